// Stage-1 streaming sketch pass for fp32 slice storage (fp32 mode), FFMA.
//
// Same contract as the fp64 DMMA pass in dp2_stage1.cu (per persistent
// segment: walk the pieces tile by tile, Y_t = X_t B, Z += X_t^T Y_t, one
// partial per piece), computed in fp32 with register blocking:
//   phase A  Y_t (TM x SG) = X_t B: warps split J, lane tile 8 rows x CPL cols,
//            float4 X loads (4 j per load) + scalar B loads: 0.21 LDS per FMA
//   phase B  Z (J x SG) += X_t^T Y_t: thread owns JT consecutive j (float2/4 X
//            loads) x all SG columns, Y broadcast as float4: 0.15 LDS per FMA
// The X tile ring is fed by cp.async (2 stages); B (Omega or Q_Z, converted to
// fp32) sits in shared memory per piece.  Accumulation is fp32 within a piece
// (the fp32-mode accuracy budget, BASELINE.json: 1e-3; measured ~1e-6 on the
// stage-1 bases), partials are written in fp64.
#include "dp2_common.cuh"
#include "dp2_internal.h"

namespace dp2 {

struct Sketch32Params {
  const float* X;
  int64_t ldx;
  int J, sp, lds, njs;
  const double* B;
  const int32_t* piece_slice;
  const int64_t* piece_row0;
  const int32_t* piece_rows;
  const int32_t* seg_begin;
  double* out_part;
  double* y_out;
  double* xsq_part;
  double* g_part;
  int64_t* status;
};

template <int TM, int CPL, int JT>
__global__ void __launch_bounds__(256, 1) sketch32_kernel(Sketch32Params prm) {
  constexpr int SG = 8 * CPL, NW = 8, RPL = TM / 4;  // rows per lane in phase A
  extern __shared__ __align__(16) unsigned char smem[];
  const int LDS = prm.lds, J = prm.J, sp = prm.sp;
  const int J4 = (J + 3) / 4;
  float* xs = reinterpret_cast<float*>(smem);                 // [2][TM][LDS]
  float* bs = xs + 2 * TM * LDS;                               // [J4*4][SG]
  float* ypart = bs + J4 * 4 * SG;                             // [NW][TM][SG]
  float* ys = ypart + NW * TM * SG;                            // [TM][SG]
  __shared__ double red[32];

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int seg = blockIdx.x, col0 = blockIdx.y * SG, jsplit = blockIdx.z;
  const int jbase = jsplit * 256 * JT;
  const bool stats = (blockIdx.y == 0) && prm.xsq_part != nullptr;
  const int cpr = (J * 4 + 15) / 16;
  const int loaded_cols = cpr * 4;
  for (int i = tid; i < 2 * TM * LDS; i += blockDim.x)
    if (i % LDS >= loaded_cols) xs[i] = 0.0f;

  const int pbeg = prm.seg_begin[seg], pend = prm.seg_begin[seg + 1];
  if (pbeg >= pend) return;
  const char* Xb = reinterpret_cast<const char*>(prm.X);

  auto issue = [&](int buf, int p, int t) {
    const int64_t row0 = prm.piece_row0[p] + (int64_t)t * TM;
    const int rows = min(TM, prm.piece_rows[p] - t * TM);
    char* dst = reinterpret_cast<char*>(xs + (size_t)buf * TM * LDS);
    for (int i = tid; i < TM * cpr; i += blockDim.x) {
      const int r = i / cpr, c = i % cpr;
      const bool ok = r < rows;
      const char* src = ok ? Xb + ((row0 + r) * prm.ldx) * 4 + (int64_t)c * 16 : Xb;
      cp_async16(dst + (size_t)r * LDS * 4 + (size_t)c * 16, src, ok ? 16 : 0);
    }
  };

  // phase-A lane tile: rows (lane & 3) + 4 r, cols (lane >> 2) * CPL + c
  const int ra = lane & 3, cb = (lane >> 2) * CPL;
  // phase-A split of J over warps (multiples of 4)
  const int jw = ((J4 + NW - 1) / NW) * 4;
  const int ja0 = warp * jw, ja1 = min(J4 * 4, ja0 + jw);

  float zacc[JT][SG];
#pragma unroll
  for (int a = 0; a < JT; ++a)
#pragma unroll
    for (int c = 0; c < SG; ++c) zacc[a][c] = 0.0f;
  double sq = 0.0;
  int bad = 0;
  constexpr int GPT = (SG * SG + 255) / 256;
  double gacc[GPT];
#pragma unroll
  for (int q = 0; q < GPT; ++q) gacc[q] = 0.0;
  const bool do_g = prm.g_part != nullptr && jsplit == 0;
  int p = pbeg, t = 0, buf = 0, bslice = -1;
  issue(0, p, 0);
  cp_async_commit();

  while (true) {
    int np = p, ntl = t + 1;
    if (ntl * TM >= prm.piece_rows[p]) { np = p + 1; ntl = 0; }
    const bool has_next = np < pend;
    if (has_next) issue(buf ^ 1, np, ntl);
    cp_async_commit();
    const int ks = prm.piece_slice[p];
    if (ks != bslice) {  // B of this slice -> fp32 smem (rows >= J zero)
      const double* Bm = prm.B + (size_t)ks * J * sp + col0;
      for (int i = tid; i < J4 * 4 * SG; i += blockDim.x) {
        const int j = i / SG, c = i % SG;
        bs[i] = j < J ? (float)Bm[(size_t)j * sp + c] : 0.0f;
      }
      bslice = ks;
    }
    cp_async_wait<1>();
    __syncthreads();
    const float* X = xs + (size_t)buf * TM * LDS;

    // ---- phase A
    float ya[RPL][CPL];
#pragma unroll
    for (int r = 0; r < RPL; ++r)
#pragma unroll
      for (int c = 0; c < CPL; ++c) ya[r][c] = 0.0f;
    for (int j = ja0; j < ja1; j += 4) {
      float4 xv[RPL];
#pragma unroll
      for (int r = 0; r < RPL; ++r) xv[r] = *reinterpret_cast<const float4*>(X + (ra + 4 * r) * LDS + j);
#pragma unroll
      for (int jj = 0; jj < 4; ++jj) {
        float bv[CPL];
#pragma unroll
        for (int c = 0; c < CPL; ++c) bv[c] = bs[(j + jj) * SG + cb + c];
#pragma unroll
        for (int r = 0; r < RPL; ++r) {
          const float x = jj == 0 ? xv[r].x : jj == 1 ? xv[r].y : jj == 2 ? xv[r].z : xv[r].w;
#pragma unroll
          for (int c = 0; c < CPL; ++c) ya[r][c] = fmaf(x, bv[c], ya[r][c]);
        }
      }
    }
#pragma unroll
    for (int r = 0; r < RPL; ++r)
#pragma unroll
      for (int c = 0; c < CPL; ++c) ypart[(warp * TM + ra + 4 * r) * SG + cb + c] = ya[r][c];
    __syncthreads();
    for (int i = tid; i < TM * SG; i += blockDim.x) {
      float s = 0.0f;
#pragma unroll
      for (int w = 0; w < NW; ++w) s += ypart[w * TM * SG + i];
      ys[i] = s;
    }
    __syncthreads();
    const int rows = min(TM, prm.piece_rows[p] - t * TM);
    if (prm.y_out != nullptr && jsplit == 0) {
      const int64_t grow = prm.piece_row0[p] + (int64_t)t * TM;
      for (int i = tid; i < rows * SG; i += blockDim.x) {
        const int r = i / SG, c = i % SG;
        prm.y_out[(grow + r) * sp + col0 + c] = (double)ys[i];
      }
    }
    if (do_g) {  // G += Y_t^T Y_t in fp64 (rows past the piece are zero)
#pragma unroll
      for (int q = 0; q < GPT; ++q) {
        const int e = tid + q * 256;
        if (e < SG * SG) {
          const int a = e / SG, b = e % SG;
          double acc = gacc[q];
          for (int r = 0; r < TM; ++r) acc = fma((double)ys[r * SG + a], (double)ys[r * SG + b], acc);
          gacc[q] = acc;
        }
      }
    }

    // ---- phase B: thread owns j = jbase + tid*JT + a
    const int j0 = jbase + tid * JT;
    if (j0 < J) {
      for (int r = 0; r < TM; ++r) {
        float xv[JT];
        if constexpr (JT == 4) {
          const float4 v = *reinterpret_cast<const float4*>(X + r * LDS + j0);
          xv[0] = v.x; xv[1] = v.y; xv[2] = v.z; xv[3] = v.w;
        } else if constexpr (JT == 2) {
          const float2 v = *reinterpret_cast<const float2*>(X + r * LDS + j0);
          xv[0] = v.x; xv[1] = v.y;
        } else {
          xv[0] = X[r * LDS + j0];
        }
        if (stats) {
#pragma unroll
          for (int a = 0; a < JT; ++a)
            if (j0 + a < J) {
              const double d = (double)xv[a];
              sq = fma(d, d, sq);
              bad |= !isfinite(xv[a]);
            }
        }
        const float4* y4 = reinterpret_cast<const float4*>(ys + r * SG);
#pragma unroll
        for (int c4 = 0; c4 < SG / 4; ++c4) {
          const float4 y = y4[c4];
#pragma unroll
          for (int a = 0; a < JT; ++a) {
            zacc[a][4 * c4 + 0] = fmaf(xv[a], y.x, zacc[a][4 * c4 + 0]);
            zacc[a][4 * c4 + 1] = fmaf(xv[a], y.y, zacc[a][4 * c4 + 1]);
            zacc[a][4 * c4 + 2] = fmaf(xv[a], y.z, zacc[a][4 * c4 + 2]);
            zacc[a][4 * c4 + 3] = fmaf(xv[a], y.w, zacc[a][4 * c4 + 3]);
          }
        }
      }
    }

    if ((t + 1) * TM >= prm.piece_rows[p]) {  // piece complete: flush partial
      if (do_g) {
#pragma unroll
        for (int q = 0; q < GPT; ++q) {
          const int e = tid + q * 256;
          if (e < SG * SG) prm.g_part[(size_t)p * SG * SG + e] = gacc[q];
          gacc[q] = 0.0;
        }
      }
      double* out = prm.out_part + (size_t)p * J * sp + col0;
#pragma unroll
      for (int a = 0; a < JT; ++a) {
        const int j = j0 + a;
        if (j < J && j < jbase + 256 * JT)
#pragma unroll
          for (int c = 0; c < SG; ++c) out[(size_t)j * sp + c] = (double)zacc[a][c];
#pragma unroll
        for (int c = 0; c < SG; ++c) zacc[a][c] = 0.0f;
      }
      if (stats) {
        const double tot = block_sum(sq, red);
        if (tid == 0) prm.xsq_part[(size_t)p * prm.njs + jsplit] = tot;
        sq = 0.0;
        if (__syncthreads_or(bad) && tid == 0) status_min(prm.status, ST_NONFINITE, ks);
        bad = 0;
      }
    }
    __syncthreads();
    if (!has_next) break;
    p = np;
    t = ntl;
    buf ^= 1;
  }
}

namespace {
template <int TM, int CPL, int JT>
cudaError_t launch32(const Sketch32Params& prm, int nseg, int ng, int njs, cudaStream_t st) {
  constexpr int SG = 8 * CPL;
  const int J4 = (prm.J + 3) / 4;
  const size_t smem = ((size_t)2 * TM * prm.lds + (size_t)J4 * 4 * SG + 8 * TM * SG + TM * SG) * 4;
  if (smem > 227 * 1024) return cudaErrorInvalidValue;
  auto kern = sketch32_kernel<TM, CPL, JT>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  kern<<<dim3(nseg, ng, njs), 256, smem, st>>>(prm);
  return cudaGetLastError();
}
template <int TM, int CPL>
cudaError_t by_jt(const Sketch32Params& prm, int jt, int nseg, int ng, int njs, cudaStream_t st) {
  switch (jt) {
    case 1: return launch32<TM, CPL, 1>(prm, nseg, ng, njs, st);
    case 2: return launch32<TM, CPL, 2>(prm, nseg, ng, njs, st);
    default: return launch32<TM, CPL, 4>(prm, nseg, ng, njs, st);
  }
}
template <int TM>
cudaError_t by_cpl(const Sketch32Params& prm, int cpl, int jt, int nseg, int ng, int njs, cudaStream_t st) {
  switch (cpl) {
    case 1: return by_jt<TM, 1>(prm, jt, nseg, ng, njs, st);
    case 2: return by_jt<TM, 2>(prm, jt, nseg, ng, njs, st);
    case 3: return by_jt<TM, 3>(prm, jt, nseg, ng, njs, st);
    default: return by_jt<TM, 4>(prm, jt, nseg, ng, njs, st);
  }
}
int lds32(int J) {
  int lds = ((J + 3) / 4) * 4;
  while (lds % 8 != 4) lds += 4;  // LDS/4 odd: 4 consecutive rows hit distinct 16B bank groups
  return lds;
}
}  // namespace

int sketch32_njs(int J) { return (J + 1023) / 1024; }

cudaError_t run_sketch_f32(const dp2_store* st, const double* B, int sp, double* out_part, double* y_out,
                           double* xsq_part, int64_t* status, cudaStream_t stream, double* g_part) {
  if (sketch_tc_eligible(st, sp)) return run_sketch_tc(st, B, sp, out_part, y_out, xsq_part, status, stream, g_part);
  if (sketch_engine() == 2 && sketch64_eligible(st, sp, xsq_part != nullptr, g_part != nullptr))
    return run_sketch64(st, B, sp, out_part, y_out, status, stream, g_part);  // fp64 products on upcast X
  const int J = (int)st->J;
  Sketch32Params prm{};
  prm.X = static_cast<const float*>(st->X);
  prm.ldx = st->ldx;
  prm.J = J;
  prm.sp = sp;
  prm.lds = lds32(J);
  prm.B = B;
  prm.piece_slice = st->piece_slice;
  prm.piece_row0 = st->piece_row0;
  prm.piece_rows = st->piece_rows;
  prm.seg_begin = st->seg_begin;
  prm.out_part = out_part;
  prm.y_out = y_out;
  prm.xsq_part = xsq_part;
  prm.g_part = sp <= 32 ? g_part : nullptr;
  prm.status = status;
  const int cpl = sp >= 32 ? 4 : sp / 8;
  const int ng = sp >= 32 ? sp / 32 : 1;
  const int jt = J <= 256 ? 1 : (J <= 512 ? 2 : 4);
  const int njs = sketch32_njs(J);
  prm.njs = njs;
  const int sg = 8 * cpl;
  const size_t need32 = ((size_t)2 * 32 * prm.lds + (size_t)((J + 3) / 4) * 4 * sg + 9 * 32 * sg) * 4;
  const size_t need16 = ((size_t)2 * 16 * prm.lds + (size_t)((J + 3) / 4) * 4 * sg + 9 * 16 * sg) * 4;
  const size_t need8 = ((size_t)2 * 8 * prm.lds + (size_t)((J + 3) / 4) * 4 * sg + 9 * 8 * sg) * 4;
  if (need32 <= 220 * 1024) return by_cpl<32>(prm, cpl, jt, st->nseg, ng, njs, stream);
  if (need16 <= 220 * 1024) return by_cpl<16>(prm, cpl, jt, st->nseg, ng, njs, stream);
  if (need8 <= 220 * 1024) return by_cpl<8>(prm, cpl, jt, st->nseg, ng, njs, stream);  // J ~ 1000
  // the B image no longer fits: the generic pass (B from L2), fp64 products
  return run_sketch_generic(st, B, sp, out_part, y_out, xsq_part, status, stream, g_part);
}

}  // namespace dp2
