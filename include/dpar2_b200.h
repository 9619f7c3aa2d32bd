/*
 * dpar2_b200.h -- C ABI of the B200-native DPar2 hot path (libdpar2_b200.so).
 *
 * The reference (dpar2, /root/reference/pkg/src/dpar2 = "P/") is pure
 * Python/NumPy and has no FFI layer; its boundary is the Python API
 * (fit_dpar2 / compress / the per-iteration kernels, P/__init__.py:19-32).
 * This header is the native boundary underneath our Python mirror of that API
 * (paper_2203_12798_b200/), bound with ctypes (INTEGRATION.md shows the stub).
 *
 * Conventions
 *   - Every pointer named *_dev or documented "device" is device memory owned
 *     by the caller; calls are stream-ordered on ``stream`` (cudaStream_t, may
 *     be NULL for the legacy stream) and return before the GPU finishes.
 *   - Return value: a dp2_status for argument / launch errors.  Numeric
 *     failures found on the device (non-finite input, non-converged Jacobi,
 *     rank-deficient slices) are written to a caller-owned device ``status``
 *     block of DP2_STATUS_WORDS int64 (initialise with dp2_status_init) and
 *     read by the host after synchronising -- mirroring the reference's
 *     NonFiniteInputError / NumericFailure(slice_index) (P/errors.py:36-43).
 *   - Row-major everywhere.  Irregular slices live in one packed store: slice
 *     k is rows [row_off[k], row_off[k+1]) of a (total_rows x ldx) matrix.
 *   - No torch types, no global mutable state.
 */
#ifndef DPAR2_B200_H_
#define DPAR2_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DP2_ABI_VERSION 1
#define DP2_STATUS_WORDS 8

enum dp2_status {
  DP2_OK = 0,
  DP2_ERR_NONFINITE = 1, /* NonFiniteInputError       (P/linalg.py:57-58, P/tensor.py:61) */
  DP2_ERR_NOCONV = 2,    /* NumericFailure             (P/linalg.py:88-89)                 */
  DP2_ERR_SHAPE = 3,     /* RankTooLarge/ShapeMismatch (P/compress.py:84-90)               */
  DP2_ERR_CUDA = 4,      /* launch / runtime failure; see dp2_last_error()                 */
  DP2_ERR_ARG = 5        /* invalid argument (ValueError in the reference)                 */
};

enum dp2_dtype { DP2_F64 = 0, DP2_F32 = 1 };

/* Device view of a packed irregular tensor plus its work plan.  The plan
 * splits the global row space into ``nseg`` equal segments (one persistent
 * CTA each); a "piece" is the intersection of a segment with a slice.  Build
 * the host arrays with dp2_plan_pieces and copy them to the device. */
typedef struct dp2_store {
  const void* X;              /* device, total_rows x ldx, dtype; cols [J, ldx) zero  */
  int32_t dtype;              /* dp2_dtype                                            */
  int32_t nseg;               /* segments (CTAs of a streaming pass)                  */
  int64_t ldx;                /* row stride in elements, ldx*size % 16 == 0           */
  int64_t J;                  /* shared column count                                  */
  int64_t K;                  /* slice count                                          */
  int64_t total_rows;         /* sum_k I_k                                            */
  int64_t npieces;            /* pieces in the plan                                   */
  const int64_t* row_off;     /* device, K+1                                          */
  const int32_t* piece_slice; /* device, npieces                                      */
  const int64_t* piece_row0;  /* device, npieces: first global row of the piece       */
  const int32_t* piece_rows;  /* device, npieces                                      */
  const int32_t* seg_begin;   /* device, nseg+1: pieces of segment g                  */
  const int32_t* slice_piece; /* device, K+1: pieces of slice k (contiguous)          */
} dp2_store;

/* ------------------------------------------------------------------ misc */
int dp2_abi_version(void);
const char* dp2_status_string(int status);
const char* dp2_last_error(void);
int dp2_device_sm_count(void);
/* Kernels enqueued by this library so far (every launch, including the
 * kernels inside the ALS graph); reset != 0 returns the count and zeroes it. */
int64_t dp2_launch_count(int32_t reset);
/* Persistent segments (CTAs) of the stage-1 streaming passes for a store of
 * this dtype / column count on a device with `sms` SMs: one per SM for fp64
 * (DMMA) and for fp32 with J <= 512 (tcgen05 tf32 pass), two per SM for the
 * fp32 FFMA pass.  Planning aid for dp2_plan_pieces(nseg). */
int32_t dp2_stream_segments(int32_t dtype, int64_t J, int32_t sms);
/* fp32-storage streaming-pass engine: 2 = fp64 DMMA products on the exactly
 * upcast values where dp2_sketch_kind reports 3, else fp32 FFMA products
 * (default; at least the fp32 mode of BASELINE.json), 1 = fp32 FFMA products
 * everywhere, 0 = single-pass tf32 products on
 * tcgen05 tensor cores where eligible (opt-in speed mode: ~5e-4 relative
 * product error, passes the 1e-3 fp32-mode bound on c2 but not on slices of
 * ~50 rows).
 * The environment variable DP2_SKETCH_ENGINE sets the initial value.
 * Returns the previous setting. */
int32_t dp2_set_sketch_engine(int32_t engine);
/* Which streaming pass a dp2_stream_pass(st, sp, ...) call takes (xsq / gram:
 * whether the per-piece sums of squares / Y^T Y partials are requested):
 * 0 = fp64 DMMA per-tile pass, 1 = fp32 FFMA pass, 2 = tf32 tcgen05 pass,
 * 3 = warp-specialised fp64 DMMA pass (fp64, or fp32 storage with engine 2);
 * -1 on invalid arguments. */
int32_t dp2_sketch_kind(const dp2_store* st, int32_t sp, int32_t xsq, int32_t gram);
/* status block: words 0 and 2/3 <- INT64_MAX, others 0 */
int dp2_status_init(int64_t* status_dev, void* stream);
/* Stream-ordered upload of a small PINNED host buffer by a kernel reading it
 * through the UVA mapping (no copy engine: it cannot queue behind bulk
 * uploads submitted earlier on another stream).  The host buffer must stay
 * valid until the stream reaches the copy. */
int dp2_copy_h2d_small(void* dst_dev, const void* src_pinned, size_t nbytes, void* stream);

/* ------------------------------------------------------------------ host planning
 * Alg. 4 LPT partition, bit-exact with P/scheduler.py:29-51 (greedy_partition):
 * visit slices by (-count, index); each goes to the lightest set, lowest set
 * index on ties.  order_out[K] = visit order, owner_out[K] = set of slice k,
 * loads_out[workers] = row loads.  Returns DP2_ERR_ARG like the reference's
 * ValueError (P/scheduler.py:39-44). */
int dp2_greedy_partition(const int64_t* row_counts, int64_t K, int32_t workers, int64_t* order_out,
                         int32_t* owner_out, int64_t* loads_out);
/* Upper bound on pieces for (K, nseg). */
int64_t dp2_piece_capacity(int64_t K, int32_t nseg);
/* Split rows [0, row_off[K]) into nseg equal segments, cut at slice bounds.
 * Host arrays; sizes as in dp2_store.  Replaces the reference's per-thread
 * slice groups (P/compress.py:93-105) with equal-row persistent segments. */
int dp2_plan_pieces(const int64_t* row_off, int64_t K, int32_t nseg, int32_t* piece_slice,
                    int64_t* piece_row0, int32_t* piece_rows, int32_t* seg_begin,
                    int32_t* slice_piece, int64_t* npieces_out);

/* ------------------------------------------------------------------ sketch matrices
 * derived_seed(seed, index) of P/linalg.py:187-194 (numpy SeedSequence hash),
 * computed natively (host). */
uint64_t dp2_derived_seed(uint64_t seed, uint64_t index);
/* Omega_k for K slices on the device, bit-exact with the reference's
 * Generator(PCG64(derived_seed(seed, id_k))).standard_normal((J, s_k))
 * (P/linalg.py:122-123): out is K x J x sp (zero padded beyond s_k).
 * id_k = slice_ids_dev[k] (device, nullable -> k).  Layer-0 tail draws
 * (~2.6e-4 of draws) depend on libm log1p rounding: each is written to
 * ``recs`` (dp2_tail_record, capacity ``cap``, count in *nrec_dev) for the
 * host to replay with the reference's log1p and patch; redo_dev[k] != 0 asks
 * the host to regenerate slice k (record overflow).  See rng.py. */
typedef struct dp2_tail_record {
  int64_t slice, index;   /* local slice, output index (C order in J x s_k) */
  int32_t attempts;       /* accepted on attempt #attempts (<= 4)           */
  int32_t negative;       /* sign of the output                              */
  double u[8];            /* (u1, u2) uniforms of each attempt               */
} dp2_tail_record;
int dp2_omega_generate(uint64_t seed, int64_t K, int32_t J, const int32_t* s_dev, int32_t sp,
                       const int64_t* slice_ids_dev, double* out, dp2_tail_record* recs, int32_t cap,
                       int32_t* nrec_dev, int32_t* redo_dev, void* stream);
/* One stream: out (rows x width, row-major) = Generator(PCG64(seed))
 * .standard_normal((rows, width)) byte-exact -- the stage-2 sketch matrix
 * (P/compress.py:109-111, seed = derived_seed(seed, K) computed by the
 * caller).  The stream is cut into segments parsed in parallel and stitched
 * exactly; tail records as for dp2_omega_generate (slice 0).  width_dev:
 * device int32 holding width. */
int dp2_omega_generate_stream(uint64_t seed, int64_t rows, int32_t width, const int32_t* width_dev, double* out,
                              dp2_tail_record* recs, int32_t cap, int32_t* nrec_dev, int32_t* redo_dev,
                              void* stream);
/* Host-side replay of tail records (host pointers): for each record, re-run
 * its attempts with this process's libm log1p -- the function NumPy's
 * ziggurat calls (npy_log1p) -- giving the reference's output value in
 * vals[i] and ok[i] = 1, or ok[i] = 0 when the device's acceptance decision
 * differed (the slice must then be regenerated on the host). */
int dp2_omega_replay(const dp2_tail_record* recs, int64_t count, double* vals, int32_t* ok);
/* Replay (multithreaded) and patch in one call: the accepted values are
 * scattered into out_dev (K x J x sp, slice k's J x widths_host[k] block) on
 * ``stream``; records whose acceptance decision differs set redo_host[slice]
 * = 1 (the caller regenerates those slices); *patched_out = values patched. */
int dp2_omega_patch(const dp2_tail_record* recs, int64_t count, int64_t J, const int32_t* widths_host, int32_t sp,
                    double* out_dev, int32_t* redo_host, int32_t* patched_out, void* stream);

/* ------------------------------------------------------------------ tensor checks
 * Per-slice squared Frobenius norms (sqnorm_dev[K]) and the lowest slice with
 * a NaN/Inf (status[0]); mirrors IrregularTensor's isfinite check
 * (P/tensor.py:61) and total_sq_norm (P/tensor.py:79-80). */
int dp2_slice_stats(const dp2_store* st, double* sqnorm_dev, int64_t* status_dev, void* stream);
/* 1 when the streaming sketch of this store at padded width sp runs on the
 * tf32 tensor-core pass (fp32 storage, J <= 512, sp <= 32), else 0. */
int dp2_sketch_uses_tc(const dp2_store* st, int32_t sp);
/* The same isfinite check on HOST slices (ptrs[k]: rows[k] x J, row stride
 * ld[k] elements, dtype DP2_F32/DP2_F64), multithreaded (threads <= 0: all
 * hardware threads), so it runs while the upload of the same slices is in
 * flight; *first_bad = lowest non-finite slice or INT64_MAX. */
int dp2_host_first_nonfinite(const void* const* ptrs, const int64_t* rows, const int64_t* ld, int64_t K, int64_t J,
                             int32_t dtype, int32_t threads, int64_t* first_bad);

/* ------------------------------------------------------------------ stage 1
 * Per-slice randomized SVD (P/linalg.py:97-132 with power_iters = 1, as called
 * from P/compress.py:96-105), two streaming passes over X:
 *   pass 1: Z_k = X_k^T (X_k Omega_k)         -> Q_Z = orth(Z_k)
 *   pass 2: Y_k = X_k Q_Z, C_k = Y_k^T X_k    -> range(Y_k) = range of the
 *           reference's X (X^T X Omega) sketch; B_k = Q^T X_k via G = Y^T Y.
 * Outputs: A_out (total_rows x rank) = U of each slice with the sign rule of
 * P/linalg.py:62-70; M_out (J x K*rank, row-major) = [V_k S_k] in slice order
 * (P/compress.py:108); rank_out[K] = numerical rank found (>= rank unless the
 * slice is rank deficient, where A is completed orthonormally).
 * omega_dev: K x J x sp (slice k's J x s_k Gaussian in the first s_k columns,
 * zero padded; P/linalg.py:122-123).  s_dev[K] = per-slice sketch width.
 * timing_ms (host, nullable, >= 8 floats): per-phase CUDA-event times
 * [sketch1, orth, sketch2, factor, signs+A, total]; forces a sync. */
size_t dp2_stage1_workspace(const dp2_store* st, int32_t sp, int32_t rank);
int dp2_stage1(const dp2_store* st, const double* omega_dev, const int32_t* s_dev, int32_t sp,
               int32_t rank, double* A_out, double* M_out, int32_t* rank_out, void* ws,
               size_t ws_bytes, int64_t* status_dev, float* timing_ms, void* stream);
/* dp2_stage1 with the column signs of A (P/linalg.py:42-49 sign rule)
 * deferred: A_out holds A_k up to column signs and a_signs_out (K x rank)
 * the signs, A_k(reference) = A_out_k diag(a_signs_out[k]) exactly (+1 for
 * completed columns of rank-deficient slices).  M_out is identical to
 * dp2_stage1's.  Saves the sign pass over A when the consumer can fold the
 * signs (dp2_assemble_q_signed). */
int dp2_stage1_signs(const dp2_store* st, const double* omega_dev, const int32_t* s_dev, int32_t sp,
                     int32_t rank, double* A_out, double* M_out, int32_t* rank_out, double* a_signs_out,
                     void* ws, size_t ws_bytes, int64_t* status_dev, float* timing_ms, void* stream);

/* dp2_stage1 / dp2_stage1_signs (a_signs_out nullable) with ``power_iters``
 * power iterations (RsvdParams.power_iters, P/linalg.py:124-126): q sketch
 * passes Z = X^T (X B) each followed by B <- orth(Z), then the final pass on B
 * (q = 0: on Omega itself).  dp2_stage1 is q = 1. */
int dp2_stage1_power(const dp2_store* st, const double* omega_dev, const int32_t* s_dev, int32_t sp, int32_t rank,
                     int32_t power_iters, double* A_out, double* M_out, int32_t* rank_out, double* a_signs_out,
                     void* ws, size_t ws_bytes, int64_t* status_dev, float* timing_ms, void* stream);

/* One streaming pass of stage 1 (the two sketch products of
 * P/linalg.py:124-127 fused per piece): for every piece p (segment x slice)
 *   out_part[p] (J x sp)  = X_p^T (X_p B_k),  B = b_dev[k] (K x J x sp, fp64)
 * and, when non-null: y_out (total_rows x sp) = X_k B_k rows, g_part[p]
 * (sp x sp) = Y_p^T Y_p, xsq_part[p] = sum of squares of X_p (non-finite
 * values set status word 0).  Pieces follow dp2_plan_pieces for st->nseg.
 * fp32 stores use the tcgen05 tf32 pass when eligible (dp2_set_sketch_engine). */
int dp2_stream_pass(const dp2_store* st, const double* b_dev, int32_t sp, double* out_part, double* y_out,
                    double* g_part, double* xsq_part, int64_t* status_dev, void* stream);

/* ------------------------------------------------------------------ stage 2
 * Randomized SVD of M (J x KR) (P/compress.py:109-111): D (J x rank), E (rank),
 * F (KR x rank), sign rule on D.  omega2_dev: KR x s2 (P/linalg.py:122-123
 * seeded with derived_seed(seed, K)). */
size_t dp2_stage2_workspace(int64_t J, int64_t KR, int32_t s2, int32_t rank);
/* dp2_stage2 with Y2 = (M M^T)^q M Omega2 (power_iters = q; dp2_stage2 is q = 1). */
int dp2_stage2_power(const double* M_dev, int64_t J, int64_t KR, const double* omega2_dev, int32_t s2,
                     int32_t rank, int32_t power_iters, double* D_out, double* E_out, double* F_out, void* ws,
                     size_t ws_bytes, int64_t* status_dev, void* stream);
int dp2_stage2(const double* M_dev, int64_t J, int64_t KR, const double* omega2_dev, int32_t s2,
               int32_t rank, double* D_out, double* E_out, double* F_out, void* ws, size_t ws_bytes,
               int64_t* status_dev, void* stream);

/* ------------------------------------------------------------------ ALS
 * Compressed-space iterations (P/solver.py:152-190).  Inputs D (J x R), E (R),
 * F (K*R x R); state H (R x R), V (J x R), W (K x R) in/out.  Runs up to
 * max_iters iterations with the reference's stop rule on the device
 * (``prev == 0 || |prev - e| <= tol * prev``, P/solver.py:180-184); writes the
 * objective trace, globaltimer stamps (ns, max_iters+1) and the executed
 * iteration count; polar_out (K x R x R) holds Z_k P_k^T of the last executed
 * iteration.  use_graph != 0 captures the loop in a CUDA graph (multi-kernel
 * path only).  For R <= 16 the loop is one cooperative launch; with the
 * environment variable DP2_ALS_STAMPS set it also records 16 globaltimer
 * slots per iteration (first 64 iterations) at byte offset
 * dp2_als_stamp_offset(K, J, R) of the workspace (profiling aid). */
size_t dp2_als_workspace(int64_t K, int64_t J, int32_t R);
size_t dp2_als_stamp_offset(int64_t K, int64_t J, int32_t R);
int dp2_als_run(const double* F, const double* D, const double* E, int64_t K, int64_t J, int32_t R,
                double* H, double* V, double* W, double* polar_out, int32_t max_iters, double tol,
                int32_t normalize, double* trace_out, int64_t* tstamp_out, int32_t* iters_out,
                int32_t use_graph, void* ws, size_t ws_bytes, int64_t* status_dev, void* stream);

/* The same iteration split at its reduction points for multi-GPU runs
 * (DESIGN.md §7): phase 0 prep; 1 rotate -> red_out[2R^2] = [G1 | W^T W]
 * partials; 2 solve_h(red_in = allreduced [G1 | W^T W]); 3 mode2 -> red_out =
 * [summed | gram(W nh)]; 4 solve_v(red_in); 5 mode3 + metric -> red_out[0] =
 * local e; 6 finish(red_in[0] = global e: trace, stop rule).  K, F, W, polar
 * are the caller's local slices; D, E, H, V replicated.  The workspace
 * (dp2_als_workspace(K, J, R)) carries state between phases. */
int dp2_als_phase(int32_t phase, const double* F, const double* D, const double* E, int64_t K, int64_t J,
                  int32_t R, double* H, double* V, double* W, double* polar, int32_t it, double tol,
                  int32_t normalize, double* trace_out, int64_t* tstamp_out, int32_t* iters_out,
                  const double* red_in, double* red_out, void* ws, size_t ws_bytes, int64_t* status_dev,
                  void* stream);

/* Kernel-granular entry points (the reference's test-level API,
 * P/solver.py:48-149).  theta (K x R x R) = (P_k Z_k^T) F_k. */
int dp2_update_rotations(const double* F, const double* D, const double* E, int64_t K, int64_t J,
                         int32_t R, const double* H, const double* V, const double* W,
                         double* polar_out, double* theta_out, void* ws, size_t ws_bytes,
                         int64_t* status_dev, void* stream);
/* mode 1: out R x R (P/solver.py:81-89); mode 2: out J x R (:92-100);
 * mode 3: out K x R (:103-111). */
int dp2_mttkrp(int32_t mode, const double* theta, const double* D, const double* E, int64_t K,
               int64_t J, int32_t R, const double* H, const double* V, const double* W, double* out,
               void* ws, size_t ws_bytes, void* stream);
/* One Gauss-Seidel sweep (P/solver.py:114-130); H, V, W updated in place. */
int dp2_update_factors(const double* theta, const double* D, const double* E, int64_t K, int64_t J,
                       int32_t R, double* H, double* V, double* W, int32_t normalize, void* ws,
                       size_t ws_bytes, int64_t* status_dev, void* stream);
/* e = sum_k ||Theta_k E D^T - (H * w_k) V^T||_F^2 (P/solver.py:133-149);
 * out: one device double. */
int dp2_convergence_metric(const double* theta, const double* D, const double* E, int64_t K,
                           int64_t J, int32_t R, const double* H, const double* V, const double* W,
                           double* out, void* ws, size_t ws_bytes, void* stream);

/* Device -> pageable host copy at link speed (the NumPy readback of Q,
 * P/solver.py:186-189 returns host arrays): chunks through a persistent
 * pinned staging ring, copied out by a persistent host thread team while the
 * next chunks are in flight.  Returns after the data is in dst_host. */
int dp2_d2h_staged(void* dst_host, const void* src_dev, size_t nbytes, void* stream);

/* ------------------------------------------------------------------ outputs
 * Q_k = A_k (Z_k P_k^T) for every slice (P/solver.py:186-189). */
int dp2_assemble_q(const dp2_store* st, const double* A, int32_t R, const double* polar,
                   double* Q_out, void* stream);
/* dp2_assemble_q for an A from dp2_stage1_signs: Q_k = A_k diag(a_signs[k]) Pi_k
 * (bit-identical to dp2_assemble_q on the signed A). */
int dp2_assemble_q_signed(const dp2_store* st, const double* A, int32_t R, const double* a_signs,
                          const double* polar, double* Q_out, void* stream);
/* fitness terms (P/analysis.py:23-45): out2_dev[0] = sum ||X_k||^2,
 * out2_dev[1] = sum ||X_k - Q_k (H * w_k) V^T||^2, fixed-order reductions. */
size_t dp2_fitness_workspace(const dp2_store* st);
int dp2_fitness(const dp2_store* st, const double* Q, int32_t R, const double* H, const double* V,
                const double* W, double* out2_dev, void* ws, size_t ws_bytes, void* stream);

/* out (K x n) = A^T B for row-major A (m x K) and B (m x n), fp64 on the DMMA
 * pipe (the tall-skinny product of stage 2): the fit's M^T V for the
 * zero-pass fitness. */
int dp2_gemm_tn(const double* A, int64_t m, int64_t K, const double* B, int32_t n, double* out, void* stream);
/* Zero-pass fitness terms (P/analysis.py:23-45 restated): for
 * factors fresh from a fit on an fp64 tensor, with G_k = H diag(w_k),
 * B_k = V^T M_k (MtV = M^T V, K R x R) and the polar factors Pi_k,
 *   ||X_k - Q_k G_k V^T||^2 = ||X_k||^2 - 2 tr(Pi_k G_k B_k) + ||G_k V^T||^2;
 * out2_dev = [sum_k ||X_k||^2, sum_k residual_k], slice-order reductions.
 * sqnorm: per-slice ||X_k||^2 (dp2_slice_stats). */
size_t dp2_zero_pass_workspace(int64_t K, int32_t R);
int dp2_fitness_zero_pass(const double* MtV, int64_t K, int64_t J, int32_t R, const double* H, const double* V,
                          const double* W, const double* polar, const double* sqnorm, double* out2_dev, void* ws,
                          size_t ws_bytes, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* DPAR2_B200_H_ */
