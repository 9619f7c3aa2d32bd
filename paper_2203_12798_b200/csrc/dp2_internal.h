// Host-side declarations shared between the .cu translation units.
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include "../../include/dpar2_b200.h"

namespace dp2 {

// detail appended to the next dp2_last_error() message
void note_error(const char* what);

struct Stage1Layout {
  size_t part, qz, y2, Pm, Sv, Vt, cand_abs, cand_row, cand_neg, xsq, scr, gpart, CCg, Gg, sgn, total;
};
Stage1Layout stage1_layout(const dp2_store* st, int sp, int R);
cudaError_t run_stage1(const dp2_store* st, const double* omega, const int32_t* s_dev, int sp, int R,
                       double* A_out, double* M_out, int32_t* rank_out, char* ws, int64_t* status,
                       float* timing, cudaStream_t stream, double* a_signs = nullptr, int power_iters = 1);
cudaError_t run_stage1_small(const dp2_store* st, const int32_t* s_dev, int sp, int R, const double* part1,
                             const double* part2, const double* gpart, double* qz, double* Ct, double* CCg,
                             double* Gg, const double* y2, double* Pm, double* Sv, double* sgn, double* cand_abs,
                             int64_t* cand_row, int32_t* cand_neg, double* A, double* M, int32_t* rank_out,
                             int64_t* status, int phase, cudaStream_t stream, bool y32, double* gscratch,
                             double* a_signs);
cudaError_t run_sketch_f32(const dp2_store* st, const double* B, int sp, double* out_part, double* y_out,
                           double* xsq_part, int64_t* status, cudaStream_t stream, double* g_part);
bool sketch_tc_eligible(const dp2_store* st, int sp);
cudaError_t run_sketch_tc(const dp2_store* st, const double* B, int sp, double* out_part, double* y_out,
                          double* xsq_part, int64_t* status, cudaStream_t stream, double* g_part, bool y32 = false);
// fp64 DMMA warp-specialised pass (dp2_sketch64.cu): fp64 or fp32 (upcast) storage
bool sketch64_eligible(const dp2_store* st, int sp, bool xsq, bool gram);
cudaError_t run_sketch_generic(const dp2_store* st, const double* B, int sp, double* out_part, double* y_out,
                               double* xsq_part, int64_t* status, cudaStream_t stream, double* g_part);
bool sketch64_pairs(int64_t J);  // the DMMA pass runs as CTA pairs (one segment per pair)
cudaError_t run_sketch64(const dp2_store* st, const double* B, int sp, double* out_part, double* y_out,
                         int64_t* status, cudaStream_t stream, double* g_part);
void set_sketch_engine(int e);
int sketch_engine();
cudaError_t run_sketch(const dp2_store* st, const double* B, int sp, double* out_part, double* y_out,
                       double* xsq_part, int64_t* status, cudaStream_t stream, double* g_part = nullptr);

size_t stage2_bytes(int64_t J, int64_t KR, int s2, int R);
cudaError_t run_stage2(const double* M, int64_t J, int64_t KR, const double* omega2, int s2, int R,
                       double* D, double* E, double* F, char* ws, int64_t* status, cudaStream_t stream,
                       int power_iters = 1);

size_t als_bytes(int64_t K, int64_t J, int R);
size_t als_stamp_offset(int64_t K, int64_t J, int R);
struct AlsCtx;  // defined in dp2_als.cu
cudaError_t als_run(const double* F, const double* D, const double* E, int64_t K, int64_t J, int R,
                    double* H, double* V, double* W, double* polar, int max_iters, double tol,
                    int normalize, double* trace, int64_t* tstamp, int32_t* iters, int use_graph,
                    char* ws, int64_t* status, cudaStream_t stream, int64_t* launches = nullptr);
cudaError_t als_phase(int phase, const double* F, const double* D, const double* E, int64_t K, int64_t J, int R,
                      double* H, double* V, double* W, double* polar, int it, double tol, int normalize,
                      double* trace, int64_t* tstamp, int32_t* iters, const double* red_in, double* red_out,
                      char* ws, int64_t* status, cudaStream_t st);
cudaError_t als_rotations(const double* F, const double* D, const double* E, int64_t K, int64_t J, int R,
                          const double* H, const double* V, const double* W, double* polar,
                          double* theta, char* ws, int64_t* status, cudaStream_t stream);
cudaError_t als_mttkrp(int mode, const double* theta, const double* D, const double* E, int64_t K,
                       int64_t J, int R, const double* H, const double* V, const double* W, double* out,
                       char* ws, cudaStream_t stream);
cudaError_t als_update_factors(const double* theta, const double* D, const double* E, int64_t K,
                               int64_t J, int R, double* H, double* V, double* W, int normalize,
                               char* ws, int64_t* status, cudaStream_t stream);
cudaError_t als_metric(const double* theta, const double* D, const double* E, int64_t K, int64_t J,
                       int R, const double* H, const double* V, const double* W, double* out, char* ws,
                       cudaStream_t stream);

cudaError_t run_assemble_q(const dp2_store* st, const double* A, int R, const double* polar, double* Q,
                           cudaStream_t stream, const double* a_signs);
size_t fitness_bytes(const dp2_store* st);
cudaError_t run_fitness(const dp2_store* st, const double* Q, int R, const double* H, const double* V,
                        const double* W, double* out2, char* ws, cudaStream_t stream);
int gemm_tn_splits(int64_t m, int64_t K, int n);
cudaError_t run_gemm_tn(const double* A, int64_t m, int64_t K, const double* B, int n, double* out,
                        cudaStream_t st, double* parts = nullptr);
int gemm_nn_splits(int64_t m, int64_t K, int n);
cudaError_t run_gemm_nn(const double* A, int64_t m, int64_t K, const double* B, int n, double* out, cudaStream_t st,
                        double* parts = nullptr);
size_t zero_pass_bytes(int64_t K, int R);
cudaError_t run_zero_pass_fitness(const double* MtV, int64_t K, int64_t J, int R, const double* H, const double* V,
                                  const double* W, const double* polar, const double* sq, double* out2, char* ws,
                                  cudaStream_t st);
cudaError_t run_slice_stats(const dp2_store* st, double* sqnorm, int64_t* status, cudaStream_t stream);

cudaError_t run_omega(uint64_t seed, int64_t K, int J, const int32_t* s_k, int sp, const int64_t* slice_ids,
                      double* out, void* recs, int cap, int32_t* nrec, int32_t* redo, cudaStream_t st, int* launches = nullptr,
                      bool raw = false);
size_t tail_record_bytes();
cudaError_t d2h_staged(void* dst, const void* src, size_t n, cudaStream_t st);
uint64_t derived_seed_host(uint64_t seed, uint64_t index);

// shared small kernels (stage 1 / stage 2)
__global__ void cgs2_cols_kernel(double* Q, int64_t rows, int ncols, double* scr);

}  // namespace dp2
