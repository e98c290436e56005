// Internal launcher declarations shared by the libsvb translation units.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/svb.h"

namespace svb {

// gates_basic.cu — one HBM pass per gate
template <typename R> void launch_gate_basic(void* state, int n, const svb_gate& g, cudaStream_t st);
template <typename R> void launch_zero(void* state, int n, cudaStream_t st);

// measure.cu — reductions over the state
template <typename R>
void launch_marginal(const void* state, int n, const int32_t* qubits, int k, double* d_out,
                     double* d_ws, size_t ws_doubles, cudaStream_t st);
size_t marginal_ws_doubles(int n, int k);
template <typename R>
void launch_expect_z(const void* state, int n, const uint64_t* h_masks, int m, double* d_out,
                     double* d_ws, cudaStream_t st);
size_t expect_ws_doubles(int n, int m);
// out[r] = sum_c partial[r * cols + c]
void launch_sum_rows(const double* d_partial, uint64_t rows, uint64_t cols, double* d_out, cudaStream_t st);
// Measure/reset qubit q with the device PCG64 stream d_rng; outcome recorded in
// d_out[0] (int32) and, when d_codes != nullptr, OR-ed into d_codes[0] << rank.
template <typename R>
void launch_measure(void* state, int n, int q, bool reset, uint64_t* d_rng, double* d_ws,
                    int32_t* d_outcome, uint64_t* d_code, int rank, cudaStream_t st);
size_t measure_ws_doubles(int n);
template <typename R> void launch_half_copy(void* state, int n, void* buf, int L, int bit, int to_buf, cudaStream_t st);
// a, b: 2^n amplitudes; out (device, 5 doubles) = {sum|a-b|^2, sum|a|^2, sum|b|^2, Re<a|b>, Im<a|b>}
template <typename RA, typename RB>
void launch_compare(const void* a, const void* b, int n, double* d_ws, double* d_out, cudaStream_t st);
size_t compare_ws_doubles(int n);
struct BlockSel {
  int g;          // local bits selecting the block
  int L[8];       // their positions, ascending
  uint64_t bits;  // the block's value deposited at those positions
};
template <typename R>
void launch_block_copy(void* state, void* buf, const BlockSel& sel, uint64_t off, uint64_t count, int to_buf,
                       cudaStream_t st);
template <typename R> void launch_outer(void* dst, const void* a, const void* b, int na, int nb, cudaStream_t st);

// dense.cu — one dense 2^k x 2^k block per HBM pass (mat: row-major complex128)
bool dense_tc_supported(int precision, int n, int k);
bool dense_fma_supported(int precision, int n, int k);
void launch_dense_tc(void* state, int n, const int32_t* q, int k, const double* mat, cudaStream_t st);
template <typename R>
void launch_dense_fma(void* state, int n, const int32_t* q, int k, const double* mat, cudaStream_t st);

// sample.cu — PCG64, pairwise sum, alias table, samplers, histogram
void host_pcg_advance(uint64_t* pcg4, uint64_t delta);
double pairwise_sum_device(const double* d_x, uint64_t m, double* d_ws, cudaStream_t st);
struct SampleOut {
  uint64_t* codes;
  uint64_t* counts;
  uint64_t n_unique;
};
void alias_build(double* d_probs, uint64_t m, double* d_prob_row, int64_t* d_alias_row,
                 cudaStream_t st);
void alias_draw(const double* d_prob_row, const int64_t* d_alias_row, uint64_t m, uint64_t shots,
                const uint64_t* pcg, const int32_t* bit_src, int w, uint64_t* d_codes,
                cudaStream_t st);
template <typename R>
void cdf_draw(const void* state, int n, uint64_t shots, const uint64_t* pcg, const int32_t* bit_src,
              int w, uint64_t* d_codes, cudaStream_t st);
// scratch: >= cdf_scratch_doubles(n) doubles of device memory (else per-call pool buffers)
template <typename R>
void cdf_draw_scratch(const void* state, int n, uint64_t shots, const uint64_t* pcg, const int32_t* bit_src,
                      int w, uint64_t* d_codes, cudaStream_t st, double* scratch);
uint64_t cdf_scratch_doubles(int n);
void cdf_draw_probs(const double* d_probs, uint64_t m, uint64_t shots, const uint64_t* pcg,
                    const int32_t* bit_src, int w, uint64_t* d_codes, cudaStream_t st);
void slice_draw(const void* state, int prec128, int n, uint64_t shots, const uint64_t* pcg, double lo, double hi,
                double total, const int32_t* bit_src, int w, uint64_t code_or, uint64_t* d_codes, cudaStream_t st);
uint64_t histogram_codes(uint64_t* d_codes, uint64_t shots, int w, uint64_t* h_codes,
                         uint64_t* h_counts, cudaStream_t st);

}  // namespace svb
