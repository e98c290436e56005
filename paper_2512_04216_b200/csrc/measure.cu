// Read-only reductions over the state vector (HBM-bound, s·2^n bytes read):
//   * marginal probabilities      — marginal_probs, statevector.py:131-139
//   * multi-mask <Z_mask>         — expectation,    statevector.py:277-292
//   * measure / reset collapse    — _measure_qubit / _reset_qubit, statevector.py:142-154
// Every reduction has a fixed, size-determined partition and a fixed combine
// order, so results are bitwise reproducible run to run (seed determinism,
// SPEC.md:155).
#include <vector>

#include "common.cuh"
#include "kernels.h"

namespace svb {

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Fixed-order block sum (blockDim.x == 256); result valid in thread 0.
__device__ __forceinline__ double block_sum256(double v, double* sh) {
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) sh[w] = v;
  __syncthreads();
  double r = 0.0;
  if (threadIdx.x == 0) {
    r = ((sh[0] + sh[1]) + (sh[2] + sh[3])) + ((sh[4] + sh[5]) + (sh[6] + sh[7]));
  }
  __syncthreads();
  return r;
}

static inline int reduce_blocks(uint64_t work) {
  // size-determined (not device-determined) so results are reproducible anywhere;
  // 1184 = 8 x 148: whole waves of 256-thread blocks
  uint64_t b = work / 4096;
  if (b < 1) b = 1;
  if (b > 1184) b = 1184;
  return (int)b;
}

// ---------------------------------------------------------------- marginals
template <typename R>
__global__ void k_probs_full(const cplx<R>* __restrict__ s, double* __restrict__ out, uint64_t len) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < len; i += stride) {
    cplx<R> a = s[i];
    double x = (double)a.x, y = (double)a.y;
    out[i] = x * x + y * y;
  }
}

__device__ __forceinline__ uint64_t deposit(uint64_t v, uint64_t mask) {
  uint64_t r = 0;
  for (uint64_t bb = 1; mask; bb <<= 1) {
    uint64_t low = mask & (~mask + 1);
    if (v & bb) r |= low;
    mask &= mask - 1;
  }
  return r;
}

// partial[o * nch + ch] = sum over r in chunk ch of |a[dep(o,Q) | dep(r,~Q)]|^2
template <typename R>
__global__ void k_marg_partial(const cplx<R>* __restrict__ s, uint64_t qmask, uint64_t rmask,
                               uint64_t rlen, uint64_t nch, uint64_t chunk, double* partial) {
  __shared__ double sh[8];
  const uint64_t blk = blockIdx.x;
  const uint64_t o = blk / nch, ch = blk % nch;
  const uint64_t obase = deposit(o, qmask);
  double acc = 0.0;
  uint64_t r0 = ch * chunk, r1 = r0 + chunk < rlen ? r0 + chunk : rlen;
  for (uint64_t r = r0 + threadIdx.x; r < r1; r += blockDim.x) {
    cplx<R> a = s[obase | deposit(r, rmask)];
    double x = (double)a.x, y = (double)a.y;
    acc += x * x + y * y;
  }
  double t = block_sum256(acc, sh);
  if (threadIdx.x == 0) partial[blk] = t;
}

__global__ void k_sum_rows(const double* __restrict__ partial, uint64_t rows, uint64_t cols,
                           double* __restrict__ out) {
  uint64_t o = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (o >= rows) return;
  double acc = 0.0;
  for (uint64_t c = 0; c < cols; ++c) acc += partial[o * cols + c];
  out[o] = acc;
}

void launch_sum_rows(const double* d_partial, uint64_t rows, uint64_t cols, double* d_out, cudaStream_t st) {
  k_sum_rows<<<(unsigned)((rows + 255) / 256), 256, 0, st>>>(d_partial, rows, cols, d_out);
  SVB_CHECK_LAUNCH();
}

static void marg_geometry(int n, int k, uint64_t* nch, uint64_t* chunk) {
  uint64_t rlen = 1ull << (n - k);
  *chunk = rlen < 16384 ? rlen : 16384;
  *nch = (rlen + *chunk - 1) / *chunk;
}

size_t marginal_ws_doubles(int n, int k) {
  if (k == n) return 0;
  uint64_t nch, chunk;
  marg_geometry(n, k, &nch, &chunk);
  return (size_t)((1ull << k) * nch);
}

template <typename R>
void launch_marginal(const void* state, int n, const int32_t* qubits, int k, double* d_out,
                     double* d_ws, size_t ws_doubles, cudaStream_t st) {
  const cplx<R>* s = static_cast<const cplx<R>*>(state);
  if (k == n) {
    uint64_t len = 1ull << n;
    k_probs_full<R><<<grid_for(len, 256), 256, 0, st>>>(s, d_out, len);
    SVB_CHECK_LAUNCH();
    return;
  }
  uint64_t qmask = 0;
  for (int j = 0; j < k; ++j) qmask |= 1ull << qubits[j];
  uint64_t full = (n == 64) ? ~0ull : ((1ull << n) - 1);
  uint64_t rmask = full & ~qmask;
  uint64_t nch, chunk;
  marg_geometry(n, k, &nch, &chunk);
  uint64_t rows = 1ull << k;
  require(ws_doubles >= rows * nch, SVB_E_ARG, "marginal workspace too small");
  uint64_t nblk = rows * nch;
  require(nblk < (1ull << 31), SVB_E_ARG, "marginal grid too large");
  k_marg_partial<R><<<(unsigned)nblk, 256, 0, st>>>(s, qmask, rmask, 1ull << (n - k), nch, chunk, d_ws);
  SVB_CHECK_LAUNCH();
  k_sum_rows<<<(unsigned)((rows + 255) / 256), 256, 0, st>>>(d_ws, rows, nch, d_out);
  SVB_CHECK_LAUNCH();
}

// ------------------------------------------------------- multi-mask <Z...Z>
// For 16 amplitudes differing in 4 index bits, sum_j p_j (-1)^popc(i & mask)
// = (-1)^popc(fixed bits & mask) * W[mask restricted to the 4 bits], where W is
// the 16-point Walsh-Hadamard transform of the p_j — so any number of masks
// costs one 64-add transform per 16 amplitudes plus one lookup per mask.
constexpr int kMaskBatch = 32;
struct MaskSet { uint64_t m[kMaskBatch]; };

template <typename R>
__global__ void __launch_bounds__(256) k_expect_partial(const cplx<R>* __restrict__ s, uint64_t nchunks,
                                                        MaskSet ms, int nm, double* partial) {
  // a warp owns chunks of 512 amplitudes; lane l holds index bits 0..4 = l and
  // its 16 values differ in bits 5..8 (coalesced loads); the Walsh-Hadamard
  // transform runs over bits 5..8, the sign of the other bits is per lane/chunk
  __shared__ double sh[8];
  __shared__ double wsh[256 * 17];
  double* W = wsh + threadIdx.x * 17;  // padded: conflict-free
  const uint32_t lane = threadIdx.x & 31u;
  double acc[kMaskBatch];
#pragma unroll
  for (int j = 0; j < kMaskBatch; ++j) acc[j] = 0.0;
  const uint64_t gw = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t c = gw; c < nchunks; c += nw) {
    const cplx<R>* base = s + c * 512 + lane;
    double w[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const cplx<R> a = __ldcs(base + 32 * j);
      const double x = (double)a.x, y = (double)a.y;
      w[j] = x * x + y * y;
    }
#pragma unroll
    for (int h = 1; h < 16; h <<= 1)
#pragma unroll
      for (int j = 0; j < 16; ++j)
        if (!(j & h)) {
          const double u = w[j], v = w[j | h];
          w[j] = u + v;
          w[j | h] = u - v;
        }
#pragma unroll
    for (int j = 0; j < 16; ++j) W[j] = w[j];
    const uint64_t fixed = c * 512 + lane;  // bits 0..4 and >= 9
#pragma unroll
    for (int k = 0; k < kMaskBatch; ++k) {
      if (k < nm) {
        const double v = W[(ms.m[k] >> 5) & 15ull];
        acc[k] += (__popcll(fixed & ms.m[k] & ~0x1e0ull) & 1) ? -v : v;
      }
    }
  }
#pragma unroll
  for (int j = 0; j < kMaskBatch; ++j) {
    if (j < nm) {  // nm is uniform: the barriers inside block_sum256 are safe
      double t = block_sum256(acc[j], sh);
      if (threadIdx.x == 0) partial[(uint64_t)j * gridDim.x + blockIdx.x] = t;
    }
  }
}

// small states (< 16 amplitudes): direct sum
template <typename R>
__global__ void k_expect_small(const cplx<R>* __restrict__ s, uint64_t len, MaskSet ms, int nm, double* out) {
  const int k = threadIdx.x;
  if (k >= nm) return;
  double acc = 0.0;
  for (uint64_t i = 0; i < len; ++i) {
    const double x = (double)s[i].x, y = (double)s[i].y;
    const double p = x * x + y * y;
    acc += (__popcll(i & ms.m[k]) & 1) ? -p : p;
  }
  out[k] = acc;
}

size_t expect_ws_doubles(int n, int m) {
  return (size_t)reduce_blocks(1ull << n) * (size_t)kMaskBatch;
}

template <typename R>
void launch_expect_z(const void* state, int n, const uint64_t* h_masks, int m, double* d_out,
                     double* d_ws, cudaStream_t st) {
  const cplx<R>* s = static_cast<const cplx<R>*>(state);
  uint64_t len = 1ull << n;
  int G = reduce_blocks(len);
  for (int b = 0; b < m; b += kMaskBatch) {
    int nm = m - b < kMaskBatch ? m - b : kMaskBatch;
    MaskSet ms;
    for (int j = 0; j < kMaskBatch; ++j) ms.m[j] = j < nm ? h_masks[b + j] : 0;
    if (len < 512) {
      k_expect_small<R><<<1, 32, 0, st>>>(s, len, ms, nm, d_out + b);
      SVB_CHECK_LAUNCH();
      continue;
    }
    k_expect_partial<R><<<G, 256, 0, st>>>(s, len / 512, ms, nm, d_ws);
    SVB_CHECK_LAUNCH();
    k_sum_rows<<<(nm + 255) / 256, 256, 0, st>>>(d_ws, nm, G, d_out + b);
    SVB_CHECK_LAUNCH();
  }
}

// ------------------------------------------------------------ measure/reset
__device__ __forceinline__ double pcg_next_double(uint64_t* rng);

template <typename R>
__global__ void k_p1_partial(const cplx<R>* __restrict__ s, uint64_t npairs, int q, double* partial) {
  __shared__ double sh[8];
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t bit = 1ull << q;
  double acc = 0.0;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < npairs; i += stride) {
    cplx<R> a = s[insert0(i, q) | bit];
    double x = (double)a.x, y = (double)a.y;
    acc += x * x + y * y;
  }
  double t = block_sum256(acc, sh);
  if (threadIdx.x == 0) partial[blockIdx.x] = t;
}

// numpy PCG64 (XSL-RR 128/64), one step per draw — see sample.cu for the derivation.
__device__ __forceinline__ double pcg_next_double(uint64_t* rng) {
  const unsigned __int128 mult =
      ((unsigned __int128)0x2360ED051FC65DA4ull << 64) | 0x4385DF649FCCF645ull;
  unsigned __int128 st = ((unsigned __int128)rng[0] << 64) | rng[1];
  unsigned __int128 inc = ((unsigned __int128)rng[2] << 64) | rng[3];
  st = st * mult + inc;
  rng[0] = (uint64_t)(st >> 64);
  rng[1] = (uint64_t)st;
  uint64_t hi = (uint64_t)(st >> 64), lo = (uint64_t)st;
  uint64_t x = hi ^ lo;
  unsigned r = (unsigned)(hi >> 58);
  uint64_t v = (x >> r) | (x << ((64u - r) & 63u));
  return (double)(v >> 11) * (1.0 / 9007199254740992.0);
}

// ws[0..G) partials; ws[G] = scale; d_outcome[0] = outcome
__global__ void k_measure_decide(double* ws, int G, uint64_t* rng, int32_t* d_outcome,
                                 uint64_t* d_code, int rank) {
  if (threadIdx.x != 0) return;
  double p1 = 0.0;
  for (int b = 0; b < G; ++b) p1 += ws[b];
  double u = pcg_next_double(rng);
  int out = (u < p1) ? 1 : 0;
  double p = out ? p1 : 1.0 - p1;
  ws[G] = 1.0 / sqrt(p);
  d_outcome[0] = out;
  if (d_code) d_code[0] = (d_code[0] & ~(1ull << rank)) | ((uint64_t)out << rank);  // last write wins
}

template <typename R>
__global__ void k_collapse(cplx<R>* __restrict__ s, uint64_t npairs, int q, const double* ws, int G,
                           const int32_t* d_outcome, int reset) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t bit = 1ull << q;
  const int out = d_outcome[0];
  const R sc = (R)ws[G];
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < npairs; i += stride) {
    uint64_t i0 = insert0(i, q), i1 = i0 | bit;
    cplx<R> keep = out ? s[i1] : s[i0];
    keep.x *= sc;
    keep.y *= sc;
    cplx<R> z = mk<R>(R(0), R(0));
    if (reset || !out) {
      s[i0] = keep;
      s[i1] = z;
    } else {
      s[i0] = z;
      s[i1] = keep;
    }
  }
}

size_t measure_ws_doubles(int n) { return (size_t)reduce_blocks(1ull << (n - 1)) + 1; }

template <typename R>
void launch_measure(void* state, int n, int q, bool reset, uint64_t* d_rng, double* d_ws,
                    int32_t* d_outcome, uint64_t* d_code, int rank, cudaStream_t st) {
  cplx<R>* s = static_cast<cplx<R>*>(state);
  uint64_t np = 1ull << (n - 1);
  int G = reduce_blocks(np);
  k_p1_partial<R><<<G, 256, 0, st>>>(s, np, q, d_ws);
  SVB_CHECK_LAUNCH();
  k_measure_decide<<<1, 32, 0, st>>>(d_ws, G, d_rng, d_outcome, d_code, rank);
  SVB_CHECK_LAUNCH();
  k_collapse<R><<<grid_for(np, 256), 256, 0, st>>>(s, np, q, d_ws, G, d_outcome, reset ? 1 : 0);
  SVB_CHECK_LAUNCH();
}

#define INST(R)                                                                                 \
  template void launch_marginal<R>(const void*, int, const int32_t*, int, double*, double*,     \
                                   size_t, cudaStream_t);                                       \
  template void launch_expect_z<R>(const void*, int, const uint64_t*, int, double*, double*,    \
                                   cudaStream_t);                                               \
  template void launch_measure<R>(void*, int, int, bool, uint64_t*, double*, int32_t*, uint64_t*, \
                                  int, cudaStream_t);
INST(float)
INST(double)

}  // namespace svb

namespace svb {
// ------------------------------------------------- sharded-mode data moves
// Gather / scatter the half of the state whose bit L equals `bit` into / out
// of a contiguous buffer (global<->local qubit swap, sharded mode).
template <typename R>
__global__ void k_half_copy(cplx<R>* __restrict__ s, cplx<R>* __restrict__ buf, uint64_t nhalf, int L, int bit,
                            int to_buf) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t b = (uint64_t)bit << L;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nhalf; i += stride) {
    const uint64_t j = insert0(i, L) | b;
    if (to_buf) buf[i] = s[j];
    else s[j] = buf[i];
  }
}

template <typename R> void launch_half_copy(void* state, int n, void* buf, int L, int bit, int to_buf, cudaStream_t st) {
  const uint64_t nh = 1ull << (n - 1);
  k_half_copy<R><<<grid_for(nh, 256), 256, 0, st>>>(static_cast<cplx<R>*>(state), static_cast<cplx<R>*>(buf), nh, L,
                                                    bit, to_buf);
  SVB_CHECK_LAUNCH();
}
template void launch_half_copy<float>(void*, int, void*, int, int, int, cudaStream_t);

// dst[ib << na | ia] = b[ib] * a[ia]  (np.multiply.outer(b, a).reshape(-1),
// the block merge of pblock.py:76-83)
template <typename R>
__global__ void k_outer(cplx<R>* __restrict__ dst, const cplx<R>* __restrict__ a, const cplx<R>* __restrict__ b,
                        int na, uint64_t total) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t amask = (1ull << na) - 1;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += stride)
    dst[i] = cmul<R>(b[i >> na], a[i & amask]);
}

template <typename R> void launch_outer(void* dst, const void* a, const void* b, int na, int nb, cudaStream_t st) {
  const uint64_t total = 1ull << (na + nb);
  k_outer<R><<<grid_for(total, 256), 256, 0, st>>>(static_cast<cplx<R>*>(dst), static_cast<const cplx<R>*>(a),
                                                     static_cast<const cplx<R>*>(b), na, total);
  SVB_CHECK_LAUNCH();
}
template void launch_outer<float>(void*, const void*, const void*, int, int, cudaStream_t);
template void launch_outer<double>(void*, const void*, const void*, int, int, cudaStream_t);
template void launch_half_copy<double>(void*, int, void*, int, int, int, cudaStream_t);
// Distance and overlap of two states (possibly of different precisions):
// out[0] = sum |a-b|^2, out[1] = sum |a|^2, out[2] = sum |b|^2,
// out[3] + i out[4] = <a|b>.  Per-block partials in fixed order, then k_sum_rows.
template <typename RA, typename RB>
__global__ void k_compare_partial(const cplx<RA>* __restrict__ a, const cplx<RB>* __restrict__ b, uint64_t len,
                                  double* __restrict__ partial) {
  __shared__ double sh[8];
  double acc[5] = {0, 0, 0, 0, 0};
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < len; i += stride) {
    const double ax = (double)a[i].x, ay = (double)a[i].y, bx = (double)b[i].x, by = (double)b[i].y;
    const double dx = ax - bx, dy = ay - by;
    acc[0] += dx * dx + dy * dy;
    acc[1] += ax * ax + ay * ay;
    acc[2] += bx * bx + by * by;
    acc[3] += ax * bx + ay * by;
    acc[4] += ax * by - ay * bx;
  }
#pragma unroll
  for (int j = 0; j < 5; ++j) {
    const double r = block_sum256(acc[j], sh);
    if (threadIdx.x == 0) partial[(uint64_t)j * gridDim.x + blockIdx.x] = r;
  }
}

template <typename RA, typename RB>
void launch_compare(const void* a, const void* b, int n, double* d_ws, double* d_out, cudaStream_t st) {
  const uint64_t len = 1ull << n;
  const int G = reduce_blocks(len);
  k_compare_partial<RA, RB><<<G, 256, 0, st>>>(static_cast<const cplx<RA>*>(a), static_cast<const cplx<RB>*>(b), len,
                                                d_ws);
  SVB_CHECK_LAUNCH();
  k_sum_rows<<<1, 256, 0, st>>>(d_ws, 5, G, d_out);
  SVB_CHECK_LAUNCH();
}
size_t compare_ws_doubles(int n) { return 5 * (size_t)reduce_blocks(1ull << n) + 8; }
template void launch_compare<double, double>(const void*, const void*, int, double*, double*, cudaStream_t);
template void launch_compare<double, float>(const void*, const void*, int, double*, double*, cudaStream_t);
template void launch_compare<float, double>(const void*, const void*, int, double*, double*, cudaStream_t);
template void launch_compare<float, float>(const void*, const void*, int, double*, double*, cudaStream_t);
// Block pack / unpack for a grouped global<->local remap (sharded mode):
// block `blk` = the amplitudes whose local bits L[0..g) (ascending) equal
// the bits of blk; element j of the block (j in [off, off + count)) is the
// state index with j's bits deposited around the L positions.
template <typename R>
__global__ void k_block_copy(cplx<R>* __restrict__ s, cplx<R>* __restrict__ buf, BlockSel sel, uint64_t off,
                             uint64_t count, int to_buf) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < count; t += stride) {
    uint64_t j = off + t;
    for (int b = 0; b < sel.g; ++b) j = insert0(j, sel.L[b]);
    j |= sel.bits;
    if (to_buf) buf[t] = s[j];
    else s[j] = buf[t];
  }
}

template <typename R>
void launch_block_copy(void* state, void* buf, const BlockSel& sel, uint64_t off, uint64_t count, int to_buf,
                       cudaStream_t st) {
  k_block_copy<R><<<grid_for(count, 256), 256, 0, st>>>(static_cast<cplx<R>*>(state), static_cast<cplx<R>*>(buf),
                                                          sel, off, count, to_buf);
  SVB_CHECK_LAUNCH();
}
template void launch_block_copy<float>(void*, void*, const BlockSel&, uint64_t, uint64_t, int, cudaStream_t);
template void launch_block_copy<double>(void*, void*, const BlockSel&, uint64_t, uint64_t, int, cudaStream_t);
}  // namespace svb
