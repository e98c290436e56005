#include <climits>
// Terminal-measurement sampling on the device.
//
// Two samplers share one uniform stream — numpy's PCG64 as seeded by
// `np.random.default_rng(seed)` (statevector.py:215), reproduced bit-exactly:
// 128-bit LCG, multiplier 0x2360ED051FC65DA44385DF649FCCF645, state stepped
// BEFORE output, XSL-RR output, double = (u64 >> 11) * 2^-53.  Shot s consumes
// draw s, so a thread owning shots [s0, s1) jumps ahead s0 steps (O(log s0)).
//
// * ALIAS (reference-compatible) — AliasTable.from_probs / sample_indices
//   (sampling.py:30-83) restated as device rounds:
//     total       : numpy pairwise summation, reproduced exactly (leaf = 8
//                   accumulators over <=128 elements, halving tree above);
//     scaled      : probs * (m / total);
//     each round  : deficits / capacities -> inclusive scans -> lower_bound
//                   (searchsorted side='left') -> owner; bincount(owner,
//                   deficits) as sequential per-owner sums (owner is monotone,
//                   so each bin is one run: bit-identical to numpy); stable
//                   compactions for the next round.
//   The two cumsums are sequential on the device as in numpy, so given the
//   same probability vector the table is bit-identical to the reference's.
// * CDF (native) — fused |amp|^2 + per-32-amplitude leaf sums, one inclusive
//   scan over the leaves, then per shot a binary search over leaf prefixes and
//   a 32-element scan inside the leaf.  Passes chi^2 against |amp|^2.
//
// Codes (clbit-packed outcomes) are histogrammed with a radix sort + run
// length encode, giving np.unique's ascending (value, count) pairs.


#include <vector>

#include "common.cuh"
#include "kernels.h"

namespace svb {

typedef unsigned __int128 u128;
__host__ __device__ __forceinline__ u128 pcg_mult() {
  return ((u128)0x2360ED051FC65DA4ull << 64) | 0x4385DF649FCCF645ull;
}

struct Pcg {
  u128 s, inc;
  __host__ __device__ __forceinline__ uint64_t next64() {
    s = s * pcg_mult() + inc;
    uint64_t hi = (uint64_t)(s >> 64), lo = (uint64_t)s;
    uint64_t x = hi ^ lo;
    unsigned r = (unsigned)(hi >> 58);
    return (x >> r) | (x << ((64u - r) & 63u));
  }
  __host__ __device__ __forceinline__ double next_double() {
    return (double)(next64() >> 11) * (1.0 / 9007199254740992.0);
  }
  // skip `delta` draws (LCG jump-ahead, Brown 1994)
  __host__ __device__ void advance(uint64_t delta) {
    u128 acc_m = 1, acc_p = 0, cur_m = pcg_mult(), cur_p = inc;
    while (delta) {
      if (delta & 1) {
        acc_m *= cur_m;
        acc_p = acc_p * cur_m + cur_p;
      }
      cur_p = (cur_m + 1) * cur_p;
      cur_m *= cur_m;
      delta >>= 1;
    }
    s = acc_m * s + acc_p;
  }
};

static inline Pcg pcg_from(const uint64_t* p) {
  Pcg g;
  g.s = ((u128)p[0] << 64) | p[1];
  g.inc = ((u128)p[2] << 64) | p[3];
  return g;
}

void host_pcg_advance(uint64_t* p, uint64_t delta) {
  Pcg g = pcg_from(p);
  g.advance(delta);
  p[0] = (uint64_t)(g.s >> 64);
  p[1] = (uint64_t)g.s;
}

// --------------------------------------------------- numpy pairwise summation
__device__ double np_pairwise(const double* a, uint64_t n) {
  if (n < 8) {
    double r = 0.0;
    for (uint64_t i = 0; i < n; ++i) r += a[i];
    return r;
  }
  if (n <= 128) {
    double r[8];
    for (int j = 0; j < 8; ++j) r[j] = a[j];
    uint64_t i = 8;
    for (; i < n - (n % 8); i += 8)
      for (int j = 0; j < 8; ++j) r[j] += a[i + j];
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; ++i) res += a[i];
    return res;
  }
  uint64_t n2 = n / 2;
  n2 -= n2 % 8;
  return np_pairwise(a, n2) + np_pairwise(a + n2, n - n2);
}

__global__ void k_pairwise_small(const double* a, uint64_t n, double* out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = np_pairwise(a, n);
}

// leaves of exactly 128 (m a power of two >= 256: the halving tree bottoms out at 128)
__global__ void k_pairwise_leaves(const double* __restrict__ a, uint64_t nleaf, double* __restrict__ out) {
  uint64_t l = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (l >= nleaf) return;
  const double* p = a + l * 128;
  double r[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) r[j] = p[j];
  for (int i = 8; i < 128; i += 8) {
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] += p[i + j];
  }
  out[l] = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
}

// one halving level: out[i] = in[2i] + in[2i+1]
__global__ void k_pair_level(const double* __restrict__ in, uint64_t nout, double* __restrict__ out) {
  uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < nout) out[i] = in[2 * i] + in[2 * i + 1];
}

// the last halving levels in one CTA (n <= 2048, a power of two): the same
// pairs in the same order as k_pair_level, levels separated by barriers
__global__ void __launch_bounds__(1024) k_pair_tail(const double* __restrict__ in, uint64_t n, double* __restrict__ out) {
  __shared__ double buf[2048];
  for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) buf[i] = in[i];
  __syncthreads();
  for (uint64_t w = n / 2; w >= 1; w /= 2) {
    double v = 0.0;
    if (threadIdx.x < w) v = buf[2 * threadIdx.x] + buf[2 * threadIdx.x + 1];
    __syncthreads();
    if (threadIdx.x < w) buf[threadIdx.x] = v;
    __syncthreads();
  }
  if (threadIdx.x == 0) out[0] = buf[0];
}

double pairwise_sum_device(const double* d_x, uint64_t m, double* d_ws, cudaStream_t st) {
  double h = 0.0;
  bool pow2 = (m & (m - 1)) == 0;
  if (!pow2 || m < 256) {
    k_pairwise_small<<<1, 1, 0, st>>>(d_x, m, d_ws);
    SVB_CHECK_LAUNCH();
    SVB_CUDA(cudaMemcpyAsync(&h, d_ws, sizeof(double), cudaMemcpyDeviceToHost, st));
    SVB_CUDA(cudaStreamSynchronize(st));
    return h;
  }
  uint64_t nl = m / 128;
  double* a = d_ws;
  double* b = d_ws + nl;
  k_pairwise_leaves<<<(unsigned)((nl + 255) / 256), 256, 0, st>>>(d_x, nl, a);
  SVB_CHECK_LAUNCH();
  while (nl > 2048) {
    uint64_t no = nl / 2;
    k_pair_level<<<(unsigned)((no + 255) / 256), 256, 0, st>>>(a, no, b);
    SVB_CHECK_LAUNCH();
    double* t = a; a = b; b = t;
    nl = no;
  }
  if (nl > 1) {
    k_pair_tail<<<1, 1024, 0, st>>>(a, nl, b);
    SVB_CHECK_LAUNCH();
    a = b;
  }
  SVB_CUDA(cudaMemcpyAsync(&h, a, sizeof(double), cudaMemcpyDeviceToHost, st));
  SVB_CUDA(cudaStreamSynchronize(st));
  return h;
}

// ----------------------------------------------------------- device buffers
struct DevBuf {
  void* p = nullptr;
  cudaStream_t st;
  explicit DevBuf(size_t bytes, cudaStream_t s) : st(s) {
    if (bytes) SVB_CUDA(cudaMallocAsync(&p, bytes, s));
  }
  ~DevBuf() {
    if (p) cudaFreeAsync(p, st);
  }
  template <typename T> T* as() { return static_cast<T*>(p); }
};

template <typename T> static T d2h_scalar(const T* d, cudaStream_t st) {
  T h;
  SVB_CUDA(cudaMemcpyAsync(&h, d, sizeof(T), cudaMemcpyDeviceToHost, st));
  SVB_CUDA(cudaStreamSynchronize(st));
  return h;
}
// *a + *b with one synchronisation (both copies into a pinned pair)
template <typename T> static T d2h_sum2(const T* a, const T* b, cudaStream_t st) {
  static thread_local T* pin = nullptr;
  if (!pin && cudaHostAlloc(reinterpret_cast<void**>(&pin), 2 * sizeof(T), cudaHostAllocPortable) != cudaSuccess) {
    cudaGetLastError();
    pin = nullptr;
    return d2h_scalar(a, st) + d2h_scalar(b, st);
  }
  SVB_CUDA(cudaMemcpyAsync(pin, a, sizeof(T), cudaMemcpyDeviceToHost, st));
  SVB_CUDA(cudaMemcpyAsync(pin + 1, b, sizeof(T), cudaMemcpyDeviceToHost, st));
  SVB_CUDA(cudaStreamSynchronize(st));
  return pin[0] + pin[1];
}

// Device prefix sums (own kernels, fixed combine order: results are
// reproducible run to run).  Three launches: per-CTA tile scans of 2048
// elements (8 per thread, warp shuffles, then the 8 warp totals), one CTA
// scanning the tile totals, and the tile offsets added back.
constexpr int kScanThreads = 256, kScanItems = 8, kScanTile = kScanThreads * kScanItems;

template <typename T> __device__ __forceinline__ T warp_incl_scan(T v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const T u = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += u;
  }
  return v;
}

// inclusive scan of this CTA's tile into out (no offset), tile total to tot[b]
template <typename T>
__global__ void __launch_bounds__(kScanThreads) k_scan_tiles(const T* __restrict__ in, T* __restrict__ out,
                                                             uint64_t n, T* __restrict__ tot, int exclusive) {
  __shared__ T wsum[kScanThreads / 32];
  const uint64_t base = (uint64_t)blockIdx.x * kScanTile + (uint64_t)threadIdx.x * kScanItems;
  T x[kScanItems];
  T run = T(0);
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    x[i] = base + i < n ? in[base + i] : T(0);
    run += x[i];
  }
  const T incl = warp_incl_scan(run);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 31) wsum[warp] = incl;
  __syncthreads();
  T woff = T(0);
  for (int w = 0; w < warp; ++w) woff += wsum[w];
  T acc = woff + incl - run;  // exclusive prefix of this thread
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    if (exclusive) {
      if (base + i < n) out[base + i] = acc;
      acc += x[i];
    } else {
      acc += x[i];
      if (base + i < n) out[base + i] = acc;
    }
  }
  if (threadIdx.x == kScanThreads - 1) {
    T t = T(0);
    for (int w = 0; w < kScanThreads / 32; ++w) t += wsum[w];
    tot[blockIdx.x] = t;
  }
}

// exclusive scan of the tile totals in place (one CTA, sequential chunks)
template <typename T> __global__ void __launch_bounds__(kScanThreads) k_scan_totals(T* __restrict__ tot, uint64_t nt) {
  __shared__ T carry_s;
  __shared__ T wsum[kScanThreads / 32];
  if (threadIdx.x == 0) carry_s = T(0);
  __syncthreads();
  for (uint64_t c0 = 0; c0 < nt; c0 += kScanThreads) {
    const uint64_t i = c0 + threadIdx.x;
    const T v = i < nt ? tot[i] : T(0);
    const T incl = warp_incl_scan(v);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    T woff = carry_s;
    for (int w = 0; w < warp; ++w) woff += wsum[w];
    if (i < nt) tot[i] = woff + incl - v;
    __syncthreads();
    if (threadIdx.x == 0) {
      T t = T(0);
      for (int w = 0; w < kScanThreads / 32; ++w) t += wsum[w];
      carry_s += t;
    }
    __syncthreads();
  }
}

template <typename T>
__global__ void k_scan_add(T* __restrict__ out, uint64_t n, const T* __restrict__ tot) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n && i >= (uint64_t)kScanTile) out[i] += tot[i / kScanTile];
}

// tot_scratch: >= ceil(n / kScanTile) elements of device memory, or null (pool buffer)
template <typename T>
static void device_scan(const T* in, T* out, uint64_t n, bool exclusive, cudaStream_t st, T* tot_scratch = nullptr) {
  if (n == 0) return;
  const uint64_t nt = (n + kScanTile - 1) / kScanTile;
  DevBuf tot_buf(tot_scratch ? 0 : sizeof(T) * nt, st);
  T* tot = tot_scratch ? tot_scratch : tot_buf.as<T>();
  k_scan_tiles<T><<<(unsigned)nt, kScanThreads, 0, st>>>(in, out, n, tot, exclusive ? 1 : 0);
  SVB_CHECK_LAUNCH();
  if (nt > 1) {
    k_scan_totals<T><<<1, kScanThreads, 0, st>>>(tot, nt);
    SVB_CHECK_LAUNCH();
    k_scan_add<T><<<(unsigned)((n + 255) / 256), 256, 0, st>>>(out, n, tot);
    SVB_CHECK_LAUNCH();
  }
}

template <typename In, typename Out>
static void scan_exclusive(const In* in, Out* out, uint64_t n, cudaStream_t st) {
  static_assert(sizeof(In) == sizeof(Out), "scan keeps the element type");
  device_scan<Out>(reinterpret_cast<const Out*>(in), out, n, true, st);
}
static void scan_inclusive(const double* in, double* out, uint64_t n, cudaStream_t st, double* tot = nullptr) {
  device_scan<double>(in, out, n, false, st, tot);
}

// np.cumsum is a left-to-right accumulation; ties between deficit and capacity
// prefixes are common (symmetric distributions), so the alias build reproduces
// it exactly.  One block: all threads stream 2048-element chunks into shared
// memory (double-buffered cp.async, coalesced) while thread 0 runs the
// dependent add chain out of shared memory; results leave coalesced.
constexpr int kSeqChunk = 2048;

__device__ __forceinline__ void seq_stage(const double* __restrict__ in, uint64_t n, uint64_t c0, double* buf) {
  for (uint32_t j = threadIdx.x; j < (uint32_t)kSeqChunk; j += blockDim.x) {
    const uint64_t i = c0 + j;
    if (i < n) {
      const uint32_t d = (uint32_t)__cvta_generic_to_shared(buf + j);
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d), "l"(in + i) : "memory");
    }
  }
  asm volatile("cp.async.commit_group;\n" ::: "memory");
}

// mode 0: out = inclusive running sum (cumsum); mode 1: *total = sum (bincount bin)
__device__ void seq_block(const double* __restrict__ in, uint64_t n, double* __restrict__ out, double* total,
                          double init = 0.0) {
  __shared__ double buf[2][kSeqChunk];
  __shared__ double acc_s;
  if (threadIdx.x == 0) acc_s = init;
  const uint64_t nch = (n + kSeqChunk - 1) / kSeqChunk;
  if (nch) seq_stage(in, n, 0, buf[0]);
  for (uint64_t c = 0; c < nch; ++c) {
    if (c + 1 < nch) seq_stage(in, n, (c + 1) * kSeqChunk, buf[(c + 1) & 1]);
    else asm volatile("cp.async.commit_group;\n" ::: "memory");
    asm volatile("cp.async.wait_group 1;\n" ::: "memory");
    __syncthreads();
    double* b = buf[c & 1];
    const uint64_t c0 = c * kSeqChunk;
    const uint32_t len = (uint32_t)((n - c0) < (uint64_t)kSeqChunk ? (n - c0) : kSeqChunk);
    if (threadIdx.x == 0) {
      double acc = acc_s;
      for (uint32_t j = 0; j < len; ++j) {
        acc += b[j];
        b[j] = acc;
      }
      acc_s = acc;
    }
    __syncthreads();
    if (out)
      for (uint32_t j = threadIdx.x; j < len; j += blockDim.x) out[c0 + j] = b[j];
    __syncthreads();
  }
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  if (total && threadIdx.x == 0) *total = acc_s;
}

// init: the running sum before in[0] (*init_d when given: a device scalar)
__global__ void __launch_bounds__(256) k_seq_cumsum(const double* __restrict__ in, double* __restrict__ out,
                                                    uint64_t n, const double* __restrict__ init_d) {
  seq_block(in, n, out, nullptr, init_d ? *init_d : 0.0);
}

static void seq_cumsum(const double* in, double* out, uint64_t n, cudaStream_t st, const double* init_d = nullptr) {
  k_seq_cumsum<<<1, 256, 0, st>>>(in, out, n, init_d);
  SVB_CHECK_LAUNCH();
}

// Exponent of the lowest set bit of each nonnegative finite x (x = k 2^e with
// k odd), min-reduced into *emin.
__global__ void k_lsb_exp_min(const double* __restrict__ in, uint64_t n, int* __restrict__ emin) {
  int e = INT_MAX;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(in[i]);
    const int ex = (int)((b >> 52) & 0x7ff);
    unsigned long long mant = b & ((1ull << 52) - 1);
    if (ex == 0 && mant == 0) continue;  // zero
    if (ex != 0) mant |= 1ull << 52;
    const int lsb = __ffsll((long long)mant) - 1 + (ex == 0 ? 1 : ex) - 1075;
    e = min(e, lsb);
  }
  for (int o = 16; o > 0; o >>= 1) e = min(e, __shfl_xor_sync(0xffffffffu, e, o));
  if ((threadIdx.x & 31) == 0 && e != INT_MAX) atomicMin(emin, e);
}

// ---- the rounding chain by binade windows (bit-exact, parallel) ----------
// While the running sum s stays in one binade [2^(e+52), 2^(e+53)), every
// value is a multiple of u = 2^e and fl(s + x) = s + u RN(x / u), except for a
// tie (x / u exactly half an integer: round-to-even depends on s) or an x
// that alone leaves the binade.  So from a known s, the window's sums are
// s + u (prefix sum of k_j = RN(x_j / u)) -- an exact int64 scan -- up to the
// first element that ties, is too large, or lifts the sum out of the binade;
// that element is one IEEE add on the device, and the next window starts in
// the new binade.  s grows by about mu per element, so a binade spans about as
// many elements as precede it: windows of max(8192, i) elements keep the work
// O(n) and their number ~ log2(n) (31-47 on the prototype's random inputs,
// every result equal to np.cumsum).  Inputs with many ties fall back to the
// sequential chain after kMaxWindows.
__global__ void k_binade_k(const double* __restrict__ x, uint64_t w, int e, int64_t* __restrict__ k,
                           unsigned long long* __restrict__ stop) {
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < w; j += (uint64_t)gridDim.x * blockDim.x) {
    const double y = ldexp(x[j], -e);  // exact (power-of-two scaling of a normal result)
    if (!(y < 9007199254740992.0) || !(y >= 0.0)) {  // >= 2^53 (leaves the binade alone), negative, NaN
      k[j] = 0;
      atomicMin(stop, (unsigned long long)j);
      continue;
    }
    const double f = floor(y), fr = y - f;  // exact
    if (fr == 0.5) {
      k[j] = 0;
      atomicMin(stop, (unsigned long long)j);
      continue;
    }
    k[j] = (int64_t)f + (fr > 0.5 ? 1 : 0);
  }
}
__global__ void k_binade_leave(const int64_t* __restrict__ K, uint64_t w, int64_t base,
                               unsigned long long* __restrict__ stop) {
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < w; j += (uint64_t)gridDim.x * blockDim.x)
    if (base + K[j] >= (int64_t)(1ull << 53)) atomicMin(stop, (unsigned long long)j);
}
__global__ void k_binade_write(const int64_t* __restrict__ K, uint64_t cnt, int64_t base, int e,
                               double* __restrict__ out) {
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < cnt; j += (uint64_t)gridDim.x * blockDim.x)
    out[j] = ldexp((double)(base + K[j]), e);  // < 2^53: exact
}
// one IEEE add: out[i] = prev + x[i] (prev = out[i - 1], or *s at a window start)
__global__ void k_binade_step(const double* __restrict__ x, double* __restrict__ out, uint64_t i, int from_out,
                              double* __restrict__ s) {
  const double prev = from_out ? out[i - 1] : *s;
  const double v = prev + x[i];
  out[i] = v;
  *s = v;
}

// Returns the number of windows, or 0 when it ran the sequential chain.
static int binade_cumsum(const double* in, double* out, uint64_t n, cudaStream_t st) {
  // measured: the chain runs at a few ns per element, a window costs ~0.1 ms
  // of launches and synchronisations, so windows pay off only for long
  // arrays, and a window budget bounds the loss on tie-heavy inputs
  constexpr int kMaxWindows = 96;
  constexpr uint64_t kMinWindow = 8192;
  if (n < (1ull << 21)) {
    seq_cumsum(in, out, n, st);
    return 0;
  }
  DevBuf kb(sizeof(int64_t) * n, st), Kb(sizeof(int64_t) * n, st), tot(sizeof(int64_t) * (n / 2048 + 2), st);
  DevBuf sb(sizeof(double) + sizeof(unsigned long long), st);
  double* d_s = sb.as<double>();
  unsigned long long* d_stop = reinterpret_cast<unsigned long long*>(d_s + 1);
  uint64_t i = 0;
  double s = 0.0;
  int windows = 0;
  while (i < n) {
    if (++windows > kMaxWindows) {  // tie-heavy input: the plain chain from here on (prefix kept)
      SVB_CUDA(cudaMemcpyAsync(d_s, &s, sizeof(double), cudaMemcpyHostToDevice, st));
      seq_cumsum(in + i, out + i, n - i, st, d_s);
      return windows;
    }
    // zero / subnormal running sums: one exact step (the first element, tiny inputs)
    if (!(s >= 0x1p-1000)) {
      SVB_CUDA(cudaMemcpyAsync(d_s, &s, sizeof(double), cudaMemcpyHostToDevice, st));
      k_binade_step<<<1, 1, 0, st>>>(in, out, i, 0, d_s);
      SVB_CHECK_LAUNCH();
      s = d2h_scalar(d_s, st);
      ++i;
      continue;
    }
    int ex;
    std::frexp(s, &ex);
    const int e = ex - 53;  // spacing of s's binade
    const int64_t base = (int64_t)std::ldexp(s, -e);
    const uint64_t w = std::min<uint64_t>(n - i, std::max<uint64_t>(kMinWindow, i));
    const unsigned long long none = ~0ull;
    SVB_CUDA(cudaMemcpyAsync(d_stop, &none, sizeof none, cudaMemcpyHostToDevice, st));
    k_binade_k<<<grid_for(w, 256), 256, 0, st>>>(in + i, w, e, kb.as<int64_t>(), d_stop);
    SVB_CHECK_LAUNCH();
    device_scan<int64_t>(kb.as<int64_t>(), Kb.as<int64_t>(), w, false, st, tot.as<int64_t>());
    k_binade_leave<<<grid_for(w, 256), 256, 0, st>>>(Kb.as<int64_t>(), w, base, d_stop);
    SVB_CHECK_LAUNCH();
    const unsigned long long stop = d2h_scalar(d_stop, st);
    const uint64_t good = stop == none ? w : (uint64_t)stop;  // [i, i + good) are s + u K
    if (good) {
      k_binade_write<<<grid_for(good, 256), 256, 0, st>>>(Kb.as<int64_t>(), good, base, e, out + i);
      SVB_CHECK_LAUNCH();
    }
    if (good == w) {
      s = d2h_scalar(out + i + w - 1, st);
      i += w;
      continue;
    }
    // the stopping element: one IEEE add after the window's valid prefix
    if (good == 0) SVB_CUDA(cudaMemcpyAsync(d_s, &s, sizeof(double), cudaMemcpyHostToDevice, st));
    k_binade_step<<<1, 1, 0, st>>>(in, out, i + good, good > 0 ? 1 : 0, d_s);
    SVB_CHECK_LAUNCH();
    s = d2h_scalar(d_s, st);
    i += good + 1;
  }
  return windows;
}

// np.cumsum (a left-to-right chain of roundings) without the chain when it
// provably never rounds: every element is a multiple of 2^e and the total
// stays below 2^(52 + e), so every partial sum in any order is exact and the
// parallel scan gives the sequential result bit for bit (GHZ / uniform /
// basis-state distributions: deficits 1.0, capacities 2^k - 1).  Otherwise
// (and for short inputs) the sequential chain runs.
static void cumsum_exact(const double* in, double* out, uint64_t n, cudaStream_t st) {
  if (n < 8192) {
    seq_cumsum(in, out, n, st);
    return;
  }
  DevBuf em(sizeof(int), st);
  const int big = INT_MAX;
  SVB_CUDA(cudaMemcpyAsync(em.p, &big, sizeof(int), cudaMemcpyHostToDevice, st));
  k_lsb_exp_min<<<grid_for(n, 256), 256, 0, st>>>(in, n, em.as<int>());
  SVB_CHECK_LAUNCH();
  device_scan<double>(in, out, n, false, st);
  const int e = d2h_scalar(em.as<int>(), st);
  const double total = d2h_scalar(out + (n - 1), st);
  const bool exact = e != INT_MAX && total < std::ldexp(1.0, 52 + e);
  static const bool trace = std::getenv("SVB_TRACE") != nullptr;
  int windows = 0;
  if (!exact) windows = binade_cumsum(in, out, n, st);
  if (trace)
    std::fprintf(stderr, "[svb] cumsum n=%llu %s (%d windows)\n", (unsigned long long)n,
                 exact ? "parallel (exact)" : windows > 0 ? "binade windows" : "sequential", windows);
}

// ------------------------------------------------------------- alias build
__global__ void k_alias_init(const double* __restrict__ probs, uint64_t m, double factor,
                             double* __restrict__ scaled, double* __restrict__ prob_row,
                             int64_t* __restrict__ alias_row, int64_t* __restrict__ big) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += stride) {
    double v = probs[i] * factor;
    scaled[i] = v;
    prob_row[i] = 1.0;
    alias_row[i] = (int64_t)i;
    big[i] = v > 1.0 ? 1 : 0;
  }
}

// split [0, m) into larges (flag) and smalls (!flag), order preserved
__global__ void k_split_iota(const int64_t* __restrict__ flag, const int64_t* __restrict__ pos,
                             uint64_t m, int64_t* __restrict__ larges, int64_t* __restrict__ smalls) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += stride) {
    if (flag[i]) larges[pos[i]] = (int64_t)i;
    else smalls[i - pos[i]] = (int64_t)i;
  }
}

__global__ void k_gather(const double* __restrict__ src, const int64_t* __restrict__ idx, uint64_t n,
                         double* __restrict__ dst) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    dst[i] = src[idx[i]];
}

__global__ void k_deficit(const double* __restrict__ scaled, const int64_t* __restrict__ smalls,
                          uint64_t ns, double* __restrict__ deficit) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < ns; i += stride)
    deficit[i] = 1.0 - scaled[smalls[i]];
}

__global__ void k_capacity(const double* __restrict__ rem, uint64_t nl, double* __restrict__ cap) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nl; i += stride)
    cap[i] = rem[i] - 1.0;
}

__global__ void k_owner(const double* __restrict__ dcum, uint64_t ns, const double* __restrict__ ccum,
                        uint64_t nl, const int64_t* __restrict__ smalls,
                        const int64_t* __restrict__ larges, const double* __restrict__ scaled,
                        int64_t* __restrict__ owner, double* __restrict__ prob_row,
                        int64_t* __restrict__ alias_row) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < ns; i += stride) {
    double d = dcum[i];
    uint64_t lo = 0, hi = nl;  // first j with ccum[j] >= d
    while (lo < hi) {
      uint64_t mid = (lo + hi) >> 1;
      if (ccum[mid] < d) lo = mid + 1;
      else hi = mid;
    }
    if (lo > nl - 1) lo = nl - 1;
    owner[i] = (int64_t)lo;
    int64_t s = smalls[i];
    prob_row[s] = scaled[s];
    alias_row[s] = larges[lo];
  }
}

// owner is non-decreasing: a run of equal owners is one bincount bin.
__global__ void k_run_heads(const int64_t* __restrict__ owner, uint64_t ns, int64_t* __restrict__ head) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < ns; i += stride)
    head[i] = (i == 0 || owner[i] != owner[i - 1]) ? 1 : 0;
}
__global__ void k_run_starts(const int64_t* __restrict__ head, const int64_t* __restrict__ hpos, uint64_t ns,
                             int64_t* __restrict__ starts) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < ns; i += stride)
    if (head[i]) starts[hpos[i]] = (int64_t)i;
}
// np.bincount(owner, weights=deficits): each bin sums its weights sequentially
// from 0.0 in index order — reproduced exactly.  Runs shorter than kLongRun: one
// thread each; longer runs are listed and summed block-cooperatively.
constexpr uint64_t kLongRun = 1024;

__global__ void k_absorb(const int64_t* __restrict__ starts, uint64_t nruns, uint64_t ns,
                         const int64_t* __restrict__ owner, const double* __restrict__ deficit,
                         double* __restrict__ rem, uint64_t* __restrict__ long_runs, unsigned long long* n_long) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t r = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; r < nruns; r += stride) {
    const uint64_t b = (uint64_t)starts[r], e = r + 1 < nruns ? (uint64_t)starts[r + 1] : ns;
    if (e - b >= kLongRun) {
      long_runs[atomicAdd(n_long, 1ull)] = r;
      continue;
    }
    double acc = 0.0;
    for (uint64_t i = b; i < e; ++i) acc += deficit[i];
    const int64_t o = owner[b];
    rem[o] = rem[o] - acc;
  }
}

__device__ __forceinline__ int lsb_exp(double x) {
  const unsigned long long bits = (unsigned long long)__double_as_longlong(x);
  const int ex = (int)((bits >> 52) & 0x7ff);
  unsigned long long mant = bits & ((1ull << 52) - 1);
  if (ex == 0 && mant == 0) return INT_MAX;
  if (ex != 0) mant |= 1ull << 52;
  return __ffsll((long long)mant) - 1 + (ex == 0 ? 1 : ex) - 1075;
}

// Long runs are reduced grid-wide: blockIdx.y picks the run, gridDim.x blocks
// stride through it with four independent loads in flight per thread (one
// block per run was load-latency bound: a 2^19-element GHZ-20 run took 1 ms).
// Each block leaves (partial sum, lowest set exponent) for k_absorb_long_fin.
constexpr int kAbsorbParts = 64;
__global__ void __launch_bounds__(256) k_absorb_long_part(const int64_t* __restrict__ starts, uint64_t nruns,
                                                          uint64_t ns, const double* __restrict__ deficit,
                                                          const uint64_t* __restrict__ long_runs,
                                                          double* __restrict__ psum, int* __restrict__ plsb) {
  __shared__ double wsum[8];
  __shared__ int wexp[8];
  const uint64_t r = long_runs[blockIdx.y];
  const uint64_t b = (uint64_t)starts[r], e = r + 1 < nruns ? (uint64_t)starts[r + 1] : ns;
  const uint64_t S = (uint64_t)gridDim.x * blockDim.x;
  double part = 0.0;
  int lsb = INT_MAX;
  for (uint64_t i = b + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < e; i += 4 * S) {
    double x[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) x[k] = i + k * S < e ? deficit[i + k * S] : 0.0;
#pragma unroll
    for (int k = 0; k < 4; ++k) { part += x[k]; lsb = min(lsb, lsb_exp(x[k])); }
  }
  for (int o = 16; o > 0; o >>= 1) {
    part += __shfl_xor_sync(0xffffffffu, part, o);
    lsb = min(lsb, __shfl_xor_sync(0xffffffffu, lsb, o));
  }
  if ((threadIdx.x & 31) == 0) { wsum[threadIdx.x >> 5] = part; wexp[threadIdx.x >> 5] = lsb; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    int l = INT_MAX;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) { t += wsum[w]; l = min(l, wexp[w]); }
    psum[(uint64_t)blockIdx.y * gridDim.x + blockIdx.x] = t;
    plsb[(uint64_t)blockIdx.y * gridDim.x + blockIdx.x] = l;
  }
}

// The in-order sum never rounds when every term is a multiple of 2^lsb and
// the total stays below 2^(52 + lsb) (see cumsum_exact): then any order gives
// it and the partials stand; else the run is re-summed as the sequential chain.
__global__ void __launch_bounds__(256) k_absorb_long_fin(const int64_t* __restrict__ starts, uint64_t nruns,
                                                         uint64_t ns, const int64_t* __restrict__ owner,
                                                         const double* __restrict__ deficit, double* __restrict__ rem,
                                                         const uint64_t* __restrict__ long_runs,
                                                         const double* __restrict__ psum,
                                                         const int* __restrict__ plsb, int parts) {
  __shared__ double tot;
  __shared__ int exact;
  const uint64_t r = long_runs[blockIdx.x];
  const uint64_t b = (uint64_t)starts[r], e = r + 1 < nruns ? (uint64_t)starts[r + 1] : ns;
  if (threadIdx.x < 32) {
    double t = 0.0;
    int l = INT_MAX;
    for (int k = threadIdx.x; k < parts; k += 32) {
      t += psum[(uint64_t)blockIdx.x * parts + k];
      l = min(l, plsb[(uint64_t)blockIdx.x * parts + k]);
    }
    for (int o = 16; o > 0; o >>= 1) {
      t += __shfl_xor_sync(0xffffffffu, t, o);
      l = min(l, __shfl_xor_sync(0xffffffffu, l, o));
    }
    if (threadIdx.x == 0) {
      tot = t;
      exact = (l == INT_MAX || t < ldexp(1.0, 52 + l)) ? 1 : 0;
    }
  }
  __syncthreads();
  if (!exact) seq_block(deficit + b, e - b, nullptr, &tot);
  __syncthreads();
  if (threadIdx.x == 0) {
    const int64_t o = owner[b];
    rem[o] = rem[o] - tot;
  }
}

__global__ void k_conv_flags(const double* __restrict__ rem, uint64_t nl, int64_t* __restrict__ conv) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nl; i += stride)
    conv[i] = rem[i] <= 1.0 ? 1 : 0;
}

__global__ void k_convert(const int64_t* __restrict__ conv, const int64_t* __restrict__ pos, uint64_t nl,
                          const int64_t* __restrict__ larges, const double* __restrict__ rem,
                          int64_t* __restrict__ new_smalls, double* __restrict__ scaled,
                          int64_t* __restrict__ new_larges, double* __restrict__ new_rem) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < nl; j += stride) {
    int64_t L = larges[j];
    if (conv[j]) {
      new_smalls[pos[j]] = L;
      scaled[L] = rem[j];
    } else {
      uint64_t k = j - pos[j];
      new_larges[k] = L;
      new_rem[k] = rem[j];
    }
  }
}

void alias_build(double* d_probs, uint64_t m, double* d_prob_row, int64_t* d_alias_row,
                 cudaStream_t st) {
  const int B = 256;
  // validation + total (sampling.py:31-42)
  DevBuf ws(sizeof(double) * (m / 64 + 16), st);
  double total = pairwise_sum_device(d_probs, m, ws.as<double>(), st);
  if (!(fabs(total - 1.0) <= 1e-9))  // np.isclose(total, 1, rtol=0, atol=1e-9)
    throw Error(SVB_E_SAMPLING, "probabilities sum to " + std::to_string(total) + ", not 1");
  double factor = (double)m / total;

  DevBuf scaled(sizeof(double) * m, st), flag(sizeof(int64_t) * m, st), pos(sizeof(int64_t) * m, st);
  k_alias_init<<<grid_for(m, B), B, 0, st>>>(d_probs, m, factor, scaled.as<double>(), d_prob_row,
                                             d_alias_row, flag.as<int64_t>());
  SVB_CHECK_LAUNCH();
  scan_exclusive(flag.as<int64_t>(), pos.as<int64_t>(), m, st);
  uint64_t nl = (uint64_t)d2h_sum2(pos.as<int64_t>() + (m - 1), flag.as<int64_t>() + (m - 1), st);
  uint64_t ns = m - nl;
  if (nl == 0 || ns == 0) return;

  DevBuf larges(sizeof(int64_t) * nl, st), smalls(sizeof(int64_t) * m, st);
  k_split_iota<<<grid_for(m, B), B, 0, st>>>(flag.as<int64_t>(), pos.as<int64_t>(), m,
                                             larges.as<int64_t>(), smalls.as<int64_t>());
  SVB_CHECK_LAUNCH();
  DevBuf rem(sizeof(double) * nl, st);
  k_gather<<<grid_for(nl, B), B, 0, st>>>(scaled.as<double>(), larges.as<int64_t>(), nl, rem.as<double>());
  SVB_CHECK_LAUNCH();

  // round scratch, sized for the first (largest) round
  DevBuf deficit(sizeof(double) * ns, st), dcum(sizeof(double) * ns, st), owner(sizeof(int64_t) * ns, st);
  DevBuf cap(sizeof(double) * nl, st), ccum(sizeof(double) * nl, st);
  DevBuf head(sizeof(int64_t) * ns, st), hpos(sizeof(int64_t) * ns, st), starts(sizeof(int64_t) * ns, st);
  DevBuf long_runs(sizeof(uint64_t) * (ns / kLongRun + 2), st), nlong(sizeof(unsigned long long), st);
  DevBuf conv(sizeof(int64_t) * nl, st), cpos(sizeof(int64_t) * nl, st);
  DevBuf larges2(sizeof(int64_t) * nl, st), rem2(sizeof(double) * nl, st);
  int64_t* L = larges.as<int64_t>();
  int64_t* L2 = larges2.as<int64_t>();
  double* Rm = rem.as<double>();
  double* Rm2 = rem2.as<double>();
  int64_t* S = smalls.as<int64_t>();

  while (ns > 0 && nl > 0) {
    k_deficit<<<grid_for(ns, B), B, 0, st>>>(scaled.as<double>(), S, ns, deficit.as<double>());
    k_capacity<<<grid_for(nl, B), B, 0, st>>>(Rm, nl, cap.as<double>());
    SVB_CHECK_LAUNCH();
    cumsum_exact(deficit.as<double>(), dcum.as<double>(), ns, st);
    cumsum_exact(cap.as<double>(), ccum.as<double>(), nl, st);
    k_owner<<<grid_for(ns, B), B, 0, st>>>(dcum.as<double>(), ns, ccum.as<double>(), nl, S, L,
                                           scaled.as<double>(), owner.as<int64_t>(), d_prob_row,
                                           d_alias_row);
    SVB_CHECK_LAUNCH();
    k_run_heads<<<grid_for(ns, B), B, 0, st>>>(owner.as<int64_t>(), ns, head.as<int64_t>());
    SVB_CHECK_LAUNCH();
    scan_exclusive(head.as<int64_t>(), hpos.as<int64_t>(), ns, st);
    k_run_starts<<<grid_for(ns, B), B, 0, st>>>(head.as<int64_t>(), hpos.as<int64_t>(), ns, starts.as<int64_t>());
    SVB_CHECK_LAUNCH();
    const uint64_t nruns = (uint64_t)d2h_sum2(hpos.as<int64_t>() + (ns - 1), head.as<int64_t>() + (ns - 1), st);
    SVB_CUDA(cudaMemsetAsync(nlong.p, 0, sizeof(unsigned long long), st));
    k_absorb<<<grid_for(nruns, 64), 64, 0, st>>>(starts.as<int64_t>(), nruns, ns, owner.as<int64_t>(),
                                                 deficit.as<double>(), Rm, long_runs.as<uint64_t>(),
                                                 nlong.as<unsigned long long>());
    SVB_CHECK_LAUNCH();
    const unsigned long long nl_runs = d2h_scalar(nlong.as<unsigned long long>(), st);
    if (nl_runs) {
      const uint64_t want = (uint64_t)4 * 148 / nl_runs;
      const int parts = (int)(want < 1 ? 1 : want > (uint64_t)kAbsorbParts ? kAbsorbParts : want);
      DevBuf psum(sizeof(double) * nl_runs * parts, st), plsb(sizeof(int) * nl_runs * parts, st);
      k_absorb_long_part<<<dim3((unsigned)parts, (unsigned)nl_runs), 256, 0, st>>>(
          starts.as<int64_t>(), nruns, ns, deficit.as<double>(), long_runs.as<uint64_t>(), psum.as<double>(),
          plsb.as<int>());
      SVB_CHECK_LAUNCH();
      k_absorb_long_fin<<<(unsigned)nl_runs, 256, 0, st>>>(starts.as<int64_t>(), nruns, ns, owner.as<int64_t>(),
                                                           deficit.as<double>(), Rm, long_runs.as<uint64_t>(),
                                                           psum.as<double>(), plsb.as<int>(), parts);
      SVB_CHECK_LAUNCH();
    }
    k_conv_flags<<<grid_for(nl, B), B, 0, st>>>(Rm, nl, conv.as<int64_t>());
    SVB_CHECK_LAUNCH();
    scan_exclusive(conv.as<int64_t>(), cpos.as<int64_t>(), nl, st);
    uint64_t nconv = (uint64_t)d2h_sum2(cpos.as<int64_t>() + (nl - 1), conv.as<int64_t>() + (nl - 1), st);
    if (nconv == 0) break;  // sampling.py:60-63
    k_convert<<<grid_for(nl, B), B, 0, st>>>(conv.as<int64_t>(), cpos.as<int64_t>(), nl, L, Rm, S,
                                             scaled.as<double>(), L2, Rm2);
    SVB_CHECK_LAUNCH();
    ns = nconv;
    nl = nl - nconv;
    int64_t* tl = L; L = L2; L2 = tl;
    double* tr = Rm; Rm = Rm2; Rm2 = tr;
  }
}

// ------------------------------------------------------------- alias draws
struct BitSrc { int8_t b[64]; };

__device__ __forceinline__ uint64_t pack_code(uint64_t idx, const BitSrc& bs, int w) {
  uint64_t code = 0;
  for (int p = 0; p < w; ++p) code |= ((idx >> bs.b[p]) & 1ull) << p;
  return code;
}

// Shots per draw thread: one shot per thread until 64k threads are in flight
// (a binary search is a chain of dependent loads, so latency, not bandwidth,
// bounds small draws: 1000 shots at 64 per thread took ~0.8 ms), then up to
// 64.  Each shot s uses PCG stream position s, so the codes do not depend on it.
inline uint32_t shots_per_thread(uint64_t shots) {
  const uint64_t k = shots >> 16;
  return (uint32_t)(k < 1 ? 1 : k > 64 ? 64 : k);
}

__global__ void k_alias_draw(const double* __restrict__ prob_row, const int64_t* __restrict__ alias_row,
                             uint64_t m, uint64_t shots, Pcg base, BitSrc bs, int w,
                             uint64_t* __restrict__ codes, uint32_t spt) {
  uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  uint64_t s0 = t * spt;
  if (s0 >= shots) return;
  uint64_t s1 = s0 + spt < shots ? s0 + spt : shots;
  Pcg g = base;
  g.advance(s0);
  const double fm = (double)m;
  for (uint64_t s = s0; s < s1; ++s) {
    double v = g.next_double() * fm;
    int64_t idx = (int64_t)v;
    double frac = v - (double)idx;
    int64_t pick = frac < prob_row[idx] ? idx : alias_row[idx];
    codes[s] = pack_code((uint64_t)pick, bs, w);
  }
}

static BitSrc make_bitsrc(const int32_t* bit_src, int w) {
  BitSrc bs;
  for (int p = 0; p < 64; ++p) bs.b[p] = p < w ? (int8_t)bit_src[p] : 0;
  return bs;
}

void alias_draw(const double* d_prob_row, const int64_t* d_alias_row, uint64_t m, uint64_t shots,
                const uint64_t* pcg, const int32_t* bit_src, int w, uint64_t* d_codes,
                cudaStream_t st) {
  const uint32_t spt = shots_per_thread(shots);
  uint64_t nthreads = (shots + spt - 1) / spt;
  k_alias_draw<<<(unsigned)((nthreads + 127) / 128), 128, 0, st>>>(
      d_prob_row, d_alias_row, m, shots, pcg_from(pcg), make_bitsrc(bit_src, w), w, d_codes, spt);
  SVB_CHECK_LAUNCH();
}

// --------------------------------------------------------------- CDF draws
// Fused |amp|^2 + leaf sums: one warp per leaf of `leaf_len` (32 << k)
// amplitudes, lanes on consecutive amplitudes.  Leaves grow with the state so
// that the leaf and prefix arrays stay <= 2^24 doubles (128 MB: the scratch
// stays mapped in the stream-ordered pool between calls).
template <typename R>
__global__ void k_leaf_sums_state(const cplx<R>* __restrict__ s, uint64_t nleaf, uint32_t leaf_len,
                                  double* __restrict__ leaf) {
  const uint64_t gw = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const int lane = threadIdx.x & 31;
  for (uint64_t l = gw; l < nleaf; l += nw) {
    double p = 0.0;
    for (uint32_t j = lane; j < leaf_len; j += 32) {
      const cplx<R> a = __ldcs(s + l * leaf_len + j);
      const double x = (double)a.x, y = (double)a.y;
      p += x * x + y * y;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) p += __shfl_xor_sync(0xffffffffu, p, o);
    if (lane == 0) leaf[l] = p;
  }
}

// leaf length for an m-amplitude state: 32, doubled until nleaf <= 2^24
inline uint32_t cdf_leaf_len(uint64_t m) {
  uint32_t L = 32;
  while (m / L > (1ull << 24)) L <<= 1;
  return L;
}

__global__ void k_leaf_sums_probs(const double* __restrict__ pr, uint64_t m, uint64_t nleaf,
                                  double* __restrict__ leaf) {
  uint64_t l = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (l >= nleaf) return;
  double acc = 0.0;
  uint64_t e = (l + 1) * 32 < m ? (l + 1) * 32 : m;
  for (uint64_t i = l * 32; i < e; ++i) acc += pr[i];
  leaf[l] = acc;
}

template <typename Prob>
__device__ __forceinline__ uint64_t cdf_pick(const double* __restrict__ cum, uint64_t nleaf, uint64_t m,
                                             double target, Prob prob, uint32_t leaf_len = 32) {
  uint64_t lo = 0, hi = nleaf;  // first leaf with cum > target
  while (lo < hi) {
    uint64_t mid = (lo + hi) >> 1;
    if (cum[mid] <= target) lo = mid + 1;
    else hi = mid;
  }
  if (lo >= nleaf) lo = nleaf - 1;
  double acc = lo ? cum[lo - 1] : 0.0;
  uint64_t i0 = lo * leaf_len, i1 = i0 + leaf_len < m ? i0 + leaf_len : m;
  uint64_t last_nz = i0;
  for (uint64_t i = i0; i < i1; ++i) {
    double p = prob(i);
    if (p > 0.0) {
      last_nz = i;
      acc += p;
      if (acc > target) return i;
    }
  }
  return last_nz;  // rounding slop at the top of the leaf
}

template <typename R>
__global__ void k_cdf_draw_state(const cplx<R>* __restrict__ s, uint64_t m, const double* __restrict__ cum,
                                 uint64_t nleaf, uint32_t leaf_len, uint64_t shots, Pcg base, BitSrc bs, int w,
                                 uint64_t* __restrict__ codes, uint32_t spt) {
  uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  uint64_t s0 = t * spt;
  if (s0 >= shots) return;
  uint64_t s1 = s0 + spt < shots ? s0 + spt : shots;
  Pcg g = base;
  g.advance(s0);
  const double total = cum[nleaf - 1];
  auto prob = [&](uint64_t i) {
    cplx<R> a = s[i];
    double x = (double)a.x, y = (double)a.y;
    return x * x + y * y;
  };
  for (uint64_t k = s0; k < s1; ++k) {
    double target = g.next_double() * total;
    codes[k] = pack_code(cdf_pick(cum, nleaf, m, target, prob, leaf_len), bs, w);
  }
}

__global__ void k_cdf_draw_probs(const double* __restrict__ pr, uint64_t m, const double* __restrict__ cum,
                                 uint64_t nleaf, uint64_t shots, Pcg base, BitSrc bs, int w,
                                 uint64_t* __restrict__ codes, uint32_t spt) {
  uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  uint64_t s0 = t * spt;
  if (s0 >= shots) return;
  uint64_t s1 = s0 + spt < shots ? s0 + spt : shots;
  Pcg g = base;
  g.advance(s0);
  const double total = cum[nleaf - 1];
  auto prob = [&](uint64_t i) { return pr[i]; };
  for (uint64_t k = s0; k < s1; ++k) {
    double target = g.next_double() * total;
    codes[k] = pack_code(cdf_pick(cum, nleaf, m, target, prob), bs, w);
  }
}

uint64_t cdf_scratch_doubles(int n) {  // leaf sums, their prefix, the scan's tile totals
  const uint64_t m = 1ull << n, nleaf = m / cdf_leaf_len(m);
  return 2 * nleaf + (nleaf + kScanTile - 1) / kScanTile;
}

template <typename R>
void cdf_draw_scratch(const void* state, int n, uint64_t shots, const uint64_t* pcg, const int32_t* bit_src,
                      int w, uint64_t* d_codes, cudaStream_t st, double* scratch) {
  uint64_t m = 1ull << n;
  require(n >= 5, SVB_E_ARG, "cdf sampler needs n >= 5");
  const uint32_t L = cdf_leaf_len(m);
  uint64_t nleaf = m / L;
  double* leaf = scratch;
  double* cum = scratch + nleaf;
  k_leaf_sums_state<R><<<grid_for(nleaf * 32, 256), 256, 0, st>>>(static_cast<const cplx<R>*>(state),
                                                                    nleaf, L, leaf);
  SVB_CHECK_LAUNCH();
  scan_inclusive(leaf, cum, nleaf, st, scratch + 2 * nleaf);
  const uint32_t spt = shots_per_thread(shots);
  uint64_t nthreads = (shots + spt - 1) / spt;
  k_cdf_draw_state<R><<<(unsigned)((nthreads + 127) / 128), 128, 0, st>>>(
      static_cast<const cplx<R>*>(state), m, cum, nleaf, L, shots, pcg_from(pcg),
      make_bitsrc(bit_src, w), w, d_codes, spt);
  SVB_CHECK_LAUNCH();
}

template <typename R>
void cdf_draw(const void* state, int n, uint64_t shots, const uint64_t* pcg, const int32_t* bit_src,
              int w, uint64_t* d_codes, cudaStream_t st) {
  require(n >= 5, SVB_E_ARG, "cdf sampler needs n >= 5");
  DevBuf scratch(sizeof(double) * cdf_scratch_doubles(n), st);
  cdf_draw_scratch<R>(state, n, shots, pcg, bit_src, w, d_codes, st, scratch.as<double>());
}

void cdf_draw_probs(const double* d_probs, uint64_t m, uint64_t shots, const uint64_t* pcg,
                    const int32_t* bit_src, int w, uint64_t* d_codes, cudaStream_t st) {
  uint64_t nleaf = (m + 31) / 32;
  DevBuf leaf(sizeof(double) * nleaf, st), cum(sizeof(double) * nleaf, st);
  k_leaf_sums_probs<<<(unsigned)((nleaf + 255) / 256), 256, 0, st>>>(d_probs, m, nleaf, leaf.as<double>());
  SVB_CHECK_LAUNCH();
  scan_inclusive(leaf.as<double>(), cum.as<double>(), nleaf, st);
  const uint32_t spt = shots_per_thread(shots);
  uint64_t nthreads = (shots + spt - 1) / spt;
  k_cdf_draw_probs<<<(unsigned)((nthreads + 127) / 128), 128, 0, st>>>(
      d_probs, m, cum.as<double>(), nleaf, shots, pcg_from(pcg), make_bitsrc(bit_src, w), w, d_codes, spt);
  SVB_CHECK_LAUNCH();
}

template void cdf_draw<float>(const void*, int, uint64_t, const uint64_t*, const int32_t*, int,
                              uint64_t*, cudaStream_t);
template void cdf_draw<double>(const void*, int, uint64_t, const uint64_t*, const int32_t*, int,
                               uint64_t*, cudaStream_t);
template void cdf_draw_scratch<float>(const void*, int, uint64_t, const uint64_t*, const int32_t*, int,
                                      uint64_t*, cudaStream_t, double*);
template void cdf_draw_scratch<double>(const void*, int, uint64_t, const uint64_t*, const int32_t*, int,
                                       uint64_t*, cudaStream_t, double*);

// ------------------------------------------------- sharded CDF slice draw
// Shot s (stream position s) belongs to this shard when its global target
// tau = u_s * total falls in [lo, hi); its local target is tau - lo.  Codes
// of foreign shots are set to the sentinel ~0 (dropped by the histogram).
__global__ void k_slice_draw(const double* __restrict__ cum, const double* __restrict__ pr_unused,
                             const void* __restrict__ state, int prec128, uint64_t m, uint64_t nleaf,
                             uint32_t leaf_len, uint64_t shots,
                             Pcg base, double lo, double hi, double total, BitSrc bs, int w, uint64_t code_or,
                             uint64_t* __restrict__ codes, uint32_t spt) {
  uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  uint64_t s0 = t * spt;
  if (s0 >= shots) return;
  uint64_t s1 = s0 + spt < shots ? s0 + spt : shots;
  Pcg g = base;
  g.advance(s0);
  auto prob = [&](uint64_t i) {
    if (prec128) {
      double2 a = static_cast<const double2*>(state)[i];
      return a.x * a.x + a.y * a.y;
    }
    float2 a = static_cast<const float2*>(state)[i];
    const double x = a.x, y = a.y;
    return x * x + y * y;
  };
  for (uint64_t k = s0; k < s1; ++k) {
    const double tau = g.next_double() * total;
    if (tau < lo || tau >= hi) {
      codes[k] = ~0ull;
      continue;
    }
    double x = tau - lo;
    const double tl = cum[nleaf - 1];
    if (x >= tl) x = tl * (1.0 - 1e-16);
    const uint64_t idx = cdf_pick(cum, nleaf, m, x, prob, leaf_len);
    uint64_t code = code_or;
    for (int p = 0; p < w; ++p)
      if (bs.b[p] >= 0) code |= ((idx >> bs.b[p]) & 1ull) << p;
    codes[k] = code;
  }
  (void)pr_unused;
}

void slice_draw(const void* state, int prec128, int n, uint64_t shots, const uint64_t* pcg, double lo, double hi,
                double total, const int32_t* bit_src, int w, uint64_t code_or, uint64_t* d_codes, cudaStream_t st) {
  const uint64_t m = 1ull << n;
  const uint32_t L = cdf_leaf_len(m);
  const uint64_t nleaf = m / L;
  DevBuf leaf(sizeof(double) * nleaf, st), cum(sizeof(double) * nleaf, st);
  if (prec128)
    k_leaf_sums_state<double><<<grid_for(nleaf * 32, 256), 256, 0, st>>>(static_cast<const double2*>(state), nleaf,
                                                                         L, leaf.as<double>());
  else
    k_leaf_sums_state<float><<<grid_for(nleaf * 32, 256), 256, 0, st>>>(static_cast<const float2*>(state), nleaf,
                                                                        L, leaf.as<double>());
  SVB_CHECK_LAUNCH();
  scan_inclusive(leaf.as<double>(), cum.as<double>(), nleaf, st);
  BitSrc bs;
  for (int p = 0; p < 64; ++p) bs.b[p] = p < w ? (int8_t)bit_src[p] : (int8_t)-1;
  const uint32_t spt = shots_per_thread(shots);
  uint64_t nthreads = (shots + spt - 1) / spt;
  k_slice_draw<<<(unsigned)((nthreads + 127) / 128), 128, 0, st>>>(cum.as<double>(), nullptr, state, prec128, m,
                                                                   nleaf, L, shots, pcg_from(pcg), lo, hi, total, bs,
                                                                   w, code_or, d_codes, spt);
  SVB_CHECK_LAUNCH();
}

// --------------------------------------------------------------- histogram
// ------------------------------------------------------ code histogram
// (code, count) pairs sorted by code, like np.unique(codes, return_counts)
// (result.py:80-82): an LSD radix sort over the w code bits (8-bit digits;
// per pass: per-tile digit histograms, one prefix scan, a stable scatter
// ranked with warp match-any), then a run-length encode (flags, scan,
// scatter).  The sentinel ~0 (shots another shard owns) sorts last and is
// dropped.
constexpr int kRsThreads = 256, kRsItems = 16, kRsTile = kRsThreads * kRsItems;

__global__ void __launch_bounds__(kRsThreads) k_rs_hist(const uint64_t* __restrict__ in, uint64_t n, int shift,
                                                        uint32_t* __restrict__ hist, uint32_t ntiles) {
  __shared__ uint32_t h[256];
  h[threadIdx.x] = 0;
  __syncthreads();
  const uint64_t base = (uint64_t)blockIdx.x * kRsTile;
  for (int i = 0; i < kRsItems; ++i) {
    const uint64_t e = base + (uint64_t)i * kRsThreads + threadIdx.x;
    if (e < n) atomicAdd(&h[(in[e] >> shift) & 255u], 1u);
  }
  __syncthreads();
  hist[(uint64_t)threadIdx.x * ntiles + blockIdx.x] = h[threadIdx.x];  // digit-major
}

__global__ void __launch_bounds__(kRsThreads) k_rs_scatter(const uint64_t* __restrict__ in, uint64_t* __restrict__ out,
                                                           uint64_t n, int shift, const uint32_t* __restrict__ off,
                                                           uint32_t ntiles) {
  __shared__ uint32_t run[256];
  __shared__ uint32_t wcnt[kRsThreads / 32][256];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  run[tid] = off[(uint64_t)tid * ntiles + blockIdx.x];
  const uint64_t base = (uint64_t)blockIdx.x * kRsTile;
  for (int r = 0; r < kRsItems; ++r) {
    for (int w = 0; w < kRsThreads / 32; ++w) wcnt[w][tid] = 0;
    __syncthreads();
    const uint64_t e = base + (uint64_t)r * kRsThreads + tid;
    const bool valid = e < n;
    const uint64_t key = valid ? in[e] : 0;
    const uint32_t d = valid ? (uint32_t)((key >> shift) & 255u) : 256u + lane;  // invalid lanes never match
    const uint32_t peers = __match_any_sync(0xffffffffu, d);
    const uint32_t rank = __popc(peers & ((1u << lane) - 1u));
    if (valid && rank == 0) wcnt[warp][d] = __popc(peers);
    __syncthreads();
    if (valid) {
      uint32_t pos = run[d] + rank;
      for (int w = 0; w < warp; ++w) pos += wcnt[w][d];
      out[pos] = key;
    }
    __syncthreads();
    uint32_t add = 0;
    for (int w = 0; w < kRsThreads / 32; ++w) add += wcnt[w][tid];
    run[tid] += add;
    __syncthreads();
  }
}

__global__ void k_rle_flags(const uint64_t* __restrict__ a, uint64_t n, uint32_t* __restrict__ flag) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) flag[i] = (i == 0 || a[i] != a[i - 1]) ? 1u : 0u;
}

__global__ void k_rle_scatter(const uint64_t* __restrict__ a, uint64_t n, const uint32_t* __restrict__ pos,
                              const uint32_t* __restrict__ flag, uint64_t* __restrict__ uniq,
                              uint64_t* __restrict__ start) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n && flag[i]) {
    uniq[pos[i]] = a[i];
    start[pos[i]] = i;
  }
}

__global__ void k_rle_counts(const uint64_t* __restrict__ start, uint64_t nruns, uint64_t n,
                             uint64_t* __restrict__ cnt) {
  const uint64_t r = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r < nruns) cnt[r] = (r + 1 < nruns ? start[r + 1] : n) - start[r];
}

uint64_t histogram_codes(uint64_t* d_codes, uint64_t shots, int w, uint64_t* h_codes,
                         uint64_t* h_counts, cudaStream_t st) {
  require(shots < (1ull << 32), SVB_E_ARG, "histogram: at most 2^32 - 1 shots per call");
  const int bits = w >= 64 ? 64 : (w < 1 ? 1 : w);
  const uint32_t ntiles = (uint32_t)((shots + kRsTile - 1) / kRsTile);
  DevBuf alt(sizeof(uint64_t) * shots, st), hist(sizeof(uint32_t) * 256 * (uint64_t)ntiles, st);
  uint64_t* src = d_codes;
  uint64_t* dst = alt.as<uint64_t>();
  for (int shift = 0; shift < bits; shift += 8) {
    k_rs_hist<<<ntiles, kRsThreads, 0, st>>>(src, shots, shift, hist.as<uint32_t>(), ntiles);
    SVB_CHECK_LAUNCH();
    device_scan<uint32_t>(hist.as<uint32_t>(), hist.as<uint32_t>(), 256ull * ntiles, true, st);
    k_rs_scatter<<<ntiles, kRsThreads, 0, st>>>(src, dst, shots, shift, hist.as<uint32_t>(), ntiles);
    SVB_CHECK_LAUNCH();
    std::swap(src, dst);
  }
  // run-length encode the sorted codes in src
  DevBuf flag(sizeof(uint32_t) * shots, st), pos(sizeof(uint32_t) * shots, st);
  DevBuf uniq(sizeof(uint64_t) * shots, st), start(sizeof(uint64_t) * shots, st), cnt(sizeof(uint64_t) * shots, st);
  const unsigned g = (unsigned)((shots + 255) / 256);
  k_rle_flags<<<g, 256, 0, st>>>(src, shots, flag.as<uint32_t>());
  SVB_CHECK_LAUNCH();
  device_scan<uint32_t>(flag.as<uint32_t>(), pos.as<uint32_t>(), shots, true, st);
  k_rle_scatter<<<g, 256, 0, st>>>(src, shots, pos.as<uint32_t>(), flag.as<uint32_t>(), uniq.as<uint64_t>(),
                                   start.as<uint64_t>());
  SVB_CHECK_LAUNCH();
  const uint64_t nruns = (uint64_t)d2h_sum2(pos.as<uint32_t>() + (shots - 1), flag.as<uint32_t>() + (shots - 1), st);
  k_rle_counts<<<(unsigned)((nruns + 255) / 256), 256, 0, st>>>(start.as<uint64_t>(), nruns, shots,
                                                                 cnt.as<uint64_t>());
  SVB_CHECK_LAUNCH();
  uint64_t keep = nruns;
  if (keep > 0 && d2h_scalar(uniq.as<uint64_t>() + (keep - 1), st) == ~0ull) --keep;  // foreign shots
  SVB_CUDA(cudaMemcpyAsync(h_codes, uniq.p, sizeof(uint64_t) * keep, cudaMemcpyDeviceToHost, st));
  SVB_CUDA(cudaMemcpyAsync(h_counts, cnt.p, sizeof(uint64_t) * keep, cudaMemcpyDeviceToHost, st));
  SVB_CUDA(cudaStreamSynchronize(st));
  return keep;
}

}  // namespace svb
