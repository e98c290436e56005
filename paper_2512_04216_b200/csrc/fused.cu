// sm_100a fused gate-pass kernel and the qubit-permutation pass.
//
// k_pass: one CTA per tile of 2^m amplitudes (the tile qubit set S always
// contains physical qubits 0..4).  Each thread holds 2^RB amplitudes in
// registers.  Round 0 loads straight from HBM (lanes <-> qubits 0..4, so each
// warp-wide load is 32 consecutive amplitudes = 512 B for complex128); later
// rounds re-distribute the tile through XOR-swizzled shared memory; the last
// layout stores straight back to HBM.  HBM traffic per pass is one read and
// one write of the state (2·s·2^n bytes) regardless of how many gates the
// pass applies.
//
// k_permute: out-of-place bit permutation of the index (restores the qubit
// order after swap relabeling).  Tiles cover input bits 0..4 plus the input
// bits that land on output bits 0..4, so both the reads and the writes are
// 32-amplitude contiguous runs.
#include <algorithm>
#include <chrono>
#include <deque>
#include <list>
#include <memory>
#include <mutex>
#include <unordered_map>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "jit.h"
#include "kernels.h"
#include "program.h"

namespace svb {

// ---------------------------------------------------------------- permute
// Out-of-place bit permutation of the index: output bit dest[p] = input bit p.
// A tile holds the ml input bits {0..4} ∪ dest^-1({0..4}) (plus fill up to 12),
// so both the HBM reads (input bits 0..4 innermost) and the writes (output bits
// 0..4 innermost) are 32-amplitude contiguous runs.  Per-element offsets come
// from split tables (6 + 6 bits) built once per CTA; the tile is XOR-swizzled.
struct PermDev {
  int32_t n, ml;
  int32_t lin[16];       // input bit of local bit l (ascending)
  int32_t lout_src[16];  // output-local bit e (ascending output positions) -> input-local bit
  int32_t lout_pos[16];  // output bit of output-local bit e
  int32_t nout;
  int32_t outin[48];     // input bits outside the tile, ascending
  int32_t dest[64];      // output bit of input bit p
};

template <typename R>
__global__ void __launch_bounds__(256) k_permute(const cplx<R>* __restrict__ in, cplx<R>* __restrict__ out,
                                                 const PermDev pd, uint64_t ntiles) {
  extern __shared__ __align__(16) unsigned char smraw[];
  __shared__ uint64_t in_lo[64], in_hi[64], out_lo[64], out_hi[64];
  __shared__ uint32_t src_lo[64], src_hi[64];
  cplx<R>* tile = reinterpret_cast<cplx<R>*>(smraw);
  const int ml = pd.ml, lb = ml < 6 ? ml : 6, hb = ml - lb;
  for (int x = threadIdx.x; x < 64; x += blockDim.x) {
    uint64_t a = 0, b = 0, c = 0, d = 0;
    uint32_t e = 0, f = 0;
    for (int l = 0; l < lb; ++l)
      if ((x >> l) & 1) {
        a |= 1ull << pd.lin[l];
        c |= 1ull << pd.lout_pos[l];
        e |= 1u << pd.lout_src[l];
      }
    for (int l = 0; l < hb; ++l)
      if ((x >> l) & 1) {
        b |= 1ull << pd.lin[lb + l];
        d |= 1ull << pd.lout_pos[lb + l];
        f |= 1u << pd.lout_src[lb + l];
      }
    in_lo[x] = a; in_hi[x] = b; out_lo[x] = c; out_hi[x] = d; src_lo[x] = e; src_hi[x] = f;
  }
  __syncthreads();
  const uint32_t T = 1u << ml, lmask = (1u << lb) - 1;
  for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    uint64_t bin = 0, bout = 0;
    for (int i = 0; i < pd.nout; ++i)
      if ((t >> i) & 1ull) {
        bin |= 1ull << pd.outin[i];
        bout |= 1ull << pd.dest[pd.outin[i]];
      }
    if (T == 4096 && blockDim.x == 256) {  // full tiles: 16 independent loads in flight per thread
      cplx<R> v[16];
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        const uint32_t j = threadIdx.x + 256u * k;
        v[k] = __ldcs(in + (bin | in_lo[j & lmask] | in_hi[j >> lb]));
      }
#pragma unroll
      for (int k = 0; k < 16; ++k) tile[swz<R>(threadIdx.x + 256u * k)] = v[k];
      __syncthreads();
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        const uint32_t o = threadIdx.x + 256u * k;
        const uint32_t j = src_lo[o & lmask] | src_hi[o >> lb];
        v[k] = tile[swz<R>(j)];
      }
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        const uint32_t o = threadIdx.x + 256u * k;
        __stcs(out + (bout | out_lo[o & lmask] | out_hi[o >> lb]), v[k]);
      }
    } else {
      for (uint32_t j = threadIdx.x; j < T; j += blockDim.x)
        tile[swz<R>(j)] = __ldcs(in + (bin | in_lo[j & lmask] | in_hi[j >> lb]));
      __syncthreads();
      for (uint32_t o = threadIdx.x; o < T; o += blockDim.x) {
        const uint32_t j = src_lo[o & lmask] | src_hi[o >> lb];
        __stcs(out + (bout | out_lo[o & lmask] | out_hi[o >> lb]), tile[swz<R>(j)]);
      }
    }
    __syncthreads();
  }
}

// complex128 full tiles (4096 amplitudes, 256 threads): persistent CTA per SM
// with a 2-stage cp.async ring, so tile t+1 streams in while tile t is
// permuted through shared memory and stored.
__global__ void __launch_bounds__(256, 1) k_permute_pipe(const cplx<double>* __restrict__ in,
                                                        cplx<double>* __restrict__ out, const PermDev pd,
                                                        uint64_t ntiles) {
  extern __shared__ __align__(128) unsigned char smraw[];
  __shared__ uint64_t in_lo[64], in_hi[64], out_lo[64], out_hi[64];
  __shared__ uint32_t src_lo[64], src_hi[64];
  __shared__ uint64_t t_in[48], t_out[48];
  cplx<double>* ring = reinterpret_cast<cplx<double>*>(smraw);
  constexpr int lb = 6;  // ml == 12
  for (int x = threadIdx.x; x < 64; x += blockDim.x) {
    uint64_t a = 0, b = 0, c = 0, d = 0;
    uint32_t e = 0, f = 0;
    for (int l = 0; l < lb; ++l)
      if ((x >> l) & 1) {
        a |= 1ull << pd.lin[l];
        c |= 1ull << pd.lout_pos[l];
        e |= 1u << pd.lout_src[l];
        b |= 1ull << pd.lin[lb + l];
        d |= 1ull << pd.lout_pos[lb + l];
        f |= 1u << pd.lout_src[lb + l];
      }
    in_lo[x] = a; in_hi[x] = b; out_lo[x] = c; out_hi[x] = d; src_lo[x] = e; src_hi[x] = f;
  }
  for (int i = threadIdx.x; i < pd.nout; i += blockDim.x) {
    t_in[i] = 1ull << pd.outin[i];
    t_out[i] = 1ull << pd.dest[pd.outin[i]];
  }
  __syncthreads();
  const uint32_t tid = threadIdx.x;
  auto bases = [&](uint64_t t, uint64_t& bin, uint64_t& bout) {
    bin = 0;
    bout = 0;
    for (int i = 0; i < pd.nout; ++i)
      if ((t >> i) & 1ull) { bin |= t_in[i]; bout |= t_out[i]; }
  };
  auto issue = [&](uint64_t t, int b) {
    uint64_t bin, bout;
    bases(t, bin, bout);
    cplx<double>* dst = ring + (size_t)b * 4096;
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const uint32_t j = tid + 256u * k;
      cp_async16(dst + swz<double>(j), in + (bin | in_lo[j & 63u] | in_hi[j >> lb]));
    }
  };
  uint64_t t = blockIdx.x;
  if (t < ntiles) issue(t, 0);
  cp_async_commit();
  for (int it = 0; t < ntiles; t += gridDim.x, ++it) {
    const uint64_t tn = t + gridDim.x;
    if (tn < ntiles) issue(tn, (it + 1) & 1);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    uint64_t bin, bout;
    bases(t, bin, bout);
    const cplx<double>* cur = ring + (size_t)(it & 1) * 4096;
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const uint32_t o = tid + 256u * k;
      const uint32_t j = src_lo[o & 63u] | src_hi[o >> lb];
      __stcs(out + (bout | out_lo[o & 63u] | out_hi[o >> lb]), cur[swz<double>(j)]);
    }
    __syncthreads();
  }
  cp_async_wait<0>();
}

static PermDev make_perm(int n, const std::vector<int>& dest) {
  PermDev pd{};
  pd.n = n;
  uint64_t inset = 0x1full;
  for (int p = 0; p < n; ++p)
    if (dest[p] < 5) inset |= 1ull << p;
  for (int p = 0; p < n && __builtin_popcountll(inset) < 12; ++p) inset |= 1ull << p;
  int ml = 0;
  for (int p = 0; p < n; ++p)
    if (inset & (1ull << p)) pd.lin[ml++] = p;
  pd.ml = ml;
  // output-local order: ascending output bit positions of the tile's bits
  std::vector<std::pair<int, int>> outs;  // (output bit, input-local bit)
  for (int l = 0; l < ml; ++l) outs.push_back({dest[pd.lin[l]], l});
  std::sort(outs.begin(), outs.end());
  for (int e = 0; e < ml; ++e) {
    pd.lout_pos[e] = outs[e].first;
    pd.lout_src[e] = outs[e].second;
  }
  pd.nout = 0;
  for (int p = 0; p < n; ++p)
    if (!(inset & (1ull << p))) pd.outin[pd.nout++] = p;
  for (int p = 0; p < n; ++p) pd.dest[p] = dest[p];
  return pd;
}

// --------------------------------------------------------------- profiler
void Profiler::begin(cudaStream_t st, int kind, double nbytes, int idx) {
  Rec r;
  SVB_CUDA(cudaEventCreate(&r.a));
  SVB_CUDA(cudaEventCreate(&r.b));
  r.kind = kind;
  r.idx = idx;
  r.bytes = nbytes;
  SVB_CUDA(cudaEventRecord(r.a, st));
  pending.push_back(r);
  bytes[kind] += nbytes;
}
void Profiler::end(cudaStream_t st) { SVB_CUDA(cudaEventRecord(pending.back().b, st)); }
void Profiler::collect() {
  static const bool trace = std::getenv("SVB_TRACE") != nullptr;
  for (size_t i = 0; i < pending.size(); ++i) {
    Rec& r = pending[i];
    float t = 0.f, gap = 0.f;
    SVB_CUDA(cudaEventSynchronize(r.b));
    SVB_CUDA(cudaEventElapsedTime(&t, r.a, r.b));
    if (i > 0) SVB_CUDA(cudaEventElapsedTime(&gap, pending[i - 1].b, r.a));
    if (trace) std::fprintf(stderr, "[svb] launch kind=%d %.3f ms (gap %.3f ms)\n", r.kind, t, gap);
    ms[r.kind] += t;
    count[r.kind] += 1;
    if (r.idx >= 0) {
      if ((int)idx_ms.size() <= r.idx) {
        idx_ms.resize(r.idx + 1, 0.0);
        idx_bytes.resize(r.idx + 1, 0.0);
        idx_count.resize(r.idx + 1, 0);
      }
      idx_ms[r.idx] += t;
      idx_bytes[r.idx] += r.bytes;
      idx_count[r.idx] += 1;
    }
  }
  for (Rec& r : pending) {
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  pending.clear();
}

// ------------------------------------------------------- fused <Z> finish
// Block (k, slice) sums value k of the last pass's <Z> slots (zsum_store) over
// a slice of the `ncta` CTAs: register bits (W_i), thread bits (per-thread T
// with the sign of thread bit b), tile bits (per-warp lane sums), the total.
// partial[k * kZsumSlices + slice]; k_sum_rows finishes.
constexpr int kZsumSlices = 32;
__global__ void __launch_bounds__(256) k_zsum_finish(const double* __restrict__ zacc, uint32_t ncta, uint32_t nthr,
                                                     int rb, int nt, int nout, double* __restrict__ partial) {
  __shared__ double sh[256];
  const int k = blockIdx.x;
  const uint32_t nw = nthr >> 5;
  const uint32_t c0 = (uint32_t)(((uint64_t)ncta * blockIdx.y) / kZsumSlices);
  const uint32_t c1 = (uint32_t)(((uint64_t)ncta * (blockIdx.y + 1)) / kZsumSlices);
  const double* zw = zacc + (uint64_t)kZaccCols * (rb + 1) * nthr;
  double acc = 0.0;
  if (k < rb + nt || k == rb + nt + nout) {
    const int row = k < rb ? 1 + k : 0;
    const int b = k - rb;
    for (uint64_t i = (uint64_t)c0 * nthr + threadIdx.x; i < (uint64_t)c1 * nthr; i += blockDim.x) {
      const uint64_t cta = i / nthr, t = i % nthr;
      const double v = zacc[(cta * (rb + 1) + row) * nthr + t];
      acc += (k >= rb && k < rb + nt && ((t >> b) & 1u)) ? -v : v;
    }
  } else {
    const int j = k - rb - nt;
    for (uint64_t i = (uint64_t)c0 * nw + threadIdx.x; i < (uint64_t)c1 * nw; i += blockDim.x) acc += zw[i * 64 + j];
  }
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[(uint64_t)k * kZsumSlices + blockIdx.y] = sh[0];
}

// ------------------------------------------------------------ run_program

// Pinned staging for program uploads.  A cudaMemcpyAsync from pageable memory
// synchronises the stream before it starts, which would serialise the host
// preparation of a program with the device work queued before it (the batch
// executor queues one circuit after another on each stream).  Uploads go
// through a per-thread pinned ring instead; a region is reused only after
// the copy that read it has completed (its event).
namespace {
struct PinnedRing {
  uint8_t* base = nullptr;
  size_t cap = 0, head = 0;
  struct Span { size_t off, len; cudaEvent_t ev; };
  std::deque<Span> live;
  ~PinnedRing() {
    for (auto& sp : live) cudaEventDestroy(sp.ev);
    if (base) cudaFreeHost(base);
  }
  void retire_all() {
    for (auto& sp : live) {
      cudaEventSynchronize(sp.ev);
      cudaEventDestroy(sp.ev);
    }
    live.clear();
  }
  // host staging of n bytes, free of in-flight copies
  uint8_t* take(size_t n) {
    n = (n + 255) & ~size_t(255);
    if (n > cap) {
      retire_all();
      if (base) cudaFreeHost(base);
      cap = std::max<size_t>(n, 8u << 20);
      if (cudaHostAlloc(reinterpret_cast<void**>(&base), cap, cudaHostAllocPortable) != cudaSuccess) {
        base = nullptr;
        cap = 0;
        throw Error(SVB_E_OOM, "pinned staging allocation failed");
      }
      head = 0;
    }
    if (head + n > cap) head = 0;
    const size_t lo = head, hi = head + n;
    while (!live.empty() && (!live.front().ev || cudaEventQuery(live.front().ev) == cudaSuccess)) {
      if (live.front().ev) cudaEventDestroy(live.front().ev);
      live.pop_front();
    }
    cudaGetLastError();  // a not-ready query is not an error
    for (auto it = live.begin(); it != live.end();) {
      if (it->off < hi && it->off + it->len > lo) {  // an in-flight copy still reads this region
        if (it->ev) {
          cudaEventSynchronize(it->ev);
          cudaEventDestroy(it->ev);
        }
        it = live.erase(it);
      } else {
        ++it;
      }
    }
    head = hi;
    uint8_t* p = base + lo;
    live.push_back({lo, n, nullptr});
    return p;
  }
  void recorded(cudaStream_t st) {  // the copy from the last take() is queued on st
    cudaEvent_t ev;
    SVB_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    SVB_CUDA(cudaEventRecord(ev, st));
    live.back().ev = ev;
  }
};
thread_local PinnedRing t_ring;
}  // namespace

static void upload(void* dst, const void* src, size_t n, cudaStream_t st) {
  // opt-in (SVB_PINNED_UPLOAD=1): measured no steady gain on config 4 and a
  // pathological slowdown combined with the heavy-circuit limit
  static const bool pinned = std::getenv("SVB_PINNED_UPLOAD") && std::atoi(std::getenv("SVB_PINNED_UPLOAD")) != 0;
  if (!pinned) {
    SVB_CUDA(cudaMemcpyAsync(dst, src, n, cudaMemcpyHostToDevice, st));
    return;
  }
  uint8_t* h = t_ring.take(n);
  std::memcpy(h, src, n);
  SVB_CUDA(cudaMemcpyAsync(dst, h, n, cudaMemcpyHostToDevice, st));
  t_ring.recorded(st);
}

// Device-resident programs of large states.  A state of >= 2^26 amplitudes is
// usually driven by the same program again and again (the bench step, a VQE
// loop at fixed structure, expectations after final_state): its descriptors and
// op stream stay on the device, keyed by their content, the stream and the
// fused-<Z> pointer, so an apply issues no upload before its first launch.
// Entries are immutable once uploaded and used only on the stream that
// uploaded them (stream order covers the upload); an evicted entry is freed
// stream-ordered behind its last use.  Small states (the batch executor's
// thousands of distinct programs) keep the per-apply upload.
constexpr int kResidentProgMinQubits = 26;
namespace {
struct ResidentProg {
  uint64_t h0, h1;
  cudaStream_t st;
  const double* zacc;
  size_t bytes;
  uint8_t* buf;
  cudaEvent_t last_use;
};
std::mutex g_res_mu;
std::list<ResidentProg> g_res;  // most recent first
constexpr size_t kResidentProgs = 8;
}  // namespace

template <class Fill>
static uint8_t* resident_program(const Program& prog, size_t pbytes, size_t obytes, cudaStream_t st,
                                 const double* zacc, Fill&& fill) {
  uint64_t h0 = 0x9E3779B97F4A7C15ull ^ pbytes, h1 = 0xC2B2AE3D27D4EB4Full ^ prog.ops.size();
  auto mix = [&](const void* data, size_t nb) {
    const unsigned char* p = static_cast<const unsigned char*>(data);
    size_t i = 0;
    for (; i + 16 <= nb; i += 16) {
      uint64_t w[2];
      std::memcpy(w, p + i, 16);
      h0 = (((h0 ^ (w[0] * 0x87C37B91114253D5ull)) << 31) | ((h0 ^ (w[0] * 0x87C37B91114253D5ull)) >> 33)) *
           0x4CF5AD432745937Full;
      h1 = (((h1 ^ (w[1] * 0x4CF5AD432745937Full)) << 29) | ((h1 ^ (w[1] * 0x4CF5AD432745937Full)) >> 35)) *
           0x87C37B91114253D5ull;
    }
    for (; i < nb; ++i) h0 = (h0 ^ p[i]) * 0x100000001B3ull;
  };
  mix(prog.passes.data(), pbytes);
  mix(prog.ops.data(), prog.ops.size());
  std::lock_guard<std::mutex> lk(g_res_mu);
  for (auto it = g_res.begin(); it != g_res.end(); ++it)
    if (it->h0 == h0 && it->h1 == h1 && it->st == st && it->zacc == zacc && it->bytes == pbytes + obytes) {
      // same stream value: ordered after the upload, unless the stream was
      // destroyed and its handle reused (then this orders it explicitly)
      if (it->last_use) SVB_CUDA(cudaStreamWaitEvent(st, it->last_use, 0));
      g_res.splice(g_res.begin(), g_res, it);
      return it->buf;
    }
  ResidentProg e{h0, h1, st, zacc, pbytes + obytes, nullptr, nullptr};
  SVB_CUDA(cudaMallocAsync(&e.buf, e.bytes, st));
  fill(e.buf);
  g_res.push_front(e);
  if (g_res.size() > kResidentProgs) {
    ResidentProg& old = g_res.back();
    if (old.last_use) {
      SVB_CUDA(cudaStreamWaitEvent(st, old.last_use, 0));
      cudaEventDestroy(old.last_use);
    }
    SVB_CUDA(cudaFreeAsync(old.buf, st));
    g_res.pop_back();
  }
  return e.buf;
}

// the launches reading buf are queued on st: record where its last use ends
static void resident_program_used(uint8_t* buf, cudaStream_t st) {
  std::lock_guard<std::mutex> lk(g_res_mu);
  for (auto& e : g_res)
    if (e.buf == buf) {
      if (!e.last_use) SVB_CUDA(cudaEventCreateWithFlags(&e.last_use, cudaEventDisableTiming));
      SVB_CUDA(cudaEventRecord(e.last_use, st));
      return;
    }
}

// Interpreter launches of a program's passes (k_pass<R, RB>).
template <typename R, int RB>
static void interp_passes(cplx<R>* state, cplx<R>* out, const Program& prog, const PassDev* dpass,
                          const uint8_t* dops, cudaStream_t st, ProgramStats* stats, int nsm, bool zero_input) {
  // the attribute is per function and device: set it once per device to the
  // largest size any program can request (a per-call value would race between
  // threads launching different programs)
  static std::atomic<uint64_t> once_pass{0};
  once_per_device(once_pass, [] {
    cudaFuncSetAttribute(k_pass<R, RB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemMaxPerCTA);
    cudaFuncSetAttribute(k_pass<R, RB>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  });
  cplx<R>* cur = state;
  cplx<R>* other = out;
  for (size_t p = 0; p < prog.passes.size(); ++p) {
    const PassDev& pd = prog.passes[p];
    uint64_t tiles = 1ull << pd.nout;
    unsigned threads = 1u << (pd.m - RB);
    int stages = pass_stages<R>(RB, pd.m, pd.ops_bytes, pd.ndiag, 0, 0, kInterpMinBlocks<R, RB>);
    if (stages == 1 && pd.direct && !pd.perm_in && (pd.dmask || std::getenv("SVB_DIRECT"))) stages = 0;  // see jit.cu
    // perm_in / perm_out passes write the other buffer, which then holds the state
    cplx<R>* const src = cur;
    cplx<R>* const dst = (pd.perm_in || pd.perm_out) ? other : cur;
    if (dst != src) std::swap(cur, other);
    unsigned grid = (unsigned)std::min<uint64_t>(tiles, (uint64_t)nsm * (stages <= 1 ? kInterpMinBlocks<R, RB> : 1));
    Profiler* pf = (stats->prof && stats->prof->on) ? stats->prof : nullptr;
    const int zin = (zero_input && p == 0) ? 1 : 0;
    if (pf) pf->begin(st, 0, pass_hbm_bytes<R>(pd, zin != 0), (int)p);
    k_pass<R, RB><<<grid, threads, pass_smem<R>(RB, pd.m, pd.ops_bytes, pd.ndiag, 0, stages, 0, pd.nrounds), st>>>(
        src, dst, dpass + p, dops, (uint32_t)tiles, zin, stages);
    SVB_CHECK_LAUNCH();
    if (pf) pf->end(st);
    stats->passes += 1;
    stats->launches += 1;
  }
}

// out: destination of the last pass when the program's final permutation is
// fused into it (prog.perm_fused; a second state-sized buffer), else unused.
// zacc: fused <Z> accumulators (zacc_doubles) when the last pass has zsum.
template <typename R>
static void launch_passes(cplx<R>* state, cplx<R>* out, int n, const Program& prog, cudaStream_t st,
                          ProgramStats* stats, bool use_jit, bool zero_input, double* zacc = nullptr) {
  if (prog.passes.empty()) return;
  size_t pbytes = prog.passes.size() * sizeof(PassDev);
  size_t obytes = std::max<size_t>(prog.ops.size(), 16);
  if (prog.passes.back().zsum && zacc == nullptr) throw Error(SVB_E_CUDA, "fused <Z> without a scratch buffer");
  auto fill = [&](uint8_t* dbuf) {  // one upload of descriptors + op stream (+ the fused <Z> pointer)
    std::vector<uint8_t> blob(pbytes + prog.ops.size());
    std::memcpy(blob.data(), prog.passes.data(), pbytes);
    if (!prog.ops.empty()) std::memcpy(blob.data() + pbytes, prog.ops.data(), prog.ops.size());
    if (prog.passes.back().zsum) {  // device-side pointer only: the host PassDev (and JIT cache keys) keep zacc = 0
      const uint64_t zp = (uint64_t)(uintptr_t)zacc;
      std::memcpy(blob.data() + (prog.passes.size() - 1) * sizeof(PassDev) + offsetof(PassDev, zacc), &zp, sizeof zp);
    }
    upload(dbuf, blob.data(), blob.size(), st);
  };
  uint8_t* dbuf = nullptr;
  const bool resident = n >= kResidentProgMinQubits;
  if (resident) {
    dbuf = resident_program(prog, pbytes, obytes, st, zacc, fill);
  } else {
    SVB_CUDA(cudaMallocAsync(&dbuf, pbytes + obytes, st));
    fill(dbuf);
  }
  const PassDev* dpass = reinterpret_cast<const PassDev*>(dbuf);
  const uint8_t* dops = dbuf + pbytes;
  if (prog.passes.back().zsum) {
    // zsum_store writes every slot of a launched CTA; cleared so that the finish
    // kernel may sum over an upper bound of the grid
    const PassDev& lp = prog.passes.back();
    SVB_CUDA(cudaMemsetAsync(zacc, 0, sizeof(double) * zacc_doubles(1u << (lp.m - lp.rb), lp.rb), st));
  }
  int dev = 0, nsm = 148;
  SVB_CUDA(cudaGetDevice(&dev));
  SVB_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  if ((prog.perm_fused || prog.passes[0].perm_in) && out == nullptr)
    throw Error(SVB_E_CUDA, "permuted load / store without a second buffer");
  if (use_jit && jit_launch_passes<R>(state, out, prog, dpass, dops, st, stats, nsm, zero_input)) {
    if (resident) resident_program_used(dbuf, st);
    else SVB_CUDA(cudaFreeAsync(dbuf, st));
    return;
  }
  const int rb = prog.passes[0].rb;
  if constexpr (sizeof(R) == 4) {
    if (rb == 5) interp_passes<R, 5>(state, out, prog, dpass, dops, st, stats, nsm, zero_input);
    else interp_passes<R, 4>(state, out, prog, dpass, dops, st, stats, nsm, zero_input);
  } else {
    if (rb != 4) throw Error(SVB_E_ARG, "complex128 passes have 4 register bits");
    interp_passes<R, 4>(state, out, prog, dpass, dops, st, stats, nsm, zero_input);
  }
  if (resident) resident_program_used(dbuf, st);
  else SVB_CUDA(cudaFreeAsync(dbuf, st));
}

template <typename R>
static void launch_permute(cplx<R>** state, cplx<R>** spare, int n, const std::vector<int>& dest, cudaStream_t st,
                           ProgramStats* stats) {
  PermDev pd = make_perm(n, dest);
  cplx<R>* out = *spare;
  size_t bytes = sizeof(cplx<R>) << n;
  uint64_t tiles = 1ull << pd.nout;
  int dev = 0, nsm = 148;
  SVB_CUDA(cudaGetDevice(&dev));
  SVB_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  const size_t smem = sizeof(cplx<R>) << pd.ml;
  static std::atomic<uint64_t> once_perm{0};
  once_per_device(once_perm, [] {
    cudaFuncSetAttribute(k_permute<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(sizeof(cplx<R>) << 12));
  });
  Profiler* pf = (stats->prof && stats->prof->on) ? stats->prof : nullptr;
  if (pf) pf->begin(st, 1, 2.0 * (double)bytes);
  if constexpr (sizeof(R) == 8) {
    if (pd.ml == 12) {
      static std::atomic<uint64_t> once_pipe{0};
      once_per_device(once_pipe, [] {
        cudaFuncSetAttribute(k_permute_pipe, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * 4096 * 16);
      });
      const unsigned g1 = (unsigned)std::min<uint64_t>(tiles, (uint64_t)nsm);
      k_permute_pipe<<<g1, 256, 2 * 4096 * 16, st>>>(*state, out, pd, tiles);
    } else {
      const unsigned grid = (unsigned)std::min<uint64_t>(tiles, (uint64_t)nsm * 3);
      k_permute<R><<<grid, 256, smem, st>>>(*state, out, pd, tiles);
    }
  } else {
    const unsigned grid = (unsigned)std::min<uint64_t>(tiles, (uint64_t)nsm * 3);
    k_permute<R><<<grid, 256, smem, st>>>(*state, out, pd, tiles);
  }
  SVB_CHECK_LAUNCH();
  if (pf) pf->end(st);
  // swap buffers rather than copy back (a copy would double the traffic)
  *spare = *state;
  *state = out;
  stats->passes += 1;
  stats->launches += 1;
}

template <typename R>
void run_program(void* state, int n, const svb_gate* g, int ng, int fusion, int max_high, cudaStream_t st,
                 ProgramStats* stats) {
  (void)max_high;
  stats->gates += ng;
  const SchedOptions opt = default_options(sizeof(R) == 8 ? SVB_C128 : SVB_C64, n);
  if (!fusion || n < opt.rb + 5) {
    for (int i = 0; i < ng; ++i) {
      launch_gate_basic<R>(state, n, g[i], st);
      stats->passes += 1;
      stats->launches += 1;
    }
    return;
  }
  SchedOptions o = opt;
  o.relabel_swaps = false;  // the handle owns its buffer; permutation passes need run_program_owned
  Program prog = build_program<R>(n, g, ng, o);
  launch_passes<R>(static_cast<cplx<R>*>(state), nullptr, n, prog, st, stats, false, false);
}

// Qubit permutation of a whole state (qubit p moves to bit dest[p]), out of
// place through the handle's spare buffer (pblock reorders, svb_permute_qubits).
template <typename R>
void run_permutation(void** state, void** spare, int n, const std::vector<int>& dest, cudaStream_t st,
                     ProgramStats* stats) {
  bool ident = true;
  for (int p = 0; p < n; ++p) ident = ident && dest[p] == p;
  if (ident) return;
  if (*spare == nullptr) SVB_CUDA(state_malloc(spare, sizeof(cplx<R>) << n));
  launch_permute<R>(reinterpret_cast<cplx<R>**>(state), reinterpret_cast<cplx<R>**>(spare), n, dest, st, stats);
}
template void run_permutation<float>(void**, void**, int, const std::vector<int>&, cudaStream_t, ProgramStats*);
template void run_permutation<double>(void**, void**, int, const std::vector<int>&, cudaStream_t, ProgramStats*);

// Host compile cache: the scheduled program of a gate list (fusion, pass and
// round selection, encoding: milliseconds for large circuits) keyed by a hash
// of the gate records and the options.  Small LRU, shared by all handles.
namespace {
struct ProgKey {
  uint64_t a, b;
  bool operator==(const ProgKey& o) const { return a == o.a && b == o.b; }
};
struct ProgKeyHash {
  size_t operator()(const ProgKey& k) const { return (size_t)(k.a ^ (k.b * 0x9E3779B97F4A7C15ull)); }
};
std::mutex g_prog_mu;
std::list<std::pair<ProgKey, std::shared_ptr<const void>>> g_prog_lru;
std::unordered_map<ProgKey, decltype(g_prog_lru)::iterator, ProgKeyHash> g_prog_idx;
constexpr size_t kProgCacheEntries = 32;

// 128-bit key of the gate records: four independent multiply-rotate lanes
// over 32-byte blocks (the hash runs on every apply: ~0.6 MB for QFT-30, so
// it must be memory-speed, not a serial FNV chain)
ProgKey prog_key(const void* data, size_t n, uint64_t salt) {
  const unsigned char* p = static_cast<const unsigned char*>(data);
  uint64_t h[4] = {0x9E3779B97F4A7C15ull ^ salt, 0xC2B2AE3D27D4EB4Full + salt, 0x165667B19E3779F9ull,
                   0x27D4EB2F165667C5ull ^ (salt << 1)};
  auto mix = [](uint64_t x, uint64_t w) {
    x ^= w * 0x87C37B91114253D5ull;
    x = (x << 31) | (x >> 33);
    return x * 0x4CF5AD432745937Full;
  };
  size_t i = 0;
  for (; i + 32 <= n; i += 32) {
    uint64_t w[4];
    std::memcpy(w, p + i, 32);
    for (int l = 0; l < 4; ++l) h[l] = mix(h[l], w[l]);
  }
  for (int l = 0; i < n; i += 8, ++l) {
    uint64_t w = 0;
    std::memcpy(&w, p + i, std::min<size_t>(8, n - i));
    h[l & 3] = mix(h[l & 3], w);
  }
  ProgKey k{h[0] ^ (h[2] * 0x9E3779B97F4A7C15ull) ^ n, h[1] ^ (h[3] * 0xC2B2AE3D27D4EB4Full) ^ (n << 7)};
  k.a ^= k.a >> 29;
  k.b ^= k.b >> 31;
  return k;
}
}  // namespace

template <typename R>
static Program cached_program(int n, const svb_gate* g, int ng, const SchedOptions& opt) {
  const uint64_t salt = (uint64_t)n | ((uint64_t)sizeof(R) << 8) | ((uint64_t)opt.rb << 16) |
                        ((uint64_t)opt.m << 24) | ((uint64_t)opt.relabel_swaps << 32) |
                        ((uint64_t)opt.round_search << 33) | ((uint64_t)opt.zero_start << 34) |
                        ((uint64_t)opt.initial_perm << 35) | ((uint64_t)opt.structural << 36);
  const ProgKey key = prog_key(g, sizeof(svb_gate) * (size_t)ng, salt);
  {
    std::lock_guard<std::mutex> lk(g_prog_mu);
    auto it = g_prog_idx.find(key);
    if (it != g_prog_idx.end()) {
      g_prog_lru.splice(g_prog_lru.begin(), g_prog_lru, it->second);
      return *static_cast<const Program*>(it->second->second.get());
    }
  }
  auto prog = std::make_shared<const Program>(build_program<R>(n, g, ng, opt));
  std::lock_guard<std::mutex> lk(g_prog_mu);
  if (g_prog_idx.find(key) == g_prog_idx.end()) {
    g_prog_lru.emplace_front(key, prog);
    g_prog_idx[key] = g_prog_lru.begin();
    if (g_prog_lru.size() > kProgCacheEntries) {
      g_prog_idx.erase(g_prog_lru.back().first);
      g_prog_lru.pop_back();
    }
  }
  return *prog;
}

static bool trace_on() {
  static int on = -1;
  if (on < 0) on = std::getenv("SVB_TRACE") ? 1 : 0;
  return on == 1;
}
struct TraceTimer {
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  double lap() {
    auto t1 = std::chrono::steady_clock::now();
    double ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
    t0 = t1;
    return ms;
  }
};

template <typename R>
void run_program_owned(void** state, void** spare, int n, const svb_gate* g, int ng, int fusion, int jit_min_n,
                       cudaStream_t st, ProgramStats* stats, bool* zero_pending, ZRequest* z) {
  TraceTimer tt;
  stats->gates += ng;
  SchedOptions opt = default_options(sizeof(R) == 8 ? SVB_C128 : SVB_C64, n, jit_min_n >= 0 && n >= jit_min_n);
  auto write_zero = [&] {
    if (zero_pending && *zero_pending) {
      launch_zero<R>(*state, n, st);
      *zero_pending = false;
    }
  };
  if (!fusion || n < opt.rb + 5 || ng == 0) {
    write_zero();
    for (int i = 0; i < ng; ++i) {
      launch_gate_basic<R>(*state, n, g[i], st);
      stats->passes += 1;
      stats->launches += 1;
    }
    return;
  }
  // swap relabeling needs a second state-sized buffer for the final permutation;
  // it is allocated once per handle (lazily) and reused
  const double t_info = tt.lap();
  opt.zero_start = zero_pending && *zero_pending;
  Program prog = cached_program<R>(n, g, ng, opt);
  // fused <Z>: the last pass's value k -> logical qubit
  auto z_setup = [&](Program& pr) {
    if (!z || !z->want || pr.passes.empty()) return;
    PassDev& pd = pr.passes.back();
    const RoundDev& rd = pd.rounds[pd.nrounds - 1];
    const int RBv = pd.rb, nt = pd.m - pd.rb;
    if (RBv + nt + pd.nout + 1 > kZaccRows) return;
    std::vector<int> phys;
    for (int i = 0; i < RBv; ++i) phys.push_back(pd.pos[rd.reg_local[i]]);
    for (int b = 0; b < nt; ++b) phys.push_back(pd.pos[rd.thr_local[b]]);
    for (int j = 0; j < pd.nout; ++j) phys.push_back(pd.outpos[j]);
    z->logical.clear();
    for (int p : phys) z->logical.push_back(pr.final_perm.empty() ? p : pr.final_perm[p]);
    z->logical.push_back(-1);
    pd.zsum = 1;
    z->fused = true;
  };
  if (z) z->fused = false;
  if ((!prog.final_perm.empty() || !prog.init_perm.empty()) && *spare == nullptr) {
    if (state_malloc(spare, sizeof(cplx<R>) << n) != cudaSuccess) {
      cudaGetLastError();
      *spare = nullptr;
      opt.relabel_swaps = false;  // no room: swaps become in-tile permutation ops
      prog = build_program<R>(n, g, ng, opt);
    }
  }
  const double t_build = tt.lap();
  // the input's permutation into the layout that absorbs the swap relabeling:
  // folded into the first pass's loads when they stay coalesced, else a pass
  const bool perm_in = !prog.init_perm.empty() && *spare != nullptr && fuse_initial_permutation<R>(prog, n);
  if (!prog.init_perm.empty() && !perm_in) {
    write_zero();
    cplx<R>* s0 = static_cast<cplx<R>*>(*state);
    cplx<R>* sp0 = static_cast<cplx<R>*>(*spare);
    launch_permute<R>(&s0, &sp0, n, prog.init_perm, st, stats);
    *state = s0;
    *spare = sp0;
  }
  z_setup(prog);
  const bool zin = zero_pending && *zero_pending && !prog.passes.empty();
  if (prog.passes.empty()) write_zero();
  const uint64_t full = n == 64 ? ~0ull : (1ull << n) - 1;
  if (zin && (prog.support & full) != full)  // positions outside the passes' support are never written
    SVB_CUDA(cudaMemsetAsync(*state, 0, sizeof(cplx<R>) << n, st));
  launch_passes<R>(static_cast<cplx<R>*>(*state), (prog.perm_fused || perm_in) ? static_cast<cplx<R>*>(*spare) : nullptr,
                   n, prog, st, stats, jit_min_n >= 0 && n >= jit_min_n, zin, z && z->fused ? z->d_acc : nullptr);
  if (z && z->fused) {
    const PassDev& lp = prog.passes.back();
    // CTAs of the last pass (the launch shapes of launch_passes / jit_launch_passes)
    int dev = 0, nsm = 148;
    SVB_CUDA(cudaGetDevice(&dev));
    SVB_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    const uint64_t ncta = std::min<uint64_t>(1ull << lp.nout, (uint64_t)nsm * std::max(kDirectMinBlocks, direct_min_blocks()));  // upper bound
    const unsigned nv = (unsigned)z->logical.size();
    double* partial = z->d_out + kZaccRows;
    k_zsum_finish<<<dim3(nv, kZsumSlices), 256, 0, st>>>(z->d_acc, (uint32_t)ncta, 1u << (lp.m - lp.rb), lp.rb,
                                                          lp.m - lp.rb, lp.nout, partial);
    SVB_CHECK_LAUNCH();
    launch_sum_rows(partial, nv, kZsumSlices, z->d_out, st);
  }
  if (zin) *zero_pending = false;
  const double t_launch = tt.lap();
  if (perm_in) std::swap(*state, *spare);  // the first pass wrote the spare buffer
  if (prog.perm_fused) {
    std::swap(*state, *spare);  // the last pass wrote the permuted state into the spare buffer
  } else if (!prog.final_perm.empty()) {
    cplx<R>* s = static_cast<cplx<R>*>(*state);
    cplx<R>* sp = static_cast<cplx<R>*>(*spare);
    launch_permute<R>(&s, &sp, n, prog.final_perm, st, stats);
    *state = s;
    *spare = sp;
  }
  const double t_perm = tt.lap();
  if (trace_on())
    std::fprintf(stderr, "[svb] n=%d gates=%d passes=%zu memgetinfo=%.2fms build=%.2fms launch=%.2fms permute=%.2fms\n",
                 n, ng, prog.passes.size(), t_info, t_build, t_launch, t_perm);
}

template void run_program<float>(void*, int, const svb_gate*, int, int, int, cudaStream_t, ProgramStats*);
template void run_program<double>(void*, int, const svb_gate*, int, int, int, cudaStream_t, ProgramStats*);
template void run_program_owned<float>(void**, void**, int, const svb_gate*, int, int, int, cudaStream_t,
                                       ProgramStats*, bool*, ZRequest*);
template void run_program_owned<double>(void**, void**, int, const svb_gate*, int, int, int, cudaStream_t,
                                        ProgramStats*, bool*, ZRequest*);

}  // namespace svb

using namespace svb;

extern "C" {

// Schedule a gate program on the host only (no GPU needed): pass/round/op
// statistics for tests and the design notes.
int svb_plan(int n, int precision, const svb_gate* gates, int ng, int64_t* n_passes, int64_t* n_rounds,
             int64_t* op_bytes, int32_t* has_perm) {
  try {
    const bool zero_start = (precision & 0x100) != 0;  // flag bit: schedule for a lazy |0...0> input
    precision &= 0xff;
    SchedOptions o = default_options(precision, n, n >= kDefaultJitMinQubits);
    o.zero_start = zero_start;
    Program p = precision == SVB_C128 ? build_program<double>(n, gates, ng, o) : build_program<float>(n, gates, ng, o);
    int64_t r = 0;
    for (auto& pd : p.passes) r += pd.nrounds;
    *n_passes = (int64_t)p.passes.size();
    *n_rounds = r;
    *op_bytes = (int64_t)p.ops.size();
    // 1: final permutation pass, 2: fused into the last pass, 3: initial
    // permutation pass, 4: initial permutation fused into the first pass's loads
    bool in_fused = false;
    if (!p.init_perm.empty())
      in_fused = precision == SVB_C128 ? fuse_initial_permutation<double>(p, n) : fuse_initial_permutation<float>(p, n);
    *has_perm = !p.init_perm.empty() ? (in_fused ? 4 : 3) : p.final_perm.empty() ? 0 : (p.perm_fused ? 2 : 1);
    return SVB_OK;
  } catch (const Error& e) {
    set_last_error(e.what());
    return e.code;
  }
}

// CPU emulation of the fused program (same scheduler, same op interpreter);
// amps are complex128 in/out.  Test hook for the scheduler without a GPU.
int svb_emulate_apply(int n, int precision, const svb_gate* gates, int ng, double* amps, int relabel) {
  try {
    SchedOptions o = default_options(precision, n, n >= kDefaultJitMinQubits);
    o.relabel_swaps = relabel != 0;
    o.zero_start = relabel == 2;  // caller passes |0...0> (lazy-zero layout choice)
    uint64_t len = 1ull << n;
    if (precision == SVB_C128) {
      Program p = build_program<double>(n, gates, ng, o);
      emulate_program<double>(reinterpret_cast<double2*>(amps), n, p);
    } else {
      Program p = build_program<float>(n, gates, ng, o);
      std::vector<float2> s(len);
      for (uint64_t i = 0; i < len; ++i) s[i] = make_float2((float)amps[2 * i], (float)amps[2 * i + 1]);
      emulate_program<float>(s.data(), n, p);
      for (uint64_t i = 0; i < len; ++i) { amps[2 * i] = s[i].x; amps[2 * i + 1] = s[i].y; }
    }
    return SVB_OK;
  } catch (const Error& e) {
    set_last_error(e.what());
    return e.code;
  }
}

}  // extern "C"
