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
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "kernels.h"
#include "program.h"

namespace svb {

// ------------------------------------------------ TMA bulk / mbarrier PTX
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}\n" ::"r"(
          smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(smem_dst)), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async8(void* smem_dst, const void* gsrc) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(smem_dst)), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N> __device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

constexpr int kStages = 2;

template <typename R> __host__ __device__ constexpr uint32_t tile_bytes_of(int m) { return (uint32_t)sizeof(cplx<R>) << m; }

// Tile base (bits outside S) computed warp-parallel: lane l owns tile bit l.
__device__ __forceinline__ uint64_t tile_base_warp(const PassDev& pd, uint64_t t, uint32_t lane) {
  uint64_t v = 0;
  if ((int)lane < pd.nout && ((t >> lane) & 1ull)) v = 1ull << pd.outpos[lane];
  if ((int)lane + 32 < pd.nout && ((t >> (lane + 32)) & 1ull)) v |= 1ull << pd.outpos[lane + 32];
  const uint32_t lo = __reduce_or_sync(0xffffffffu, (uint32_t)v);
  const uint32_t hi = __reduce_or_sync(0xffffffffu, (uint32_t)(v >> 32));
  return ((uint64_t)hi << 32) | lo;
}

template <typename R> __device__ __forceinline__ cplx<R> shfl_xor_c(cplx<R> x, int o) {
  x.x = __shfl_xor_sync(0xffffffffu, x.x, o);
  x.y = __shfl_xor_sync(0xffffffffu, x.y, o);
  return x;
}

// Tile-uniform factors of one DIAG payload, lanes in parallel over the terms.
template <typename R, int RB>
__device__ void diag_uniform_warp(const uint8_t* payload, uint64_t base, cplx<R>* slot, uint32_t lane) {
  const int4 h0 = reinterpret_cast<const int4*>(payload)[0];
  const int4 h1 = reinterpret_cast<const int4*>(payload)[1];
  const int nur[6] = {h0.x, h0.y, h0.z, h0.w, h1.x, h1.y};
  const int nuc = h1.z;
  const DiagTerm<R>* t = reinterpret_cast<const DiagTerm<R>*>(payload + sizeof(DiagHdr));
  const cplx<R> one = mk<R>(R(1), R(0));
  for (int i = 0; i < RB; ++i) {
    const int n = nur[i];
    cplx<R> u0 = one, u1 = one;
    if (n > 0) {
      for (int k = (int)lane; k < n; k += 32) {
        const int qb = t[k].qb;
        const int f = qb >= 0 ? (int)((base >> qb) & 1ull) : 0;
        u0 = cmul<R>(u0, t[k].d[2 * f]);
        u1 = cmul<R>(u1, t[k].d[2 * f + 1]);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        u0 = cmul<R>(u0, shfl_xor_c<R>(u0, o));
        u1 = cmul<R>(u1, shfl_xor_c<R>(u1, o));
      }
    }
    if (lane == 0) {
      slot[1 + i] = u0;
      slot[1 + 5 + i] = u1;
    }
    t += n;
  }
  cplx<R> c = one;
  if (nuc > 0) {
    for (int k = (int)lane; k < nuc; k += 32) {
      const int qa = t[k].qa, qb = t[k].qb;
      const int fa = qa >= 0 ? (int)((base >> qa) & 1ull) : 0, fb = qb >= 0 ? (int)((base >> qb) & 1ull) : 0;
      c = cmul<R>(c, t[k].d[fa + 2 * fb]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c = cmul<R>(c, shfl_xor_c<R>(c, o));
  }
  if (lane == 0) slot[0] = c;
}

// Persistent fused pass: one CTA per SM walks tiles blockIdx.x, +gridDim.x, ...
// Tiles stream HBM -> shared memory with cp.async (LDGSTS, 16 B per thread,
// lanes on consecutive amplitudes: 512 B per warp request) kStages-1 tiles
// ahead into an XOR-swizzled ring; warps first evaluate the tile-uniform
// factors of the pass's diagonal ops, then run the tile's rounds out of shared
// memory; the last round stores straight from registers to HBM (lanes <->
// qubits 0..4).  The swizzle is GF(2)-linear, so every shared-memory slot is
// an XOR of a per-thread base and per-register-bit offsets.
template <typename R, int RB>
__global__ void __launch_bounds__(256, 1)
    k_pass(cplx<R>* __restrict__ state, const PassDev* __restrict__ pdg, const uint8_t* __restrict__ ops_g,
           uint32_t ntiles) {
  extern __shared__ __align__(128) unsigned char smraw[];
  __shared__ PassDev pd;
  __shared__ cplx<R> uni[kMaxDiag * kUniStride];
  __shared__ uint64_t s_ldk[32];
  __shared__ uint32_t s_sdk[32];
  {
    const int4* src = reinterpret_cast<const int4*>(pdg);
    int4* dst = reinterpret_cast<int4*>(&pd);
    for (int i = threadIdx.x; i < (int)(sizeof(PassDev) / 16); i += blockDim.x) dst[i] = __ldg(src + i);
  }
  __syncthreads();
  // stage this pass's op stream after the tile ring; `ops` is rebased so that
  // stream offsets index shared memory
  const uint32_t ring_bytes = (uint32_t)kStages * ((uint32_t)sizeof(cplx<R>) << pd.m);
  {
    const int4* src = reinterpret_cast<const int4*>(ops_g + pd.ops_begin);
    int4* dst = reinterpret_cast<int4*>(smraw + ring_bytes);
    for (uint32_t i = threadIdx.x; i < pd.ops_bytes / 16; i += blockDim.x) dst[i] = __ldg(src + i);
  }
  const uint8_t* ops = smraw + ring_bytes - pd.ops_begin;
  __syncthreads();
  constexpr int V = 1 << RB;
  constexpr int kHoist = 4;  // rounds whose thread constants live in registers
  const uint32_t tid = threadIdx.x, nthr = blockDim.x, lane = tid & 31u, warp = tid >> 5;
  const uint32_t nwarps = nthr >> 5;
  const int m = pd.m, nrounds = pd.nrounds, ndiag = pd.ndiag;
  const uint32_t T = 1u << m;
  cplx<R>* ring = reinterpret_cast<cplx<R>*>(smraw);
  // loads: element j = (tid + k*nthr)*kPer; 16 B per copy (one c128 amplitude
  // or an aligned c64 pair); global and smem offsets split into a tid part and
  // a tile-independent k part (tables in shared memory)
  constexpr int kPer = sizeof(cplx<R>) == 16 ? 1 : 2;
  const int lo_bits = (31 - __clz(nthr)) + (kPer == 2 ? 1 : 0);
  uint64_t ld_tid = 0;
  for (int l = 0; l < lo_bits; ++l)
    if (((tid * kPer) >> l) & 1u) ld_tid |= 1ull << pd.pos[l];
  const uint32_t sd_tid = swz<R>(tid * kPer);
  const uint32_t nld = T / (nthr * kPer);
  if (tid < nld) {
    uint64_t g = 0;
    const uint32_t j = tid * nthr * kPer;
    for (int l = lo_bits; l < m; ++l)
      if ((j >> l) & 1u) g |= 1ull << pd.pos[l];
    s_ldk[tid] = g;
    s_sdk[tid] = swz<R>(j);
  }
  __syncthreads();
  uint32_t sFl_r[kHoist];
  uint64_t Fg_r[kHoist];
#pragma unroll
  for (int k = 0; k < kHoist; ++k) {
    if (k < nrounds) {
      uint32_t Fl;
      thread_fixed(pd, pd.rounds[k], tid, 0, &Fl, &Fg_r[k]);
      sFl_r[k] = swz<R>(Fl);
    }
  }
  auto issue = [&](uint64_t base, int b) {
    cplx<R>* dst = ring + (size_t)b * T;
    const cplx<R>* src = state + (base | ld_tid);
    // swizzle is linear over XOR: slot(tid part ^ k part) = swz(tid part) ^ swz(k part)
    for (uint32_t k = 0; k < nld; ++k) cp_async16(dst + (sd_tid ^ s_sdk[k]), src + s_ldk[k]);
  };
  const uint32_t t0 = blockIdx.x;
#pragma unroll
  for (int s = 0; s < kStages - 1; ++s) {
    const uint32_t ts = t0 + (uint32_t)s * gridDim.x;
    if (ts < ntiles) issue(tile_base_warp(pd, ts, lane), s);
    cp_async_commit();
  }
  cplx<R> a[V];
  int it = 0;
  for (uint32_t t = t0; t < ntiles; t += gridDim.x, ++it) {
    const uint32_t tn = t + (uint32_t)(kStages - 1) * gridDim.x;
    if (tn < ntiles) issue(tile_base_warp(pd, tn, lane), (it + kStages - 1) % kStages);
    cp_async_commit();
    const uint64_t base = tile_base_warp(pd, t, lane);
    if (ndiag > 0) {  // tile-uniform diagonal factors (before the ring wait: overlaps the copies)
      for (int d = (int)warp; d < ndiag; d += (int)nwarps)
        diag_uniform_warp<R, RB>(ops + pd.diag_off[d], base, uni + d * kUniStride, lane);
    }
    cp_async_wait<kStages - 1>();
    __syncthreads();
    cplx<R>* cur = ring + (size_t)(it % kStages) * T;
    for (int k = 0; k < nrounds; ++k) {
      const RoundDev& rd = pd.rounds[k];
      uint32_t sFl;
      uint64_t Fg;
      if (k < kHoist) {
#pragma unroll
        for (int q = 0; q < kHoist; ++q)
          if (q == k) { sFl = sFl_r[q]; Fg = Fg_r[q] | base; }
      } else {
        uint32_t Fl;
        thread_fixed(pd, rd, tid, base, &Fl, &Fg);
        sFl = swz<R>(Fl);
      }
      uint32_t sl[RB];
#pragma unroll
      for (int i = 0; i < RB; ++i) sl[i] = swz<R>(1u << rd.reg_local[i]);
      uint32_t slot[V];
      slot[0] = sFl;
#pragma unroll
      for (int i = 0; i < RB; ++i)
#pragma unroll
        for (int v = 0; v < (1 << i); ++v) slot[v | (1 << i)] = slot[v] ^ sl[i];
#pragma unroll
      for (int v = 0; v < V; ++v) a[v] = cur[slot[v]];
      run_ops<R, RB>(a, Fg, ops, rd.op_off, rd.op_end, uni);
      if (k + 1 < nrounds) {
        // each slot of a layout is read and rewritten by its owner only, so one
        // barrier (after the writes) separates consecutive layouts
#pragma unroll
        for (int v = 0; v < V; ++v) cur[slot[v]] = a[v];
        __syncthreads();
      } else {
        cplx<R>* g0 = state + Fg;
        size_t goff[RB];
#pragma unroll
        for (int i = 0; i < RB; ++i) goff[i] = (size_t)1 << pd.pos[rd.reg_local[i]];
        size_t gv[V];
        gv[0] = 0;
#pragma unroll
        for (int i = 0; i < RB; ++i)
#pragma unroll
          for (int v = 0; v < (1 << i); ++v) gv[v | (1 << i)] = gv[v] | goff[i];
#pragma unroll
        for (int v = 0; v < V; ++v) __stcs(g0 + gv[v], a[v]);
      }
    }
    __syncthreads();  // ring slot and uniform factors are rewritten next tile
  }
  cp_async_wait<0>();
}

// ---------------------------------------------------------------- permute
struct PermDev {
  int32_t n, ml;        // tile local bits
  int32_t lin[12];      // input bit of local bit l (ascending)
  int32_t lout_src[12]; // output-local bit e (ascending output positions) -> input-local bit
  int32_t lout_pos[12]; // output bit of output-local bit e
  int32_t nout;
  int32_t outin[48];    // input bits outside the tile, ascending
  int32_t dest[64];     // output bit of input bit p
};

template <typename R>
__global__ void __launch_bounds__(256) k_permute(const cplx<R>* __restrict__ in, cplx<R>* __restrict__ out,
                                                 PermDev pd) {
  extern __shared__ __align__(16) unsigned char smraw[];
  cplx<R>* sm = reinterpret_cast<cplx<R>*>(smraw);
  const uint64_t t = blockIdx.x;
  uint64_t bin = 0, bout = 0;
  for (int i = 0; i < pd.nout; ++i)
    if ((t >> i) & 1ull) {
      bin |= 1ull << pd.outin[i];
      bout |= 1ull << pd.dest[pd.outin[i]];
    }
  const uint32_t T = 1u << pd.ml;
  for (uint32_t j = threadIdx.x; j < T; j += blockDim.x) {
    uint64_t g = bin;
    for (int l = 0; l < pd.ml; ++l)
      if ((j >> l) & 1u) g |= 1ull << pd.lin[l];
    sm[j] = __ldcs(in + g);
  }
  __syncthreads();
  for (uint32_t o = threadIdx.x; o < T; o += blockDim.x) {
    uint64_t g = bout;
    uint32_t j = 0;
    for (int e = 0; e < pd.ml; ++e)
      if ((o >> e) & 1u) {
        g |= 1ull << pd.lout_pos[e];
        j |= 1u << pd.lout_src[e];
      }
    __stcs(out + g, sm[j]);
  }
}

static PermDev make_perm(int n, const std::vector<int>& dest) {
  PermDev pd{};
  pd.n = n;
  uint64_t inset = 0x1full;
  for (int p = 0; p < n; ++p)
    if (dest[p] < 5) inset |= 1ull << p;
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
void Profiler::begin(cudaStream_t st, int kind, double nbytes) {
  Rec r;
  SVB_CUDA(cudaEventCreate(&r.a));
  SVB_CUDA(cudaEventCreate(&r.b));
  r.kind = kind;
  SVB_CUDA(cudaEventRecord(r.a, st));
  pending.push_back(r);
  bytes[kind] += nbytes;
}
void Profiler::end(cudaStream_t st) { SVB_CUDA(cudaEventRecord(pending.back().b, st)); }
void Profiler::collect() {
  for (Rec& r : pending) {
    float t = 0.f;
    SVB_CUDA(cudaEventSynchronize(r.b));
    SVB_CUDA(cudaEventElapsedTime(&t, r.a, r.b));
    ms[r.kind] += t;
    count[r.kind] += 1;
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  pending.clear();
}

// ------------------------------------------------------------ run_program
template <typename R> static constexpr int rb_of() { return sizeof(R) == 8 ? 4 : 5; }

template <typename R>
static void launch_passes(cplx<R>* state, int n, const Program& prog, cudaStream_t st, ProgramStats* stats) {
  constexpr int RB = rb_of<R>();
  if (prog.passes.empty()) return;
  size_t pbytes = prog.passes.size() * sizeof(PassDev);
  size_t obytes = std::max<size_t>(prog.ops.size(), 16);
  uint8_t* dbuf = nullptr;
  SVB_CUDA(cudaMallocAsync(&dbuf, pbytes + obytes, st));
  SVB_CUDA(cudaMemcpyAsync(dbuf, prog.passes.data(), pbytes, cudaMemcpyHostToDevice, st));
  if (!prog.ops.empty())
    SVB_CUDA(cudaMemcpyAsync(dbuf + pbytes, prog.ops.data(), prog.ops.size(), cudaMemcpyHostToDevice, st));
  const PassDev* dpass = reinterpret_cast<const PassDev*>(dbuf);
  const uint8_t* dops = dbuf + pbytes;
  size_t smem = 0;
  for (const PassDev& pd : prog.passes)
    smem = std::max(smem, kStages * (size_t)tile_bytes_of<R>(pd.m) + pd.ops_bytes);
  SVB_CUDA(cudaFuncSetAttribute(k_pass<R, RB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int dev = 0, nsm = 148;
  SVB_CUDA(cudaGetDevice(&dev));
  SVB_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  for (size_t p = 0; p < prog.passes.size(); ++p) {
    const PassDev& pd = prog.passes[p];
    uint64_t tiles = 1ull << pd.nout;
    unsigned threads = 1u << (pd.m - RB);
    unsigned grid = (unsigned)std::min<uint64_t>(tiles, (uint64_t)nsm);
    Profiler* pf = (stats->prof && stats->prof->on) ? stats->prof : nullptr;
    if (pf) pf->begin(st, 0, 2.0 * (double)(sizeof(cplx<R>) << n));
    k_pass<R, RB><<<grid, threads, kStages * (size_t)tile_bytes_of<R>(pd.m) + pd.ops_bytes, st>>>(
        state, dpass + p, dops, (uint32_t)tiles);
    SVB_CHECK_LAUNCH();
    if (pf) pf->end(st);
    stats->passes += 1;
    stats->launches += 1;
  }
  SVB_CUDA(cudaFreeAsync(dbuf, st));
}

template <typename R>
static void launch_permute(cplx<R>** state, cplx<R>** spare, int n, const std::vector<int>& dest, cudaStream_t st,
                           ProgramStats* stats) {
  PermDev pd = make_perm(n, dest);
  cplx<R>* out = *spare;
  size_t bytes = sizeof(cplx<R>) << n;
  uint64_t tiles = 1ull << pd.nout;
  Profiler* pf = (stats->prof && stats->prof->on) ? stats->prof : nullptr;
  if (pf) pf->begin(st, 1, 2.0 * (double)bytes);
  k_permute<R><<<(unsigned)tiles, 256, sizeof(cplx<R>) << pd.ml, st>>>(*state, out, pd);
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
  launch_passes<R>(static_cast<cplx<R>*>(state), n, prog, st, stats);
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
void run_program_owned(void** state, void** spare, int n, const svb_gate* g, int ng, int fusion, cudaStream_t st,
                       ProgramStats* stats) {
  TraceTimer tt;
  stats->gates += ng;
  SchedOptions opt = default_options(sizeof(R) == 8 ? SVB_C128 : SVB_C64, n);
  if (!fusion || n < opt.rb + 5) {
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
  Program prog = build_program<R>(n, g, ng, opt);
  if (!prog.final_perm.empty() && *spare == nullptr) {
    if (cudaMalloc(spare, sizeof(cplx<R>) << n) != cudaSuccess) {
      cudaGetLastError();
      *spare = nullptr;
      opt.relabel_swaps = false;  // no room: swaps become in-tile permutation ops
      prog = build_program<R>(n, g, ng, opt);
    }
  }
  const double t_build = tt.lap();
  launch_passes<R>(static_cast<cplx<R>*>(*state), n, prog, st, stats);
  const double t_launch = tt.lap();
  if (!prog.final_perm.empty()) {
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
template void run_program_owned<float>(void**, void**, int, const svb_gate*, int, int, cudaStream_t, ProgramStats*);
template void run_program_owned<double>(void**, void**, int, const svb_gate*, int, int, cudaStream_t, ProgramStats*);

}  // namespace svb

using namespace svb;

extern "C" {

// Schedule a gate program on the host only (no GPU needed): pass/round/op
// statistics for tests and the design notes.
int svb_plan(int n, int precision, const svb_gate* gates, int ng, int64_t* n_passes, int64_t* n_rounds,
             int64_t* op_bytes, int32_t* has_perm) {
  try {
    SchedOptions o = default_options(precision, n);
    Program p = precision == SVB_C128 ? build_program<double>(n, gates, ng, o) : build_program<float>(n, gates, ng, o);
    int64_t r = 0;
    for (auto& pd : p.passes) r += pd.nrounds;
    *n_passes = (int64_t)p.passes.size();
    *n_rounds = r;
    *op_bytes = (int64_t)p.ops.size();
    *has_perm = p.final_perm.empty() ? 0 : 1;
    return SVB_OK;
  } catch (const Error& e) {
    return e.code;
  }
}

// CPU emulation of the fused program (same scheduler, same op interpreter);
// amps are complex128 in/out.  Test hook for the scheduler without a GPU.
int svb_emulate_apply(int n, int precision, const svb_gate* gates, int ng, double* amps, int relabel) {
  try {
    SchedOptions o = default_options(precision, n);
    o.relabel_swaps = relabel != 0;
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
    return e.code;
  }
}

}  // extern "C"
