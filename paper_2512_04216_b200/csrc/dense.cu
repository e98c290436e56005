// Dense k-qubit block passes (north_star item 3, SURVEY §7 step 7 "K6"):
// apply one dense 2^k x 2^k complex matrix U to qubits q[0..k) of the state
// in one HBM pass (read + write the state once).
//
// The state is viewed as 2^(n-k) columns x 2^k rows: column c holds the 2^k
// amplitudes that differ only in the block qubits, y_c = U x_c (local index
// bit i <-> q[i], the svb_gate convention of gates.py:3-5).  A CTA stages a
// tile of 128 columns (2^(k+7) amplitudes: the block qubits plus the 7 lowest
// other qubits, so warps read 256 contiguous bytes) in shared memory.
//
// * k_dense_tc (complex64, 3 <= k <= 5; k_dense_tc6 for k = 6, with the
//   unitary as the TMEM operand): the block is a real GEMM on the
//   5th-generation tensor cores.  With x in interleaved real form
//   (x_re, x_im per amplitude) D[c][2i+e] = sum_kk A[c][kk] * B[2i+e][kk],
//   A = the tile (M = 128 columns, K = 2^(k+1)), B = U in real form
//   (N = K).  kind::tf32 with a 4-term TF32 split (A_lo B_lo + A_lo B_hi +
//   A_hi B_lo + A_hi B_hi, small terms first; hi = x rounded to TF32, lo =
//   x - hi rounded to TF32) keeps ~2^-21 relative
//   accuracy per block, inside complex64's 1e-5 (TF32 alone would miss it).
//   One thread issues tcgen05.mma from shared-memory descriptors (canonical
//   K-major, no swizzle; the K-chunk stride is padded by 16 B so the tile
//   writes are bank-conflict free), the accumulator lives in TMEM
//   (128 lanes x 2^(k+1) fp32 columns) and returns through tcgen05.ld.
//   The next tile's loads are issued before the MMA wait, so HBM traffic
//   overlaps the tensor work and the epilogue.
// * k_dense_fma (either precision, 1 <= k <= 6): the same tile staging with
//   the products on the FP32/FP64 FMA pipes: the CUDA-core path for small or
//   complex128 blocks, and the baseline the tensor path is measured against.
//
// Roofline: 2*s*2^n bytes per pass; 8*2^k flop per amplitude
// (complex MAC) on CUDA cores, 3*8*2^k TF32 flop on tensor cores.  complex64
// leaves the HBM roofline on CUDA cores at k = 5 (128 FFMA per amplitude),
// where the tensor path stays HBM-bound.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "kernels.h"

namespace svb {

constexpr int kDenseCols = 128;  // columns per tile (= UMMA M)
constexpr int kDenseMaxK = 6;
constexpr int kTcMaxK = 6;

struct DenseGeom {
  int k = 0;          // block qubits
  int kb = 0;         // tile bits = k + 7
  int nout = 0;       // qubits outside the tile
  int8_t tq[kDenseMaxK + 12] = {};   // qubit of tile position b (ascending)
  uint32_t sb[kDenseMaxK + 12] = {};  // shared-memory byte contribution of tile position b
  int8_t outq[48] = {};              // qubits outside the tile, ascending
};

// ------------------------------------------------------------ tcgen05 PTX
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  // SWIZZLE_NONE K-major canonical layout: core matrices of 8 rows x 16 B,
  // rows 16 B apart, row groups SBO apart, the two K chunks LBO apart;
  // version 1 (bits 46-47) for sm_100
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}

__device__ __forceinline__ void umma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }

// 16 consecutive fp32 accumulator columns of this thread's TMEM lane
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// round to the nearest TF32 (ties away): unbiased hi / lo split, and a lo part
// the tensor core then reads exactly (its own conversion truncates, which
// would bias every product toward zero and decay the norm block by block)
__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// Per-CTA constants in shared memory: the tile-base deposit tables (tile
// index -> amplitude offset of the bits outside the tile, 8 index bits per
// table: base = sum of 4 lookups) and the element-offset tables.
struct DenseSmemHdr {
  uint64_t tb[4][256];
};

__device__ __forceinline__ void dense_tile_tables(const DenseGeom& g, DenseSmemHdr* h) {
  for (int e = threadIdx.x; e < 4 * 256; e += blockDim.x) {
    const int c = e >> 8, v = e & 255;
    uint64_t b = 0;
    for (int j = 0; j < 8; ++j)
      if (((v >> j) & 1) && 8 * c + j < g.nout) b |= 1ull << g.outq[8 * c + j];
    h->tb[c][v] = b;
  }
}
__device__ __forceinline__ uint64_t dense_tile_base(const DenseSmemHdr* h, uint64_t t) {
  return h->tb[0][t & 255] + h->tb[1][(t >> 8) & 255] + h->tb[2][(t >> 16) & 255] + h->tb[3][(t >> 24) & 255];
}

// per-thread constant part of the element offsets (element e = it * NT + tid)
template <int NT>
__device__ __forceinline__ void dense_thread_offsets(const DenseGeom& g, uint32_t tid, uint64_t& goff,
                                                     uint32_t& soff) {
  goff = 0;
  soff = 0;
  constexpr int lb = NT == 128 ? 7 : 8;
  for (int b = 0; b < lb; ++b)
    if ((tid >> b) & 1u) {
      goff += 1ull << g.tq[b];
      soff += g.sb[b];
    }
}

// it-part of the offsets, one table entry per element slot
template <int NT>
__device__ __forceinline__ void dense_it_tables(const DenseGeom& g, int ept, uint64_t* git, uint32_t* sit) {
  constexpr int lb = NT == 128 ? 7 : 8;
  for (int it = threadIdx.x; it < ept; it += NT) {
    uint64_t go = 0;
    uint32_t so = 0;
    for (int b = lb; b < g.kb; ++b)
      if ((it >> (b - lb)) & 1) {
        go += 1ull << g.tq[b];
        so += g.sb[b];
      }
    git[it] = go;
    sit[it] = so;
  }
}

constexpr int kTcThreads = 128;

// smem: [hdr | Ahi | Alo | Bhi | Blo | git | sit | bar | tmem slot]
// Two register sets of the tile (cur / nxt): tile t + grid is loaded at the
// top of tile t's iteration, a whole iteration ahead of its use.
template <int K>
__global__ void __launch_bounds__(kTcThreads, 2)
    k_dense_tc(float2* __restrict__ state, const float* __restrict__ bsrc, const DenseGeom g, uint64_t ntiles,
               uint32_t chunk_stride) {
  constexpr int KR = 2 << K;             // real K = N
  constexpr int EPT = (1 << (K + 7)) / kTcThreads;  // elements per thread
  constexpr int NCH = KR / 4;            // 16-byte K chunks
  extern __shared__ __align__(1024) uint8_t smem[];
  DenseSmemHdr* hdr = reinterpret_cast<DenseSmemHdr*>(smem);
  const uint32_t abytes = NCH * chunk_stride;
  uint8_t* ahi = smem + sizeof(DenseSmemHdr);
  uint8_t* alo = ahi + abytes;
  uint8_t* bhi = alo + abytes;
  uint8_t* blo = bhi + KR * KR * 4;
  uint64_t* git = reinterpret_cast<uint64_t*>(blo + KR * KR * 4);
  uint32_t* sit = reinterpret_cast<uint32_t*>(git + EPT);
  uint64_t* bar = reinterpret_cast<uint64_t*>(sit + EPT + (EPT & 1));
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 1);
  const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  constexpr uint32_t TCOLS = KR < 32 ? 32 : KR;

  // B operand (hi, lo: real-form U, K-major rows) from global, once per CTA
  for (int i = tid; i < 2 * KR * KR / 4; i += kTcThreads)
    reinterpret_cast<float4*>(bhi)[i] = reinterpret_cast<const float4*>(bsrc)[i];
  dense_it_tables<kTcThreads>(g, EPT, git, sit);
  dense_tile_tables(g, hdr);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tslot)),
                 "n"(TCOLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
  }
  if (tid == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  uint64_t goff;
  uint32_t soff;
  dense_thread_offsets<kTcThreads>(g, tid, goff, soff);
  // instruction descriptor: F32 accumulator, TF32 A and B, K-major both, N = KR, M = 128
  const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(KR >> 3) << 17) | ((128u >> 4) << 24);
  uint32_t phase = 0;

  auto load = [&](float2 (&v)[EPT], uint64_t t) {
    const uint64_t base = dense_tile_base(hdr, t) + goff;
#pragma unroll
    for (int i = 0; i < EPT; ++i) v[i] = __ldcs(state + base + git[i]);
  };
  auto step = [&](float2 (&cur)[EPT], float2 (&nxt)[EPT], uint64_t t) {
    const uint64_t base = dense_tile_base(hdr, t) + goff;
    if (t + gridDim.x < ntiles) load(nxt, t + gridDim.x);
    // A tile, split hi / lo
#pragma unroll
    for (int i = 0; i < EPT; ++i) {
      const float hx = tf32_rna(cur[i].x), hy = tf32_rna(cur[i].y);
      const uint32_t o = soff + sit[i];
      *reinterpret_cast<float2*>(ahi + o) = make_float2(hx, hy);
      *reinterpret_cast<float2*>(alo + o) = make_float2(tf32_rna(cur[i].x - hx), tf32_rna(cur[i].y - hy));
    }
    fence_proxy_async();
    __syncthreads();
    if (tid == 0) {
      tc_fence_after();
      const uint32_t a0 = smem_u32(ahi), a1 = smem_u32(alo), b0 = smem_u32(bhi), b1 = smem_u32(blo);
      // small terms first (lo*lo, lo*hi, hi*lo), hi*hi last: the accumulator
      // holds the small partial sums before the large one arrives
      const uint32_t as[4] = {a1, a1, a0, a0}, bs[4] = {b1, b0, b1, b0};
#pragma unroll
      for (int term = 0; term < 4; ++term)
#pragma unroll
        for (int s = 0; s < KR / 8; ++s) {
          const uint32_t ao = s * 2 * chunk_stride, bo = s * 2 * (KR * 16);
          umma_tf32(tmem, umma_desc(as[term] + ao, chunk_stride, 128), umma_desc(bs[term] + bo, KR * 16, 128),
                    idesc, (term | s) != 0);
        }
      umma_commit(bar);
    }
    mbar_wait(bar, phase);
    phase ^= 1u;
    tc_fence_after();
    // epilogue: row c = 32*warp + lane; columns 2i+e -> amplitude i of the column,
    // written back into the A-hi layout (16 B = two amplitudes per chunk)
    {
      const uint32_t c = 32 * warp + lane;
#pragma unroll
      for (int col = 0; col < KR; col += 16) {
        float y[16];
        tmem_ld16(tmem + ((32 * warp) << 16) + col, y);
#pragma unroll
        for (int q = 0; q < 4; ++q)
          *reinterpret_cast<float4*>(ahi + (uint32_t)(col / 4 + q) * chunk_stride + c * 16) =
              make_float4(y[4 * q], y[4 * q + 1], y[4 * q + 2], y[4 * q + 3]);
      }
    }
    tc_fence_before();
    __syncthreads();
#pragma unroll
    for (int i = 0; i < EPT; ++i)
      __stcs(state + base + git[i], *reinterpret_cast<const float2*>(ahi + soff + sit[i]));
    __syncthreads();
  };

  float2 va[EPT], vb[EPT];
  const uint64_t G = gridDim.x;
  if (blockIdx.x < ntiles) load(va, blockIdx.x);
  for (uint64_t t = blockIdx.x; t < ntiles; t += 2 * G) {
    step(va, vb, t);
    if (t + G < ntiles) step(vb, va, t + G);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(TCOLS) : "memory");
  }
}

// Pipelined variant (one CTA of 256 threads per SM): two A tiles and two
// TMEM accumulators, so the split of tile i+1 and its MMAs run while tile i
// is in its epilogue and stores, and the loads of tile i+2 are in flight.
//   iteration i:  split(i+1) -> A[(i+1)&1]; MMA(i+1) -> D[(i+1)&1] (async);
//                 load(i+2) -> registers; wait MMA(i); epilogue D[i&1] ->
//                 A[i&1]; store tile i.
constexpr int kTcpThreads = 256;

__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float* v) {
  uint32_t r[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}

template <int K>
__global__ void __launch_bounds__(kTcpThreads, 1)
    k_dense_tcp(float2* __restrict__ state, const float* __restrict__ bsrc, const DenseGeom g, uint64_t ntiles,
                uint32_t chunk_stride) {
  constexpr int KR = 2 << K;
  constexpr int EPT = (1 << (K + 7)) / kTcpThreads;
  constexpr int NCH = KR / 4;
  constexpr uint32_t TCOLS = 2 * KR < 32 ? 32 : 2 * KR;
  extern __shared__ __align__(1024) uint8_t smem[];
  DenseSmemHdr* hdr = reinterpret_cast<DenseSmemHdr*>(smem);
  const uint32_t abytes = NCH * chunk_stride;
  uint8_t* abuf = smem + sizeof(DenseSmemHdr);  // [slot][hi, lo]
  uint8_t* bhi = abuf + 4 * abytes;
  uint8_t* blo = bhi + KR * KR * 4;
  uint64_t* git = reinterpret_cast<uint64_t*>(blo + KR * KR * 4);
  uint32_t* sit = reinterpret_cast<uint32_t*>(git + EPT);
  uint64_t* bar = reinterpret_cast<uint64_t*>(sit + EPT + (EPT & 1));  // 2 mbarriers
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 2);
  const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, quad = warp & 3, half = warp >> 2;

  for (int i = tid; i < 2 * KR * KR / 4; i += kTcpThreads)
    reinterpret_cast<float4*>(bhi)[i] = reinterpret_cast<const float4*>(bsrc)[i];
  dense_it_tables<kTcpThreads>(g, EPT, git, sit);
  dense_tile_tables(g, hdr);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tslot)),
                 "n"(TCOLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
  }
  if (tid == 0) {
    mbar_init(bar, 1);
    mbar_init(bar + 1, 1);
    fence_mbar_init();
  }
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  uint64_t goff;
  uint32_t soff;
  dense_thread_offsets<kTcpThreads>(g, tid, goff, soff);
  const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(KR >> 3) << 17) | ((128u >> 4) << 24);
  const uint64_t G = gridDim.x;
  uint32_t phase[2] = {0, 0};

  auto ahi = [&](int b) { return abuf + (2 * b) * abytes; };
  auto alo = [&](int b) { return abuf + (2 * b + 1) * abytes; };
  auto load = [&](float2 (&v)[EPT], uint64_t t) {
    const uint64_t base = dense_tile_base(hdr, t) + goff;
#pragma unroll
    for (int i = 0; i < EPT; ++i) v[i] = __ldcs(state + base + git[i]);
  };
  auto split = [&](const float2 (&v)[EPT], int b) {
    uint8_t* h = ahi(b);
    uint8_t* l = alo(b);
#pragma unroll
    for (int i = 0; i < EPT; ++i) {
      const float hx = tf32_rna(v[i].x), hy = tf32_rna(v[i].y);
      const uint32_t o = soff + sit[i];
      *reinterpret_cast<float2*>(h + o) = make_float2(hx, hy);
      *reinterpret_cast<float2*>(l + o) = make_float2(tf32_rna(v[i].x - hx), tf32_rna(v[i].y - hy));
    }
  };
  auto mma = [&](int b) {  // one thread
    tc_fence_after();
    const uint32_t a0 = smem_u32(ahi(b)), a1 = smem_u32(alo(b)), b0 = smem_u32(bhi), b1 = smem_u32(blo);
    const uint32_t as[4] = {a1, a1, a0, a0}, bs[4] = {b1, b0, b1, b0};
    const uint32_t d = tmem + b * KR;
#pragma unroll
    for (int term = 0; term < 4; ++term)
#pragma unroll
      for (int s = 0; s < KR / 8; ++s)
        umma_tf32(d, umma_desc(as[term] + s * 2 * chunk_stride, chunk_stride, 128),
                  umma_desc(bs[term] + s * 2 * (KR * 16), KR * 16, 128), idesc, (term | s) != 0);
    umma_commit(bar + b);
  };
  auto finish = [&](uint64_t t, int b) {  // wait MMA(b), epilogue, store tile t
    mbar_wait(bar + b, phase[b]);
    phase[b] ^= 1u;
    tc_fence_after();
    const uint32_t c = 32 * quad + lane;
    uint8_t* h = ahi(b);
    constexpr int HALF = KR / 2;
#pragma unroll
    for (int col = 0; col < HALF; col += 8) {
      const int cc = half * HALF + col;
      float y[8];
      tmem_ld8(tmem + b * KR + ((32 * quad) << 16) + cc, y);
#pragma unroll
      for (int q = 0; q < 2; ++q)
        *reinterpret_cast<float4*>(h + (uint32_t)(cc / 4 + q) * chunk_stride + c * 16) =
            make_float4(y[4 * q], y[4 * q + 1], y[4 * q + 2], y[4 * q + 3]);
    }
    tc_fence_before();
    __syncthreads();
    const uint64_t base = dense_tile_base(hdr, t) + goff;
#pragma unroll
    for (int i = 0; i < EPT; ++i)
      __stcs(state + base + git[i], *reinterpret_cast<const float2*>(h + soff + sit[i]));
  };

  float2 va[EPT], vb[EPT];
  uint64_t t = blockIdx.x;
  if (t >= ntiles) {
    tc_fence_before();
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(TCOLS));
    return;
  }
  // prologue: tile t into slot 0, its MMAs in flight, loads of t + G
  load(va, t);
  split(va, 0);
  fence_proxy_async();
  __syncthreads();
  if (tid == 0) mma(0);
  if (t + G < ntiles) load(vb, t + G);
  int b = 0;
  for (; t < ntiles; t += G) {
    const uint64_t tn = t + G;
    if (tn < ntiles) {  // split + MMA of the next tile while this one drains
      split(vb, b ^ 1);
      fence_proxy_async();
      __syncthreads();
      if (tid == 0) mma(b ^ 1);
      if (tn + G < ntiles) load(vb, tn + G);
    }
    finish(t, b);
    __syncthreads();  // slot b is split into again two tiles later
    b ^= 1;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(TCOLS) : "memory");
  }
}

// ------------------------------------------- TMA-staged tensor-core pass
// The tile is a box of a <= 5-dimensional tensor-map view of the state: one
// dimension per run of tile qubits (<= 8 qubits each), each spanning up to
// the next run, so the tile's other bits are the box coordinates; tile
// pieces beyond five become extra copies.  Tiles land in a ring of raw slots
// (natural tile order) by cp.async.bulk.tensor, one elected thread keeping
// kTmaSlots tiles in flight (no registers hold prefetched data); the threads
// split each raw tile into the TF32 hi / lo A operand, one thread issues the
// MMAs, the epilogue writes the results back into the raw slot in natural
// order and the same tensor map stores it (bulk async store).
constexpr int kTmaThreads = 256, kTmaSlots = 3, kTmaMaxCopies = 16;

struct TmaGeom {
  int ncopy;                          // copies per tile (extra pieces enumerated)
  int32_t copy_c4[kTmaMaxCopies];     // dim-4 coordinate offset of each copy
  int8_t tdim[48];                    // tile-index bit b -> tensor dim
  int8_t tshift[48];                  // ... and the bit's position in that dim's coordinate
  int ntb;                            // tile-index bits
  uint32_t erow[128];                 // natural tile index of D row (state column) c
  uint32_t ecol[64];                  // natural tile index of block amplitude j
};

__device__ __forceinline__ void tma_load_5d(void* dst, const CUtensorMap* map, const int32_t* c, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], "
      "[%7];\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4]), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_store_5d(const CUtensorMap* map, const int32_t* c, const void* src) {
  asm volatile("cp.async.bulk.tensor.5d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4, %5}], [%6];\n" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4]), "r"(smem_u32(src))
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read1() { asm volatile("cp.async.bulk.wait_group.read 1;\n" ::: "memory"); }

__device__ __forceinline__ void tma_coords(const TmaGeom& tg, uint64_t t, int32_t* c) {
  c[0] = c[1] = c[2] = c[3] = c[4] = 0;
  for (int b = 0; b < tg.ntb; ++b)
    if ((t >> b) & 1ull) c[tg.tdim[b]] += 1 << tg.tshift[b];
}

// Warp roles: warps 0-7 (256 threads) split tiles, issue the MMAs (thread 0)
// and run the epilogue; warp 8 is the TMA producer (loads and stores).  The
// roles meet only at mbarriers: full[s] (tile in slot s: TMA transaction
// bytes), done[s] (its results are back in slot s: 256 arrivals), mma.
template <int K>
__global__ void __launch_bounds__(kTmaThreads + 32, 1)
    k_dense_tma(const __grid_constant__ CUtensorMap tmap, const float* __restrict__ bsrc, const DenseGeom g,
                const TmaGeom tg, uint64_t ntiles, uint32_t chunk_stride) {
  constexpr int KR = 2 << K;
  constexpr int TILE = 1 << (K + 7);  // amplitudes per tile
  constexpr int EPT = TILE / kTmaThreads;
  constexpr int NCH = KR / 4;
  constexpr uint32_t TCOLS = KR < 32 ? 32 : KR;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* raw = smem;  // kTmaSlots x TILE x 8 B
  const uint32_t abytes = NCH * chunk_stride;
  uint8_t* ahi = raw + kTmaSlots * TILE * 8;
  uint8_t* alo = ahi + abytes;
  uint8_t* bhi = alo + abytes;
  uint8_t* blo = bhi + KR * KR * 4;
  uint32_t* sit = reinterpret_cast<uint32_t*>(blo + KR * KR * 4);  // EPT
  uint32_t* erow = sit + EPT;                                       // 128
  uint32_t* ecol = erow + 128;                                      // 2^K
  uint64_t* bars = reinterpret_cast<uint64_t*>(ecol + (1 << K) + ((1 << K) & 1));
  uint64_t* full = bars;
  uint64_t* done = bars + kTmaSlots;
  uint64_t* mmab = bars + 2 * kTmaSlots;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(mmab + 1);
  const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, quad = warp & 3, half = (warp >> 2) & 1;
  const uint64_t G = gridDim.x;
  constexpr uint32_t kTileBytes = TILE * 8;
  const uint32_t copy_elems = TILE / tg.ncopy;

  for (int i = tid; i < 2 * KR * KR / 4; i += blockDim.x)
    reinterpret_cast<float4*>(bhi)[i] = reinterpret_cast<const float4*>(bsrc)[i];
  for (int r = tid; r < EPT; r += blockDim.x) {
    uint32_t so = 0;
    for (int b = 8; b < g.kb; ++b)
      if ((r >> (b - 8)) & 1) so += g.sb[b];
    sit[r] = so;
  }
  for (int c = tid; c < 128; c += blockDim.x) erow[c] = tg.erow[c];
  for (int j = tid; j < (1 << K); j += blockDim.x) ecol[j] = tg.ecol[j];
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tslot)),
                 "n"(TCOLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
  }
  if (tid == 0) {
    for (int i = 0; i < kTmaSlots; ++i) {
      mbar_init(full + i, 1);
      mbar_init(done + i, kTmaThreads);
    }
    mbar_init(mmab, 1);
    fence_mbar_init();
  }
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;

  if (warp == kTmaThreads / 32) {  // ---------------- TMA producer
    if (lane == 0) {
      auto issue = [&](uint64_t t, int slot) {
        int32_t c[5];
        tma_coords(tg, t, c);
        mbar_expect_tx(full + slot, kTileBytes);
        for (int x = 0; x < tg.ncopy; ++x) {
          int32_t cx[5] = {c[0], c[1], c[2], c[3], c[4] + tg.copy_c4[x]};
          tma_load_5d(raw + (size_t)slot * kTileBytes + (size_t)x * copy_elems * 8, &tmap, cx, full + slot);
        }
      };
      for (int j = 0; j < kTmaSlots; ++j) {
        const uint64_t t = blockIdx.x + (uint64_t)j * G;
        if (t < ntiles) issue(t, j);
      }
      uint32_t phase_done = 0;
      int slot = 0;
      for (uint64_t t = blockIdx.x; t < ntiles; t += G) {
        mbar_wait(done + slot, (phase_done >> slot) & 1u);  // results of tile t are in the slot
        phase_done ^= 1u << slot;
        int32_t c[5];
        tma_coords(tg, t, c);
        const uint8_t* rs = raw + (size_t)slot * kTileBytes;
        for (int x = 0; x < tg.ncopy; ++x) {
          int32_t cx[5] = {c[0], c[1], c[2], c[3], c[4] + tg.copy_c4[x]};
          tma_store_5d(&tmap, cx, rs + (size_t)x * copy_elems * 8);
        }
        bulk_commit();
        const uint64_t tn = t + (uint64_t)kTmaSlots * G;
        if (tn < ntiles) {
          bulk_wait_read0();  // the store has read the slot (the compute warps work on the next tiles meanwhile)
          issue(tn, slot);
        }
        slot = slot + 1 == kTmaSlots ? 0 : slot + 1;
      }
      bulk_wait0();
    }
  } else {  // ------------------------------------------- compute warps
    uint32_t soff = 0;
    for (int b = 0; b < 8; ++b)
      if ((tid >> b) & 1u) soff += g.sb[b];
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(KR >> 3) << 17) | ((128u >> 4) << 24);
    uint32_t phase_full = 0, phase_mma = 0;
    int slot = 0;
    for (uint64_t t = blockIdx.x; t < ntiles; t += G) {
      uint8_t* rs = raw + (size_t)slot * kTileBytes;
      mbar_wait(full + slot, (phase_full >> slot) & 1u);
      phase_full ^= 1u << slot;
#pragma unroll
      for (int r = 0; r < EPT; ++r) {
        const float2 v = *reinterpret_cast<const float2*>(rs + ((size_t)r * kTmaThreads + tid) * 8);
        const float hx = tf32_rna(v.x), hy = tf32_rna(v.y);
        const uint32_t o = soff + sit[r];
        *reinterpret_cast<float2*>(ahi + o) = make_float2(hx, hy);
        *reinterpret_cast<float2*>(alo + o) = make_float2(tf32_rna(v.x - hx), tf32_rna(v.y - hy));
      }
      fence_proxy_async();
      tc_fence_before();
      asm volatile("bar.sync 1, %0;\n" ::"n"(kTmaThreads) : "memory");
      if (tid == 0) {
        tc_fence_after();
        const uint32_t a0 = smem_u32(ahi), a1 = smem_u32(alo), b0 = smem_u32(bhi), b1 = smem_u32(blo);
        const uint32_t as[4] = {a1, a1, a0, a0}, bs[4] = {b1, b0, b1, b0};
#pragma unroll
        for (int term = 0; term < 4; ++term)
#pragma unroll
          for (int s = 0; s < KR / 8; ++s)
            umma_tf32(tmem, umma_desc(as[term] + s * 2 * chunk_stride, chunk_stride, 128),
                      umma_desc(bs[term] + s * 2 * (KR * 16), KR * 16, 128), idesc, (term | s) != 0);
        umma_commit(mmab);
      }
      mbar_wait(mmab, phase_mma);
      phase_mma ^= 1u;
      tc_fence_after();
      {  // D row c (lane), columns -> amplitudes j of column c, natural order into the raw slot
        const uint32_t c = 32 * quad + lane, er = erow[c];
        constexpr int HALF = KR / 2;
#pragma unroll
        for (int col = 0; col < HALF; col += 8) {
          const int cc = half * HALF + col;
          float y[8];
          tmem_ld8(tmem + ((32 * quad) << 16) + cc, y);
#pragma unroll
          for (int q = 0; q < 4; ++q)
            *reinterpret_cast<float2*>(rs + (size_t)(er + ecol[cc / 2 + q]) * 8) =
                make_float2(y[2 * q], y[2 * q + 1]);
        }
      }
      fence_proxy_async();  // generic writes of the slot before the TMA store reads it
      tc_fence_before();
      mbar_arrive(done + slot);
      slot = slot + 1 == kTmaSlots ? 0 : slot + 1;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(TCOLS) : "memory");
  }
}

// ---------------------------------------------- k = 6: U as the TMEM operand
// For 6-qubit blocks the real-form unitary (128 x 128 fp32, hi and lo) does
// not fit in shared memory next to the tile, so the roles swap: A = U lives in
// TMEM (lane = output row, columns = K; written once per CTA with
// tcgen05.st), B = the tile (N = 128 state columns, K = 128 reals) in shared
// memory, D[out][column] in TMEM.  3-term split (U_lo X_hi, U_hi X_lo,
// U_hi X_hi).  TMEM: U_hi [0,128), U_lo [128,256), D [256,384).
constexpr int kTc6Threads = 256;

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const float* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};\n" ::"r"(
          taddr),
      "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])), "r"(__float_as_uint(v[3])),
      "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])), "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])),
      "r"(__float_as_uint(v[8])), "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])), "r"(__float_as_uint(v[11])),
      "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])), "r"(__float_as_uint(v[14])), "r"(__float_as_uint(v[15]))
      : "memory");
}

__device__ __forceinline__ void umma_tf32_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc,
                                             uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, {%5, %5, %5, %5}, p;\n}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate), "r"(0u)
      : "memory");
}

// usrc: real-form U rows (128 x 128 fp32, row-major) hi then lo
__global__ void __launch_bounds__(kTc6Threads, 1)
    k_dense_tc6(float2* __restrict__ state, const float* __restrict__ usrc, const DenseGeom g, uint64_t ntiles,
                uint32_t chunk_stride) {
  constexpr int KR = 128;
  constexpr int EPT = (1 << 13) / kTc6Threads;  // 32
  constexpr int NCH = KR / 4;
  extern __shared__ __align__(1024) uint8_t smem[];
  DenseSmemHdr* hdr = reinterpret_cast<DenseSmemHdr*>(smem);
  const uint32_t xbytes = NCH * chunk_stride;
  uint8_t* xhi = smem + sizeof(DenseSmemHdr);
  uint8_t* xlo = xhi + xbytes;
  uint64_t* git = reinterpret_cast<uint64_t*>(xlo + xbytes);
  uint32_t* sit = reinterpret_cast<uint32_t*>(git + EPT);
  uint64_t* bar = reinterpret_cast<uint64_t*>(sit + EPT);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 1);
  const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, quad = warp & 3;

  dense_it_tables<kTc6Threads>(g, EPT, git, sit);
  dense_tile_tables(g, hdr);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tslot)),
                 "n"(512)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
  }
  if (tid == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  const uint32_t t_uhi = tmem, t_ulo = tmem + 128, t_d = tmem + 256;
  {  // U rows into TMEM: warps 0-3 the hi half, warps 4-7 the lo half; lane = row
    const int row = 32 * quad + lane;
    const float* src = usrc + (warp >= 4 ? KR * KR : 0) + (size_t)row * KR;
    const uint32_t base = (warp >= 4 ? t_ulo : t_uhi) + ((32 * quad) << 16);
#pragma unroll
    for (int c = 0; c < KR; c += 16) {
      float v[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) v[i] = src[c + i];
      tmem_st16(base + c, v);
    }
    asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  uint64_t goff;
  uint32_t soff;
  dense_thread_offsets<kTc6Threads>(g, tid, goff, soff);
  // M = 128 (U rows), N = 128 (state columns), TF32 A (TMEM) and B (smem), F32 D
  const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((128u >> 3) << 17) | ((128u >> 4) << 24);
  uint32_t phase = 0;

  auto load = [&](float2 (&v)[EPT], uint64_t t) {
    const uint64_t base = dense_tile_base(hdr, t) + goff;
#pragma unroll
    for (int i = 0; i < EPT; ++i) v[i] = __ldcs(state + base + git[i]);
  };
  auto step = [&](float2 (&cur)[EPT], float2 (&nxt)[EPT], uint64_t t) {
    const uint64_t base = dense_tile_base(hdr, t) + goff;
    if (t + gridDim.x < ntiles) load(nxt, t + gridDim.x);
#pragma unroll
    for (int i = 0; i < EPT; ++i) {
      const float hx = tf32_rna(cur[i].x), hy = tf32_rna(cur[i].y);
      const uint32_t o = soff + sit[i];
      *reinterpret_cast<float2*>(xhi + o) = make_float2(hx, hy);
      *reinterpret_cast<float2*>(xlo + o) = make_float2(tf32_rna(cur[i].x - hx), tf32_rna(cur[i].y - hy));
    }
    fence_proxy_async();
    __syncthreads();
    if (tid == 0) {
      tc_fence_after();
      const uint32_t b0 = smem_u32(xhi), b1 = smem_u32(xlo);
      const uint32_t as[3] = {t_ulo, t_uhi, t_uhi}, bs[3] = {b0, b1, b0};
#pragma unroll
      for (int term = 0; term < 3; ++term)
#pragma unroll
        for (int s = 0; s < KR / 8; ++s)
          umma_tf32_ts(t_d, as[term] + 8 * s, umma_desc(bs[term] + s * 2 * chunk_stride, chunk_stride, 128), idesc,
                       (term | s) != 0);
      umma_commit(bar);
    }
    mbar_wait(bar, phase);
    phase ^= 1u;
    tc_fence_after();
    {  // D row n = output real index (re/im of amplitude n / 2), columns = state columns
      const uint32_t n = 32 * quad + lane;
      const uint32_t nb = (n >> 2) * chunk_stride + ((n >> 1) & 1) * 8 + (n & 1) * 4;
      const int c0 = warp >= 4 ? 64 : 0;
#pragma unroll
      for (int c = 0; c < 64; c += 16) {
        float y[16];
        tmem_ld16(t_d + ((32 * quad) << 16) + c0 + c, y);
#pragma unroll
        for (int i = 0; i < 16; ++i) *reinterpret_cast<float*>(xhi + nb + (c0 + c + i) * 16) = y[i];
      }
    }
    tc_fence_before();
    __syncthreads();
#pragma unroll
    for (int i = 0; i < EPT; ++i)
      __stcs(state + base + git[i], *reinterpret_cast<const float2*>(xhi + soff + sit[i]));
    __syncthreads();
  };

  float2 va[EPT], vb[EPT];
  const uint64_t G = gridDim.x;
  if (blockIdx.x < ntiles) load(va, blockIdx.x);
  for (uint64_t t = blockIdx.x; t < ntiles; t += 2 * G) {
    step(va, vb, t);
    if (t + G < ntiles) step(vb, va, t + G);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(512) : "memory");
  }
}

// ----------------------------------------------------- CUDA-core baseline
constexpr int kFmaThreads = 256;
constexpr int kFmaOut = 8;  // outputs accumulated per thread per sweep over the inputs

// smem: [hdr | X | Y | U | git | sit]; X/Y layout [j][c] complex with
// 2^cb columns per tile (EPT * 256 amplitudes).  The next tile's loads are
// issued as soon as this tile is in shared memory, so they are in flight
// during the products and the stores.
template <typename R, int EPT>
__global__ void __launch_bounds__(kFmaThreads, 2)
    k_dense_fma(cplx<R>* __restrict__ state, const cplx<R>* __restrict__ u, const DenseGeom g, uint64_t ntiles) {
  const int k = g.k, D = 1 << k, cb = g.kb - g.k, cols = 1 << cb;
  const int ob = D < kFmaOut ? D : kFmaOut;
  extern __shared__ __align__(16) uint8_t smem[];
  DenseSmemHdr* hdr = reinterpret_cast<DenseSmemHdr*>(smem);
  cplx<R>* X = reinterpret_cast<cplx<R>*>(smem + sizeof(DenseSmemHdr));
  cplx<R>* Y = X + (D << cb);
  cplx<R>* U = Y + (D << cb);
  uint64_t* git = reinterpret_cast<uint64_t*>(U + D * D);
  uint32_t* sit = reinterpret_cast<uint32_t*>(git + EPT);
  const uint32_t tid = threadIdx.x;
  for (int i = tid; i < D * D; i += kFmaThreads) U[i] = u[i];
  dense_it_tables<kFmaThreads>(g, EPT, git, sit);
  dense_tile_tables(g, hdr);
  uint64_t goff;
  uint32_t soff;
  dense_thread_offsets<kFmaThreads>(g, tid, goff, soff);
  __syncthreads();
  const int items = cols * (D / ob);
  cplx<R> v[EPT];
  uint64_t t = blockIdx.x;
  if (t < ntiles) {
    const uint64_t base = dense_tile_base(hdr, t) + goff;
#pragma unroll
    for (int i = 0; i < EPT; ++i) v[i] = __ldcs(state + base + git[i]);
  }
  for (; t < ntiles; t += gridDim.x) {
    const uint64_t base = dense_tile_base(hdr, t) + goff;
#pragma unroll
    for (int i = 0; i < EPT; ++i) *reinterpret_cast<cplx<R>*>(reinterpret_cast<uint8_t*>(X) + soff + sit[i]) = v[i];
    if (t + gridDim.x < ntiles) {
      const uint64_t nb = dense_tile_base(hdr, t + gridDim.x) + goff;
#pragma unroll
      for (int i = 0; i < EPT; ++i) v[i] = __ldcs(state + nb + git[i]);
    }
    __syncthreads();
    for (int p = tid; p < items; p += kFmaThreads) {
      const int c = p & (cols - 1), i0 = (p >> cb) * ob;
      cplx<R> acc[kFmaOut];
#pragma unroll
      for (int o = 0; o < kFmaOut; ++o) acc[o] = mk<R>(0, 0);
      for (int j = 0; j < D; ++j) {
        const cplx<R> xj = X[(j << cb) + c];
#pragma unroll
        for (int o = 0; o < kFmaOut; ++o)
          if (o < ob) acc[o] = cfma_scalar<R>(U[(i0 + o) * D + j], xj, acc[o]);
      }
#pragma unroll
      for (int o = 0; o < kFmaOut; ++o)
        if (o < ob) Y[((i0 + o) << cb) + c] = acc[o];
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < EPT; ++i)
      __stcs(state + base + git[i],
             *reinterpret_cast<const cplx<R>*>(reinterpret_cast<const uint8_t*>(Y) + soff + sit[i]));
  }
}

// ------------------------------------------------------------------ host
// Tile = block qubits + the 7 lowest other qubits; `layout` 0: [j][c] complex
// of size s (FMA kernel), 1: the UMMA A-operand layout (TC kernel).
static DenseGeom make_geom(int n, const int32_t* q, int k, int cb, int layout, size_t s, uint32_t chunk_stride) {
  DenseGeom g;
  g.k = k;
  g.kb = k + cb;
  std::vector<int> blk(q, q + k), cols, tile;
  for (int x = 0; x < n && (int)cols.size() < cb; ++x)
    if (std::find(blk.begin(), blk.end(), x) == blk.end()) cols.push_back(x);
  tile = cols;
  tile.insert(tile.end(), blk.begin(), blk.end());
  std::sort(tile.begin(), tile.end());
  for (int b = 0; b < g.kb; ++b) {
    const int x = tile[b];
    g.tq[b] = (int8_t)x;
    const auto bi = std::find(blk.begin(), blk.end(), x);
    if (bi != blk.end()) {
      const int i = (int)(bi - blk.begin());  // local index bit i of U
      if (layout == 0) g.sb[b] = (uint32_t)(s << cb) << i;
      else g.sb[b] = i == 0 ? 8u : chunk_stride << (i - 1);
    } else {
      const int r = (int)(std::find(cols.begin(), cols.end(), x) - cols.begin());  // column bit r
      if (layout == 0) g.sb[b] = (uint32_t)s << r;
      else g.sb[b] = 16u << r;  // (c % 8) * 16 + (c / 8) * 128 = 16 c
    }
  }
  g.nout = 0;
  for (int x = 0; x < n; ++x)
    if (std::find(tile.begin(), tile.end(), x) == tile.end()) g.outq[g.nout++] = (int8_t)x;
  return g;
}

static int sm_count() {
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  return nsm;
}

bool dense_tc_supported(int precision, int n, int k) {
  return precision == SVB_C64 && k >= 3 && k <= kTcMaxK && n >= k + 7;
}
bool dense_fma_supported(int precision, int n, int k) {
  return k >= 1 && k <= (precision == SVB_C128 ? kDenseMaxK - 1 : kDenseMaxK) && n >= k + 7;
}

// mat: 2^k x 2^k complex, row-major (re, im) doubles, local bit i <-> q[i]
static void launch_dense_tc6(void* state, int n, const int32_t* q, const double* mat, cudaStream_t st,
                             uint32_t chunk_stride) {
  constexpr int D = 64, KR = 128;
  auto rna = [](float x) {
    uint32_t bits;
    std::memcpy(&bits, &x, 4);
    bits = (bits + 0x1000u) & 0xFFFFE000u;
    float r;
    std::memcpy(&r, &bits, 4);
    return r;
  };
  // real-form rows U_real[nrow][kk], row-major, hi then lo
  std::vector<float> hu(2 * KR * KR);
  auto put = [&](int nrow, int kk, double val) {
    const float x = (float)val, hi = rna(x);
    hu[(size_t)nrow * KR + kk] = hi;
    hu[(size_t)KR * KR + (size_t)nrow * KR + kk] = rna(x - hi);
  };
  for (int i = 0; i < D; ++i)
    for (int j = 0; j < D; ++j) {
      const double re = mat[2 * (i * D + j)], im = mat[2 * (i * D + j) + 1];
      put(2 * i, 2 * j, re);
      put(2 * i, 2 * j + 1, -im);
      put(2 * i + 1, 2 * j, im);
      put(2 * i + 1, 2 * j + 1, re);
    }
  float* du = nullptr;
  SVB_CUDA(cudaMallocAsync(&du, hu.size() * sizeof(float), st));
  SVB_CUDA(cudaMemcpyAsync(du, hu.data(), hu.size() * sizeof(float), cudaMemcpyHostToDevice, st));
  const DenseGeom g = make_geom(n, q, 6, 7, 1, 8, chunk_stride);
  require(g.nout <= 32, SVB_E_ARG, "dense block: state too large for the tile-base tables");
  const uint64_t ntiles = 1ull << (n - 13);
  const int ept = (1 << 13) / kTc6Threads;
  const size_t smem = sizeof(DenseSmemHdr) + 2 * (size_t)(KR / 4) * chunk_stride + (size_t)ept * 12 + 64;
  const unsigned grid = (unsigned)std::min<uint64_t>(ntiles, (uint64_t)sm_count());
  static std::atomic<uint64_t> attr{0};
  once_per_device(attr, [] {
    cudaFuncSetAttribute(k_dense_tc6, cudaFuncAttributeMaxDynamicSharedMemorySize, 150 * 1024);
  });
  k_dense_tc6<<<grid, kTc6Threads, smem, st>>>(static_cast<float2*>(state), du, g, ntiles, chunk_stride);
  SVB_CHECK_LAUNCH();
  SVB_CUDA(cudaFreeAsync(du, st));
}

// Tensor map of the state for the TMA-staged kernel (see k_dense_tma);
// false when the geometry does not fit (then the register-prefetch kernels run).
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static bool make_tma(void* state, int n, const DenseGeom& g, const int32_t* q, int k, CUtensorMap* map,
                     TmaGeom* tg) {
  static EncodeTiledFn encode = [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      fn = nullptr;
    cudaGetLastError();
    return reinterpret_cast<EncodeTiledFn>(fn);
  }();
  if (!encode || n > 36) return false;
  // pieces: runs of consecutive tile qubits, <= 8 qubits each
  std::vector<std::pair<int, int>> pc;  // (start, len)
  for (int b = 0; b < g.kb; ++b) {
    const int qb = g.tq[b];
    if (!pc.empty() && pc.back().first + pc.back().second == qb && pc.back().second < 8) ++pc.back().second;
    else pc.push_back({qb, 1});
  }
  if (pc[0].first != 0) return false;
  const int nd = std::min<int>(5, (int)pc.size());
  std::vector<int> extra;  // tile qubits beyond the fifth piece: enumerated by copies
  for (size_t i = nd; i < pc.size(); ++i)
    for (int j = 0; j < pc[i].second; ++j) extra.push_back(pc[i].first + j);
  if ((1 << extra.size()) > kTmaMaxCopies) return false;
  cuuint64_t gdim[5], gstr[4];
  cuuint32_t box[5], es[5] = {1, 1, 1, 1, 1};
  for (int d = 0; d < 5; ++d) {
    if (d < nd) {
      const int s0 = pc[d].first, e0 = d + 1 < nd ? pc[d + 1].first : n;
      if (e0 - s0 > 31) return false;
      gdim[d] = 1ull << (e0 - s0);
      box[d] = 1u << pc[d].second;
      if (d >= 1) gstr[d - 1] = 8ull << s0;
    } else {
      gdim[d] = 1;
      box[d] = 1;
      gstr[d - 1] = 8ull << n;
    }
  }
  if (encode(map, CU_TENSOR_MAP_DATA_TYPE_UINT64, 5, state, gdim, gstr, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
      CUDA_SUCCESS)
    return false;
  std::memset(tg, 0, sizeof *tg);
  tg->ncopy = 1 << extra.size();
  for (int x = 0; x < tg->ncopy; ++x) {
    int32_t c4 = 0;
    for (size_t i = 0; i < extra.size(); ++i)
      if ((x >> i) & 1) c4 += 1 << (extra[i] - pc[nd - 1].first);
    tg->copy_c4[x] = c4;
  }
  // tile-index bit b (outside qubit g.outq[b]) -> dim and coordinate bit
  tg->ntb = g.nout;
  for (int b = 0; b < g.nout; ++b) {
    const int qb = g.outq[b];
    int d = 0;
    while (d + 1 < nd && pc[d + 1].first <= qb) ++d;
    tg->tdim[b] = (int8_t)d;
    tg->tshift[b] = (int8_t)(qb - pc[d].first);
  }
  // natural tile index of (row c, amplitude j): tile position b holds qubit
  // g.tq[b], a block qubit (local bit i of U) or the r-th column qubit
  std::vector<int> role(g.kb);  // >= 0: block bit i; < 0: column bit -(r + 1)
  int r = 0;
  for (int b = 0; b < g.kb; ++b) {
    const int i = (int)(std::find(q, q + k, (int32_t)g.tq[b]) - q);
    role[b] = i < k ? i : -(++r);
  }
  for (int c = 0; c < 128; ++c) {
    uint32_t e = 0;
    for (int b = 0; b < g.kb; ++b)
      if (role[b] < 0 && ((c >> (-role[b] - 1)) & 1)) e |= 1u << b;
    tg->erow[c] = e;
  }
  for (int j = 0; j < (1 << k); ++j) {
    uint32_t e = 0;
    for (int b = 0; b < g.kb; ++b)
      if (role[b] >= 0 && ((j >> role[b]) & 1)) e |= 1u << b;
    tg->ecol[j] = e;
  }
  return true;
}

void launch_dense_tc(void* state, int n, const int32_t* q, int k, const double* mat, cudaStream_t st) {
  require(k >= 3 && k <= kTcMaxK && n >= k + 7, SVB_E_ARG, "tensor-core dense block: need 3 <= k <= 6, n >= k + 7");
  const int D = 1 << k, KR = 2 * D;
  const uint32_t chunk_stride = kDenseCols * 16 + 16;  // 2064 B: +16 B keeps tile writes bank-conflict free
  if (k == 6) {
    launch_dense_tc6(state, n, q, mat, st, chunk_stride);
    return;
  }
  // real form B[n_out][kk] (K-major rows), split into TF32 hi / lo, in the
  // canonical layout byte(nrow, kk) = (kk / 4) * KR * 16 + nrow * 16 + (kk % 4) * 4
  std::vector<float> hb(2 * KR * KR);
  auto rna = [](float x) {  // cvt.rna.tf32.f32 on the host (finite inputs)
    uint32_t bits;
    std::memcpy(&bits, &x, 4);
    bits = (bits + 0x1000u) & 0xFFFFE000u;
    float r;
    std::memcpy(&r, &bits, 4);
    return r;
  };
  auto put = [&](int nrow, int kk, double val) {
    const float x = (float)val, hi = rna(x);
    const size_t idx = (size_t)(kk / 4) * KR * 4 + (size_t)nrow * 4 + (kk % 4);
    hb[idx] = hi;
    hb[(size_t)KR * KR + idx] = rna(x - hi);
  };
  for (int i = 0; i < D; ++i)
    for (int j = 0; j < D; ++j) {
      const double re = mat[2 * (i * D + j)], im = mat[2 * (i * D + j) + 1];
      put(2 * i, 2 * j, re);
      put(2 * i, 2 * j + 1, -im);
      put(2 * i + 1, 2 * j, im);
      put(2 * i + 1, 2 * j + 1, re);
    }
  float* db = nullptr;
  SVB_CUDA(cudaMallocAsync(&db, hb.size() * sizeof(float), st));
  SVB_CUDA(cudaMemcpyAsync(db, hb.data(), hb.size() * sizeof(float), cudaMemcpyHostToDevice, st));
  const DenseGeom g = make_geom(n, q, k, 7, 1, 8, chunk_stride);
  require(g.nout <= 32, SVB_E_ARG, "dense block: state too large for the tile-base tables");
  const uint64_t ntiles = 1ull << (n - k - 7);
  // TMA-staged kernel on request (SVB_TC_TMA=1): at n = 30 it measured 5.4 ms
  // (k = 5, mixed qubits) against 5.1-5.3 ms for the register-prefetch
  // kernels below and is slower for k <= 4 (one CTA per SM, one A buffer:
  // the MMA latency is exposed), so those stay the default
  static const bool use_tma = std::getenv("SVB_TC_TMA") && std::atoi(std::getenv("SVB_TC_TMA")) != 0;
  CUtensorMap tmap;
  TmaGeom tg;
  if (use_tma && make_tma(state, n, g, q, k, &tmap, &tg)) {
    const int tile = 1 << (k + 7);
    const size_t smem = (size_t)kTmaSlots * tile * 8 + 2 * (size_t)(KR / 4) * chunk_stride + 2 * (size_t)KR * KR * 4 +
                        (size_t)(tile / kTmaThreads) * 4 + 128 * 4 + 64 * 4 + 8 * (2 * kTmaSlots + 2) + 64;
    const unsigned grid = (unsigned)std::min<uint64_t>(ntiles, (uint64_t)sm_count());
    static std::atomic<uint64_t> tattr[3] = {{0}, {0}, {0}};
    auto go = [&](auto kern, int slot) {
      once_per_device(tattr[slot], [&] {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
      });
      kern<<<grid, kTmaThreads + 32, smem, st>>>(tmap, db, g, tg, ntiles, chunk_stride);
    };
    if (k == 3) go(k_dense_tma<3>, 0);
    else if (k == 4) go(k_dense_tma<4>, 1);
    else go(k_dense_tma<5>, 2);
    SVB_CHECK_LAUNCH();
    SVB_CUDA(cudaFreeAsync(db, st));
    return;
  }
  // k = 5: the pipelined one-CTA kernel (measured 5.1 vs 5.7 ms at n = 30);
  // k <= 4: two CTAs per SM with register prefetch (smaller tiles need the
  // second CTA's loads in flight: 4.6 vs 8.2 ms at k = 3).  SVB_TC_PIPE=0/1 overrides.
  const char* pe = std::getenv("SVB_TC_PIPE");
  const bool pipe = pe ? std::atoi(pe) != 0 : k == 5;
  static std::atomic<uint64_t> attr[6] = {{0}, {0}, {0}, {0}, {0}, {0}};
  if (pipe) {
    const int ept = (1 << (k + 7)) / kTcpThreads;
    const size_t smem = sizeof(DenseSmemHdr) + 4 * (size_t)(KR / 4) * chunk_stride + 2 * (size_t)KR * KR * 4 +
                        (size_t)ept * 12 + 64;
    const unsigned grid = (unsigned)std::min<uint64_t>(ntiles, (uint64_t)sm_count());
    auto go = [&](auto kern, int slot) {
      once_per_device(attr[slot], [&] {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      });
      kern<<<grid, kTcpThreads, smem, st>>>(static_cast<float2*>(state), db, g, ntiles, chunk_stride);
    };
    if (k == 3) go(k_dense_tcp<3>, 3);
    else if (k == 4) go(k_dense_tcp<4>, 4);
    else go(k_dense_tcp<5>, 5);
  } else {
    const int ept = (1 << (k + 7)) / kTcThreads;
    const size_t smem = sizeof(DenseSmemHdr) + 2 * (size_t)(KR / 4) * chunk_stride + 2 * (size_t)KR * KR * 4 +
                        (size_t)ept * 12 + 64;
    const unsigned grid = (unsigned)std::min<uint64_t>(ntiles, (uint64_t)sm_count() * 2);
    auto go = [&](auto kern, int slot) {
      once_per_device(attr[slot], [&] {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 112 * 1024);
      });
      kern<<<grid, kTcThreads, smem, st>>>(static_cast<float2*>(state), db, g, ntiles, chunk_stride);
    };
    if (k == 3) go(k_dense_tc<3>, 0);
    else if (k == 4) go(k_dense_tc<4>, 1);
    else go(k_dense_tc<5>, 2);
  }
  SVB_CHECK_LAUNCH();
  SVB_CUDA(cudaFreeAsync(db, st));
}

template <typename R>
void launch_dense_fma(void* state, int n, const int32_t* q, int k, const double* mat, cudaStream_t st) {
  require(dense_fma_supported(sizeof(R) == 8 ? SVB_C128 : SVB_C64, n, k), SVB_E_ARG,
          "dense block: need n >= k + 7 and 1 <= k <= 6 (complex64) / 5 (complex128)");
  const int D = 1 << k;
  std::vector<cplx<R>> hu(D * D);
  for (int i = 0; i < D * D; ++i) hu[i] = mk<R>((R)mat[2 * i], (R)mat[2 * i + 1]);
  cplx<R>* du = nullptr;
  SVB_CUDA(cudaMallocAsync(&du, hu.size() * sizeof(cplx<R>), st));
  SVB_CUDA(cudaMemcpyAsync(du, hu.data(), hu.size() * sizeof(cplx<R>), cudaMemcpyHostToDevice, st));
  const int cb = std::min(n - k, std::max(7, 12 - k));  // 4096 amplitudes per tile (8192 for k = 6)
  require((D << cb) >= kFmaThreads && (D << cb) <= 32 * kFmaThreads, SVB_E_ARG, "dense block: bad tile size");
  const DenseGeom g = make_geom(n, q, k, cb, 0, sizeof(cplx<R>), 0);
  require(g.nout <= 32, SVB_E_ARG, "dense block: state too large for the tile-base tables");
  const uint64_t ntiles = 1ull << (n - k - cb);
  const int ept = (D << cb) / kFmaThreads;
  const size_t smem = sizeof(DenseSmemHdr) + (2 * ((size_t)D << cb) + (size_t)D * D) * sizeof(cplx<R>) +
                      (size_t)ept * 12 + 16;
  const int per_sm = smem <= 110 * 1024 ? 2 : 1;  // two CTAs per SM when their tiles fit
  const unsigned grid = (unsigned)std::min<uint64_t>(ntiles, (uint64_t)sm_count() * per_sm);
  static std::atomic<uint64_t> attr[6] = {{0}, {0}, {0}, {0}, {0}, {0}};
  auto go = [&](auto kern, int slot) {
    once_per_device(attr[slot], [&] {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    });
    kern<<<grid, kFmaThreads, smem, st>>>(static_cast<cplx<R>*>(state), du, g, ntiles);
  };
  switch (ept) {
    case 1: go(k_dense_fma<R, 1>, 0); break;
    case 2: go(k_dense_fma<R, 2>, 1); break;
    case 4: go(k_dense_fma<R, 4>, 2); break;
    case 8: go(k_dense_fma<R, 8>, 3); break;
    case 16: go(k_dense_fma<R, 16>, 4); break;
    default: go(k_dense_fma<R, 32>, 5); break;
  }
  SVB_CHECK_LAUNCH();
  SVB_CUDA(cudaFreeAsync(du, st));
}
template void launch_dense_fma<float>(void*, int, const int32_t*, int, const double*, cudaStream_t);
template void launch_dense_fma<double>(void*, int, const int32_t*, int, const double*, cudaStream_t);

}  // namespace svb
