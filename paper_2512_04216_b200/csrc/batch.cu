// Persistent batch kernel for many small circuits (config 4).
//
// Replaces the reference's sequential batch runner (`batch.run_batch`,
// batch.py:104-222: one `run_circuit(c, "sv", shots, seed)` per circuit) for
// the circuits whose state fits in shared memory (2^n x s <= 64 KB: n <= 12
// complex128, n <= 13 complex64).  One CTA per SM walks the batch; per circuit
// it keeps the whole state in shared memory, applies the gates as shared
// memory sweeps, builds the CDF of |amp|^2 with a block scan, and draws the
// shots from the circuit's PCG64 stream (numpy default_rng(seed) positions
// 0..shots-1) by binary search.  HBM traffic is only the gate records in and
// the shot codes out.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "kernels.h"

namespace svb {

// per-gate record: kind 0 = dense 1q, 1 = dense 2q, 2 = monomial 2q
struct BatchGate {
  int32_t kind, q0, q1, src;  // src: 4 x 2-bit source indices (monomial)
  double m[32];               // row-major complex (re, im)
};

struct BatchCirc {
  int32_t n, gate_off, ngates, w;
  uint64_t pcg[4];
  int8_t bit_src[64];
};

typedef unsigned __int128 u128b;
__device__ __forceinline__ u128b mult128() { return ((u128b)0x2360ED051FC65DA4ull << 64) | 0x4385DF649FCCF645ull; }
__device__ __forceinline__ void lcg_jump(u128b inc, uint64_t delta, u128b& am, u128b& ap) {
  u128b acc_m = 1, acc_p = 0, cur_m = mult128(), cur_p = inc;
  while (delta) {
    if (delta & 1) {
      acc_m *= cur_m;
      acc_p = acc_p * cur_m + cur_p;
    }
    cur_p = (cur_m + 1) * cur_p;
    cur_m *= cur_m;
    delta >>= 1;
  }
  am = acc_m;
  ap = acc_p;
}
__device__ __forceinline__ double pcg_out(u128b s) {
  uint64_t hi = (uint64_t)(s >> 64), lo = (uint64_t)s;
  uint64_t x = hi ^ lo;
  unsigned r = (unsigned)(hi >> 58);
  uint64_t v = (x >> r) | (x << ((64u - r) & 63u));
  return (double)(v >> 11) * (1.0 / 9007199254740992.0);
}

template <typename R>
__global__ void __launch_bounds__(256, 1) k_batch_small(const BatchCirc* __restrict__ circs, int ncirc,
                                                        const BatchGate* __restrict__ gates, uint64_t shots,
                                                        uint64_t* __restrict__ codes) {
  extern __shared__ __align__(16) unsigned char smraw[];
  cplx<R>* st = reinterpret_cast<cplx<R>*>(smraw);                        // <= 64 KB
  double* cum = reinterpret_cast<double*>(smraw + 65536);                 // <= 8192 doubles
  __shared__ double warp_tot[8];
  const uint32_t tid = threadIdx.x;
  for (int ci = blockIdx.x; ci < ncirc; ci += gridDim.x) {
    const BatchCirc C = circs[ci];
    const uint32_t len = 1u << C.n;
    for (uint32_t i = tid; i < len; i += blockDim.x) st[i] = mk<R>(i == 0 ? R(1) : R(0), R(0));
    for (int gi = 0; gi < C.ngates; ++gi) {
      __syncthreads();
      const BatchGate& g = gates[C.gate_off + gi];
      const int kind = g.kind;
      if (kind == 0) {
        const int q = g.q0;
        const cplx<R> m0 = mk<R>((R)g.m[0], (R)g.m[1]), m1 = mk<R>((R)g.m[2], (R)g.m[3]);
        const cplx<R> m2 = mk<R>((R)g.m[4], (R)g.m[5]), m3 = mk<R>((R)g.m[6], (R)g.m[7]);
        for (uint32_t p = tid; p < len / 2; p += blockDim.x) {
          const uint32_t i0 = (uint32_t)insert0(p, q), i1 = i0 | (1u << q);
          const cplx<R> x0 = st[i0], x1 = st[i1];
          st[i0] = cfma<R>(m1, x1, cmul<R>(m0, x0));
          st[i1] = cfma<R>(m3, x1, cmul<R>(m2, x0));
        }
      } else {
        const int qa = g.q0, qb = g.q1;
        const int lo = qa < qb ? qa : qb, hi = qa < qb ? qb : qa;
        for (uint32_t p = tid; p < len / 4; p += blockDim.x) {
          const uint32_t base = (uint32_t)insert0(insert0(p, lo), hi);
          const uint32_t idx[4] = {base, base | (1u << qa), base | (1u << qb), base | (1u << qa) | (1u << qb)};
          cplx<R> x[4];
#pragma unroll
          for (int k = 0; k < 4; ++k) x[k] = st[idx[k]];
          if (kind == 2) {
#pragma unroll
            for (int r = 0; r < 4; ++r) {
              const int sidx = (g.src >> (2 * r)) & 3;
              const cplx<R> e = mk<R>((R)g.m[2 * (4 * r + sidx)], (R)g.m[2 * (4 * r + sidx) + 1]);
              st[idx[r]] = cmul<R>(e, x[sidx]);
            }
          } else {
#pragma unroll
            for (int r = 0; r < 4; ++r) {
              cplx<R> acc = mk<R>(R(0), R(0));
#pragma unroll
              for (int c = 0; c < 4; ++c)
                acc = cfma<R>(mk<R>((R)g.m[2 * (4 * r + c)], (R)g.m[2 * (4 * r + c) + 1]), x[c], acc);
              st[idx[r]] = acc;
            }
          }
        }
      }
    }
    __syncthreads();
    // CDF: each thread sums a contiguous chunk, warp + block exclusive scan
    const uint32_t per = (len + blockDim.x - 1) / blockDim.x;
    const uint32_t b0 = tid * per, b1 = b0 + per < len ? b0 + per : len;
    double loc = 0.0;
    for (uint32_t i = b0; i < b1; ++i) {
      const double x = (double)st[i].x, y = (double)st[i].y;
      loc += x * x + y * y;
      cum[i] = loc;
    }
    double inc = loc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double v = __shfl_up_sync(0xffffffffu, inc, o);
      if ((tid & 31u) >= (uint32_t)o) inc += v;
    }
    if ((tid & 31u) == 31u) warp_tot[tid >> 5] = inc;
    __syncthreads();
    double woff = 0.0;
    for (uint32_t w = 0; w < (tid >> 5); ++w) woff += warp_tot[w];
    const double off = woff + inc - loc;
    for (uint32_t i = b0; i < b1; ++i) cum[i] += off;
    __syncthreads();
    const double total = cum[len - 1];
    // shots s = tid, tid + 256, ...: stream position s of the circuit's PCG64
    const u128b inc128 = ((u128b)C.pcg[2] << 64) | C.pcg[3];
    u128b s = ((u128b)C.pcg[0] << 64) | C.pcg[1];
    u128b am, ap, sm, sp;
    lcg_jump(inc128, tid + 1, am, ap);  // state after draw `tid` (step precedes output)
    s = am * s + ap;
    lcg_jump(inc128, blockDim.x, sm, sp);
    uint64_t* out = codes + (uint64_t)ci * shots;
    for (uint64_t k = tid; k < shots; k += blockDim.x) {
      const double target = pcg_out(s) * total;
      s = sm * s + sp;
      uint32_t lo = 0, hi = len;  // first i with cum[i] > target
      while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (cum[mid] <= target) lo = mid + 1;
        else hi = mid;
      }
      if (lo >= len) lo = len - 1;
      uint64_t code = 0;
      for (int p = 0; p < C.w; ++p) code |= (uint64_t)((lo >> C.bit_src[p]) & 1u) << p;
      out[k] = code;
    }
    __syncthreads();
  }
}

}  // namespace svb

using namespace svb;

// Batch of small terminal circuits (n <= 12 complex128 / 13 complex64).
//   gates[]   svb_gate records of all circuits, circuit i at [gate_off[i], gate_off[i] + ngates[i]);
//   pcg[4i..]  numpy PCG64 state of default_rng(seed_i);
//   bit_src[64i..]  output bit p of circuit i <- bit bit_src of the sampled index;
//   out_codes[shots * i + s]  packed clbits of shot s.
extern "C" int svb_batch_small(int device, int precision, int ncirc, const int32_t* nq, const int32_t* gate_off,
                               const int32_t* ngates, const svb_gate* gates, int total_gates, const uint64_t* pcg,
                               const int32_t* w, const int8_t* bit_src, uint64_t shots, uint64_t* out_codes) {
  try {
    require(ncirc >= 0 && shots >= 1, SVB_E_ARG, "bad batch arguments");
    if (ncirc == 0) return SVB_OK;
    const int nmax = precision == SVB_C128 ? 12 : 13;
    std::vector<BatchCirc> hc(ncirc);
    for (int i = 0; i < ncirc; ++i) {
      require(nq[i] >= 1 && nq[i] <= nmax, SVB_E_ARG, "circuit too large for the shared-memory batch kernel");
      require(w[i] >= 1 && w[i] <= 63, SVB_E_ARG, "bad clbit count");
      require(gate_off[i] >= 0 && ngates[i] >= 0 && gate_off[i] + ngates[i] <= total_gates, SVB_E_ARG, "bad gate range");
      hc[i].n = nq[i];
      hc[i].gate_off = gate_off[i];
      hc[i].ngates = ngates[i];
      hc[i].w = w[i];
      for (int k = 0; k < 4; ++k) hc[i].pcg[k] = pcg[4 * i + k];
      for (int p = 0; p < 64; ++p) hc[i].bit_src[p] = bit_src[64 * i + p];
    }
    std::vector<BatchGate> hg(total_gates);
    for (int i = 0; i < total_gates; ++i) {
      const svb_gate& g = gates[i];
      BatchGate& b = hg[i];
      std::memcpy(b.m, g.mat, sizeof b.m);
      b.q0 = g.qubits[0];
      b.q1 = g.k == 2 ? g.qubits[1] : 0;
      b.src = 0;
      if (g.k == 1) {
        b.kind = 0;
        continue;
      }
      bool mono = true;
      for (int r = 0; r < 4 && mono; ++r) {
        int nz = 0, src = 0;
        for (int c = 0; c < 4; ++c)
          if (g.mat[2 * (4 * r + c)] != 0.0 || g.mat[2 * (4 * r + c) + 1] != 0.0) { ++nz; src = c; }
        if (nz != 1) mono = false;
        b.src |= src << (2 * r);
      }
      b.kind = mono ? 2 : 1;
    }
    SVB_CUDA(cudaSetDevice(device));
    cudaStream_t st;
    SVB_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    BatchCirc* dc = nullptr;
    BatchGate* dg = nullptr;
    uint64_t* dcodes = nullptr;
    SVB_CUDA(cudaMallocAsync(&dc, sizeof(BatchCirc) * ncirc, st));
    SVB_CUDA(cudaMallocAsync(&dg, sizeof(BatchGate) * std::max(total_gates, 1), st));
    SVB_CUDA(cudaMallocAsync(&dcodes, sizeof(uint64_t) * shots * ncirc, st));
    SVB_CUDA(cudaMemcpyAsync(dc, hc.data(), sizeof(BatchCirc) * ncirc, cudaMemcpyHostToDevice, st));
    if (total_gates)
      SVB_CUDA(cudaMemcpyAsync(dg, hg.data(), sizeof(BatchGate) * total_gates, cudaMemcpyHostToDevice, st));
    int nsm = 148;
    SVB_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device));
    const size_t smem = 65536 + 8192 * sizeof(double);
    const unsigned grid = (unsigned)std::min(ncirc, nsm);
    if (precision == SVB_C128) {  // constant size: no race between threads
      SVB_CUDA(cudaFuncSetAttribute(k_batch_small<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      k_batch_small<double><<<grid, 256, smem, st>>>(dc, ncirc, dg, shots, dcodes);
    } else {
      SVB_CUDA(cudaFuncSetAttribute(k_batch_small<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      k_batch_small<float><<<grid, 256, smem, st>>>(dc, ncirc, dg, shots, dcodes);
    }
    SVB_CHECK_LAUNCH();
    SVB_CUDA(cudaMemcpyAsync(out_codes, dcodes, sizeof(uint64_t) * shots * ncirc, cudaMemcpyDeviceToHost, st));
    cudaFreeAsync(dc, st);
    cudaFreeAsync(dg, st);
    cudaFreeAsync(dcodes, st);
    SVB_CUDA(cudaStreamSynchronize(st));
    cudaStreamDestroy(st);
    return SVB_OK;
  } catch (const Error& e) {
    set_last_error(e.what());
    return e.code;
  }
}

// ------------------------------------------------ mid-circuit replay (smem)
// All shots of `_replay_shots` (statevector.py:157-179) for states that fit in
// shared memory.  Shot s uses PCG64 draws [s*M, (s+1)*M) (M = measures +
// resets in the suffix): the reference's single-stream order.  Ops: kind 0 =
// gate (index), 1 = measure (qubit, clbit rank), 2 = reset (qubit).
namespace svb {

template <typename R>
__device__ double block_sum_p1(const cplx<R>* st, uint32_t len, int q, double* red) {
  double acc = 0.0;
  for (uint32_t p = threadIdx.x; p < len / 2; p += blockDim.x) {
    const uint32_t i = (uint32_t)insert0(p, q) | (1u << q);
    const double x = (double)st[i].x, y = (double)st[i].y;
    acc += x * x + y * y;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31u) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  double t = 0.0;
  for (uint32_t w = 0; w < blockDim.x / 32; ++w) t += red[w];  // same order in every thread
  __syncthreads();
  return t;
}

template <typename R>
__global__ void __launch_bounds__(256, 1) k_replay_small(const cplx<R>* __restrict__ prefix, int n,
                                                         const int32_t* __restrict__ ops, int nops,
                                                         const BatchGate* __restrict__ gates, int M, uint64_t shots,
                                                         uint64_t pcg0, uint64_t pcg1, uint64_t pcg2, uint64_t pcg3,
                                                         uint64_t* __restrict__ codes) {
  extern __shared__ __align__(16) unsigned char smraw[];
  cplx<R>* st = reinterpret_cast<cplx<R>*>(smraw);
  __shared__ double red[8];
  const uint32_t len = 1u << n, tid = threadIdx.x;
  const u128b inc = ((u128b)pcg2 << 64) | pcg3, s0 = ((u128b)pcg0 << 64) | pcg1;
  for (uint64_t shot = blockIdx.x; shot < shots; shot += gridDim.x) {
    for (uint32_t i = tid; i < len; i += blockDim.x) st[i] = prefix[i];
    u128b am, ap;
    lcg_jump(inc, shot * (uint64_t)M, am, ap);
    u128b s = am * s0 + ap;  // state before this shot's first draw
    uint64_t code = 0;
    for (int k = 0; k < nops; ++k) {
      __syncthreads();
      const int kind = ops[3 * k], a = ops[3 * k + 1], b = ops[3 * k + 2];
      if (kind == 0) {
        const BatchGate& g = gates[a];
        if (g.kind == 0) {
          const int q = g.q0;
          const cplx<R> m0 = mk<R>((R)g.m[0], (R)g.m[1]), m1 = mk<R>((R)g.m[2], (R)g.m[3]);
          const cplx<R> m2 = mk<R>((R)g.m[4], (R)g.m[5]), m3 = mk<R>((R)g.m[6], (R)g.m[7]);
          for (uint32_t p = tid; p < len / 2; p += blockDim.x) {
            const uint32_t i0 = (uint32_t)insert0(p, q), i1 = i0 | (1u << q);
            const cplx<R> x0 = st[i0], x1 = st[i1];
            st[i0] = cfma<R>(m1, x1, cmul<R>(m0, x0));
            st[i1] = cfma<R>(m3, x1, cmul<R>(m2, x0));
          }
        } else {
          const int qa = g.q0, qb = g.q1;
          const int lo = qa < qb ? qa : qb, hi = qa < qb ? qb : qa;
          for (uint32_t p = tid; p < len / 4; p += blockDim.x) {
            const uint32_t base = (uint32_t)insert0(insert0(p, lo), hi);
            const uint32_t idx[4] = {base, base | (1u << qa), base | (1u << qb), base | (1u << qa) | (1u << qb)};
            cplx<R> x[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) x[j] = st[idx[j]];
#pragma unroll
            for (int r = 0; r < 4; ++r) {
              cplx<R> acc = mk<R>(R(0), R(0));
#pragma unroll
              for (int c = 0; c < 4; ++c)
                acc = cfma<R>(mk<R>((R)g.m[2 * (4 * r + c)], (R)g.m[2 * (4 * r + c) + 1]), x[c], acc);
              st[idx[r]] = acc;
            }
          }
        }
      } else {
        const int q = a;
        const double p1 = block_sum_p1<R>(st, len, q, red);
        s = s * mult128() + inc;
        const double u = pcg_out(s);
        const int out = u < p1 ? 1 : 0;
        const double p = out ? p1 : 1.0 - p1;
        const R sc = (R)(1.0 / sqrt(p));
        for (uint32_t pp = tid; pp < len / 2; pp += blockDim.x) {
          const uint32_t i0 = (uint32_t)insert0(pp, q), i1 = i0 | (1u << q);
          cplx<R> keep = out ? st[i1] : st[i0];
          keep.x *= sc;
          keep.y *= sc;
          const cplx<R> z = mk<R>(R(0), R(0));
          if (kind == 2 || !out) {  // reset: |1> -> X -> |0>
            st[i0] = keep;
            st[i1] = z;
          } else {
            st[i0] = z;
            st[i1] = keep;
          }
        }
        if (kind == 1) code = (code & ~(1ull << b)) | ((uint64_t)out << b);
      }
    }
    if (tid == 0) codes[shot] = code;
    __syncthreads();
  }
}

}  // namespace svb

extern "C" int svb_replay_small(int device, int precision, int n, const double* prefix_c128, const int32_t* ops,
                                int nops, const svb_gate* gates, int ngates, uint64_t shots, const uint64_t* pcg,
                                uint64_t* out_codes) {
  try {
    const int nmax = precision == SVB_C128 ? 12 : 13;
    require(n >= 1 && n <= nmax && shots >= 1 && nops >= 0 && ngates >= 0, SVB_E_ARG, "bad replay arguments");
    int M = 0;
    for (int k = 0; k < nops; ++k) {
      require(ops[3 * k] >= 0 && ops[3 * k] <= 2, SVB_E_ARG, "bad replay op");
      require(ops[3 * k] != 1 || (ops[3 * k + 2] >= 0 && ops[3 * k + 2] < 64), SVB_E_ARG,
              "replay: clbit rank must be in [0, 64)");
      if (ops[3 * k] != 0) ++M;
      else require(ops[3 * k + 1] >= 0 && ops[3 * k + 1] < ngates, SVB_E_ARG, "bad gate index");
    }
    std::vector<BatchGate> hg(ngates);
    for (int i = 0; i < ngates; ++i) {
      std::memcpy(hg[i].m, gates[i].mat, sizeof hg[i].m);
      hg[i].kind = gates[i].k == 1 ? 0 : 1;
      hg[i].q0 = gates[i].qubits[0];
      hg[i].q1 = gates[i].k == 2 ? gates[i].qubits[1] : 0;
      hg[i].src = 0;
    }
    const uint64_t len = 1ull << n;
    const size_t sz = precision == SVB_C128 ? 16 : 8;
    std::vector<unsigned char> hp(len * sz);
    for (uint64_t i = 0; i < len; ++i) {
      if (precision == SVB_C128) {
        double2 v = make_double2(prefix_c128[2 * i], prefix_c128[2 * i + 1]);
        std::memcpy(hp.data() + i * sz, &v, sz);
      } else {
        float2 v = make_float2((float)prefix_c128[2 * i], (float)prefix_c128[2 * i + 1]);
        std::memcpy(hp.data() + i * sz, &v, sz);
      }
    }
    SVB_CUDA(cudaSetDevice(device));
    cudaStream_t st;
    SVB_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    void* dpre = nullptr;
    int32_t* dops = nullptr;
    BatchGate* dg = nullptr;
    uint64_t* dcodes = nullptr;
    SVB_CUDA(cudaMallocAsync(&dpre, len * sz, st));
    SVB_CUDA(cudaMallocAsync(&dops, sizeof(int32_t) * 3 * std::max(nops, 1), st));
    SVB_CUDA(cudaMallocAsync(&dg, sizeof(BatchGate) * std::max(ngates, 1), st));
    SVB_CUDA(cudaMallocAsync(&dcodes, sizeof(uint64_t) * shots, st));
    SVB_CUDA(cudaMemcpyAsync(dpre, hp.data(), len * sz, cudaMemcpyHostToDevice, st));
    if (nops) SVB_CUDA(cudaMemcpyAsync(dops, ops, sizeof(int32_t) * 3 * nops, cudaMemcpyHostToDevice, st));
    if (ngates) SVB_CUDA(cudaMemcpyAsync(dg, hg.data(), sizeof(BatchGate) * ngates, cudaMemcpyHostToDevice, st));
    int nsm = 148;
    SVB_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device));
    const unsigned grid = (unsigned)std::min<uint64_t>(shots, (uint64_t)nsm * 2);
    const size_t smem = len * sz;
    if (precision == SVB_C128) {
      SVB_CUDA(cudaFuncSetAttribute(k_replay_small<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536));
      k_replay_small<double><<<grid, 256, smem, st>>>(static_cast<const double2*>(dpre), n, dops, nops, dg, M, shots,
                                                      pcg[0], pcg[1], pcg[2], pcg[3], dcodes);
    } else {
      SVB_CUDA(cudaFuncSetAttribute(k_replay_small<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536));
      k_replay_small<float><<<grid, 256, smem, st>>>(static_cast<const float2*>(dpre), n, dops, nops, dg, M, shots,
                                                     pcg[0], pcg[1], pcg[2], pcg[3], dcodes);
    }
    SVB_CHECK_LAUNCH();
    SVB_CUDA(cudaMemcpyAsync(out_codes, dcodes, sizeof(uint64_t) * shots, cudaMemcpyDeviceToHost, st));
    cudaFreeAsync(dpre, st);
    cudaFreeAsync(dops, st);
    cudaFreeAsync(dg, st);
    cudaFreeAsync(dcodes, st);
    SVB_CUDA(cudaStreamSynchronize(st));
    cudaStreamDestroy(st);
    return SVB_OK;
  } catch (const Error& e) {
    set_last_error(e.what());
    return e.code;
  }
}

// ------------------------------------------ batch of HBM-resident circuits
// Terminal circuits too large for the shared-memory kernel (config 4: 13-24
// qubits, `batch.run_batch`'s per-circuit `run_circuit(c, "sv", shots, seed)`
// loop, batch.py:104-222).  The whole batch is one C call: `nthreads` host
// workers, each with its own CUDA stream and state buffer (sized once for
// its largest circuit: circuits are taken largest first from a shared
// counter), schedule each circuit's fused program natively (program.cu; the
// NVRTC kernels of identical structures are shared), run it from a lazy
// |0...0> and draw the shots with the CDF sampler into one device code
// buffer.  No per-circuit host synchronisation: the codes come back with a
// single copy at the end.  status[i] = 0 or the svb_status of circuit i.
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <mutex>
#include <thread>
namespace {
std::mutex g_batch_pool_mu;
int g_batch_calls = 0;  // svb_batch_run calls in flight (pool release threshold)

// Per-device arena of the workers' state buffers and sampler scratch, kept
// across svb_batch_run calls.  Growing the stream-ordered pool by a few GiB at
// the start of every call stalled all workers for 8-600 ms (the growth waits
// for work already on the device, e.g. the shared-memory batch beside it);
// the arena is allocated once (cudaMalloc), grown only for a larger state,
// and released when a state allocation runs out of memory (state_malloc).
struct BatchArena {
  std::mutex mu;
  std::vector<void*> bufs;
  std::vector<double*> scratch;
  size_t buf_bytes = 0, scratch_doubles = 0;
  void release() {
    for (void* p : bufs) cudaFree(p);
    for (double* p : scratch) cudaFree(p);
    bufs.clear();
    scratch.clear();
    buf_bytes = scratch_doubles = 0;
  }
  // T buffers of >= bytes and scratch of >= sd doubles (caller holds mu)
  bool ensure(int T, size_t bytes, size_t sd) {
    if ((int)bufs.size() >= T && buf_bytes >= bytes && scratch_doubles >= sd) return true;
    release();
    for (int t = 0; t < T; ++t) {
      void* b = nullptr;
      double* d = nullptr;
      if (cudaMalloc(&b, bytes) != cudaSuccess || cudaMalloc(reinterpret_cast<void**>(&d), sizeof(double) * sd) != cudaSuccess) {
        if (b) cudaFree(b);
        cudaGetLastError();
        release();
        return false;
      }
      bufs.push_back(b);
      scratch.push_back(d);
    }
    buf_bytes = bytes;
    scratch_doubles = sd;
    return true;
  }
};
BatchArena g_arena[16];
}  // namespace

namespace svb {
// state_malloc's out-of-memory path: give the idle batch arenas back
void release_batch_arenas() {
  for (BatchArena& a : g_arena) {
    std::unique_lock<std::mutex> lk(a.mu, std::try_to_lock);
    if (lk.owns_lock()) a.release();
  }
}
}  // namespace svb

#include "jit.h"
#include "program.h"

namespace svb {
void expand_gate(const svb_gate_op& op, const svb_gate* fixed, svb_gate& g);
}

extern "C" int svb_batch_run(int device, int precision, int ncirc, const int32_t* nq, const int32_t* gate_off,
                             const int32_t* ngates, const svb_gate_op* ops, const svb_gate* fixed, int nfixed,
                             int total_gates, const uint64_t* pcg,
                             const int32_t* w, const int8_t* bit_src, uint64_t shots, int nthreads,
                             int jit_mode, uint64_t* out_codes, int32_t* status) {
  using namespace svb;
  try {
    require(ncirc >= 0 && shots >= 1 && nthreads >= 1, SVB_E_ARG, "bad batch arguments");
    if (ncirc == 0) return SVB_OK;
    std::vector<int> order(ncirc);
    for (int i = 0; i < ncirc; ++i) {
      status[i] = SVB_OK;
      order[i] = i;
      if (!(nq[i] >= 5 && nq[i] <= 36) || !(w[i] >= 1 && w[i] <= 63) ||
          !(gate_off[i] >= 0 && ngates[i] >= 0 && gate_off[i] + ngates[i] <= total_gates))
        status[i] = SVB_E_ARG;
      for (int p = 0; status[i] == SVB_OK && p < w[i]; ++p)
        if (bit_src[64 * i + p] < 0 || bit_src[64 * i + p] >= nq[i]) status[i] = SVB_E_ARG;
      for (int gi = 0; status[i] == SVB_OK && gi < ngates[i]; ++gi) {
        const svb_gate_op& g = ops[gate_off[i] + gi];
        if (g.kind < 0 || g.kind >= 4 + nfixed) {
          status[i] = SVB_E_ARG;
          break;
        }
        const int k = g.kind >= 4 ? fixed[g.kind - 4].k : 1;
        if (k < 1 || k > 2 || g.q0 < 0 || g.q0 >= nq[i] || (k == 2 && (g.q1 < 0 || g.q1 >= nq[i] || g.q1 == g.q0)))
          status[i] = SVB_E_ARG;
      }
    }
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return nq[a] > nq[b]; });
    SVB_CUDA(cudaSetDevice(device));
    const size_t s_amp = precision == SVB_C128 ? 16 : 8;
    int nmax = 0;
    for (int i = 0; i < ncirc; ++i)
      if (status[i] == SVB_OK) nmax = std::max(nmax, (int)nq[i]);
    const int T = std::min(nthreads, ncirc);
    BatchArena* arena = device >= 0 && device < 16 ? &g_arena[device] : nullptr;
    std::unique_lock<std::mutex> arena_lk;
    const auto ta0 = std::chrono::steady_clock::now();
    if (arena && nmax > 0) {  // a concurrent call uses the pool instead
      arena_lk = std::unique_lock<std::mutex>(arena->mu, std::try_to_lock);
      if (!arena_lk.owns_lock() || !arena->ensure(T, s_amp << nmax, cdf_scratch_doubles(nmax))) arena = nullptr;
    } else {
      arena = nullptr;
    }
    const double arena_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - ta0).count();
    // every buffer of the batch comes from the stream-ordered pool, kept
    // mapped for the whole call (cudaMalloc / cudaFree would synchronise the
    // device at every worker's start and end); trimmed back afterwards
    // (concurrent calls: the first one in raises the threshold, the last one
    // out restores it, so no call trims the pool under another's workers)
    cudaMemPool_t pool = nullptr;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
      std::lock_guard<std::mutex> lk(g_batch_pool_mu);
      if (g_batch_calls++ == 0) {
        uint64_t keep = ~0ull;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
      }
    }
    cudaGetLastError();
    cudaStream_t main_st;
    SVB_CUDA(cudaStreamCreateWithFlags(&main_st, cudaStreamNonBlocking));
    uint64_t* dcodes = nullptr;
    SVB_CUDA(cudaMallocAsync(&dcodes, sizeof(uint64_t) * shots * (uint64_t)ncirc, main_st));
    SVB_CUDA(cudaStreamSynchronize(main_st));
    static const bool prof = std::getenv("SVB_BATCH_PROFILE") != nullptr;
    std::atomic<int64_t> t_host_prog{0}, t_host_draw{0}, t_wait{0};
    // SVB_BATCH_TRACE=file: per circuit host timestamps and device start/end
    // events, appended as CSV (i, n, worker, host begin/launched/drawn us,
    // device begin/end us; all relative to the call's start)
    static const char* trace_path = std::getenv("SVB_BATCH_TRACE");
    struct TraceRec { int worker = -1; double h0 = 0, h1 = 0, h2 = 0; cudaEvent_t e0 = nullptr, e1 = nullptr; };
    std::vector<TraceRec> trace(trace_path ? ncirc : 0);
    const auto tr0 = std::chrono::steady_clock::now();
    cudaEvent_t tr_ev0 = nullptr;
    if (trace_path) {
      cudaEventCreate(&tr_ev0);
      cudaEventRecord(tr_ev0, main_st);
    }
    std::atomic<int> worker_ids{0};
    auto us_since = [&](std::chrono::steady_clock::time_point t) {
      return std::chrono::duration<double, std::micro>(t - tr0).count();
    };
    const size_t s = precision == SVB_C128 ? 16 : 8;
    // jit_mode 0: interpreter kernels up to 24 qubits, NVRTC above (no compile
    // in a config-4 batch; deterministic); 1: NVRTC from 24 qubits, compiled
    // synchronously (the engine sv.run uses: identical results); 2: as 1 but
    // compiled in the background while the interpreter serves (fastest once
    // warm; which engine ran, hence the last bits, depends on timing).
    require(jit_mode >= 0 && jit_mode <= 2, SVB_E_ARG, "bad jit mode");
    const int jit_min = jit_mode == 0 ? 25 : 24;
    std::atomic<int> next{0};
    std::mutex err_mu;
    std::string first_err;
    // SVB_BATCH_HEAVY=k: states that overflow L2 (>= 256 MB) run at most k at
    // a time (an experiment: 200 fresh 24-qubit circuits took 0.25 s on one
    // stream and 2-16 s on eight, but whole-batch timings did not improve)
    static const int heavy_max = std::getenv("SVB_BATCH_HEAVY") ? std::max(1, std::atoi(std::getenv("SVB_BATCH_HEAVY")))
                                                                 : 1 << 30;  // off unless set (no steady gain measured)
    std::mutex heavy_mu;
    std::condition_variable heavy_cv;
    int heavy_running = 0;
    auto worker = [&] {
      const int wid = worker_ids++;
      const bool own = arena == nullptr;  // buffers from the pool (else the arena's slot wid)
      cudaSetDevice(device);
      jit_set_async(jit_mode == 2);  // never wait for NVRTC: the interpreter runs until the kernels exist
      cudaStream_t st = nullptr;
      void *buf = nullptr, *spare = nullptr, *buf_pool = nullptr;
      double* cdf_scratch = nullptr;  // leaf sums / prefix of the CDF draw, sized for the worker's first (largest) circuit
      if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess) return;
      ProgramStats stats{};
      std::vector<svb_gate> gates;
      for (int j = next++; j < ncirc; j = next++) {
        const int i = order[j];
        if (status[i] != SVB_OK) continue;
        const int n = nq[i];
        const bool heavy = (s << n) >= (256ull << 20);
        if (heavy) {
          std::unique_lock<std::mutex> lk(heavy_mu);
          heavy_cv.wait(lk, [&] { return heavy_running < heavy_max; });
          ++heavy_running;
        }
        auto heavy_done = [&] {
          if (!heavy) return;
          cudaStreamSynchronize(st);  // its passes are done before another heavy circuit starts
          std::lock_guard<std::mutex> lk(heavy_mu);
          --heavy_running;
          heavy_cv.notify_one();
        };
        try {
          const auto c0 = std::chrono::steady_clock::now();
          if (trace_path) {
            trace[i].worker = wid;
            trace[i].h0 = us_since(c0);
            cudaEventCreate(&trace[i].e0);
            cudaEventCreate(&trace[i].e1);
            cudaEventRecord(trace[i].e0, st);
          }
          gates.resize(ngates[i]);
          for (int gi = 0; gi < ngates[i]; ++gi) expand_gate(ops[gate_off[i] + gi], fixed, gates[gi]);
          if (!buf) {  // largest first: the first size is the maximum
            if (own) {
              SVB_CUDA(cudaMallocAsync(&buf, s << n, st));
              SVB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&cdf_scratch), sizeof(double) * cdf_scratch_doubles(n), st));
            } else {
              buf = arena->bufs[wid];
              cdf_scratch = arena->scratch[wid];
            }
            buf_pool = buf;
          }
          bool zp = true;
          if (precision == SVB_C128)
            run_program_owned<double>(&buf, &spare, n, gates.data(), ngates[i], 1, jit_min, st, &stats, &zp);
          else
            run_program_owned<float>(&buf, &spare, n, gates.data(), ngates[i], 1, jit_min, st, &stats, &zp);
          if (zp) {
            if (precision == SVB_C128) launch_zero<double>(buf, n, st);
            else launch_zero<float>(buf, n, st);
          }
          const auto c1 = std::chrono::steady_clock::now();
          int32_t bs[64];
          for (int p = 0; p < 64; ++p) bs[p] = p < w[i] ? bit_src[64 * i + p] : 0;
          if (precision == SVB_C128)
            cdf_draw_scratch<double>(buf, n, shots, pcg + 4 * i, bs, w[i], dcodes + shots * i, st, cdf_scratch);
          else
            cdf_draw_scratch<float>(buf, n, shots, pcg + 4 * i, bs, w[i], dcodes + shots * i, st, cdf_scratch);
          if (trace_path) {
            cudaEventRecord(trace[i].e1, st);
            trace[i].h1 = us_since(c1);
            trace[i].h2 = us_since(std::chrono::steady_clock::now());
          }
          if (prof) {
            const auto c2 = std::chrono::steady_clock::now();
            t_host_prog += std::chrono::duration_cast<std::chrono::microseconds>(c1 - c0).count();
            t_host_draw += std::chrono::duration_cast<std::chrono::microseconds>(c2 - c1).count();
          }
        } catch (const Error& e) {
          status[i] = e.code;
          std::lock_guard<std::mutex> lk(err_mu);
          if (first_err.empty()) first_err = e.what();
        } catch (const std::exception& e) {
          status[i] = SVB_E_CUDA;
          std::lock_guard<std::mutex> lk(err_mu);
          if (first_err.empty()) first_err = e.what();
        }
        heavy_done();
      }
      jit_set_async(false);
      const auto w0 = std::chrono::steady_clock::now();
      // buf came from the pool; a spare the engine allocated (permutation
      // passes) came from cudaMalloc; the two may have been swapped
      void* pooled = buf_pool;
      void* other = buf == buf_pool ? spare : buf;
      if (own && pooled) cudaFreeAsync(pooled, st);
      if (own && cdf_scratch) cudaFreeAsync(cdf_scratch, st);
      cudaStreamSynchronize(st);
      if (other) cudaFree(other);
      if (prof) t_wait += std::chrono::duration_cast<std::chrono::microseconds>(std::chrono::steady_clock::now() - w0).count();
      cudaStreamDestroy(st);
    };
    std::vector<std::thread> th;
    for (int t = 0; t < T; ++t) th.emplace_back(worker);
    for (auto& t : th) t.join();
    const cudaError_t e = cudaMemcpyAsync(out_codes, dcodes, sizeof(uint64_t) * shots * (uint64_t)ncirc,
                                          cudaMemcpyDeviceToHost, main_st);
    cudaFreeAsync(dcodes, main_st);
    cudaStreamSynchronize(main_st);
    cudaStreamDestroy(main_st);
    if (trace_path) {
      if (FILE* f = std::fopen(trace_path, "a")) {
        for (int i = 0; i < ncirc; ++i) {
          const TraceRec& r = trace[i];
          float g0 = -1, g1 = -1;
          if (r.e0 && r.e1) {
            cudaEventElapsedTime(&g0, tr_ev0, r.e0);
            cudaEventElapsedTime(&g1, tr_ev0, r.e1);
          }
          std::fprintf(f, "%d,%d,%d,%.1f,%.1f,%.1f,%.1f,%.1f\n", i, nq[i], r.worker, r.h0, r.h1, r.h2, g0 * 1e3, g1 * 1e3);
          if (r.e0) cudaEventDestroy(r.e0);
          if (r.e1) cudaEventDestroy(r.e1);
        }
        std::fprintf(f, "end,%.1f\n", us_since(std::chrono::steady_clock::now()));
        std::fclose(f);
      }
      cudaEventDestroy(tr_ev0);
      cudaGetLastError();
    }
    if (pool) {  // back to the library's usual threshold (keep_pool_mapped) and release the rest
      std::lock_guard<std::mutex> lk(g_batch_pool_mu);
      if (--g_batch_calls == 0) {
        uint64_t keep = 1ull << 30;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
        cudaMemPoolTrimTo(pool, keep);
      }
    }
    if (prof)
      std::fprintf(stderr, "[svb] batch_run %d circuits: arena %.1f ms, setup %.1f ms, host program %.1f ms, host draw %.1f ms, final wait %.1f ms (summed over workers), total %.1f ms\n",
                   ncirc, arena_ms, std::chrono::duration<double, std::milli>(tr0 - ta0).count() - arena_ms,
                   t_host_prog / 1e3, t_host_draw / 1e3, t_wait / 1e3,
                   std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - ta0).count());
    SVB_CUDA(e);
    if (!first_err.empty()) set_last_error(first_err.c_str());
    return SVB_OK;
  } catch (const Error& e) {
    set_last_error(e.what());
    return e.code;
  }
}

// ------------------------------------------------ compact gate records
// 40-byte (kind, qubits, params) records expanded to svb_gate matrices in
// C++ (batch workers expand their own circuits in parallel).  Parametric
// kinds evaluate gates.py's formulas (gates.py:43-65) with the same libm
// calls numpy / math make; fixed kinds copy `fixed[kind]` (the exact
// matrices gates.py holds, passed in by the caller).
namespace svb {
enum : int32_t { GK_RX = 0, GK_RY = 1, GK_RZ = 2, GK_U = 3, GK_FIXED = 4 };

void expand_gate(const svb_gate_op& op, const svb_gate* fixed, svb_gate& g) {
  if (op.kind >= GK_FIXED) {
    g = fixed[op.kind - GK_FIXED];
  } else {
    std::memset(&g, 0, sizeof g);
    g.k = 1;
    double* m = g.mat;
    const double t = op.p[0];
    if (op.kind == GK_RZ) {  // np.exp(-0.5j t), np.exp(0.5j t)
      m[0] = std::cos(-0.5 * t);
      m[1] = std::sin(-0.5 * t);
      m[6] = std::cos(0.5 * t);
      m[7] = std::sin(0.5 * t);
    } else {
      const double c = std::cos(t / 2), s = std::sin(t / 2);
      if (op.kind == GK_RX) {  // [[c, -1j s], [-1j s, c]]
        m[0] = c;
        m[2] = -0.0 * s;
        m[3] = -s;
        m[4] = -0.0 * s;
        m[5] = -s;
        m[6] = c;
      } else if (op.kind == GK_RY) {
        m[0] = c;
        m[2] = -s;
        m[4] = s;
        m[6] = c;
      } else {  // u(t, p, l): [[c, -e^{il} s], [e^{ip} s, e^{i(p+l)} c]]
        const double p = op.p[1], l = op.p[2];
        m[0] = c;
        m[2] = -std::cos(l) * s;
        m[3] = -std::sin(l) * s;
        m[4] = std::cos(p) * s;
        m[5] = std::sin(p) * s;
        m[6] = std::cos(p + l) * c;
        m[7] = std::sin(p + l) * c;
      }
    }
  }
  g.qubits[0] = op.q0;
  g.qubits[1] = g.k == 2 ? op.q1 : 0;
}
}  // namespace svb

extern "C" int svb_expand_gates(const svb_gate_op* ops, int n, const svb_gate* fixed, svb_gate* out) {
  for (int i = 0; i < n; ++i) svb::expand_gate(ops[i], fixed, out[i]);
  return SVB_OK;
}
