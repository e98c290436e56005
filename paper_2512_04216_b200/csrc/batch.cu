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
