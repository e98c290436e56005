// Per-gate kernels: one HBM pass per 1q/2q gate.
//
// These restate the reference gate kernels `apply_1q` (statevector.py:33-53)
// and `apply_2q` (statevector.py:71-113) one gate at a time.  They serve the
// kernel-level API (svb_apply on a single gate) and are the unfused baseline
// the fused pass kernel (gates_fused.cu) is checked against.  Special-cased
// structure (diagonal / anti-diagonal / monomial) is detected on the host and
// dispatched to cheaper kernels that skip the multiply-adds.
#include "common.cuh"
#include "kernels.h"

namespace svb {

template <typename R> struct M2 { cplx<R> m[4]; };
template <typename R> struct M4 { cplx<R> m[16]; };

template <typename R>
__global__ void k_gate1_dense(cplx<R>* __restrict__ s, uint64_t npairs, int q, M2<R> g) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t bit = 1ull << q;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < npairs; i += stride) {
    uint64_t i0 = insert0(i, q), i1 = i0 | bit;
    cplx<R> a0 = s[i0], a1 = s[i1];
    cplx<R> b0 = cmul<R>(g.m[0], a0), b1 = cmul<R>(g.m[2], a0);
    s[i0] = cfma<R>(g.m[1], a1, b0);
    s[i1] = cfma<R>(g.m[3], a1, b1);
  }
}

// diag(d0, d1) or antidiag: out0 = m01 a1, out1 = m10 a0
template <typename R>
__global__ void k_gate1_mono(cplx<R>* __restrict__ s, uint64_t npairs, int q, cplx<R> f0,
                             cplx<R> f1, int swap) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t bit = 1ull << q;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < npairs; i += stride) {
    uint64_t i0 = insert0(i, q), i1 = i0 | bit;
    cplx<R> a0 = s[i0], a1 = s[i1];
    if (swap) { cplx<R> t = a0; a0 = a1; a1 = t; }
    s[i0] = cmul<R>(f0, a0);
    s[i1] = cmul<R>(f1, a1);
  }
}

// Dense or monomial 4x4 on (qa, qb); local index = bit(qa) + 2 bit(qb).
template <typename R>
__global__ void k_gate2(cplx<R>* __restrict__ s, uint64_t nquads, int qa, int qb, M4<R> g,
                        int mono, int4 src) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const int lo = qa < qb ? qa : qb, hi = qa < qb ? qb : qa;
  const uint64_t ba = 1ull << qa, bb = 1ull << qb;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nquads; i += stride) {
    uint64_t base = insert0(insert0(i, lo), hi);
    uint64_t idx[4] = {base, base | ba, base | bb, base | ba | bb};
    cplx<R> a[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) a[k] = s[idx[k]];
    if (mono) {
      const int sr[4] = {src.x, src.y, src.z, src.w};
#pragma unroll
      for (int r = 0; r < 4; ++r) s[idx[r]] = cmul<R>(g.m[r * 4 + sr[r]], a[sr[r]]);
    } else {
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        cplx<R> acc = cmul<R>(g.m[r * 4], a[0]);
        acc = cfma<R>(g.m[r * 4 + 1], a[1], acc);
        acc = cfma<R>(g.m[r * 4 + 2], a[2], acc);
        acc = cfma<R>(g.m[r * 4 + 3], a[3], acc);
        s[idx[r]] = acc;
      }
    }
  }
}

template <typename R>
__global__ void k_zero_state(cplx<R>* __restrict__ s, uint64_t len) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < len; i += stride)
    s[i] = mk<R>(i == 0 ? R(1) : R(0), R(0));
}

static inline bool is_zero(const double* c) { return c[0] == 0.0 && c[1] == 0.0; }

template <typename R>
void launch_gate_basic(void* state, int n, const svb_gate& g, cudaStream_t st) {
  cplx<R>* s = static_cast<cplx<R>*>(state);
  const int B = 256;
  if (g.k == 1) {
    const double* m = g.mat;
    uint64_t np = 1ull << (n - 1);
    int q = g.qubits[0];
    bool diag = is_zero(m + 2) && is_zero(m + 4);
    bool anti = is_zero(m + 0) && is_zero(m + 6);
    if (diag || anti) {
      cplx<R> f0 = diag ? mk<R>((R)m[0], (R)m[1]) : mk<R>((R)m[2], (R)m[3]);
      cplx<R> f1 = diag ? mk<R>((R)m[6], (R)m[7]) : mk<R>((R)m[4], (R)m[5]);
      k_gate1_mono<R><<<grid_for(np, B), B, 0, st>>>(s, np, q, f0, f1, anti ? 1 : 0);
    } else {
      M2<R> mm;
      for (int i = 0; i < 4; ++i) mm.m[i] = mk<R>((R)m[2 * i], (R)m[2 * i + 1]);
      k_gate1_dense<R><<<grid_for(np, B), B, 0, st>>>(s, np, q, mm);
    }
  } else {
    M4<R> mm;
    int src[4];
    bool mono = true;
    for (int r = 0; r < 4; ++r) {
      int nz = 0;
      src[r] = 0;
      for (int c = 0; c < 4; ++c) {
        mm.m[r * 4 + c] = mk<R>((R)g.mat[2 * (r * 4 + c)], (R)g.mat[2 * (r * 4 + c) + 1]);
        if (!is_zero(g.mat + 2 * (r * 4 + c))) { ++nz; src[r] = c; }
      }
      if (nz != 1) mono = false;
    }
    uint64_t nqd = 1ull << (n - 2);
    k_gate2<R><<<grid_for(nqd, B), B, 0, st>>>(s, nqd, g.qubits[0], g.qubits[1], mm, mono ? 1 : 0,
                                               make_int4(src[0], src[1], src[2], src[3]));
  }
  SVB_CHECK_LAUNCH();
}

template <typename R> void launch_zero(void* state, int n, cudaStream_t st) {
  uint64_t len = 1ull << n;
  k_zero_state<R><<<grid_for(len, 256), 256, 0, st>>>(static_cast<cplx<R>*>(state), len);
  SVB_CHECK_LAUNCH();
}

template void launch_gate_basic<float>(void*, int, const svb_gate&, cudaStream_t);
template void launch_gate_basic<double>(void*, int, const svb_gate&, cudaStream_t);
template void launch_zero<float>(void*, int, cudaStream_t);
template void launch_zero<double>(void*, int, cudaStream_t);

}  // namespace svb
