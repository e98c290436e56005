// Device code shared by the libsvb kernels (nvcc) and the JIT-compiled pass
// kernels (NVRTC): complex arithmetic, the op/pass data layout, the per-thread
// op interpreter, and the persistent fused-pass skeleton.  No host-only
// includes here: NVRTC compiles this header as-is.
#pragma once
#ifndef __CUDACC_RTC__
#include <stddef.h>
#include <stdint.h>
#ifndef __CUDACC_RTC__
#include <cstdlib>
#endif
#else
typedef unsigned long long uint64_t;
typedef long long int64_t;
typedef unsigned int uint32_t;
typedef unsigned short uint16_t;
typedef int int32_t;
typedef signed char int8_t;
typedef unsigned char uint8_t;
#endif

namespace svb {

// ---- complex arithmetic on float2 / double2 --------------------------------
template <typename R> struct CT;
template <> struct CT<float> { using T = float2; };
template <> struct CT<double> { using T = double2; };
template <typename R> using cplx = typename CT<R>::T;

template <typename R> __host__ __device__ __forceinline__ cplx<R> mk(R x, R y) {
  cplx<R> r; r.x = x; r.y = y; return r;
}
// complex64 on sm_100: both components of a complex value go through one
// packed f32x2 instruction (FFMA2 / FMUL2, each lane an IEEE fp32 operation
// rounded to nearest, as the scalar form).  The scalar-operand broadcast and
// the swapped / lane-negated operand are FFMA2 operand modifiers, so a complex
// multiply-add is 2 instructions instead of 4 and the Sycamore-style c64
// passes, which were issue-bound, issue half the FMA instructions.
#if defined(__CUDA_ARCH__) && __CUDA_ARCH__ >= 1000 && !defined(SVB_NO_FFMA2)
#define SVB_FFMA2 1
#endif
template <typename R>
__host__ __device__ __forceinline__ cplx<R> cmul(cplx<R> a, cplx<R> b) {
#ifdef SVB_FFMA2
  if constexpr (sizeof(R) == 4)
    return __ffma2_rn(make_float2(a.y, a.y), make_float2(-b.y, b.x), __fmul2_rn(make_float2(a.x, a.x), b));
  else
#endif
    return mk<R>(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
// acc + a*b
template <typename R>
__host__ __device__ __forceinline__ cplx<R> cfma(cplx<R> a, cplx<R> b, cplx<R> acc) {
#ifdef SVB_FFMA2
  if constexpr (sizeof(R) == 4)
    return __ffma2_rn(make_float2(a.y, a.y), make_float2(-b.y, b.x), __ffma2_rn(make_float2(a.x, a.x), b, acc));
  else
#endif
  {
    acc.x = fma(a.x, b.x, acc.x); acc.x = fma(-a.y, b.y, acc.x);
    acc.y = fma(a.x, b.y, acc.y); acc.y = fma(a.y, b.x, acc.y);
    return acc;
  }
}
// acc + a*b as four scalar FMAs: for loops bound by the FMA pipe itself (the
// dense-block engine), where FFMA2 with the swapped operand measured ~20%
// fewer FMAs per clock (profiles/r02_fma_pipe_microbench.txt)
template <typename R>
__host__ __device__ __forceinline__ cplx<R> cfma_scalar(cplx<R> a, cplx<R> b, cplx<R> acc) {
  acc.x = fma(a.x, b.x, acc.x); acc.x = fma(-a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y); acc.y = fma(a.y, b.x, acc.y);
  return acc;
}
// s*x, acc + s*x and acc + i*s*x for a real s
template <typename R> __host__ __device__ __forceinline__ cplx<R> rmul(R s, cplx<R> x) {
#ifdef SVB_FFMA2
  if constexpr (sizeof(R) == 4) return __fmul2_rn(make_float2(s, s), x);
  else
#endif
    return mk<R>(s * x.x, s * x.y);
}
template <typename R> __host__ __device__ __forceinline__ cplx<R> rfma(R s, cplx<R> x, cplx<R> acc) {
#ifdef SVB_FFMA2
  if constexpr (sizeof(R) == 4) return __ffma2_rn(make_float2(s, s), x, acc);
  else
#endif
    return mk<R>(fma(s, x.x, acc.x), fma(s, x.y, acc.y));
}
template <typename R> __host__ __device__ __forceinline__ cplx<R> ifma(R s, cplx<R> x, cplx<R> acc) {
#ifdef SVB_FFMA2
  if constexpr (sizeof(R) == 4) return __ffma2_rn(make_float2(s, s), make_float2(-x.y, x.x), acc);
  else
#endif
    return mk<R>(fma(-s, x.y, acc.x), fma(s, x.x, acc.y));
}
// i*s*x
template <typename R> __host__ __device__ __forceinline__ cplx<R> imul(R s, cplx<R> x) {
#ifdef SVB_FFMA2
  if constexpr (sizeof(R) == 4) return __fmul2_rn(make_float2(s, s), make_float2(-x.y, x.x));
  else
#endif
    return mk<R>(-s * x.y, s * x.x);
}
template <typename R> __host__ __device__ __forceinline__ R norm2(cplx<R> a) {
  return a.x * a.x + a.y * a.y;
}

// insert a zero bit at position q
__host__ __device__ __forceinline__ uint64_t insert0(uint64_t i, int q) {
  uint64_t lo = i & ((1ull << q) - 1ull);
  return ((i >> q) << (q + 1)) | lo;
}

// OP_U1P / OP_U1PR: unit-pivot 1q op y_r = x_pc[r] + ratio_r * x_(1-pc[r])
// (pc bits in OpHdr::n; payload ratio_0, ratio_1; PR = both ratios real)
enum : int32_t { OP_DIAG = 0, OP_U1 = 1, OP_U1ANTI = 2, OP_U2 = 3, OP_PERM2 = 4, OP_U1R = 5, OP_U1X = 6,
                 OP_U1P = 7, OP_U1PR = 8 };

// Every op: header, then a kind-specific payload.  `bytes` = total size
// (multiple of 16).  Condition: the op applies where
// (Fg & fmask) == fval  and  (v & rmask) == rval  (v = register index).
struct alignas(16) OpHdr {
  int32_t kind, a, b, n;      // a, b: register bits; n: DIAG term count
  uint64_t fmask, fval;       // condition on fixed global index bits
  uint32_t rmask, rval, bytes, pad;
};
static_assert(sizeof(OpHdr) == 48, "OpHdr layout");
constexpr uint32_t kOpHdrBytesOff = 40;  // offsetof(OpHdr, bytes) (no offsetof under NVRTC)
#ifndef __CUDACC_RTC__
static_assert(offsetof(OpHdr, bytes) == kOpHdrBytesOff, "OpHdr layout");
#endif

// Diagonal factor d[bit(qa) + 2 bit(qb)]; ra/rb = register bit or -1 (then
// the bit is read from the fixed global index at position qa/qb; q = -1 -> 0).
template <typename R> struct alignas(16) DiagTerm {
  int8_t ra, rb, qa, qb;
  int32_t pad[3];
  cplx<R> d[4];
};

// DIAG payload: DiagHdr, then DiagTerm entries in class order
//   UR (register bit i x tile bit, grouped by i) | UC (tile x tile) |
//   UT (thread bit x tile bit, grouped by thread qubit) |
//   TR (register bit x thread bit) | TC (thread-bit constants) | RR (register x register)
// Classes U* depend only on the tile index and are evaluated once per tile per
// CTA into the pass's uniform slots (shared memory); T* and RR per thread.
// A UT term stores, per tile-bit value f, the constant part d[2f] = e(0, f)
// (folded into the slot's C) and the ratio d[2f+1] = e(1, f) / e(0, f) that
// the thread applies when its thread bit is set (group product V[g]).
struct alignas(16) DiagHdr {
  int32_t nUR[6];
  int32_t nUC, nTR, nTC, nRR;
  int32_t slot;
  int32_t nUTg;       // UT groups (one per thread qubit)
  uint8_t utn[16];    // terms per UT group
};
static_assert(sizeof(DiagHdr) == 64, "DiagHdr layout");
constexpr int kMaxUT = 12;
// cplx per uniform slot: C, U0[5], U1[5], V[kMaxUT], pad
constexpr int kUniStride = 24;
// one-round direct passes: tile-uniform factors are produced kUPipeAhead tiles
// ahead into a ring of 2 * kUPipeAhead + 1 shared-memory slots (pass_kernel)
// (SVB_UPIPE_AHEAD: experiments; the JIT defines it from the environment)
#ifndef SVB_UPIPE_AHEAD
#define SVB_UPIPE_AHEAD 1
#endif
// SVB_UWAIT_FIRST: wait for the tile's uniform slot before issuing its loads
// SVB_BULK_ROWS (set by the JIT per kernel): the one-round direct pass stores
// its tile through shared memory with one 4 KB bulk copy per register row
// (thread bits = the state's lowest qubits, so each row is one contiguous run)
#ifndef SVB_BULK_ROWS
#define SVB_BULK_ROWS 0
#endif
#ifndef SVB_UPIPE_PROBE
// timing probes only (results are wrong): 1 = skip the uniform-slot waits,
// 2 = also skip evaluating the uniform factors
#define SVB_UPIPE_PROBE 0
#endif
#ifndef SVB_UWAIT_FIRST
#define SVB_UWAIT_FIRST 0
#endif
// SVB_UIN: the JIT body waits for the tile's slot before its first uniform
// factor (pass_kernel's UIN; needs one more slot).  Measured slower: off.
#ifndef SVB_UIN
#define SVB_UIN 0
#endif
// SVB_UGROUP: tiles per ring slot (one wait + one arrive per group of tiles;
// the default loop path only)
#ifndef SVB_UGROUP
#define SVB_UGROUP 1
#endif
constexpr int kUPipeAhead = SVB_UPIPE_AHEAD, kUPipeSlots = 2 * kUPipeAhead + 1 + (SVB_UIN ? 1 : 0);
constexpr int kUGroup = SVB_UGROUP;
constexpr int kUniV = 11;

constexpr int kMaxRounds = 24;
constexpr int kMaxM = 14;
constexpr int kMaxDiag = 48;
constexpr int kMaxItems = 256;

struct RoundDev {
  int32_t reg_local[8];  // local bit of register bit i
  uint32_t op_off, op_end;
  uint32_t regmask_local, pad;
  // local bit of thread-index bit tb (the non-register local bits; ascending
  // except in a permuted-store round, whose lanes sit on the bits that land
  // on output qubits 0..4)
  uint8_t thr_local[16];
};

struct PassDev {
  int32_t m, nrounds, nout, rb;
  int32_t pos[16];      // physical qubit of local bit l
  int32_t outpos[48];   // physical qubits outside S, ascending (tile index bits)
  RoundDev rounds[kMaxRounds];
  int32_t ndiag;
  uint32_t ops_begin, ops_bytes;  // this pass's slice of the op stream (staged in smem)
  int32_t direct;                 // round 0 has no lane register bits (see pass_kernel)
  uint32_t diag_off[kMaxDiag];  // op-stream offsets of this pass's DIAG payloads
  // tile-uniform work items (one per non-empty UR register bit, constant and
  // UT group of each uniform DIAG payload): d | kind << 8 | index << 10,
  // kind 0 = UR, 1 = constant, 2 = UT group
  int32_t nitems;
  // permuted store (the program's final qubit permutation fused into its last
  // pass): the last round writes out-of-place to bit dest(p) for every
  // physical bit p; dpos[l] = dest(pos[l]), doutpos[i] = dest(outpos[i])
  int32_t perm_out;
  // fused <Z_q> sums (last pass of an apply that asked for single-qubit <Z>):
  // sums of p (-1)^bit for every register bit of the last round, every
  // thread bit and every tile bit, plus sum p, accumulate in zacc (see
  // zsum_tile; reduced by k_zsum_finish)
  int32_t zsum;
  int32_t pad2;
  uint16_t items[kMaxItems];
  int32_t dpos[16];
  int32_t doutpos[48];
  uint64_t zacc;
  // zero_start support tracking: positions of the tile with a bit in dmask are
  // |0...0>-only so far (never written): the loader synthesises zeros there
  uint64_t dmask;
  // fused initial permutation (first pass of a program on a written input
  // whose swap relabeling needs the input in another qubit order): the tile
  // loads read the input buffer at bit ipos[l] for local bit l and ioutpos[i]
  // for tile bit i, and the pass stores into the output buffer in the
  // program's layout.  ld_local[b]: the local bit of load-order bit b (the
  // low load-order bits are the threads', so they are the local bits with
  // the lowest input positions: the loads stay coalesced).
  int32_t perm_in;
  int32_t pad3[3];
  int32_t ipos[16];
  int32_t ioutpos[48];
  uint8_t ld_local[16];
};
static_assert(sizeof(PassDev) % 16 == 0, "PassDev is copied in 16-byte units");
constexpr uint32_t kMaxPassOpBytes = 72 * 1024;
constexpr int kZaccRows = 64, kZaccCols = 1024;  // fused <Z>: values, CTAs (grid <= kZaccCols)
// fused <Z> accumulators (doubles) for up to kZaccCols CTAs of nthr threads
__host__ __device__ constexpr uint64_t zacc_doubles(uint32_t nthr, int rb) {
  return (uint64_t)kZaccCols * ((uint64_t)(rb + 1) * nthr + (nthr >> 5) * 64u);
}

// ------------------------------------------------------------ interpreter
#define SVB_HD __host__ __device__ __forceinline__

// op data is staged in shared memory by the pass kernel: plain loads
template <typename T> SVB_HD T ldop(const T* p) { return *p; }
template <typename R> SVB_HD cplx<R> ldc(const cplx<R>* p) { return *p; }

template <typename R, int RB, int B, bool COND>
SVB_HD void u1_dense(cplx<R>* a, const cplx<R>* m, uint32_t rmask, uint32_t rval) {
  const cplx<R> m0 = ldc<R>(m), m1 = ldc<R>(m + 1), m2 = ldc<R>(m + 2), m3 = ldc<R>(m + 3);
#pragma unroll
  for (int v = 0; v < (1 << RB); ++v) {
    if (v & (1 << B)) continue;
    if (COND && (v & rmask) != rval) continue;
    cplx<R> x0 = a[v], x1 = a[v | (1 << B)];
    a[v] = cfma<R>(m1, x1, cmul<R>(m0, x0));
    a[v | (1 << B)] = cfma<R>(m3, x1, cmul<R>(m2, x0));
  }
}

// real 2x2 (h, ry, ...): half the multiplies of the complex form
template <typename R, int RB, int B, bool COND>
SVB_HD void u1_real(cplx<R>* a, const cplx<R>* m, uint32_t rmask, uint32_t rval) {
  const R m0 = ldc<R>(m).x, m1 = ldc<R>(m + 1).x, m2 = ldc<R>(m + 2).x, m3 = ldc<R>(m + 3).x;
#pragma unroll
  for (int v = 0; v < (1 << RB); ++v) {
    if (v & (1 << B)) continue;
    if (COND && (v & rmask) != rval) continue;
    const cplx<R> x0 = a[v], x1 = a[v | (1 << B)];
    a[v] = rfma<R>(m1, x1, rmul<R>(m0, x0));
    a[v | (1 << B)] = rfma<R>(m3, x1, rmul<R>(m2, x0));
  }
}

// [[a, i b], [i c, d]] with a, b, c, d real (rx-like: sqrt(X), rx(t)): 4 FMA per output
template <typename R, int RB, int B, bool COND>
SVB_HD void u1_rx(cplx<R>* a, const cplx<R>* m, uint32_t rmask, uint32_t rval) {
  const R ma = ldc<R>(m).x, mb = ldc<R>(m + 1).y, mc = ldc<R>(m + 2).y, md = ldc<R>(m + 3).x;
#pragma unroll
  for (int v = 0; v < (1 << RB); ++v) {
    if (v & (1 << B)) continue;
    if (COND && (v & rmask) != rval) continue;
    const cplx<R> x0 = a[v], x1 = a[v | (1 << B)];
    a[v] = ifma<R>(mb, x1, rmul<R>(ma, x0));
    a[v | (1 << B)] = ifma<R>(mc, x0, rmul<R>(md, x1));
  }
}

// [[0, m1], [m2, 0]]
template <typename R, int RB, int B, bool COND>
SVB_HD void u1_anti(cplx<R>* a, const cplx<R>* m, uint32_t rmask, uint32_t rval) {
  const cplx<R> m1 = ldc<R>(m + 1), m2 = ldc<R>(m + 2);
  const bool plain = m1.x == R(1) && m1.y == R(0) && m2.x == R(1) && m2.y == R(0);
  if (plain) {
#pragma unroll
    for (int v = 0; v < (1 << RB); ++v) {
      if (v & (1 << B)) continue;
      if (COND && (v & rmask) != rval) continue;
      const cplx<R> x0 = a[v];
      a[v] = a[v | (1 << B)];
      a[v | (1 << B)] = x0;
    }
  } else {
#pragma unroll
    for (int v = 0; v < (1 << RB); ++v) {
      if (v & (1 << B)) continue;
      if (COND && (v & rmask) != rval) continue;
      const cplx<R> x0 = a[v], x1 = a[v | (1 << B)];
      a[v] = cmul<R>(m1, x1);
      a[v | (1 << B)] = cmul<R>(m2, x0);
    }
  }
}

// one output row of a unit-pivot op: p + r*o; RK: 0 r = 0, 1 real, 2 imaginary, 3 complex
template <typename R, int RK> SVB_HD cplx<R> piv_row(cplx<R> p, cplx<R> o, cplx<R> r) {
  if constexpr (RK == 0) return p;
  else if constexpr (RK == 1) return rfma<R>(r.x, o, p);
  else if constexpr (RK == 2) return ifma<R>(r.y, o, p);
  else return cfma<R>(r, o, p);
}

template <typename R, int RB, int B, int PC0, int PC1, int RK0, int RK1>
SVB_HD void u1_piv(cplx<R>* a, cplx<R> r0, cplx<R> r1) {
#pragma unroll
  for (int v = 0; v < (1 << RB); ++v) {
    if (v & (1 << B)) continue;
    const cplx<R> x0 = a[v], x1 = a[v | (1 << B)];
    a[v] = piv_row<R, RK0>(PC0 ? x1 : x0, PC0 ? x0 : x1, r0);
    a[v | (1 << B)] = piv_row<R, RK1>(PC1 ? x1 : x0, PC1 ? x0 : x1, r1);
  }
}

// u1_piv with registers known to be zero (bit v of ZM: a[v] == 0, e.g. the
// never-written positions of a support-tracked pass): no work on zero
// operands (JIT only; the generator tracks ZM through the ops)
template <typename R, int RK> SVB_HD cplx<R> piv_mul(cplx<R> o, cplx<R> r) {  // r*o
  if constexpr (RK == 0) return mk<R>(R(0), R(0));
  else if constexpr (RK == 1) return rmul<R>(r.x, o);
  else if constexpr (RK == 2) return imul<R>(r.y, o);
  else return cmul<R>(r, o);
}
template <typename R, int RK, bool PZ, bool OZ> SVB_HD cplx<R> piv_row_z(cplx<R> p, cplx<R> o, cplx<R> r) {
  if constexpr (PZ && OZ) return mk<R>(R(0), R(0));
  else if constexpr (OZ) return p;
  else if constexpr (PZ) return piv_mul<R, RK>(o, r);
  else return piv_row<R, RK>(p, o, r);
}
template <typename R, int RB, int B, int PC0, int PC1, int RK0, int RK1, uint32_t ZM>
SVB_HD void u1_piv_z(cplx<R>* a, cplx<R> r0, cplx<R> r1) {
#pragma unroll
  for (int v = 0; v < (1 << RB); ++v) {
    if (v & (1 << B)) continue;
    const int w = v | (1 << B);
    const cplx<R> x0 = a[v], x1 = a[w];
    if (((ZM >> v) & 1u) && ((ZM >> w) & 1u)) continue;
    if ((ZM >> v) & 1u) {
      a[v] = PC0 ? piv_row_z<R, RK0, false, true>(x1, x0, r0) : piv_row_z<R, RK0, true, false>(x0, x1, r0);
      a[w] = PC1 ? piv_row_z<R, RK1, false, true>(x1, x0, r1) : piv_row_z<R, RK1, true, false>(x0, x1, r1);
    } else if ((ZM >> w) & 1u) {
      a[v] = PC0 ? piv_row_z<R, RK0, true, false>(x1, x0, r0) : piv_row_z<R, RK0, false, true>(x0, x1, r0);
      a[w] = PC1 ? piv_row_z<R, RK1, true, false>(x1, x0, r1) : piv_row_z<R, RK1, false, true>(x0, x1, r1);
    } else {
      a[v] = piv_row<R, RK0>(PC0 ? x1 : x0, PC0 ? x0 : x1, r0);
      a[w] = piv_row<R, RK1>(PC1 ? x1 : x0, PC1 ? x0 : x1, r1);
    }
  }
}

// op-stream form (interpreter and structure-only JIT): ratios from the payload
template <typename R, int RB, int B, int PC, bool REAL>
SVB_HD void u1_piv_p(cplx<R>* a, const cplx<R>* r) {
  constexpr int RK = REAL ? 1 : 3;
  u1_piv<R, RB, B, (PC & 1), (PC >> 1), RK, RK>(a, ldc<R>(r), ldc<R>(r + 1));
}

template <typename R, int RB, int B1, int B2>
SVB_HD void u2_dense(cplx<R>* a, const cplx<R>* m, uint32_t rmask, uint32_t rval) {
#pragma unroll
  for (int v = 0; v < (1 << RB); ++v) {
    if (v & ((1 << B1) | (1 << B2))) continue;
    if ((v & rmask) != rval) continue;
    const int i0 = v, i1 = v | (1 << B1), i2 = v | (1 << B2), i3 = v | (1 << B1) | (1 << B2);
    cplx<R> x[4] = {a[i0], a[i1], a[i2], a[i3]};
    cplx<R> y[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      cplx<R> acc = cmul<R>(ldc<R>(m + 4 * r), x[0]);
      acc = cfma<R>(ldc<R>(m + 4 * r + 1), x[1], acc);
      acc = cfma<R>(ldc<R>(m + 4 * r + 2), x[2], acc);
      acc = cfma<R>(ldc<R>(m + 4 * r + 3), x[3], acc);
      y[r] = acc;
    }
    a[i0] = y[0]; a[i1] = y[1]; a[i2] = y[2]; a[i3] = y[3];
  }
}

// out[r] = ph[r] * in[src[r]]
template <typename R, int RB, int B1, int B2>
SVB_HD void u2_perm(cplx<R>* a, const int32_t* src, const cplx<R>* ph, uint32_t rmask, uint32_t rval) {
  const int s0 = ldop(src), s1 = ldop(src + 1), s2 = ldop(src + 2), s3 = ldop(src + 3);
  const cplx<R> p0 = ldc<R>(ph), p1 = ldc<R>(ph + 1), p2 = ldc<R>(ph + 2), p3 = ldc<R>(ph + 3);
#pragma unroll
  for (int v = 0; v < (1 << RB); ++v) {
    if (v & ((1 << B1) | (1 << B2))) continue;
    if ((v & rmask) != rval) continue;
    const int i0 = v, i1 = v | (1 << B1), i2 = v | (1 << B2), i3 = v | (1 << B1) | (1 << B2);
    const cplx<R> x0 = a[i0], x1 = a[i1], x2 = a[i2], x3 = a[i3];
    // selects, not an indexed array (a runtime index into x[] put it in local memory)
    auto pick = [x0, x1, x2, x3](int s) {
      cplx<R> r = x0;
      r = s == 1 ? x1 : r;
      r = s == 2 ? x2 : r;
      r = s == 3 ? x3 : r;
      return r;
    };
    a[i0] = cmul<R>(p0, pick(s0));
    a[i1] = cmul<R>(p1, pick(s1));
    a[i2] = cmul<R>(p2, pick(s2));
    a[i3] = cmul<R>(p3, pick(s3));
  }
}

template <typename R> SVB_HD int fbit(uint64_t F, int q) { return q >= 0 ? (int)((F >> q) & 1ull) : 0; }

SVB_HD int diag_nut(const DiagHdr* h) {
  int n = 0;
  for (int g = 0; g < h->nUTg; ++g) n += h->utn[g];
  return n;
}

// Tile-uniform factors of one DIAG payload (host emulator / reference order).
template <typename R, int RB>
SVB_HD void diag_uniform_serial(const uint8_t* payload, uint64_t base, cplx<R>* slot) {
  const DiagHdr* h = reinterpret_cast<const DiagHdr*>(payload);
  const DiagTerm<R>* t = reinterpret_cast<const DiagTerm<R>*>(payload + sizeof(DiagHdr));
  const cplx<R> one = mk<R>(R(1), R(0));
  for (int i = 0; i < RB; ++i) {
    cplx<R> u0 = one, u1 = one;
    for (int k = 0; k < h->nUR[i]; ++k, ++t) {
      const int f = fbit<R>(base, t->qb);
      u0 = cmul<R>(u0, t->d[2 * f]);
      u1 = cmul<R>(u1, t->d[2 * f + 1]);
    }
    slot[1 + i] = u0;
    slot[1 + 5 + i] = u1;
  }
  cplx<R> c = one;
  for (int k = 0; k < h->nUC; ++k, ++t) c = cmul<R>(c, t->d[fbit<R>(base, t->qa) + 2 * fbit<R>(base, t->qb)]);
  for (int g = 0; g < h->nUTg; ++g) {
    cplx<R> v = one;
    for (int k = 0; k < h->utn[g]; ++k, ++t) {
      const int f = fbit<R>(base, t->qb);
      c = cmul<R>(c, t->d[2 * f]);
      v = cmul<R>(v, t->d[2 * f + 1]);
    }
    slot[kUniV + g] = v;
  }
  slot[0] = c;
}

// A register-pair diagonal term (quadrant factors e[ba + 2 bb]) with the pair
// as template arguments: the quadrant of every register is then a constant
// (a runtime pair cost three selects per register -- ~17% of the interpreter's
// instructions on the config-4 QAOA passes), and a quadrant whose factor is
// exactly 1 is skipped (a warp-uniform branch: controlled phases touch one).
template <typename R, int RB, int RA, int RBB>
SVB_HD void rr_quads(cplx<R>* a, const cplx<R>* e) {
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const cplx<R> f = ldc<R>(e + q);
    if (f.x == R(1) && f.y == R(0)) continue;
#pragma unroll
    for (int v = 0; v < (1 << RB); ++v)
      if ((((v >> RA) & 1) | (((v >> RBB) & 1) << 1)) == q) a[v] = cmul<R>(a[v], f);
  }
}
template <typename R, int RB>
SVB_HD void rr_apply(cplx<R>* a, int ra, int rb, const cplx<R>* e) {
#define SVB_RR(A, B) \
  case (A) * 8 + (B): \
    if constexpr ((A) < RB && (B) < RB) rr_quads<R, RB, A, B>(a, e); \
    break;
  switch (ra * 8 + rb) {
    SVB_RR(0, 1) SVB_RR(0, 2) SVB_RR(0, 3) SVB_RR(0, 4)
    SVB_RR(1, 0) SVB_RR(1, 2) SVB_RR(1, 3) SVB_RR(1, 4)
    SVB_RR(2, 0) SVB_RR(2, 1) SVB_RR(2, 3) SVB_RR(2, 4)
    SVB_RR(3, 0) SVB_RR(3, 1) SVB_RR(3, 2) SVB_RR(3, 4)
    SVB_RR(4, 0) SVB_RR(4, 1) SVB_RR(4, 2) SVB_RR(4, 3)
    default: break;
  }
#undef SVB_RR
}

template <typename R, int RB>
SVB_HD void diag_apply(cplx<R>* a, uint64_t Fg, const uint8_t* payload, const cplx<R>* uni) {
  constexpr int V = 1 << RB;
  const int4 h0 = ldop(reinterpret_cast<const int4*>(payload));      // nUR[0..3]
  const int4 h1 = ldop(reinterpret_cast<const int4*>(payload) + 1);  // nUR[4..5], nUC, nTR
  const int4 h2 = ldop(reinterpret_cast<const int4*>(payload) + 2);  // nTC, nRR, slot, -
  const DiagHdr* hd = reinterpret_cast<const DiagHdr*>(payload);
  const int nut = diag_nut(hd);
  const int nskip = h0.x + h0.y + h0.z + h0.w + h1.x + h1.y + h1.z + nut;
  const int nTR = h1.w, nTC = h2.x, nRR = h2.y;
  cplx<R> C = mk<R>(R(1), R(0));
  cplx<R> D0[RB], D1[RB];
#pragma unroll
  for (int i = 0; i < RB; ++i) D0[i] = D1[i] = C;
  if (h2.z >= 0) {
    // only entries with terms are evaluated (see PassDev::items)
    const cplx<R>* us = uni + (size_t)h2.z * kUniStride;
    const int nur[6] = {h0.x, h0.y, h0.z, h0.w, h1.x, h1.y};
    if (h1.z + nut > 0) C = us[0];
#pragma unroll
    for (int i = 0; i < RB; ++i)
      if (nur[i] > 0) {
        D0[i] = us[1 + i];
        D1[i] = us[1 + 5 + i];
      }
    // UT groups: the thread's own bit of each group's thread qubit selects V[g]
    const DiagTerm<R>* tu = reinterpret_cast<const DiagTerm<R>*>(payload + sizeof(DiagHdr)) + (nskip - nut);
    for (int g = 0; g < hd->nUTg; ++g) {
      const uint32_t w = ldop(reinterpret_cast<const uint32_t*>(tu));
      const int qa = (int8_t)((w >> 16) & 0xff);
      if (fbit<R>(Fg, qa)) C = cmul<R>(C, us[kUniV + g]);
      tu += hd->utn[g];
    }
  }
  const DiagTerm<R>* t = reinterpret_cast<const DiagTerm<R>*>(payload + sizeof(DiagHdr)) + nskip;
  for (int k = 0; k < nTR; ++k, ++t) {
    const uint32_t w = ldop(reinterpret_cast<const uint32_t*>(t));
    const int ra = (int8_t)(w & 0xff), qb = (int8_t)((w >> 24) & 0xff);
    const int f = fbit<R>(Fg, qb);
    const cplx<R> e0 = ldc<R>(t->d + 2 * f), e1 = ldc<R>(t->d + 2 * f + 1);
#pragma unroll
    for (int i = 0; i < RB; ++i)
      if (i == ra) {
        D0[i] = cmul<R>(D0[i], e0);
        D1[i] = cmul<R>(D1[i], e1);
      }
  }
  for (int k = 0; k < nTC; ++k, ++t) {
    const uint32_t w = ldop(reinterpret_cast<const uint32_t*>(t));
    const int qa = (int8_t)((w >> 16) & 0xff), qb = (int8_t)((w >> 24) & 0xff);
    C = cmul<R>(C, ldc<R>(t->d + fbit<R>(Fg, qa) + 2 * fbit<R>(Fg, qb)));
  }
  for (int k = 0; k < nRR; ++k, ++t) {
    const uint32_t w = ldop(reinterpret_cast<const uint32_t*>(t));
    const int ra = (int8_t)(w & 0xff), rb = (int8_t)((w >> 8) & 0xff);
    rr_apply<R, RB>(a, ra, rb, t->d);
  }
  // a[v] *= C * prod_i (v_i ? D1[i] : D0[i]).  Fold D0[i] into C so each
  // register bit contributes one ratio on its v_i = 1 half; skip factors that
  // are exactly 1 (controlled phases leave the v_i = 0 half untouched).
  auto is_one = [](cplx<R> z) { return z.x == R(1) && z.y == R(0); };
#pragma unroll
  for (int i = 0; i < RB; ++i) {
    if (!is_one(D0[i])) {
      C = cmul<R>(C, D0[i]);
      // unitary diagonal entries have unit modulus: 1/D0 = conj(D0)
      D1[i] = cmul<R>(D1[i], mk<R>(D0[i].x, -D0[i].y));
    }
  }
  if (!is_one(C)) {
#pragma unroll
    for (int v = 0; v < V; ++v) a[v] = cmul<R>(a[v], C);
  }
#pragma unroll
  for (int i = 0; i < RB; ++i) {
    if (!is_one(D1[i])) {
#pragma unroll
      for (int v = 0; v < V; ++v)
        if (v & (1 << i)) a[v] = cmul<R>(a[v], D1[i]);
    }
  }
}

// Value-taking entry points (JIT bodies pass immediates).
template <typename R, int RB, int B, bool COND>
SVB_HD void u1_real_v(cplx<R>* a, R m0, R m1, R m2, R m3, uint32_t rmask, uint32_t rval) {
  const cplx<R> m[4] = {mk<R>(m0, R(0)), mk<R>(m1, R(0)), mk<R>(m2, R(0)), mk<R>(m3, R(0))};
  u1_real<R, RB, B, COND>(a, m, rmask, rval);
}
template <typename R, int RB, int B, bool COND>
SVB_HD void u1_dense_v(cplx<R>* a, cplx<R> m0, cplx<R> m1, cplx<R> m2, cplx<R> m3, uint32_t rmask, uint32_t rval) {
  const cplx<R> m[4] = {m0, m1, m2, m3};
  u1_dense<R, RB, B, COND>(a, m, rmask, rval);
}
template <typename R, int RB, int B, bool COND>
SVB_HD void u1_anti_v(cplx<R>* a, cplx<R> m1, cplx<R> m2, uint32_t rmask, uint32_t rval) {
  const cplx<R> m[4] = {mk<R>(R(0), R(0)), m1, m2, mk<R>(R(0), R(0))};
  u1_anti<R, RB, B, COND>(a, m, rmask, rval);
}

template <typename R, int RB, int B, bool COND>
SVB_HD void u1_rx_v(cplx<R>* a, R ma, R mb, R mc, R md, uint32_t rmask, uint32_t rval) {
  const cplx<R> m[4] = {mk<R>(ma, R(0)), mk<R>(R(0), mb), mk<R>(R(0), mc), mk<R>(md, R(0))};
  u1_rx<R, RB, B, COND>(a, m, rmask, rval);
}

template <typename R, int RB, int B, bool COND>
SVB_HD void u1_kind(int kind, cplx<R>* a, const cplx<R>* m, uint32_t rmask, uint32_t rval) {
  if (kind == OP_U1R) u1_real<R, RB, B, COND>(a, m, rmask, rval);
  else if (kind == OP_U1X) u1_rx<R, RB, B, COND>(a, m, rmask, rval);
  else if (kind == OP_U1) u1_dense<R, RB, B, COND>(a, m, rmask, rval);
  else u1_anti<R, RB, B, COND>(a, m, rmask, rval);
}

template <typename R, int RB, int B, bool REAL>
SVB_HD void u1_piv_pc(int pc, cplx<R>* a, const cplx<R>* r) {
  switch (pc) {
    case 0: u1_piv_p<R, RB, B, 0, REAL>(a, r); break;
    case 1: u1_piv_p<R, RB, B, 1, REAL>(a, r); break;
    case 2: u1_piv_p<R, RB, B, 2, REAL>(a, r); break;
    default: u1_piv_p<R, RB, B, 3, REAL>(a, r); break;
  }
}

template <typename R, int RB, int B>
SVB_HD void u1_piv_any(bool real, int pc, cplx<R>* a, const cplx<R>* r) {
  if constexpr (B < RB) {
    if (real) u1_piv_pc<R, RB, B, true>(pc, a, r);
    else u1_piv_pc<R, RB, B, false>(pc, a, r);
  }
}

template <typename R, int RB>
SVB_HD void dispatch_u1p(bool real, int b, int pc, cplx<R>* a, const cplx<R>* r) {
  switch (b) {
    case 0: u1_piv_any<R, RB, 0>(real, pc, a, r); break;
    case 1: u1_piv_any<R, RB, 1>(real, pc, a, r); break;
    case 2: u1_piv_any<R, RB, 2>(real, pc, a, r); break;
    case 3: u1_piv_any<R, RB, 3>(real, pc, a, r); break;
    default: u1_piv_any<R, RB, 4>(real, pc, a, r); break;
  }
}

template <typename R, int RB, bool COND>
SVB_HD void dispatch_u1_c(int kind, int b, cplx<R>* a, const cplx<R>* m, uint32_t rmask, uint32_t rval) {
  switch (b) {
    case 0: u1_kind<R, RB, 0, COND>(kind, a, m, rmask, rval); break;
    case 1: u1_kind<R, RB, 1, COND>(kind, a, m, rmask, rval); break;
    case 2: u1_kind<R, RB, 2, COND>(kind, a, m, rmask, rval); break;
    case 3: u1_kind<R, RB, 3, COND>(kind, a, m, rmask, rval); break;
    default:
      if constexpr (RB > 4) u1_kind<R, RB, (RB > 4 ? 4 : 0), COND>(kind, a, m, rmask, rval);
      break;
  }
}

template <typename R, int RB>
SVB_HD void dispatch_u1(int kind, int b, cplx<R>* a, const cplx<R>* m, uint32_t rmask, uint32_t rval) {
  if (rmask == 0) dispatch_u1_c<R, RB, false>(kind, b, a, m, 0, 0);
  else dispatch_u1_c<R, RB, true>(kind, b, a, m, rmask, rval);
}

template <typename R, int RB, int B1, int B2>
SVB_HD void u2_any(int kind, cplx<R>* a, const uint8_t* payload, uint32_t rmask, uint32_t rval) {
  if constexpr (B1 == B2 || B1 >= RB || B2 >= RB) {
    return;
  } else {
    if (kind == OP_U2)
      u2_dense<R, RB, B1, B2>(a, reinterpret_cast<const cplx<R>*>(payload), rmask, rval);
    else
      u2_perm<R, RB, B1, B2>(a, reinterpret_cast<const int32_t*>(payload),
                             reinterpret_cast<const cplx<R>*>(payload + 16), rmask, rval);
  }
}

template <typename R, int RB, int B1>
SVB_HD void dispatch_u2_b2(int kind, int b2, cplx<R>* a, const uint8_t* p, uint32_t rm, uint32_t rv) {
  switch (b2) {
    case 0: u2_any<R, RB, B1, 0>(kind, a, p, rm, rv); break;
    case 1: u2_any<R, RB, B1, 1>(kind, a, p, rm, rv); break;
    case 2: u2_any<R, RB, B1, 2>(kind, a, p, rm, rv); break;
    case 3: u2_any<R, RB, B1, 3>(kind, a, p, rm, rv); break;
    case 4: u2_any<R, RB, B1, 4>(kind, a, p, rm, rv); break;
    default: break;
  }
}

template <typename R, int RB>
SVB_HD void dispatch_u2(int kind, int b1, int b2, cplx<R>* a, const uint8_t* p, uint32_t rm, uint32_t rv) {
  switch (b1) {
    case 0: dispatch_u2_b2<R, RB, 0>(kind, b2, a, p, rm, rv); break;
    case 1: dispatch_u2_b2<R, RB, 1>(kind, b2, a, p, rm, rv); break;
    case 2: dispatch_u2_b2<R, RB, 2>(kind, b2, a, p, rm, rv); break;
    case 3: dispatch_u2_b2<R, RB, 3>(kind, b2, a, p, rm, rv); break;
    case 4: dispatch_u2_b2<R, RB, 4>(kind, b2, a, p, rm, rv); break;
    default: break;
  }
}

// Run the ops in [off, end) of the op stream on one thread's registers.
template <typename R, int RB>
SVB_HD void run_ops(cplx<R>* a, uint64_t Fg, const uint8_t* ops, uint32_t off, uint32_t end, const cplx<R>* uni) {
  while (off < end) {
    const OpHdr* h = reinterpret_cast<const OpHdr*>(ops + off);
    const int4 w0 = ldop(reinterpret_cast<const int4*>(h));          // kind, a, b, n
    const ulonglong2 w1 = ldop(reinterpret_cast<const ulonglong2*>(h) + 1);  // fmask, fval
    const uint4 w2 = ldop(reinterpret_cast<const uint4*>(h) + 2);     // rmask, rval, bytes
    const uint8_t* payload = ops + off + sizeof(OpHdr);
    off += w2.z;
    if ((Fg & w1.x) != w1.y) continue;
    switch (w0.x) {
      case OP_DIAG:
        diag_apply<R, RB>(a, Fg, payload, uni);
        break;
      case OP_U1:
      case OP_U1R:
      case OP_U1X:
      case OP_U1ANTI:
        dispatch_u1<R, RB>(w0.x, w0.y, a, reinterpret_cast<const cplx<R>*>(payload), w2.x, w2.y);
        break;
      case OP_U1P:
      case OP_U1PR:
        dispatch_u1p<R, RB>(w0.x == OP_U1PR, w0.y, w0.w, a, reinterpret_cast<const cplx<R>*>(payload));
        break;
      default:
        dispatch_u2<R, RB>(w0.x, w0.y, w0.z, a, payload, w2.x, w2.y);
        break;
    }
  }
}

// Shared-memory slot of local index j (XOR swizzle of the bank group).
template <typename R> SVB_HD uint32_t swz(uint32_t j);
template <> SVB_HD uint32_t swz<double>(uint32_t j) {
  return j ^ (((j >> 3) ^ (j >> 6) ^ (j >> 9) ^ (j >> 12)) & 7u);
}
// complex64: bit 0 is left alone so an aligned pair (j, j^1) stays one 16-byte
// unit (cp.async copies c64 amplitudes in pairs)
template <> SVB_HD uint32_t swz<float>(uint32_t j) {
  return j ^ ((((j >> 4) ^ (j >> 7) ^ (j >> 10)) & 7u) << 1);
}

// Thread layout of round `rd`: fixed local index and fixed global index.
SVB_HD void thread_fixed(const PassDev& pd, const RoundDev& rd, uint32_t tid, uint64_t base,
                         uint32_t* Fl, uint64_t* Fg) {
  uint32_t fl = 0;
  uint64_t fg = base;
  const int nt = pd.m - pd.rb;
  for (int tb = 0; tb < nt; ++tb) {
    if ((tid >> tb) & 1u) {
      const int l = rd.thr_local[tb];
      fl |= 1u << l;
      fg |= 1ull << pd.pos[l];
    }
  }
  *Fl = fl;
  *Fg = fg;
}

// Permuted-store round: the thread's fixed index with every bit moved to its
// destination (dest is a bit permutation, so it distributes over OR).
SVB_HD uint64_t thread_fixed_perm(const PassDev& pd, const RoundDev& rd, uint32_t tid) {
  uint64_t fg = 0;
  const int nt = pd.m - pd.rb;
  for (int tb = 0; tb < nt; ++tb)
    if ((tid >> tb) & 1u) fg |= 1ull << pd.dpos[rd.thr_local[tb]];
  return fg;
}

SVB_HD uint64_t tile_base(const PassDev& pd, uint64_t t) {
  uint64_t b = 0;
  for (int i = 0; i < pd.nout; ++i)
    if ((t >> i) & 1ull) b |= 1ull << pd.outpos[i];
  return b;
}
SVB_HD uint64_t tile_base_perm(const PassDev& pd, uint64_t t) {
  uint64_t b = 0;
  for (int i = 0; i < pd.nout; ++i)
    if ((t >> i) & 1ull) b |= 1ull << pd.doutpos[i];
  return b;
}

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
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(smem_dst)), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async8(void* smem_dst, const void* gsrc) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(smem_dst)), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void prefetch_l2(const void* g) {
  asm volatile("prefetch.global.L2::evict_last [%0];\n" ::"l"(g));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
// bulk (TMA-engine) stores of contiguous rows from shared memory
__device__ __forceinline__ void bulk_store_row(void* gdst, const void* ssrc, uint32_t bytes) {
  const uint32_t s = (uint32_t)__cvta_generic_to_shared(ssrc);
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(gdst), "r"(s), "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
}
// this thread's bulk stores have finished reading shared memory
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory"); }
// generic-proxy shared-memory writes visible to the async (bulk copy) proxy
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}
template <int N> __device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

constexpr int kStages = 2;
// Register bits per thread and threads per CTA of the pass kernel:
// complex128: 16 amplitudes x 256 threads (m = 12); complex64: 16 x 512 (m = 13),
// i.e. twice the warps per SM for the cheaper type.
template <typename R> constexpr int kRegBits = 4;
// NVRTC-specialised complex64 passes hold 32 amplitudes per thread (5 register
// bits): a 2^13 tile is 256 threads and two CTAs share an SM, so one CTA's
// shared-memory exchange and barrier overlap the other's FFMA2 bursts
// (Sycamore-32 c64: 347 -> 300 ms).  The interpreter keeps 4 (at 5 it spills).
#ifdef SVB_C64_RB4
template <typename R> constexpr int kJitRegBits = 4;
#else
template <typename R> constexpr int kJitRegBits = sizeof(R) == 8 ? 4 : 5;
#endif
// Launch shape of a pass with RB register bits: the threads of a default tile
// (m = 12 complex128, 13 complex64) and the CTAs per SM it is compiled for.
// complex128 passes run two CTAs per SM (single-stage ring each, <= 128
// registers per thread): 16 warps hide the FP64 and shared-memory latency;
// complex64 at RB = 4: one 512-thread CTA; at RB = 5: two 256-thread CTAs.
#ifdef SVB_C64_M14  // experiment: NVRTC complex64 tiles of 2^14 (512 threads x 32 amplitudes, one CTA per SM)
__host__ __device__ constexpr int pass_tile_m(int rsize, int rb = 4) { return rsize == 8 ? 12 : (rb >= 5 ? 14 : 13); }
__host__ __device__ constexpr int pass_min_blocks_of(int rsize, int rb) { return rsize == 8 ? 2 : 1; }
#else
__host__ __device__ constexpr int pass_tile_m(int rsize, int rb = 4) { return rsize == 8 ? 12 : 13; }
__host__ __device__ constexpr int pass_min_blocks_of(int rsize, int rb) { return (rsize == 8 || rb >= 5) ? 2 : 1; }
#endif
template <typename R, int RB> constexpr int kPassThreads = 1 << (pass_tile_m((int)sizeof(R), RB) - RB);
template <typename R, int RB> constexpr int kPassMinBlocks = pass_min_blocks_of((int)sizeof(R), RB);
// the interpreter kernel k_pass<R, RB>: one CTA per SM with a double ring.
// At two CTAs (<= 128 registers) the complex128 body spilled 5.4 KB; without
// the cap it does not spill, and config 4 (every circuit on the interpreter)
// measured 1.52 vs 1.63 s.  (SVB_INTERP_MINB2: the two-CTA shape, A/B runs.)
#ifdef SVB_INTERP_MINB2
template <typename R, int RB> constexpr int kInterpMinBlocks = kPassMinBlocks<R, RB>;
#else
template <typename R, int RB> constexpr int kInterpMinBlocks = 1;
#endif

template <typename R> __host__ __device__ constexpr uint32_t tile_bytes_of(int m) { return (uint32_t)sizeof(cplx<R>) << m; }

// Tile base (bits outside S) computed warp-parallel: lane l owns tile bit l.
__device__ __forceinline__ uint64_t tile_base_warp(const PassDev& pd, uint64_t t, uint32_t lane,
                                                  bool perm = false) {
  const int32_t* op = perm ? pd.doutpos : pd.outpos;
  uint64_t v = 0;
  if ((int)lane < pd.nout && ((t >> lane) & 1ull)) v = 1ull << op[lane];
  if ((int)lane + 32 < pd.nout && ((t >> (lane + 32)) & 1ull)) v |= 1ull << op[lane + 32];
  const uint32_t lo = __reduce_or_sync(0xffffffffu, (uint32_t)v);
  const uint32_t hi = __reduce_or_sync(0xffffffffu, (uint32_t)(v >> 32));
  return ((uint64_t)hi << 32) | lo;
}

// Tile base in the input buffer's layout (differs only for a perm_in pass).
template <int PERMIN>
__device__ __forceinline__ uint64_t tile_base_ld(const PassDev& pd, uint64_t t, uint32_t lane) {
  if (!PERMIN || !pd.perm_in) return tile_base_warp(pd, t, lane);
  uint64_t v = 0;
  if ((int)lane < pd.nout && ((t >> lane) & 1ull)) v = 1ull << pd.ioutpos[lane];
  if ((int)lane + 32 < pd.nout && ((t >> (lane + 32)) & 1ull)) v |= 1ull << pd.ioutpos[lane + 32];
  const uint32_t lo = __reduce_or_sync(0xffffffffu, (uint32_t)v);
  const uint32_t hi = __reduce_or_sync(0xffffffffu, (uint32_t)(v >> 32));
  return ((uint64_t)hi << 32) | lo;
}
// Local index of load-order index j (identity unless perm_in).
__host__ __device__ __forceinline__ uint32_t ld_order_local(const PassDev& pd, uint32_t j) {
  if (!pd.perm_in) return j;
  uint32_t r = 0;
  for (int b = 0; b < pd.m; ++b)
    if ((j >> b) & 1u) r |= 1u << pd.ld_local[b];
  return r;
}

template <typename R> __device__ __forceinline__ cplx<R> shfl_xor_c(cplx<R> x, int o) {
  x.x = __shfl_xor_sync(0xffffffffu, x.x, o);
  x.y = __shfl_xor_sync(0xffffffffu, x.y, o);
  return x;
}

// Tile-uniform factors of one DIAG payload, lanes in parallel over the terms.
// Product over lanes of a warp (all lanes return it).
template <typename R> __device__ __forceinline__ cplx<R> warp_prod(cplx<R> x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x = cmul<R>(x, shfl_xor_c<R>(x, o));
  return x;
}

// Tile-uniform factors of a pass's DIAG payloads: the host lists one work item
// per non-empty factor (PassDev::items); warp w evaluates items w, w+nwarps,
// ... as lane-parallel products over the item's terms.
template <typename R, int RB>
__device__ void diag_uniform_items(const uint8_t* ops, const uint32_t* diag_off, const uint16_t* items, int nitems,
                                   uint64_t base, cplx<R>* uni, uint32_t warp, uint32_t nwarps, uint32_t lane) {
  const cplx<R> one = mk<R>(R(1), R(0));
  for (int it = (int)warp; it < nitems; it += (int)nwarps) {
    const uint32_t code = items[it];
    const int d = (int)(code & 0xffu), kind = (int)((code >> 8) & 3u), idx = (int)(code >> 10);
    const uint8_t* payload = ops + diag_off[d];
    const DiagHdr* h = reinterpret_cast<const DiagHdr*>(payload);
    cplx<R>* slot = uni + d * kUniStride;
    const DiagTerm<R>* t = reinterpret_cast<const DiagTerm<R>*>(payload + sizeof(DiagHdr));
    int nur_all = 0;
    for (int i = 0; i < 6; ++i) nur_all += h->nUR[i];
    if (kind == 0) {  // register bit idx x tile bits
      for (int i = 0; i < idx; ++i) t += h->nUR[i];
      const int n = h->nUR[idx];
      cplx<R> u0 = one, u1 = one;
      for (int k = (int)lane; k < n; k += 32) {
        const int f = fbit<R>(base, t[k].qb);
        u0 = cmul<R>(u0, t[k].d[2 * f]);
        u1 = cmul<R>(u1, t[k].d[2 * f + 1]);
      }
      if (n > 1) { u0 = warp_prod<R>(u0); u1 = warp_prod<R>(u1); }
      if (lane == 0) { slot[1 + idx] = u0; slot[1 + 5 + idx] = u1; }
    } else if (kind == 1) {  // constant: UC terms and the UT constant parts
      t += nur_all;
      const DiagTerm<R>* tut = t + h->nUC;
      const int nut = diag_nut(h);
      cplx<R> c = one;
      for (int k = (int)lane; k < h->nUC; k += 32)
        c = cmul<R>(c, t[k].d[fbit<R>(base, t[k].qa) + 2 * fbit<R>(base, t[k].qb)]);
      for (int k = (int)lane; k < nut; k += 32) c = cmul<R>(c, tut[k].d[2 * fbit<R>(base, tut[k].qb)]);
      if (h->nUC + nut > 1) c = warp_prod<R>(c);
      if (lane == 0) slot[0] = c;
    } else {  // UT group idx: thread-bit ratio
      t += nur_all + h->nUC;
      for (int g = 0; g < idx; ++g) t += h->utn[g];
      const int n = h->utn[idx];
      cplx<R> v = one;
      for (int k = (int)lane; k < n; k += 32) v = cmul<R>(v, t[k].d[2 * fbit<R>(base, t[k].qb) + 1]);
      if (n > 1) v = warp_prod<R>(v);
      if (lane == 0) slot[kUniV + idx] = v;
    }
  }
}

// ------------------------------------------------------- pass skeleton
// Per-CTA context of a fused pass, shared by the interpreter body and the
// JIT-generated bodies.
template <typename R, int RB> struct PassCtx {
#ifndef SVB_HOIST
#define SVB_HOIST 4
#endif
  static constexpr int kHoist = SVB_HOIST;  // rounds whose thread constants live in registers
  const PassDev& pd;
  cplx<R>* state;
  cplx<R>* out;          // destination of the last round (== state unless pd.perm_out / pd.perm_in: the launchers pass it always)
  uint64_t pthr, pbase;  // permuted store: the thread's and the tile's destination bits
  double* zl;            // fused <Z>: the thread's running sums [RB + 3] (zsum_tile)
  double* zsm;           // or (ZSM kernels) in shared memory: [RB + 3][nthr], null otherwise
  const uint8_t* ops;  // op stream rebased onto shared memory
  const cplx<R>* uni;  // tile-uniform diagonal factors (shared memory)
  uint32_t tid;
  uint32_t sFl_r[kHoist];
  uint64_t Fg_r[kHoist];
  // single-stage ring: the body calls prefetch_next() once the last round's
  // layout is in registers, which refills the ring with the next tile
  cplx<R>* ring;
  cplx<R>* pro;        // per-thread prologue slots, [slot][thread] (shared memory)
  uint32_t nthr;
  const uint64_t* ldk;
  const uint32_t* sdk;
  uint64_t ld_tid, next_base;
  uint32_t sd_tid, nld;
  int prefetch, zero_input;
  int direct;  // round 0 loads straight from HBM into registers (no ring)
  int l2next;  // direct: the next tile exists (next_base); round 0 prefetches its live data into L2
  // uniform-slot sync inside the body (UIN kernels, upipe_sync): the tile's
  // slot wait and the production of tile it+D's factors run where the JIT
  // body first needs a uniform factor, after the ops that need none
  int usync;              // this tile's slot wait is the body's (0: done by the loop)
  uint32_t uslot;         // wait slot | parity << 16
  uint64_t* ubar;         // the slot barriers (shared memory)
  __device__ PassCtx(const PassDev& p) : pd(p) {}
};

// Copy (or, for a lazy |0...0>, synthesise) the tile at `base` into `dst`:
// element j = (tid + k*nthr)*kPer, 16 B per cp.async (one c128 amplitude or
// an aligned c64 pair); global and smem offsets split into a tid part and a
// tile-independent k part (tables in shared memory; the swizzle is linear
// over XOR: slot(tid part ^ k part) = swz(tid part) ^ swz(k part)).
template <typename R, int RB>
__device__ __forceinline__ void issue_tile(const PassCtx<R, RB>& c, uint64_t base, cplx<R>* dst) {
  constexpr int kPer = sizeof(cplx<R>) == 16 ? 1 : 2;
  if (c.zero_input) {
    for (uint32_t k = 0; k < c.nld; ++k) {
      const uint64_t g = base | c.ld_tid | c.ldk[k];
      cplx<R>* d = dst + (c.sd_tid ^ c.sdk[k]);
      d[0] = mk<R>(g == 0 ? R(1) : R(0), R(0));
      if (kPer == 2) d[1] = mk<R>(R(0), R(0));
    }
    return;
  }
  const cplx<R>* src = c.state + (base | c.ld_tid);
  if (c.pd.dmask) {
    for (uint32_t k = 0; k < c.nld; ++k) {
      cplx<R>* d = dst + (c.sd_tid ^ c.sdk[k]);
      if ((c.ld_tid | c.ldk[k]) & c.pd.dmask) {
        d[0] = mk<R>(R(0), R(0));
        if (kPer == 2) d[1] = mk<R>(R(0), R(0));
      } else {
        cp_async16(d, src + c.ldk[k]);
      }
    }
    return;
  }
  for (uint32_t k = 0; k < c.nld; ++k) cp_async16(dst + (c.sd_tid ^ c.sdk[k]), src + c.ldk[k]);
}

template <typename R, int RB, class Body> __device__ __forceinline__ void prefetch_next(const PassCtx<R, RB>& c) {
  if (c.prefetch) {
    __syncthreads();  // every thread holds its last layout: the ring is free
    Body::template issue<R, RB>(c, c.next_base, c.ring);
    cp_async_commit();
  }
}

// Thread constants of round k for the tile at `base`: swizzled local slot base
// and the fixed global index.
template <typename R, int RB>
__device__ __forceinline__ void round_fixed(const PassCtx<R, RB>& c, int k, uint64_t base, uint32_t& sFl,
                                            uint64_t& Fg) {
  if (k < PassCtx<R, RB>::kHoist) {
#pragma unroll
    for (int q = 0; q < PassCtx<R, RB>::kHoist; ++q)
      if (q == k) {
        sFl = c.sFl_r[q];
        Fg = c.Fg_r[q] | base;
      }
  } else {
    uint32_t Fl;
    thread_fixed(c.pd, c.pd.rounds[k], c.tid, base, &Fl, &Fg);
    sFl = swz<R>(Fl);
  }
}

template <typename R, int RB>
__device__ __forceinline__ uint64_t thread_fixed_g(const PassCtx<R, RB>& c, int k) {
  uint32_t Fl;
  uint64_t Fg;
  thread_fixed(c.pd, c.pd.rounds[k], c.tid, 0, &Fl, &Fg);
  return Fg;
}

// Shared-memory slots of the thread's 2^RB amplitudes in round layout `rd`:
// the swizzle is GF(2)-linear, so slot(v) = swz(Fl) ^ XOR_i v_i swz(1 << reg_local[i]).
template <typename R, int RB>
__device__ __forceinline__ void layout_slots(uint32_t sFl, const RoundDev& rd, uint32_t* slot) {
  uint32_t sl[RB];
#pragma unroll
  for (int i = 0; i < RB; ++i) sl[i] = swz<R>(1u << rd.reg_local[i]);
  slot[0] = sFl;
#pragma unroll
  for (int i = 0; i < RB; ++i)
#pragma unroll
    for (int v = 0; v < (1 << i); ++v) slot[v | (1 << i)] = slot[v] ^ sl[i];
}

template <typename R, int RB>
__device__ __forceinline__ void load_slots(cplx<R>* a, const cplx<R>* cur, const uint32_t* slot) {
#pragma unroll
  for (int v = 0; v < (1 << RB); ++v) a[v] = cur[slot[v]];
}
template <typename R, int RB>
__device__ __forceinline__ void store_slots(const cplx<R>* a, cplx<R>* cur, const uint32_t* slot) {
#pragma unroll
  for (int v = 0; v < (1 << RB); ++v) cur[slot[v]] = a[v];
}

// Last round: straight from registers to HBM (lanes <-> qubits 0..4, or with a
// permuted store lanes <-> the qubits whose destinations are 0..4).
template <typename R, int RB>
__device__ __forceinline__ void store_global(const PassCtx<R, RB>& c, uint64_t Fg, const RoundDev& rd,
                                             const cplx<R>* a) {
  const PassDev& pd = c.pd;
  cplx<R>* g0 = pd.perm_out ? c.out + (c.pbase | c.pthr) : c.out + Fg;
  const int32_t* dp = pd.perm_out ? pd.dpos : pd.pos;
  size_t goff[RB];
#pragma unroll
  for (int i = 0; i < RB; ++i) goff[i] = (size_t)1 << dp[rd.reg_local[i]];
  size_t gv[1 << RB];
  gv[0] = 0;
#pragma unroll
  for (int i = 0; i < RB; ++i)
#pragma unroll
    for (int v = 0; v < (1 << i); ++v) gv[v | (1 << i)] = gv[v] | goff[i];
#pragma unroll
  for (int v = 0; v < (1 << RB); ++v) __stcs(g0 + gv[v], a[v]);
}

// Direct first round: the round-0 layout has no lane register bits, so the
// warp's lanes read consecutive amplitudes (512 B per request).
template <typename R, int RB>
__device__ __forceinline__ void load_global(const PassCtx<R, RB>& c, uint64_t Fg, const RoundDev& rd, cplx<R>* a) {
  size_t goff[RB];
#pragma unroll
  for (int i = 0; i < RB; ++i) goff[i] = (size_t)1 << c.pd.pos[rd.reg_local[i]];
#pragma unroll
  for (int v = 0; v < (1 << RB); ++v) {
    size_t g = 0;
#pragma unroll
    for (int i = 0; i < RB; ++i)
      if (v & (1 << i)) g |= goff[i];
    if (c.zero_input) a[v] = mk<R>((Fg | g) == 0 ? R(1) : R(0), R(0));
    else if ((Fg | g) & c.pd.dmask) a[v] = mk<R>(R(0), R(0));  // never written (support tracking)
    else a[v] = __ldcs(c.state + (Fg | g));
  }
}

// Fused <Z_q> of the last round (pd.zsum): p_v = |a_v|^2 of the thread's 2^RB
// amplitudes; the thread adds T = sum p and W_i = sum p (-1)^(v_i) to its
// running sums, and lane j adds +-(warp sum of T) for tile bits j and j + 32.
// The running sums are thread-local (c.zl: local memory if the registers run
// out -- no shared memory, no atomics); zsum_store writes them once per thread
// at the end, and k_zsum_finish (fused.cu) applies the thread-bit signs and
// sums over the CTAs.
// Global layout (doubles): per thread [cta][RB + 1][nthr], then per warp [cta][nwarps][64].
template <typename R, int RB>
__device__ __forceinline__ void zsum_tile(const PassCtx<R, RB>& c, const cplx<R>* a, uint64_t base) {
  // halving tree over the register bits: level i sums the pairs along bit i
  // (their odd halves give s1[i] = sum of p_v with bit i set); ~2^(RB+1)
  // additions instead of 2^RB (RB/2 + 1)
  double q[1 << RB], s1[RB];
#pragma unroll
  for (int v = 0; v < (1 << RB); ++v) q[v] = (double)a[v].x * (double)a[v].x + (double)a[v].y * (double)a[v].y;
#pragma unroll
  for (int i = 0; i < RB; ++i) {
    const int h = 1 << (RB - 1 - i);  // pairs at this level
    double odd = q[1];
#pragma unroll
    for (int j = 1; j < h; ++j) odd += q[2 * j + 1];
    s1[i] = odd;
#pragma unroll
    for (int j = 0; j < h; ++j) q[j] = q[2 * j] + q[2 * j + 1];
  }
  const double T = q[0];
  double tw = T;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) tw += __shfl_xor_sync(0xffffffffu, tw, o);
  const uint32_t lane = c.tid & 31u;
  const double t0 = ((int)lane < c.pd.nout) ? (((base >> c.pd.outpos[lane]) & 1ull) ? -tw : tw) : 0.0;
  const double t1 = ((int)lane + 32 < c.pd.nout) ? (((base >> c.pd.outpos[lane + 32]) & 1ull) ? -tw : tw) : 0.0;
  if (c.zsm) {  // shared-memory running sums: no registers held across the tile's ops
    double* z = c.zsm + c.tid;
    const uint32_t st = c.nthr;
    z[0] += T;
#pragma unroll
    for (int i = 0; i < RB; ++i) z[(1 + i) * st] += fma(-2.0, s1[i], T);
    z[(RB + 1) * st] += t0;
    z[(RB + 2) * st] += t1;
    return;
  }
  double* zl = c.zl;
  zl[0] += T;
#pragma unroll
  for (int i = 0; i < RB; ++i) zl[1 + i] += fma(-2.0, s1[i], T);
  zl[RB + 1] += t0;
  zl[RB + 2] += t1;
}

template <typename R, int RB>
__device__ __forceinline__ void zsum_store(const PassCtx<R, RB>& c) {
  const uint32_t nthr = c.nthr, tid = c.tid, lane = tid & 31u;
  double* zs = reinterpret_cast<double*>(c.pd.zacc) + (size_t)blockIdx.x * (RB + 1) * nthr;
  double* zw = reinterpret_cast<double*>(c.pd.zacc) + (size_t)kZaccCols * (RB + 1) * nthr +
               ((size_t)blockIdx.x * (nthr >> 5) + (tid >> 5)) * 64;
  if (c.zsm) {
    const double* z = c.zsm + tid;
#pragma unroll
    for (int i = 0; i <= RB; ++i) zs[i * nthr + tid] = z[i * nthr];
    zw[lane] = z[(RB + 1) * nthr];
    zw[lane + 32] = z[(RB + 2) * nthr];
    return;
  }
#pragma unroll
  for (int i = 0; i <= RB; ++i) zs[i * nthr + tid] = c.zl[i];
  zw[lane] = c.zl[RB + 1];
  zw[lane + 32] = c.zl[RB + 2];
}

// Helpers for JIT-generated diagonal code.
template <typename R> __device__ __forceinline__ cplx<R> csel(int f, cplx<R> x0, cplx<R> x1) { return f ? x1 : x0; }
template <typename R> __device__ __forceinline__ cplx<R> conj_mul(cplx<R> x, cplx<R> u) {
  return cmul<R>(x, mk<R>(u.x, -u.y));
}
template <typename R, int RB, int I>
__device__ __forceinline__ void mul_half(cplx<R>* a, cplx<R> d) {  // a[v] *= d for v with bit I set
#pragma unroll
  for (int v = 0; v < (1 << RB); ++v)
    if (v & (1 << I)) a[v] = cmul<R>(a[v], d);
}
template <typename R, int RB, int I>
__device__ __forceinline__ void mul_half_r(cplx<R>* a, R d) {  // real factor (e.g. cz signs)
#pragma unroll
  for (int v = 0; v < (1 << RB); ++v)
    if (v & (1 << I)) a[v] = rmul<R>(d, a[v]);
}
template <typename R, int RB>
__device__ __forceinline__ void mul_all_r(cplx<R>* a, R d) {
#pragma unroll
  for (int v = 0; v < (1 << RB); ++v) a[v] = rmul<R>(d, a[v]);
}
template <typename R, int RB>
__device__ __forceinline__ void mul_all(cplx<R>* a, cplx<R> d) {
#pragma unroll
  for (int v = 0; v < (1 << RB); ++v) a[v] = cmul<R>(a[v], d);
}
template <typename R, int RB, int IA, int IB, int Q>
__device__ __forceinline__ void neg_quad(cplx<R>* a) {  // factor exactly -1 (cz)
#pragma unroll
  for (int v = 0; v < (1 << RB); ++v)
    if ((((v >> IA) & 1) + 2 * ((v >> IB) & 1)) == Q) a[v] = mk<R>(-a[v].x, -a[v].y);
}
template <typename R, int RB, int IA, int IB, int Q, int S>
__device__ __forceinline__ void imul_quad(cplx<R>* a) {  // factor exactly S*i (S = +-1): no flops
#pragma unroll
  for (int v = 0; v < (1 << RB); ++v)
    if ((((v >> IA) & 1) + 2 * ((v >> IB) & 1)) == Q) a[v] = S > 0 ? mk<R>(-a[v].y, a[v].x) : mk<R>(a[v].y, -a[v].x);
}
template <typename R, int RB, int IA, int IB, int Q>
__device__ __forceinline__ void mul_quad(cplx<R>* a, cplx<R> d) {  // amps with bit(IA) + 2 bit(IB) == Q
#pragma unroll
  for (int v = 0; v < (1 << RB); ++v)
    if ((((v >> IA) & 1) + 2 * ((v >> IB) & 1)) == Q) a[v] = cmul<R>(a[v], d);
}
template <typename R, int RB, int IA, int IB>
__device__ __forceinline__ void mul_rr(cplx<R>* a, cplx<R> e0, cplx<R> e1, cplx<R> e2, cplx<R> e3) {
#pragma unroll
  for (int v = 0; v < (1 << RB); ++v) {
    const int k = ((v >> IA) & 1) + 2 * ((v >> IB) & 1);
    a[v] = cmul<R>(a[v], k == 0 ? e0 : k == 1 ? e1 : k == 2 ? e2 : e3);
  }
}

// Interpreter body: rounds and ops read from the pass descriptor / op stream.
struct InterpBody {
  template <typename R, int RB> struct State {};
  template <typename R, int RB>
  __device__ static __forceinline__ void issue(const PassCtx<R, RB>& c, uint64_t base, cplx<R>* dst) {
    issue_tile<R, RB>(c, base, dst);
  }
  template <typename R, int RB>
  __device__ static __forceinline__ void prologue(const PassCtx<R, RB>&, State<R, RB>&) {}
  // direct first round: the tile's round-0 amplitudes straight from HBM
  template <typename R, int RB>
  __device__ static __forceinline__ void preload(const PassCtx<R, RB>& c, cplx<R>* a, uint64_t base) {
    uint32_t sFl;
    uint64_t Fg;
    round_fixed<R, RB>(c, 0, base, sFl, Fg);
    load_global<R, RB>(c, Fg, c.pd.rounds[0], a);
  }
  template <typename R, int RB>
  __device__ static __forceinline__ void tile(int, const PassCtx<R, RB>& c, cplx<R>* a, cplx<R>* cur,
                                              uint64_t base, const State<R, RB>&) {
    const int nrounds = c.pd.nrounds;
    for (int k = 0; k < nrounds; ++k) {
      const RoundDev& rd = c.pd.rounds[k];
      uint32_t sFl;
      uint64_t Fg;
      round_fixed<R, RB>(c, k, base, sFl, Fg);
      uint32_t slot[1 << RB];
      layout_slots<R, RB>(sFl, rd, slot);
      if (!(k == 0 && c.direct)) load_slots<R, RB>(a, cur, slot);  // direct: preload() filled a
      if (k + 1 == nrounds) prefetch_next<R, RB, InterpBody>(c);
      run_ops<R, RB>(a, Fg, c.ops, rd.op_off, rd.op_end, c.uni);
      if (k + 1 < nrounds) {
        // each slot of a layout is read and rewritten by its owner only, so one
        // barrier (after the writes) separates consecutive layouts
        store_slots<R, RB>(a, cur, slot);
        __syncthreads();
      } else {
        if (c.pd.zsum) zsum_tile<R, RB>(c, a, base);
        store_global<R, RB>(c, Fg, rd, a);
      }
    }
  }
};

// The tile's uniform-slot wait (UIN kernels, see pass_kernel), placed by the
// JIT right before the body's first tile-uniform factor.
template <typename R, int RB>
__device__ __forceinline__ void upipe_sync(const PassCtx<R, RB>& c) {
  if (c.usync) mbar_wait(&c.ubar[c.uslot & 0xffu], (c.uslot >> 16) & 1u);
}

// Persistent fused pass: each CTA walks tiles blockIdx.x, +gridDim.x, ...
// Tiles stream HBM -> shared memory with cp.async (LDGSTS, 16 B per thread,
// lanes on consecutive amplitudes: 512 B per warp request) into an
// XOR-swizzled ring of `stages` tiles: with 2 stages the next tile is issued
// at the top of the loop; with 1 stage (two CTAs per SM) the body issues it
// through prefetch_next() as soon as the last round's layout is in registers.
// Warps first evaluate the tile-uniform factors of the pass's diagonal ops,
// then Body runs the tile's rounds out of shared memory and stores the last
// layout straight from registers to HBM.
// Dynamic shared memory: ring | op stream (16-B padded) | uniform slots.
// PERMIN: the kernel may serve a perm_in pass (the JIT sets it only for one;
// the extra load addressing costs the others registers)
// STAGES >= 0: the launch's ring depth as a compile-time constant (NVRTC
// kernels: the other paths are dead code -- fewer instructions and spills)
// NR >= 0 / ZIN >= 0: the pass's round count and lazy-|0..0> input flag, also
// compiled in by the NVRTC kernels
template <typename R, int RB, class Body, int ZSM = 0, int UIN = 0, int PERMIN = 0, int STAGES = -1, int NR = -1,
          int ZIN = -1>
__device__ __forceinline__ void pass_kernel(cplx<R>* state, cplx<R>* out,
                                            const PassDev* __restrict__ pdg,
                                            const uint8_t* __restrict__ ops_g, uint32_t ntiles, int pass = 0,
                                            int zero_input_arg = 0, int stages_arg = kStages, int ops_mode = 0,
                                            int nslots = 0) {
  const int stages = STAGES >= 0 ? STAGES : stages_arg;
  const int zero_input = ZIN >= 0 ? ZIN : zero_input_arg;
  extern __shared__ __align__(128) unsigned char smraw[];
  __shared__ PassDev pd;
  __shared__ uint64_t s_ldk[32];
  __shared__ uint32_t s_sdk[32];
  __shared__ uint32_t s_doff[kMaxDiag];  // staged offsets of the uniform DIAG payloads
  __shared__ uint64_t s_ubar[kUPipeSlots];  // one-round direct passes: uniform-slot barriers
  {
    const int4* src = reinterpret_cast<const int4*>(pdg);
    int4* dst = reinterpret_cast<int4*>(&pd);
    for (int i = threadIdx.x; i < (int)(sizeof(PassDev) / 16); i += blockDim.x) dst[i] = __ldg(src + i);
  }
  __syncthreads();
  // Stage the op stream after the tile ring: ops_mode 0 copies this pass's
  // whole slice (offsets rebased so that stream offsets index shared memory);
  // ops_mode 1 (bodies with immediate coefficients) packs only the DIAG
  // payloads that have uniform slots.
  // stages: 2 = double ring, 1 = single ring + prefetch, 0 = direct first round
  // (one tile of shared memory for the inter-round layouts, no cp.async)
  // a one-round direct pass never touches the ring (registers from HBM, to HBM)
  const int nrounds_c = NR >= 0 ? NR : pd.nrounds;
  // (SVB_BULK_ROWS: the tile-sized region is the store staging of the rows)
  const uint32_t ring_bytes = (stages == 0 && nrounds_c == 1 && !SVB_BULK_ROWS)
                                  ? 0u
                                  : (uint32_t)(stages > 0 ? stages : 1) * ((uint32_t)sizeof(cplx<R>) << pd.m);
  uint32_t staged = 0;
  if (ops_mode == 0) {
    const int4* src = reinterpret_cast<const int4*>(ops_g + pd.ops_begin);
    int4* dst = reinterpret_cast<int4*>(smraw + ring_bytes);
    for (uint32_t i = threadIdx.x; i < pd.ops_bytes / 16; i += blockDim.x) dst[i] = __ldg(src + i);
    for (int d = threadIdx.x; d < pd.ndiag; d += blockDim.x) s_doff[d] = pd.diag_off[d] - pd.ops_begin;
    staged = pd.ops_bytes;
  } else {
    for (int d = 0; d < pd.ndiag; ++d) {
      const uint32_t off = pd.diag_off[d];
      const uint32_t bytes = __ldg(reinterpret_cast<const uint32_t*>(ops_g + off - sizeof(OpHdr) + kOpHdrBytesOff)) -
                             (uint32_t)sizeof(OpHdr);
      const int4* src = reinterpret_cast<const int4*>(ops_g + off);
      int4* dst = reinterpret_cast<int4*>(smraw + ring_bytes + staged);
      for (uint32_t i = threadIdx.x; i < bytes / 16; i += blockDim.x) dst[i] = __ldg(src + i);
      if (threadIdx.x == 0) s_doff[d] = staged;
      staged += bytes;
    }
  }
  cplx<R>* uni = reinterpret_cast<cplx<R>*>(smraw + ring_bytes + ((staged + 15u) & ~15u));
  PassCtx<R, RB> c(pd);
  c.state = state;
  c.out = out;
  c.pthr = pd.perm_out ? thread_fixed_perm(pd, pd.rounds[nrounds_c - 1], threadIdx.x) : 0;
  c.pbase = 0;
  c.ops = smraw + ring_bytes - pd.ops_begin;  // ops_mode 0 only
  c.uni = uni;
  // uniform slots are double-buffered by tile parity (the next tile's factors
  // are written while slow warps may still read this tile's).  One-round
  // direct passes (no ring) replace the per-tile CTA barrier by split
  // arrive/wait mbarriers over a ring of K = 2D + 1 slots (D = kUPipeAhead):
  // before tile it a warp waits on s_ubar[it%K], then evaluates its share of
  // tile it+D's factors into slot (it+D)%K and arrives on that slot's barrier.
  // Passing the wait for tile it means every warp has passed the wait for tile
  // it-D, i.e. finished tile it-D-1 -- the last user of slot (it+D)%K.  Warps
  // may drift D tiles apart instead of one.
  const bool upipe = stages == 0 && nrounds_c == 1;
  c.pro = uni + (upipe ? kUPipeSlots * kUGroup : 2) * pd.ndiag * kUniStride;
  c.nthr = blockDim.x;
  // fused <Z> running sums: registers, or (ZSM) shared memory after the
  // prologue slots (pass_smem counts them), which frees RB + 3 doubles of
  // registers across the tile's ops
  double zl[ZSM ? 1 : RB + 3];
#pragma unroll
  for (int i = 0; i < (ZSM ? 1 : RB + 3); ++i) zl[i] = 0.0;
  c.zl = zl;
  c.zsm = nullptr;
  if (ZSM && pd.zsum) {
    c.zsm = reinterpret_cast<double*>(c.pro + (size_t)nslots * blockDim.x);
    for (uint32_t i = threadIdx.x; i < (RB + 3) * blockDim.x; i += blockDim.x) c.zsm[i] = 0.0;
  }
  const uint32_t tid = threadIdx.x, nthr = blockDim.x, lane = tid & 31u, warp = tid >> 5;
  c.tid = tid;
  const uint32_t nwarps = nthr >> 5;
  const int m = pd.m, nrounds = nrounds_c, ndiag = pd.ndiag;
  const uint32_t T = 1u << m;
  cplx<R>* ring = reinterpret_cast<cplx<R>*>(smraw);
  constexpr int kPer = sizeof(cplx<R>) == 16 ? 1 : 2;
  const int lo_bits = (31 - __clz(nthr)) + (kPer == 2 ? 1 : 0);
  uint64_t ld_tid = 0;
  const uint32_t nld = T / (nthr * kPer);
  if (PERMIN && pd.perm_in) {
    // load-order element j -> local index ld_order_local(j) -> input offset
    // (ipos) and shared-memory slot
    const uint32_t lj = ld_order_local(pd, tid * kPer);
    for (int l = 0; l < m; ++l)
      if ((lj >> l) & 1u) ld_tid |= 1ull << pd.ipos[l];
    if (tid < nld) {
      uint64_t g = 0;
      const uint32_t lk = ld_order_local(pd, tid * nthr * kPer);
      for (int l = 0; l < m; ++l)
        if ((lk >> l) & 1u) g |= 1ull << pd.ipos[l];
      s_ldk[tid] = g;
      s_sdk[tid] = swz<R>(lk);
    }
  } else {
    for (int l = 0; l < lo_bits; ++l)
      if (((tid * kPer) >> l) & 1u) ld_tid |= 1ull << pd.pos[l];
    if (tid < nld) {
      uint64_t g = 0;
      const uint32_t j = tid * nthr * kPer;
      for (int l = lo_bits; l < m; ++l)
        if ((j >> l) & 1u) g |= 1ull << pd.pos[l];
      s_ldk[tid] = g;
      s_sdk[tid] = swz<R>(j);
    }
  }
  c.ring = ring;
  c.ldk = s_ldk;
  c.sdk = s_sdk;
  c.ld_tid = ld_tid;
  c.sd_tid = swz<R>(PERMIN ? ld_order_local(pd, tid * kPer) : tid * kPer);
  c.nld = nld;
  c.zero_input = zero_input;
  c.prefetch = 0;
  c.next_base = 0;
  c.direct = stages == 0;  // launch chose the direct first round (pd.direct, single stage)
  c.l2next = 0;
  c.usync = 0;
  c.uslot = 0;
  c.ubar = s_ubar;
  if (upipe && tid == 0) {
    for (int i = 0; i < kUPipeSlots; ++i) mbar_init(&s_ubar[i], nwarps);
    fence_mbar_init();
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < PassCtx<R, RB>::kHoist; ++k) {
    if (k < nrounds) {
      uint32_t Fl;
      thread_fixed(pd, pd.rounds[k], tid, 0, &Fl, &c.Fg_r[k]);
      c.sFl_r[k] = swz<R>(Fl);
    }
  }
  const uint32_t t0 = blockIdx.x;
  if (stages > 0) {
    if (t0 < ntiles) Body::template issue<R, RB>(c, tile_base_ld<PERMIN>(pd, t0, lane), ring);
    cp_async_commit();
  }
  // tile-independent per-thread constants of the body (e.g. products of
  // diagonal factors that depend only on the thread's own local bits)
  typename Body::template State<R, RB> bs;
  Body::template prologue<R, RB>(c, bs);
  cplx<R> a[1 << RB];
  const bool upipe_d = upipe && ndiag > 0;
  if (upipe) {
    if (upipe_d) {
      for (int d = 0; d < kUPipeAhead; ++d) {
        if (t0 + (uint64_t)d * kUGroup * gridDim.x >= ntiles) break;
        for (int g = 0; g < kUGroup; ++g) {
          const uint64_t td = t0 + (uint64_t)(d * kUGroup + g) * gridDim.x;
          if (td >= ntiles) break;
          diag_uniform_items<R, RB>(smraw + ring_bytes, s_doff, pd.items, pd.nitems,
                                    tile_base_warp(pd, (uint32_t)td, lane),
                                    uni + (d * kUGroup + g) * ndiag * kUniStride, warp, nwarps, lane);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&s_ubar[d]);
      }
    }
    __syncthreads();  // prologue slots visible
  }
  int it = 0;
  for (uint32_t t = t0; t < ntiles; t += gridDim.x, ++it) {
    const uint32_t tn = t + gridDim.x;
    if (stages > 1) {
      if (tn < ntiles)
        Body::template issue<R, RB>(c, tile_base_ld<PERMIN>(pd, tn, lane), ring + (size_t)((it + 1) & 1) * T);
      cp_async_commit();
    }
    const uint64_t base = tile_base_warp(pd, t, lane);
    if (pd.perm_out) c.pbase = tile_base_warp(pd, t, lane, true);
    const int u = it % kUPipeSlots;
    if (SVB_UWAIT_FIRST && upipe_d) mbar_wait(&s_ubar[u], (uint32_t)(it / kUPipeSlots) & 1u);
    if (UIN && upipe_d) {
      // produce tile it+D's factors first (registers are free between tiles);
      // the body waits for tile it's slot where it first needs it.  Starting
      // iteration it means this warp passed the wait for tile it-1, i.e. every
      // warp has finished tile it-D-2, the last user of slot (it+D)%K when
      // K = 2D + 2
      const int un = (it + kUPipeAhead) % kUPipeSlots;
      const uint64_t tf = (uint64_t)t + (uint64_t)kUPipeAhead * gridDim.x;
      if (tf < ntiles) {
        diag_uniform_items<R, RB>(smraw + ring_bytes, s_doff, pd.items, pd.nitems,
                                  tile_base_warp(pd, (uint32_t)tf, lane), uni + un * ndiag * kUniStride, warp,
                                  nwarps, lane);
        __syncwarp();
        if (lane == 0) mbar_arrive(&s_ubar[un]);
      }
      c.usync = 1;
      c.uslot = (uint32_t)u | (((uint32_t)(it / kUPipeSlots) & 1u) << 16);
    }
    if (stages == 0) {
      // direct first round: issue the tile's HBM loads (and the next tile's L2
      // prefetches) before the uniform factors and the barrier, so their
      // latency overlaps them; a[] is free between tiles
      c.l2next = tn < ntiles;
      if (c.l2next) c.next_base = tile_base_warp(pd, tn, lane);
      Body::template preload<R, RB>(c, a, base);
    }
    if (upipe) {
      if (upipe_d) {
        if (kUGroup > 1 && !UIN && !SVB_UWAIT_FIRST) {
          // groups of kUGroup tiles per slot: group P = it / G waits once and
          // produces group P + D (same ring argument with groups as units)
          const int P = it / kUGroup, gi = it % kUGroup, ug = P % kUPipeSlots;
          if (gi == 0) {
            const int ung = (P + kUPipeAhead) % kUPipeSlots;
            mbar_wait(&s_ubar[ug], (uint32_t)(P / kUPipeSlots) & 1u);
            if ((uint64_t)t + (uint64_t)kUPipeAhead * kUGroup * gridDim.x < ntiles) {
              for (int g = 0; g < kUGroup; ++g) {
                const uint64_t tf = (uint64_t)t + (uint64_t)(kUPipeAhead * kUGroup + g) * gridDim.x;
                if (tf >= ntiles) break;
                diag_uniform_items<R, RB>(smraw + ring_bytes, s_doff, pd.items, pd.nitems,
                                          tile_base_warp(pd, (uint32_t)tf, lane),
                                          uni + (ung * kUGroup + g) * ndiag * kUniStride, warp, nwarps, lane);
              }
              __syncwarp();
              if (lane == 0) mbar_arrive(&s_ubar[ung]);
            }
          }
          c.uni = uni + (ug * kUGroup + gi) * ndiag * kUniStride;
        } else {
          const int un = (it + kUPipeAhead) % kUPipeSlots;
          const uint64_t tf = (uint64_t)t + (uint64_t)kUPipeAhead * gridDim.x;
          if (!SVB_UWAIT_FIRST && !UIN && SVB_UPIPE_PROBE == 0) mbar_wait(&s_ubar[u], (uint32_t)(it / kUPipeSlots) & 1u);
          if (!UIN && tf < ntiles && SVB_UPIPE_PROBE < 2) {
            diag_uniform_items<R, RB>(smraw + ring_bytes, s_doff, pd.items, pd.nitems,
                                      tile_base_warp(pd, (uint32_t)tf, lane), uni + un * ndiag * kUniStride, warp,
                                      nwarps, lane);
            __syncwarp();
            if (lane == 0) mbar_arrive(&s_ubar[un]);
          }
          c.uni = uni + u * ndiag * kUniStride;
        }
      }
      Body::template tile<R, RB>(pass, c, a, ring, base, bs);
      continue;
    }
    c.uni = uni + (it & 1) * ndiag * kUniStride;
    if (ndiag > 0)  // tile-uniform diagonal factors (before the ring wait: overlaps the copies)
      diag_uniform_items<R, RB>(smraw + ring_bytes, s_doff, pd.items, pd.nitems, base, const_cast<cplx<R>*>(c.uni),
                                warp, nwarps, lane);
    if (stages > 1) cp_async_wait<1>();
    else if (stages == 1) cp_async_wait<0>();
    // ring data and uniform factors visible; (direct) the previous tile's last
    // shared-memory reads are done before round 0 stores this tile's layout
    __syncthreads();
    if (stages == 1) {
      c.prefetch = tn < ntiles;
      if (c.prefetch) c.next_base = tile_base_ld<PERMIN>(pd, tn, lane);
    }
    Body::template tile<R, RB>(pass, c, a, ring + (size_t)(stages > 1 ? (it & 1) : 0) * T, base, bs);
    // two stages: the ring slot is rewritten by the next iteration's issue.
    // One stage: prefetch_next() already fenced the ring, and the uniform
    // slots alternate, so the next tile's leading barrier is enough.
    if (stages > 1) __syncthreads();
  }
  cp_async_wait<0>();
  if (SVB_BULK_ROWS && threadIdx.x < (1u << RB)) bulk_wait_all();
  if (pd.zsum) zsum_store<R, RB>(c);
}

template <typename R, int RB>
__global__ void __launch_bounds__(kPassThreads<R, RB>, kInterpMinBlocks<R, RB>)
    k_pass(cplx<R>* state, cplx<R>* out, const PassDev* __restrict__ pdg,
           const uint8_t* __restrict__ ops_g, uint32_t ntiles, int zero_input, int stages) {
  pass_kernel<R, RB, InterpBody, 0, 0, 1>(state, out, pdg, ops_g, ntiles, 0, zero_input, stages, 0, 0);
}

// Launch shape of a pass: single-stage ring and kPassMinBlocks CTAs per SM
// when the op stream fits the per-CTA shared memory budget, else two stages
// and one CTA per SM.  Returns the dynamic shared memory bytes.
// HBM bytes a pass moves: every live tile is written; reads skip the
// never-written positions (dmask) and the lazy |0...0> input (zin).
#ifndef __CUDACC_RTC__
template <typename R> inline double pass_hbm_bytes(const PassDev& pd, bool zin) {
  const double tile = (double)(sizeof(cplx<R>) << pd.m) * (double)(1ull << pd.nout);
  const double rd = zin ? 0.0 : tile / (double)(1ull << __builtin_popcountll(pd.dmask));
  return tile + rd;
}
#endif

// host: the uniform-slot ring depth the JIT kernels are compiled with
__host__ __device__ inline int upipe_slots() {
#if defined(__CUDA_ARCH__) || defined(__CUDACC_RTC__)
  return kUPipeSlots;
#else
  static const int k = [] {
    const char* e = std::getenv("SVB_UPIPE_AHEAD");
    const char* ui = std::getenv("SVB_UIN");
    const int extra = ui ? (std::atoi(ui) != 0 ? 1 : 0) : (SVB_UIN ? 1 : 0);
    const char* gr = std::getenv("SVB_UGROUP");
    const int group = gr ? (std::atoi(gr) > 1 ? std::atoi(gr) : 1) : SVB_UGROUP;
    return ((e ? 2 * std::atoi(e) : 2 * SVB_UPIPE_AHEAD) + 1 + extra) * group;  // slots x tiles per slot
  }();
  return k;
#endif
}
template <typename R>
__host__ __device__ inline uint32_t pass_smem(int rb, int m, uint32_t staged_ops, int ndiag, int nslots, int stages,
                                              int zsum = 0, int nrounds = 2, int bulk = 0) {
  const uint32_t nthr = 1u << (m - rb);
  const uint32_t ring = (stages == 0 && nrounds == 1 && !bulk)
                            ? 0u
                            : (uint32_t)(stages > 0 ? stages : 1) * ((uint32_t)sizeof(cplx<R>) << m);
  return ring + ((staged_ops + 15u) & ~15u) +
         (((stages == 0 && nrounds == 1) ? (uint32_t)upipe_slots() : 2u) * (uint32_t)ndiag * kUniStride +
          (uint32_t)nslots * nthr) *
             (uint32_t)sizeof(cplx<R>) +
         // zsum != 0: a ZSM kernel keeps the fused <Z> running sums in shared memory
         (zsum ? (uint32_t)(rb + 3) * nthr * (uint32_t)sizeof(double) : 0u);
}
constexpr uint32_t kSmemPerSM = 228u * 1024u, kSmemReservedPerCTA = 1024u, kPassStaticSmem = 4096u;
// One-round direct passes of a support-tracked program (the QFT bench's last
// pass): no ring, so three CTAs per SM fit; the JIT gives them
// __launch_bounds__(.., 3) (<= 85 registers) for more warps in flight.
__host__ __device__ inline bool direct_one_round(const PassDev& pd) {
  return pd.direct && pd.dmask && pd.nrounds == 1;
}
constexpr int kDirectMinBlocks = 3;
#ifndef __CUDACC_RTC__
// CTAs per SM of one-round direct c128 passes (SVB_DIRECT_MINB: experiments)
inline int direct_min_blocks() {
  static const int k = [] {
    const char* e = std::getenv("SVB_DIRECT_MINB");
    return e ? std::atoi(e) : kDirectMinBlocks;
  }();
  return k;
}
#endif
// JIT kernels of one-round direct passes with fused <Z> keep the running sums
// in shared memory (pass_kernel's ZSM; pass_smem's zsum argument)
__host__ __device__ inline int zsm_pass(const PassDev& pd) { return direct_one_round(pd) && pd.zsum ? 1 : 0; }
// ... and (SVB_UIN=1, measured slower) wait for the uniform slot inside the body
#ifndef __CUDACC_RTC__
inline bool uin_pass(const PassDev& pd) {  // host (JIT generation); SVB_UIN=0: sync in the loop
  if (const char* e = std::getenv("SVB_UIN")) return std::atoi(e) != 0 && direct_one_round(pd);
  return SVB_UIN && direct_one_round(pd);
}
#endif
constexpr uint32_t kSmemMaxPerCTA = 227u * 1024u - kPassStaticSmem;
template <typename R>
__host__ __device__ inline int pass_stages(int rb, int m, uint32_t staged_ops, int ndiag, int nslots, int zsum = 0,
                                           int minb = 0) {
  if ((minb > 0 ? minb : pass_min_blocks_of((int)sizeof(R), rb)) < 2)
    return pass_smem<R>(rb, m, staged_ops, ndiag, nslots, 2, zsum) <= kSmemMaxPerCTA ? 2 : 1;
  const uint32_t per_cta = kSmemPerSM / 2 - kSmemReservedPerCTA - kPassStaticSmem;
  return pass_smem<R>(rb, m, staged_ops, ndiag, nslots, 1, zsum) <= per_cta ? 1 : 2;
}

}  // namespace svb
