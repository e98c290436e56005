// Fused gate programs: the host scheduler's output format and the per-thread
// op interpreter shared by the sm_100a pass kernel (fused.cu) and its CPU
// emulator (emulate.cpp).
//
// A program is a list of HBM passes.  Pass p owns a tile qubit set S (m
// physical qubits, always containing qubits 0..4 so that 32 lanes read 32
// consecutive amplitudes).  One CTA processes one tile = the 2^m amplitudes
// that share the bits outside S.  Inside a tile, work proceeds in rounds:
// in round k every thread holds 2^RB amplitudes in registers whose local
// indices differ in the round's RB "register" local bits; ops of the round
// touch only those registers, bits of the thread's fixed index, or the
// tile's fixed bits.  Rounds are separated by a shared-memory exchange.
#pragma once
#include <stdint.h>

#include <vector>

#include "common.cuh"

namespace svb {

// Optional per-kernel CUDA-event timing on the launching stream.
struct Profiler {
  bool on = false;
  struct Rec { cudaEvent_t a, b; int kind; };  // kind 0 = k_pass, 1 = k_permute
  std::vector<Rec> pending;
  double ms[2] = {0, 0};
  int64_t count[2] = {0, 0};
  double bytes[2] = {0, 0};
  void begin(cudaStream_t st, int kind, double nbytes);
  void end(cudaStream_t st);
  void collect();  // after a stream sync
};

struct ProgramStats {
  int64_t passes = 0, gates = 0, launches = 0;
  Profiler* prof = nullptr;
};

enum : int32_t { OP_DIAG = 0, OP_U1 = 1, OP_U1ANTI = 2, OP_U2 = 3, OP_PERM2 = 4 };

// Every op: header, then a kind-specific payload.  `bytes` = total size
// (multiple of 16).  Condition: the op applies where
// (Fg & fmask) == fval  and  (v & rmask) == rval  (v = register index).
struct alignas(16) OpHdr {
  int32_t kind, a, b, n;      // a, b: register bits; n: DIAG term count
  uint64_t fmask, fval;       // condition on fixed global index bits
  uint32_t rmask, rval, bytes, pad;
};
static_assert(sizeof(OpHdr) == 48, "OpHdr layout");

// Diagonal factor d[bit(qa) + 2 bit(qb)]; ra/rb = register bit or -1 (then
// the bit is read from the fixed global index at position qa/qb; q = -1 -> 0).
template <typename R> struct alignas(16) DiagTerm {
  int8_t ra, rb, qa, qb;
  int32_t pad[3];
  cplx<R> d[4];
};

constexpr int kMaxRounds = 24;
constexpr int kMaxM = 14;

struct RoundDev {
  int32_t reg_local[8];  // local bit of register bit i
  uint32_t op_off, op_end;
  uint32_t regmask_local, pad;
};

struct PassDev {
  int32_t m, nrounds, nout, rb;
  int32_t pos[16];      // physical qubit of local bit l
  int32_t outpos[48];   // physical qubits outside S, ascending (tile index bits)
  RoundDev rounds[kMaxRounds];
};

// ------------------------------------------------------------ interpreter
#define SVB_HD __host__ __device__ __forceinline__

template <typename T> SVB_HD T ldop(const T* p) {
#ifdef __CUDA_ARCH__
  return __ldg(p);
#else
  return *p;
#endif
}

template <typename R> SVB_HD cplx<R> ldc(const cplx<R>* p) {
#ifdef __CUDA_ARCH__
  return __ldg(p);
#else
  return *p;
#endif
}

template <typename R, int RB, int B>
SVB_HD void u1_dense(cplx<R>* a, const cplx<R>* m, uint32_t rmask, uint32_t rval) {
  const cplx<R> m0 = ldc<R>(m), m1 = ldc<R>(m + 1), m2 = ldc<R>(m + 2), m3 = ldc<R>(m + 3);
#pragma unroll
  for (int v = 0; v < (1 << RB); ++v) {
    if (v & (1 << B)) continue;
    if ((v & rmask) != rval) continue;
    cplx<R> x0 = a[v], x1 = a[v | (1 << B)];
    a[v] = cfma<R>(m1, x1, cmul<R>(m0, x0));
    a[v | (1 << B)] = cfma<R>(m3, x1, cmul<R>(m2, x0));
  }
}

// [[0, m1], [m2, 0]]
template <typename R, int RB, int B>
SVB_HD void u1_anti(cplx<R>* a, const cplx<R>* m, uint32_t rmask, uint32_t rval) {
  const cplx<R> m1 = ldc<R>(m + 1), m2 = ldc<R>(m + 2);
  const bool plain = m1.x == R(1) && m1.y == R(0) && m2.x == R(1) && m2.y == R(0);
#pragma unroll
  for (int v = 0; v < (1 << RB); ++v) {
    if (v & (1 << B)) continue;
    if ((v & rmask) != rval) continue;
    cplx<R> x0 = a[v], x1 = a[v | (1 << B)];
    if (plain) {
      a[v] = x1;
      a[v | (1 << B)] = x0;
    } else {
      a[v] = cmul<R>(m1, x1);
      a[v | (1 << B)] = cmul<R>(m2, x0);
    }
  }
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
    cplx<R> x[4] = {a[i0], a[i1], a[i2], a[i3]};
    auto pick = [&](int s) { return s == 0 ? x[0] : s == 1 ? x[1] : s == 2 ? x[2] : x[3]; };
    a[i0] = cmul<R>(p0, pick(s0));
    a[i1] = cmul<R>(p1, pick(s1));
    a[i2] = cmul<R>(p2, pick(s2));
    a[i3] = cmul<R>(p3, pick(s3));
  }
}

template <typename R, int RB>
SVB_HD void diag_apply(cplx<R>* a, uint64_t Fg, const DiagTerm<R>* t, int nt) {
  constexpr int V = 1 << RB;
  cplx<R> C = mk<R>(R(1), R(0));
  cplx<R> D0[RB], D1[RB];
#pragma unroll
  for (int i = 0; i < RB; ++i) D0[i] = D1[i] = mk<R>(R(1), R(0));
  for (int k = 0; k < nt; ++k) {
    const int8_t* hb = reinterpret_cast<const int8_t*>(t + k);
    const uint32_t w = ldop(reinterpret_cast<const uint32_t*>(hb));
    const int ra = (int8_t)(w & 0xff), rb = (int8_t)((w >> 8) & 0xff);
    const int qa = (int8_t)((w >> 16) & 0xff), qb = (int8_t)((w >> 24) & 0xff);
    const int fa = (qa >= 0 && ra < 0) ? (int)((Fg >> qa) & 1) : 0;
    const int fb = (qb >= 0 && rb < 0) ? (int)((Fg >> qb) & 1) : 0;
    const cplx<R>* d = t[k].d;
    if (ra < 0 && rb < 0) {
      C = cmul<R>(C, ldc<R>(d + fa + 2 * fb));
    } else if (rb < 0) {
      const cplx<R> e0 = ldc<R>(d + 2 * fb), e1 = ldc<R>(d + 1 + 2 * fb);
#pragma unroll
      for (int i = 0; i < RB; ++i)
        if (i == ra) { D0[i] = cmul<R>(D0[i], e0); D1[i] = cmul<R>(D1[i], e1); }
    } else if (ra < 0) {
      const cplx<R> e0 = ldc<R>(d + fa), e1 = ldc<R>(d + fa + 2);
#pragma unroll
      for (int i = 0; i < RB; ++i)
        if (i == rb) { D0[i] = cmul<R>(D0[i], e0); D1[i] = cmul<R>(D1[i], e1); }
    } else {
      const cplx<R> e0 = ldc<R>(d), e1 = ldc<R>(d + 1), e2 = ldc<R>(d + 2), e3 = ldc<R>(d + 3);
#pragma unroll
      for (int v = 0; v < V; ++v) {
        const int ba = (v >> ra) & 1, bb = (v >> rb) & 1;
        const cplx<R> e = ba ? (bb ? e3 : e1) : (bb ? e2 : e0);
        a[v] = cmul<R>(a[v], e);
      }
    }
  }
  // a[v] *= C * prod_i (v_i ? D1[i] : D0[i]): two half tables (low / high
  // register bits) keep the register footprint at 2^(RB/2) + 2^(RB - RB/2).
  constexpr int LB = RB / 2, HB = RB - RB / 2;
  cplx<R> TL[1 << LB], TH[1 << HB];
  TL[0] = C;
#pragma unroll
  for (int i = 0; i < LB; ++i) {
#pragma unroll
    for (int v = 0; v < (1 << i); ++v) {
      TL[v | (1 << i)] = cmul<R>(TL[v], D1[i]);
      TL[v] = cmul<R>(TL[v], D0[i]);
    }
  }
  TH[0] = mk<R>(R(1), R(0));
#pragma unroll
  for (int i = 0; i < HB; ++i) {
#pragma unroll
    for (int v = 0; v < (1 << i); ++v) {
      TH[v | (1 << i)] = cmul<R>(TH[v], D1[LB + i]);
      TH[v] = cmul<R>(TH[v], D0[LB + i]);
    }
  }
#pragma unroll
  for (int v = 0; v < V; ++v) a[v] = cmul<R>(a[v], cmul<R>(TL[v & ((1 << LB) - 1)], TH[v >> LB]));
}

#define SVB_CASE_B(FN, RB_, BB, ...) \
  case BB: FN<R, RB_, BB>(__VA_ARGS__); break;

template <typename R, int RB>
SVB_HD void dispatch_u1(int kind, int b, cplx<R>* a, const cplx<R>* m, uint32_t rmask, uint32_t rval) {
  if (kind == OP_U1) {
    switch (b) {
      SVB_CASE_B(u1_dense, RB, 0, a, m, rmask, rval)
      SVB_CASE_B(u1_dense, RB, 1, a, m, rmask, rval)
      SVB_CASE_B(u1_dense, RB, 2, a, m, rmask, rval)
      SVB_CASE_B(u1_dense, RB, 3, a, m, rmask, rval)
      default:
        if constexpr (RB > 4) { u1_dense<R, RB, (RB > 4 ? 4 : 0)>(a, m, rmask, rval); }
    }
  } else {
    switch (b) {
      SVB_CASE_B(u1_anti, RB, 0, a, m, rmask, rval)
      SVB_CASE_B(u1_anti, RB, 1, a, m, rmask, rval)
      SVB_CASE_B(u1_anti, RB, 2, a, m, rmask, rval)
      SVB_CASE_B(u1_anti, RB, 3, a, m, rmask, rval)
      default:
        if constexpr (RB > 4) { u1_anti<R, RB, (RB > 4 ? 4 : 0)>(a, m, rmask, rval); }
    }
  }
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
SVB_HD void run_ops(cplx<R>* a, uint64_t Fg, const uint8_t* ops, uint32_t off, uint32_t end) {
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
        diag_apply<R, RB>(a, Fg, reinterpret_cast<const DiagTerm<R>*>(payload), w0.w);
        break;
      case OP_U1:
      case OP_U1ANTI:
        dispatch_u1<R, RB>(w0.x, w0.y, a, reinterpret_cast<const cplx<R>*>(payload), w2.x, w2.y);
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
template <> SVB_HD uint32_t swz<float>(uint32_t j) {
  return j ^ (((j >> 4) ^ (j >> 8) ^ (j >> 12)) & 15u);
}

// Thread layout of round `rd`: fixed local index and fixed global index.
SVB_HD void thread_fixed(const PassDev& pd, const RoundDev& rd, uint32_t tid, uint64_t base,
                         uint32_t* Fl, uint64_t* Fg) {
  uint32_t fl = 0;
  uint64_t fg = base;
  int tb = 0;
  for (int l = 0; l < pd.m; ++l) {
    if (rd.regmask_local & (1u << l)) continue;
    if ((tid >> tb) & 1u) {
      fl |= 1u << l;
      fg |= 1ull << pd.pos[l];
    }
    ++tb;
  }
  *Fl = fl;
  *Fg = fg;
}

SVB_HD uint64_t tile_base(const PassDev& pd, uint64_t t) {
  uint64_t b = 0;
  for (int i = 0; i < pd.nout; ++i)
    if ((t >> i) & 1ull) b |= 1ull << pd.outpos[i];
  return b;
}

// ------------------------------------------------------------- host side
struct Program {
  std::vector<PassDev> passes;
  std::vector<uint8_t> ops;          // op stream (all passes)
  std::vector<int> final_perm;       // physical bit p must move to bit final_perm[p]; empty = identity
  int64_t gates = 0;
};

struct SchedOptions {
  int rb = 4;        // register bits per thread
  int m = 12;        // tile qubits
  bool relabel_swaps = true;
};

SchedOptions default_options(int precision, int n);

template <typename R>
Program build_program(int n, const svb_gate* gates, int ng, const SchedOptions& opt);

template <typename R>
void run_program(void* state, int n, const svb_gate* g, int ng, int fusion, int max_high,
                 cudaStream_t st, ProgramStats* stats);

// As run_program, but may replace *state (swap relabeling ends with an
// out-of-place permutation pass into a fresh cudaMalloc buffer).
template <typename R>
void run_program_owned(void** state, int n, const svb_gate* g, int ng, int fusion, cudaStream_t st,
                       ProgramStats* stats);

// CPU emulation of a program on a host state (same op interpreter).
template <typename R>
void emulate_program(cplx<R>* state, int n, const Program& prog);

}  // namespace svb
