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

enum : int32_t { OP_DIAG = 0, OP_U1 = 1, OP_U1ANTI = 2, OP_U2 = 3, OP_PERM2 = 4, OP_U1R = 5 };

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

// DIAG payload: DiagHdr, then DiagTerm entries in class order
//   UR (register bit i x tile bit, grouped by i) | UC (tile x tile) |
//   TR (register bit x thread bit) | TC (thread-bit constants) | RR (register x register)
// Classes U* depend only on the tile index and are evaluated once per tile per
// CTA into the pass's uniform slots (shared memory); T* and RR per thread.
struct alignas(16) DiagHdr {
  int32_t nUR[6];
  int32_t nUC, nTR, nTC, nRR;
  int32_t slot;
  int32_t pad[5];
};
static_assert(sizeof(DiagHdr) == 64, "DiagHdr layout");
constexpr int kUniStride = 12;  // cplx per slot: C, U0[5], U1[5], pad

constexpr int kMaxRounds = 24;
constexpr int kMaxM = 14;
constexpr int kMaxDiag = 48;

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
  int32_t ndiag;
  uint32_t ops_begin, ops_bytes;  // this pass's slice of the op stream (staged in smem)
  int32_t pad;
  uint32_t diag_off[kMaxDiag];  // op-stream offsets of this pass's DIAG payloads
};
constexpr uint32_t kMaxPassOpBytes = 72 * 1024;

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
    a[v] = mk<R>(fma(m1, x1.x, m0 * x0.x), fma(m1, x1.y, m0 * x0.y));
    a[v | (1 << B)] = mk<R>(fma(m3, x1.x, m2 * x0.x), fma(m3, x1.y, m2 * x0.y));
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

template <typename R> SVB_HD int fbit(uint64_t F, int q) { return q >= 0 ? (int)((F >> q) & 1ull) : 0; }

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
  slot[0] = c;
}

template <typename R, int RB>
SVB_HD void diag_apply(cplx<R>* a, uint64_t Fg, const uint8_t* payload, const cplx<R>* uni) {
  constexpr int V = 1 << RB;
  const int4 h0 = ldop(reinterpret_cast<const int4*>(payload));      // nUR[0..3]
  const int4 h1 = ldop(reinterpret_cast<const int4*>(payload) + 1);  // nUR[4..5], nUC, nTR
  const int4 h2 = ldop(reinterpret_cast<const int4*>(payload) + 2);  // nTC, nRR, slot, -
  const int nskip = h0.x + h0.y + h0.z + h0.w + h1.x + h1.y + h1.z;
  const int nTR = h1.w, nTC = h2.x, nRR = h2.y;
  cplx<R> C = mk<R>(R(1), R(0));
  cplx<R> D0[RB], D1[RB];
#pragma unroll
  for (int i = 0; i < RB; ++i) D0[i] = D1[i] = C;
  if (h2.z >= 0) {
    const cplx<R>* us = uni + (size_t)h2.z * kUniStride;
    C = us[0];
#pragma unroll
    for (int i = 0; i < RB; ++i) {
      D0[i] = us[1 + i];
      D1[i] = us[1 + 5 + i];
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
    const cplx<R> e0 = ldc<R>(t->d), e1 = ldc<R>(t->d + 1), e2 = ldc<R>(t->d + 2), e3 = ldc<R>(t->d + 3);
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const int ba = (v >> ra) & 1, bb = (v >> rb) & 1;
      a[v] = cmul<R>(a[v], ba ? (bb ? e3 : e1) : (bb ? e2 : e0));
    }
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

template <typename R, int RB, int B, bool COND>
SVB_HD void u1_kind(int kind, cplx<R>* a, const cplx<R>* m, uint32_t rmask, uint32_t rval) {
  if (kind == OP_U1R) u1_real<R, RB, B, COND>(a, m, rmask, rval);
  else if (kind == OP_U1) u1_dense<R, RB, B, COND>(a, m, rmask, rval);
  else u1_anti<R, RB, B, COND>(a, m, rmask, rval);
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
// *spare: a second state-sized buffer owned by the handle (allocated on first
// use, nullptr if it cannot be); the permutation writes into it and swaps.
template <typename R>
void run_program_owned(void** state, void** spare, int n, const svb_gate* g, int ng, int fusion, cudaStream_t st,
                       ProgramStats* stats);

// CPU emulation of a program on a host state (same op interpreter).
template <typename R>
void emulate_program(cplx<R>* state, int n, const Program& prog);

}  // namespace svb
