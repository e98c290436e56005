// Host-side gate fusion, pass scheduling and op encoding; CPU emulation of a
// scheduled program.
//
// Pipeline (replaces the reference's one-numpy-pass-per-gate loop,
// statevector.py:210-212 / 269-272):
//  1. swap relabeling: an exact SWAP permutes the logical->physical qubit map
//     instead of moving data; one permutation pass restores the order at the end;
//  2. forward fusion: a gate merges into the open block of its qubit(s)
//     (1q into 1q/2q blocks, 2q into the 2q block on the same pair), so
//     cx·u·cx·u·u (the conftest controlled phase) fuses to one diagonal;
//  3. classification: diagonal terms, 1q dense / anti-diagonal ops (with fixed
//     controls when a 2q block preserves one of its qubits), 2q monomial or
//     dense ops;
//  4. pass scheduling: greedy over the op list with commutation (ops commute
//     when every shared qubit is acted on diagonally by both); a pass admits
//     an op when its active qubits fit in the tile set S (|S| = m);
//  5. rounds: consecutive ops whose active qubits fit in RB register bits.
#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <cstddef>
#include <cmath>
#include <complex>
#include <cstring>
#include <vector>

#include "program.h"

namespace svb {

using cd = std::complex<double>;

namespace {

struct Block {
  int k;
  int q[2];
  cd M[16];
};

struct FOp {
  int type;                               // OP_DIAG, OP_U1, OP_U1ANTI, OP_U2, OP_PERM2
  int q[2];                               // DIAG: qa, qb(-1); U1: target; U2/PERM2: (qa, qb)
  std::vector<std::pair<int, int>> conds; // (qubit, value) fixed controls (U1 only)
  cd c[16];
  int src[4];
  uint64_t touched = 0, active = 0;
};

inline bool zero(cd z) { return z.real() == 0.0 && z.imag() == 0.0; }
inline bool one(cd z) { return z.real() == 1.0 && z.imag() == 0.0; }

// new = G(on q of block) * block.M
void left_mul_1q(Block& b, int q, const cd* g) {
  if (b.k == 1) {
    cd r[4];
    for (int i = 0; i < 2; ++i)
      for (int j = 0; j < 2; ++j) r[i * 2 + j] = g[i * 2 + 0] * b.M[0 * 2 + j] + g[i * 2 + 1] * b.M[1 * 2 + j];
    std::copy(r, r + 4, b.M);
    return;
  }
  int bitpos = (q == b.q[0]) ? 0 : 1;
  cd r[16];
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j < 4; ++j) {
      int bi = (i >> bitpos) & 1;
      int i0 = i & ~(1 << bitpos), i1 = i | (1 << bitpos);
      r[i * 4 + j] = g[bi * 2 + 0] * b.M[i0 * 4 + j] + g[bi * 2 + 1] * b.M[i1 * 4 + j];
    }
  std::copy(r, r + 16, b.M);
}

// new = G(on (qa,qb) in gate order) * block.M   (block is 2q on the same pair)
void left_mul_2q(Block& b, int qa, int qb, const cd* g) {
  cd gg[16];
  if (qa == b.q[0]) {
    std::copy(g, g + 16, gg);
  } else {  // reorder the gate into the block's (q0, q1) basis: swap bit roles
    auto sw = [](int i) { return ((i & 1) << 1) | ((i >> 1) & 1); };
    for (int i = 0; i < 4; ++i)
      for (int j = 0; j < 4; ++j) gg[sw(i) * 4 + sw(j)] = g[i * 4 + j];
  }
  cd r[16];
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j < 4; ++j) {
      cd acc = 0;
      for (int k = 0; k < 4; ++k) acc += gg[i * 4 + k] * b.M[k * 4 + j];
      r[i * 4 + j] = acc;
    }
  std::copy(r, r + 16, b.M);
}

// Fused products of exact gates pick up 1-ulp noise (e^{-it/2} e^{it/2} may
// round to 1 - 2^-53): snap such entries back to exactly 1 / 0 so the diagonal
// and trivial-factor structure is recognised (error <= 2^-50 per entry).
inline cd snap(cd z) {
  const double t = 0x1p-50;
  double re = z.real(), im = z.imag();
  if (std::fabs(re - 1.0) <= t && std::fabs(im) <= t) return cd(1.0, 0.0);
  if (std::fabs(re) <= t * 1e-3 && std::fabs(im) <= t * 1e-3) return cd(0.0, 0.0);
  // the other unit phases (-1, +-i: e.g. e^{i pi/2} = 6e-17 + 1i) become exact,
  // so the code generator emits swaps / negations instead of complex products
  if (std::fabs(re + 1.0) <= t && std::fabs(im) <= t) return cd(-1.0, 0.0);
  if (std::fabs(re) <= t && std::fabs(std::fabs(im) - 1.0) <= t) return cd(0.0, im > 0 ? 1.0 : -1.0);
  return z;
}

void emit_block(const Block& b0, std::vector<FOp>& out) {
  Block b = b0;
  for (int e = 0; e < (b.k == 1 ? 4 : 16); ++e) b.M[e] = snap(b.M[e]);
  if (b.k == 1) {
    FOp f;
    f.q[0] = b.q[0];
    f.q[1] = -1;
    f.touched = 1ull << b.q[0];
    const cd* M = b.M;
    if (zero(M[1]) && zero(M[2])) {
      if (one(M[0]) && one(M[3])) return;  // identity
      f.type = OP_DIAG;
      f.c[0] = M[0]; f.c[1] = M[3]; f.c[2] = M[0]; f.c[3] = M[3];
    } else {
      f.type = (zero(M[0]) && zero(M[3])) ? OP_U1ANTI : OP_U1;
      if (f.type == OP_U1 && M[0].imag() == 0 && M[1].imag() == 0 && M[2].imag() == 0 && M[3].imag() == 0)
        f.type = OP_U1R;
      else if (f.type == OP_U1 && M[0].imag() == 0 && M[3].imag() == 0 && M[1].real() == 0 && M[2].real() == 0)
        f.type = OP_U1X;
      std::copy(M, M + 4, f.c);
      f.active = f.touched;
    }
    out.push_back(f);
    return;
  }
  const cd* M = b.M;
  const int qa = b.q[0], qb = b.q[1];
  bool diag = true, pres_a = true, pres_b = true;
  for (int r = 0; r < 4; ++r)
    for (int c = 0; c < 4; ++c) {
      if (zero(M[r * 4 + c])) continue;
      if (r != c) diag = false;
      if ((r & 1) != (c & 1)) pres_a = false;
      if ((r & 2) != (c & 2)) pres_b = false;
    }
  uint64_t touched = (1ull << qa) | (1ull << qb);
  if (diag) {
    bool ident = true;
    for (int r = 0; r < 4; ++r) ident = ident && one(M[r * 5]);
    if (ident) return;
    FOp f;
    f.type = OP_DIAG;
    f.q[0] = qa; f.q[1] = qb;
    for (int r = 0; r < 4; ++r) f.c[r] = M[r * 5];
    f.touched = touched;
    out.push_back(f);
    return;
  }
  if (pres_a || pres_b) {
    // controlled structure: for each value of the preserved qubit, a 2x2 on the other
    const int ctl = pres_a ? qa : qb, tgt = pres_a ? qb : qa;
    const int cbit = pres_a ? 1 : 2, tbit = pres_a ? 2 : 1;
    for (int v = 0; v < 2; ++v) {
      int i0 = v ? cbit : 0, i1 = i0 | tbit;
      cd U[4] = {M[i0 * 4 + i0], M[i0 * 4 + i1], M[i1 * 4 + i0], M[i1 * 4 + i1]};
      if (zero(U[1]) && zero(U[2]) && one(U[0]) && one(U[3])) continue;
      FOp f;
      f.touched = touched;
      if (zero(U[1]) && zero(U[2])) {  // conditional diagonal -> 2q diag term
        f.type = OP_DIAG;
        f.q[0] = qa; f.q[1] = qb;
        for (int r = 0; r < 4; ++r) f.c[r] = 1.0;
        f.c[i0] = U[0];
        f.c[i1] = U[3];
        out.push_back(f);
        continue;
      }
      f.type = (zero(U[0]) && zero(U[3])) ? OP_U1ANTI : OP_U1;
      if (f.type == OP_U1 && U[0].imag() == 0 && U[1].imag() == 0 && U[2].imag() == 0 && U[3].imag() == 0)
        f.type = OP_U1R;
      else if (f.type == OP_U1 && U[0].imag() == 0 && U[3].imag() == 0 && U[1].real() == 0 && U[2].real() == 0)
        f.type = OP_U1X;
      f.q[0] = tgt; f.q[1] = -1;
      std::copy(U, U + 4, f.c);
      f.conds.push_back({ctl, v});
      f.active = 1ull << tgt;
      out.push_back(f);
    }
    return;
  }
  FOp f;
  f.q[0] = qa; f.q[1] = qb;
  f.touched = f.active = touched;
  bool mono = true;
  for (int r = 0; r < 4 && mono; ++r) {
    int nz = 0;
    for (int c = 0; c < 4; ++c)
      if (!zero(M[r * 4 + c])) { ++nz; f.src[r] = c; }
    if (nz != 1) mono = false;
  }
  if (mono) {
    f.type = OP_PERM2;
    for (int r = 0; r < 4; ++r) f.c[r] = M[r * 4 + f.src[r]];
  } else {
    f.type = OP_U2;
    std::copy(M, M + 16, f.c);
  }
  out.push_back(f);
}

// every row has at most one non-zero entry
bool monomial4(const cd* M) {
  for (int r = 0; r < 4; ++r) {
    int nz = 0;
    for (int c = 0; c < 4; ++c) nz += !zero(snap(M[r * 4 + c]));
    if (nz > 1) return false;
  }
  return true;
}
bool monomial2(const cd* G) {
  return (zero(snap(G[1])) && zero(snap(G[2]))) || (zero(snap(G[0])) && zero(snap(G[3])));
}

bool is_plain_swap(const svb_gate& g) {
  if (g.k != 2) return false;
  static const int src[4] = {0, 2, 1, 3};
  for (int r = 0; r < 4; ++r)
    for (int c = 0; c < 4; ++c) {
      double re = g.mat[2 * (r * 4 + c)], im = g.mat[2 * (r * 4 + c) + 1];
      double want = (src[r] == c) ? 1.0 : 0.0;
      if (re != want || im != 0.0) return false;
    }
  return true;
}

// Fuse the gate list into classified ops over physical qubits.
// zero_start: the input is |0...0>, which every qubit layout represents, so
// the initial logical -> physical map is chosen such that the swap relabeling
// ends on the identity (no final permutation at all).
std::vector<FOp> fuse(int n, const svb_gate* gates, int ng, bool relabel, bool zero_start, std::vector<int>& phys) {
  phys.resize(n);
  for (int q = 0; q < n; ++q) phys[q] = q;
  if (relabel && zero_start) {
    std::vector<int> tau(phys);
    for (int i = 0; i < ng; ++i)
      if (gates[i].k == 2 && is_plain_swap(gates[i])) std::swap(tau[gates[i].qubits[0]], tau[gates[i].qubits[1]]);
    for (int q = 0; q < n; ++q) phys[tau[q]] = q;
  }
  std::vector<Block> blocks;
  std::vector<int> order;  // block indices in creation order
  std::vector<int> open(n, -1);
  std::vector<bool> closed;
  auto close = [&](int bi) {
    if (bi < 0) return;
    for (int j = 0; j < blocks[bi].k; ++j) open[blocks[bi].q[j]] = -1;
  };
  for (int i = 0; i < ng; ++i) {
    const svb_gate& g = gates[i];
    cd G[16];
    int dim = g.k == 1 ? 2 : 4;
    for (int e = 0; e < dim * dim; ++e) G[e] = cd(g.mat[2 * e], g.mat[2 * e + 1]);
    if (g.k == 1) {
      int a = phys[g.qubits[0]];
      // a dense 1q gate does not enter a monomial (diagonal / permutation) 2q
      // block: that would turn a cheap cz-like op into a dense 4x4 (four
      // complex MACs per amplitude instead of one pivoted 1q op)
      if (open[a] >= 0 && blocks[open[a]].k == 2 && monomial4(blocks[open[a]].M) && !monomial2(G)) close(open[a]);
      if (open[a] >= 0) {
        left_mul_1q(blocks[open[a]], a, G);
      } else {
        Block b;
        b.k = 1; b.q[0] = a; b.q[1] = -1;
        std::copy(G, G + 4, b.M);
        blocks.push_back(b);
        open[a] = (int)blocks.size() - 1;
      }
      continue;
    }
    if (relabel && is_plain_swap(g)) {
      std::swap(phys[g.qubits[0]], phys[g.qubits[1]]);
      continue;
    }
    int a = phys[g.qubits[0]], b = phys[g.qubits[1]];
    if (open[a] >= 0 && open[a] == open[b]) {
      left_mul_2q(blocks[open[a]], a, b, G);
      continue;
    }
    // earlier open blocks on a or b are closed, not absorbed: absorbing a dense
    // 1q block would turn cheap monomial/diagonal 2q blocks dense.
    Block nb;
    nb.k = 2; nb.q[0] = a; nb.q[1] = b;
    std::copy(G, G + 16, nb.M);
    close(open[a]);
    close(open[b]);
    blocks.push_back(nb);
    open[a] = open[b] = (int)blocks.size() - 1;
  }
  std::vector<FOp> ops;
  for (const Block& b : blocks) emit_block(b, ops);
  return ops;
}

template <typename R> cplx<R> cvt(cd z) { return mk<R>((R)z.real(), (R)z.imag()); }

template <typename R> struct Encoder {
  std::vector<uint8_t>& buf;
  explicit Encoder(std::vector<uint8_t>& b) : buf(b) {}
  size_t begin(int kind, int a, int b, int n, uint64_t fmask, uint64_t fval, uint32_t rmask, uint32_t rval) {
    size_t at = buf.size();
    buf.resize(at + sizeof(OpHdr));
    OpHdr h{};
    h.kind = kind; h.a = a; h.b = b; h.n = n;
    h.fmask = fmask; h.fval = fval; h.rmask = rmask; h.rval = rval;
    std::memcpy(buf.data() + at, &h, sizeof h);
    return at;
  }
  template <typename T> void put(const T& x) {
    size_t at = buf.size();
    buf.resize(at + sizeof(T));
    std::memcpy(buf.data() + at, &x, sizeof(T));
  }
  void end(size_t at) {
    while (buf.size() % 16) buf.push_back(0);
    uint32_t bytes = (uint32_t)(buf.size() - at);
    std::memcpy(buf.data() + at + offsetof(OpHdr, bytes), &bytes, 4);
  }
};

}  // namespace

// Prologue slots the JIT body of an encoded pass will use (register x
// thread-bit chains of three or more factors, jit.cu emit_diag), and whether
// the pass still fits the two-CTA shared memory budget with them.
template <typename R> bool slots_fit(const Program& prog, const PassDev& pd) {
  int slots = 0;
  uint32_t staged = 0;
  for (int k = 0; k < pd.nrounds; ++k) {
    uint32_t off = pd.rounds[k].op_off;
    while (off < pd.rounds[k].op_end) {
      OpHdr h;
      std::memcpy(&h, prog.ops.data() + off, sizeof h);
      if (h.kind == OP_DIAG) {
        DiagHdr d;
        std::memcpy(&d, prog.ops.data() + off + sizeof(OpHdr), sizeof d);
        if (d.slot >= 0) staged += h.bytes - (uint32_t)sizeof(OpHdr);
        int nskip = d.nUC + d.nUR[0] + d.nUR[1] + d.nUR[2] + d.nUR[3] + d.nUR[4] + d.nUR[5];
        for (int g = 0; g < d.nUTg; ++g) nskip += d.utn[g];
        const DiagTerm<R>* tr =
            reinterpret_cast<const DiagTerm<R>*>(prog.ops.data() + off + sizeof(OpHdr) + sizeof(DiagHdr)) + nskip;
        for (int i = 0; i < pd.rb; ++i)
          for (int half = 0; half < 2; ++half) {
            int cnt = 0;
            for (int t = 0; t < d.nTR; ++t) {
              if (tr[t].ra != i) continue;
              const cplx<R> e0 = tr[t].d[half], e1 = tr[t].d[2 + half];
              if (!(e0.x == 1 && e0.y == 0 && e1.x == 1 && e1.y == 0)) ++cnt;
            }
            if (cnt >= 3) ++slots;
          }
      }
      off += h.bytes;
    }
  }
  if (pass_min_blocks_of((int)sizeof(R), pd.rb) < 2) return true;
  const uint32_t per_cta = kSmemPerSM / 2 - kSmemReservedPerCTA - kPassStaticSmem;
  return pass_smem<R>(pd.rb, pd.m, staged, pd.ndiag, slots, 1) <= per_cta;
}

// Fuse the program's final qubit permutation into its last pass: when that
// pass's tile set holds every physical qubit whose destination is 0..4, its
// last round can store out-of-place straight to the permuted addresses with
// the warp's lanes on those qubits (512 contiguous bytes per warp store), so
// the separate permutation pass (a full read + write of the state) goes away.
// The last round must not keep those qubits in registers; if it does, an
// op-free round with other register bits is appended.
static void fuse_final_permutation(Program& prog, int n) {
  if (prog.passes.empty() || prog.final_perm.empty()) return;
  PassDev& pd = prog.passes.back();
  if (std::getenv("SVB_TRACE")) {
    for (size_t p = 0; p < prog.passes.size(); ++p) {
      std::fprintf(stderr, "[svb] pass %zu S =", p);
      for (int l = 0; l < prog.passes[p].m; ++l) std::fprintf(stderr, " %d", prog.passes[p].pos[l]);
      std::fprintf(stderr, "\n");
    }
    std::fprintf(stderr, "[svb] final_perm:");
    for (int p = 0; p < n; ++p) std::fprintf(stderr, " %d", prog.final_perm[p]);
    std::fprintf(stderr, "\n");
  }
  int lane_l[5];
  uint32_t lmask = 0;
  for (int j = 0; j < 5; ++j) {
    lane_l[j] = -1;
    for (int p = 0; p < n; ++p)
      if (prog.final_perm[p] == j)
        for (int l = 0; l < pd.m; ++l)
          if (pd.pos[l] == p) lane_l[j] = l;
    if (lane_l[j] < 0) return;
    lmask |= 1u << lane_l[j];
  }
  if (pd.rounds[pd.nrounds - 1].regmask_local & lmask) {
    if (pd.nrounds >= kMaxRounds) return;
    const RoundDev& prev = pd.rounds[pd.nrounds - 1];
    RoundDev rd{};
    uint32_t regs = 0;
    for (int b = 0, i = 0; b < pd.m && i < pd.rb; ++b)
      if (!(lmask & (1u << b))) { regs |= 1u << b; rd.reg_local[i++] = b; }
    rd.regmask_local = regs;
    rd.op_off = rd.op_end = prev.op_end;
    pd.rounds[pd.nrounds++] = rd;
  }
  RoundDev& last = pd.rounds[pd.nrounds - 1];
  int t = 0;
  for (int j = 0; j < 5; ++j) last.thr_local[t++] = (uint8_t)lane_l[j];
  for (int b = 0; b < pd.m; ++b)
    if (!(last.regmask_local & (1u << b)) && !(lmask & (1u << b))) last.thr_local[t++] = (uint8_t)b;
  for (int l = 0; l < pd.m; ++l) pd.dpos[l] = prog.final_perm[pd.pos[l]];
  for (int i = 0; i < pd.nout; ++i) pd.doutpos[i] = prog.final_perm[pd.outpos[i]];
  pd.perm_out = 1;
  prog.perm_fused = true;
}

// absorb: start from the qubit layout that makes the swap relabeling end on
// the identity (a lazy |0...0> input, or an input permuted into that layout)
template <typename R>
static Program build_program_layout(int n, const svb_gate* gates, int ng, const SchedOptions& opt, bool absorb) {
  Program prog;
  prog.gates = ng;
  prog.n = n;
  std::vector<int> phys;
  std::vector<FOp> ops = fuse(n, gates, ng, opt.relabel_swaps, absorb, phys);
  const int m = std::min(opt.m, n);
  const int RB = opt.rb;
  require(m - RB >= 5 && m <= kMaxM, SVB_E_ARG, "fused program needs n >= rb + 5");
  const uint64_t lanes = 0x1full;

  std::vector<int> remaining(ops.size());
  for (size_t i = 0; i < ops.size(); ++i) remaining[i] = (int)i;
  uint64_t support = 0;  // zero_start: physical qubits written by an earlier pass

  while (!remaining.empty()) {
    // ---- choose S and the ops of this pass
    auto op_bytes = [](const FOp& f) -> size_t {
      const size_t c = sizeof(cplx<R>);
      if (f.type == OP_DIAG) return sizeof(OpHdr) + sizeof(DiagHdr) + sizeof(DiagTerm<R>) + 16;
      if (f.type == OP_U2) return sizeof(OpHdr) + 16 * c + 16;
      return sizeof(OpHdr) + 4 * c + 32;
    };
    // One in-order scan over the remaining ops: an op is placed when it does not
    // depend on a skipped op and its active qubits lie in S (grow: S may gain
    // qubits up to m).  Returns the number of placed ops.
    auto place = [&](uint64_t& S, bool grow, std::vector<int>* placed, std::vector<int>* skipped) {
      uint64_t blkA = 0, blkD = 0;
      size_t est_bytes = 0;  // upper bound of the encoded op bytes of this pass
      int count = 0;
      for (int idx : remaining) {
        const FOp& f = ops[idx];
        bool conflict = (f.touched & blkA) || (f.active & blkD);
        if (!conflict && est_bytes + op_bytes(f) <= kMaxPassOpBytes) {
          uint64_t need = f.active & ~S;
          if (need == 0 || (grow && __builtin_popcountll(S | need) <= m)) {
            S |= need;
            if (placed) placed->push_back(idx);
            est_bytes += op_bytes(f);
            ++count;
            continue;
          }
        }
        if (skipped) skipped->push_back(idx);
        blkA |= f.active;
        blkD |= f.touched & ~f.active;
      }
      return count;
    };
    uint64_t S = (m == n) ? ((n == 64) ? ~0ull : ((1ull << n) - 1)) : lanes;
    int best = place(S, true, nullptr, nullptr);
    for (int q = 0; q < n && __builtin_popcountll(S) < m; ++q) S |= 1ull << q;
    if (m < n) {
      // Local search over S: the in-order greedy fills S with the first qubits
      // it meets (e.g. the whole state-prep layer), which can starve the long
      // dependency chains (QFT).  Swap one non-lane qubit for one that a
      // remaining op acts on while that places more ops.
      uint64_t cand = 0;
      for (int idx : remaining) cand |= ops[idx].active;
      cand &= ~lanes;
      for (int it = 0; it < 4 * m; ++it) {
        int gain = 0;
        uint64_t bestS = S;
        for (uint64_t outs = S & ~lanes; outs; outs &= outs - 1) {
          const uint64_t qo = outs & (~outs + 1);
          for (uint64_t ins = cand & ~S; ins; ins &= ins - 1) {
            const uint64_t qi = ins & (~ins + 1);
            uint64_t T = (S & ~qo) | qi;
            const int c = place(T, false, nullptr, nullptr);
            if (c > best + gain) { gain = c - best; bestS = T; }
          }
        }
        if (gain == 0) break;
        best += gain;
        S = bestS;
      }
    }
    std::vector<int> placed, skipped;
    place(S, false, &placed, &skipped);

    PassDev pd{};
    pd.m = m;
    pd.rb = RB;
    int l = 0;
    int local_of[64];
    for (int q = 0; q < 64; ++q) local_of[q] = -1;
    for (int q = 0; q < n; ++q)
      if (S & (1ull << q)) { pd.pos[l] = q; local_of[q] = l; ++l; }
    pd.nout = 0;
    // zero_start: only tiles whose fixed bits lie in the support (qubits some
    // earlier pass has already written) hold anything but zeros, and they stay
    // zero through a pass (non-diagonal ops act inside the tile): those tiles
    // are the whole launch; inside a tile, positions with a bit outside the
    // support are synthesised as zeros instead of read (PassDev::dmask)
    for (int q = 0; q < n; ++q)
      if (!(S & (1ull << q)) && (!opt.zero_start || (support & (1ull << q)))) pd.outpos[pd.nout++] = q;
    pd.dmask = opt.zero_start && !prog.passes.empty() ? (S & ~support) : 0;

    // Rounds are built with op reordering first; if that needs more
    // per-thread prologue slots (register x thread-bit products, see jit.cu)
    // than two CTAs per SM leave room for, the pass is re-encoded in program
    // order.
    const PassDev pd_saved = pd;
    const size_t ops_saved = prog.ops.size();
    const std::vector<int> skipped_saved = skipped;
    for (int attempt = 0; attempt < 2; ++attempt) {
    const bool search = opt.round_search && attempt == 0;
      // ---- split into rounds: each round picks RB register bits and runs every
      // op (in dependency order, commuting where allowed) whose active qubits
      // lie in them; the register set is grown greedily, then improved by
      // single-bit swaps while that runs more ops (same scheme as the tile set)
      std::vector<std::pair<uint32_t, std::vector<int>>> rounds;
      {
        std::vector<int> rem = placed;
        std::vector<uint32_t> actl(ops.size(), 0);
        for (int idx : placed)
          for (int q = 0; q < n; ++q)
            if (ops[idx].active & (1ull << q)) actl[idx] |= 1u << local_of[q];
        auto place_r = [&](uint32_t& Rl, bool grow, std::vector<int>* took, std::vector<int>* left) {
          uint64_t blkA = 0, blkD = 0;
          int cnt = 0;
          for (int idx : rem) {
            const FOp& f = ops[idx];
            if (!((f.touched & blkA) || (f.active & blkD))) {
              const uint32_t need = actl[idx] & ~Rl;
              if (need == 0 || (grow && __builtin_popcount(Rl | need) <= RB)) {
                Rl |= need;
                if (took) took->push_back(idx);
                ++cnt;
                continue;
              }
            }
            if (left) left->push_back(idx);
            blkA |= f.active;
            blkD |= f.touched & ~f.active;
          }
          return cnt;
        };
        while (!rem.empty()) {
          uint32_t Rl = 0;
          int best = place_r(Rl, true, nullptr, nullptr);
          if (search) {
            uint32_t cand = 0;
            for (int idx : rem) cand |= actl[idx];
            for (int iter = 0; iter < 4 * RB; ++iter) {
              int gain = 0;
              uint32_t bestR = Rl;
              for (uint32_t ins = cand & ~Rl; ins; ins &= ins - 1) {
                const uint32_t qi = ins & (~ins + 1);
                if (__builtin_popcount(Rl) < RB) {
                  uint32_t T = Rl | qi;
                  const int c2 = place_r(T, false, nullptr, nullptr);
                  if (c2 > best + gain) { gain = c2 - best; bestR = T; }
                }
                for (uint32_t outs = Rl; outs; outs &= outs - 1) {
                  const uint32_t qo = outs & (~outs + 1);
                  uint32_t T = (Rl & ~qo) | qi;
                  const int c2 = place_r(T, false, nullptr, nullptr);
                  if (c2 > best + gain) { gain = c2 - best; bestR = T; }
                }
              }
              if (gain == 0) break;
              best += gain;
              Rl = bestR;
            }
          }
          std::vector<int> took, left;
          if (search) {
            place_r(Rl, false, &took, &left);
          } else {  // in program order: a new round whenever the register need overflows
            Rl = 0;
            size_t i = 0;
            for (; i < rem.size(); ++i) {
              const uint32_t need = actl[rem[i]];
              if (__builtin_popcount(Rl | need) > RB) break;
              Rl |= need;
              took.push_back(rem[i]);
            }
            left.assign(rem.begin() + (long)i, rem.end());
          }
          require(!took.empty(), SVB_E_CUDA, "scheduler: empty round");
          rounds.push_back({Rl, took});
          rem.swap(left);
        }
      }
      const uint32_t lane_local = 0x1fu;  // local bits 0..4 are physical 0..4
      auto fill = [&](uint32_t r) {
        for (int b = 5; b < m && __builtin_popcount(r) < RB; ++b) r |= 1u << b;
        for (int b = 0; b < 5 && __builtin_popcount(r) < RB; ++b) r |= 1u << b;
        return r;
      };
      std::vector<uint32_t> regsets;
      for (auto& rd : rounds) regsets.push_back(fill(rd.first));
      if (regsets.back() & lane_local) {
        rounds.push_back({0u, {}});
        regsets.push_back(fill(0u));
      }
      // (direct is set after the kMaxRounds trim below)
      if ((int)rounds.size() > kMaxRounds) {
        // defer the tail of this pass's ops to the next pass (original order kept)
        std::vector<int> keep_ops;
        std::vector<std::pair<uint32_t, std::vector<int>>> kept(rounds.begin(), rounds.begin() + kMaxRounds - 1);
        std::vector<int> deferred;
        for (size_t k = kMaxRounds - 1; k < rounds.size(); ++k)
          deferred.insert(deferred.end(), rounds[k].second.begin(), rounds[k].second.end());
        rounds = kept;
        regsets.resize(kMaxRounds - 1);
        if (regsets.back() & lane_local) {
          rounds.push_back({0u, {}});
          regsets.push_back(fill(0u));
        }
        skipped.insert(skipped.end(), deferred.begin(), deferred.end());
        std::sort(skipped.begin(), skipped.end());
      }
      // round 0 without lane register bits: its layout is coalesced in HBM, so
      // a single-stage kernel can load it straight into registers (no ring)
      pd.direct = (regsets[0] & lane_local) == 0 ? 1 : 0;

      // ---- encode the rounds
      //
      // Deferred pivot diagonals: an unconditional 1q op M on q (after the
      // pending diagonal diag(1, dl[q]) of q) is factored as diag(p0, p1) * P,
      // where each row of P has a unit pivot: y_r = x_pc[r] + ratio_r x_(1-pc[r]).
      // P costs one complex FMA per amplitude (two real FMAs for a real ratio)
      // instead of two complex products; diag(p0, p1) = p0 * diag(1, p1/p0) is
      // carried forward: the scalar p0 into the pass-global K, the rest into dl[q].
      // Diagonals commute with diagonal ops; a conditional 1q op on q sees
      // D^-1 M D; a 2q op absorbs its qubits' pending diagonals into its
      // columns.  The pass's last unconditional dense 1q op absorbs K and is
      // emitted in full; leftover pending diagonals and K are flushed as one
      // DIAG op at the end of the last round.
      Encoder<R> enc(prog.ops);
      pd.nrounds = (int)rounds.size();
      pd.ops_begin = (uint32_t)prog.ops.size();
      std::vector<cd> dl(n, cd(1.0, 0.0));
      cd K(1.0, 0.0);
      // structural mode: which pending diagonals were ever set (flushed even
      // when they come out as 1) and pivots since the last rescale
      std::vector<char> dtouch(n, 0);
      bool ktouch = false;
      int npiv = 0;
      int last_u1 = -1;
      for (auto& rd : rounds)
        for (int idx : rd.second) {
          const FOp& f = ops[idx];
          if ((f.type == OP_U1 || f.type == OP_U1R || f.type == OP_U1X) && f.conds.empty()) last_u1 = idx;
        }
      auto u1_type = [](const cd* M) {
        if (zero(M[0]) && zero(M[3])) return (int)OP_U1ANTI;
        if (M[0].imag() == 0 && M[1].imag() == 0 && M[2].imag() == 0 && M[3].imag() == 0) return (int)OP_U1R;
        if (M[0].imag() == 0 && M[3].imag() == 0 && M[1].real() == 0 && M[2].real() == 0) return (int)OP_U1X;
        return (int)OP_U1;
      };
      struct DT { int qa, qb; cd e[4]; };
      for (size_t k = 0; k < rounds.size(); ++k) {
        RoundDev& rd = pd.rounds[k];
        uint32_t regs = regsets[k];
        rd.regmask_local = regs;
        int regidx_of_local[kMaxM];
        for (int b = 0, i = 0; b < m; ++b) {
          regidx_of_local[b] = -1;
          if (regs & (1u << b)) { rd.reg_local[i] = b; regidx_of_local[b] = i; ++i; }
        }
        for (int b = 0, t = 0; b < m; ++b)
          if (!(regs & (1u << b))) rd.thr_local[t++] = (uint8_t)b;
        auto ridx = [&](int q) { return (q >= 0 && local_of[q] >= 0) ? regidx_of_local[local_of[q]] : -1; };
        // one DIAG op from a list of 2-qubit (or 1-qubit, qb = -1) factors
        auto encode_diag = [&](const std::vector<DT>& terms) {
          // classify each factor by where its qubits live in this round
          enum { NONE, TILE, THREAD, REG };
          auto cls = [&](int q) {
            if (q < 0) return (int)NONE;
            if (local_of[q] < 0) return (int)TILE;
            return regidx_of_local[local_of[q]] >= 0 ? (int)REG : (int)THREAD;
          };
          const bool uniform_ok = pd.ndiag < kMaxDiag && pd.nitems + 7 + kMaxUT <= kMaxItems;
          std::vector<DiagTerm<R>> ur[6], uc, tr, tc, rr;
          std::vector<int> ut_q;                       // thread qubit of each UT group
          std::vector<std::vector<DiagTerm<R>>> ut;    // UT terms per group
          for (const DT& d : terms) {
            int qa = d.qa, qb = d.qb;
            cd e[4] = {d.e[0], d.e[1], d.e[2], d.e[3]};
            int ca = cls(qa), cb = cls(qb);
            // register qubit first; else thread qubit first
            if ((ca != REG && cb == REG) || ((ca == TILE || ca == NONE) && cb == THREAD)) {
              std::swap(qa, qb);
              std::swap(ca, cb);
              std::swap(e[1], e[2]);
            }
            DiagTerm<R> term{};
            term.qa = (int8_t)qa;
            term.qb = (int8_t)qb;
            term.ra = (int8_t)(ca == REG ? ridx(qa) : -1);
            term.rb = (int8_t)(cb == REG ? ridx(qb) : -1);
            for (int k2 = 0; k2 < 4; ++k2) term.d[k2] = cvt<R>(e[k2]);
            const bool ubit = (cb == TILE || cb == NONE);
            if (ca == REG && cb == REG) rr.push_back(term);
            else if (ca == REG && cb == THREAD) tr.push_back(term);
            else if (ca == REG) (uniform_ok ? ur[term.ra] : tr).push_back(term);
            else if ((ca == TILE || ca == NONE) && ubit && uniform_ok) uc.push_back(term);
            else if (ca == THREAD && ubit && uniform_ok && !zero(e[0]) && !zero(e[2])) {
              size_t g = 0;
              while (g < ut_q.size() && ut_q[g] != qa) ++g;
              if (g == ut_q.size()) {
                if ((int)g == kMaxUT) { tc.push_back(term); continue; }
                ut_q.push_back(qa);
                ut.emplace_back();
              }
              // constant part per tile-bit value and the thread-bit ratio
              const cd r0 = snap(e[1] / e[0]), r1 = snap(e[3] / e[2]);
              term.d[0] = cvt<R>(e[0]);
              term.d[1] = cvt<R>(r0);
              term.d[2] = cvt<R>(e[2]);
              term.d[3] = cvt<R>(r1);
              ut[g].push_back(term);
            } else tc.push_back(term);
          }
          size_t at = enc.begin(OP_DIAG, 0, 0, (int)terms.size(), 0, 0, 0, 0);
          DiagHdr hd{};
          for (int k2 = 0; k2 < 6; ++k2) hd.nUR[k2] = (int32_t)ur[k2].size();
          hd.nUC = (int32_t)uc.size();
          hd.nTR = (int32_t)tr.size();
          hd.nTC = (int32_t)tc.size();
          hd.nRR = (int32_t)rr.size();
          bool any_uniform = !uc.empty() || !ut.empty();
          for (int k2 = 0; k2 < 6; ++k2) any_uniform = any_uniform || !ur[k2].empty();
          hd.slot = (uniform_ok && any_uniform) ? pd.ndiag : -1;
          if (hd.slot >= 0) {  // the pass's tile-uniform work items (PassDev::items)
            auto item = [&](int kind, int idx) {
              require(pd.nitems < kMaxItems, SVB_E_CUDA, "scheduler: too many uniform items");
              pd.items[pd.nitems++] = (uint16_t)(hd.slot | (kind << 8) | (idx << 10));
            };
            for (int k2 = 0; k2 < 6; ++k2)
              if (!ur[k2].empty()) item(0, k2);
            if (!uc.empty() || !ut.empty()) item(1, 0);
            for (size_t g = 0; g < ut.size(); ++g) item(2, (int)g);
          }
          hd.nUTg = (int32_t)ut.size();
          for (size_t g = 0; g < ut.size(); ++g) {
            require(ut[g].size() <= 255, SVB_E_CUDA, "scheduler: UT group too large");
            hd.utn[g] = (uint8_t)ut[g].size();
          }
          if (hd.slot >= 0) pd.diag_off[pd.ndiag++] = (uint32_t)prog.ops.size();
          enc.put(hd);
          for (int k2 = 0; k2 < 6; ++k2)
            for (auto& x : ur[k2]) enc.put(x);
          for (auto& x : uc) enc.put(x);
          for (auto& g : ut)
            for (auto& x : g) enc.put(x);
          for (auto* lst : {&tr, &tc, &rr})
            for (auto& x : *lst) enc.put(x);
          enc.end(at);
        };
        auto encode_u1 = [&](int type, int b, const cd* M, uint64_t fm, uint64_t fv, uint32_t rm, uint32_t rv) {
          size_t at = enc.begin(type, b, 0, 0, fm, fv, rm, rv);
          for (int e = 0; e < 4; ++e) enc.put(cvt<R>(M[e]));
          enc.end(at);
        };
        rd.op_off = (uint32_t)prog.ops.size();
        const std::vector<int>& list = rounds[k].second;
        size_t i = 0;
        while (i < list.size()) {
          const FOp& f = ops[list[i]];
          if (f.type == OP_DIAG) {
            size_t j = i;
            while (j < list.size() && ops[list[j]].type == OP_DIAG) ++j;
            std::vector<DT> terms;
            for (size_t t = i; t < j; ++t) {
              const FOp& d = ops[list[t]];
              if (d.q[1] < 0 && d.q[0] >= 0 && local_of[d.q[0]] >= 0 && !zero(d.c[0])) {
                // 1q diagonal on a tile qubit: fold into the pending diagonal
                K *= d.c[0];
                dl[d.q[0]] *= d.c[1] / d.c[0];
                dtouch[d.q[0]] = 1;
                ktouch = true;
                continue;
              }
              terms.push_back(DT{d.q[0], d.q[1], {d.c[0], d.c[1], d.c[2], d.c[3]}});
            }
            if (!terms.empty()) encode_diag(terms);
            i = j;
            continue;
          }
          if (f.type == OP_U1 || f.type == OP_U1R || f.type == OP_U1X || f.type == OP_U1ANTI) {
            uint64_t fm = 0, fv = 0;
            uint32_t rm = 0, rv = 0;
            for (auto& cv : f.conds) {
              int ri = ridx(cv.first);
              if (ri >= 0) { rm |= 1u << ri; rv |= (uint32_t)cv.second << ri; }
              else { fm |= 1ull << cv.first; fv |= (uint64_t)cv.second << cv.first; }
            }
            const int q = f.q[0];
            int b = ridx(q);
            require(b >= 0, SVB_E_CUDA, "scheduler: U1 target not in registers");
            const cd d1 = dl[q];
            if (!f.conds.empty()) {
              // conditional op: pass the pending diagonal through (D^-1 M D)
              cd M[4] = {f.c[0], f.c[1] * d1, f.c[2] / d1, f.c[3]};
              for (auto& z : M) z = snap(z);
              encode_u1(u1_type(M), b, M, fm, fv, rm, rv);
              ++i;
              continue;
            }
            cd M[4] = {f.c[0], f.c[1] * d1, f.c[2], f.c[3] * d1};  // M * diag(1, d1)
            dl[q] = cd(1.0, 0.0);
            if (zero(M[1]) && zero(M[2])) {  // diagonal: defer entirely
              K *= M[0];
              dl[q] = snap(M[3] / M[0]);
              dtouch[q] = 1;
              ktouch = true;
              ++i;
              continue;
            }
            if (zero(M[0]) && zero(M[3])) {  // anti-diagonal: plain swap + deferred diag(m01, m10)
              K *= M[1];
              dl[q] = snap(M[2] / M[1]);
              dtouch[q] = 1;
              ktouch = true;
              const cd sw[4] = {cd(0.0, 0.0), cd(1.0, 0.0), cd(1.0, 0.0), cd(0.0, 0.0)};
              encode_u1(OP_U1ANTI, b, sw, 0, 0, 0, 0);
              ++i;
              continue;
            }
            // the stored amplitudes carry 1/K: once |K| drifts far from 1 (long
            // passes of pivoted ops), emit this op in full to rescale (keeps
            // complex64 values far from overflow / underflow)
            // (structural mode: every 8 / 64 pivots; a pivot scales by >= 2^-8.5,
            // so |K| stays within 2^68 (c64) / 2^544 (c128) of 1)
            const double klog = std::fabs(std::log2(std::abs(K)));
            const bool rescale = opt.structural ? npiv >= (sizeof(R) == 4 ? 8 : 64)
                                                : klog > (sizeof(R) == 4 ? 20.0 : 100.0);
            if (list[i] == last_u1 || rescale) {  // absorbs K; emitted in full
              for (auto& z : M) z = snap(z) * K;  // snap is absolute: before scaling
              K = cd(1.0, 0.0);
              npiv = 0;
              encode_u1(u1_type(M), b, M, 0, 0, 0, 0);
              ++i;
              continue;
            }
            // pivots: the diagonal entry unless it is much smaller than its
            // neighbour; row 1 prefers an entry equal to p0 (keeps D scalar)
            const int pc0 = (std::abs(M[0]) >= 0x1p-8 * std::abs(M[1])) ? 0 : 1;
            const cd p0 = M[pc0];
            auto close = [](cd x, cd y) { return std::abs(x - y) <= 0x1p-50 * std::abs(y); };
            int pc1;
            if (close(M[2], p0) && std::abs(M[2]) >= 0x1p-8 * std::abs(M[3])) pc1 = 0;
            else if (close(M[3], p0)) pc1 = 1;
            else pc1 = (std::abs(M[3]) >= 0x1p-8 * std::abs(M[2])) ? 1 : 0;
            const cd p1 = M[2 + pc1];
            const cd r0 = snap(M[1 - pc0] / p0), r1 = snap(M[2 + (1 - pc1)] / p1);
            K *= p0;
            dl[q] = close(p1, p0) ? cd(1.0, 0.0) : snap(p1 / p0);
            dtouch[q] = 1;
            ktouch = true;
            ++npiv;
            const bool real = r0.imag() == 0 && r1.imag() == 0;
            size_t at = enc.begin(real ? OP_U1PR : OP_U1P, b, 0, pc0 | (pc1 << 1), 0, 0, 0, 0);
            enc.put(cvt<R>(r0));
            enc.put(cvt<R>(r1));
            enc.end(at);
          } else {
            int b1 = ridx(f.q[0]), b2 = ridx(f.q[1]);
            require(b1 >= 0 && b2 >= 0, SVB_E_CUDA, "scheduler: U2 qubits not in registers");
            // absorb the pending diagonals of both qubits into the input columns
            const cd da = dl[f.q[0]], db = dl[f.q[1]];
            auto colf = [&](int c) { return ((c & 1) ? da : cd(1.0, 0.0)) * ((c & 2) ? db : cd(1.0, 0.0)); };
            dl[f.q[0]] = dl[f.q[1]] = cd(1.0, 0.0);
            size_t at = enc.begin(f.type, b1, b2, 0, 0, 0, 0, 0);
            if (f.type == OP_U2) {
              for (int e = 0; e < 16; ++e) enc.put(cvt<R>(snap(f.c[e] * colf(e & 3))));
            } else {
              int32_t s4[4] = {f.src[0], f.src[1], f.src[2], f.src[3]};
              enc.put(s4);
              for (int e = 0; e < 4; ++e) enc.put(cvt<R>(snap(f.c[e] * colf(f.src[e]))));
            }
            enc.end(at);
          }
          ++i;
        }
        if (k + 1 == rounds.size()) {
          // flush: pending per-qubit diagonals and the global scalar
          std::vector<DT> terms;
          for (int q = 0; q < n; ++q) {
            const cd d1 = snap(dl[q]);
            if (!(d1.real() == 1.0 && d1.imag() == 0.0) || (opt.structural && dtouch[q]))
              terms.push_back(DT{q, -1, {cd(1.0, 0.0), d1, cd(1.0, 0.0), d1}});
          }
          if (std::abs(K - cd(1.0, 0.0)) <= 0x1p-50) K = cd(1.0, 0.0);  // not snap(): |K| may be tiny
          if (!(K.real() == 1.0 && K.imag() == 0.0) || (opt.structural && ktouch)) terms.push_back(DT{-1, -1, {K, K, K, K}});
          if (!terms.empty()) encode_diag(terms);
        }
        rd.op_end = (uint32_t)prog.ops.size();
      }
      pd.ops_bytes = (uint32_t)prog.ops.size() - pd.ops_begin;
      require(pd.ops_bytes <= kMaxPassOpBytes, SVB_E_CUDA, "scheduler: pass op stream too large");
    if (!search || slots_fit<R>(prog, pd)) break;
    pd = pd_saved;
    prog.ops.resize(ops_saved);
    skipped = skipped_saved;
    }
    prog.passes.push_back(pd);
    support |= S;
    remaining = skipped;
  }
  prog.support = opt.zero_start ? support : ~0ull;
  if (std::getenv("SVB_TRACE_OPS")) {  // the op stream per pass and round (scheduler debugging)
    static const char* kname[] = {"DIAG", "U1", "U1ANTI", "U2", "PERM2", "U1R", "U1X", "U1P", "U1PR"};
    for (size_t p = 0; p < prog.passes.size(); ++p) {
      const PassDev& pd = prog.passes[p];
      for (int k = 0; k < pd.nrounds; ++k) {
        std::fprintf(stderr, "[svb] pass %zu round %d regs", p, k);
        for (int i = 0; i < pd.rb; ++i) std::fprintf(stderr, " q%d", pd.pos[pd.rounds[k].reg_local[i]]);
        std::fprintf(stderr, " thr");
        for (int b = 0; b < pd.m - pd.rb; ++b) std::fprintf(stderr, " q%d", pd.pos[pd.rounds[k].thr_local[b]]);
        std::fprintf(stderr, ":");
        for (uint32_t off = pd.rounds[k].op_off; off < pd.rounds[k].op_end;) {
          OpHdr h;
          std::memcpy(&h, prog.ops.data() + off, sizeof h);
          std::fprintf(stderr, " %s(a%d b%d n%d%s%s)", h.kind >= 0 && h.kind <= 8 ? kname[h.kind] : "?", h.a, h.b, h.n,
                       h.fmask ? " F" : "", h.rmask ? " R" : "");
          if (h.kind == OP_DIAG) {
            DiagHdr d;
            std::memcpy(&d, prog.ops.data() + off + sizeof(OpHdr), sizeof d);
            std::fprintf(stderr, "[UR%d UC%d TR%d TC%d RR%d UT%d]", d.nUR[0] + d.nUR[1] + d.nUR[2] + d.nUR[3] + d.nUR[4] + d.nUR[5],
                         d.nUC, d.nTR, d.nTC, d.nRR, d.nUTg);
          }
          off += h.bytes;
        }
        std::fprintf(stderr, "\n");
      }
    }
  }
  if (opt.zero_start && std::getenv("SVB_TRACE"))
    std::fprintf(stderr, "[svb] zero-start support %llx over %zu passes\n", (unsigned long long)support,
                 prog.passes.size());
  bool ident = true;
  for (int q = 0; q < n; ++q) ident = ident && phys[q] == q;
  if (!ident) {
    // data of logical qubit q sits at physical bit phys[q]; move it to bit q
    prog.final_perm.assign(n, 0);
    for (int q = 0; q < n; ++q) prog.final_perm[phys[q]] = q;
    fuse_final_permutation(prog, n);
  }
  return prog;
}

static int64_t total_rounds(const Program& p) {
  int64_t r = 0;
  for (const PassDev& pd : p.passes) r += pd.nrounds;
  return r;
}

// With swap relabeling on a written (non-lazy) input the final layout must be
// undone by a permutation either way; doing it FIRST (permute the input into
// the layout that absorbs the relabeling) can give much cheaper passes (the
// QFT's bit reversal: 14 -> 8 rounds over its 4 passes), so both schedules are
// built and the one with fewer passes, then fewer rounds, is kept.
template <typename R>
Program build_program(int n, const svb_gate* gates, int ng, const SchedOptions& opt) {
  if (!opt.relabel_swaps || opt.zero_start) return build_program_layout<R>(n, gates, ng, opt, opt.zero_start);
  Program a = build_program_layout<R>(n, gates, ng, opt, false);
  if (a.final_perm.empty() || a.perm_fused || !opt.initial_perm) return a;
  Program b = build_program_layout<R>(n, gates, ng, opt, true);
  if (!b.final_perm.empty()) return a;
  if (b.passes.size() > a.passes.size() ||
      (b.passes.size() == a.passes.size() && total_rounds(b) >= total_rounds(a)))
    return a;
  // input bit q moves to physical bit phys_init[q] = tau^-1(q), and a's final
  // map (physical bit p -> logical bit final_perm[p]) is that same tau^-1
  b.init_perm = a.final_perm;
  return b;
}

template Program build_program<float>(int, const svb_gate*, int, const SchedOptions&);
template Program build_program<double>(int, const svb_gate*, int, const SchedOptions&);

// Fold the program's initial permutation (input bit q -> layout bit
// init_perm[q]) into the first pass's tile loads (PassDev::perm_in): the pass
// reads the input buffer at the permuted addresses and writes the other
// buffer in the program's layout, which saves the separate permutation sweep
// (2 s 2^n bytes).  The tile's load order takes its local bits by ascending
// input position, so a warp's 32 loads cover one contiguous run; when the
// tile does not contain input bits 0..4 (complex128) / 0..5 (complex64),
// the loads would not be coalesced and the permutation stays a pass.
template <typename R>
bool fuse_initial_permutation(Program& prog, int n) {
  if (prog.init_perm.empty() || prog.passes.empty()) return false;
  PassDev& pd = prog.passes[0];
  if (pd.dmask || pd.perm_out || pd.m > 16) return false;
  std::vector<int> inv(n, -1);
  for (int q = 0; q < n; ++q) inv[prog.init_perm[q]] = q;
  std::vector<std::pair<int, int>> ord;  // (input position, local bit)
  for (int l = 0; l < pd.m; ++l) ord.push_back({inv[pd.pos[l]], l});
  std::sort(ord.begin(), ord.end());
  if (std::getenv("SVB_TRACE")) {
    std::fprintf(stderr, "[svb] perm_in candidate: input positions of the first tile:");
    for (auto& o : ord) std::fprintf(stderr, " %d(l%d)", o.first, o.second);
    std::fprintf(stderr, "\n");
  }
  const int run_bits = sizeof(R) == 8 ? 5 : 6;
  for (int b = 0; b < run_bits; ++b)
    if (ord[b].first != b) return false;
  // complex64 copies aligned pairs (local bits 0 of slot and address agree)
  if (sizeof(R) == 4 && ord[0].second != 0) return false;
  for (int l = 0; l < pd.m; ++l) pd.ipos[l] = inv[pd.pos[l]];
  for (int i = 0; i < pd.nout; ++i) pd.ioutpos[i] = inv[pd.outpos[i]];
  for (int b = 0; b < pd.m; ++b) pd.ld_local[b] = (uint8_t)ord[b].second;
  pd.perm_in = 1;
  pd.direct = 0;  // the direct first round reads through pos: the ring path loads
  return true;
}
template bool fuse_initial_permutation<float>(Program&, int);
template bool fuse_initial_permutation<double>(Program&, int);

// ------------------------------------------------------------- emulation
static uint64_t permute_index(const PassDev& pd, uint64_t g) {
  uint64_t o = 0;
  for (int l = 0; l < pd.m; ++l)
    if ((g >> pd.pos[l]) & 1ull) o |= 1ull << pd.dpos[l];
  for (int i = 0; i < pd.nout; ++i)
    if ((g >> pd.outpos[i]) & 1ull) o |= 1ull << pd.doutpos[i];
  return o;
}

// out: destination of a permuted-store pass (pd.perm_out), else unused
template <typename R, int RB>
static void emulate_pass(cplx<R>* state, cplx<R>* out, int n, const PassDev& pd, const uint8_t* ops) {
  constexpr int V = 1 << RB;
  const int m = pd.m;
  const uint32_t NT = 1u << (m - RB);
  std::vector<cplx<R>> tile((size_t)1 << m);
  const uint64_t ntiles = 1ull << pd.nout;
  std::vector<cplx<R>> uni((size_t)kMaxDiag * kUniStride);
  for (uint64_t t = 0; t < ntiles; ++t) {
    const uint64_t base = tile_base(pd, t);
    for (int d = 0; d < pd.ndiag; ++d)
      diag_uniform_serial<R, RB>(ops + pd.diag_off[d], base, uni.data() + (size_t)d * kUniStride);
    for (int k = 0; k < pd.nrounds; ++k) {
      const RoundDev& rd = pd.rounds[k];
      for (uint32_t tid = 0; tid < NT; ++tid) {
        uint32_t Fl;
        uint64_t Fg;
        thread_fixed(pd, rd, tid, base, &Fl, &Fg);
        cplx<R> a[V];
        uint64_t gidx[V];
        uint32_t lidx[V];
        for (int v = 0; v < V; ++v) {
          uint64_t g = Fg;
          uint32_t lo = Fl;
          for (int i = 0; i < RB; ++i)
            if ((v >> i) & 1) { g |= 1ull << pd.pos[rd.reg_local[i]]; lo |= 1u << rd.reg_local[i]; }
          gidx[v] = g;
          lidx[v] = lo;
          a[v] = (k == 0) ? state[g] : tile[lo];
        }
        run_ops<R, RB>(a, Fg, ops, rd.op_off, rd.op_end, uni.data());
        for (int v = 0; v < V; ++v) {
          if (k < pd.nrounds - 1) tile[lidx[v]] = a[v];
          else if (pd.perm_out) out[permute_index(pd, gidx[v])] = a[v];
          else state[gidx[v]] = a[v];
        }
      }
    }
  }
}

template <typename R>
void emulate_program(cplx<R>* state, int n, const Program& prog) {
  if (!prog.init_perm.empty()) {
    const uint64_t len = 1ull << n;
    std::vector<cplx<R>> tmp(len);
    for (uint64_t i = 0; i < len; ++i) {
      uint64_t o = 0;
      for (int p = 0; p < n; ++p)
        if ((i >> p) & 1) o |= 1ull << prog.init_perm[p];
      tmp[o] = state[i];
    }
    std::copy(tmp.begin(), tmp.end(), state);
  }
  std::vector<cplx<R>> out(prog.perm_fused ? (size_t)1 << n : 0);
  for (const PassDev& pd : prog.passes) {
    if (pd.rb == 4) emulate_pass<R, 4>(state, out.data(), n, pd, prog.ops.data());
    else emulate_pass<R, 5>(state, out.data(), n, pd, prog.ops.data());
  }
  if (prog.perm_fused) {
    std::copy(out.begin(), out.end(), state);
  } else if (!prog.final_perm.empty()) {
    uint64_t len = 1ull << n;
    std::vector<cplx<R>> out(len);
    for (uint64_t i = 0; i < len; ++i) {
      uint64_t o = 0;
      for (int p = 0; p < n; ++p)
        if ((i >> p) & 1) o |= 1ull << prog.final_perm[p];
      out[o] = state[i];
    }
    std::copy(out.begin(), out.end(), state);
  }
}

template void emulate_program<float>(cplx<float>*, int, const Program&);
template void emulate_program<double>(cplx<double>*, int, const Program&);

SchedOptions default_options(int precision, int n, bool jit) {
  SchedOptions o;
  if (precision == SVB_C128) { o.rb = jit ? kJitRegBits<double> : kRegBits<double>; o.m = 12; }
  else { o.rb = jit ? kJitRegBits<float> : kRegBits<float>; o.m = pass_tile_m(4, o.rb); }
  o.structural = jit && n < kJitImmMinQubits;
  if (const char* e = std::getenv("SVB_STRUCTURAL")) o.structural = o.structural && std::atoi(e) != 0;  // A/B runs
  return o;
}

}  // namespace svb
