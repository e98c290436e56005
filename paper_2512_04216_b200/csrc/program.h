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
#include "device_core.cuh"

namespace svb {

// Optional per-kernel CUDA-event timing on the launching stream.
struct Profiler {
  bool on = false;
  struct Rec { cudaEvent_t a, b; int kind, idx; double bytes; };  // kind 0 = k_pass, 1 = k_permute
  std::vector<Rec> pending;
  double ms[2] = {0, 0};
  int64_t count[2] = {0, 0};
  double bytes[2] = {0, 0};
  // per pass index of a program (idx): summed ms, HBM bytes and launches,
  // so the dominant pass of repeated applies can be reported on its own
  std::vector<double> idx_ms, idx_bytes;
  std::vector<int64_t> idx_count;
  void begin(cudaStream_t st, int kind, double nbytes, int idx = -1);
  void end(cudaStream_t st);
  void collect();  // after a stream sync
};

struct ProgramStats {
  int64_t passes = 0, gates = 0, launches = 0;
  Profiler* prof = nullptr;
};

// ------------------------------------------------------------- host side
struct Program {
  std::vector<PassDev> passes;
  std::vector<uint8_t> ops;          // op stream (all passes)
  std::vector<int> final_perm;       // physical bit p must move to bit final_perm[p]; empty = identity
  bool perm_fused = false;
  std::vector<int> init_perm;        // input bit q moves to bit init_perm[q] before the passes; empty = none
  uint64_t support = ~0ull;          // zero_start: qubits the passes wrote; positions with other bits are never written           // final_perm is done by the last pass's permuted store (PassDev::perm_out)
  int64_t gates = 0;
  int n = 0;                         // qubits of the state
};

struct SchedOptions {
  int rb = 4;        // register bits per thread
  int m = 12;        // tile qubits
  bool relabel_swaps = true;
  bool zero_start = false;   // input is |0...0>: choose the initial qubit layout so no final permutation is needed
  bool initial_perm = true;  // written input + swaps: may permute the input first (see build_program)
  bool round_search = true;  // reorder ops across rounds (else program order)
  // structure-only NVRTC code (n < kJitImmMinQubits): the op stream's shape
  // must not depend on the angles, so that circuits differing only in angles
  // share kernels -- deferred pivot diagonals are flushed for every qubit that
  // had one (even when the factor comes out as exactly 1) and the rescale of
  // the carried scalar happens every few pivots instead of when |K| drifts
  bool structural = false;
};
constexpr int kJitImmMinQubits = 28;  // from here the NVRTC passes take coefficients as immediates

// jit: the options of a program the NVRTC passes will run (kJitRegBits)
SchedOptions default_options(int precision, int n, bool jit = false);
constexpr int kDefaultJitMinQubits = 24;  // a handle's NVRTC threshold (SVB_OPT_JIT_MIN_N)

template <typename R>
Program build_program(int n, const svb_gate* gates, int ng, const SchedOptions& opt);

// the initial permutation of `prog` folded into its first pass (PassDev::perm_in)
template <typename R>
bool fuse_initial_permutation(Program& prog, int n);

template <typename R>
void run_program(void* state, int n, const svb_gate* g, int ng, int fusion, int max_high,
                 cudaStream_t st, ProgramStats* stats);

// As run_program, but may replace *state (swap relabeling ends with an
// out-of-place permutation pass into a fresh cudaMalloc buffer).
// *spare: a second state-sized buffer owned by the handle (allocated on first
// use, nullptr if it cannot be); the permutation writes into it and swaps.
// fusion: 0 = one pass per gate, 1 = fused passes.  jit_min_n: specialise the
// fused passes with NVRTC when n >= jit_min_n (negative: never).
template <typename R>
void run_permutation(void** state, void** spare, int n, const std::vector<int>& dest, cudaStream_t st,
                     ProgramStats* stats);

// Fused single-qubit <Z> (optional argument of run_program_owned): when
// `want`, the last fused pass accumulates sum p (-1)^bit for every qubit and
// d_out (device, >= kZaccRows doubles) receives them; `fused` reports whether
// that happened (else the caller runs a separate reduction) and logical[k] is
// the logical qubit of value k (-1: the total sum p).
struct ZRequest {
  bool want = false;
  double* d_out = nullptr;
  double* d_acc = nullptr;  // zacc_doubles() accumulators (device)
  bool fused = false;
  std::vector<int> logical;
};

// zero_pending (may be null): the state is a lazy |0...0>; the first fused
// pass synthesises it instead of reading HBM (other paths write it first).
template <typename R>
void run_program_owned(void** state, void** spare, int n, const svb_gate* g, int ng, int fusion, int jit_min_n,
                       cudaStream_t st, ProgramStats* stats, bool* zero_pending, ZRequest* z = nullptr);

// CPU emulation of a program on a host state (same op interpreter).
template <typename R>
void emulate_program(cplx<R>* state, int n, const Program& prog);

}  // namespace svb
