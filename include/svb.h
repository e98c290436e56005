/*
 * svb.h — C ABI of the B200 state-vector backend (libsvb.so).
 *
 * This is the drop-in boundary for the reference's dense state-vector path
 * (`polysim/statevector.py`).  Every entry point below names the reference
 * interface it replaces.  Signatures carry plain pointers and sizes only; the
 * Python boundary module `paper_2512_04216_b200/statevector.py` binds them
 * with ctypes, exactly as a maintainer of the reference would.
 *
 * Conventions (identical to the reference):
 *   - qubit 0 is the least significant bit of the amplitude index
 *     (statevector.py:3-4);
 *   - a 2-qubit matrix acts on local index bit(q[0]) + 2*bit(q[1])
 *     (gates.py:3-5, 69-74);
 *   - host amplitude buffers are interleaved complex128 (re, im) doubles,
 *     i.e. numpy complex128 memory, regardless of the device precision.
 *
 * Errors: every function returns an svb_status; the message of the last
 * failure on the calling thread is svb_last_error().  The Python layer maps
 *   SVB_E_CAP -> QubitCapError, SVB_E_ARG -> ValueError,
 *   SVB_E_SAMPLING -> SamplingError (a ValueError, sampling.py:17-18),
 *   SVB_E_OOM / SVB_E_CUDA / SVB_E_NCCL -> BackendError  (result.py:12-21).
 *
 * Thread-safety: distinct handles may be used from distinct threads; one
 * handle is confined to one thread at a time.  Every call that
 * takes host buffers is synchronous on return.
 */
#ifndef SVB_H
#define SVB_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  SVB_OK = 0,
  SVB_E_ARG = 1,
  SVB_E_CAP = 2,
  SVB_E_OOM = 3,
  SVB_E_CUDA = 4,
  SVB_E_NCCL = 5,
  SVB_E_SAMPLING = 6
} svb_status;

typedef enum { SVB_C64 = 0, SVB_C128 = 1 } svb_precision;

typedef enum {
  SVB_SAMPLER_ALIAS = 0, /* reference-compatible Walker/Vose table, sampling.py:30-83 */
  SVB_SAMPLER_CDF = 1    /* fused |amp|^2 block prefix + binary-search multinomial */
} svb_sampler;

typedef struct svb_state* svb_handle;

/* One unitary of a gate program.  k = 1 or 2 qubits; mat is the row-major
 * 2^k x 2^k complex matrix as (re, im) pairs (2x2 uses the first 8 doubles).
 * Replaces one `apply_instruction` call (statevector.py:116-122). */
typedef struct {
  int32_t k;
  int32_t qubits[2];
  int32_t reserved;
  double mat[32];
} svb_gate;

/* Compact gate record (40 B) for batches: kind 0 = rx, 1 = ry, 2 = rz,
 * 3 = u(p[0], p[1], p[2]) (matrices from gates.py's formulas, evaluated in
 * C++), kind >= 4 = fixed gate `fixed[kind - 4]` (a caller-supplied table of
 * svb_gate matrices, e.g. h x y z s sdg t tdg cx cz swap). */
typedef struct {
  int32_t kind;
  int32_t q0, q1;
  int32_t reserved;
  double p[3];
} svb_gate_op;
/* ops[i] -> out[i] (host-only; the batch executor's expansion, for tests). */
int svb_expand_gates(const svb_gate_op* ops, int n, const svb_gate* fixed, svb_gate* out);

/* Library / device info. */
const char* svb_last_error(void);
int svb_version(void);
/* Largest n whose state (plus sampling workspace) fits on `device`. */
int svb_max_qubits(int device, int precision, int* out_n);
/* Page-locked host buffers (fast final_state copies). */
int svb_host_alloc(uint64_t bytes, void** out);
int svb_host_free(void* p);

typedef enum {
  SVB_OPT_FUSION = 0,   /* 1 (default): fused multi-gate HBM passes; 0: one pass per gate */
  SVB_OPT_MAX_HIGH = 1,  /* fused pass: max non-lane qubits per pass (tuning; default auto) */
  SVB_OPT_JIT_MIN_N = 2, /* NVRTC-specialise fused passes for n >= value (default 24; -1 never) */
  SVB_OPT_TC_MIN_K = 3   /* svb_apply_matrix (engine AUTO): tensor cores for complex64 blocks of >= value qubits (default 5) */
} svb_option;
int svb_set_option(svb_handle h, int option, int value);
/* Statistics of the last svb_apply: HBM passes launched, gates applied. */
int svb_last_stats(svb_handle h, int64_t* n_passes, int64_t* n_gates, int64_t* n_launches);
int svb_sync(svb_handle h);
/* CUDA-event timing on the handle's stream (the stream every kernel of the
 * handle is launched on).  svb_profile(h, 1) additionally times every fused
 * pass and permutation launch; svb_profile_read fills out[6] =
 * {pass_ms, pass_launches, pass_bytes, perm_ms, perm_launches, perm_bytes}
 * (bytes = algorithmic 2*s*2^n per launch). */
int svb_timer_start(svb_handle h);
int svb_timer_stop(svb_handle h, double* ms);
int svb_profile(svb_handle h, int enable);
int svb_profile_read(svb_handle h, double* out);
/* Per pass index of the programs applied while profiling: out[3*i .. 3*i+2] =
 * (summed ms, summed HBM bytes moved, launches) for i < min(*n, cap). */
int svb_profile_passes(svb_handle h, double* out, int cap, int* n);

/* State lifetime: zero_state (statevector.py:125-128). */
int svb_create(int n_qubits, int precision, int device, svb_handle* out);
int svb_destroy(svb_handle h);
int svb_set_zero(svb_handle h);
int svb_copy_state(svb_handle dst, svb_handle src); /* prefix.copy(), statevector.py:168 */
int svb_n_qubits(svb_handle h);
/* Kernel-level numpy API on device-resident memory (statevector.py:33-154 as
 * used by calibration.py:215-228 and pblock.py:93-154): a complex128 state in
 * CUDA managed memory (svb_managed_alloc) wrapped by a handle that does not
 * own it (svb_create_view).  Calls on the view run on the device in place;
 * the host sees the result after the call returns (every call synchronises). */
int svb_managed_alloc(uint64_t bytes, int device, void** out);
int svb_managed_free(void* p);
int svb_create_view(int n_qubits, int device, void* amps, svb_handle* out);

/* Host <-> device amplitudes (final_state, statevector.py:259-274; and the
 * kernel-level numpy-array API used by pblock.py:93-154, calibration.py:215-228). */
int svb_set_amplitudes(svb_handle h, const double* host, uint64_t offset, uint64_t count);
int svb_get_amplitudes(svb_handle h, double* host, uint64_t offset, uint64_t count);

/* Gate program: apply_1q / apply_2q / apply_instruction over a whole circuit
 * (statevector.py:33-122, 210-212).  The program is fused and scheduled into
 * HBM passes natively; the result equals applying the gates
 * one by one in order. */
int svb_apply(svb_handle h, const svb_gate* gates, int n_gates);
/* Apply a gate program and return out[j] = <Z_{z_qubits[j]}> of the resulting
 * state (single-qubit Z; statevector.py:277-292 per qubit, after
 * statevector.py:116-122 for every gate).  The sums are accumulated by the
 * program's last fused pass as it stores the state, so no separate read pass
 * is needed; unfused programs fall back to one reduction pass.  nz may be 0.
 * z_qubits[j] = -1 returns sum |a|^2 (the norm: a shard's share of the <Z> of
 * a qubit held in the rank bits). */
int svb_apply_z(svb_handle h, const svb_gate* gates, int n_gates, const int32_t* z_qubits, int nz,
                double* out);

/* One dense 2^k x 2^k block (a fused k-qubit gate; apply_2q's dense path,
 * statevector.py:105-113, generalised to k <= 6) in one HBM pass.  mat is
 * row-major complex128 (re, im); local index bit i <-> qubits[i].  engine:
 *   SVB_ENGINE_AUTO   tensor cores (tcgen05 kind::tf32, 3xTF32 split) for
 *                     complex64 and k >= SVB_OPT_TC_MIN_K, else CUDA cores;
 *   SVB_ENGINE_TENSOR tensor cores (complex64, 3 <= k <= 6), else SVB_E_ARG;
 *   SVB_ENGINE_FMA    CUDA cores (k <= 6 complex64, k <= 5 complex128).
 * Needs n >= k + 7.  svb_last_engine reports which engine ran. */
typedef enum { SVB_ENGINE_AUTO = 0, SVB_ENGINE_TENSOR = 1, SVB_ENGINE_FMA = 2 } svb_engine;
int svb_apply_matrix(svb_handle h, const int32_t* qubits, int k, const double* mat, int engine);
int svb_last_engine(svb_handle h);

/* Reduced |amp|^2 over ascending `qubits` (marginal_probs, statevector.py:131-139). */
int svb_marginal_probs(svb_handle h, const int32_t* qubits, int k, double* out);

/* <Z_mask> for M masks in one pass over the state (expectation, statevector.py:277-292). */
int svb_expect_z(svb_handle h, const uint64_t* masks, int m, double* out);

/* Distance and overlap of two states of the same size on the same device
 * (either precision): out[5] = {sum|a-b|^2, sum|a|^2, sum|b|^2, Re<a|b>,
 * Im<a|b>}.  State fidelity |<a|b>|^2 as in metrics.mirror_fidelity
 * (metrics.py:33-56), and the device-side parity check of large states. */
int svb_compare(svb_handle a, svb_handle b, double* out);

/* Terminal sampling (statevector.py:213-216 + result.py:50-82 + sampling.py:30-83).
 *   qubits[k]      ascending measured qubits;
 *   bit_src[w]     for output bit p (clbit rank p): bit index into the marginal index;
 *   pcg[4]         numpy PCG64 (state_hi, state_lo, inc_hi, inc_lo) of default_rng(seed);
 *   out_codes/out_counts: capacity >= min(shots, 2^w); sorted ascending like np.unique. */
int svb_sample(svb_handle h, const int32_t* qubits, int k, const int32_t* bit_src, int w,
               uint64_t shots, const uint64_t* pcg, int sampler, uint64_t* out_codes,
               uint64_t* out_counts, uint64_t* n_unique);

/* AliasTable.from_probs (sampling.py:30-70) on the device for a given
 * probability vector: the table the ALIAS sampler draws from.  Errors:
 * SVB_E_SAMPLING for an invalid vector (sampling.py:31-40). */
int svb_alias_table(int device, const double* probs, uint64_t m, double* prob_row, int64_t* alias_row);

/* AliasTable.from_probs(probs).sample_indices(rng, shots) (sampling.py:30-83):
 * table build and draws on the device from the numpy PCG64 state pcg[4];
 * m must be a power of two (a marginal).  out_idx[shots]: outcome indices. */
int svb_alias_draw(int device, const double* probs, uint64_t m, uint64_t shots, const uint64_t* pcg,
                   uint64_t* out_idx);

/* AliasTable.sample_indices(rng, shots) (sampling.py:78-83) for a table
 * already built (prob_row/alias_row as svb_alias_table returns; any m): the
 * next `shots` doubles of the numpy PCG64 state pcg[4], one per draw. */
int svb_alias_sample(int device, const double* prob_row, const int64_t* alias_row, uint64_t m, uint64_t shots,
                     const uint64_t* pcg, uint64_t* out_idx);
/* The same draws from a device-resident table (uploaded once): handle from
 * svb_alias_upload, freed by svb_alias_release.  sampling.py:72-77 */
int svb_alias_upload(int device, const double* prob_row, const int64_t* alias_row, uint64_t m, void** out_table);
int svb_alias_sample_table(void* table, uint64_t shots, const uint64_t* pcg, uint64_t* out_idx);
int svb_alias_release(void* table);

/* Sharded mode (global<->local qubit swaps, svb_dist in sharded.py):
 * raw device pointer of the state (synchronised), and gather/scatter of the
 * half whose bit L == bit to/from a contiguous device buffer of 2^(n-1)
 * amplitudes (to_buf = 1: state -> buffer). */
int svb_device_ptr(svb_handle h, void** ptr, uint64_t* bytes, int64_t* stream);
int svb_half_copy(svb_handle h, int L, int bit, void* dev_buf, int to_buf);
int svb_clear(svb_handle h); /* all amplitudes 0 (a shard that holds no part of |0..0>) */
/* Grouped remap of g global qubits (sharded.py): block `block` of the shard
 * = the amplitudes whose local bits lbits[0..g) (ascending) equal block's
 * bits; copy its elements [offset, offset + count) to (to_buf = 1) or from
 * a contiguous device buffer of count amplitudes.  sync = 0 leaves the copy
 * queued on the handle's stream (svb_sync before the buffer is read). */
int svb_block_copy(svb_handle h, const int32_t* lbits, int g, uint64_t block, uint64_t offset, uint64_t count,
                   void* dev_buf, int to_buf, int sync);
/* Distributed terminal sampling: the shots of the shared PCG64 stream whose
 * global CDF target u*total falls in [lo, hi) are drawn from this shard;
 * bit_src[p] = local bit of output bit p or -1 (then taken from code_or). */
int svb_sample_slice(svb_handle h, uint64_t shots, const uint64_t* pcg, double lo, double hi, double total,
                     const int32_t* bit_src, int w, uint64_t code_or, uint64_t* out_codes, uint64_t* out_counts,
                     uint64_t* n_unique);

/* Batched terminal circuits that fit in shared memory (n <= 12 complex128,
 * n <= 13 complex64): one persistent kernel, state per CTA in shared memory,
 * CDF sampling from each circuit's PCG64 stream (replaces the sequential
 * batch.run_batch loop, batch.py:104-222, for small circuits).  Circuit i:
 * nq[i] qubits, gates[gate_off[i] .. +ngates[i]), pcg[4i..4i+3], w[i] output
 * bits with sources bit_src[64i + p]; codes to out_codes[shots*i + s]. */
int svb_batch_small(int device, int precision, int ncirc, const int32_t* nq, const int32_t* gate_off,
                    const int32_t* ngates, const svb_gate* gates, int total_gates, const uint64_t* pcg,
                    const int32_t* w, const int8_t* bit_src, uint64_t shots, uint64_t* out_codes);

/* Batched terminal circuits of any size (5 <= n <= 36; config 4's 13-24
 * qubit circuits): one call for the whole batch.  `nthreads` host workers,
 * each with its own stream and state buffer, run each circuit's fused program
 * from |0...0> and draw `shots` CDF samples from its PCG64 stream pcg[4i..];
 * bit_src[64i + p] is the state-index bit of output bit p; codes to
 * out_codes[shots*i + s] (one device->host copy at the end).  Per-circuit
 * errors land in status[i] (svb_status); the call itself fails only on
 * bad arguments or a device error outside a circuit.  jit_mode: 0 =
 * interpreter kernels up to 24 qubits (no NVRTC compile; deterministic),
 * 1 = NVRTC-specialised passes from 24 qubits, compiled synchronously (same
 * engine and results as svb_apply), 2 = as 1 but compiled in the background
 * while the interpreter serves (fastest once warm, engine per circuit depends
 * on timing). */
int svb_batch_run(int device, int precision, int ncirc, const int32_t* nq, const int32_t* gate_off,
                  const int32_t* ngates, const svb_gate_op* ops, const svb_gate* fixed, int nfixed,
                  int total_gates, const uint64_t* pcg,
                  const int32_t* w, const int8_t* bit_src, uint64_t shots, int nthreads, int jit_mode,
                  uint64_t* out_codes, int32_t* status);

/* Mid-circuit replay (statevector.py:142-179).  The PCG64 stream lives on the
 * device; each measure/reset consumes one draw, exactly as rng.random(). */
/* Partitioned-block support (pblock.py:34-43,76-120): the block merge
   np.multiply.outer(b, a) into dst (a.n + b.n qubits), a qubit reorder
   (qubit p -> bit dest[p], reorder_qubits), and the kept half of a measured
   block (state.reshape(-1, 2, 2^q)[:, bit, :]) into dst (src.n - 1 qubits). */
int svb_outer(svb_handle dst, svb_handle a, svb_handle b);
int svb_permute_qubits(svb_handle h, const int32_t* dest);
int svb_select_half(svb_handle dst, svb_handle src, int qubit, int bit);
int svb_rng_seed(svb_handle h, const uint64_t* pcg);
int svb_measure(svb_handle h, int qubit, int32_t* outcome);      /* _measure_qubit */
int svb_reset(svb_handle h, int qubit);                          /* _reset_qubit   */

/* Whole-shot replay of a suffix program on device: for each shot, copy
 * `prefix`, run ops, record clbits.  ops: kind 0 = gate (index into gates),
 * 1 = measure (qubit, clbit), 2 = reset (qubit).  out_codes[s] = packed clbits
 * (bit p = clbit rank p), computed with the device PCG64 stream seeded by pcg. */
int svb_replay(svb_handle work, svb_handle prefix, const int32_t* ops, int n_ops,
               const svb_gate* gates, const int32_t* clbit_rank, uint64_t shots,
               const uint64_t* pcg, uint64_t* out_codes);

/* Host-only helpers (no GPU): schedule statistics of a gate program, and CPU
 * emulation of the fused program with the same scheduler and op interpreter
 * as the device kernel (complex128 amps in/out).  Test/diagnostic hooks.
 * svb_plan: precision | 0x100 schedules for a lazy |0...0> input; *has_perm =
 * 0 (no permutation), 1 (separate final permutation pass), 2 (fused into the
 * last pass's store), 3 (the input is permuted first into the layout that
 * absorbs the swap relabeling), 4 (that permutation fused into the first
 * pass's loads).  svb_emulate_apply: relabel_swaps 0 = swaps as ops,
 * 1 = relabeling + final permutation, 2 = relabeling for a |0...0> input. */
int svb_plan(int n, int precision, const svb_gate* gates, int n_gates, int64_t* n_passes,
             int64_t* n_rounds, int64_t* op_bytes, int32_t* has_perm);
int svb_emulate_apply(int n, int precision, const svb_gate* gates, int n_gates, double* amps,
                      int relabel_swaps);
/* Generate and NVRTC-compile the specialised pass kernels of a program (no
 * GPU needed); cubin size out, compiler log into log[log_cap]. */
int svb_jit_check(int n, int precision, const svb_gate* gates, int n_gates, int64_t* cubin_bytes, char* log,
                  int log_cap);

/* All shots of the mid-circuit replay in one launch for states that fit in
 * shared memory (n <= 12 complex128 / 13 complex64); same op encoding and
 * draw order as svb_replay (shot s uses draws [s*M, (s+1)*M)).  prefix is the
 * complex128 prefix state on the host; ops[3k] as in svb_replay with the
 * clbit operand already mapped to its output bit rank. */
int svb_replay_small(int device, int precision, int n, const double* prefix_c128, const int32_t* ops, int n_ops,
                     const svb_gate* gates, int n_gates, uint64_t shots, const uint64_t* pcg,
                     uint64_t* out_codes);

#ifdef __cplusplus
}
#endif
#endif /* SVB_H */
