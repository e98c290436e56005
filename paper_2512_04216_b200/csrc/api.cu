// libsvb C ABI (include/svb.h): handle lifetime, host<->device transfers and
// the dispatch of gate programs, reductions and samplers to the kernels.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "common.cuh"
#include "kernels.h"
#include "program.h"

using namespace svb;

struct svb_state {
  int n = 0, prec = SVB_C128, device = 0;
  void* amps = nullptr;
  void* spare = nullptr;  // second state buffer for out-of-place permutation passes
  cudaStream_t st = nullptr;
  uint64_t* d_rng = nullptr;     // PCG64 (state_hi, state_lo, inc_hi, inc_lo)
  int32_t* d_outcome = nullptr;  // last measure outcome
  double* d_ws = nullptr;        // reduction scratch
  size_t ws_doubles = 0;
  int fusion = 1, max_high = -1;
  bool zero_pending = false;  // |0...0> not yet written: the next fused pass synthesises it
  int jit_min_n = kDefaultJitMinQubits;  // NVRTC-specialised passes from this many qubits up (-1: never)
  int tc_min_k = 5;    // svb_apply_matrix: tensor cores for dense blocks of >= this many qubits (complex64)
  int last_engine = 0;
  void* external = nullptr;  // svb_create_view: caller-owned amplitudes (never freed, always current)
  ProgramStats stats{};
  Profiler prof;
  cudaEvent_t t0 = nullptr, t1 = nullptr;
  size_t amp_bytes() const { return (size_t)(prec == SVB_C128 ? 16 : 8) << n; }
};

static thread_local std::string g_err;
namespace svb {
void set_last_error(const char* msg) { g_err = msg; }
}  // namespace svb

template <class F> static int guard(F&& f) {
  try {
    f();
    return SVB_OK;
  } catch (const Error& e) {
    g_err = e.what();
    return e.code;
  } catch (const std::exception& e) {
    g_err = e.what();
    return SVB_E_CUDA;
  }
}

static void check_handle_nomat(svb_handle h) {
  require(h != nullptr && h->amps != nullptr, SVB_E_ARG, "invalid svb handle");
  SVB_CUDA(cudaSetDevice(h->device));
}

// Write a pending lazy |0...0> before anything reads or partially writes the state.
static void materialize(svb_handle h) {
  if (!h->zero_pending) return;
  if (h->prec == SVB_C128) launch_zero<double>(h->amps, h->n, h->st);
  else launch_zero<float>(h->amps, h->n, h->st);
  h->zero_pending = false;
}

static void check_handle(svb_handle h) {
  check_handle_nomat(h);
  materialize(h);
}

// A view's amplitudes must stay in the caller's buffer: when a program ended
// with an out-of-place permutation into the spare buffer, copy back.
static void restore_view(svb_handle h) {
  if (!h->external || h->amps == h->external) return;
  SVB_CUDA(cudaMemcpyAsync(h->external, h->amps, h->amp_bytes(), cudaMemcpyDeviceToDevice, h->st));
  h->spare = h->amps;
  h->amps = h->external;
}

static void ensure_ws(svb_handle h, size_t doubles) {
  if (doubles <= h->ws_doubles) return;
  if (h->d_ws) SVB_CUDA(cudaFreeAsync(h->d_ws, h->st));
  h->d_ws = nullptr;
  h->ws_doubles = 0;
  SVB_CUDA(cudaMallocAsync(&h->d_ws, doubles * sizeof(double), h->st));
  h->ws_doubles = doubles;
}

// complex128 <-> complex64 conversion through a device staging buffer
__global__ void k_c128_to_c64(const double2* __restrict__ in, float2* __restrict__ out, uint64_t n) {
  uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    out[i] = make_float2((float)in[i].x, (float)in[i].y);
}
__global__ void k_c64_to_c128(const float2* __restrict__ in, double2* __restrict__ out, uint64_t n) {
  uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    out[i] = make_double2((double)in[i].x, (double)in[i].y);
}

extern "C" {

const char* svb_last_error(void) { return g_err.c_str(); }
int svb_version(void) { return 1; }

int svb_max_qubits(int device, int precision, int* out_n) {
  return guard([&] {
    SVB_CUDA(cudaSetDevice(device));
    size_t fr = 0, tot = 0;
    SVB_CUDA(cudaMemGetInfo(&fr, &tot));
    size_t s = precision == SVB_C128 ? 16 : 8;
    int n = 1;
    while (n < 40 && ((s << (n + 1)) + (s << (n + 1)) / 8) < fr) ++n;
    *out_n = n;
  });
}

int svb_host_alloc(uint64_t bytes, void** out) {
  return guard([&] { SVB_CUDA(cudaHostAlloc(out, bytes, cudaHostAllocPortable)); });
}
int svb_host_free(void* p) {
  return guard([&] { SVB_CUDA(cudaFreeHost(p)); });
}

int svb_create(int n_qubits, int precision, int device, svb_handle* out) {
  svb_state* h = nullptr;
  int rc = guard([&] {
    require(n_qubits >= 1 && n_qubits <= 40, SVB_E_ARG, "n_qubits out of range");
    require(precision == SVB_C64 || precision == SVB_C128, SVB_E_ARG, "bad precision");
    SVB_CUDA(cudaSetDevice(device));
    {
      // small per-call scratch (program upload, reduction workspaces) comes from
      // the stream-ordered pool; keep its memory mapped across synchronisations
      cudaMemPool_t pool;
      if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
        uint64_t keep = 1ull << 30;  // (unbounded measured slower for the 2 GiB sampler scratch)
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
      }
      cudaGetLastError();
    }
    h = new svb_state();
    h->n = n_qubits;
    h->prec = precision;
    h->device = device;
    SVB_CUDA(cudaStreamCreateWithFlags(&h->st, cudaStreamNonBlocking));
    cudaError_t e = state_malloc(&h->amps, h->amp_bytes());
    if (e != cudaSuccess) {
      cudaGetLastError();
      h->amps = nullptr;
      throw Error(SVB_E_OOM, "cannot allocate " + std::to_string(h->amp_bytes()) +
                                 " bytes for a " + std::to_string(n_qubits) + "-qubit state");
    }
    SVB_CUDA(cudaMalloc(&h->d_rng, 4 * sizeof(uint64_t) + 16));
    h->d_outcome = reinterpret_cast<int32_t*>(h->d_rng + 4);
    h->zero_pending = true;  // |0...0>, written lazily (see materialize)
  });
  if (rc != SVB_OK) {
    if (h) {
      if (h->amps) cudaFree(h->amps);
      if (h->st) cudaStreamDestroy(h->st);
      delete h;
    }
    *out = nullptr;
    return rc;
  }
  *out = h;
  return SVB_OK;
}

// Managed (unified) memory for the kernel-level numpy API: zero_state()
// returns an array in this memory, so apply_1q / apply_2q / marginal_probs on
// it run on the device with no host<->device copy (pages migrate on demand
// and stay in HBM while only kernels touch them).
int svb_managed_alloc(uint64_t bytes, int device, void** out) {
  return guard([&] {
    SVB_CUDA(cudaSetDevice(device));
    SVB_CUDA(cudaMallocManaged(out, bytes, cudaMemAttachGlobal));
    cudaMemLocation loc{};
    loc.type = cudaMemLocationTypeDevice;
    loc.id = device;
    cudaMemAdvise(*out, bytes, cudaMemAdviseSetPreferredLocation, loc);
    cudaGetLastError();
  });
}
int svb_managed_free(void* p) {
  return guard([&] { SVB_CUDA(cudaFree(p)); });
}

int svb_create_view(int n_qubits, int device, void* amps, svb_handle* out) {
  svb_state* h = nullptr;
  int rc = guard([&] {
    require(n_qubits >= 1 && n_qubits <= 40 && amps != nullptr, SVB_E_ARG, "bad view");
    SVB_CUDA(cudaSetDevice(device));
    h = new svb_state();
    h->n = n_qubits;
    h->prec = SVB_C128;
    h->device = device;
    h->amps = amps;
    h->external = amps;
    SVB_CUDA(cudaStreamCreateWithFlags(&h->st, cudaStreamNonBlocking));
    SVB_CUDA(cudaMalloc(&h->d_rng, 4 * sizeof(uint64_t) + 16));
    h->d_outcome = reinterpret_cast<int32_t*>(h->d_rng + 4);
  });
  if (rc != SVB_OK) {
    if (h) {
      if (h->st) cudaStreamDestroy(h->st);
      delete h;
    }
    *out = nullptr;
    return rc;
  }
  *out = h;
  return SVB_OK;
}

int svb_destroy(svb_handle h) {
  if (!h) return SVB_OK;
  return guard([&] {
    SVB_CUDA(cudaSetDevice(h->device));
    SVB_CUDA(cudaStreamSynchronize(h->st));
    if (h->d_ws) cudaFreeAsync(h->d_ws, h->st);
    SVB_CUDA(cudaStreamSynchronize(h->st));
    if (h->amps != h->external) cudaFree(h->amps);
    if (h->spare && h->spare != h->external) cudaFree(h->spare);
    cudaFree(h->d_rng);
    if (h->t0) cudaEventDestroy(h->t0);
    if (h->t1) cudaEventDestroy(h->t1);
    cudaStreamDestroy(h->st);
    delete h;
  });
}

int svb_n_qubits(svb_handle h) { return h ? h->n : -1; }

int svb_sync(svb_handle h) {
  return guard([&] {
    check_handle(h);
    SVB_CUDA(cudaStreamSynchronize(h->st));
  });
}

int svb_set_option(svb_handle h, int option, int value) {
  return guard([&] {
    check_handle(h);
    if (option == SVB_OPT_FUSION) h->fusion = value;
    else if (option == SVB_OPT_MAX_HIGH) h->max_high = value;
    else if (option == SVB_OPT_JIT_MIN_N) h->jit_min_n = value;
    else if (option == SVB_OPT_TC_MIN_K) h->tc_min_k = value;
    else throw Error(SVB_E_ARG, "unknown option");
  });
}

int svb_last_stats(svb_handle h, int64_t* n_passes, int64_t* n_gates, int64_t* n_launches) {
  return guard([&] {
    check_handle(h);
    *n_passes = h->stats.passes;
    *n_gates = h->stats.gates;
    *n_launches = h->stats.launches;
  });
}

int svb_set_zero(svb_handle h) {
  return guard([&] {
    check_handle_nomat(h);
    h->zero_pending = true;  // lazy: written by the first consumer (or synthesised by the next pass)
    if (h->external) {       // a view is read by the host directly: write it now
      materialize(h);
      SVB_CUDA(cudaStreamSynchronize(h->st));
    }
  });
}

int svb_copy_state(svb_handle dst, svb_handle src) {
  return guard([&] {
    check_handle(dst);
    check_handle(src);
    require(dst->n == src->n && dst->prec == src->prec, SVB_E_ARG, "state shape mismatch");
    SVB_CUDA(cudaStreamSynchronize(src->st));
    SVB_CUDA(cudaMemcpyAsync(dst->amps, src->amps, src->amp_bytes(), cudaMemcpyDeviceToDevice, dst->st));
    SVB_CUDA(cudaStreamSynchronize(dst->st));
  });
}

static constexpr uint64_t kStage = 1ull << 24;  // amplitudes per c64 conversion chunk

int svb_set_amplitudes(svb_handle h, const double* host, uint64_t offset, uint64_t count) {
  return guard([&] {
    check_handle(h);
    uint64_t len = 1ull << h->n;
    require(offset <= len && count <= len - offset, SVB_E_ARG, "amplitude range out of bounds");
    if (h->prec == SVB_C128) {
      SVB_CUDA(cudaMemcpyAsync(static_cast<double2*>(h->amps) + offset, host, count * 16,
                               cudaMemcpyHostToDevice, h->st));
    } else {
      double2* stage = nullptr;
      uint64_t chunk = std::min(count, kStage);
      SVB_CUDA(cudaMallocAsync(&stage, std::max<uint64_t>(chunk, 1) * 16, h->st));
      for (uint64_t done = 0; done < count; done += chunk) {
        uint64_t c = std::min(chunk, count - done);
        SVB_CUDA(cudaMemcpyAsync(stage, host + 2 * done, c * 16, cudaMemcpyHostToDevice, h->st));
        k_c128_to_c64<<<grid_for(c, 256), 256, 0, h->st>>>(stage, static_cast<float2*>(h->amps) + offset + done, c);
        SVB_CHECK_LAUNCH();
      }
      SVB_CUDA(cudaFreeAsync(stage, h->st));
    }
    SVB_CUDA(cudaStreamSynchronize(h->st));
  });
}

int svb_get_amplitudes(svb_handle h, double* host, uint64_t offset, uint64_t count) {
  return guard([&] {
    check_handle(h);
    uint64_t len = 1ull << h->n;
    require(offset <= len && count <= len - offset, SVB_E_ARG, "amplitude range out of bounds");
    if (h->prec == SVB_C128) {
      SVB_CUDA(cudaMemcpyAsync(host, static_cast<double2*>(h->amps) + offset, count * 16,
                               cudaMemcpyDeviceToHost, h->st));
    } else {
      double2* stage = nullptr;
      uint64_t chunk = std::min(count, kStage);
      SVB_CUDA(cudaMallocAsync(&stage, std::max<uint64_t>(chunk, 1) * 16, h->st));
      for (uint64_t done = 0; done < count; done += chunk) {
        uint64_t c = std::min(chunk, count - done);
        k_c64_to_c128<<<grid_for(c, 256), 256, 0, h->st>>>(static_cast<float2*>(h->amps) + offset + done, stage, c);
        SVB_CHECK_LAUNCH();
        SVB_CUDA(cudaMemcpyAsync(host + 2 * done, stage, c * 16, cudaMemcpyDeviceToHost, h->st));
      }
      SVB_CUDA(cudaFreeAsync(stage, h->st));
    }
    SVB_CUDA(cudaStreamSynchronize(h->st));
  });
}

static void validate_gates(svb_handle h, const svb_gate* g, int ng) {
  require(ng >= 0 && (ng == 0 || g != nullptr), SVB_E_ARG, "bad gate list");
  for (int i = 0; i < ng; ++i) {
    require(g[i].k == 1 || g[i].k == 2, SVB_E_ARG, "gate arity must be 1 or 2");
    for (int j = 0; j < g[i].k; ++j)
      require(g[i].qubits[j] >= 0 && g[i].qubits[j] < h->n, SVB_E_ARG, "gate qubit out of range");
    require(g[i].k == 1 || g[i].qubits[0] != g[i].qubits[1], SVB_E_ARG, "gate repeats a qubit");
  }
}

int svb_apply(svb_handle h, const svb_gate* gates, int n_gates) {
  return guard([&] {
    auto t0 = std::chrono::steady_clock::now();
    check_handle_nomat(h);
    validate_gates(h, gates, n_gates);
    h->stats = ProgramStats{};
    h->stats.prof = &h->prof;
    if (h->prec == SVB_C128)
      run_program_owned<double>(&h->amps, &h->spare, h->n, gates, n_gates, h->fusion, h->jit_min_n, h->st, &h->stats, &h->zero_pending);
    else
      run_program_owned<float>(&h->amps, &h->spare, h->n, gates, n_gates, h->fusion, h->jit_min_n, h->st, &h->stats, &h->zero_pending);
    restore_view(h);
    auto t1 = std::chrono::steady_clock::now();
    SVB_CUDA(cudaStreamSynchronize(h->st));
    if (h->prof.on) h->prof.collect();
    if (std::getenv("SVB_TRACE")) {
      auto t2 = std::chrono::steady_clock::now();
      std::fprintf(stderr, "[svb] apply host=%.2fms sync=%.2fms\n",
                   std::chrono::duration<double, std::milli>(t1 - t0).count(),
                   std::chrono::duration<double, std::milli>(t2 - t1).count());
    }
  });
}

// Apply a gate program and return <Z_q> for single qubits q (after the
// program).  The sums are accumulated by the program's last fused pass while it
// stores the state (no separate read pass); programs that are not fused fall
// back to one multi-mask reduction pass.  statevector.py:277-292 per qubit.
int svb_apply_z(svb_handle h, const svb_gate* gates, int n_gates, const int32_t* z_qubits, int nz, double* out) {
  return guard([&] {
    check_handle_nomat(h);
    validate_gates(h, gates, n_gates);
    require(nz >= 0, SVB_E_ARG, "bad qubit count");
    // qubit -1: sum p (the norm; a shard's share of a global qubit's <Z>)
    for (int j = 0; j < nz; ++j) require(z_qubits[j] >= -1 && z_qubits[j] < h->n, SVB_E_ARG, "qubit out of range");
    h->stats = ProgramStats{};
    h->stats.prof = &h->prof;
    const size_t zacc = std::max({zacc_doubles(kPassThreads<float, 4>, 4), zacc_doubles(kPassThreads<float, 5>, 5),
                                  zacc_doubles(kPassThreads<double, 4>, 4)});
    ensure_ws(h, zacc + kZaccRows + (size_t)kZaccRows * 32 + expect_ws_doubles(h->n, nz > 0 ? nz : 1) + 64);
    ZRequest z;
    z.want = nz > 0;
    z.d_acc = h->d_ws;
    z.d_out = h->d_ws + zacc;
    if (h->prec == SVB_C128)
      run_program_owned<double>(&h->amps, &h->spare, h->n, gates, n_gates, h->fusion, h->jit_min_n, h->st, &h->stats,
                                &h->zero_pending, &z);
    else
      run_program_owned<float>(&h->amps, &h->spare, h->n, gates, n_gates, h->fusion, h->jit_min_n, h->st, &h->stats,
                               &h->zero_pending, &z);
    restore_view(h);
    if (nz == 0) {
      SVB_CUDA(cudaStreamSynchronize(h->st));
      if (h->prof.on) h->prof.collect();
      return;
    }
    if (z.fused) {
      std::vector<double> vals(z.logical.size());
      SVB_CUDA(cudaMemcpyAsync(vals.data(), z.d_out, vals.size() * sizeof(double), cudaMemcpyDeviceToHost, h->st));
      SVB_CUDA(cudaStreamSynchronize(h->st));
      std::vector<double> by_q(h->n, 0.0);
      std::vector<int> seen(h->n, 0);
      for (size_t k = 0; k < z.logical.size(); ++k)
        if (z.logical[k] >= 0) { by_q[z.logical[k]] = vals[k]; seen[z.logical[k]] = 1; }
      // a qubit outside the passes' support (zero_start) is |0> in every
      // amplitude that is not zero: <Z> = sum p
      for (int j = 0; j < nz; ++j) out[j] = (z_qubits[j] >= 0 && seen[z_qubits[j]]) ? by_q[z_qubits[j]] : vals.back();
    } else {
      materialize(h);
      std::vector<uint64_t> masks(nz);
      for (int j = 0; j < nz; ++j) masks[j] = z_qubits[j] >= 0 ? 1ull << z_qubits[j] : 0ull;
      double* d_out = z.d_out;
      double* d_ws = z.d_out + kZaccRows + (size_t)kZaccRows * 32;
      if (h->prec == SVB_C128) launch_expect_z<double>(h->amps, h->n, masks.data(), nz, d_out, d_ws, h->st);
      else launch_expect_z<float>(h->amps, h->n, masks.data(), nz, d_out, d_ws, h->st);
      SVB_CUDA(cudaMemcpyAsync(out, d_out, nz * sizeof(double), cudaMemcpyDeviceToHost, h->st));
      SVB_CUDA(cudaStreamSynchronize(h->st));
    }
    if (h->prof.on) h->prof.collect();
  });
}

int svb_profile(svb_handle h, int enable) {
  return guard([&] {
    check_handle_nomat(h);  // timing/profiling never materialises a lazy |0...0>
    h->prof.on = enable != 0;
    h->prof.ms[0] = h->prof.ms[1] = 0;
    h->prof.count[0] = h->prof.count[1] = 0;
    h->prof.bytes[0] = h->prof.bytes[1] = 0;
    h->prof.idx_ms.clear();
    h->prof.idx_bytes.clear();
    h->prof.idx_count.clear();
  });
}

int svb_profile_read(svb_handle h, double* out) {
  return guard([&] {
    check_handle_nomat(h);  // timing/profiling never materialises a lazy |0...0>
    out[0] = h->prof.ms[0];
    out[1] = (double)h->prof.count[0];
    out[2] = h->prof.bytes[0];
    out[3] = h->prof.ms[1];
    out[4] = (double)h->prof.count[1];
    out[5] = h->prof.bytes[1];
  });
}

// Per pass index of the applied programs since profiling was enabled:
// out[3*i + {0,1,2}] = (ms, HBM bytes, launches); returns the count in *n.
int svb_profile_passes(svb_handle h, double* out, int cap, int* n) {
  return guard([&] {
    check_handle_nomat(h);  // timing/profiling never materialises a lazy |0...0>
    const int k = (int)h->prof.idx_ms.size();
    *n = k;
    for (int i = 0; i < k && i < cap; ++i) {
      out[3 * i] = h->prof.idx_ms[i];
      out[3 * i + 1] = h->prof.idx_bytes[i];
      out[3 * i + 2] = (double)h->prof.idx_count[i];
    }
  });
}

int svb_timer_start(svb_handle h) {
  return guard([&] {
    check_handle_nomat(h);  // timing/profiling never materialises a lazy |0...0>
    if (!h->t0) {
      SVB_CUDA(cudaEventCreate(&h->t0));
      SVB_CUDA(cudaEventCreate(&h->t1));
    }
    SVB_CUDA(cudaEventRecord(h->t0, h->st));
  });
}

int svb_timer_stop(svb_handle h, double* ms) {
  return guard([&] {
    check_handle_nomat(h);  // timing/profiling never materialises a lazy |0...0>
    require(h->t0 != nullptr, SVB_E_ARG, "timer not started");
    SVB_CUDA(cudaEventRecord(h->t1, h->st));
    SVB_CUDA(cudaEventSynchronize(h->t1));
    float t = 0.f;
    SVB_CUDA(cudaEventElapsedTime(&t, h->t0, h->t1));
    *ms = t;
  });
}

int svb_marginal_probs(svb_handle h, const int32_t* qubits, int k, double* out) {
  return guard([&] {
    check_handle(h);
    require(k >= 1 && k <= h->n, SVB_E_ARG, "bad qubit count");
    for (int j = 0; j < k; ++j) {
      require(qubits[j] >= 0 && qubits[j] < h->n, SVB_E_ARG, "qubit out of range");
      require(j == 0 || qubits[j] > qubits[j - 1], SVB_E_ARG, "qubits must be ascending");
    }
    uint64_t m = 1ull << k;
    double* d_out = nullptr;
    SVB_CUDA(cudaMallocAsync(&d_out, m * sizeof(double), h->st));
    size_t wsd = marginal_ws_doubles(h->n, k);
    ensure_ws(h, wsd + 1);
    if (h->prec == SVB_C128) launch_marginal<double>(h->amps, h->n, qubits, k, d_out, h->d_ws, h->ws_doubles, h->st);
    else launch_marginal<float>(h->amps, h->n, qubits, k, d_out, h->d_ws, h->ws_doubles, h->st);
    SVB_CUDA(cudaMemcpyAsync(out, d_out, m * sizeof(double), cudaMemcpyDeviceToHost, h->st));
    SVB_CUDA(cudaFreeAsync(d_out, h->st));
    SVB_CUDA(cudaStreamSynchronize(h->st));
  });
}

int svb_expect_z(svb_handle h, const uint64_t* masks, int m, double* out) {
  return guard([&] {
    check_handle(h);
    require(m >= 0, SVB_E_ARG, "bad mask count");
    if (m == 0) return;
    uint64_t full = (1ull << h->n) - 1;
    for (int j = 0; j < m; ++j) require((masks[j] & ~full) == 0, SVB_E_ARG, "mask names a qubit out of range");
    ensure_ws(h, expect_ws_doubles(h->n, m) + 64);
    double* d_out = nullptr;
    SVB_CUDA(cudaMallocAsync(&d_out, m * sizeof(double), h->st));
    if (h->prec == SVB_C128) launch_expect_z<double>(h->amps, h->n, masks, m, d_out, h->d_ws, h->st);
    else launch_expect_z<float>(h->amps, h->n, masks, m, d_out, h->d_ws, h->st);
    SVB_CUDA(cudaMemcpyAsync(out, d_out, m * sizeof(double), cudaMemcpyDeviceToHost, h->st));
    SVB_CUDA(cudaFreeAsync(d_out, h->st));
    SVB_CUDA(cudaStreamSynchronize(h->st));
  });
}

int svb_apply_matrix(svb_handle h, const int32_t* qubits, int k, const double* mat, int engine) {
  return guard([&] {
    check_handle(h);
    require(k >= 1 && k <= 6 && qubits != nullptr && mat != nullptr, SVB_E_ARG, "bad dense block");
    for (int i = 0; i < k; ++i) {
      require(qubits[i] >= 0 && qubits[i] < h->n, SVB_E_ARG, "block qubit out of range");
      for (int j = 0; j < i; ++j) require(qubits[i] != qubits[j], SVB_E_ARG, "block repeats a qubit");
    }
    const bool tc = dense_tc_supported(h->prec, h->n, k);
    require(engine != SVB_ENGINE_TENSOR || tc, SVB_E_ARG,
            "tensor-core engine needs complex64, 3 <= k <= 6 and n >= k + 7");
    const bool use_tc = engine == SVB_ENGINE_TENSOR || (engine == SVB_ENGINE_AUTO && tc && k >= h->tc_min_k);
    Profiler* pf = h->prof.on ? &h->prof : nullptr;
    if (pf) pf->begin(h->st, 0, 2.0 * (double)h->amp_bytes(), 0);
    if (use_tc) launch_dense_tc(h->amps, h->n, qubits, k, mat, h->st);
    else if (h->prec == SVB_C128) launch_dense_fma<double>(h->amps, h->n, qubits, k, mat, h->st);
    else launch_dense_fma<float>(h->amps, h->n, qubits, k, mat, h->st);
    if (pf) pf->end(h->st);
    h->stats = ProgramStats{};
    h->stats.passes = 1;
    h->stats.launches = 1;
    h->stats.gates = 1;
    h->last_engine = use_tc ? SVB_ENGINE_TENSOR : SVB_ENGINE_FMA;
    SVB_CUDA(cudaStreamSynchronize(h->st));
  });
}

int svb_last_engine(svb_handle h) { return h ? h->last_engine : -1; }

int svb_compare(svb_handle a, svb_handle b, double* out) {
  return guard([&] {
    check_handle(b);
    check_handle(a);
    require(a->n == b->n && a->device == b->device, SVB_E_ARG, "states differ in size or device");
    SVB_CUDA(cudaStreamSynchronize(b->st));
    ensure_ws(a, compare_ws_doubles(a->n));
    double* d_out = nullptr;
    SVB_CUDA(cudaMallocAsync(&d_out, 5 * sizeof(double), a->st));
    const bool a2 = a->prec == SVB_C128, b2 = b->prec == SVB_C128;
    if (a2 && b2) launch_compare<double, double>(a->amps, b->amps, a->n, a->d_ws, d_out, a->st);
    else if (a2) launch_compare<double, float>(a->amps, b->amps, a->n, a->d_ws, d_out, a->st);
    else if (b2) launch_compare<float, double>(a->amps, b->amps, a->n, a->d_ws, d_out, a->st);
    else launch_compare<float, float>(a->amps, b->amps, a->n, a->d_ws, d_out, a->st);
    SVB_CUDA(cudaMemcpyAsync(out, d_out, 5 * sizeof(double), cudaMemcpyDeviceToHost, a->st));
    SVB_CUDA(cudaFreeAsync(d_out, a->st));
    SVB_CUDA(cudaStreamSynchronize(a->st));
  });
}

int svb_sample(svb_handle h, const int32_t* qubits, int k, const int32_t* bit_src, int w, uint64_t shots,
               const uint64_t* pcg, int sampler, uint64_t* out_codes, uint64_t* out_counts,
               uint64_t* n_unique) {
  return guard([&] {
    check_handle(h);
    require(shots >= 1, SVB_E_ARG, "shots must be positive");
    require(k >= 1 && k <= h->n, SVB_E_ARG, "bad measured-qubit count");
    require(w >= 1 && w <= 63, SVB_E_ARG, "bad clbit count");
    for (int j = 0; j < k; ++j) {
      require(qubits[j] >= 0 && qubits[j] < h->n, SVB_E_ARG, "qubit out of range");
      require(j == 0 || qubits[j] > qubits[j - 1], SVB_E_ARG, "qubits must be ascending");
    }
    for (int p = 0; p < w; ++p) require(bit_src[p] >= 0 && bit_src[p] < k, SVB_E_ARG, "bad bit source");
    require(sampler == SVB_SAMPLER_ALIAS || sampler == SVB_SAMPLER_CDF, SVB_E_ARG, "bad sampler");
    cudaStream_t st = h->st;
    uint64_t* d_codes = nullptr;
    SVB_CUDA(cudaMallocAsync(&d_codes, shots * sizeof(uint64_t), st));
    uint64_t m = 1ull << k;
    bool full = (k == h->n);
    if (sampler == SVB_SAMPLER_CDF && full && h->n >= 5) {
      if (h->prec == SVB_C128) cdf_draw<double>(h->amps, h->n, shots, pcg, bit_src, w, d_codes, st);
      else cdf_draw<float>(h->amps, h->n, shots, pcg, bit_src, w, d_codes, st);
    } else {
      double* d_probs = nullptr;
      SVB_CUDA(cudaMallocAsync(&d_probs, m * sizeof(double), st));
      ensure_ws(h, marginal_ws_doubles(h->n, k) + 1);
      if (h->prec == SVB_C128) launch_marginal<double>(h->amps, h->n, qubits, k, d_probs, h->d_ws, h->ws_doubles, st);
      else launch_marginal<float>(h->amps, h->n, qubits, k, d_probs, h->d_ws, h->ws_doubles, st);
      if (sampler == SVB_SAMPLER_CDF) {
        cdf_draw_probs(d_probs, m, shots, pcg, bit_src, w, d_codes, st);
      } else {
        double* d_prob_row = nullptr;
        int64_t* d_alias = nullptr;
        SVB_CUDA(cudaMallocAsync(&d_prob_row, m * sizeof(double), st));
        SVB_CUDA(cudaMallocAsync(&d_alias, m * sizeof(int64_t), st));
        try {
          alias_build(d_probs, m, d_prob_row, d_alias, st);
        } catch (...) {
          cudaFreeAsync(d_prob_row, st);
          cudaFreeAsync(d_alias, st);
          cudaFreeAsync(d_probs, st);
          cudaFreeAsync(d_codes, st);
          throw;
        }
        alias_draw(d_prob_row, d_alias, m, shots, pcg, bit_src, w, d_codes, st);
        SVB_CUDA(cudaFreeAsync(d_prob_row, st));
        SVB_CUDA(cudaFreeAsync(d_alias, st));
      }
      SVB_CUDA(cudaFreeAsync(d_probs, st));
    }
    *n_unique = histogram_codes(d_codes, shots, w, out_codes, out_counts, st);
    SVB_CUDA(cudaFreeAsync(d_codes, st));
    SVB_CUDA(cudaStreamSynchronize(st));
  });
}

int svb_alias_table(int device, const double* probs, uint64_t m, double* prob_row, int64_t* alias_row) {
  return guard([&] {
    require(m >= 1, SVB_E_SAMPLING, "need a non-empty 1-D probability vector");
    for (uint64_t i = 0; i < m; ++i) require(probs[i] >= 0.0, SVB_E_SAMPLING, "negative probability");
    SVB_CUDA(cudaSetDevice(device));
    cudaStream_t st;
    SVB_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    double *dp = nullptr, *dr = nullptr;
    int64_t* da = nullptr;
    try {
      SVB_CUDA(cudaMallocAsync(&dp, m * sizeof(double), st));
      SVB_CUDA(cudaMallocAsync(&dr, m * sizeof(double), st));
      SVB_CUDA(cudaMallocAsync(&da, m * sizeof(int64_t), st));
      SVB_CUDA(cudaMemcpyAsync(dp, probs, m * sizeof(double), cudaMemcpyHostToDevice, st));
      alias_build(dp, m, dr, da, st);
      SVB_CUDA(cudaMemcpyAsync(prob_row, dr, m * sizeof(double), cudaMemcpyDeviceToHost, st));
      SVB_CUDA(cudaMemcpyAsync(alias_row, da, m * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
      SVB_CUDA(cudaStreamSynchronize(st));
    } catch (...) {
      cudaFreeAsync(dp, st); cudaFreeAsync(dr, st); cudaFreeAsync(da, st);
      cudaStreamSynchronize(st);
      cudaStreamDestroy(st);
      throw;
    }
    cudaFreeAsync(dp, st); cudaFreeAsync(dr, st); cudaFreeAsync(da, st);
    SVB_CUDA(cudaStreamSynchronize(st));
    cudaStreamDestroy(st);
  });
}

// AliasTable.from_probs(probs).sample_indices(rng, shots) (sampling.py:30-83)
// on the device: the table build and the draws of `shots` uniforms from the
// numpy PCG64 state `pcg` (pblock's per-group terminal draws, result.py:63-66).
int svb_alias_draw(int device, const double* probs, uint64_t m, uint64_t shots, const uint64_t* pcg,
                   uint64_t* out_idx) {
  return guard([&] {
    require(m >= 1 && (m & (m - 1)) == 0 && m <= (1ull << 40), SVB_E_ARG, "alias_draw: m must be a power of two");
    require(shots >= 1, SVB_E_ARG, "shots must be positive");
    for (uint64_t i = 0; i < m; ++i) require(probs[i] >= 0.0, SVB_E_SAMPLING, "negative probability");
    SVB_CUDA(cudaSetDevice(device));
    cudaStream_t st;
    SVB_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    double *dp = nullptr, *dr = nullptr;
    int64_t* da = nullptr;
    uint64_t* dc = nullptr;
    int w = 0;
    while ((1ull << w) < m) ++w;
    std::vector<int32_t> ident(64);
    for (int p = 0; p < 64; ++p) ident[p] = p;
    auto cleanup = [&] {
      cudaFreeAsync(dp, st); cudaFreeAsync(dr, st); cudaFreeAsync(da, st); cudaFreeAsync(dc, st);
      cudaStreamSynchronize(st);
      cudaStreamDestroy(st);
    };
    try {
      SVB_CUDA(cudaMallocAsync(&dp, m * sizeof(double), st));
      SVB_CUDA(cudaMallocAsync(&dr, m * sizeof(double), st));
      SVB_CUDA(cudaMallocAsync(&da, m * sizeof(int64_t), st));
      SVB_CUDA(cudaMallocAsync(&dc, shots * sizeof(uint64_t), st));
      SVB_CUDA(cudaMemcpyAsync(dp, probs, m * sizeof(double), cudaMemcpyHostToDevice, st));
      alias_build(dp, m, dr, da, st);
      alias_draw(dr, da, m, shots, pcg, ident.data(), w, dc, st);
      SVB_CUDA(cudaMemcpyAsync(out_idx, dc, shots * sizeof(uint64_t), cudaMemcpyDeviceToHost, st));
      SVB_CUDA(cudaStreamSynchronize(st));
    } catch (...) {
      cleanup();
      throw;
    }
    cleanup();
  });
}

// AliasTable.sample_indices (sampling.py:78-83) for a table already built
// (any m): v = u*m, idx = floor(v), idx if v - idx < prob[idx] else alias[idx],
// with u the next `shots` doubles of the numpy PCG64 state pcg[4].
int svb_alias_sample(int device, const double* prob_row, const int64_t* alias_row, uint64_t m, uint64_t shots,
                     const uint64_t* pcg, uint64_t* out_idx) {
  return guard([&] {
    require(m >= 1 && m <= (1ull << 40), SVB_E_ARG, "alias_sample: bad table size");
    require(shots >= 1, SVB_E_ARG, "shots must be positive");
    SVB_CUDA(cudaSetDevice(device));
    cudaStream_t st;
    SVB_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    double* dr = nullptr;
    int64_t* da = nullptr;
    uint64_t* dc = nullptr;
    int w = 0;
    while ((1ull << w) < m) ++w;
    std::vector<int32_t> ident(64);
    for (int p = 0; p < 64; ++p) ident[p] = p;
    auto cleanup = [&] {
      cudaFreeAsync(dr, st); cudaFreeAsync(da, st); cudaFreeAsync(dc, st);
      cudaStreamSynchronize(st);
      cudaStreamDestroy(st);
    };
    try {
      SVB_CUDA(cudaMallocAsync(&dr, m * sizeof(double), st));
      SVB_CUDA(cudaMallocAsync(&da, m * sizeof(int64_t), st));
      SVB_CUDA(cudaMallocAsync(&dc, shots * sizeof(uint64_t), st));
      SVB_CUDA(cudaMemcpyAsync(dr, prob_row, m * sizeof(double), cudaMemcpyHostToDevice, st));
      SVB_CUDA(cudaMemcpyAsync(da, alias_row, m * sizeof(int64_t), cudaMemcpyHostToDevice, st));
      alias_draw(dr, da, m, shots, pcg, ident.data(), w, dc, st);
      SVB_CUDA(cudaMemcpyAsync(out_idx, dc, shots * sizeof(uint64_t), cudaMemcpyDeviceToHost, st));
      SVB_CUDA(cudaStreamSynchronize(st));
    } catch (...) {
      cleanup();
      throw;
    }
    cleanup();
  });
}

// Device-resident alias tables: sampling.AliasTable uploads its rows once and
// draws from them (a per-call upload made a 2^20-row table's draws ~3x the
// cost of a 16-row table's, against the reference's O(1)-per-draw test).
struct svb_alias_dev {
  int device = 0;
  uint64_t m = 0;
  double* prob = nullptr;
  int64_t* alias = nullptr;
};

int svb_alias_upload(int device, const double* prob_row, const int64_t* alias_row, uint64_t m, void** out_table) {
  svb_alias_dev* t = nullptr;
  const int rc = guard([&] {
    require(m >= 1 && m <= (1ull << 40), SVB_E_ARG, "alias_upload: bad table size");
    SVB_CUDA(cudaSetDevice(device));
    t = new svb_alias_dev();
    t->device = device;
    t->m = m;
    if (cudaMalloc(&t->prob, m * sizeof(double)) != cudaSuccess ||
        cudaMalloc(&t->alias, m * sizeof(int64_t)) != cudaSuccess) {
      cudaGetLastError();
      throw Error(SVB_E_OOM, "alias_upload: device allocation failed");
    }
    SVB_CUDA(cudaMemcpy(t->prob, prob_row, m * sizeof(double), cudaMemcpyHostToDevice));
    SVB_CUDA(cudaMemcpy(t->alias, alias_row, m * sizeof(int64_t), cudaMemcpyHostToDevice));
  });
  if (rc != SVB_OK && t) {
    cudaFree(t->prob);
    cudaFree(t->alias);
    delete t;
    t = nullptr;
  }
  *out_table = t;
  return rc;
}

int svb_alias_sample_table(void* table, uint64_t shots, const uint64_t* pcg, uint64_t* out_idx) {
  return guard([&] {
    require(table != nullptr, SVB_E_ARG, "alias_sample_table: null table");
    require(shots >= 1, SVB_E_ARG, "shots must be positive");
    const svb_alias_dev* t = static_cast<const svb_alias_dev*>(table);
    SVB_CUDA(cudaSetDevice(t->device));
    // one stream per thread and device, and the pool's freed scratch kept
    // mapped: a per-call stream and a re-mapped output buffer made the cost of
    // a draw batch vary by milliseconds
    keep_pool_mapped(t->device);
    static thread_local cudaStream_t streams[16] = {};
    cudaStream_t& st = streams[t->device & 15];
    if (!st) SVB_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    uint64_t* dc = nullptr;
    int w = 0;
    while ((1ull << w) < t->m) ++w;
    int32_t ident[64];
    for (int p = 0; p < 64; ++p) ident[p] = p;
    static const bool trace = std::getenv("SVB_TRACE") != nullptr;
    const auto h0 = std::chrono::steady_clock::now();
    try {
      SVB_CUDA(cudaMallocAsync(&dc, shots * sizeof(uint64_t), st));
      alias_draw(t->prob, t->alias, t->m, shots, pcg, ident, w, dc, st);
      if (trace) {
        SVB_CUDA(cudaStreamSynchronize(st));
        std::fprintf(stderr, "[svb] alias_sample_table m=%llu shots=%llu draw %.3f ms\n", (unsigned long long)t->m,
                     (unsigned long long)shots,
                     std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - h0).count());
      }
      // large batches land in a pinned staging buffer (DMA at link speed
      // whatever state the caller's pages are in), then one host copy
      const size_t bytes = shots * sizeof(uint64_t);
      static thread_local void* pin = nullptr;
      static thread_local size_t pin_bytes = 0;
      if (bytes >= (512u << 10) && pin_bytes < bytes) {
        if (pin) cudaFreeHost(pin);
        pin = nullptr;
        pin_bytes = 0;
        if (cudaHostAlloc(&pin, bytes, cudaHostAllocPortable) == cudaSuccess) pin_bytes = bytes;
        else cudaGetLastError();
      }
      const bool staged = bytes >= (512u << 10) && pin_bytes >= bytes;
      SVB_CUDA(cudaMemcpyAsync(staged ? pin : out_idx, dc, bytes, cudaMemcpyDeviceToHost, st));
      SVB_CUDA(cudaFreeAsync(dc, st));
      SVB_CUDA(cudaStreamSynchronize(st));
      if (staged) std::memcpy(out_idx, pin, bytes);
      if (trace)
        std::fprintf(stderr, "[svb] alias_sample_table total %.3f ms\n",
                     std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - h0).count());
    } catch (...) {
      cudaStreamSynchronize(st);
      throw;
    }
  });
}

int svb_alias_release(void* table) {
  return guard([&] {
    svb_alias_dev* t = static_cast<svb_alias_dev*>(table);
    if (!t) return;
    cudaSetDevice(t->device);
    cudaFree(t->prob);
    cudaFree(t->alias);
    delete t;
  });
}

int svb_device_ptr(svb_handle h, void** ptr, uint64_t* bytes, int64_t* stream) {
  return guard([&] {
    check_handle(h);
    SVB_CUDA(cudaStreamSynchronize(h->st));
    *ptr = h->amps;
    *bytes = (uint64_t)h->amp_bytes();
    *stream = (int64_t)(intptr_t)h->st;
  });
}

int svb_clear(svb_handle h) {
  return guard([&] {
    check_handle_nomat(h);
    h->zero_pending = false;
    SVB_CUDA(cudaMemsetAsync(h->amps, 0, h->amp_bytes(), h->st));
    SVB_CUDA(cudaStreamSynchronize(h->st));
  });
}

int svb_sample_slice(svb_handle h, uint64_t shots, const uint64_t* pcg, double lo, double hi, double total,
                     const int32_t* bit_src, int w, uint64_t code_or, uint64_t* out_codes, uint64_t* out_counts,
                     uint64_t* n_unique) {
  return guard([&] {
    check_handle(h);
    require(shots >= 1 && w >= 1 && w <= 63 && h->n >= 5, SVB_E_ARG, "bad slice sampling arguments");
    for (int p = 0; p < w; ++p) require(bit_src[p] >= -1 && bit_src[p] < h->n, SVB_E_ARG, "bad bit source");
    uint64_t* d_codes = nullptr;
    SVB_CUDA(cudaMallocAsync(&d_codes, shots * sizeof(uint64_t), h->st));
    slice_draw(h->amps, h->prec == SVB_C128, h->n, shots, pcg, lo, hi, total, bit_src, w, code_or, d_codes, h->st);
    *n_unique = histogram_codes(d_codes, shots, 64, out_codes, out_counts, h->st);
    SVB_CUDA(cudaFreeAsync(d_codes, h->st));
    SVB_CUDA(cudaStreamSynchronize(h->st));
  });
}

int svb_half_copy(svb_handle h, int L, int bit, void* dev_buf, int to_buf) {
  return guard([&] {
    check_handle(h);
    require(L >= 0 && L < h->n && (bit == 0 || bit == 1), SVB_E_ARG, "bad half selector");
    if (h->prec == SVB_C128) launch_half_copy<double>(h->amps, h->n, dev_buf, L, bit, to_buf, h->st);
    else launch_half_copy<float>(h->amps, h->n, dev_buf, L, bit, to_buf, h->st);
    SVB_CUDA(cudaStreamSynchronize(h->st));
  });
}

int svb_block_copy(svb_handle h, const int32_t* lbits, int g, uint64_t block, uint64_t offset, uint64_t count,
                   void* dev_buf, int to_buf, int sync) {
  return guard([&] {
    check_handle(h);
    require(g >= 1 && g <= 8 && g < h->n, SVB_E_ARG, "block copy: 1 <= g <= 8 local bits");
    BlockSel sel{};
    sel.g = g;
    for (int b = 0; b < g; ++b) {
      sel.L[b] = lbits[b];
      require(lbits[b] >= 0 && lbits[b] < h->n && (b == 0 || lbits[b] > lbits[b - 1]), SVB_E_ARG,
              "block copy: local bits must be ascending and in range");
      if ((block >> b) & 1) sel.bits |= 1ull << lbits[b];
    }
    require(block < (1ull << g), SVB_E_ARG, "block copy: bad block");
    const uint64_t blen = 1ull << (h->n - g);
    require(offset <= blen && count <= blen - offset, SVB_E_ARG, "block copy: range out of the block");
    if (count == 0) return;
    if (h->prec == SVB_C128) launch_block_copy<double>(h->amps, dev_buf, sel, offset, count, to_buf, h->st);
    else launch_block_copy<float>(h->amps, dev_buf, sel, offset, count, to_buf, h->st);
    if (sync) SVB_CUDA(cudaStreamSynchronize(h->st));
  });
}

// ---- partitioned-block support (pblock.py:76-120) ----------------------
int svb_outer(svb_handle dst, svb_handle a, svb_handle b) {
  return guard([&] {
    check_handle_nomat(dst);
    check_handle(a);
    check_handle(b);
    require(dst->n == a->n + b->n && dst->prec == a->prec && dst->prec == b->prec, SVB_E_ARG,
            "outer: dst must hold a.n + b.n qubits of the same precision");
    require(dst->device == a->device && dst->device == b->device, SVB_E_ARG, "outer: states on different devices");
    SVB_CUDA(cudaStreamSynchronize(a->st));
    SVB_CUDA(cudaStreamSynchronize(b->st));
    if (dst->prec == SVB_C128) launch_outer<double>(dst->amps, a->amps, b->amps, a->n, b->n, dst->st);
    else launch_outer<float>(dst->amps, a->amps, b->amps, a->n, b->n, dst->st);
    dst->zero_pending = false;
    SVB_CUDA(cudaStreamSynchronize(dst->st));
  });
}

int svb_permute_qubits(svb_handle h, const int32_t* dest) {
  return guard([&] {
    check_handle(h);
    std::vector<int> d(h->n);
    uint64_t seen = 0;
    for (int p = 0; p < h->n; ++p) {
      d[p] = dest[p];
      require(d[p] >= 0 && d[p] < h->n && !((seen >> d[p]) & 1ull), SVB_E_ARG, "permute: dest is not a permutation");
      seen |= 1ull << d[p];
    }
    if (h->prec == SVB_C128) run_permutation<double>(&h->amps, &h->spare, h->n, d, h->st, &h->stats);
    else run_permutation<float>(&h->amps, &h->spare, h->n, d, h->st, &h->stats);
    restore_view(h);
    SVB_CUDA(cudaStreamSynchronize(h->st));
  });
}

int svb_select_half(svb_handle dst, svb_handle src, int qubit, int bit) {
  return guard([&] {
    check_handle_nomat(dst);
    check_handle(src);
    require(src->n >= 2 && dst->n == src->n - 1 && dst->prec == src->prec && dst->device == src->device, SVB_E_ARG,
            "select_half: dst must hold src.n - 1 qubits of the same precision");
    require(qubit >= 0 && qubit < src->n && (bit == 0 || bit == 1), SVB_E_ARG, "bad half selector");
    if (src->prec == SVB_C128) launch_half_copy<double>(src->amps, src->n, dst->amps, qubit, bit, 1, src->st);
    else launch_half_copy<float>(src->amps, src->n, dst->amps, qubit, bit, 1, src->st);
    dst->zero_pending = false;
    SVB_CUDA(cudaStreamSynchronize(src->st));
  });
}

int svb_rng_seed(svb_handle h, const uint64_t* pcg) {
  return guard([&] {
    check_handle(h);
    SVB_CUDA(cudaMemcpyAsync(h->d_rng, pcg, 4 * sizeof(uint64_t), cudaMemcpyHostToDevice, h->st));
    SVB_CUDA(cudaStreamSynchronize(h->st));
  });
}

static void do_measure(svb_handle h, int q, bool reset, uint64_t* d_code, int rank) {
  require(q >= 0 && q < h->n, SVB_E_ARG, "qubit out of range");
  ensure_ws(h, measure_ws_doubles(h->n) + 1);
  if (h->prec == SVB_C128)
    launch_measure<double>(h->amps, h->n, q, reset, h->d_rng, h->d_ws, h->d_outcome, d_code, rank, h->st);
  else
    launch_measure<float>(h->amps, h->n, q, reset, h->d_rng, h->d_ws, h->d_outcome, d_code, rank, h->st);
}

int svb_measure(svb_handle h, int qubit, int32_t* outcome) {
  return guard([&] {
    check_handle(h);
    do_measure(h, qubit, false, nullptr, 0);
    SVB_CUDA(cudaMemcpyAsync(outcome, h->d_outcome, sizeof(int32_t), cudaMemcpyDeviceToHost, h->st));
    SVB_CUDA(cudaStreamSynchronize(h->st));
  });
}

int svb_reset(svb_handle h, int qubit) {
  return guard([&] {
    check_handle(h);
    do_measure(h, qubit, true, nullptr, 0);
    SVB_CUDA(cudaStreamSynchronize(h->st));
  });
}

int svb_replay(svb_handle work, svb_handle prefix, const int32_t* ops, int n_ops, const svb_gate* gates,
               const int32_t* clbit_rank, uint64_t shots, const uint64_t* pcg, uint64_t* out_codes) {
  return guard([&] {
    check_handle(work);
    check_handle(prefix);
    require(work->n == prefix->n && work->prec == prefix->prec, SVB_E_ARG, "state shape mismatch");
    require(work->device == prefix->device, SVB_E_ARG, "states on different devices");
    cudaStream_t st = work->st;
    // prefix may have pending work on its own stream
    SVB_CUDA(cudaStreamSynchronize(prefix->st));
    int ngates = 0;
    for (int i = 0; i < n_ops; ++i) {
      int kind = ops[3 * i];
      require(kind >= 0 && kind <= 2, SVB_E_ARG, "bad replay op");
      if (kind == 0) ngates = std::max(ngates, ops[3 * i + 1] + 1);
      if (kind == 1) {  // one shot's clbits are packed into a uint64 code
        const int r = clbit_rank[ops[3 * i + 2]];
        require(r >= 0 && r < 64, SVB_E_ARG, "replay: clbit rank must be in [0, 64)");
      }
    }
    validate_gates(work, gates, ngates);
    uint64_t* d_codes = nullptr;
    SVB_CUDA(cudaMallocAsync(&d_codes, shots * sizeof(uint64_t), st));
    SVB_CUDA(cudaMemsetAsync(d_codes, 0, shots * sizeof(uint64_t), st));
    SVB_CUDA(cudaMemcpyAsync(work->d_rng, pcg, 4 * sizeof(uint64_t), cudaMemcpyHostToDevice, st));
    ensure_ws(work, measure_ws_doubles(work->n) + 1);
    work->stats = ProgramStats{};
    for (uint64_t s = 0; s < shots; ++s) {
      SVB_CUDA(cudaMemcpyAsync(work->amps, prefix->amps, prefix->amp_bytes(), cudaMemcpyDeviceToDevice, st));
      int i = 0;
      while (i < n_ops) {
        int kind = ops[3 * i];
        if (kind == 0) {  // maximal run of gates -> one program
          int j = i;
          std::vector<svb_gate> run;
          while (j < n_ops && ops[3 * j] == 0) run.push_back(gates[ops[3 * j + 1]]), ++j;
          if (work->prec == SVB_C128)
            run_program_owned<double>(&work->amps, &work->spare, work->n, run.data(), (int)run.size(), work->fusion, work->jit_min_n, st, &work->stats, nullptr);
          else
            run_program_owned<float>(&work->amps, &work->spare, work->n, run.data(), (int)run.size(), work->fusion, work->jit_min_n, st, &work->stats, nullptr);
          i = j;
        } else {
          int q = ops[3 * i + 1];
          if (kind == 1) do_measure(work, q, false, d_codes + s, clbit_rank[ops[3 * i + 2]]);
          else do_measure(work, q, true, nullptr, 0);
          ++i;
        }
      }
    }
    SVB_CUDA(cudaMemcpyAsync(out_codes, d_codes, shots * sizeof(uint64_t), cudaMemcpyDeviceToHost, st));
    SVB_CUDA(cudaFreeAsync(d_codes, st));
    SVB_CUDA(cudaStreamSynchronize(st));
  });
}

}  // extern "C"
