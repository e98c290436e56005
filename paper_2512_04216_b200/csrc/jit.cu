// JIT specialisation of fused gate programs (NVRTC -> sm_100a cubin).
//
// The interpreter kernel (InterpBody) decodes ops at run time; that costs a
// header decode per op and, worse, forces the compiler to shuffle the whole
// register-resident amplitude array at every dispatch merge.  Here every pass
// of a scheduled program becomes a kernel whose Body is straight-line code:
// round layouts unrolled, register-bit positions as template arguments,
// matrix coefficients as hexfloat immediates, conditions folded.  The skeleton
// (streaming ring, uniform diagonal factors, stores) is the same
// pass_kernel<> the interpreter uses: device_core.cuh is embedded in the
// library and handed to NVRTC as an in-memory header.
//
// NVRTC is dlopen'ed and the driver API is reached through
// cudaGetDriverEntryPoint, so the library loads (and runs the interpreter) on
// machines without either.  Modules are cached per process by source hash.
#include <cuda.h>
#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <memory>
#include <chrono>
#include <mutex>
#include <shared_mutex>
#include <sstream>
#include <thread>
#include <string>
#include <unordered_map>
#include <unordered_set>
#include <vector>

#include "jit.h"
#include "program.h"

extern const char svb_device_core_src[];

namespace svb {

namespace {

// ---------------------------------------------------------------- NVRTC
typedef int nvrtcResult_t;
struct Nvrtc {
  void* h = nullptr;
  nvrtcResult_t (*create)(void**, const char*, const char*, int, const char* const*, const char* const*) = nullptr;
  nvrtcResult_t (*compile)(void*, int, const char* const*) = nullptr;
  nvrtcResult_t (*log_size)(void*, size_t*) = nullptr;
  nvrtcResult_t (*log)(void*, char*) = nullptr;
  nvrtcResult_t (*cubin_size)(void*, size_t*) = nullptr;
  nvrtcResult_t (*cubin)(void*, char*) = nullptr;
  nvrtcResult_t (*destroy)(void**) = nullptr;
  bool ok = false;
  Nvrtc() {
    const char* names[] = {"libnvrtc.so.12", "/usr/local/cuda/lib64/libnvrtc.so.12", "libnvrtc.so"};
    for (const char* n : names)
      if ((h = dlopen(n, RTLD_NOW | RTLD_LOCAL))) break;
    if (!h) return;
    create = (decltype(create))dlsym(h, "nvrtcCreateProgram");
    compile = (decltype(compile))dlsym(h, "nvrtcCompileProgram");
    log_size = (decltype(log_size))dlsym(h, "nvrtcGetProgramLogSize");
    log = (decltype(log))dlsym(h, "nvrtcGetProgramLog");
    cubin_size = (decltype(cubin_size))dlsym(h, "nvrtcGetCUBINSize");
    cubin = (decltype(cubin))dlsym(h, "nvrtcGetCUBIN");
    destroy = (decltype(destroy))dlsym(h, "nvrtcDestroyProgram");
    ok = create && compile && log_size && log && cubin_size && cubin && destroy;
  }
};

// ---------------------------------------------------------- driver API
struct Driver {
  CUresult (*load)(CUmodule*, const void*) = nullptr;
  CUresult (*getfn)(CUfunction*, CUmodule, const char*) = nullptr;
  CUresult (*setattr)(CUfunction, CUfunction_attribute, int) = nullptr;
  CUresult (*unload)(CUmodule) = nullptr;
  CUresult (*launch)(CUfunction, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned, CUstream,
                     void**, void**) = nullptr;
  bool ok = false;
  Driver() {
    auto get = [](const char* name, void** fn) {
      cudaDriverEntryPointQueryResult q;
      return cudaGetDriverEntryPoint(name, fn, cudaEnableDefault, &q) == cudaSuccess &&
             q == cudaDriverEntryPointSuccess && *fn;
    };
    ok = get("cuModuleLoadData", (void**)&load) && get("cuModuleGetFunction", (void**)&getfn) &&
         get("cuFuncSetAttribute", (void**)&setattr) && get("cuLaunchKernel", (void**)&launch) &&
         get("cuModuleUnload", (void**)&unload);
    if (!ok) cudaGetLastError();
  }
};

struct Module {
  CUmodule mod = nullptr;
  std::vector<CUfunction> fns;
  uint64_t last_use = 0;
};

std::mutex g_mu;
std::unordered_map<std::string, Module> g_cache;  // key: device + source
std::unordered_map<std::string, std::shared_ptr<std::mutex>> g_key_locks;  // in-flight compiles
std::unordered_set<std::string> g_inflight;  // background compiles (asynchronous mode)
thread_local bool t_async_jit = false;
uint64_t g_tick = 0;  // LRU clock (under g_mu)
// Bounds of the in-memory caches: programs whose coefficients are compiled in
// as immediates (n >= 28) make a new kernel per angle set, so a parameter
// sweep would otherwise grow them (and the loaded modules) without limit.
constexpr size_t kMaxModules = 768, kMaxPrograms = 256;
// Launchers hold it shared from the cache lookup to the last launch; module
// eviction holds it exclusively (and synchronises the device) before
// cuModuleUnload, so no function of an unloaded module is ever launched.
std::shared_mutex g_launch_mu;
// Whole programs seen before: their kernels and launch parameters, keyed by a
// 128-bit hash of the encoded program (passes + op stream), so repeated
// applies skip source generation (tens of ms of host time the GPU would idle).
struct ProgKernels {
  std::vector<CUfunction> fns;
  std::vector<int> nslots;
  std::vector<uint32_t> staged;
  uint64_t last_use = 0;
};
struct Key128 {
  uint64_t a, b;
  bool operator==(const Key128& o) const { return a == o.a && b == o.b; }
};
struct Key128Hash {
  size_t operator()(const Key128& k) const { return (size_t)(k.a ^ (k.b * 0x9E3779B97F4A7C15ull)); }
};
std::unordered_map<Key128, ProgKernels, Key128Hash> g_prog;

// four independent multiply-rotate lanes over 32-byte blocks (runs on every
// apply over the program's pass descriptors and op stream)
void mix_bytes(Key128& k, const void* data, size_t n) {
  const unsigned char* p = static_cast<const unsigned char*>(data);
  uint64_t h[4] = {k.a, k.b, k.a ^ 0x165667B19E3779F9ull, k.b + 0x27D4EB2F165667C5ull};
  auto mix = [](uint64_t x, uint64_t w) {
    x ^= w * 0x87C37B91114253D5ull;
    x = (x << 31) | (x >> 33);
    return x * 0x4CF5AD432745937Full;
  };
  size_t i = 0;
  for (; i + 32 <= n; i += 32) {
    uint64_t w[4];
    std::memcpy(w, p + i, 32);
    for (int l = 0; l < 4; ++l) h[l] = mix(h[l], w[l]);
  }
  for (int l = 0; i < n; i += 8, ++l) {
    uint64_t w = 0;
    std::memcpy(&w, p + i, std::min<size_t>(8, n - i));
    h[l & 3] = mix(h[l & 3], w);
  }
  k.a = h[0] ^ (h[2] * 0x9E3779B97F4A7C15ull) ^ n;
  k.b = h[1] ^ (h[3] * 0xC2B2AE3D27D4EB4Full) + n * 0x9E3779B97F4A7C15ull;
  k.a ^= k.a >> 29;
  k.b ^= k.b >> 31;
}

std::string hexf(double x, bool single) {
  char buf[64];
  if (single) std::snprintf(buf, sizeof buf, "%af", (double)(float)x);
  else std::snprintf(buf, sizeof buf, "%a", x);
  std::string s(buf);
  if (!std::isfinite(single ? (double)(float)x : x)) {
    // non-finite coefficients keep their bit pattern (inf / NaN propagate
    // exactly as in the interpreter and the reference)
    if (single) {
      const float f = (float)x;
      uint32_t b;
      std::memcpy(&b, &f, 4);
      std::snprintf(buf, sizeof buf, "__int_as_float(0x%08x)", b);
    } else {
      uint64_t b;
      std::memcpy(&b, &x, 8);
      std::snprintf(buf, sizeof buf, "__longlong_as_double((long long)0x%016llxull)", (unsigned long long)b);
    }
    return std::string(buf);
  }
  return s;
}

template <typename R> std::string cimm(const cplx<R>& z) {
  const bool single = sizeof(R) == 4;
  return "svb::mk<R>(" + hexf((double)z.x, single) + ", " + hexf((double)z.y, single) + ")";
}

template <typename C> bool is1(const C& z) { return z.x == 1 && z.y == 0; }

// Straight-line code of one DIAG payload (see DiagHdr): tile-uniform factors
// come from the pass's uniform slot, thread-dependent factors are evaluated
// with immediates, and factors that are exactly 1 by construction are dropped
// at generation time (controlled phases leave half the amplitudes untouched).
struct PrologueCtx {
  std::ostringstream* o = nullptr;  // prologue code (runs once per thread)
  std::ostringstream* pre = nullptr;  // preload(): round-0 HBM loads of a direct first round
  int nslots = 0;                   // per-thread complex slots
  int round = 0;                    // round of the op being emitted
};

// A DIAG that only multiplies each amplitude by per-register-bit factors
// (no tile/thread-uniform scalar C, no |0>-half factors, no register pairs):
// it can be fused with a preceding product state (emit_diag's `prod`).
template <typename R> bool diag_per_bit_only(const uint8_t* payload, int RB) {
  DiagHdr h;
  std::memcpy(&h, payload, sizeof h);
  if (h.nUC || h.nUTg || h.nTC || h.nRR) return false;
  const DiagTerm<R>* u = reinterpret_cast<const DiagTerm<R>*>(payload + sizeof(DiagHdr));
  int nur = 0;
  for (int i = 0; i < RB; ++i) nur += h.nUR[i];
  for (int k = 0; k < nur + h.nTR; ++k)
    if (!is1(u[k].d[0]) || !is1(u[k].d[2])) return false;
  return true;
}

// prod (support-tracked round 0, immediates): the registers hold the product
// state a[v] = a[0] * prod_{i in v} prod[i] of leading pivot ops that were not
// emitted; the DIAG (diag_per_bit_only) then builds a[v] = a[0] * prod E_i with
// E_i = prod[i] * D1_i in one tree: 15 complex products instead of the pivot
// expansions, the factor tree and a multiply per amplitude.
template <typename R>
void emit_diag(std::ostringstream& o, const uint8_t* payload, uint32_t pay_off, int RB, bool imm,
               PrologueCtx& pc, const cplx<R>* prod = nullptr) {
  // factor e of a term: an immediate (large programs) or a load from the op
  // payload in shared memory (structure-only code shared across angles)
  auto dref = [&](const void* term, int e) {
    if (imm) return cimm<R>(reinterpret_cast<const DiagTerm<R>*>(term)->d[e]);
    const uint32_t addr = pay_off + (uint32_t)((const uint8_t*)term - payload) + 16 + e * (uint32_t)sizeof(cplx<R>);
    return "reinterpret_cast<const svb::cplx<R>*>(c.ops + " + std::to_string(addr) + ")[0]";
  };
  DiagHdr h;
  std::memcpy(&h, payload, sizeof h);
  const DiagTerm<R>* t = reinterpret_cast<const DiagTerm<R>*>(payload + sizeof(DiagHdr));
  bool d0one[8], d1one[8], cone = true;
  bool d0real[8], d1real[8], creal = true;  // every contributing entry real
  for (int i = 0; i < RB; ++i) d0one[i] = d1one[i] = d0real[i] = d1real[i] = true;
  const DiagTerm<R>* u = t;
  for (int i = 0; i < RB; ++i)
    for (int k = 0; k < h.nUR[i]; ++k, ++u) {
      if (!is1(u->d[0]) || !is1(u->d[2])) d0one[i] = false;
      if (!is1(u->d[1]) || !is1(u->d[3])) d1one[i] = false;
      if (u->d[0].y != 0 || u->d[2].y != 0) d0real[i] = false;
      if (u->d[1].y != 0 || u->d[3].y != 0) d1real[i] = false;
    }
  for (int k = 0; k < h.nUC; ++k, ++u)
    for (int e = 0; e < 4; ++e) {
      cone = cone && is1(u->d[e]);
      creal = creal && u->d[e].y == 0;
    }
  // UT groups: C also takes the group ratios selected by the thread's own bits
  std::vector<int> ut_q;
  for (int g = 0; g < h.nUTg; ++g) {
    ut_q.push_back(u->qa);
    for (int k = 0; k < h.utn[g]; ++k, ++u)
      for (int e = 0; e < 4; ++e) {
        cone = cone && is1(u->d[e]);
        creal = creal && u->d[e].y == 0;
      }
  }
  const DiagTerm<R>* tr = u;
  const DiagTerm<R>* tc = tr + h.nTR;
  const DiagTerm<R>* rr = tc + h.nTC;
  for (int k = 0; k < h.nTR; ++k) {
    const int i = tr[k].ra;
    if (!is1(tr[k].d[0]) || !is1(tr[k].d[2])) d0one[i] = false;
    if (!is1(tr[k].d[1]) || !is1(tr[k].d[3])) d1one[i] = false;
    if (tr[k].d[0].y != 0 || tr[k].d[2].y != 0) d0real[i] = false;
    if (tr[k].d[1].y != 0 || tr[k].d[3].y != 0) d1real[i] = false;
  }
  for (int k = 0; k < h.nTC; ++k)
    for (int e = 0; e < 4; ++e) {
      cone = cone && is1(tc[k].d[e]);
      creal = creal && tc[k].d[e].y == 0;
    }
  if (!imm) {
    // structure-only code: a factor is skipped only when no term contributes
    // to it (a value that happens to be 1 -- e.g. the deferred scale of a
    // pivot whose choice flips with the angle -- must not change the source)
    for (int i = 0; i < RB; ++i) d0one[i] = d1one[i] = h.nUR[i] == 0;
    for (int k = 0; k < h.nTR; ++k) d0one[tr[k].ra] = d1one[tr[k].ra] = false;
    cone = h.nUC == 0 && h.nUTg == 0 && h.nTC == 0;
  }
  o << "    {\n";
  const std::string us = "c.uni + " + std::to_string(h.slot * kUniStride);
  const bool has_uc = h.slot >= 0 && (h.nUC > 0 || h.nUTg > 0);
  if (!cone) o << "      svb::cplx<R> C = " << (has_uc ? "(" + us + ")[0]" : "svb::mk<R>(R(1), R(0))") << ";\n";
  for (size_t g = 0; g < ut_q.size(); ++g)
    o << "      if ((Fg >> " << ut_q[g] << ") & 1ull) C = svb::cmul<R>(C, (" << us << ")[" << (kUniV + (int)g) << "]);\n";
  for (int i = 0; i < RB; ++i) {
    const bool has_ur = h.slot >= 0 && h.nUR[i] > 0;
    if (!d0one[i])
      o << "      svb::cplx<R> D0_" << i << " = "
        << (has_ur ? "(" + us + ")[" + std::to_string(1 + i) + "]" : "svb::mk<R>(R(1), R(0))") << ";\n";
    if (!d1one[i])
      o << "      svb::cplx<R> D1_" << i << " = "
        << (has_ur ? "(" + us + ")[" + std::to_string(6 + i) + "]" : "svb::mk<R>(R(1), R(0))") << ";\n";
  }
  uint32_t pro_scaled = 0;  // prod: bits whose ratio went into a prologue slot
  // register-bit x thread-bit terms depend only on the thread's own local bits:
  // their products are evaluated once per thread in the prologue (st.v[slot])
  for (int i = 0; i < RB; ++i) {
    bool any0 = false, any1 = false;
    for (int k = 0; k < h.nTR; ++k) {
      if (tr[k].ra != i) continue;
      any0 = any0 || !(is1(tr[k].d[0]) && is1(tr[k].d[2]));
      any1 = any1 || !(is1(tr[k].d[1]) && is1(tr[k].d[3]));
    }
    for (int half = 0; half < 2; ++half) {
      if (!(half ? any1 : any0)) continue;
      std::vector<int> terms;
      for (int k = 0; k < h.nTR; ++k) {
        if (tr[k].ra != i) continue;
        if (half == 0 && is1(tr[k].d[0]) && is1(tr[k].d[2])) continue;
        if (half == 1 && is1(tr[k].d[1]) && is1(tr[k].d[3])) continue;
        terms.push_back(k);
      }
      if (terms.size() <= 2) {  // short chains: a select or one product per tile, no slot
        std::string f;
        for (int k : terms) {
          const std::string sel = "svb::csel<R>((int)((Fg >> " + std::to_string((int)tr[k].qb) + ") & 1ull), " +
                                  dref(tr + k, half) + ", " + dref(tr + k, 2 + half) + ")";
          f = f.empty() ? sel : "svb::cmul<R>(" + f + ", " + sel + ")";
        }
        o << "      D" << half << "_" << i << " = svb::cmul<R>(D" << half << "_" << i << ", " << f << ");\n";
        continue;
      }
      const int slot = pc.nslots++;
      std::ostringstream& P = *pc.o;
      P << "    { svb::cplx<R> acc = svb::mk<R>(R(1), R(0)); const uint64_t F = svb::thread_fixed_g<R, RB>(c, "
        << pc.round << ");\n";
      for (int k = 0; k < h.nTR; ++k) {
        if (tr[k].ra != i) continue;
        if (half == 0 && is1(tr[k].d[0]) && is1(tr[k].d[2])) continue;
        if (half == 1 && is1(tr[k].d[1]) && is1(tr[k].d[3])) continue;
        P << "      acc = svb::cmul<R>(acc, svb::csel<R>((int)((F >> " << (int)tr[k].qb << ") & 1ull), "
          << dref(tr + k, half) << ", " << dref(tr + k, 2 + half) << "));\n";
      }
      if (prod && half == 1) {  // the product tree's ratio of this bit, once per thread
        if (prod[i].y == 0) P << "      acc = svb::rmul<R>(" << hexf((double)prod[i].x, sizeof(R) == 4) << ", acc);\n";
        else P << "      acc = svb::cmul<R>(acc, " << cimm<R>(prod[i]) << ");\n";
        pro_scaled |= 1u << i;
      }
      P << "      c.pro[" << slot << " * c.nthr + c.tid] = acc; }\n";
      o << "      D" << half << "_" << i << " = svb::cmul<R>(D" << half << "_" << i << ", c.pro[" << slot
        << " * c.nthr + c.tid]);\n";
    }
  }
  for (int k = 0; k < h.nTC; ++k) {
    const int qa = tc[k].qa, qb = tc[k].qb;
    const std::string fa = qa >= 0 ? "(int)((Fg >> " + std::to_string(qa) + ") & 1ull)" : "0";
    const std::string fb = qb >= 0 ? "(int)((Fg >> " + std::to_string(qb) + ") & 1ull)" : "0";
    o << "      { const int fa = " << fa << ", fb = " << fb << "; C = svb::cmul<R>(C, fb ? svb::csel<R>(fa, "
      << dref(tc + k, 2) << ", " << dref(tc + k, 3) << ") : svb::csel<R>(fa, " << dref(tc + k, 0)
      << ", " << dref(tc + k, 1) << ")); }\n";
  }
  for (int k = 0; k < h.nRR; ++k)  // only the quadrants whose factor is not exactly 1
    for (int q = 0; q < 4; ++q)
      if (!is1(rr[k].d[q])) {
        if (rr[k].d[q].x == -1 && rr[k].d[q].y == 0)
          o << "      svb::neg_quad<R, RB, " << (int)rr[k].ra << ", " << (int)rr[k].rb << ", " << q << ">(a);\n";
        else if (rr[k].d[q].x == 0 && (rr[k].d[q].y == 1 || rr[k].d[q].y == -1))
          o << "      svb::imul_quad<R, RB, " << (int)rr[k].ra << ", " << (int)rr[k].rb << ", " << q << ", "
            << (rr[k].d[q].y > 0 ? 1 : -1) << ">(a);\n";
        else
          o << "      svb::mul_quad<R, RB, " << (int)rr[k].ra << ", " << (int)rr[k].rb << ", " << q << ">(a, "
            << dref(rr + k, q) << ");\n";
      }
  if (prod) {
    for (int i = 0; i < RB; ++i) {
      const bool preal = prod[i].y == 0;
      o << "      const svb::cplx<R> E_" << i << " = ";
      if ((pro_scaled >> i) & 1u) o << "D1_" << i;
      else if (d1one[i]) o << cimm<R>(prod[i]);
      else if (preal) o << "svb::rmul<R>(" << hexf((double)prod[i].x, sizeof(R) == 4) << ", D1_" << i << ")";
      else o << "svb::cmul<R>(D1_" << i << ", " << cimm<R>(prod[i]) << ")";
      o << ";\n";
    }
    for (int v = 1; v < (1 << RB); ++v) {
      const int low = __builtin_ctz((unsigned)v);
      const int rest = v & (v - 1);
      if (d1one[low] && prod[low].y == 0)
        o << "      a[" << v << "] = svb::rmul<R>(E_" << low << ".x, a[" << rest << "]);\n";
      else
        o << "      a[" << v << "] = svb::cmul<R>(a[" << rest << "], E_" << low << ");\n";
    }
    o << "    }\n";
    return;
  }
  // fold D0 into C (unit-modulus entries: 1/D0 = conj(D0)), then apply
  bool need_c = !cone;
  for (int i = 0; i < RB; ++i)
    if (!d0one[i]) {
      if (!need_c) {
        o << "      svb::cplx<R> C = svb::mk<R>(R(1), R(0));\n";
        need_c = true;
      }
      o << "      C = svb::cmul<R>(C, D0_" << i << ");\n";
      creal = creal && d0real[i];
      if (!d1one[i]) {
        o << "      D1_" << i << " = svb::conj_mul<R>(D1_" << i << ", D0_" << i << ");\n";
        d1real[i] = d1real[i] && d0real[i];
      } else {
        o << "      svb::cplx<R> D1_" << i << " = svb::mk<R>(D0_" << i << ".x, -D0_" << i << ".y);\n";
        d1one[i] = false;
        d1real[i] = d0real[i];
      }
    }
  // complex factors: with two or more, one product per register index (a
  // product tree over the bits: F_v = F_(v - lowbit) * D1_lowbit, C folded into
  // F_0) replaces a complex multiply per factor per amplitude
  uint32_t cbits = 0;
  for (int i = 0; i < RB; ++i)
    if (!d1one[i] && !d1real[i]) cbits |= 1u << i;
  const bool cc = need_c && !creal;
  if (__builtin_popcount(cbits) + (cc ? 1 : 0) >= 2) {
    if (need_c && creal) o << "      svb::mul_all_r<R, RB>(a, C.x);\n";
    o << "      { svb::cplx<R> F[" << (1 << RB) << "];\n";
    for (int v = 0; v < (1 << RB); ++v) {
      const uint32_t act = (uint32_t)v & cbits;
      if (act == 0) {
        if (cc) o << "        F[" << v << "] = C;\n";
        continue;
      }
      if (act != (uint32_t)v) continue;  // F depends only on the active bits: reuse F[act]
      const int low = __builtin_ctz(act);
      const uint32_t rest = act & (act - 1);
      if (rest == 0 && !cc) o << "        F[" << v << "] = D1_" << low << ";\n";
      else o << "        F[" << v << "] = svb::cmul<R>(F[" << rest << "], D1_" << low << ");\n";
    }
    for (int v = 0; v < (1 << RB); ++v) {
      const uint32_t act = (uint32_t)v & cbits;
      if (act == 0 && !cc) continue;
      o << "        a[" << v << "] = svb::cmul<R>(a[" << v << "], F[" << act << "]);\n";
    }
    o << "      }\n";
    for (int i = 0; i < RB; ++i)
      if (!d1one[i] && d1real[i]) o << "      svb::mul_half_r<R, RB, " << i << ">(a, D1_" << i << ".x);\n";
  } else {
    if (need_c) {
      if (creal) o << "      svb::mul_all_r<R, RB>(a, C.x);\n";
      else o << "      svb::mul_all<R, RB>(a, C);\n";
    }
    for (int i = 0; i < RB; ++i)
      if (!d1one[i]) {
        if (d1real[i]) o << "      svb::mul_half_r<R, RB, " << i << ">(a, D1_" << i << ".x);\n";
        else o << "      svb::mul_half<R, RB, " << i << ">(a, D1_" << i << ");\n";
      }
  }
  o << "    }\n";
}

// One-round direct complex128 passes whose thread bits are the state's lowest
// qubits in order: each register row of a tile is one contiguous run, so the
// tile can leave through shared memory as bulk copies (SVB_BULK_ROWS, chosen
// at launch when the launch is direct).  SVB_BULK_ROWS=0 in the environment
// keeps register stores.
bool bulk_rows_eligible(const PassDev& pd, int rsize) {
  static const bool off = std::getenv("SVB_BULK_ROWS") && std::atoi(std::getenv("SVB_BULK_ROWS")) == 0;
  if (off || rsize != 8 || !direct_one_round(pd) || pd.perm_out || pd.perm_in) return false;
  const RoundDev& rd = pd.rounds[0];
  for (int b = 0; b < pd.m - pd.rb; ++b)
    if (pd.pos[rd.thr_local[b]] != b) return false;
  return true;
}

// Emit the straight-line Body of one pass.
template <typename R>
void emit_body(std::ostringstream& o, const Program& prog, int p, int RB, bool imm, PrologueCtx& pc) {
  const PassDev& pd = prog.passes[p];
  o << "    case " << p << ": {\n";
  // one-round direct passes: the uniform-slot sync (upipe_sync) goes right
  // before the first op that reads a tile-uniform factor
  const bool uin = uin_pass(pd);
  bool usynced = false;
  for (int k = 0; k < pd.nrounds; ++k) {
    const RoundDev& rd = pd.rounds[k];
    o << "    // round " << k << "\n"
      << "    svb::round_fixed<R, RB>(c, " << k << ", base, sFl, Fg);\n";
    // layout constants are known here: slot(v) = sFl ^ K[v] (GF(2)-linear
    // swizzle), global offset(v) = G[v]; immediates keep them out of registers
    uint32_t K[1 << 5];
    uint64_t G[1 << 5];
    K[0] = 0;
    G[0] = 0;
    for (int i = 0; i < RB; ++i)
      for (int v = 0; v < (1 << i); ++v) {
        K[v | (1 << i)] = K[v] ^ swz<R>(1u << rd.reg_local[i]);
        G[v | (1 << i)] = G[v] | (1ull << pd.pos[rd.reg_local[i]]);
      }
    if (k == 0) {  // direct first round (launch-time choice): preload() already filled a[]
      {
        std::ostringstream& P = *pc.pre;
        P << "    const svb::cplx<R>* g0 = c.state + Fg;\n    if (c.zero_input) {\n";
        for (int v = 0; v < (1 << RB); ++v)
          P << "      a[" << v << "] = svb::mk<R>((Fg | " << G[v] << "ull) == 0 ? R(1) : R(0), R(0));\n";
        P << "    } else {\n";
        if (pd.dmask) {  // support tracking: only written positions are read; the next tile's go to L2
          P << "      const bool tdead0 = (Fg & " << pd.dmask << "ull) != 0;\n";
          for (int v = 0; v < (1 << RB); ++v) {
            if (G[v] & pd.dmask) P << "      a[" << v << "] = svb::mk<R>(R(0), R(0));\n";
            else P << "      a[" << v << "] = tdead0 ? svb::mk<R>(R(0), R(0)) : __ldcs(g0 + " << G[v] << "ull);\n";
          }
          P << "      if (c.l2next && !tdead0) {\n"
               "        const svb::cplx<R>* gn = c.state + ((Fg & ~base) | c.next_base);\n";
          for (int v = 0; v < (1 << RB); ++v)
            if (!(G[v] & pd.dmask)) P << "        svb::prefetch_l2(gn + " << G[v] << "ull);\n";
          P << "      }\n";
        } else {
          for (int v = 0; v < (1 << RB); ++v) P << "      a[" << v << "] = __ldcs(g0 + " << G[v] << "ull);\n";
        }
        P << "    }\n";
      }
      o << "    if (!c.direct) {\n";
      if (pd.dmask) {  // never-written positions (support tracking) are zeros, not loaded
        o << "      const bool tdead0 = (Fg & " << pd.dmask << "ull) != 0;\n";
        for (int v = 0; v < (1 << RB); ++v) {
          if (G[v] & pd.dmask) o << "      a[" << v << "] = svb::mk<R>(R(0), R(0));\n";
          else o << "      a[" << v << "] = tdead0 ? svb::mk<R>(R(0), R(0)) : cur[sFl ^ " << K[v] << "u];\n";
        }
      } else {
        for (int v = 0; v < (1 << RB); ++v) o << "      a[" << v << "] = cur[sFl ^ " << K[v] << "u];\n";
      }
      o << "    }\n";
    } else {
      for (int v = 0; v < (1 << RB); ++v) o << "    a[" << v << "] = cur[sFl ^ " << K[v] << "u];\n";
    }
    if (k + 1 == pd.nrounds) o << "    svb::prefetch_next<R, RB, PassBody>(c);\n";
    // registers statically zero: round 0 of a support-tracked pass (never-written
    // positions), tracked through the leading pivot ops (any other op ends it)
    uint32_t zm = 0;
    if (k == 0 && pd.dmask && imm)
      for (int v = 0; v < (1 << RB); ++v)
        if (G[v] & pd.dmask) zm |= 1u << v;
    // product-state fusion (see emit_diag's prod): while round 0 starts from a
    // single live register (a[0]) and each leading pivot op expands it along a
    // new register bit, the ops are held back (deferred) with their ratios;
    // a following per-bit DIAG then builds the whole product in one tree
    const uint32_t nregs = 1u << RB, allv = (nregs >= 32 ? 0xffffffffu : (1u << nregs) - 1u);
    bool prod_ok = zm == (allv & ~1u) && !std::getenv("SVB_NO_PROD_FUSE");
    uint32_t prod_bits = 0;
    cplx<R> prodf[8];
    std::string deferred;
    auto zm_of = [&](uint32_t bits) {  // zero registers of a product over `bits`
      uint32_t z = 0;
      for (uint32_t v = 0; v < nregs; ++v)
        if (v & ~bits) z |= 1u << v;
      return z;
    };
    uint32_t off = rd.op_off;
    while (off < rd.op_end) {
      OpHdr h;
      std::memcpy(&h, prog.ops.data() + off, sizeof h);
      const uint32_t pay = off + (uint32_t)sizeof(OpHdr);
      const cplx<R>* coef = reinterpret_cast<const cplx<R>*>(prog.ops.data() + pay);
      bool fuse_diag = false;
      if (h.kind != OP_U1P && h.kind != OP_U1PR && !deferred.empty()) {
        if (h.kind == OP_DIAG && prod_bits == nregs - 1 && diag_per_bit_only<R>(prog.ops.data() + pay, RB)) {
          fuse_diag = true;
        } else {
          o << deferred;
        }
        deferred.clear();
        prod_ok = false;
      }
      std::string guard;
      if (h.fmask) {
        char buf[96];
        std::snprintf(buf, sizeof buf, "if ((Fg & 0x%llxull) == 0x%llxull) ", (unsigned long long)h.fmask,
                      (unsigned long long)h.fval);
        guard = buf;
      }
      const std::string cond = h.rmask ? "true" : "false";
      const std::string rm = std::to_string(h.rmask) + "u, " + std::to_string(h.rval) + "u";
      if (h.kind != OP_U1P && h.kind != OP_U1PR) zm = 0;  // zero tracking covers leading pivot ops only
      const std::streampos mark = o.tellp();
      switch (h.kind) {
        case OP_DIAG:
          pc.round = k;
          emit_diag<R>(o, prog.ops.data() + pay, pay, RB, imm, pc, fuse_diag ? prodf : nullptr);
          break;
        case OP_U1R:
          if (imm) {
            o << "    " << guard << "svb::u1_real_v<R, RB, " << h.a << ", " << cond << ">(a, "
              << hexf((double)coef[0].x, sizeof(R) == 4) << ", " << hexf((double)coef[1].x, sizeof(R) == 4) << ", "
              << hexf((double)coef[2].x, sizeof(R) == 4) << ", " << hexf((double)coef[3].x, sizeof(R) == 4) << ", "
              << rm << ");\n";
            break;
          }
          [[fallthrough]];
        case OP_U1X:
        case OP_U1:
        case OP_U1ANTI: {
          const char* fn = h.kind == OP_U1R ? "u1_real" : h.kind == OP_U1X ? "u1_rx" : h.kind == OP_U1 ? "u1_dense" : "u1_anti";
          if (imm) {  // constant local array: folded into immediates
            o << "    " << guard << "{ const svb::cplx<R> M[4] = {";
            for (int e = 0; e < 4; ++e) o << (e ? ", " : "") << cimm<R>(coef[e]);
            o << "}; svb::" << fn << "<R, RB, " << h.a << ", " << cond << ">(a, M, " << rm << "); }\n";
            break;
          }
          // structure-only: coefficients stay in the op payload (shared memory), so
          // circuits that differ only in angles share one compiled kernel
          o << "    " << guard << "svb::" << fn << "<R, RB, " << h.a << ", " << cond
            << ">(a, reinterpret_cast<const svb::cplx<R>*>(c.ops + " << pay << "), " << rm << ");\n";
          break;
        }
        case OP_U1P:
        case OP_U1PR: {
          const int pc0 = h.n & 1, pc1 = (h.n >> 1) & 1;
          if (imm && zm && !h.fmask) {
            auto rk = [](const cplx<R>& z) { return z.x == 0 && z.y == 0 ? 0 : z.y == 0 ? 1 : z.x == 0 ? 2 : 3; };
            const int rk0 = rk(coef[0]), rk1 = rk(coef[1]);
            // along a new bit with the live half as pivot of row 0 and the
            // other of row 1: a[v] stays, a[v | bit] = ratio1 * a[v]
            const bool expands = prod_ok && !((prod_bits >> h.a) & 1u) && pc0 == 0 && pc1 == 1 && zm == zm_of(prod_bits);
            if (!expands && !deferred.empty()) {
              o << deferred;
              deferred.clear();
            }
            if (!expands) prod_ok = false;
            std::ostringstream call;
            call << "    svb::u1_piv_z<R, RB, " << h.a << ", " << pc0 << ", " << pc1 << ", " << rk0 << ", " << rk1 << ", "
                 << zm << "u>(a, " << cimm<R>(coef[0]) << ", " << cimm<R>(coef[1]) << ");\n";
            if (expands) {
              prodf[h.a] = coef[1];
              prod_bits |= 1u << h.a;
              deferred += call.str();
            } else {
              o << call.str();
            }
            uint32_t nz = zm;  // zero outputs: both inputs zero, or (p zero and the ratio term zero)
            for (int v = 0; v < (1 << RB); ++v) {
              if (v & (1 << h.a)) continue;
              const int w = v | (1 << h.a);
              const bool z0 = (zm >> v) & 1u, z1 = (zm >> w) & 1u;
              const bool p0z = pc0 ? z1 : z0, o0z = pc0 ? z0 : z1, p1z = pc1 ? z1 : z0, o1z = pc1 ? z0 : z1;
              const bool y0z = p0z && (o0z || rk0 == 0), y1z = p1z && (o1z || rk1 == 0);
              nz = (nz & ~((1u << v) | (1u << w))) | (y0z ? 1u << v : 0u) | (y1z ? 1u << w : 0u);
            }
            zm = nz;
            break;
          }
          if (!deferred.empty()) {
            o << deferred;
            deferred.clear();
          }
          prod_ok = false;
          zm = 0;
          if (imm) {
            auto rk = [](const cplx<R>& z) { return z.x == 0 && z.y == 0 ? 0 : z.y == 0 ? 1 : z.x == 0 ? 2 : 3; };
            o << "    " << guard << "svb::u1_piv<R, RB, " << h.a << ", " << pc0 << ", " << pc1 << ", " << rk(coef[0])
              << ", " << rk(coef[1]) << ">(a, " << cimm<R>(coef[0]) << ", " << cimm<R>(coef[1]) << ");\n";
          } else {
            // (the pivot choice is part of the source: it depends on the
            // angles only near a singular pivot, |m_rr| < 2^-8 |m_r,1-r|)
            o << "    " << guard << "svb::u1_piv_p<R, RB, " << h.a << ", " << (h.n & 3) << ", "
              << (h.kind == OP_U1PR ? "true" : "false") << ">(a, reinterpret_cast<const svb::cplx<R>*>(c.ops + "
              << pay << "));\n";
          }
          break;
        }
        case OP_U2:
          if (imm) {
            o << "    " << guard << "{ const svb::cplx<R> M[16] = {";
            for (int e = 0; e < 16; ++e) o << (e ? ", " : "") << cimm<R>(coef[e]);
            o << "}; svb::u2_dense<R, RB, " << h.a << ", " << h.b << ">(a, M, " << rm << "); }\n";
            break;
          }
          o << "    " << guard << "svb::u2_dense<R, RB, " << h.a << ", " << h.b
            << ">(a, reinterpret_cast<const svb::cplx<R>*>(c.ops + " << pay << "), " << rm << ");\n";
          break;
        case OP_PERM2:
          if (imm) {
            int32_t src4[4];
            std::memcpy(src4, prog.ops.data() + pay, sizeof src4);
            const cplx<R>* ph = reinterpret_cast<const cplx<R>*>(prog.ops.data() + pay + 16);
            o << "    " << guard << "{ const int32_t S[4] = {" << src4[0] << ", " << src4[1] << ", " << src4[2] << ", "
              << src4[3] << "}; const svb::cplx<R> P[4] = {";
            for (int e = 0; e < 4; ++e) o << (e ? ", " : "") << cimm<R>(ph[e]);
            o << "}; svb::u2_perm<R, RB, " << h.a << ", " << h.b << ">(a, S, P, " << rm << "); }\n";
            break;
          }
          o << "    " << guard << "svb::u2_perm<R, RB, " << h.a << ", " << h.b
            << ">(a, reinterpret_cast<const int32_t*>(c.ops + " << pay
            << "), reinterpret_cast<const svb::cplx<R>*>(c.ops + " << (pay + 16) << "), " << rm << ");\n";
          break;
        default:
          throw Error(SVB_E_CUDA, "jit: unknown op kind");
      }
      off += h.bytes;
      if (uin && !usynced) {
        std::string all = o.str();
        if (all.find("c.uni", (size_t)mark) != std::string::npos) {
          all.insert((size_t)mark, "    svb::upipe_sync<R, RB>(c);\n");
          o.str(all);
          o.seekp(0, std::ios::end);
          usynced = true;
        }
      }
    }
    if (!deferred.empty()) o << deferred;  // the round ended inside the expansion
    if (uin && !usynced && k + 1 == pd.nrounds) {
      o << "    svb::upipe_sync<R, RB>(c);\n";
      usynced = true;
    }
    if (k + 1 == pd.nrounds && pd.zsum) o << "    svb::zsum_tile<R, RB>(c, a, base);\n";
    if (k + 1 < pd.nrounds) {
      for (int v = 0; v < (1 << RB); ++v) o << "    cur[sFl ^ " << K[v] << "u] = a[" << v << "];\n";
      o << "    __syncthreads();\n";
    } else if (pd.perm_out) {  // permuted store: every bit to its destination (see fuse_final_permutation)
      uint64_t PG[1 << 5];
      PG[0] = 0;
      for (int i = 0; i < RB; ++i)
        for (int v = 0; v < (1 << i); ++v) PG[v | (1 << i)] = PG[v] | (1ull << pd.dpos[rd.reg_local[i]]);
      o << "    { svb::cplx<R>* g0 = c.out + (c.pbase | c.pthr);\n";
      for (int v = 0; v < (1 << RB); ++v) o << "      __stcs(g0 + " << PG[v] << "ull, a[" << v << "]);\n";
      o << "    }\n";
    } else {
      const bool rows = bulk_rows_eligible(pd, (int)sizeof(R));
      if (rows) {
        // SVB_BULK_ROWS (decided at launch): register row v of the tile is one
        // contiguous run of nthr amplitudes at Fg - tid + G[v]; rows go through
        // shared memory and leave as bulk copies issued by threads 0..2^RB-1
        o << "#if SVB_BULK_ROWS\n"
             "    { svb::cplx<R>* stg = c.ring;\n"
             "      if (c.tid < " << (1 << RB) << "u) svb::bulk_wait_read();\n"
             "      __syncthreads();\n";
        for (int v = 0; v < (1 << RB); ++v) o << "      stg[" << v << " * c.nthr + c.tid] = a[" << v << "];\n";
        o << "      svb::fence_proxy_async_smem();\n"
             "      __syncthreads();\n"
             "      if (c.tid < " << (1 << RB) << "u) {\n"
             "        uint64_t go = 0;\n";
        for (int i = 0; i < RB; ++i) o << "        if (c.tid & " << (1u << i) << "u) go |= " << G[1 << i] << "ull;\n";
        o << "        svb::bulk_store_row(c.out + (Fg - c.tid) + go, stg + c.tid * c.nthr, c.nthr * (uint32_t)sizeof(svb::cplx<R>));\n"
             "      }\n"
             "    }\n"
             "#else\n";
      }
      o << "    { svb::cplx<R>* g0 = c.out + Fg;\n";  // == c.state unless perm_in
      for (int v = 0; v < (1 << RB); ++v) o << "      __stcs(g0 + " << G[v] << "ull, a[" << v << "]);\n";
      o << "    }\n";
      if (rows) o << "#endif\n";
    }
  }
  o << "    } break;\n";
  (void)RB;
}

}  // namespace

bool jit_available() {
  static Nvrtc nv;
  static Driver dr;
  return nv.ok && dr.ok;
}

// Source of one pass kernel (skeleton + straight-line body).
// Programs on at least this many qubits get coefficients as immediates (a
// one-off compile is negligible next to their passes); smaller ones get
// structure-only code that circuits differing only in angles share.
constexpr int kImmMinQubits = kJitImmMinQubits;

// `nslots`: per-thread prologue slots (shared memory, [slot][thread]);
// `imm`: coefficients are immediates, so only the uniform DIAG payloads are
// staged in shared memory (ops_mode 1).
template <typename R> std::string jit_source_pass(const Program& prog, int p, int* nslots, bool* imm_out) {
  const int RB = prog.passes[p].rb;
  std::ostringstream body, pro, pre;
  PrologueCtx pc;
  pc.o = &pro;
  pc.pre = &pre;
  const PassDev& pd0 = prog.passes[p];
  const bool imm = prog.n >= kImmMinQubits;  // (not m + nout: support tracking shrinks nout)
  emit_body<R>(body, prog, p, RB, imm, pc);
  if (nslots) *nslots = pc.nslots;
  if (imm_out) *imm_out = imm;
  std::ostringstream o;
  if (const char* e = std::getenv("SVB_UPIPE_AHEAD")) o << "#define SVB_UPIPE_AHEAD " << std::atoi(e) << "\n";
  if (const char* e = std::getenv("SVB_UWAIT_FIRST")) o << "#define SVB_UWAIT_FIRST " << std::atoi(e) << "\n";
  if (const char* e = std::getenv("SVB_UIN")) o << "#define SVB_UIN " << (std::atoi(e) != 0 ? 1 : 0) << "\n";
  if (const char* e = std::getenv("SVB_UGROUP")) o << "#define SVB_UGROUP " << std::max(1, std::atoi(e)) << "\n";
  if (const char* e = std::getenv("SVB_UPIPE_PROBE")) o << "#define SVB_UPIPE_PROBE " << std::atoi(e) << "\n";
  if (const char* e = std::getenv("SVB_HOIST")) o << "#define SVB_HOIST " << std::max(1, std::atoi(e)) << "\n";
  o << "#include \"device_core.cuh\"\nusing R = " << (sizeof(R) == 8 ? "double" : "float") << ";\n";
  // tile loads with the layout's offsets as immediates (see issue_tile)
  std::ostringstream iss;
  {
    const int m = pd0.m;
    const uint32_t nthr = 1u << (m - RB);
    const int kPer = sizeof(cplx<R>) == 16 ? 1 : 2;
    int lo_bits = 0;
    while ((1u << lo_bits) < nthr) ++lo_bits;
    lo_bits += (kPer == 2 ? 1 : 0);
    const uint32_t nld = (1u << m) / (nthr * (uint32_t)kPer);
    iss << "  template <typename R, int RB>\n"
           "  __device__ static __forceinline__ void issue(const svb::PassCtx<R, RB>& c, uint64_t base, "
           "svb::cplx<R>* dst) {\n"
           "    if (c.zero_input) { svb::issue_tile<R, RB>(c, base, dst); return; }\n"
           "    const svb::cplx<R>* src = c.state + (base | c.ld_tid);\n"
           "    const uint32_t s0 = c.sd_tid;\n";
    // support tracking (PassDev::dmask): never-written positions load as zeros;
    // the k part of the offset is known here, the thread part at run time
    uint64_t tmask = 0;
    for (int l = 0; l < lo_bits; ++l) tmask |= 1ull << pd0.pos[l];
    const uint64_t dm_thr = pd0.dmask & tmask;
    if (dm_thr) iss << "    const bool tdead = (c.ld_tid & " << dm_thr << "ull) != 0;\n";
    const int32_t* lpos = pd0.perm_in ? pd0.ipos : pd0.pos;  // input positions (perm_in: see PassDev)
    for (uint32_t k = 0; k < nld; ++k) {
      const uint32_t j = ld_order_local(pd0, k * nthr * (uint32_t)kPer);
      uint64_t g = 0;
      for (int l = 0; l < m; ++l)
        if ((j >> l) & 1u) g |= 1ull << lpos[l];
      // never-written positions are not stored at all: round 0 of a pass with a
      // dmask takes them as constant zeros (emit_body), later rounds read what
      // round 0 wrote
      if (g & pd0.dmask) {
        continue;
      } else if (dm_thr) {
        iss << "    if (!tdead) svb::cp_async16(dst + (s0 ^ " << swz<R>(j) << "u), src + " << g << "ull);\n";
      } else {
        iss << "    svb::cp_async16(dst + (s0 ^ " << swz<R>(j) << "u), src + " << g << "ull);\n";
      }
    }
    iss << "  }\n";
  }
  o << "struct PassBody {\n"
       "  template <typename R, int RB> struct State {};\n"
    << iss.str()
    << "  template <typename R, int RB>\n"
       "  __device__ static __forceinline__ void prologue(const svb::PassCtx<R, RB>& c, State<R, RB>& st) {\n"
    << pro.str() << "    (void)c; (void)st;\n  }\n"
       "  template <typename R, int RB>\n"
       "  __device__ static __forceinline__ void preload(const svb::PassCtx<R, RB>& c, svb::cplx<R>* a, "
       "uint64_t base) {\n"
       "    uint32_t sFl; uint64_t Fg;\n    svb::round_fixed<R, RB>(c, 0, base, sFl, Fg); (void)sFl;\n"
    << pre.str() << "  }\n"
       "  template <typename R, int RB>\n"
       "  __device__ static __forceinline__ void tile(int pass, const svb::PassCtx<R, RB>& c, svb::cplx<R>* a, "
       "svb::cplx<R>* cur, uint64_t base, const State<R, RB>& st) {\n"
       "    uint32_t sFl; uint64_t Fg;\n    (void)st;\n    switch (0) {\n";
  std::string b = body.str();
  const std::string from = "    case " + std::to_string(p) + ": {";
  const size_t at = b.find(from);
  if (at != std::string::npos) b.replace(at, from.size(), "    case 0: {");
  o << b << "    default: break;\n    }\n    (void)pass;\n  }\n};\n";
  const int minb = (sizeof(R) == 8 && direct_one_round(pd0)) ? direct_min_blocks() : pass_min_blocks_of((int)sizeof(R), RB);
  // bulk row stores: the staging tile leaves room for two CTAs per SM
  const std::string minb_s = bulk_rows_eligible(pd0, (int)sizeof(R))
                                 ? "(SVB_BULK_ROWS ? " + std::to_string(pass_min_blocks_of((int)sizeof(R), RB)) + " : " +
                                       std::to_string(minb) + ")"
                                 : std::to_string(minb);
  o << "extern \"C\" __global__ void __launch_bounds__(" << (1 << (pass_tile_m((int)sizeof(R), RB) - RB)) << ", " << minb_s
    << ") svb_jit(svb::cplx<R>* state, svb::cplx<R>* out, "
       "const svb::PassDev* __restrict__ pdg, const uint8_t* __restrict__ ops_g, uint32_t ntiles, int pass, "
       "int zero_input, int stages) {\n"
       "  svb::pass_kernel<R, "
    << RB << ", PassBody, " << zsm_pass(pd0) << ", " << (uin_pass(pd0) ? 1 : 0) << ", " << (pd0.perm_in ? 1 : 0)
    << ">(state, out, pdg, ops_g, ntiles, pass, zero_input, stages, " << (imm ? 1 : 0) << ", "
    << pc.nslots << ");\n}\n";
  return o.str();
}

uint64_t fnv1a(const std::string& s, uint64_t h = 1469598103934665603ull) {
  for (unsigned char ch : s) {
    h ^= ch;
    h *= 1099511628211ull;
  }
  return h;
}

std::string cache_dir() {
  const char* env = std::getenv("SVB_JIT_CACHE");
  if (env) return env;
  const char* home = std::getenv("HOME");
  return std::string(home ? home : "/tmp") + "/.cache/svb_jit";
}

// NVRTC -> cubin; empty on failure (log in *log).
static std::vector<char> jit_compile(const std::string& src, std::string* log) {
  static Nvrtc nv;
  if (!nv.ok) {
    if (log) *log = "libnvrtc not found";
    return {};
  }
  void* prog_h = nullptr;
  const char* hdr_src[] = {svb_device_core_src};
  const char* hdr_name[] = {"device_core.cuh"};
  if (nv.create(&prog_h, src.c_str(), "svb_jit.cu", 1, hdr_src, hdr_name) != 0) return {};
  std::vector<const char*> opts = {"--gpu-architecture=sm_100a", "-std=c++17", "-lineinfo"};
  static const std::string extra = std::getenv("SVB_JIT_OPTS") ? std::getenv("SVB_JIT_OPTS") : "";
  if (!extra.empty()) opts.push_back(extra.c_str());
  int rc = nv.compile(prog_h, (int)opts.size(), opts.data());
  if (rc != 0) {
    size_t n = 0;
    nv.log_size(prog_h, &n);
    std::string logs(n, '\0');
    nv.log(prog_h, &logs[0]);
    nv.destroy(&prog_h);
    if (log) *log = logs;
    return {};
  }
  size_t n = 0;
  nv.cubin_size(prog_h, &n);
  std::vector<char> cubin(n);
  nv.cubin(prog_h, cubin.data());
  nv.destroy(&prog_h);
  return cubin;
}

// Keep the in-memory caches bounded (LRU).  Programs are dropped freely;
// modules of this device are unloaded only after a device synchronisation
// with every launcher excluded, and every program entry is dropped with them
// (entries hold CUfunctions of the modules).
void evict_lru(Driver& dr, int dev) {
  {
    std::lock_guard<std::mutex> lk(g_mu);
    if (g_prog.size() > kMaxPrograms) {
      std::vector<std::pair<uint64_t, Key128>> age;
      for (auto& kv : g_prog) age.push_back({kv.second.last_use, kv.first});
      std::sort(age.begin(), age.end(), [](const auto& x, const auto& y) { return x.first < y.first; });
      for (size_t i = 0; i < age.size() / 2; ++i) g_prog.erase(age[i].second);
    }
    if (g_cache.size() <= kMaxModules) return;
  }
  std::unique_lock<std::shared_mutex> ex(g_launch_mu);
  std::lock_guard<std::mutex> lk(g_mu);
  if (g_cache.size() <= kMaxModules) return;
  const std::string pre = std::to_string(dev) + ":";
  std::vector<std::pair<uint64_t, std::string>> age;
  for (auto& kv : g_cache)
    if (kv.first.compare(0, pre.size(), pre) == 0) age.push_back({kv.second.last_use, kv.first});
  if (age.empty()) return;
  std::sort(age.begin(), age.end(), [](const auto& x, const auto& y) { return x.first < y.first; });
  cudaDeviceSynchronize();
  cudaGetLastError();
  g_prog.clear();
  for (size_t i = 0; i < age.size() / 2; ++i) {
    auto it = g_cache.find(age[i].second);
    if (dr.unload) dr.unload(it->second.mod);
    g_cache.erase(it);
  }
}

// Ring depth of a pass's launch: pass_stages, and the direct first round for
// support-tracked passes (few live loads per tile, no ring barrier); for full
// passes only on request (load latency exposed)
template <typename R> static int launch_stages(const PassDev& pd, uint32_t staged, int nslots) {
  int stages = pass_stages<R>(pd.rb, pd.m, staged, pd.ndiag, nslots, zsm_pass(pd));
  if (stages == 1 && pd.direct && !pd.perm_in && (pd.dmask || std::getenv("SVB_DIRECT"))) stages = 0;
  return stages;
}
// bulk row stores need the direct launch (the tile region is free for staging)
template <typename R> static bool launch_bulk(const PassDev& pd, int stages) {
  return stages == 0 && bulk_rows_eligible(pd, (int)sizeof(R));
}

template <typename R>
bool jit_launch_passes(cplx<R>* state, cplx<R>* out, const Program& prog, const PassDev* dpass, const uint8_t* dops,
                       cudaStream_t st, ProgramStats* stats, int nsm, bool zero_input) {
  static Driver dr;
  if (!dr.ok || prog.passes.empty()) return false;
  const int RB = prog.passes[0].rb;
  static const bool jprof = std::getenv("SVB_JIT_PROFILE") != nullptr;
  const auto jt0 = std::chrono::steady_clock::now();
  auto jms = [&] { return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - jt0).count(); };
  double j_evict = 0, j_gen = 0, j_lookup = 0;
  int dev = 0;
  SVB_CUDA(cudaGetDevice(&dev));
  evict_lru(dr, dev);
  std::shared_lock<std::shared_mutex> launch_lk(g_launch_mu);
  if (jprof) j_evict = jms();
  const size_t np = prog.passes.size();
  std::vector<std::string> srcs(np), keys(np);
  std::vector<CUfunction> fns(np, nullptr);
  std::vector<int> nslots(np, 0);
  std::vector<uint32_t> staged(np, 0);
  // the engine source's hash, once per process (a byte-serial pass over ~90 KB
  // on every apply was 80 us of host time before the first launch)
  static const uint64_t salt = fnv1a(svb_device_core_src, fnv1a("svb-jit-v1 sm_100a"));
  Key128 pkey{salt ^ (uint64_t)dev, 0x243F6A8885A308D3ull + sizeof(R)};
  mix_bytes(pkey, prog.passes.data(), prog.passes.size() * sizeof(PassDev));
  mix_bytes(pkey, prog.ops.data(), prog.ops.size());
  bool hit = false;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = g_prog.find(pkey);
    if (it != g_prog.end()) {
      it->second.last_use = ++g_tick;
      fns = it->second.fns;
      nslots = it->second.nslots;
      staged = it->second.staged;
      hit = true;
    }
  }
  std::vector<size_t> todo;
  if (!hit) {
    // sources are generated without the cache lock (workers of the batch
    // executor generate theirs in parallel); only the lookups are locked
    for (size_t p = 0; p < np; ++p) {
      bool imm = false;
      srcs[p] = jit_source_pass<R>(prog, (int)p, &nslots[p], &imm);
      const PassDev& pd = prog.passes[p];
      staged[p] = pd.ops_bytes;
      if (imm) {  // only the uniform DIAG payloads are staged
        staged[p] = 0;
        for (int d = 0; d < pd.ndiag; ++d) {
          OpHdr h;
          std::memcpy(&h, prog.ops.data() + pd.diag_off[d] - sizeof(OpHdr), sizeof h);
          staged[p] += h.bytes - (uint32_t)sizeof(OpHdr);
        }
      }
      if (pass_smem<R>(pd.rb, pd.m, staged[p], pd.ndiag, nslots[p], 1, zsm_pass(pd)) > kSmemMaxPerCTA) return false;
      {  // the launch's ring depth, round count and lazy-input flag, compiled in
         // (pass_kernel's STAGES / NR / ZIN), and the bulk row stores
        const int stg = launch_stages<R>(pd, staged[p], nslots[p]);
        if (launch_bulk<R>(pd, stg)) srcs[p].insert(0, "#define SVB_BULK_ROWS 1\n");
        const int zin = (zero_input && p == 0) ? 1 : 0;
        const std::string from = "(state, out, pdg, ops_g, ntiles, pass, zero_input, stages,";
        const size_t at = srcs[p].rfind(from);
        const size_t lt = at == std::string::npos ? at : srcs[p].rfind(">", at);
        if (lt != std::string::npos)
          srcs[p].insert(lt, ", " + std::to_string(stg) + ", " + std::to_string(pd.nrounds) + ", " + std::to_string(zin));
      }
      char buf[40];
      std::snprintf(buf, sizeof buf, "%016llx", (unsigned long long)fnv1a(srcs[p], salt));
      keys[p] = std::to_string(dev) + ":" + buf;
    }
    if (jprof) j_gen = jms();
    std::lock_guard<std::mutex> lk(g_mu);
    for (size_t p = 0; p < np; ++p) {
      auto it = g_cache.find(keys[p]);
      if (it != g_cache.end()) {
        fns[p] = it->second.fns[0];
        it->second.last_use = ++g_tick;
      } else {
        todo.push_back(p);
      }
    }
  }
  if (jprof) j_lookup = jms();
  // Asynchronous mode (the batch executor): kernels not compiled yet are
  // compiled by background threads while this program runs on the
  // interpreter; later programs of the same structure pick them up.
  if (!todo.empty() && t_async_jit) {
    std::vector<std::pair<std::string, std::string>> jobs;  // (key, source)
    {
      std::lock_guard<std::mutex> lk(g_mu);
      for (size_t p : todo)
        if (!g_cache.count(keys[p]) && g_inflight.insert(keys[p]).second) jobs.push_back({keys[p], srcs[p]});
    }
    for (auto& jb : jobs) {
      std::thread([jb, dev, drp = &dr] {
        cudaSetDevice(dev);
        const std::string dir = cache_dir();
        const std::string path = dir + "/" + jb.first.substr(jb.first.find(':') + 1) + ".cubin";
        std::vector<char> cubin;
        if (FILE* f = std::fopen(path.c_str(), "rb")) {
          std::fseek(f, 0, SEEK_END);
          const long sz = std::ftell(f);
          std::fseek(f, 0, SEEK_SET);
          cubin.resize(sz > 0 ? (size_t)sz : 0);
          if (sz <= 0 || std::fread(cubin.data(), 1, (size_t)sz, f) != (size_t)sz) cubin.clear();
          std::fclose(f);
        }
        if (cubin.empty()) {
          std::string log;
          cubin = jit_compile(jb.second, &log);
          if (!cubin.empty()) {
            std::string mk = "mkdir -p '" + dir + "' 2>/dev/null";
            if (std::system(mk.c_str()) != 0) { /* best effort */ }
            const std::string tmp = path + ".tmp" + std::to_string((unsigned long long)(uintptr_t)&cubin);
            if (FILE* f = std::fopen(tmp.c_str(), "wb")) {
              const bool ok = std::fwrite(cubin.data(), 1, cubin.size(), f) == cubin.size();
              std::fclose(f);
              if (ok) std::rename(tmp.c_str(), path.c_str());
              else std::remove(tmp.c_str());
            }
          }
        }
        Module m;
        CUfunction fn = nullptr;
        const bool ok = !cubin.empty() && drp->load(&m.mod, cubin.data()) == CUDA_SUCCESS &&
                        drp->getfn(&fn, m.mod, "svb_jit") == CUDA_SUCCESS;
        std::lock_guard<std::mutex> lk(g_mu);
        if (ok) {
          m.fns.push_back(fn);
          m.last_use = ++g_tick;
          g_cache.emplace(jb.first, m);
        }
        g_inflight.erase(jb.first);
      }).detach();
    }
    return false;
  }
  // one compiler per kernel source: threads that need a source another thread
  // is compiling wait for it (the batch executor's workers meet the same
  // structures at the same time), then find it in g_cache
  std::vector<std::unique_lock<std::mutex>> key_locks;
  if (!todo.empty()) {
    std::vector<std::pair<std::string, std::shared_ptr<std::mutex>>> ks;
    {
      std::lock_guard<std::mutex> lk(g_mu);
      for (size_t p : todo) {
        auto& m = g_key_locks[keys[p]];
        if (!m) m = std::make_shared<std::mutex>();
        ks.push_back({keys[p], m});
      }
    }
    std::sort(ks.begin(), ks.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
    ks.erase(std::unique(ks.begin(), ks.end(), [](const auto& a, const auto& b) { return a.first == b.first; }),
             ks.end());
    for (auto& k : ks) key_locks.emplace_back(*k.second);
    std::lock_guard<std::mutex> lk(g_mu);
    std::vector<size_t> still;
    for (size_t p : todo) {
      auto it = g_cache.find(keys[p]);
      if (it != g_cache.end()) {
        fns[p] = it->second.fns[0];
        it->second.last_use = ++g_tick;
      } else {
        still.push_back(p);
      }
    }
    todo.swap(still);
  }
  if (!todo.empty()) {
    // disk cache, then NVRTC for the rest (one thread per pass kernel)
    const std::string dir = cache_dir();
    std::vector<std::vector<char>> cubins(np);
    std::vector<size_t> compile;
    for (size_t p : todo) {
      const std::string path = dir + "/" + keys[p].substr(keys[p].find(':') + 1) + ".cubin";
      FILE* f = std::fopen(path.c_str(), "rb");
      if (f) {
        std::fseek(f, 0, SEEK_END);
        long sz = std::ftell(f);
        std::fseek(f, 0, SEEK_SET);
        cubins[p].resize(sz > 0 ? (size_t)sz : 0);
        if (sz <= 0 || std::fread(cubins[p].data(), 1, (size_t)sz, f) != (size_t)sz) cubins[p].clear();
        std::fclose(f);
      }
      if (cubins[p].empty()) compile.push_back(p);
    }
    std::vector<std::string> logs(np);
    std::vector<std::thread> th;
    for (size_t p : compile) th.emplace_back([&, p] { cubins[p] = jit_compile(srcs[p], &logs[p]); });
    for (auto& t : th) t.join();
    if (!compile.empty()) {
      std::string mk = "mkdir -p '" + dir + "' 2>/dev/null";
      if (std::system(mk.c_str()) != 0) { /* cache is best effort */ }
    }
    for (size_t p : compile) {
      if (cubins[p].empty()) {
        if (std::getenv("SVB_JIT_STRICT"))  // tests: a compile failure must not hide behind the interpreter
          throw Error(SVB_E_CUDA, "JIT compile failed:\n" + logs[p]);
        std::fprintf(stderr, "[svb] JIT compile failed; using the interpreter kernel\n%s\n", logs[p].c_str());
        return false;
      }
      const std::string path = dir + "/" + keys[p].substr(keys[p].find(':') + 1) + ".cubin";
      const std::string tmp = path + ".tmp" + std::to_string((unsigned long long)(uintptr_t)&cubins[p]);
      FILE* f = std::fopen(tmp.c_str(), "wb");
      if (f) {
        const bool ok = std::fwrite(cubins[p].data(), 1, cubins[p].size(), f) == cubins[p].size();
        std::fclose(f);
        if (ok) std::rename(tmp.c_str(), path.c_str());
        else std::remove(tmp.c_str());
      }
    }
    std::lock_guard<std::mutex> lk(g_mu);
    for (size_t p : todo) {
      Module m;
      if (dr.load(&m.mod, cubins[p].data()) != CUDA_SUCCESS) return false;
      CUfunction f;
      if (dr.getfn(&f, m.mod, "svb_jit") != CUDA_SUCCESS) return false;
      m.fns.push_back(f);
      m.last_use = ++g_tick;
      fns[p] = f;
      g_cache.emplace(keys[p], m);
    }
  }
  if (!hit) {
    std::lock_guard<std::mutex> lk(g_mu);
    g_prog.emplace(pkey, ProgKernels{fns, nslots, staged, ++g_tick});
  }
  cplx<R>* cur = state;
  cplx<R>* other = out;
  for (size_t p = 0; p < np; ++p) {
    const PassDev& pd = prog.passes[p];
    const uint64_t tiles = 1ull << pd.nout;
    const unsigned threads = 1u << (pd.m - RB);
    int stages = launch_stages<R>(pd, staged[p], nslots[p]);
    const unsigned smem = pass_smem<R>(pd.rb, pd.m, staged[p], pd.ndiag, nslots[p], stages, zsm_pass(pd), pd.nrounds,
                                       launch_bulk<R>(pd, stages) ? 1 : 0);
    int per_sm = stages <= 1 ? pass_min_blocks_of((int)sizeof(R), pd.rb) : 1;
    if (sizeof(R) == 8 && stages == 0 && direct_one_round(pd) &&
        (uint64_t)direct_min_blocks() * (smem + kSmemReservedPerCTA + kPassStaticSmem) <= kSmemPerSM)
      per_sm = direct_min_blocks();
    const unsigned grid = (unsigned)std::min<uint64_t>(tiles, (uint64_t)nsm * per_sm);
    static const bool trace = std::getenv("SVB_TRACE") != nullptr;
    if (trace)
      std::fprintf(stderr, "[svb] jit pass %zu: m=%d rounds=%d stages=%d grid=%u smem=%u staged=%u ndiag=%d slots=%d\n",
                   p, pd.m, pd.nrounds, stages, grid, smem, staged[p], pd.ndiag, nslots[p]);
    CUfunction f = fns[p];
    // per-function attributes, set once per (function, carveout) in the
    // process (changing attributes of a function other threads are launching
    // costs driver synchronisation: the batch executor's fresh worker threads
    // must not redo it); the shared memory limit is always the maximum;
    // three-CTA one-round passes use little shared memory: leave L1 room for their spills
    const int carve = per_sm == direct_min_blocks() ? 60 : 100;
    {
      static std::mutex attr_mu;
      static std::unordered_map<CUfunction, int> configured;
      std::lock_guard<std::mutex> lk(attr_mu);
      auto cf = configured.find(f);
      if (cf == configured.end() || cf->second != carve) {
        if (dr.setattr(f, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, (int)kSmemMaxPerCTA) != CUDA_SUCCESS)
          throw Error(SVB_E_CUDA, "jit: cannot set shared memory size");
        dr.setattr(f, CU_FUNC_ATTRIBUTE_PREFERRED_SHARED_MEMORY_CARVEOUT, carve);
        configured[f] = carve;
      }
    }
    // perm_in / perm_out passes write the other buffer, which then holds the state
    cplx<R>* s = cur;
    cplx<R>* so = (pd.perm_in || pd.perm_out) ? other : cur;
    if (so != s) std::swap(cur, other);
    const PassDev* pdp = dpass + p;
    const uint8_t* ob = dops;
    uint32_t nt = (uint32_t)tiles;
    int pass = 0;
    int zin = (zero_input && p == 0) ? 1 : 0;
    void* args[] = {&s, &so, &pdp, &ob, &nt, &pass, &zin, &stages};
    Profiler* pf = (stats->prof && stats->prof->on) ? stats->prof : nullptr;
    if (pf) pf->begin(st, 0, pass_hbm_bytes<R>(pd, zin != 0), (int)p);
    if (dr.launch(f, grid, 1, 1, threads, 1, 1, smem, (CUstream)st, args, nullptr) != CUDA_SUCCESS)
      throw Error(SVB_E_CUDA, "jit: kernel launch failed");
    if (pf) pf->end(st);
    stats->passes += 1;
    stats->launches += 1;
  }
  if (jprof)
    std::fprintf(stderr, "[svb] jit_launch: evict+lock %.3f gen %.3f lookup %.3f total %.3f ms (hit %d)\n", j_evict, j_gen,
                 j_lookup, jms(), hit ? 1 : 0);
  return true;
}

void jit_set_async(bool on) { t_async_jit = on; }

template bool jit_launch_passes<float>(cplx<float>*, cplx<float>*, const Program&, const PassDev*, const uint8_t*, cudaStream_t,
                                       ProgramStats*, int, bool);
template bool jit_launch_passes<double>(cplx<double>*, cplx<double>*, const Program&, const PassDev*, const uint8_t*, cudaStream_t,
                                        ProgramStats*, int, bool);

}  // namespace svb

using namespace svb;

// Host-only check of the JIT path (no GPU needed): schedule, generate and
// NVRTC-compile the specialised kernels of a gate program.  Returns SVB_OK and
// the cubin size, or an error with the compiler log in svb_last_error-like buf.
extern "C" int svb_jit_check(int n, int precision, const svb_gate* gates, int ng, int64_t* cubin_bytes, char* log,
                             int log_cap) {
  try {
    const bool zero_start = (precision & 0x100) != 0;  // flag bit: schedule for a lazy |0...0> input
    const bool zsum = (precision & 0x200) != 0;        // flag bit: last pass accumulates fused <Z>
    precision &= 0xff;
    SchedOptions o = default_options(precision, n, true);
    o.zero_start = zero_start;
    std::vector<std::string> srcs;
    if (precision == SVB_C128) {
      Program p = build_program<double>(n, gates, ng, o);
      if (zsum && !p.passes.empty()) p.passes.back().zsum = 1;
      for (size_t k = 0; k < p.passes.size(); ++k) srcs.push_back(jit_source_pass<double>(p, (int)k, nullptr, nullptr));
      if (std::getenv("SVB_TRACE"))
        for (const PassDev& pd : p.passes)
          std::fprintf(stderr, "[svb] jit_check pass: m=%d rounds=%d ndiag=%d nitems=%d ops_bytes=%u dmask=%llx\n", pd.m,
                       pd.nrounds, pd.ndiag, pd.nitems, pd.ops_bytes, (unsigned long long)pd.dmask);
    } else {
      Program p = build_program<float>(n, gates, ng, o);
      if (zsum && !p.passes.empty()) p.passes.back().zsum = 1;
      for (size_t k = 0; k < p.passes.size(); ++k) srcs.push_back(jit_source_pass<float>(p, (int)k, nullptr, nullptr));
    }
    // passes with a bulk-row-store epilogue also compile in that variant
    // (the launch chooses it when the pass runs direct)
    for (size_t k = 0, n0 = srcs.size(); k < n0; ++k)
      if (srcs[k].find("#if SVB_BULK_ROWS") != std::string::npos) srcs.push_back("#define SVB_BULK_ROWS 1\n" + srcs[k]);
    if (std::getenv("SVB_JIT_DUMP") && !srcs.empty()) {
      FILE* f = std::fopen(std::getenv("SVB_JIT_DUMP"), "w");
      if (f) {
        for (auto& x : srcs) std::fputs(x.c_str(), f);
        std::fclose(f);
      }
    }
    if (std::getenv("SVB_JIT_NOCOMPILE")) {  // timing of source generation alone
      *cubin_bytes = 0;
      for (auto& x : srcs) *cubin_bytes += (int64_t)x.size();
      return SVB_OK;
    }
    std::vector<std::vector<char>> cubins(srcs.size());
    std::vector<std::string> logs(srcs.size());
    std::vector<std::thread> th;
    for (size_t k = 0; k < srcs.size(); ++k) th.emplace_back([&, k] { cubins[k] = jit_compile(srcs[k], &logs[k]); });
    for (auto& t : th) t.join();
    int64_t total = 0;
    for (size_t k = 0; k < srcs.size(); ++k) {
      if (cubins[k].empty()) {
        if (log && log_cap > 0) std::snprintf(log, (size_t)log_cap, "%s", logs[k].c_str());
        *cubin_bytes = total;
        return SVB_E_CUDA;
      }
      total += (int64_t)cubins[k].size();
    }
    *cubin_bytes = total;
    return SVB_OK;
  } catch (const Error& e) {
    if (log && log_cap > 0) std::snprintf(log, (size_t)log_cap, "%s", e.what());
    return e.code;
  }
}
