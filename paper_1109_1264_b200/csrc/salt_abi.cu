// salt_abi.cu — libsalt.so: the C ABI declared in include/salt.h.
//
// Host runtime around the fused kernels of salt_expr.cuh:
//   * signature parsing / validation (postfix, see salt.h),
//   * the kernel table: compiled-in (AOT, sm_100a) instantiations for the
//     trees the reference's named ops and the BASELINE configs use, plus an
//     NVRTC JIT that instantiates the SAME template for any other tree and
//     caches the cubin per signature and the module per device,
//   * launch geometry (persistent grid = SMs x resident CTAs),
//   * deterministic reductions (per-CTA double-double partials, last-CTA
//     combine) and the multi-device finish,
//   * the host-buffer streaming path (H2D / kernel / D2H pipelined over
//     three streams) used for end-to-end evaluation of host vectors.
//
// Reference anchors (pkg/src/lanevec/): engine.py:243-264 (assign loop),
// :267-292 (reduce loop), expressions.py:392-395 (commit), :457-480 (sum).
#include <cuda.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <sys/stat.h>
#include <unistd.h>

#include <atomic>
#include <chrono>
#include <condition_variable>
#include <deque>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <sstream>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <unordered_map>
#include <unordered_set>
#include <vector>

#include "../../include/salt.h"
#include "salt_expr.cuh"
#include "salt_interp.cuh"

namespace {

using salt::i64;

constexpr int kBlock = 256;
static_assert(SALT_WORKSPACE_TICKET_BYTES == salt::WsLayout::group_partials,
              "salt.h ticket prefix must match the kernel workspace layout");
// 256-bit vectors in flight per leaf per thread.  2 for assignments; 4 for
// pure reductions unless f64 with two or more leaves (profiles/
// r01_reduce_unroll_sweep.txt: nrm2 f64 6.72 -> 7.13 TB/s at 2^28 and
// +11 % at 2^24, sdot +25 % at 2^24; ddot is best at 2: TwoSum accumulation
// of two f64 streams needs the registers).
constexpr int unroll_for(int mode, int nl, int elem_bytes) {
  return mode == salt::MODE_REDUCE && (elem_bytes == 4 || nl <= 1) ? 4 : 2;
}
constexpr int kUnrollScalar = 4;  // V == 1 fallback (misaligned operands)
// Reductions: tiles (of BLOCK*UNR vectors) per CTA, so that every CTA
// streams ~64 KiB before paying its partial/ticket epilogue: 4 tiles for
// one-leaf trees (nrm2, sum), 2 for two or more leaves (dot, fused axpy->dot).
// SALT_REDUCE_TILES overrides it (tuning only; read once).
// Assignments: one tile per CTA (SALT_ASSIGN_TILES overrides; tuning only).
// SALT_UNROLL=U (tuning only): every vector kernel is JIT-built with UNR=U
// instead of the compiled-in choice.
int tuning_unroll() {
  static const int env = [] {
    const char* e = getenv("SALT_UNROLL");
    return e ? atoi(e) : 0;
  }();
  return env;
}
// SALT_JIT_MINB=B (tuning only): JIT-build every vector kernel with
// __launch_bounds__(256, B), i.e. registers capped for B CTAs per SM.
int tuning_minb() {
  static const int env = [] {
    const char* e = getenv("SALT_JIT_MINB");
    return e ? atoi(e) : 0;
  }();
  return env;
}

// Reductions whose tiles fit max_cluster() CTAs x cluster_tiles() run as
// ONE thread-block cluster (SALT_CLUSTER = max CTAs, 0 disables, <= 16;
// SALT_CLUSTER_TILES = tiles per CTA at most; tuning only).
int max_cluster() {
  static const int env = [] {
    const char* e = getenv("SALT_CLUSTER");
    int v = e ? atoi(e) : 16;
    return v < 0 ? 0 : v > 16 ? 16 : v;
  }();
  return env;
}
int cluster_tiles() {
  static const int env = [] {
    const char* e = getenv("SALT_CLUSTER_TILES");
    return e ? atoi(e) : 2;
  }();
  return env > 0 ? env : 2;
}

// SALT_CLUSTER_COMBINE=0 (test hook): keep the cluster-sized grid but
// combine through the workspace tickets — must give the same bits.
bool cluster_combine() {
  static const bool env = [] {
    const char* e = getenv("SALT_CLUSTER_COMBINE");
    return !(e && atoi(e) == 0);
  }();
  return env;
}

// Reductions of up to group_tiles() x 256 tiles run as one group of CTAs
// (SALT_GROUP_TILES overrides; tuning only).  16 (profiles/r01_group_tiles.txt):
// ddot 2^23 27.5 -> 25.8 us, sdot 2^25 44.1 -> 42.2 us vs 8; 1-4 are worse.
int group_tiles() {
  static const int env = [] {
    const char* e = getenv("SALT_GROUP_TILES");
    return e ? atoi(e) : 16;
  }();
  return env >= 0 ? env : 16;
}

int assign_tiles_per_cta() {
  static const int env = [] {
    const char* e = getenv("SALT_ASSIGN_TILES");
    return e ? atoi(e) : 0;
  }();
  return env > 0 ? env : 1;
}

int reduce_tiles_per_cta(int nl) {
  static const int env = [] {
    const char* e = getenv("SALT_REDUCE_TILES");
    return e ? atoi(e) : 0;
  }();
  if (env > 0) return env;
  return nl <= 1 ? 4 : 2;
}
constexpr int kMaxDevices = 64;

thread_local std::string g_err;
std::atomic<uint64_t> g_launches{0};
std::atomic<int> g_force_jit{0};
std::atomic<int> g_force_interp{0};
std::atomic<uint64_t> g_interp_launches{0};

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}
int cuda_fail(cudaError_t e, const char* what) {
  return fail(SALT_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
#define SALT_CUDA(call)                                  \
  do {                                                   \
    cudaError_t e_ = (call);                             \
    if (e_ != cudaSuccess) return cuda_fail(e_, #call);  \
  } while (0)

// ------------------------------------------------------------------ signatures
struct Sig {
  std::string canon;  // tokens joined by single spaces (roots joined by " ; ")
  std::string type;   // C++ type of the tree, e.g. salt::Add<salt::L<0>,salt::L<1>>
  int nl = 0, ns = 0, np = 0;
  int nroots = 0;     // assignment roots (Multi<...> when > 1)
  bool uses_d = false;
};

bool parse_index(const std::string& t, size_t from, int& k) {
  if (t.size() <= from || t.size() > from + 2) return false;
  k = 0;
  for (size_t i = from; i < t.size(); ++i) {
    if (t[i] < '0' || t[i] > '9') return false;
    k = k * 10 + (t[i] - '0');
  }
  return true;
}

// One postfix tree.  `d_limit` = how many earlier roots' values (D0 ..) it
// may read; "D" is D0.  Returns "" on success, else an error message.
std::string parse_tree(const std::string& s, int d_limit, Sig& out) {
  std::vector<std::string> toks;
  std::string cur;
  for (size_t i = 0; i <= s.size(); ++i) {
    char c = i < s.size() ? s[i] : '\0';
    if (c == ' ' || c == '\t' || c == '\0') {
      if (!cur.empty()) toks.push_back(cur), cur.clear();
    } else {
      cur.push_back(c);
    }
  }
  if (toks.empty()) return "empty signature";
  if (toks.size() > 256) return "signature too long";
  std::vector<std::string> st;
  for (const auto& t : toks) {
    int k = 0;
    if (t == "+" || t == "-" || t == "*") {
      if (st.size() < 2) return "operator '" + t + "' needs two operands in '" + s + "'";
      std::string b = st.back(); st.pop_back();
      std::string a = st.back(); st.pop_back();
      const char* node = t == "+" ? "salt::Add<" : t == "-" ? "salt::Sub<" : "salt::Mul<";
      st.push_back(std::string(node) + a + "," + b + ">");
    } else if (t[0] == 'L' && parse_index(t, 1, k)) {
      if (k >= salt::MAX_LEAVES) return "leaf index out of range: " + t;
      out.nl = std::max(out.nl, k + 1);
      st.push_back("salt::L<" + std::to_string(k) + ">");
    } else if (t[0] == 'S' && parse_index(t, 1, k)) {
      if (k >= salt::MAX_SCALARS) return "scalar index out of range: " + t;
      out.ns = std::max(out.ns, k + 1);
      st.push_back("salt::S<" + std::to_string(k) + ">");
    } else if (t[0] == 'P' && parse_index(t, 1, k)) {
      if (k >= salt::MAX_PSCALARS) return "device scalar index out of range: " + t;
      out.np = std::max(out.np, k + 1);
      st.push_back("salt::P<" + std::to_string(k) + ">");
    } else if (t[0] == 'D' && (t.size() == 1 || parse_index(t, 1, k)) && d_limit > 0) {
      if (t.size() == 1) k = 0;
      if (k >= d_limit) return "'" + t + "' reads a root that is not computed before it";
      out.uses_d = true;
      st.push_back("salt::Dk<" + std::to_string(k) + ">");
    } else {
      return "bad token '" + t + "' in signature '" + s + "'";
    }
    if (!out.canon.empty()) out.canon.push_back(' ');
    out.canon += t;
  }
  if (st.size() != 1) return std::string("signature leaves ") + std::to_string(st.size()) +
                            " values on the stack: '" + s + "'";
  out.type = st.back();
  return "";
}

// A reduce tree (d_limit = roots of the fused assignment, 0 for none).
std::string parse_sig(const char* s, int d_limit, Sig& out) {
  if (!s) return "signature is NULL";
  out = Sig();
  return parse_tree(s, d_limit, out);
}

// Assignment roots separated by ';'; root r may read D0 .. D(r-1).
std::string parse_assign(const char* s, Sig& out) {
  if (!s) return "signature is NULL";
  out = Sig();
  std::string all(s);
  std::vector<std::string> types;
  size_t pos = 0;
  while (true) {
    size_t semi = all.find(';', pos);
    std::string part = all.substr(pos, semi == std::string::npos ? std::string::npos : semi - pos);
    if ((int)types.size() == salt::MAX_ROOTS)
      return "more than " + std::to_string((int)salt::MAX_ROOTS) + " assignment roots";
    Sig r;
    std::string err = parse_tree(part, (int)types.size(), r);
    if (!err.empty()) return err;
    out.nl = std::max(out.nl, r.nl);
    out.ns = std::max(out.ns, r.ns);
    out.np = std::max(out.np, r.np);
    out.uses_d = out.uses_d || r.uses_d;
    if (!out.canon.empty()) out.canon += " ; ";
    out.canon += r.canon;
    types.push_back(r.type);
    if (semi == std::string::npos) break;
    pos = semi + 1;
  }
  out.nroots = (int)types.size();
  if (types.size() == 1) {
    out.type = types[0];
  } else {
    out.type = "salt::Multi<";
    for (size_t i = 0; i < types.size(); ++i) out.type += (i ? "," : "") + types[i];
    out.type += ">";
  }
  return "";
}

// ------------------------------------------------------------------ driver / NVRTC
struct Driver {
  bool ok = false;
  std::string why;
  CUresult (*ModuleLoadData)(CUmodule*, const void*) = nullptr;
  CUresult (*ModuleGetFunction)(CUfunction*, CUmodule, const char*) = nullptr;
  CUresult (*LaunchKernel)(CUfunction, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned,
                           unsigned, CUstream, void**, void**) = nullptr;
  CUresult (*GetErrorString)(CUresult, const char**) = nullptr;
  // optional (cluster launches of JIT kernels)
  CUresult (*LaunchKernelEx)(const CUlaunchConfig*, CUfunction, void**, void**) = nullptr;
  CUresult (*FuncSetAttribute)(CUfunction, CUfunction_attribute, int) = nullptr;
};

template <class F> bool entry(const char* name, F& fp, std::string& why) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || !p) {
    why = std::string("driver entry point missing: ") + name;
    return false;
  }
  fp = reinterpret_cast<F>(p);
  return true;
}

Driver& driver() {
  static Driver d;
  static std::once_flag once;
  std::call_once(once, [] {
    d.ok = entry("cuModuleLoadData", d.ModuleLoadData, d.why) &&
           entry("cuModuleGetFunction", d.ModuleGetFunction, d.why) &&
           entry("cuLaunchKernel", d.LaunchKernel, d.why) &&
           entry("cuGetErrorString", d.GetErrorString, d.why);
    std::string ignore;
    if (!entry("cuLaunchKernelEx", d.LaunchKernelEx, ignore) ||
        !entry("cuFuncSetAttribute", d.FuncSetAttribute, ignore))
      d.LaunchKernelEx = nullptr;
  });
  return d;
}

typedef int nvrtcResult_t;
struct Nvrtc {
  bool ok = false;
  std::string why;
  void* h = nullptr;
  nvrtcResult_t (*CreateProgram)(void**, const char*, const char*, int, const char* const*,
                                 const char* const*) = nullptr;
  nvrtcResult_t (*AddNameExpression)(void*, const char*) = nullptr;
  nvrtcResult_t (*CompileProgram)(void*, int, const char* const*) = nullptr;
  nvrtcResult_t (*GetProgramLogSize)(void*, size_t*) = nullptr;
  nvrtcResult_t (*GetProgramLog)(void*, char*) = nullptr;
  nvrtcResult_t (*GetCUBINSize)(void*, size_t*) = nullptr;
  nvrtcResult_t (*GetCUBIN)(void*, char*) = nullptr;
  nvrtcResult_t (*GetLoweredName)(void*, const char*, const char**) = nullptr;
  nvrtcResult_t (*DestroyProgram)(void**) = nullptr;
  nvrtcResult_t (*Version)(int*, int*) = nullptr;
  bool has_256bit = false;  // NVRTC >= 12.9 accepts .v8.f32 / .v4.f64
};

Nvrtc& nvrtc() {
  static Nvrtc n;
  static std::once_flag once;
  std::call_once(once, [] {
    // Prefer the toolkit's NVRTC (12.9, PTX ISA 8.8: 256-bit ld/st) by full
    // path: a bare soname would return torch's already-loaded 12.8 copy.
    const char* off = getenv("SALT_NO_JIT");  // test hook: behave as if NVRTC were absent
    if (off && atoi(off) != 0) {
      n.why = "JIT disabled (SALT_NO_JIT)";
      return;
    }
    const char* env = getenv("SALT_NVRTC_LIB");
    const char* cands[] = {env, "/usr/local/cuda/lib64/libnvrtc.so.12", "libnvrtc.so.12",
                           "libnvrtc.so"};
    for (const char* c : cands) {
      if (!c) continue;
      n.h = dlopen(c, RTLD_NOW | RTLD_LOCAL);
      if (n.h) break;
    }
    if (!n.h) {
      n.why = "libnvrtc.so.12 not found (set SALT_NVRTC_LIB)";
      return;
    }
#define SYM(F, NAME)                                               \
  n.F = reinterpret_cast<decltype(n.F)>(dlsym(n.h, NAME));         \
  if (!n.F) { n.why = std::string("nvrtc symbol missing: ") + NAME; return; }
    SYM(CreateProgram, "nvrtcCreateProgram");
    SYM(AddNameExpression, "nvrtcAddNameExpression");
    SYM(CompileProgram, "nvrtcCompileProgram");
    SYM(GetProgramLogSize, "nvrtcGetProgramLogSize");
    SYM(GetProgramLog, "nvrtcGetProgramLog");
    SYM(GetCUBINSize, "nvrtcGetCUBINSize");
    SYM(GetCUBIN, "nvrtcGetCUBIN");
    SYM(GetLoweredName, "nvrtcGetLoweredName");
    SYM(DestroyProgram, "nvrtcDestroyProgram");
    SYM(Version, "nvrtcVersion");
#undef SYM
    int major = 0, minor = 0;
    n.Version(&major, &minor);
    n.has_256bit = major > 12 || (major == 12 && minor >= 9);
    n.ok = true;
  });
  return n;
}

const char* kExprSource =
#include "salt_expr_src.inc"
    ;

// ------------------------------------------------------------------ kernel table
struct Kernel {
  const void* aot = nullptr;                 // compiled-in kernel
  std::string cubin, lowered;                // JIT kernel (device independent)
  CUfunction jit_fn[kMaxDevices] = {};       // JIT module per device
  int vec = 1;                               // lanes per vector access
  int unroll = 1;
  // cluster launches (reductions at small n): 0 unknown, 1 ok, -1 refused
  std::atomic<int> cluster_ok[kMaxDevices] = {};
  bool interp = false;                       // salt::interp_kernel (program in the parameters)
  std::atomic<int> smem_limit[kMaxDevices] = {};  // 1: dynamic shared memory cap raised on the device
};

std::string key_of(int dtype, int mode, int vec, const std::string& ta, const std::string& tr) {
  return std::to_string(dtype) + "|" + std::to_string(mode) + "|" + std::to_string(vec) + "|" +
         ta + "|" + tr;
}

std::mutex g_table_mu;
std::unordered_map<std::string, std::unique_ptr<Kernel>>& table() {
  static std::unordered_map<std::string, std::unique_ptr<Kernel>> t;
  return t;
}
std::unordered_map<std::string, std::unique_ptr<Kernel>>& jit_table() {
  // leaked: the background JIT thread may insert while the process exits
  static auto* t = new std::unordered_map<std::string, std::unique_ptr<Kernel>>;
  return *t;
}

template <class T> constexpr int dtype_of();
template <> constexpr int dtype_of<float>() { return SALT_F32; }
template <> constexpr int dtype_of<double>() { return SALT_F64; }
template <class T> constexpr int vec_of() { return 32 / (int)sizeof(T); }

template <class T, class EA, class ER, int MODE>
void reg_one(const char* asig, const char* rsig) {
  Sig sa, sr;
  std::string ta = "salt::None", tr = "salt::None";
  if (asig) { parse_assign(asig, sa); ta = sa.type; }
  if (rsig) { parse_sig(rsig, MODE == salt::MODE_ASSIGN_REDUCE ? sa.nroots : 0, sr); tr = sr.type; }
  constexpr int V = vec_of<T>();
  constexpr int U = unroll_for(MODE, salt::cmax(EA::NL, ER::NL), (int)sizeof(T));
  auto k1 = std::make_unique<Kernel>();
  k1->aot = (const void*)&salt::fused_kernel<T, EA, ER, MODE, V, U, kBlock>;
  k1->vec = V; k1->unroll = U;
  table()[key_of(dtype_of<T>(), MODE, V, ta, tr)] = std::move(k1);
  auto k2 = std::make_unique<Kernel>();
  k2->aot = (const void*)&salt::fused_kernel<T, EA, ER, MODE, 1, kUnrollScalar, kBlock>;
  k2->vec = 1; k2->unroll = kUnrollScalar;
  table()[key_of(dtype_of<T>(), MODE, 1, ta, tr)] = std::move(k2);
}

// Batch kernels (salt_assign_batch) of a single-root assignment tree.
constexpr int kBatchKind = 3;  // table key "mode" of batch kernels
template <class T, class EA> void reg_batch_one(const char* asig) {
  Sig sa;
  parse_assign(asig, sa);
  constexpr int V = vec_of<T>();
  constexpr int U = unroll_for(salt::MODE_ASSIGN, EA::NL, (int)sizeof(T));
  auto k = std::make_unique<Kernel>();
  k->aot = (const void*)&salt::batch_kernel<T, EA, V, U, kBlock>;
  k->vec = V;
  k->unroll = U;
  table()[key_of(dtype_of<T>(), kBatchKind, V, sa.type, "batch")] = std::move(k);
}

// Batched small-reduction kernels (salt_reduce_batch) of a reduce tree.
constexpr int kBatchReduceKind = 4;
template <class T, class ER> void reg_batch_reduce_one(const char* rsig) {
  Sig sr;
  parse_sig(rsig, 0, sr);
  constexpr int V = vec_of<T>();
  constexpr int U = unroll_for(salt::MODE_REDUCE, ER::NL, (int)sizeof(T));
  auto k = std::make_unique<Kernel>();
  k->aot = (const void*)&salt::batch_reduce_kernel<T, ER, V, U, kBlock>;
  k->vec = V;
  k->unroll = U;
  table()[key_of(dtype_of<T>(), kBatchReduceKind, V, "batch", sr.type)] = std::move(k);
}

template <class EA, class ER, int MODE> void reg(const char* asig, const char* rsig) {
  reg_one<float, EA, ER, MODE>(asig, rsig);
  reg_one<double, EA, ER, MODE>(asig, rsig);
  if constexpr (MODE == salt::MODE_ASSIGN) {
    if constexpr (EA::NL <= salt::BATCH_LEAVES && EA::NS <= salt::BATCH_SCALARS) {
      reg_batch_one<float, EA>(asig);
      reg_batch_one<double, EA>(asig);
    }
  }
  if constexpr (MODE == salt::MODE_REDUCE) {
    if constexpr (ER::NL <= salt::BATCH_LEAVES && ER::NS <= salt::BATCH_SCALARS) {
      reg_batch_reduce_one<float, ER>(rsig);
      reg_batch_reduce_one<double, ER>(rsig);
    }
  }
}

using namespace salt;
// Trees of the reference's named ops (ops.py:18-55) and of BASELINE.json's
// configs.  The sig string and the C++ type on each line must agree; the GPU
// tests prove it by comparing every entry against the JIT build of its sig.
void register_aot() {
  constexpr int A = MODE_ASSIGN, R = MODE_REDUCE, AR = MODE_ASSIGN_REDUCE;
  // --- assignments
  reg<L<0>, None, A>("L0", nullptr);                                      // copy
  reg<Mul<S<0>, L<0>>, None, A>("S0 L0 *", nullptr);                      // scal / scaled_copy
  reg<Add<L<0>, Mul<S<0>, L<1>>>, None, A>("L0 S0 L1 * +", nullptr);      // axpy  y + a*x
  reg<Add<Mul<S<0>, L<0>>, L<1>>, None, A>("S0 L0 * L1 +", nullptr);      // a*x + y
  reg<Add<L<0>, L<1>>, None, A>("L0 L1 +", nullptr);
  reg<Sub<L<0>, L<1>>, None, A>("L0 L1 -", nullptr);
  reg<Mul<L<0>, L<1>>, None, A>("L0 L1 *", nullptr);
  reg<Add<L<0>, Sub<L<1>, L<2>>>, None, A>("L0 L1 L2 - +", nullptr);      // C2 T1
  reg<Add<Mul<S<0>, L<0>>, Mul<S<1>, Sub<L<1>, L<2>>>>, None, A>(         // C2 T2
      "S0 L0 * S1 L1 L2 - * +", nullptr);
  reg<Add<Sub<Mul<S<0>, Add<L<0>, L<1>>>, Mul<S<1>, Sub<L<2>, L<3>>>>, Mul<S<2>, L<0>>>, None,
      A>("S0 L0 L1 + * S1 L2 L3 - * - S2 L0 * +", nullptr);               // C4 e-tree
  reg<Add<Mul<S<0>, L<0>>, Mul<S<1>, L<1>>>, None, A>("S0 L0 * S1 L1 * +", nullptr);  // axpby
  reg<Sub<L<0>, Mul<S<0>, L<1>>>, None, A>("L0 S0 L1 * -", nullptr);      // y - a*x (CG residual)
  // --- reductions
  reg<None, L<0>, R>(nullptr, "L0");                                      // sum
  reg<None, Mul<L<0>, L<1>>, R>(nullptr, "L0 L1 *");                      // dot
  reg<None, Mul<L<0>, L<0>>, R>(nullptr, "L0 L0 *");                      // dot(x,x) / nrm2
  reg<None, Mul<Sub<L<0>, L<1>>, Sub<L<0>, L<1>>>, R>(nullptr, "L0 L1 - L0 L1 - *");  // ||x-y||^2
  reg<None, Mul<Mul<L<0>, L<1>>, L<2>>, R>(nullptr, "L0 L1 * L2 *");       // weighted dot
  // --- fused assign + reduce (C5: y = y + a*x ; r = dot(y, z))
  reg<Add<L<0>, Mul<S<0>, L<1>>>, Mul<D, L<2>>, AR>("L0 S0 L1 * +", "D L2 *");
  reg<Add<L<0>, Mul<S<0>, L<1>>>, Mul<D, D>, AR>("L0 S0 L1 * +", "D D *");
  reg<Sub<L<0>, Mul<S<0>, L<1>>>, Mul<D, D>, AR>("L0 S0 L1 * -", "D D *");  // CG: r -= a*q; r.r
  // CG iteration body in one pass: x += a*p ; r -= a*q ; rr = r.r
  reg<Multi<Add<L<0>, Mul<S<0>, L<1>>>, Sub<L<2>, Mul<S<1>, L<3>>>>, Mul<Dk<1>, Dk<1>>, AR>(
      "L0 S0 L1 * + ; L2 S1 L3 * -", "D1 D1 *");
}

void ensure_table() {
  static std::once_flag once;
  std::call_once(once, [] { register_aot(); });
}

// Compile the tree with NVRTC; returns nullptr + g_err on failure.
// On-disk cubin cache for JIT kernels: $SALT_JIT_CACHE (default
// ~/.cache/salt_jit; "off" disables), one file per (source, options, kernel)
// hash holding the lowered name and the cubin.  Only a start-up cost saver:
// a miss simply compiles.
std::string jit_cache_dir() {
  const char* e = getenv("SALT_JIT_CACHE");
  if (e && std::string(e) == "off") return "";
  if (e && *e) return e;
  const char* home = getenv("HOME");
  return home ? std::string(home) + "/.cache/salt_jit" : "";
}

uint64_t fnv1a(const std::string& s, uint64_t h = 1469598103934665603ull) {
  for (unsigned char c : s) h = (h ^ c) * 1099511628211ull;
  return h;
}

bool jit_cache_load(const std::string& path, Kernel& k) {
  std::ifstream f(path, std::ios::binary);
  if (!f) return false;
  std::string name;
  if (!std::getline(f, name) || name.empty()) return false;
  std::stringstream ss;
  ss << f.rdbuf();
  std::string bin = ss.str();
  if (bin.size() < 16) return false;
  k.lowered = name;
  k.cubin = bin;
  return true;
}

void jit_cache_store(const std::string& dir, const std::string& path, const Kernel& k) {
  mkdir(dir.c_str(), 0755);  // parent of the default dir: ~/.cache
  // unique per process and thread (the background JIT thread may store too)
  std::string tmp = path + ".tmp" + std::to_string(getpid()) + "." +
                    std::to_string(std::hash<std::thread::id>()(std::this_thread::get_id()));
  {
    std::ofstream f(tmp, std::ios::binary);
    if (!f) return;
    f << k.lowered << "\n";
    f.write(k.cubin.data(), (std::streamsize)k.cubin.size());
    if (!f) return;
  }
  rename(tmp.c_str(), path.c_str());
}

// Build (or load from the disk cache) the JIT kernel of a tree; nullptr +
// g_err on failure.  cache_only: return nullptr on a cache miss instead of
// compiling.  The caller inserts the result into jit_table().
std::unique_ptr<Kernel> jit_build(int dtype, int mode, int vec, int nl, const std::string& ta,
                                  const std::string& tr, bool cache_only) {
  Nvrtc& nv = nvrtc();
  if (!nv.ok) { g_err = "NVRTC unavailable: " + nv.why; return nullptr; }
  const char* tname = dtype == SALT_F32 ? "float" : "double";
  const bool batch = mode == kBatchKind, batch_reduce = mode == kBatchReduceKind;
  const int kmode = batch ? salt::MODE_ASSIGN : batch_reduce ? salt::MODE_REDUCE : mode;
  const int unroll = vec == 1 ? kUnrollScalar
                     : tuning_unroll() > 0 ? tuning_unroll()
                     : unroll_for(kmode, nl, dtype == SALT_F32 ? 4 : 8);
  const std::string tail = std::to_string(vec) + "," + std::to_string(unroll) + "," +
                           std::to_string(kBlock) + ">";
  std::string expr =
      batch ? std::string("salt::batch_kernel<") + tname + "," + ta + "," + tail
      : batch_reduce ? std::string("salt::batch_reduce_kernel<") + tname + "," + tr + "," + tail
                     : std::string("salt::fused_kernel<") + tname + "," + ta + "," + tr + "," +
                           std::to_string(mode) + "," + tail;
  const std::string minb = "-DSALT_MIN_BLOCKS=" + std::to_string(tuning_minb());
  const char* opts[8] = {"--gpu-architecture=sm_100a", "-fmad=false", "--std=c++17",
                         "-lineinfo", "-default-device"};
  int nopts = 5;
  if (!nv.has_256bit) opts[nopts++] = "-DSALT_NO_256BIT";
  if (tuning_minb() > 0 && vec != 1) opts[nopts++] = minb.c_str();
  std::string cache_path;
  const std::string cdir = jit_cache_dir();
  if (!cdir.empty()) {
    std::string id = expr;
    for (int i = 0; i < nopts; ++i) id += std::string("|") + opts[i];
    int maj = 0, min = 0;
    nv.Version(&maj, &min);
    id += "|nvrtc" + std::to_string(maj) + "." + std::to_string(min);
    char hex[32];
    snprintf(hex, sizeof hex, "%016llx", (unsigned long long)fnv1a(id, fnv1a(kExprSource)));
    cache_path = cdir + "/" + hex + ".salt";
    auto k = std::make_unique<Kernel>();
    if (jit_cache_load(cache_path, *k)) {
      k->vec = vec;
      k->unroll = unroll;
      return k;
    }
  }
  if (cache_only) return nullptr;
  void* prog = nullptr;
  if (nv.CreateProgram(&prog, kExprSource, "salt_expr_jit.cu", 0, nullptr, nullptr) != 0) {
    g_err = "nvrtcCreateProgram failed";
    return nullptr;
  }
  nv.AddNameExpression(prog, expr.c_str());
  int rc = nv.CompileProgram(prog, nopts, opts);
  if (rc != 0) {
    size_t ls = 0;
    nv.GetProgramLogSize(prog, &ls);
    std::string log(ls, '\0');
    nv.GetProgramLog(prog, &log[0]);
    nv.DestroyProgram(&prog);
    g_err = "NVRTC compile failed for " + expr + ":\n" + log;
    return nullptr;
  }
  auto k = std::make_unique<Kernel>();
  size_t cs = 0;
  nv.GetCUBINSize(prog, &cs);
  k->cubin.resize(cs);
  nv.GetCUBIN(prog, &k->cubin[0]);
  const char* low = nullptr;
  nv.GetLoweredName(prog, expr.c_str(), &low);
  k->lowered = low ? low : "";
  nv.DestroyProgram(&prog);
  k->vec = vec;
  k->unroll = unroll;
  if (!cache_path.empty()) {
    std::string parent = cdir.substr(0, cdir.find_last_of('/'));
    if (!parent.empty()) mkdir(parent.c_str(), 0755);
    jit_cache_store(cdir, cache_path, *k);
  }
  return k;
}

Kernel* jit_insert(const std::string& key, std::unique_ptr<Kernel> k) {
  std::lock_guard<std::mutex> lk(g_table_mu);
  auto& slot = jit_table()[key];
  if (!slot) slot = std::move(k);  // a concurrent build of the same tree may have won
  return slot.get();
}

// ---- tiered JIT: a tree outside the compiled-in table runs on the
// interpreter (same bits, salt_interp.cuh) while a background thread
// compiles it with NVRTC; later calls find the compiled kernel, so no call
// waits for NVRTC.  Opt-in (SALT_JIT_ASYNC=1 / salt_set_jit_async(1)): by
// default fresh trees are built synchronously and no thread is started.
struct JitJob {
  int dtype, mode, vec, nl;
  std::string ta, tr, key;
};
struct AsyncJit {
  std::mutex mu;
  std::condition_variable cv, idle;
  std::deque<JitJob> queue;
  std::unordered_set<std::string> pending, failed;
  std::unordered_map<std::string, std::string> errors;
  int active = 0;
  bool started = false, stopping = false;
};
AsyncJit& async_jit() {
  static AsyncJit* a = new AsyncJit;  // leaked: the worker may outlive static destructors
  return *a;
}
std::atomic<int> g_jit_async{-1};  // -1: not yet read from SALT_JIT_ASYNC
bool jit_async() {
  int v = g_jit_async.load(std::memory_order_relaxed);
  if (v < 0) {
    const char* e = getenv("SALT_JIT_ASYNC");  // opt-in
    v = e && atoi(e) != 0 ? 1 : 0;
    g_jit_async.store(v);
  }
  return v == 1;
}

void jit_worker() {
  AsyncJit& A = async_jit();
  for (;;) {
    JitJob j;
    {
      std::unique_lock<std::mutex> lk(A.mu);
      // never woken once the process exits (see jit_atexit): a thread
      // returning while exit() tears down the C++ runtime can crash it
      A.cv.wait(lk, [&] { return !A.queue.empty() && !A.stopping; });
      j = std::move(A.queue.front());
      A.queue.pop_front();
      ++A.active;
    }
    std::unique_ptr<Kernel> k = jit_build(j.dtype, j.mode, j.vec, j.nl, j.ta, j.tr, false);
    std::string err = k ? std::string() : g_err;
    if (k) jit_insert(j.key, std::move(k));
    std::lock_guard<std::mutex> lk(A.mu);
    A.pending.erase(j.key);
    if (!err.empty()) {
      A.failed.insert(j.key);
      A.errors[j.key] = err;
    }
    --A.active;
    if (A.queue.empty() && A.active == 0) A.idle.notify_all();
  }
}

// At exit: drop queued builds and let a compile in flight finish (NVRTC
// must not run while the process tears its libraries down).  The worker is
// then left blocked on its condition variable — it is never woken again, so
// it cannot run any code while exit() destroys the runtime.
void jit_atexit() {
  AsyncJit& A = async_jit();
  std::unique_lock<std::mutex> lk(A.mu);
  A.stopping = true;
  A.queue.clear();
  A.pending.clear();
  A.idle.wait_for(lk, std::chrono::seconds(10), [&] { return A.active == 0; });
}

// Queue a background build; false if it failed before (g_err = why).
bool jit_enqueue(JitJob j) {
  AsyncJit& A = async_jit();
  std::lock_guard<std::mutex> lk(A.mu);
  if (A.failed.count(j.key)) {
    g_err = A.errors[j.key];
    return false;
  }
  if (A.pending.count(j.key)) return true;
  if (A.stopping) return false;
  if (!A.started) {
    A.started = true;
    std::thread(jit_worker).detach();
    atexit(jit_atexit);
  }
  A.pending.insert(j.key);
  A.queue.push_back(std::move(j));
  A.cv.notify_one();
  return true;
}

// Look up (or JIT) the kernel; nullptr + g_err on failure.  async: on a
// miss (table, JIT table and disk cache) queue a background build and return
// nullptr with *queued = true — the caller runs the interpreter meanwhile.
Kernel* get_kernel(int dtype, int mode, int vec, int nl, const std::string& ta,
                   const std::string& tr, bool async = false, bool* queued = nullptr) {
  ensure_table();
  const std::string key = key_of(dtype, mode, vec, ta, tr);
  {
    std::lock_guard<std::mutex> lk(g_table_mu);
    if (!g_force_jit.load() && tuning_unroll() <= 0 && tuning_minb() <= 0) {
      auto it = table().find(key);
      if (it != table().end()) return it->second.get();
    }
    auto jt = jit_table().find(key);
    if (jt != jit_table().end()) return jt->second.get();
  }
  if (async && nvrtc().ok) {
    if (auto k = jit_build(dtype, mode, vec, nl, ta, tr, true)) return jit_insert(key, std::move(k));
    if (queued) *queued = jit_enqueue(JitJob{dtype, mode, vec, nl, ta, tr, key});
    return nullptr;
  }
  auto k = jit_build(dtype, mode, vec, nl, ta, tr, false);
  return k ? jit_insert(key, std::move(k)) : nullptr;
}

std::mutex g_dev_mu;

// The interpreter kernels: per element type, the vector width and unroll of
// every compiled kernel (so the interpreter walks the same tiles and its
// reductions add in the same order).
template <class T> Kernel* interp_kernel_for(int vec, int unroll) {
  static Kernel k2, k4, k1;
  static std::once_flag once;
  std::call_once(once, [] {
    k2.aot = (const void*)&salt::interp_kernel<T, vec_of<T>(), 2, kBlock>;
    k4.aot = (const void*)&salt::interp_kernel<T, vec_of<T>(), 4, kBlock>;
    k1.aot = (const void*)&salt::interp_kernel<T, 1, kUnrollScalar, kBlock>;
    k2.vec = k4.vec = vec_of<T>();
    k1.vec = 1;
    k2.unroll = 2;
    k4.unroll = 4;
    k1.unroll = kUnrollScalar;
    k2.interp = k4.interp = k1.interp = true;
  });
  return vec == 1 ? &k1 : unroll == 4 ? &k4 : &k2;
}

int current_device(int& dev) {
  SALT_CUDA(cudaGetDevice(&dev));
  if (dev < 0 || dev >= kMaxDevices) return fail(SALT_EINVAL, "device ordinal out of range");
  return 0;
}

// Resolve per-device state (the JIT module) for a kernel.
int prepare(Kernel* k, int dev) {
  if (k->aot) return 0;
  std::lock_guard<std::mutex> lk(g_dev_mu);
  if (!k->jit_fn[dev]) {
    Driver& d = driver();
    if (!d.ok) return fail(SALT_EJIT, "driver API unavailable: " + d.why);
    CUmodule mod;
    CUresult r = d.ModuleLoadData(&mod, k->cubin.data());
    if (r != CUDA_SUCCESS) {
      const char* s = "?";
      d.GetErrorString(r, &s);
      return fail(SALT_EJIT, std::string("cuModuleLoadData: ") + s);
    }
    r = d.ModuleGetFunction(&k->jit_fn[dev], mod, k->lowered.c_str());
    if (r != CUDA_SUCCESS) return fail(SALT_EJIT, "cuModuleGetFunction failed for " + k->lowered);
  }
  return 0;
}

// Fused kernels are launched with programmatic stream serialization (PDL):
// the grid may be scheduled while the previous kernel on the stream drains;
// the kernel's first instruction (griddepcontrol.wait) holds every CTA until
// that kernel has completed and its writes are visible.  SALT_PDL=0 turns it
// off (tuning / A-B tests only).
bool use_pdl() {
  static const bool env = [] {
    const char* e = getenv("SALT_PDL");
    return !(e && atoi(e) == 0);
  }();
  return env;
}

// One cluster of `grid` CTAs (2..16; > 8 needs the non-portable opt-in).
// Returns false (without an error) if this kernel/device refuses clusters
// of that size, so the caller launches the ticket-combine grid instead.
template <class T> bool launch_cluster(Kernel* k, int dev, int grid, salt::Args<T>& args,
                                       cudaStream_t st, int& rc) {
  rc = 0;
  std::atomic<int>& ok = k->cluster_ok[dev];
  if (ok.load(std::memory_order_relaxed) < 0) return false;
  void* params[] = {&args};
  if (k->aot) {
    if (ok.load(std::memory_order_relaxed) == 0) {
      if (cudaFuncSetAttribute(k->aot, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) !=
          cudaSuccess) {
        cudaGetLastError();
        ok.store(-1);
        return false;
      }
      ok.store(1);
    }
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = (unsigned)grid;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kBlock);
    cfg.stream = st;
    cfg.attrs = attr;
    cfg.numAttrs = use_pdl() ? 2 : 1;
    cudaError_t e = cudaLaunchKernelExC(&cfg, k->aot, params);
    if (e != cudaSuccess) {
      cudaGetLastError();
      ok.store(-1);
      return false;
    }
  } else {
    Driver& d = driver();
    if (!d.LaunchKernelEx) return false;
    if (ok.load(std::memory_order_relaxed) == 0) {
      if (d.FuncSetAttribute(k->jit_fn[dev], CU_FUNC_ATTRIBUTE_NON_PORTABLE_CLUSTER_SIZE_ALLOWED,
                             1) != CUDA_SUCCESS) {
        ok.store(-1);
        return false;
      }
      ok.store(1);
    }
    CUlaunchConfig cfg = {};
    CUlaunchAttribute attr[2];
    attr[0].id = CU_LAUNCH_ATTRIBUTE_CLUSTER_DIMENSION;
    attr[0].value.clusterDim.x = (unsigned)grid;
    attr[0].value.clusterDim.y = 1;
    attr[0].value.clusterDim.z = 1;
    attr[1].id = CU_LAUNCH_ATTRIBUTE_PROGRAMMATIC_STREAM_SERIALIZATION;
    attr[1].value.programmaticStreamSerializationAllowed = 1;
    cfg.gridDimX = (unsigned)grid;
    cfg.gridDimY = cfg.gridDimZ = 1;
    cfg.blockDimX = kBlock;
    cfg.blockDimY = cfg.blockDimZ = 1;
    cfg.hStream = (CUstream)st;
    cfg.attrs = attr;
    cfg.numAttrs = use_pdl() ? 2 : 1;
    if (d.LaunchKernelEx(&cfg, k->jit_fn[dev], params, nullptr) != CUDA_SUCCESS) {
      ok.store(-1);
      return false;
    }
  }
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return true;
}

// One launch of `k` with its single by-value parameter at `argp` (Args<T>,
// or InterpArgs<T> for the interpreter) and `smem` dynamic shared bytes.
int launch_raw(Kernel* k, int dev, int grid, void* argp, size_t smem, cudaStream_t st) {
  void* params[] = {argp};
  const bool pdl = use_pdl();
  if (k->aot) {
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kBlock);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    cudaError_t e = cudaLaunchKernelExC(&cfg, k->aot, params);
    if (e != cudaSuccess) return cuda_fail(e, "cudaLaunchKernelExC");
  } else if (pdl && driver().LaunchKernelEx) {
    CUlaunchConfig cfg = {};
    CUlaunchAttribute attr[1];
    attr[0].id = CU_LAUNCH_ATTRIBUTE_PROGRAMMATIC_STREAM_SERIALIZATION;
    attr[0].value.programmaticStreamSerializationAllowed = 1;
    cfg.gridDimX = (unsigned)grid;
    cfg.gridDimY = cfg.gridDimZ = 1;
    cfg.blockDimX = kBlock;
    cfg.blockDimY = cfg.blockDimZ = 1;
    cfg.hStream = (CUstream)st;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    CUresult r = driver().LaunchKernelEx(&cfg, k->jit_fn[dev], params, nullptr);
    if (r != CUDA_SUCCESS) {
      const char* s = "?";
      driver().GetErrorString(r, &s);
      return fail(SALT_ECUDA, std::string("cuLaunchKernelEx: ") + s);
    }
  } else {
    CUresult r = driver().LaunchKernel(k->jit_fn[dev], grid, 1, 1, kBlock, 1, 1, 0,
                                       (CUstream)st, params, nullptr);
    if (r != CUDA_SUCCESS) {
      const char* s = "?";
      driver().GetErrorString(r, &s);
      return fail(SALT_ECUDA, std::string("cuLaunchKernel: ") + s);
    }
  }
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return 0;
}

template <class T> int launch(Kernel* k, int dev, int grid, salt::Args<T>& args, cudaStream_t st) {
  return launch_raw(k, dev, grid, &args, 0, st);
}

// Common 32-byte misalignment of all operands -> (vec, head, nvec).
template <class T>
void geometry(void* const* dsts, int ndst, const void* const* leaves, int nl, i64 n, int& vec,
              i64& head, i64& nvec) {
  constexpr int V = vec_of<T>();
  uintptr_t mis = (uintptr_t)-1;
  bool same = true;
  auto check = [&](const void* p) {
    uintptr_t m = (uintptr_t)p % 32;
    if (mis == (uintptr_t)-1) mis = m;
    else if (m != mis) same = false;
    if (m % sizeof(T)) same = false;
  };
  for (int r = 0; dsts && r < ndst; ++r) check(dsts[r]);
  for (int l = 0; leaves && l < nl; ++l) check(leaves[l]);
  if (mis == (uintptr_t)-1) mis = 0;
  if (same) {
    i64 h = (i64)(((32 - mis) % 32) / sizeof(T));
    if (h > n) h = n;
    vec = V;
    head = h;
    nvec = (n - h) / V;
  } else {
    vec = 1;
    head = 0;
    nvec = n;
  }
}

struct Plan {
  Sig sa, sr;
  int mode = 0;
  int nl = 0, ns = 0, np = 0;
  Kernel* cached[2][2] = {};  // [force_jit][vec == 1]: table / JIT lookups done once
  salt::Prog prog;            // the same trees as an interpreter program
  bool prog_ok = false;
  std::string prog_err;
};

// Encode the plan's trees for interp_kernel: assignment roots in order, each
// followed by OP_STORE r, then the reduce tree followed by OP_ACC.  Stack
// slots = the deepest push (the top of the stack stays in registers).
std::string encode_prog(const Plan& p, salt::Prog& g) {
  memset(&g, 0, sizeof(g));
  int sp = 0;
  auto emit = [&](int op, int arg) -> bool {
    if (g.len >= salt::MAX_PROG) return false;
    g.op[g.len] = (unsigned char)op;
    g.arg[g.len] = (unsigned char)arg;
    ++g.len;
    if (op <= salt::OP_D) g.slots = std::max(g.slots, ++sp);
    else if (op <= salt::OP_MUL) --sp;
    else sp = 0;
    return true;
  };
  auto tree = [&](const std::string& canon) -> bool {
    std::istringstream in(canon);
    std::string t;
    while (in >> t) {
      if (t == ";") continue;
      bool ok;
      if (t == "+") ok = emit(salt::OP_ADD, 0);
      else if (t == "-") ok = emit(salt::OP_SUB, 0);
      else if (t == "*") ok = emit(salt::OP_MUL, 0);
      else if (t == "D") ok = emit(salt::OP_D, 0);
      else {
        const int k = atoi(t.c_str() + 1);
        const int op = t[0] == 'L' ? salt::OP_LEAF : t[0] == 'S' ? salt::OP_SCALAR
                       : t[0] == 'P' ? salt::OP_PSCALAR : salt::OP_D;
        ok = emit(op, k);
      }
      if (!ok) return false;
    }
    return true;
  };
  if (p.mode != salt::MODE_REDUCE) {
    size_t pos = 0;
    int r = 0;
    const std::string& all = p.sa.canon;
    while (true) {
      size_t semi = all.find(';', pos);
      if (!tree(all.substr(pos, semi == std::string::npos ? std::string::npos : semi - pos)) ||
          !emit(salt::OP_STORE, r))
        return "tree too long for the interpreter (" + std::to_string((int)salt::MAX_PROG) + " tokens)";
      ++r;
      if (semi == std::string::npos) break;
      pos = semi + 1;
    }
    g.nroots = r;
  }
  if (p.mode != salt::MODE_ASSIGN) {
    if (!tree(p.sr.canon) || !emit(salt::OP_ACC, 0))
      return "tree too long for the interpreter (" + std::to_string((int)salt::MAX_PROG) + " tokens)";
    g.reduce = 1;
  }
  g.nl = p.nl;
  // 8 KiB per slot (32-byte vectors x 256 threads); stay below 224 KiB
  if (salt::interp_smem_bytes(g, 4, kBlock, 8) > 224 * 1024)
    return "tree needs " + std::to_string(g.nl + g.slots + g.nroots) +
           " interpreter slots (leaves + stack depth + roots > 28)";
  return "";
}

// Parsed signatures are cached per thread (keyed by the raw strings), so a
// repeated call costs one hash lookup instead of a parse + type rebuild.
int make_plan(int dtype, const char* asig, const char* rsig, int mode, int nleaves, int nscalars,
              Plan*& out) {
  if (dtype != SALT_F32 && dtype != SALT_F64) return fail(SALT_EINVAL, "dtype must be SALT_F32 or SALT_F64");
  thread_local std::unordered_map<std::string, std::unique_ptr<Plan>> cache;
  std::string key;
  key.push_back(char('0' + dtype));
  key.push_back(char('0' + mode));
  if (mode != salt::MODE_REDUCE && asig) key += asig;
  key.push_back('\x1f');
  if (mode != salt::MODE_ASSIGN && rsig) key += rsig;
  Plan* p;
  auto it = cache.find(key);
  if (it != cache.end()) {
    p = it->second.get();
  } else {
    auto np = std::make_unique<Plan>();
    np->mode = mode;
    std::string err;
    np->sa.type = np->sr.type = "salt::None";
    if (mode != salt::MODE_REDUCE) {
      err = parse_assign(asig, np->sa);
      if (!err.empty()) return fail(SALT_EINVAL, err);
    }
    if (mode != salt::MODE_ASSIGN) {
      err = parse_sig(rsig, mode == salt::MODE_ASSIGN_REDUCE ? np->sa.nroots : 0, np->sr);
      if (!err.empty()) return fail(SALT_EINVAL, err);
    }
    np->nl = std::max(np->sa.nl, np->sr.nl);
    np->ns = std::max(np->sa.ns, np->sr.ns);
    np->np = std::max(np->sa.np, np->sr.np);
    np->prog_err = encode_prog(*np, np->prog);
    np->prog_ok = np->prog_err.empty();
    if (cache.size() > 4096) cache.clear();
    p = np.get();
    cache.emplace(std::move(key), std::move(np));
  }
  if (nleaves < p->nl || nleaves > salt::MAX_LEAVES)
    return fail(SALT_EINVAL, "signature references " + std::to_string(p->nl) + " leaves but " +
                                 std::to_string(nleaves) + " were passed");
  if (nscalars < p->ns || nscalars > salt::MAX_SCALARS)
    return fail(SALT_EINVAL, "signature references " + std::to_string(p->ns) + " scalars but " +
                                 std::to_string(nscalars) + " were passed");
  out = p;
  return 0;
}

template <class T>
int run_fused(Plan& p, void* const* dsts, int ndst, const void* const* leaves, int nleaves,
              const double* scalars, int nscalars, i64 n, int flags, void* ws, size_t ws_bytes,
              void* out_dev, void* out_host, cudaStream_t st, const salt_exchange* x,
              const void* const* pscalars, int npscalars) {
  if (n < 0) return fail(SALT_EINVAL, "negative length");
  const bool reduce = p.mode != salt::MODE_ASSIGN;
  if (!reduce && n == 0) return 0;  // zero length assign is a no-op (test_engine.py:147-153)
  // Empty vectors may legitimately have NULL storage (torch gives numel-0
  // tensors a NULL data pointer); nothing is dereferenced when n == 0.
  const int nroots = p.mode == salt::MODE_REDUCE ? 0 : p.sa.nroots;
  if (ndst != nroots)
    return fail(SALT_EINVAL, "signature has " + std::to_string(nroots) + " assignment roots but " +
                                 std::to_string(ndst) + " destinations were passed");
  for (int r = 0; n > 0 && r < nroots; ++r)
    if (!dsts || !dsts[r]) return fail(SALT_EINVAL, "NULL destination");
  if (n > 0 && p.nl > 0 && !leaves) return fail(SALT_EINVAL, "NULL leaf array");
  for (int l = 0; n > 0 && l < p.nl; ++l)
    if (!leaves[l]) return fail(SALT_EINVAL, "NULL leaf pointer");
  if (reduce) {
    if (!out_dev) return fail(SALT_EINVAL, "NULL reduction output");
    if (!ws || ws_bytes < salt_reduce_workspace_bytes())
      return fail(SALT_EWORKSPACE, "reduction workspace smaller than salt_reduce_workspace_bytes()");
  }
  salt::Args<T> a;
  memset(&a, 0, sizeof(a));
  for (int r = 0; r < nroots; ++r) a.dst[r] = (T*)dsts[r];
  for (int l = 0; l < p.nl; ++l) a.leaf[l] = leaves ? (const T*)leaves[l] : nullptr;
  for (int s = 0; s < p.ns; ++s) a.sc[s] = (T)scalars[s];
  if (npscalars < p.np || npscalars > salt::MAX_PSCALARS)
    return fail(SALT_EINVAL, "signature reads " + std::to_string(p.np) + " device scalars but " +
                                 std::to_string(npscalars) + " were passed");
  for (int q = 0; q < p.np; ++q) {
    if (!pscalars || !pscalars[q]) return fail(SALT_EINVAL, "NULL device scalar");
    a.ps[q] = (const T*)pscalars[q];
  }
  a.n = n;
  a.flags = flags;
  int vec;
  geometry<T>(dsts, nroots, leaves, p.nl, n, vec, a.head, a.nvec);
  Kernel* k = nullptr;
  const bool force_interp = g_force_interp.load(std::memory_order_relaxed) != 0;
  if (!force_interp) {
    Kernel*& slot = p.cached[g_force_jit.load(std::memory_order_relaxed)][vec == 1 ? 1 : 0];
    if (!slot) {
      // tiered: trees the interpreter can run do not wait for NVRTC (unless
      // the JIT itself is being tested: salt_set_force_jit)
      // ... nor while the stream is being captured into a CUDA graph: the
      // graph would keep the interpreter kernel for good
      cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
      if (cudaStreamIsCapturing(st, &cap) != cudaSuccess) cudaGetLastError();
      const bool async = p.prog_ok && jit_async() && !g_force_jit.load(std::memory_order_relaxed) &&
                         cap == cudaStreamCaptureStatusNone;
      bool queued = false;
      slot = get_kernel(dtype_of<T>(), p.mode, vec, p.nl, p.sa.type, p.sr.type, async, &queued);
    }
    k = slot;
  }
  if (!k) {
    // Not compiled in and no JIT build (NVRTC missing or failed), or forced:
    // the postfix interpreter evaluates the same trees (salt_interp.cuh).
    if (!p.prog_ok)
      return fail(SALT_EJIT, (force_interp ? std::string() : g_err + "; ") + "interpreter: " + p.prog_err);
    k = interp_kernel_for<T>(vec, unroll_for(p.mode, p.nl, (int)sizeof(T)));
  }
  int dev;
  int rc = current_device(dev);
  if (rc) return rc;
  rc = prepare(k, dev);
  if (rc) return rc;
  // Work split (tools/stream_variants.cu, tools/reduce_variants.cu on B200):
  // assignments take one BLOCK*UNR tile per CTA — the block scheduler
  // refills an SM the moment a CTA retires, which keeps loads in flight
  // (7.29 TB/s vs 7.06 for a persistent grid-stride loop); reductions take
  // kReduceTilesPerCta tiles per CTA and combine per-CTA partials in two
  // deterministic ticket levels (7.25 vs 6.88 TB/s persistent, fused
  // axpy->dot f64 2^28).  Both grids depend only on n.
  const i64 per_tile = (i64)kBlock * k->unroll;
  const i64 ntiles = (a.nvec + per_tile - 1) / per_tile;
  i64 K = assign_tiles_per_cta(), cap = i64(0x7fffffff);
  bool cluster = false, one_group = false;
  if (reduce && ntiles > 2 && ntiles <= (i64)max_cluster() * cluster_tiles()) {
    // Small n (3 .. 16 x 2 tiles; up to 2 tiles one CTA is quicker): one cluster
    // of <= 16 CTAs, partials combined in distributed shared memory — no
    // workspace round trip, no ticket atomics.  B200, back-to-back launches
    // (profiles/r01_cluster_reduce.txt): nrm2 f64 2^16 6.33 -> 4.13 us,
    // sdot 2^17 5.35 -> 4.28 us, fused axpy->dot 2^14 5.18 -> 4.07 us.
    K = (ntiles + max_cluster() - 1) / max_cluster();
    cluster = true;
  } else if (reduce) {
    K = reduce_tiles_per_cta(p.nl);
    cap = salt::MAX_REDUCE_CTAS;
    // Small and mid sizes: if at most 16 tiles per CTA fit everything into
    // one group of CTAs, use one group with as many CTAs as possible — the
    // single-group combine skips the second ticket level (f64 dot at 2^22:
    // 7.2 vs 5.1 TB/s) and more CTAs keep more SMs streaming (nrm2 f64 at
    // 2^19: 6.39 -> 4.67 us; profiles/r01_small_n/).
    // Up to 2 tiles: one CTA (no combine at all).
    // The one group may hold 2 x GROUP = 512 CTAs when a thread keeps at
    // most 128 bytes of loads in flight per tile (nrm2 / sum: one leaf x 4
    // vectors; f64 dot: two leaves x 2): 256 such CTAs leave HBM short of
    // requests at 2^23-2^25 (tools/midred_probe.cu, profiles/
    // r01_midred_probe.txt: dnrm2 2^24 28.5 -> 26.3 us, ddot 2^24 46.9 ->
    // 44.2 us, snrm2 2^24 17.4 -> 15.8 us); with more bytes in flight per
    // thread (f32 dot, 3+ leaves) 512 CTAs are slower than 256.
    const i64 vbytes = vec == 1 ? (i64)sizeof(T) : 32;
    const i64 one = (i64)k->unroll * p.nl * vbytes <= 128 ? 2 * salt::GROUP : salt::GROUP;
    if (ntiles <= 2) K = ntiles > 0 ? ntiles : 1;
    else if (ntiles <= (i64)group_tiles() * one) {
      K = (ntiles + one - 1) / one;
      one_group = true;
    }
  }
  if ((ntiles + K - 1) / K > cap) K = (ntiles + cap - 1) / cap;
  i64 g64 = (ntiles + K - 1) / K;
  if (g64 < 1) g64 = 1;
  const int grid = (int)g64;
  a.tiles_per_cta = K;
  // CTAs per combine group: the whole grid when it was sized as one group
  // (at most 2 x GROUP), else GROUP (a grid of <= GROUP CTAs is one group
  // either way).
  a.group = one_group ? grid : salt::GROUP;
  if (reduce) {
    char* w = (char*)ws;
    a.ticket = (unsigned int*)(w + salt::WsLayout::ticket);
    a.group_tickets = (unsigned int*)(w + salt::WsLayout::group_tickets);
    a.group_partials = (salt::DD*)(w + salt::WsLayout::group_partials);
    a.partials = (salt::DD*)(w + salt::WsLayout::partials);
    a.out = out_dev;
    if (x) {
      if (x->world < 1 || x->world > salt::XCHG_MAX_RANKS || x->rank < 0 || x->rank >= x->world ||
          x->epoch == 0)
        return fail(SALT_EINVAL, "bad exchange descriptor (world 1..8, 0 <= rank < world, epoch >= 1)");
      if (flags & SALT_PARTIAL) return fail(SALT_EINVAL, "SALT_PARTIAL cannot be combined with an exchange");
      a.xchg.rank = x->rank;
      a.xchg.world = x->world;
      a.xchg.epoch = x->epoch;
      for (int r = 0; r < x->world; ++r) {
        if (!x->slots[r] || !x->flags[r]) return fail(SALT_EINVAL, "NULL exchange buffer");
        a.xchg.slots[r] = (salt::DD*)x->slots[r];
        a.xchg.flags[r] = (unsigned long long*)x->flags[r];
      }
      a.xchg.timeout_ns = x->timeout_ns;
      a.xchg.error = (unsigned int*)x->error;
    }
  }
  // the interpreter keeps the cluster-sized grid but folds through the
  // tickets (same bits, as SALT_CLUSTER_COMBINE=0 shows for compiled kernels)
  a.cluster = cluster && grid > 1 && cluster_combine() && !k->interp ? 1 : 0;
  bool launched = false;
  if (a.cluster) {
    launched = launch_cluster<T>(k, dev, grid, a, st, rc);
    if (rc) return rc;
    // refused (e.g. no 16-CTA cluster fits): same grid, ticket combine —
    // identical bits, since both fold the partials in CTA order
    if (!launched) a.cluster = 0;
  }
  if (!launched && k->interp) {
    salt::InterpArgs<T> ia;
    ia.a = a;
    ia.pg = p.prog;
    const int smem = salt::interp_smem_bytes(p.prog, vec, kBlock, (int)sizeof(T));
    if (!k->smem_limit[dev].load(std::memory_order_acquire)) {  // once per device: the cap
      SALT_CUDA(cudaFuncSetAttribute(k->aot, cudaFuncAttributeMaxDynamicSharedMemorySize, 224 * 1024));
      k->smem_limit[dev].store(1, std::memory_order_release);
    }
    rc = launch_raw(k, dev, grid, &ia, (size_t)smem, st);
    if (rc) return rc;
    g_interp_launches.fetch_add(1, std::memory_order_relaxed);
  } else if (!launched) {
    rc = launch<T>(k, dev, grid, a, st);
    if (rc) return rc;
  }
  if (reduce && out_host) {
    size_t bytes = (flags & SALT_PARTIAL) ? sizeof(salt::DD) : sizeof(T);
    SALT_CUDA(cudaMemcpyAsync(out_host, out_dev, bytes, cudaMemcpyDeviceToHost, st));
    SALT_CUDA(cudaStreamSynchronize(st));
  }
  return 0;
}

int dispatch(int dtype, Plan& p, void* const* dsts, int ndst, const void* const* leaves,
             int nleaves, const double* scalars, int nscalars, i64 n, int flags, void* ws,
             size_t ws_bytes, void* out_dev, void* out_host, cudaStream_t st,
             const salt_exchange* x = nullptr, const void* const* pscalars = nullptr,
             int npscalars = 0) {
  if (dtype == SALT_F32)
    return run_fused<float>(p, dsts, ndst, leaves, nleaves, scalars, nscalars, n, flags, ws,
                            ws_bytes, out_dev, out_host, st, x, pscalars, npscalars);
  return run_fused<double>(p, dsts, ndst, leaves, nleaves, scalars, nscalars, n, flags, ws,
                           ws_bytes, out_dev, out_host, st, x, pscalars, npscalars);
}

// Batched assignments: problem table in the kernel parameters, up to
// BATCH_MAX problems (and < 2^31 tiles) per launch; trees beyond the batch
// limits, or without a kernel (no JIT), run one launch per problem.
template <class T>
int run_batch(Plan& p, int count, void* const* dsts, const void* const* leaves, int nleaves,
              const double* scalars, int nscalars, const int64_t* ns, cudaStream_t st) {
  if (count < 0 || (count > 0 && (!dsts || !ns || (nleaves > 0 && !leaves))))
    return fail(SALT_EINVAL, "bad batch arguments");
  for (int q = 0; q < count; ++q) {
    if (ns[q] < 0) return fail(SALT_EINVAL, "negative length");
    if (ns[q] == 0) continue;
    if (!dsts[q]) return fail(SALT_EINVAL, "NULL destination");
    for (int l = 0; l < p.nl; ++l)
      if (!leaves[(size_t)q * nleaves + l]) return fail(SALT_EINVAL, "NULL leaf pointer");
  }
  Kernel* k = nullptr;
  const bool batchable = p.sa.nroots == 1 && p.np == 0 && p.nl <= salt::BATCH_LEAVES &&
                         p.ns <= salt::BATCH_SCALARS;
  if (batchable) k = get_kernel(dtype_of<T>(), kBatchKind, vec_of<T>(), p.nl, p.sa.type, "batch");
  if (!k) {  // one fused launch per problem (table, JIT or interpreter kernel)
    for (int q = 0; q < count; ++q) {
      if (ns[q] == 0) continue;
      void* d = dsts[q];
      int rc = run_fused<T>(p, &d, 1, leaves + (size_t)q * nleaves, nleaves, scalars + (size_t)q * nscalars,
                            nscalars, ns[q], 0, nullptr, 0, nullptr, nullptr, st, nullptr, nullptr, 0);
      if (rc) return rc;
    }
    return 0;
  }
  int dev;
  int rc = current_device(dev);
  if (rc) return rc;
  rc = prepare(k, dev);
  if (rc) return rc;
  constexpr int V = vec_of<T>();
  const i64 per_tile = (i64)kBlock * k->unroll;
  auto args = std::make_unique<salt::BatchArgs<T>>();  // ~17 KB: not on the stack
  auto flush = [&]() -> int {
    if (args->count == 0) return 0;
    const salt::BatchProblem<T>& last = args->p[args->count - 1];
    const i64 tiles = last.tile0 + last.nst + (last.nvec + per_tile - 1) / per_tile;
    int r = launch_raw(k, dev, (int)tiles, args.get(), 0, st);
    args->count = 0;
    return r;
  };
  memset(args.get(), 0, sizeof(salt::BatchArgs<T>));
  i64 tile = 0;
  for (int q = 0; q < count; ++q) {
    const i64 n = ns[q];
    if (n == 0) continue;
    const void* const* lq = leaves + (size_t)q * nleaves;
    void* dq = dsts[q];
    int vec;
    i64 head, nvec;
    geometry<T>(&dq, 1, lq, p.nl, n, vec, head, nvec);
    if (vec == 1) {  // operands not sharing one 32-byte alignment: all scalar
      head = n;
      nvec = 0;
    }
    const i64 nscalar = head + (n - head - nvec * V);
    const i64 nst = (nscalar + kBlock - 1) / kBlock;
    const i64 ntiles = nst + (nvec + per_tile - 1) / per_tile;
    if (args->count == salt::BATCH_MAX || (args->count > 0 && tile + ntiles > i64(0x7fffffff))) {
      if ((rc = flush())) return rc;
      tile = 0;
    }
    if (ntiles > i64(0x7fffffff)) return fail(SALT_EINVAL, "batch problem too large for one launch");
    salt::BatchProblem<T>& P = args->p[args->count++];
    P.dst = (T*)dq;
    for (int l = 0; l < p.nl; ++l) P.leaf[l] = (const T*)lq[l];
    for (int c = 0; c < p.ns; ++c) P.sc[c] = (T)scalars[(size_t)q * nscalars + c];
    P.n = n;
    P.head = head;
    P.nvec = nvec;
    P.tile0 = tile;
    P.nst = nst;
    tile += ntiles;
  }
  return flush();
}

// Batched small reductions: problems of <= 2 tiles whose operands share the
// 32-byte alignment go into batch_reduce_kernel launches (one CTA each, the
// one-CTA fused order: same bits); the others run as ordinary reductions.
template <class T>
int run_reduce_batch(Plan& p, int count, const void* const* leaves, int nleaves, const double* scalars,
                     int nscalars, const int64_t* ns, int flags, void* const* outs, void* ws,
                     size_t ws_bytes, cudaStream_t st) {
  if (count < 0 || (count > 0 && (!ns || !outs || (nleaves > 0 && !leaves))))
    return fail(SALT_EINVAL, "bad batch arguments");
  if (flags & ~(SALT_SQRT | SALT_PARTIAL)) return fail(SALT_EINVAL, "reduce flags: SALT_SQRT, SALT_PARTIAL");
  for (int q = 0; q < count; ++q) {
    if (ns[q] < 0) return fail(SALT_EINVAL, "negative length");
    if (!outs[q]) return fail(SALT_EINVAL, "NULL reduction output");
    for (int l = 0; ns[q] > 0 && l < p.nl; ++l)
      if (!leaves[(size_t)q * nleaves + l]) return fail(SALT_EINVAL, "NULL leaf pointer");
  }
  Kernel* k = nullptr;
  if (p.np == 0 && p.nl <= salt::BATCH_LEAVES && p.ns <= salt::BATCH_SCALARS)
    k = get_kernel(dtype_of<T>(), kBatchReduceKind, vec_of<T>(), p.nl, "batch", p.sr.type);
  int dev, rc;
  if (k) {
    if ((rc = current_device(dev)) || (rc = prepare(k, dev))) return rc;
  }
  constexpr int V = vec_of<T>();
  const i64 per_tile = k ? (i64)kBlock * k->unroll : 0;
  auto args = std::make_unique<salt::BatchArgs<T>>();
  memset(args.get(), 0, sizeof(salt::BatchArgs<T>));
  auto flush = [&]() -> int {
    if (args->count == 0) return 0;
    void* params[] = {args.get(), &flags};
    const bool pdl = use_pdl();
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.gridDim = dim3(args->count);
    cfg.blockDim = dim3(kBlock);
    cfg.stream = st;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    if (k->aot) {
      cudaError_t e = cudaLaunchKernelExC(&cfg, k->aot, params);
      if (e != cudaSuccess) return cuda_fail(e, "cudaLaunchKernelExC(batch reduce)");
    } else {
      CUlaunchConfig c = {};
      CUlaunchAttribute at[1];
      at[0].id = CU_LAUNCH_ATTRIBUTE_PROGRAMMATIC_STREAM_SERIALIZATION;
      at[0].value.programmaticStreamSerializationAllowed = 1;
      c.gridDimX = (unsigned)args->count;
      c.gridDimY = c.gridDimZ = 1;
      c.blockDimX = kBlock;
      c.blockDimY = c.blockDimZ = 1;
      c.hStream = (CUstream)st;
      c.attrs = at;
      c.numAttrs = pdl && driver().LaunchKernelEx ? 1 : 0;
      CUresult r = driver().LaunchKernelEx
                       ? driver().LaunchKernelEx(&c, k->jit_fn[dev], params, nullptr)
                       : driver().LaunchKernel(k->jit_fn[dev], args->count, 1, 1, kBlock, 1, 1, 0,
                                               (CUstream)st, params, nullptr);
      if (r != CUDA_SUCCESS) return fail(SALT_ECUDA, "cuLaunchKernel(batch reduce) failed");
    }
    g_launches.fetch_add(1, std::memory_order_relaxed);
    args->count = 0;
    return 0;
  };
  for (int q = 0; q < count; ++q) {
    const i64 n = ns[q];
    const void* const* lq = leaves + (size_t)q * nleaves;
    int vec = V;
    i64 head = 0, nvec = 0;
    if (n > 0) geometry<T>(nullptr, 0, lq, p.nl, n, vec, head, nvec);
    if (k && vec == V && (nvec + per_tile - 1) / per_tile <= 2) {
      if (args->count == salt::BATCH_MAX && (rc = flush())) return rc;
      salt::BatchProblem<T>& P = args->p[args->count++];
      P.dst = (T*)outs[q];
      for (int l = 0; l < p.nl; ++l) P.leaf[l] = (const T*)lq[l];
      for (int c = 0; c < p.ns; ++c) P.sc[c] = (T)scalars[(size_t)q * nscalars + c];
      P.n = n;
      P.head = head;
      P.nvec = nvec;
      continue;
    }
    if ((rc = run_fused<T>(p, nullptr, 0, lq, nleaves, scalars + (size_t)q * nscalars, nscalars, n,
                           flags, ws, ws_bytes, outs[q], nullptr, st, nullptr, nullptr, 0)))
      return rc;
  }
  return k ? flush() : 0;
}

template <class T>
int finish(const void* parts, int count, int flags, void* out_dev, void* out_host,
           cudaStream_t st) {
  if (count < 0 || (count > 0 && !parts) || !out_dev) return fail(SALT_EINVAL, "bad finish arguments");
  void* params[] = {(void*)&parts, &count, &flags, &out_dev};
  SALT_CUDA(cudaLaunchKernel((const void*)&salt::finish_kernel<T, kBlock>, dim3(1), dim3(kBlock),
                             params, 0, st));
  g_launches.fetch_add(1, std::memory_order_relaxed);
  if (out_host) {
    size_t bytes = (flags & SALT_PARTIAL) ? sizeof(salt::DD) : sizeof(T);
    SALT_CUDA(cudaMemcpyAsync(out_host, out_dev, bytes, cudaMemcpyDeviceToHost, st));
    SALT_CUDA(cudaStreamSynchronize(st));
  }
  return 0;
}

// ------------------------------------------------------------------ single-process multi-GPU
// NCCL is loaded at run time (no link-time dependency): $SALT_NCCL_LIB, else
// the soname libnccl.so.2 — which resolves to the copy torch already loaded
// when torch is in the process — else the system library.
typedef int ncclResult_v;
struct Nccl {
  bool ok = false;
  std::string why;
  ncclResult_v (*CommInitAll)(void** comms, int ndev, const int* devlist) = nullptr;
  ncclResult_v (*CommDestroy)(void* comm) = nullptr;
  ncclResult_v (*CommCuDevice)(void* comm, int* device) = nullptr;
  ncclResult_v (*CommCount)(void* comm, int* count) = nullptr;
  ncclResult_v (*CommUserRank)(void* comm, int* rank) = nullptr;
  ncclResult_v (*GroupStart)() = nullptr;
  ncclResult_v (*GroupEnd)() = nullptr;
  ncclResult_v (*AllGather)(const void* send, void* recv, size_t count, int datatype, void* comm,
                            cudaStream_t stream) = nullptr;
  const char* (*GetErrorString)(ncclResult_v) = nullptr;
};
constexpr int kNcclFloat64 = 8;  // ncclFloat64 (nccl.h)

Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* env = getenv("SALT_NCCL_LIB");
    const char* cands[] = {env, "libnccl.so.2", "/usr/lib/x86_64-linux-gnu/libnccl.so.2"};
    void* h = nullptr;
    for (const char* c : cands) {
      if (!c) continue;
      h = dlopen(c, RTLD_NOW | RTLD_LOCAL);
      if (h) break;
    }
    if (!h) {
      n.why = "libnccl.so.2 not found (set SALT_NCCL_LIB)";
      return;
    }
#define SYM(F, NAME)                                        \
  n.F = reinterpret_cast<decltype(n.F)>(dlsym(h, NAME));    \
  if (!n.F) { n.why = std::string("nccl symbol missing: ") + NAME; return; }
    SYM(CommInitAll, "ncclCommInitAll");
    SYM(CommDestroy, "ncclCommDestroy");
    SYM(CommCuDevice, "ncclCommCuDevice");
    SYM(CommCount, "ncclCommCount");
    SYM(CommUserRank, "ncclCommUserRank");
    SYM(GroupStart, "ncclGroupStart");
    SYM(GroupEnd, "ncclGroupEnd");
    SYM(AllGather, "ncclAllGather");
    SYM(GetErrorString, "ncclGetErrorString");
#undef SYM
    n.ok = true;
  });
  return n;
}

int nccl_fail(ncclResult_v r, const char* what) {
  return fail(SALT_ECUDA, std::string(what) + ": " + (nccl().GetErrorString ? nccl().GetErrorString(r) : "nccl error"));
}

// Restores the caller's current device on scope exit.
struct DeviceGuard {
  int dev = -1;
  DeviceGuard() { cudaGetDevice(&dev); }
  ~DeviceGuard() { if (dev >= 0) cudaSetDevice(dev); }
};

// G per-device {hi, lo} partials -> every device holds the rank-ordered fold
// (finish_kernel: the same arithmetic as salt_reduce_finish and the NVLink
// exchange, so all three multi-GPU paths give identical bits).  One group of
// G all-gathers of 16 bytes, then one finish kernel per device, all
// enqueued on the callers' streams; gathered partials live in stream-ordered
// allocations freed on the same streams.
int allreduce_sum(void* const* out_dev, int G, int dtype, void* const* comms, void* const* streams,
                  int flags) {
  if (G < 1 || !out_dev || !comms || !streams) return fail(SALT_EINVAL, "bad allreduce arguments");
  if (dtype != SALT_F32 && dtype != SALT_F64) return fail(SALT_EINVAL, "dtype must be SALT_F32 or SALT_F64");
  if (flags & ~SALT_SQRT) return fail(SALT_EINVAL, "allreduce flags: only SALT_SQRT");
  Nccl& nc = nccl();
  if (!nc.ok) return fail(SALT_ECUDA, nc.why);
  DeviceGuard guard;
  std::vector<int> devs(G);
  std::vector<void*> gathered(G, nullptr);
  auto release = [&]() {
    for (int g = 0; g < G; ++g)
      if (gathered[g]) {
        cudaSetDevice(devs[g]);
        cudaFreeAsync(gathered[g], (cudaStream_t)streams[g]);
      }
  };
  for (int g = 0; g < G; ++g) {
    if (!out_dev[g] || !comms[g]) return fail(SALT_EINVAL, "NULL partial or communicator");
    int count = 0, rank = -1;
    ncclResult_v r = nc.CommCuDevice(comms[g], &devs[g]);
    if (!r) r = nc.CommCount(comms[g], &count);
    if (!r) r = nc.CommUserRank(comms[g], &rank);
    if (r) return nccl_fail(r, "ncclComm query");
    if (count != G || rank != g) return fail(SALT_EINVAL, "comms[g] must be rank g of a G-rank communicator");
  }
  for (int g = 0; g < G; ++g) {
    cudaError_t e = cudaSetDevice(devs[g]);
    if (e == cudaSuccess) e = cudaMallocAsync(&gathered[g], (size_t)G * sizeof(salt::DD), (cudaStream_t)streams[g]);
    if (e != cudaSuccess) { release(); return cuda_fail(e, "cudaMallocAsync(gathered partials)"); }
  }
  ncclResult_v r = nc.GroupStart();
  for (int g = 0; g < G && !r; ++g)
    r = nc.AllGather(out_dev[g], gathered[g], 2, kNcclFloat64, comms[g], (cudaStream_t)streams[g]);
  ncclResult_v r2 = nc.GroupEnd();
  if (r || r2) { release(); return nccl_fail(r ? r : r2, "ncclAllGather"); }
  int rc = 0;
  for (int g = 0; g < G && !rc; ++g) {
    cudaError_t e = cudaSetDevice(devs[g]);
    if (e != cudaSuccess) { rc = cuda_fail(e, "cudaSetDevice"); break; }
    rc = dtype == SALT_F32 ? finish<float>(gathered[g], G, flags, out_dev[g], nullptr, (cudaStream_t)streams[g])
                           : finish<double>(gathered[g], G, flags, out_dev[g], nullptr, (cudaStream_t)streams[g]);
  }
  release();
  return rc;
}

// ------------------------------------------------------------------ host streaming
struct Events {
  std::vector<cudaEvent_t> ev;
  ~Events() { for (auto e : ev) cudaEventDestroy(e); }
  int make(int count) {
    ev.resize(count, nullptr);
    for (auto& e : ev) SALT_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    return 0;
  }
};

constexpr int kNBuf = 3;
constexpr i64 kMaxChunk = i64(1) << 23;

// Shared by assign (reduce == false) and reduce: stream chunk c of every
// operand through buffer c % 3; the fused kernel runs on streams[1].
int host_pipeline(int dtype, Plan& p, void* host_dst, const void* const* host_leaves,
                  int nleaves, const double* scalars, int nscalars, i64 n, int flags,
                  void* staging, size_t staging_bytes, void* const* streams3, void* out_host) {
  const bool reduce = p.mode != salt::MODE_ASSIGN;   // produces a sum
  const bool has_dst = p.mode != salt::MODE_REDUCE;  // streams a destination back
  const size_t esz = dtype == SALT_F32 ? 4 : 8;
  if (n < 0) return fail(SALT_EINVAL, "negative length");
  if (!streams3 || !staging) return fail(SALT_EINVAL, "NULL staging or streams");
  if (!reduce && n == 0) return 0;
  cudaStream_t sh = (cudaStream_t)streams3[0], sc = (cudaStream_t)streams3[1],
               sd = (cudaStream_t)streams3[2];
  if (has_dst && p.sa.nroots != 1)
    return fail(SALT_EINVAL, "host streaming takes exactly one assignment root");
  const int nl = p.nl;
  const int nbufs_per_set = nl + (has_dst ? 1 : 0);
  // staging: [reduce workspace][chunk partials][result 256B][kNBuf x (nl leaves + dst)]
  size_t ws = reduce ? salt_reduce_workspace_bytes() : 0;
  size_t fixed = ws + (reduce ? 256 * 1024 : 0) + 256;
  if (staging_bytes <= fixed + 256) return fail(SALT_EWORKSPACE, "staging too small");
  i64 chunk = (i64)((staging_bytes - fixed) / (kNBuf * nbufs_per_set * esz));
  chunk = chunk / 64 * 64;
  static const i64 max_chunk = [] {  // SALT_HOST_CHUNK (elements; tuning only)
    const char* e = getenv("SALT_HOST_CHUNK");
    const long long v = e ? atoll(e) : 0;
    return v >= 64 ? (i64)(v / 64 * 64) : kMaxChunk;
  }();
  if (chunk > max_chunk) chunk = max_chunk;
  if (chunk < 64) return fail(SALT_EWORKSPACE, "staging too small for one chunk");
  const i64 nchunks = (n + chunk - 1) / chunk;
  if (reduce && nchunks * (i64)sizeof(salt::DD) > 256 * 1024)
    return fail(SALT_EWORKSPACE, "too many chunks for the partial buffer; enlarge staging");
  char* base = (char*)staging;
  void* wsp = base;
  salt::DD* parts = (salt::DD*)(base + ws);
  void* result = base + ws + (reduce ? 256 * 1024 : 0);
  char* bufs = base + fixed;
  auto buf = [&](int b, int i) -> void* {
    return bufs + ((size_t)b * nbufs_per_set + i) * chunk * esz;
  };
  if (reduce) SALT_CUDA(cudaMemsetAsync(wsp, 0, SALT_WORKSPACE_TICKET_BYTES, sc));
  Events h2d, comp, d2h;
  int rc = h2d.make(kNBuf);
  if (!rc) rc = comp.make(kNBuf);
  if (!rc) rc = d2h.make(kNBuf);
  if (rc) return rc;
  for (i64 c = 0; c < nchunks; ++c) {
    const int b = (int)(c % kNBuf);
    const i64 off = c * chunk;
    const i64 m = std::min(chunk, n - off);
    if (c >= kNBuf) SALT_CUDA(cudaStreamWaitEvent(sh, comp.ev[b], 0));
    const void* dleaves[salt::MAX_LEAVES];
    for (int l = 0; l < nl; ++l) {
      SALT_CUDA(cudaMemcpyAsync(buf(b, l), (const char*)host_leaves[l] + off * esz, m * esz,
                                cudaMemcpyHostToDevice, sh));
      dleaves[l] = buf(b, l);
    }
    SALT_CUDA(cudaEventRecord(h2d.ev[b], sh));
    SALT_CUDA(cudaStreamWaitEvent(sc, h2d.ev[b], 0));
    if (has_dst && c >= kNBuf) SALT_CUDA(cudaStreamWaitEvent(sc, d2h.ev[b], 0));
    void* ddst = has_dst ? buf(b, nl) : nullptr;
    rc = dispatch(dtype, p, &ddst, has_dst ? 1 : 0, dleaves, nleaves, scalars, nscalars, m,
                  reduce ? SALT_PARTIAL : 0, wsp, ws, reduce ? (void*)(parts + c) : nullptr,
                  nullptr, sc);
    if (rc) return rc;
    SALT_CUDA(cudaEventRecord(comp.ev[b], sc));
    if (has_dst) {
      SALT_CUDA(cudaStreamWaitEvent(sd, comp.ev[b], 0));
      SALT_CUDA(cudaMemcpyAsync((char*)host_dst + off * esz, ddst, m * esz,
                                cudaMemcpyDeviceToHost, sd));
      SALT_CUDA(cudaEventRecord(d2h.ev[b], sd));
    }
  }
  if (reduce) {
    if (nchunks == 0) {
      // zero length: the sum is dtype(0) (test_engine.py:147-153)
      void* hdst = host_dst;
      rc = dispatch(dtype, p, &hdst, has_dst ? 1 : 0, host_leaves, nleaves, scalars, nscalars, 0, flags, wsp, ws,
                    result, out_host, sc);
      if (rc) return rc;
    } else {
      rc = dtype == SALT_F32 ? finish<float>(parts, (int)nchunks, flags, result, out_host, sc)
                             : finish<double>(parts, (int)nchunks, flags, result, out_host, sc);
      if (rc) return rc;
    }
  }
  SALT_CUDA(cudaStreamSynchronize(sh));
  SALT_CUDA(cudaStreamSynchronize(sc));
  SALT_CUDA(cudaStreamSynchronize(sd));
  return 0;
}

}  // namespace

// ====================================================================== C ABI
extern "C" {

int salt_abi_version(void) { return SALT_ABI_VERSION; }

const char* salt_last_error(void) { return g_err.c_str(); }

uint64_t salt_launch_count(void) { return g_launches.load(); }

void salt_set_force_jit(int on) { g_force_jit.store(on ? 1 : 0); }

void salt_set_force_interp(int on) { g_force_interp.store(on ? 1 : 0); }

void salt_set_jit_async(int on) { g_jit_async.store(on ? 1 : 0); }

int salt_jit_wait(void) {
  AsyncJit& A = async_jit();
  std::unique_lock<std::mutex> lk(A.mu);
  A.idle.wait(lk, [&] { return A.queue.empty() && A.active == 0; });
  return (int)A.failed.size();
}

uint64_t salt_interp_launch_count(void) { return g_interp_launches.load(); }

size_t salt_reduce_workspace_bytes(void) { return (size_t)salt::WsLayout::bytes; }

int salt_signature_kind(int dtype, const char* sig, const char* reduce_sig, int kind) {
  if (kind < 0 || kind > 2) return 0;
  Plan* p;
  const char* a = kind == 1 ? nullptr : sig;
  const char* r = kind == 0 ? nullptr : (kind == 1 ? sig : reduce_sig);
  if (make_plan(dtype, a, r, kind, salt::MAX_LEAVES, salt::MAX_SCALARS, p)) return 0;
  ensure_table();
  const int V = dtype == SALT_F32 ? 8 : 4;
  std::lock_guard<std::mutex> lk(g_table_mu);
  return table().count(key_of(dtype, kind, V, p->sa.type, p->sr.type)) ? 1 : 2;
}

int salt_prepare(int dtype, const char* sig, const char* reduce_sig, int kind) {
  if (kind < 0 || kind > 2) return fail(SALT_EINVAL, "kind must be 0, 1 or 2");
  Plan* p;
  const char* a = kind == 1 ? nullptr : sig;
  const char* r = kind == 0 ? nullptr : (kind == 1 ? sig : reduce_sig);
  int rc = make_plan(dtype, a, r, kind, salt::MAX_LEAVES, salt::MAX_SCALARS, p);
  if (rc) return rc;
  const int V = dtype == SALT_F32 ? 8 : 4;
  for (int vec : {V, 1})
    if (!get_kernel(dtype, kind, vec, p->nl, p->sa.type, p->sr.type)) return SALT_EJIT;
  return 0;
}

int salt_assign(int dtype, const char* sig, void* dst, const void* const* leaves, int nleaves,
                const double* scalars, int nscalars, int64_t n, void* stream) {
  Plan* p;
  int rc = make_plan(dtype, sig, nullptr, salt::MODE_ASSIGN, nleaves, nscalars, p);
  if (rc) return rc;
  return dispatch(dtype, *p, &dst, 1, leaves, nleaves, scalars, nscalars, n, 0, nullptr, 0, nullptr,
                  nullptr, (cudaStream_t)stream);
}

int salt_reduce(int dtype, const char* sig, const void* const* leaves, int nleaves,
                const double* scalars, int nscalars, int64_t n, int flags, void* workspace,
                size_t workspace_bytes, void* out_dev, void* out_host, void* stream) {
  Plan* p;
  int rc = make_plan(dtype, nullptr, sig, salt::MODE_REDUCE, nleaves, nscalars, p);
  if (rc) return rc;
  return dispatch(dtype, *p, nullptr, 0, leaves, nleaves, scalars, nscalars, n, flags, workspace,
                  workspace_bytes, out_dev, out_host, (cudaStream_t)stream);
}

int salt_assign_reduce(int dtype, const char* assign_sig, const char* reduce_sig, void* dst,
                       const void* const* leaves, int nleaves, const double* scalars,
                       int nscalars, int64_t n, int flags, void* workspace,
                       size_t workspace_bytes, void* out_dev, void* out_host, void* stream) {
  Plan* p;
  int rc = make_plan(dtype, assign_sig, reduce_sig, salt::MODE_ASSIGN_REDUCE, nleaves, nscalars, p);
  if (rc) return rc;
  return dispatch(dtype, *p, &dst, 1, leaves, nleaves, scalars, nscalars, n, flags, workspace,
                  workspace_bytes, out_dev, out_host, (cudaStream_t)stream);
}

int salt_reduce_exchange(int dtype, const char* sig, const void* const* leaves, int nleaves,
                         const double* scalars, int nscalars, int64_t n, int flags, void* workspace,
                         size_t workspace_bytes, const salt_exchange* exchange, void* out_dev,
                         void* out_host, void* stream) {
  if (!exchange) return fail(SALT_EINVAL, "NULL exchange descriptor");
  Plan* p;
  int rc = make_plan(dtype, nullptr, sig, salt::MODE_REDUCE, nleaves, nscalars, p);
  if (rc) return rc;
  return dispatch(dtype, *p, nullptr, 0, leaves, nleaves, scalars, nscalars, n, flags, workspace,
                  workspace_bytes, out_dev, out_host, (cudaStream_t)stream, exchange);
}

int salt_assign_reduce_exchange(int dtype, const char* assign_sig, const char* reduce_sig,
                                void* dst, const void* const* leaves, int nleaves,
                                const double* scalars, int nscalars, int64_t n, int flags,
                                void* workspace, size_t workspace_bytes,
                                const salt_exchange* exchange, void* out_dev, void* out_host,
                                void* stream) {
  if (!exchange) return fail(SALT_EINVAL, "NULL exchange descriptor");
  Plan* p;
  int rc = make_plan(dtype, assign_sig, reduce_sig, salt::MODE_ASSIGN_REDUCE, nleaves, nscalars, p);
  if (rc) return rc;
  return dispatch(dtype, *p, &dst, 1, leaves, nleaves, scalars, nscalars, n, flags, workspace,
                  workspace_bytes, out_dev, out_host, (cudaStream_t)stream, exchange);
}

int salt_fused_exchange(int dtype, const char* assign_sigs, const char* reduce_sig,
                        void* const* dsts, int ndst, const void* const* leaves, int nleaves,
                        const double* scalars, int nscalars, const void* const* pscalars,
                        int npscalars, int64_t n, int flags, void* workspace,
                        size_t workspace_bytes, const salt_exchange* exchange, void* out_dev,
                        void* out_host, void* stream) {
  if (!exchange) return fail(SALT_EINVAL, "NULL exchange descriptor");
  if (!reduce_sig) return fail(SALT_EINVAL, "salt_fused_exchange needs a reduction");
  Plan* p;
  const int mode = assign_sigs ? salt::MODE_ASSIGN_REDUCE : salt::MODE_REDUCE;
  int rc = make_plan(dtype, assign_sigs, reduce_sig, mode, nleaves, nscalars, p);
  if (rc) return rc;
  return dispatch(dtype, *p, dsts, ndst, leaves, nleaves, scalars, nscalars, n, flags, workspace,
                  workspace_bytes, out_dev, out_host, (cudaStream_t)stream, exchange, pscalars,
                  npscalars);
}

int salt_exchange_emulate(int world, int rounds, uint64_t epoch0, const void* totals_dev,
                          void* results_dev, void* scratch_dev, void* stream) {
  if (world < 1 || world > salt::XCHG_MAX_RANKS || rounds < 1 || epoch0 == 0 || !totals_dev ||
      !results_dev || !scratch_dev)
    return fail(SALT_EINVAL, "bad exchange emulation arguments");
  // scratch: per rank 512 bytes: [DD slots 2 x 8 | u64 flags 8]; the kernel
  // takes the slot arrays first, then the flag arrays, so lay them out apart.
  salt::DD* slots = (salt::DD*)scratch_dev;
  unsigned long long* flags =
      (unsigned long long*)((char*)scratch_dev + (size_t)world * 2 * salt::XCHG_MAX_RANKS * sizeof(salt::DD));
  const salt::DD* totals = (const salt::DD*)totals_dev;
  salt::DD* results = (salt::DD*)results_dev;
  unsigned long long e0 = epoch0;
  void* params[] = {(void*)&totals, (void*)&results, (void*)&slots, (void*)&flags, &world, &rounds, &e0};
  SALT_CUDA(cudaLaunchCooperativeKernel((const void*)&salt::exchange_emulate_kernel, dim3(world),
                                        dim3(32), params, 0, (cudaStream_t)stream));
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return 0;
}

int salt_fused(int dtype, const char* assign_sigs, const char* reduce_sig, void* const* dsts,
               int ndst, const void* const* leaves, int nleaves, const double* scalars,
               int nscalars, const void* const* pscalars, int npscalars, int64_t n, int flags,
               void* workspace, size_t workspace_bytes, void* out_dev, void* out_host,
               void* stream) {
  Plan* p;
  if (!assign_sigs && !reduce_sig) return fail(SALT_EINVAL, "nothing to evaluate");
  const int mode = !assign_sigs ? salt::MODE_REDUCE
                   : reduce_sig ? salt::MODE_ASSIGN_REDUCE : salt::MODE_ASSIGN;
  int rc = make_plan(dtype, assign_sigs, reduce_sig, mode, nleaves, nscalars, p);
  if (rc) return rc;
  return dispatch(dtype, *p, dsts, ndst, leaves, nleaves, scalars, nscalars, n, flags, workspace,
                  workspace_bytes, out_dev, out_host, (cudaStream_t)stream, nullptr, pscalars,
                  npscalars);
}

int salt_reduce_finish(int dtype, const void* partials_dev, int count, int flags, void* out_dev,
                       void* out_host, void* stream) {
  if (dtype == SALT_F32)
    return finish<float>(partials_dev, count, flags, out_dev, out_host, (cudaStream_t)stream);
  if (dtype == SALT_F64)
    return finish<double>(partials_dev, count, flags, out_dev, out_host, (cudaStream_t)stream);
  return fail(SALT_EINVAL, "dtype must be SALT_F32 or SALT_F64");
}

int salt_assign_batch(int dtype, const char* sig, int count, void* const* dsts,
                      const void* const* leaves, int nleaves, const double* scalars, int nscalars,
                      const int64_t* ns, void* stream) {
  Plan* p;
  int rc = make_plan(dtype, sig, nullptr, salt::MODE_ASSIGN, nleaves, nscalars, p);
  if (rc) return rc;
  if (dtype == SALT_F32)
    return run_batch<float>(*p, count, dsts, leaves, nleaves, scalars, nscalars, ns, (cudaStream_t)stream);
  return run_batch<double>(*p, count, dsts, leaves, nleaves, scalars, nscalars, ns, (cudaStream_t)stream);
}

int salt_reduce_batch(int dtype, const char* sig, int count, const void* const* leaves, int nleaves,
                      const double* scalars, int nscalars, const int64_t* ns, int flags,
                      void* const* outs, void* workspace, size_t workspace_bytes, void* stream) {
  Plan* p;
  int rc = make_plan(dtype, nullptr, sig, salt::MODE_REDUCE, nleaves, nscalars, p);
  if (rc) return rc;
  if (dtype == SALT_F32)
    return run_reduce_batch<float>(*p, count, leaves, nleaves, scalars, nscalars, ns, flags, outs, workspace,
                                   workspace_bytes, (cudaStream_t)stream);
  return run_reduce_batch<double>(*p, count, leaves, nleaves, scalars, nscalars, ns, flags, outs, workspace,
                                  workspace_bytes, (cudaStream_t)stream);
}

int salt_assign_host(int dtype, const char* sig, void* host_dst, const void* const* host_leaves,
                     int nleaves, const double* scalars, int nscalars, int64_t n, void* staging,
                     size_t staging_bytes, void* const* streams3) {
  Plan* p;
  int rc = make_plan(dtype, sig, nullptr, salt::MODE_ASSIGN, nleaves, nscalars, p);
  if (rc) return rc;
  if (!host_dst) return fail(SALT_EINVAL, "NULL destination");
  return host_pipeline(dtype, *p, host_dst, host_leaves, nleaves, scalars, nscalars, n, 0, staging,
                       staging_bytes, streams3, nullptr);
}

int salt_assign_reduce_host(int dtype, const char* assign_sig, const char* reduce_sig,
                            void* host_dst, const void* const* host_leaves, int nleaves,
                            const double* scalars, int nscalars, int64_t n, int flags,
                            void* staging, size_t staging_bytes, void* const* streams3,
                            void* out_host) {
  Plan* p;
  int rc = make_plan(dtype, assign_sig, reduce_sig, salt::MODE_ASSIGN_REDUCE, nleaves, nscalars, p);
  if (rc) return rc;
  if (!host_dst || !out_host) return fail(SALT_EINVAL, "NULL destination or out_host");
  return host_pipeline(dtype, *p, host_dst, host_leaves, nleaves, scalars, nscalars, n, flags,
                       staging, staging_bytes, streams3, out_host);
}

int salt_reduce_host(int dtype, const char* sig, const void* const* host_leaves, int nleaves,
                     const double* scalars, int nscalars, int64_t n, int flags, void* staging,
                     size_t staging_bytes, void* const* streams3, void* out_host) {
  Plan* p;
  int rc = make_plan(dtype, nullptr, sig, salt::MODE_REDUCE, nleaves, nscalars, p);
  if (rc) return rc;
  if (!out_host) return fail(SALT_EINVAL, "NULL out_host");
  return host_pipeline(dtype, *p, nullptr, host_leaves, nleaves, scalars, nscalars, n, flags,
                       staging, staging_bytes, streams3, out_host);
}

int salt_nccl_comm_init_all(int G, const int* devices, void** comms_out) {
  if (G < 1 || !comms_out) return fail(SALT_EINVAL, "bad communicator arguments");
  Nccl& nc = nccl();
  if (!nc.ok) return fail(SALT_ECUDA, nc.why);
  DeviceGuard guard;
  ncclResult_v r = nc.CommInitAll(comms_out, G, devices);
  return r ? nccl_fail(r, "ncclCommInitAll") : 0;
}

int salt_nccl_comm_destroy(int G, void** comms) {
  if (G < 1 || !comms) return fail(SALT_EINVAL, "bad communicator arguments");
  Nccl& nc = nccl();
  if (!nc.ok) return fail(SALT_ECUDA, nc.why);
  int rc = 0;
  for (int g = 0; g < G; ++g)
    if (comms[g]) {
      ncclResult_v r = nc.CommDestroy(comms[g]);
      if (r && !rc) rc = nccl_fail(r, "ncclCommDestroy");
      comms[g] = nullptr;
    }
  return rc;
}

int salt_allreduce_sum(void* out_dev_per_gpu[], int G, int dtype, void* comms, void* streams[]) {
  return allreduce_sum(out_dev_per_gpu, G, dtype, (void* const*)comms, streams, 0);
}

int salt_allreduce_sum_flags(void* out_dev_per_gpu[], int G, int dtype, void* comms,
                             void* streams[], int flags) {
  return allreduce_sum(out_dev_per_gpu, G, dtype, (void* const*)comms, streams, flags);
}

}  // extern "C"
