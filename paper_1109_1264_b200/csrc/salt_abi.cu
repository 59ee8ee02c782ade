// salt_abi.cu — libsalt.so: the C ABI declared in include/salt.h.
//
// Host runtime around the kernels of salt_expr.cuh / salt_interp.cuh, one
// translation unit in six parts:
//   salt_abi_signatures.inc  postfix signature parsing / validation (salt.h)
//   salt_abi_jit.inc         driver / NVRTC loading; the kernel table —
//                            compiled-in (AOT, sm_100a) instantiations for
//                            the reference's named ops and the BASELINE
//                            trees — plus the NVRTC JIT that instantiates the
//                            SAME templates for any other tree (disk cache,
//                            module per device, opt-in tiered build)
//   this file                launch geometry (tiles per CTA, reduction
//                            groups, one-cluster small reductions), PDL
//                            launches, plans, the interpreter fallback,
//                            run_fused / dispatch
//   salt_abi_batch.inc       batched assignments and small reductions
//   salt_abi_nccl.inc        single-process multi-GPU all-reduce (NCCL)
//   salt_abi_host.inc        host-buffer streaming (H2D / kernel / D2H on
//                            three streams) for end-to-end evaluation
// followed by the extern "C" entry points.
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
constexpr int kInterpSmemCap = 216 * 1024;  // dynamic shared memory of the interpreter kernel (27 slots)
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
// V == 1 fallback (operands that do not share one 32-byte misalignment):
// elements in flight per leaf per thread.  64 bytes per leaf, like the vector
// kernels' two 256-bit loads (32 with five or more leaves, for the
// registers): with 4 elements (16-32 bytes) a misaligned f64 dot ran at
// 4.6 TB/s and an f32 one at 5.3 against 7.2-7.3 aligned
// (profiles/r02_misaligned.json).
constexpr int unroll_scalar(int elem_bytes, int nl) {
  return (elem_bytes == 8 ? 8 : 16) / (nl > 4 ? 2 : 1);
}
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

// Collector combine (salt_expr.cuh collect_epilogue) for reductions whose
// grid has between collect_min() and MAX_COLLECT streaming CTAs of
// collect_tiles() tiles each; SALT_COMBINE=ticket disables it (tests,
// tuning), SALT_COLLECT_TILES / SALT_COLLECT_MIN tune it (tools/c3_probe.cu).
bool collect_enabled() {
  static const bool env = [] {
    const char* e = getenv("SALT_COMBINE");
    return !(e && std::string(e) == "ticket");
  }();
  return env;
}
int collect_tiles() {
  static const int env = [] {
    const char* e = getenv("SALT_COLLECT_TILES");
    return e ? atoi(e) : 0;
  }();
  // 1 tile per streaming CTA: the block scheduler refills an SM the moment
  // a CTA retires, as for assignments (same-box A/B over 1-4 tiles,
  // profiles/r02_collect_tiles_ab.txt: 1 equal or better for dot / nrm2,
  // f32 / f64, 2^22-2^27)
  return env > 0 ? env : 1;
}
// Collector warps for a grid of `nstream` streaming CTAs (a function of n
// only, so the fold order — and the bits — still depend only on n).  The
// collector must retire slots as fast as the streaming CTAs fill them: f32
// nrm2 at 2^28 completes ~220 slots per microsecond, and two warps x 4 slots
// per L2 round trip fell behind there once the cheap epilogue shortened the
// streaming CTAs (168 us against a 147 us floor; four warps: 148 us,
// profiles/r02_cheap_epilogue.txt).  Below 8,192 streaming CTAs two warps
// are equal or a little better (fewer warps polling beside the streaming
// CTAs of that SM), and below 128 one warp is (~0.1 us,
// profiles/r02_collector_small_grids.txt).
int collect_warps(i64 nstream) {
  static const int env = [] {
    const char* e = getenv("SALT_COLLECT_WARPS");
    return e ? atoi(e) : 0;
  }();
  if (env >= 1 && env <= 8) return env;
  return nstream >= 8192 ? 4 : nstream >= 128 ? 2 : 1;
}
int collect_min() {
  static const int env = [] {
    const char* e = getenv("SALT_COLLECT_MIN");
    return e ? atoi(e) : -1;
  }();
  return env >= 0 ? env : 3;
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

// salt_set_trace: this host thread's device trace buffer (nullptr: off)
thread_local long long* g_trace_buf = nullptr;
thread_local long long g_trace_cap = 0;

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

#include "salt_abi_signatures.inc"

#include "salt_abi_jit.inc"

std::mutex g_dev_mu;

// The interpreter kernels: per element type, the vector width and unroll of
// every compiled kernel (so the interpreter walks the same tiles and its
// reductions add in the same order).
template <class T> Kernel* interp_kernel_for(int vec, int unroll, int nl) {
  static Kernel k2, k4, k1, k1h;
  static std::once_flag once;
  constexpr int U1 = unroll_scalar((int)sizeof(T), 1), U1H = unroll_scalar((int)sizeof(T), 8);
  std::call_once(once, [] {
    k2.aot = (const void*)&salt::interp_kernel<T, vec_of<T>(), 2, kBlock>;
    k4.aot = (const void*)&salt::interp_kernel<T, vec_of<T>(), 4, kBlock>;
    k1.aot = (const void*)&salt::interp_kernel<T, 1, U1, kBlock>;
    k1h.aot = (const void*)&salt::interp_kernel<T, 1, U1H, kBlock>;
    k2.vec = k4.vec = vec_of<T>();
    k1.vec = k1h.vec = 1;
    k2.unroll = 2;
    k4.unroll = 4;
    k1.unroll = U1;
    k1h.unroll = U1H;
    k2.interp = k4.interp = k1.interp = k1h.interp = true;
  });
  if (vec == 1) return unroll_scalar((int)sizeof(T), nl) == U1 ? &k1 : &k1h;
  return unroll == 4 ? &k4 : &k2;
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
  Kernel* cached[2][4] = {};  // [force_jit][(V == 1) + 2 * (small assignment)]: lookups done once
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
  // 8 KiB per slot (32-byte vectors x 256 threads); 27 slots + the 4 KiB of
  // static shared memory the reduction epilogue's CTA fold uses stay below
  // the 227 KiB a CTA may have
  if (salt::interp_smem_bytes(g, 4, kBlock, 8) > kInterpSmemCap)
    return "tree needs " + std::to_string(g.nl + g.slots + g.nroots) +
           " interpreter slots (leaves + stack depth + roots > 27)";
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

// A reduction's result to the caller's host memory (blocking).  Copying a
// few bytes into PAGEABLE memory costs ~3 us more than into pinned memory
// (the driver stages it), so each host thread gets one 64-byte slot of a
// small pinned pool, claimed once; beyond the pool, threads copy directly.
constexpr int kResultSlots = 256;
std::atomic<int> g_result_slot_next{0};
std::atomic<bool> g_result_pool_mapped{false};
// This host thread's 64-byte pinned result slot (nullptr beyond the pool).
char* thread_result_slot() {
  static char* pool = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    if (cudaHostAlloc((void**)&pool, kResultSlots * 64, cudaHostAllocPortable | cudaHostAllocMapped) !=
        cudaSuccess) {
      cudaGetLastError();
      pool = nullptr;
    }
    // Under unified addressing a kernel can store through the host pointer
    // itself (salt_result_slot); anything else keeps the copy route.
    void* dev = nullptr;
    if (pool && cudaHostGetDevicePointer(&dev, pool, 0) == cudaSuccess && dev == (void*)pool)
      g_result_pool_mapped.store(true, std::memory_order_release);
    else
      cudaGetLastError();
  });
  thread_local int slot = -2;  // -2: not claimed yet, -1: none (direct copy)
  if (slot == -2) {
    const int k = g_result_slot_next.fetch_add(1, std::memory_order_relaxed);
    slot = pool && k < kResultSlots ? k : -1;
  }
  return slot >= 0 ? pool + 64 * slot : nullptr;
}

int result_to_host(void* out_host, const void* out_dev, size_t bytes, cudaStream_t st) {
  char* pinned = thread_result_slot();
  void* dst = pinned ? (void*)pinned : out_host;
  SALT_CUDA(cudaMemcpyAsync(dst, out_dev, bytes, cudaMemcpyDeviceToHost, st));
  SALT_CUDA(cudaStreamSynchronize(st));
  if (dst != out_host) memcpy(out_host, dst, bytes);
  return 0;
}

// Split form for hosts that release a lock while waiting (the CPython fast
// path drops the GIL): enqueue the copy into this thread's pinned slot; the
// caller synchronises the stream, then reads *host_slot.
int result_enqueue(const void* out_dev, size_t bytes, cudaStream_t st, void** host_slot) {
  char* pinned = thread_result_slot();
  if (!pinned) {  // beyond the pool's threads: a pinned slot of this thread's own
    thread_local char* own = nullptr;
    if (!own) SALT_CUDA(cudaHostAlloc((void**)&own, 64, cudaHostAllocPortable));
    pinned = own;
  }
  SALT_CUDA(cudaMemcpyAsync(pinned, out_dev, bytes, cudaMemcpyDeviceToHost, st));
  *host_slot = pinned;
  return 0;
}

// Parse a scalar program (include/salt.h salt_fused_prog): tokens
// "p<i>" (raw device scalar i), "S<j>" (host scalar j), "+ - * /", "neg",
// "=<k>" (pop into the tree's P<k>).  Checks indices and the stack; `defined`
// gets bit k for every P<k> the program writes.  Cached per thread by text.
int parse_sprog(const char* text, int nraw, int nhost, salt::SProg& out, unsigned& defined) {
  thread_local std::unordered_map<std::string, std::pair<salt::SProg, unsigned>> cache;
  auto it = cache.find(text);
  if (it == cache.end()) {
    salt::SProg sp;
    memset(&sp, 0, sizeof sp);
    unsigned def = 0;
    int depth = 0;
    std::istringstream in(text);
    std::string tok;
    while (in >> tok) {
      if (sp.len == salt::SPROG_MAX) return fail(SALT_EINVAL, "scalar program longer than 32 ops");
      int op, arg = 0;
      if ((tok[0] == 'p' || tok[0] == 'S' || tok[0] == '=') && tok.size() > 1) {
        char* end = nullptr;
        const long v = strtol(tok.c_str() + 1, &end, 10);
        if (*end || v < 0 || v > 255) return fail(SALT_EINVAL, "bad scalar program token '" + tok + "'");
        arg = (int)v;
        op = tok[0] == 'p' ? salt::SP_RAW : tok[0] == 'S' ? salt::SP_HOST : salt::SP_OUT;
      } else if (tok == "+") op = salt::SP_ADD;
      else if (tok == "-") op = salt::SP_SUB;
      else if (tok == "*") op = salt::SP_MUL;
      else if (tok == "/") op = salt::SP_DIV;
      else if (tok == "neg") op = salt::SP_NEG;
      else return fail(SALT_EINVAL, "bad scalar program token '" + tok + "'");
      if (op == salt::SP_RAW || op == salt::SP_HOST) {
        if (++depth > salt::SPROG_STACK) return fail(SALT_EINVAL, "scalar program stack deeper than 8");
      } else if (op == salt::SP_NEG) {
        if (depth < 1) return fail(SALT_EINVAL, "scalar program stack underflow");
      } else if (op == salt::SP_OUT) {
        if (depth < 1) return fail(SALT_EINVAL, "scalar program stack underflow");
        if (arg >= salt::MAX_PSCALARS) return fail(SALT_EINVAL, "scalar program output index >= 8");
        --depth;
        def |= 1u << arg;
      } else {
        if (depth < 2) return fail(SALT_EINVAL, "scalar program stack underflow");
        --depth;
      }
      sp.op[sp.len] = (unsigned char)op;
      sp.arg[sp.len] = (unsigned char)arg;
      ++sp.len;
    }
    if (depth != 0) return fail(SALT_EINVAL, "scalar program leaves values on its stack");
    it = cache.emplace(text, std::make_pair(sp, def)).first;
  }
  const salt::SProg& sp = it->second.first;
  for (int i = 0; i < sp.len; ++i) {
    if (sp.op[i] == salt::SP_RAW && sp.arg[i] >= nraw)
      return fail(SALT_EINVAL, "scalar program reads device scalar " + std::to_string(sp.arg[i]) + " of " +
                                   std::to_string(nraw));
    if (sp.op[i] == salt::SP_HOST && sp.arg[i] >= nhost)
      return fail(SALT_EINVAL, "scalar program reads host scalar " + std::to_string(sp.arg[i]) + " of " +
                                   std::to_string(nhost));
  }
  out = sp;
  defined = it->second.second;
  return 0;
}

template <class T>
int run_fused(Plan& p, void* const* dsts, int ndst, const void* const* leaves, int nleaves,
              const double* scalars, int nscalars, i64 n, int flags, void* ws, size_t ws_bytes,
              void* out_dev, void* out_host, cudaStream_t st, const salt_exchange* x,
              const void* const* pscalars, int npscalars, const char* sprog = nullptr) {
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
  if (nscalars < p.ns || nscalars > salt::MAX_SCALARS)
    return fail(SALT_EINVAL, "signature reads " + std::to_string(p.ns) + " scalars but " +
                                 std::to_string(nscalars) + " were passed (at most 32)");
  for (int s = 0; s < nscalars; ++s) a.sc[s] = (T)scalars[s];
  if (npscalars < 0 || npscalars > salt::MAX_PSCALARS)
    return fail(SALT_EINVAL, "at most 8 device scalars, got " + std::to_string(npscalars));
  if (sprog && *sprog) {
    unsigned defined = 0;
    int rc = parse_sprog(sprog, npscalars, nscalars, a.sp, defined);
    if (rc) return rc;
    for (int q = 0; q < p.np; ++q)
      if (!(defined >> q & 1u))
        return fail(SALT_EINVAL, "the scalar program does not define P" + std::to_string(q));
  } else if (npscalars < p.np) {
    return fail(SALT_EINVAL, "signature reads " + std::to_string(p.np) + " device scalars but " +
                                 std::to_string(npscalars) + " were passed");
  }
  for (int q = 0; q < npscalars; ++q) {
    if (!pscalars || !pscalars[q]) return fail(SALT_EINVAL, "NULL device scalar");
    a.ps[q] = (const T*)pscalars[q];
  }
  a.nps = npscalars;
  a.n = n;
  a.flags = flags;
  int vec;
  geometry<T>(dsts, nroots, leaves, p.nl, n, vec, a.head, a.nvec);
  Kernel* k = nullptr;
  const bool force_interp = g_force_interp.load(std::memory_order_relaxed) != 0;
  // small assignments: the UNR 1 kernel of the same tree (kAssignSmallKind)
  const bool small = p.mode == salt::MODE_ASSIGN && tuning_unroll() <= 0 &&
                     a.nvec <= (vec == 1 ? kAssignSmallElements : kAssignSmallVectors);
  const int kind = small ? kAssignSmallKind : p.mode;
  if (g_trace_buf) {
    // device-observed trace (salt_set_trace): the NVRTC build of this tree
    // with -DSALT_TRACE, recording one thread's events into the buffer
    k = get_kernel(dtype_of<T>(), kind, vec, p.nl, p.sa.type, p.sr.type, false, nullptr, true);
    if (!k) return fail(SALT_EJIT, "traced kernel: " + g_err);
    a.trace = g_trace_buf;
    a.trace_cap = g_trace_cap;
  } else if (!force_interp) {
    Kernel*& slot = p.cached[g_force_jit.load(std::memory_order_relaxed)][(vec == 1 ? 1 : 0) + (small ? 2 : 0)];
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
      slot = get_kernel(dtype_of<T>(), kind, vec, p.nl, p.sa.type, p.sr.type, async, &queued);
    }
    k = slot;
  }
  if (!k) {
    // Not compiled in and no JIT build (NVRTC missing or failed), or forced:
    // the postfix interpreter evaluates the same trees (salt_interp.cuh).
    if (!p.prog_ok)
      return fail(SALT_EJIT, (force_interp ? std::string() : g_err + "; ") + "interpreter: " + p.prog_err);
    k = interp_kernel_for<T>(vec, unroll_for(p.mode, p.nl, (int)sizeof(T)), p.nl);
  }
  // V == 1 kernels run whole tiles without bounds predicates (salt_expr.cuh):
  // the ragged end joins the scalar tail, which every CTA shares.
  if (vec == 1) a.nvec -= a.nvec % ((i64)kBlock * k->unroll);
  int dev;
  int rc = current_device(dev);
  if (rc) return rc;
  rc = prepare(k, dev);
  if (rc) return rc;
  // Work split (tools/stream_variants.cu, tools/reduce_variants.cu on B200):
  // assignments take one BLOCK*UNR tile per CTA — the block scheduler
  // refills an SM the moment a CTA retires, which keeps loads in flight
  // (7.29 TB/s vs 7.06 for a persistent grid-stride loop); reductions of
  // three or more tiles do the same and hand their per-CTA partials to one
  // collector CTA (below); the round-1 geometry — reduce_tiles_per_cta()
  // tiles per CTA, partials combined in two deterministic ticket levels,
  // 7.25 vs 6.88 TB/s persistent for the fused axpy->dot f64 2^28 — remains
  // behind SALT_COMBINE=ticket.  Every grid depends only on n.
  const i64 per_tile = (i64)kBlock * k->unroll;
  i64 ntiles = (a.nvec + per_tile - 1) / per_tile;
  // V == 1: the ragged end (up to one tile: 2,047 / 4,095 elements) runs in
  // the scalar loop, which strides over every streaming CTA — size the grid
  // for it too (one element per thread), or a short misaligned vector would
  // loop through it in a single CTA.  (The kernel derives its own tile count
  // from nvec; CTAs beyond it only take scalar elements.  Giving the ragged
  // end CTAs of its own, so that no CTA pays the scalar loop's round trip
  // before its tile's, saved 0.2-0.3 us below 10^5 elements but its index
  // arithmetic cost a misaligned f64 dot at 2^27 14 %: measured and dropped.)
  if (vec == 1) ntiles = std::max(ntiles, (n - a.nvec + kBlock - 1) / kBlock);
  i64 K = assign_tiles_per_cta(), cap = i64(0x7fffffff);
  bool cluster = false, one_group = false, collect = false;
  if (reduce && ntiles > 2 && collect_enabled() &&
      (ntiles + collect_tiles() - 1) / collect_tiles() >= collect_min()) {
    // From 3 tiles up: streaming CTAs of collect_tiles() tiles that only
    // store their partial, plus one collector CTA (tools/c3_probe.cu,
    // profiles/r02_c3_probe*.txt: at 2^24 ddot 46.6 -> 42.6 us, sdot 25.7 ->
    // 24.3 us, dnrm2 26.4 -> 25.5 us; the fence + ticket atomic each
    // streaming CTA paid in the two-level combine held its SM slot).  With
    // the warp-uniform collector loop it is also the quickest combine for
    // small grids (profiles/r02_collector_small_grids.txt, back-to-back
    // launches: 2.5-3.0 us for 3-32 tiles against 2.8-4.0 us as one
    // cluster, 2.9-3.3 us for 33-192 tiles against 3.6-4.6 us through the
    // tickets), so the cluster and ticket combines below only run when
    // SALT_COLLECT_MIN / SALT_COMBINE ask for them.
    // Beyond kCollectCtas streaming CTAs (the slots the workspace holds),
    // more tiles per CTA: 2 for the f64 2^28 fused multi-leaf trees, the
    // K round 1 measured best for them (7.26 TB/s, r01_reduce_variants.txt);
    // a cap of 32,768 (K = 4 there) cost the CG update 2.3 %
    // (profiles/r02_ncu_cgupdate.txt); 131,072 slots (K = 1 for them) was a
    // wash on one box: ddot f64 2^28 +0.7 %, the CG update -0.8 %, axpy->dot
    // equal.
    constexpr i64 kCollectCtas = salt::MAX_COLLECT;
    static_assert(kCollectCtas <= salt::MAX_COLLECT, "collector slots");
    K = collect_tiles();
    if ((ntiles + K - 1) / K > kCollectCtas) K = (ntiles + kCollectCtas - 1) / kCollectCtas;
    collect = true;
  } else if (reduce && ntiles > 2 && ntiles <= (i64)max_cluster() * cluster_tiles()) {
    // (round 1; SALT_COLLECT_MIN=33 restores it) 3 .. 16 x 2 tiles: one cluster
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
  if (collect) g64 += 1;  // CTA 0: the collector
  const int grid = (int)g64;
  a.first = collect ? 1 : 0;
  a.collect_warps = collect_warps(g64 - 1);
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
    a.slots = (unsigned long long*)(w + salt::WsLayout::slots);
    a.out = out_dev;
    // a host result too: the kernel also stores it into this thread's pinned
    // slot (mapped on the device at the host address), so no copy follows
    if (out_host && out_host != out_dev) {
      char* slot = thread_result_slot();
      if (slot && g_result_pool_mapped.load(std::memory_order_acquire) && slot != (char*)out_dev)
        a.out2 = slot;
    }
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
      SALT_CUDA(cudaFuncSetAttribute(k->aot, cudaFuncAttributeMaxDynamicSharedMemorySize, kInterpSmemCap));
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
    const size_t bytes = (flags & SALT_PARTIAL) ? sizeof(salt::DD) : sizeof(T);
    if (a.out2) {  // the kernel stored it into this thread's mapped slot itself
      SALT_CUDA(cudaStreamSynchronize(st));
      memcpy(out_host, a.out2, bytes);
      return 0;
    }
    return result_to_host(out_host, out_dev, bytes, st);
  }
  return 0;
}

int dispatch(int dtype, Plan& p, void* const* dsts, int ndst, const void* const* leaves,
             int nleaves, const double* scalars, int nscalars, i64 n, int flags, void* ws,
             size_t ws_bytes, void* out_dev, void* out_host, cudaStream_t st,
             const salt_exchange* x = nullptr, const void* const* pscalars = nullptr,
             int npscalars = 0, const char* sprog = nullptr) {
  if (dtype == SALT_F32)
    return run_fused<float>(p, dsts, ndst, leaves, nleaves, scalars, nscalars, n, flags, ws,
                            ws_bytes, out_dev, out_host, st, x, pscalars, npscalars, sprog);
  return run_fused<double>(p, dsts, ndst, leaves, nleaves, scalars, nscalars, n, flags, ws,
                           ws_bytes, out_dev, out_host, st, x, pscalars, npscalars, sprog);
}

#include "salt_abi_batch.inc"

template <class T>
int finish(const void* parts, int count, int flags, void* out_dev, void* out_host,
           cudaStream_t st) {
  if (count < 0 || (count > 0 && !parts) || !out_dev) return fail(SALT_EINVAL, "bad finish arguments");
  void* params[] = {(void*)&parts, &count, &flags, &out_dev};
  SALT_CUDA(cudaLaunchKernel((const void*)&salt::finish_kernel<T, kBlock>, dim3(1), dim3(kBlock),
                             params, 0, st));
  g_launches.fetch_add(1, std::memory_order_relaxed);
  if (out_host)
    return result_to_host(out_host, out_dev, (flags & SALT_PARTIAL) ? sizeof(salt::DD) : sizeof(T), st);
  return 0;
}

#include "salt_abi_nccl.inc"

#include "salt_abi_host.inc"

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

int salt_result_enqueue(const void* out_dev, size_t bytes, void* stream, void** host_slot) {
  if (!out_dev || !host_slot || bytes == 0 || bytes > 64) return fail(SALT_EINVAL, "bad result fetch");
  return result_enqueue(out_dev, bytes, (cudaStream_t)stream, host_slot);
}

int salt_result_slot(void** host_slot) {
  if (!host_slot) return fail(SALT_EINVAL, "null result slot pointer");
  char* slot = thread_result_slot();
  if (!slot || !g_result_pool_mapped.load(std::memory_order_acquire))
    return fail(SALT_EINVAL, "no device-mapped result slot for this thread");
  *host_slot = slot;
  return 0;
}

int salt_stream_synchronize(void* stream) {
  SALT_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
  return 0;
}

int salt_set_trace(void* trace_dev, int64_t capacity) {
  if (trace_dev && capacity < 4) return fail(SALT_EINVAL, "trace buffer needs at least 4 int64 words");
  g_trace_buf = (long long*)trace_dev;
  g_trace_cap = trace_dev ? capacity : 0;
  return 0;
}

uint64_t salt_capture_id(void* stream) {
  cudaStreamCaptureStatus status = cudaStreamCaptureStatusNone;
  unsigned long long id = 0;
  if (cudaStreamGetCaptureInfo((cudaStream_t)stream, &status, &id) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return status == cudaStreamCaptureStatusActive ? (uint64_t)id : 0;
}

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
  return salt_fused_exchange_prog(dtype, assign_sigs, reduce_sig, dsts, ndst, leaves, nleaves, scalars,
                                  nscalars, pscalars, npscalars, nullptr, n, flags, workspace,
                                  workspace_bytes, exchange, out_dev, out_host, stream);
}

int salt_fused_exchange_prog(int dtype, const char* assign_sigs, const char* reduce_sig,
                             void* const* dsts, int ndst, const void* const* leaves, int nleaves,
                             const double* scalars, int nscalars, const void* const* pscalars,
                             int npscalars, const char* scalar_prog, int64_t n, int flags,
                             void* workspace, size_t workspace_bytes, const salt_exchange* exchange,
                             void* out_dev, void* out_host, void* stream) {
  if (!exchange) return fail(SALT_EINVAL, "NULL exchange descriptor");
  if (!reduce_sig) return fail(SALT_EINVAL, "salt_fused_exchange needs a reduction");
  Plan* p;
  const int mode = assign_sigs ? salt::MODE_ASSIGN_REDUCE : salt::MODE_REDUCE;
  int rc = make_plan(dtype, assign_sigs, reduce_sig, mode, nleaves, nscalars, p);
  if (rc) return rc;
  return dispatch(dtype, *p, dsts, ndst, leaves, nleaves, scalars, nscalars, n, flags, workspace,
                  workspace_bytes, out_dev, out_host, (cudaStream_t)stream, exchange, pscalars,
                  npscalars, scalar_prog);
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
  return salt_fused_prog(dtype, assign_sigs, reduce_sig, dsts, ndst, leaves, nleaves, scalars, nscalars,
                         pscalars, npscalars, nullptr, n, flags, workspace, workspace_bytes, out_dev,
                         out_host, stream);
}

int salt_fused_prog(int dtype, const char* assign_sigs, const char* reduce_sig, void* const* dsts,
                    int ndst, const void* const* leaves, int nleaves, const double* scalars,
                    int nscalars, const void* const* pscalars, int npscalars, const char* scalar_prog,
                    int64_t n, int flags, void* workspace, size_t workspace_bytes, void* out_dev,
                    void* out_host, void* stream) {
  Plan* p;
  if (!assign_sigs && !reduce_sig) return fail(SALT_EINVAL, "nothing to evaluate");
  const int mode = !assign_sigs ? salt::MODE_REDUCE
                   : reduce_sig ? salt::MODE_ASSIGN_REDUCE : salt::MODE_ASSIGN;
  int rc = make_plan(dtype, assign_sigs, reduce_sig, mode, nleaves, nscalars, p);
  if (rc) return rc;
  return dispatch(dtype, *p, dsts, ndst, leaves, nleaves, scalars, nscalars, n, flags, workspace,
                  workspace_bytes, out_dev, out_host, (cudaStream_t)stream, nullptr, pscalars,
                  npscalars, scalar_prog);
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

#include "salt_abi_group.inc"
