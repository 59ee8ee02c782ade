// salt_expr.cuh — device-side expression templates and the fused kernel.
//
// This is SALT's idea (arXiv 1109.1264, Fig. 1 / Listing 2) moved to
// the GPU: an expression tree is a TYPE (Add<L<0>, Sub<L<1>, L<2>>>), the
// kernel is instantiated per tree shape, and the whole tree is evaluated in
// registers between one vectorised load burst and one store burst, so no
// intermediate vector ever reaches HBM.
//
// Reference semantics reproduced bit for bit (pkg/src/lanevec/...):
//   * every binary node is ONE IEEE op in the element type, left operand
//     first (expressions.py:239-249, operator.add/sub/mul :255-270);
//   * ScaleNode is alpha * child with alpha already coerced to the element
//     type (expressions.py:282, :319-320);
//   * no FMA contraction, no flush-to-zero: the __{d,f}{add,sub,mul}_rn
//     intrinsics pin round-to-nearest and forbid contraction;
//   * AssignNode computes the full value before the store, so exact
//     aliasing dst == leaf is safe (expressions.py:392-395).
//
// Reductions (SumNode, expressions.py:401-467) are NOT order-reproduced: the
// reference's order depends on its CPU unroll plan and its contract is a
// tolerance.  Here they are compensated (double-double) and
// deterministic, i.e. more accurate than the reference's own engine.
//
// The header is self-contained (no #include) so NVRTC can compile it verbatim
// for signatures that are not in the compiled-in table.
#pragma once

namespace salt {

typedef long long i64;

// ---------------------------------------------------------------- arithmetic
template <class T> struct Arith;
template <> struct Arith<double> {
  static __device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
  static __device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
  static __device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
  static __device__ __forceinline__ double sqrt_rn(double a) { return __dsqrt_rn(a); }
  static __device__ __forceinline__ double div(double a, double b) { return __ddiv_rn(a, b); }
};
template <> struct Arith<float> {
  static __device__ __forceinline__ float add(float a, float b) { return __fadd_rn(a, b); }
  static __device__ __forceinline__ float sub(float a, float b) { return __fsub_rn(a, b); }
  static __device__ __forceinline__ float mul(float a, float b) { return __fmul_rn(a, b); }
  static __device__ __forceinline__ float sqrt_rn(float a) { return __fsqrt_rn(a); }
  static __device__ __forceinline__ float div(float a, float b) { return __fdiv_rn(a, b); }
};

__host__ __device__ constexpr int cmax(int a, int b) { return a > b ? a : b; }

// ---------------------------------------------------------------- tree nodes
// Each node exposes: NL (leaves referenced = max index + 1), NS (scalars),
// USES_D (reads the just-assigned value) and ev(env, k) for lane k.
template <int I> struct L {
  enum { NL = I + 1, NS = 0, NP = 0, USES_D = 0 };
  template <class Env> static __device__ __forceinline__ typename Env::T ev(const Env& e, int k) {
    return e.x[I][k];
  }
};
template <int I> struct S {
  enum { NL = 0, NS = I + 1, NP = 0, USES_D = 0 };
  template <class Env> static __device__ __forceinline__ typename Env::T ev(const Env& e, int) {
    return e.s[I];
  }
};
// Dk<R>: the value root R of the same fused kernel has just assigned (the
// reduce tree of an assign+reduce kernel, or a later root of a multi-root
// kernel, reading an earlier root's destination).  D is Dk<0>.
// P<I>: a scalar read from device memory (a DeviceScalar operand: e.g. the
// alpha of a solver step computed on the GPU), loaded once per thread.
template <int I> struct P {
  enum { NL = 0, NS = 0, NP = I + 1, USES_D = 0 };
  template <class Env> static __device__ __forceinline__ typename Env::T ev(const Env& e, int) {
    return e.p[I];
  }
};
template <int R> struct Dk {
  enum { NL = 0, NS = 0, NP = 0, USES_D = 1 };
  template <class Env> static __device__ __forceinline__ typename Env::T ev(const Env& e, int k) {
    return e.d[R][k];
  }
};
typedef Dk<0> D;
// Placeholder for "no tree" (reduce-only kernels have no assign tree and
// vice versa).
struct None {
  enum { NL = 0, NS = 0, NP = 0, USES_D = 0 };
  template <class Env> static __device__ __forceinline__ typename Env::T ev(const Env&, int) {
    return typename Env::T(0);
  }
};

#define SALT_BINARY_NODE(NAME, FN)                                                       \
  template <class A, class B> struct NAME {                                              \
    enum { NL = cmax(A::NL, B::NL), NS = cmax(A::NS, B::NS), NP = cmax(A::NP, B::NP),      \
           USES_D = A::USES_D | B::USES_D };                                             \
    template <class Env> static __device__ __forceinline__ typename Env::T ev(const Env& e, int k) { \
      return Arith<typename Env::T>::FN(A::ev(e, k), B::ev(e, k));                      \
    }                                                                                    \
  };
SALT_BINARY_NODE(Add, add)
SALT_BINARY_NODE(Sub, sub)
SALT_BINARY_NODE(Mul, mul)
#undef SALT_BINARY_NODE

// Multi<E0, E1, ...>: several assignment roots fused into one kernel (one
// destination each), evaluated in order per element, so root R may read the
// new value of an earlier root's destination through Dk<R'> — the
// sequential semantics of the same statements run one after another.
template <class... Es> struct Multi;
template <class E0> struct Multi<E0> {
  enum { NL = E0::NL, NS = E0::NS, NP = E0::NP, ND = 1 };
};
template <class E0, class E1, class... Es> struct Multi<E0, E1, Es...> {
  enum {
    NL = cmax(E0::NL, Multi<E1, Es...>::NL),
    NS = cmax(E0::NS, Multi<E1, Es...>::NS),
    NP = cmax(E0::NP, Multi<E1, Es...>::NP),
    ND = 1 + Multi<E1, Es...>::ND
  };
};
template <int R, class... Es> struct TypeAt;
template <class E0, class... Es> struct TypeAt<0, E0, Es...> { typedef E0 type; };
template <int R, class E0, class... Es> struct TypeAt<R, E0, Es...> {
  typedef typename TypeAt<R - 1, Es...>::type type;
};
// Roots of an assign tree: a plain tree is one root.
template <class EA> struct Roots {
  enum { N = 1 };
  template <int R> struct At { typedef EA type; };
};
template <class... Es> struct Roots<Multi<Es...>> {
  enum { N = sizeof...(Es) };
  template <int R> struct At { typedef typename TypeAt<R, Es...>::type type; };
};

// ---------------------------------------------------------------- kernel ABI
enum { MAX_LEAVES = 16, MAX_SCALARS = 32, MAX_ROOTS = 4, MAX_PSCALARS = 8 };
enum { MODE_ASSIGN = 0, MODE_REDUCE = 1, MODE_ASSIGN_REDUCE = 2 };
enum { FLAG_SQRT = 1, FLAG_PARTIAL = 2 };

struct DD { double hi, lo; };  // double-double partial (same layout as double2)

// Cross-GPU exchange of per-rank totals over NVLink peer memory (sharded
// reductions).  Every rank owns a small symmetric buffer: slots DD[2][8]
// (double-buffered by epoch parity) followed by flags u64[8].  slots[p] /
// flags[p] are rank p's buffers mapped into this process (peer pointers;
// p == rank is the local one).  world == 0 disables the exchange.
enum { XCHG_MAX_RANKS = 8 };
struct Xchg {
  int rank, world;
  unsigned long long epoch;            // >= 1, +1 per exchange, same on all ranks
  DD* slots[XCHG_MAX_RANKS];
  unsigned long long* flags[XCHG_MAX_RANKS];
  unsigned long long timeout_ns;       // 0: wait forever
  unsigned int* error;                 // set to 1 on timeout (local memory)
};

// Scalar program: derived device scalars computed once per thread in the
// kernel prologue from the raw device scalars (ps[i]) and host scalars
// (sc[j]) — e.g. a CG step length rr / pq — instead of a separate launch
// per scalar operation.  Postfix; SP_OUT k pops into the tree's P<k>.
// Every op is one IEEE op in the element type (the bits of the same torch
// op on 1-element tensors).
enum { SPROG_MAX = 32, SPROG_STACK = 8 };
enum { SP_RAW = 0, SP_HOST, SP_ADD, SP_SUB, SP_MUL, SP_DIV, SP_NEG, SP_OUT };
struct SProg {
  int len;  // 0: no program, P<k> = *ps[k]
  unsigned char op[SPROG_MAX];
  unsigned char arg[SPROG_MAX];
};

// One by-value parameter block shared by AOT and JIT kernels.
template <class T> struct Args {
  T* dst[MAX_ROOTS];              // assign modes: one destination per root
  const T* leaf[MAX_LEAVES];
  T sc[MAX_SCALARS];
  const T* ps[MAX_PSCALARS];      // device-resident scalars (P<k>, or the program's inputs)
  int nps;                        // pointers in ps
  SProg sp;                       // scalar program (sp.len == 0: none)
  i64 n;                          // elements
  i64 head;                       // scalar elements before the first aligned vector
  i64 nvec;                       // aligned vectors of V elements after `head`
  i64 tiles_per_cta;              // consecutive BLOCK*UNR-vector tiles each CTA owns
  // reduce modes (workspace, see WsLayout): two-level deterministic combine
  DD* partials;                   // one partial per CTA
  DD* group_partials;             // one partial per group of GROUP CTAs
  unsigned int* group_tickets;    // arrival counters per group (zeroed, self-resetting)
  unsigned int* ticket;           // arrival counter of the groups (zeroed, self-resetting)
  void* out;                      // T result or DD partial
  void* out2;                     // optional second copy of the result (the caller's
                                  // device-mapped pinned host slot), or nullptr
  int flags;
  int cluster;                    // reduce modes: 1 = the grid is ONE thread-block cluster
  int group;                      // reduce modes: CTAs per group (GROUP, or the whole grid
                                  // when it is one group of <= MAX_ONE_GROUP CTAs)
  int collect_warps;              // collector warps (1 .. 8)
  long long* trace;               // -DSALT_TRACE builds: event buffer (salt_set_trace)
  long long trace_cap;
  int first;                      // 1: CTA 0 is the collector (see collect_epilogue), the
                                  // streaming CTAs are 1..gridDim.x-1; 0: no collector
  unsigned long long* slots;      // collector slots (2 words per streaming CTA, zero = empty)
  Xchg xchg;                      // sharded reductions over NVLink (world 0: off)
};

// Reduction workspace: [ticket | group tickets | collector slots | group
// partials | CTA partials]; everything before group_partials must be zero
// before the first use (the kernels leave it zero again).
enum { GROUP = 256, MAX_GROUPS = 4096, MAX_REDUCE_CTAS = GROUP * MAX_GROUPS, MAX_ONE_GROUP = 1024,
       MAX_COLLECT = 65536 };
struct WsLayout {
  static constexpr i64 ticket = 0;
  static constexpr i64 group_tickets = 256;
  static constexpr i64 slots = group_tickets + 4 * (i64)MAX_GROUPS;
  static constexpr i64 group_partials = slots + 16 * (i64)MAX_COLLECT;
  static constexpr i64 partials = group_partials + 16 * (i64)MAX_GROUPS;
  static constexpr i64 bytes = partials + 16 * (i64)MAX_REDUCE_CTAS;
};

// 32-byte (256-bit) vector access: LDG.E.ENL2.256 / STG.E.ENL2.256 on sm_100a.
// Plain (coherent) loads: a leaf may alias the destination (axpy, scal).
template <class T, int V> struct VecIO;
#ifndef SALT_NO_256BIT
template <> struct VecIO<double, 4> {
  static __device__ __forceinline__ void load(double (&r)[4], const double* p) {
    asm volatile("ld.global.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];"
                 : "=d"(r[0]), "=d"(r[1]), "=d"(r[2]), "=d"(r[3]) : "l"(p));
  }
  static __device__ __forceinline__ void store(double* p, const double (&r)[4]) {
    asm volatile("st.global.L1::no_allocate.v4.f64 [%0], {%1,%2,%3,%4};"
                 :: "l"(p), "d"(r[0]), "d"(r[1]), "d"(r[2]), "d"(r[3]) : "memory");
  }
};
template <> struct VecIO<float, 8> {
  static __device__ __forceinline__ void load(float (&r)[8], const float* p) {
    asm volatile("ld.global.L1::no_allocate.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(r[0]), "=f"(r[1]), "=f"(r[2]), "=f"(r[3]),
                   "=f"(r[4]), "=f"(r[5]), "=f"(r[6]), "=f"(r[7]) : "l"(p));
  }
  static __device__ __forceinline__ void store(float* p, const float (&r)[8]) {
    asm volatile("st.global.L1::no_allocate.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
                 :: "l"(p), "f"(r[0]), "f"(r[1]), "f"(r[2]), "f"(r[3]),
                    "f"(r[4]), "f"(r[5]), "f"(r[6]), "f"(r[7]) : "memory");
  }
};
#else
// NVRTC < 12.9 (PTX ISA < 8.8) has no 256-bit ld/st: two 128-bit halves.
template <> struct VecIO<double, 4> {
  static __device__ __forceinline__ void load(double (&r)[4], const double* p) {
    asm volatile("ld.global.L1::no_allocate.v2.f64 {%0,%1}, [%2];" : "=d"(r[0]), "=d"(r[1]) : "l"(p));
    asm volatile("ld.global.L1::no_allocate.v2.f64 {%0,%1}, [%2];" : "=d"(r[2]), "=d"(r[3]) : "l"(p + 2));
  }
  static __device__ __forceinline__ void store(double* p, const double (&r)[4]) {
    asm volatile("st.global.L1::no_allocate.v2.f64 [%0], {%1,%2};" :: "l"(p), "d"(r[0]), "d"(r[1]) : "memory");
    asm volatile("st.global.L1::no_allocate.v2.f64 [%0], {%1,%2};" :: "l"(p + 2), "d"(r[2]), "d"(r[3]) : "memory");
  }
};
template <> struct VecIO<float, 8> {
  static __device__ __forceinline__ void load(float (&r)[8], const float* p) {
    asm volatile("ld.global.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(r[0]), "=f"(r[1]), "=f"(r[2]), "=f"(r[3]) : "l"(p));
    asm volatile("ld.global.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(r[4]), "=f"(r[5]), "=f"(r[6]), "=f"(r[7]) : "l"(p + 4));
  }
  static __device__ __forceinline__ void store(float* p, const float (&r)[8]) {
    asm volatile("st.global.L1::no_allocate.v4.f32 [%0], {%1,%2,%3,%4};"
                 :: "l"(p), "f"(r[0]), "f"(r[1]), "f"(r[2]), "f"(r[3]) : "memory");
    asm volatile("st.global.L1::no_allocate.v4.f32 [%0], {%1,%2,%3,%4};"
                 :: "l"(p + 4), "f"(r[4]), "f"(r[5]), "f"(r[6]), "f"(r[7]) : "memory");
  }
};
#endif
// One element (operands that do not share one 32-byte misalignment).  The
// loads are volatile asm like the vector ones, so a tile's whole load burst
// is issued before the first use: with plain C++ loads the compiler merged
// the load loop into the TwoSum chain of a reduction, one pair of loads
// ahead of the arithmetic (a misaligned f64 dot: 3.5-4.6 TB/s; now 7.3,
// profiles/r02_misaligned.json).  They allocate in L1, unlike the vector
// loads: a warp's run of elements straddles two 128-byte lines here, and the
// neighbouring warp's load of the shared line then hits L1 instead of L2
// (f32 axpy at mixed offsets 6.56 -> 6.75 TB/s).
template <> struct VecIO<double, 1> {
  static __device__ __forceinline__ void load(double (&r)[1], const double* p) {
    asm volatile("ld.global.f64 %0, [%1];" : "=d"(r[0]) : "l"(p));
  }
  static __device__ __forceinline__ void store(double* p, const double (&r)[1]) {
    asm volatile("st.global.f64 [%0], %1;" :: "l"(p), "d"(r[0]) : "memory");
  }
};
template <> struct VecIO<float, 1> {
  static __device__ __forceinline__ void load(float (&r)[1], const float* p) {
    asm volatile("ld.global.f32 %0, [%1];" : "=f"(r[0]) : "l"(p));
  }
  static __device__ __forceinline__ void store(float* p, const float (&r)[1]) {
    asm volatile("st.global.f32 [%0], %1;" :: "l"(p), "f"(r[0]) : "memory");
  }
};

// Registers of one unroll slot: V lanes of every leaf, the scalars, and the
// assigned value (read back by D in fused assign+reduce trees).
template <class T_, int NL, int NS, int NP, int ND, int V> struct Env {
  typedef T_ T;
  T x[NL > 0 ? NL : 1][V];
  T s[NS > 0 ? NS : 1];
  T p[NP > 0 ? NP : 1];
  T d[ND][V];
};

// Evaluate roots R..N-1 for the V lanes of one vector and store them.
template <class EA, int R, int N> struct AssignRoots {
  template <class T, class E>
  static __device__ __forceinline__ void vec(E& e, T* const* dst, i64 off);
  template <class T, class E>
  static __device__ __forceinline__ void one(E& e, T* const* dst, i64 i);
};
template <class EA, int N> struct AssignRoots<EA, N, N> {
  template <class T, class E> static __device__ __forceinline__ void vec(E&, T* const*, i64) {}
  template <class T, class E> static __device__ __forceinline__ void one(E&, T* const*, i64) {}
};

// ---------------------------------------------------------------- reductions
// Knuth TwoSum: s + e == a + b exactly.
__device__ __forceinline__ void two_sum(double a, double b, double& s, double& e) {
  s = __dadd_rn(a, b);
  double bp = __dsub_rn(s, a);
  double ap = __dsub_rn(s, bp);
  e = __dadd_rn(__dsub_rn(a, ap), __dsub_rn(b, bp));
}
// x - x == 0 exactly for finite x; NaN for +-inf and NaN.
__device__ __forceinline__ bool finite(double x) { return __dsub_rn(x, x) == 0.0; }

// Double-double accumulation (round 2: the cheap form).  The high words are
// added exactly (TwoSum: s + e == a.hi + b.hi); the low words and e are
// summed in plain f64; the pair is NOT renormalised between additions
// (|lo| stays within a few hundred ulps of hi over any fold in this file, so
// the low word's own rounding errors are ~2^-96 of the sum).  8 FP64
// operations with a ONE-add dependency chain through hi, instead of 18 with
// a 13-deep chain for a renormalising add: at one tile per CTA the CTA
// epilogue was 40 % of an f64 nrm2's FP64 instructions, and the FP64 pipe
// (64 lanes / clk / SM) sat at ~70 % beside the loads
// (profiles/r02_cheap_epilogue.txt).
// Once a sum is not finite (an inf or NaN term, or overflow) e and lo turn
// NaN while hi carries the plain IEEE sum on — inf, or NaN for inf + -inf,
// which is what the reference's element-typed accumulation produces;
// dd_norm / finish_store drop the meaningless low word at the end.
__device__ __forceinline__ DD dd_add(DD a, DD b) {
  DD r;
  double e;
  two_sum(a.hi, b.hi, r.hi, e);
  r.lo = __dadd_rn(a.lo, __dadd_rn(b.lo, e));
  return r;
}
// Canonical form of a pair: |lo| <= ulp(hi) / 2, or (hi, 0) when hi is not
// finite.  Applied where a pair leaves the kernel (partial outputs, the
// cross-rank exchange), so every route folds the same values.
__device__ __forceinline__ DD dd_norm(DD v) {
  DD r;
  if (!finite(v.hi)) {
    r.hi = v.hi;
    r.lo = 0.0;
    return r;
  }
  two_sum(v.hi, v.lo, r.hi, r.lo);
  return r;
}

// Per-thread accumulator.  f64 terms: compensated (TwoSum per term).
// f32 terms: exact conversion to double and a plain double sum — a thread
// sums at most a few hundred terms, so its error (~1e-14 relative) is far
// below f32 eps.
template <class T> struct Acc;
template <> struct Acc<double> {
  double hi = 0.0, lo = 0.0;
  __device__ __forceinline__ void add(double v) {
    double s, e;
    two_sum(hi, v, s, e);
    hi = s;
    lo = __dadd_rn(lo, e);
  }
  // not renormalised (dd_add does not need it)
  __device__ __forceinline__ DD get() const { DD r; r.hi = hi; r.lo = lo; return r; }
};
template <> struct Acc<float> {
  double hi = 0.0;
  __device__ __forceinline__ void add(float v) { hi = __dadd_rn(hi, (double)v); }
  __device__ __forceinline__ DD get() const { DD r; r.hi = hi; r.lo = 0.0; return r; }
};

// Thread-block cluster helpers (sm_90+ PTX): a barrier across every thread
// of the cluster with release/acquire semantics for shared memory, and a
// load from another CTA's shared memory (distributed shared memory).
__device__ __forceinline__ void cluster_barrier() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\t"
               "barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ double ld_dsmem(const double* local, unsigned int rank) {
  const unsigned int addr = (unsigned int)__cvta_generic_to_shared(local);
  unsigned int remote;
  double v;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(addr), "r"(rank));
  asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(remote) : "memory");
  return v;
}

// Ticket increment with acquire-release semantics at GPU scope: it publishes
// this CTA's partial (release) and, for the CTA that turns out to be last,
// makes every other CTA's partial visible (acquire) — no separate fences.
__device__ __forceinline__ unsigned int ticket_add(unsigned int* p) {
  unsigned int old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(p) : "memory");
  return old;
}

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" :: "l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// Publish `mine` to every rank, wait for every rank's value of this epoch,
// and fold them in rank order (identical bits on every rank).  One thread.
//
// Ordering: the slot stores to peer p are made visible before the release
// store of flag[rank] at p (fence.sys); the reader's acquire load of
// flag[q] orders its slot load after it.  Slots alternate by epoch parity: a
// rank can only reach epoch e+2 after every rank has published e+1, which
// each does only after finishing its epoch-e reads, so a slot is never
// overwritten while it is still being read.
// A rank that gives up (timeout, or poisoned by an earlier one) raises the
// ABORT flag at every peer, so the others stop waiting for it at once —
// they return NaN and poison themselves too — instead of each timing out.
constexpr unsigned long long kXchgAbort = ~0ull;

__device__ DD exchange_abort(const Xchg& x) {
  DD nan; nan.hi = __longlong_as_double(0x7ff8000000000000ll); nan.lo = 0.0;
  if (x.error) *(volatile unsigned int*)x.error = 1u;
  for (int p = 0; p < x.world; ++p) st_release_sys(x.flags[p] + x.rank, kXchgAbort);
  return nan;
}

__device__ DD exchange_dd(DD mine, const Xchg& x) {
  // A previous exchange of this rank failed: the protocol's epochs are out
  // of step, so touch no slot (a late peer may have reused it) — NaN.
  if (x.error && *(volatile unsigned int*)x.error) return exchange_abort(x);
  mine = dd_norm(mine);  // what finish_store hands the all-gather route
  const int par = (int)(x.epoch & 1ull);
  for (int p = 0; p < x.world; ++p) {
    volatile DD* dst = (volatile DD*)(x.slots[p] + par * XCHG_MAX_RANKS + x.rank);
    dst->hi = mine.hi;
    dst->lo = mine.lo;
  }
  __threadfence_system();
  for (int p = 0; p < x.world; ++p) st_release_sys(x.flags[p] + x.rank, x.epoch);
  DD acc; acc.hi = 0.0; acc.lo = 0.0;
  const unsigned long long t0 = x.timeout_ns ? globaltimer_ns() : 0ull;
  for (int q = 0; q < x.world; ++q) {
    for (;;) {
      const unsigned long long f = ld_acquire_sys(x.flags[x.rank] + q);
      if (f == kXchgAbort) return exchange_abort(x);  // a peer gave up
      if (f >= x.epoch) break;
      if (x.timeout_ns && globaltimer_ns() - t0 > x.timeout_ns) return exchange_abort(x);
    }
    volatile DD* src = (volatile DD*)(x.slots[x.rank] + par * XCHG_MAX_RANKS + q);
    DD v;
    v.hi = src->hi;
    v.lo = src->lo;
    acc = dd_add(acc, v);
  }
  return acc;
}

// CTA fold of one pair per thread; `smem` holds BLOCK pairs.  Every thread
// leaves its pair in shared memory; the first warp's lane l then folds
// threads l, l + 32, ... in that order and a shuffle tree folds the lanes —
// a fixed order.  Only ONE warp runs FP64 here: 12 dd_adds per CTA instead
// of the 8 x 5 + 5 a shuffle tree in every warp costs (the FP64 pipe charges
// per warp instruction, not per useful lane).
template <int BLOCK> __device__ __forceinline__ DD block_reduce_dd(DD v, DD* smem) {
  double* const sh = (double*)smem;  // hi[BLOCK], then lo[BLOCK]: conflict-free
  sh[threadIdx.x] = v.hi;
  sh[BLOCK + threadIdx.x] = v.lo;
  __syncthreads();
  if (threadIdx.x < 32) {
#pragma unroll
    for (int w = 1; w < BLOCK / 32; ++w) {
      DD o;
      o.hi = sh[threadIdx.x + 32 * w];
      o.lo = sh[BLOCK + threadIdx.x + 32 * w];
      v = dd_add(v, o);
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      DD o;
      o.hi = __shfl_xor_sync(0xffffffffu, v.hi, off);
      o.lo = __shfl_xor_sync(0xffffffffu, v.lo, off);
      v = dd_add(v, o);
    }
  }
  return v;  // valid in thread 0
}

template <class T> __device__ __forceinline__ void finish_store(DD tot, int flags, void* out);
// The kernel's result: to a.out and, when the caller also wants it in host
// memory, to its device-mapped pinned slot (a.out2) — no copy afterwards.
template <class T> __device__ __forceinline__ void finish_result(DD tot, const Args<T>& a) {
  finish_store<T>(tot, a.flags, a.out);
  if (a.out2) finish_store<T>(tot, a.flags, a.out2);
}

// The tree's device scalars pv[0..NPV) for this thread: loaded from ps, or
// computed by the scalar program (uniform across threads; a few ops).
template <class T, int NPV>
__device__ __forceinline__ void load_pscalars(const Args<T>& a, T (&pv)[NPV], int np) {
  if (a.sp.len == 0) {
#pragma unroll
    for (int q = 0; q < NPV; ++q)
      if (q < np) pv[q] = __ldg(a.ps[q]);
    return;
  }
  T stk[SPROG_STACK];
  int top = 0;
  for (int i = 0; i < a.sp.len; ++i) {
    const int op = a.sp.op[i], k = a.sp.arg[i];
    if (op == SP_RAW) {
      stk[top++] = __ldg(a.ps[k]);
    } else if (op == SP_HOST) {
      stk[top++] = a.sc[k];
    } else if (op == SP_NEG) {
      stk[top - 1] = -stk[top - 1];
    } else if (op == SP_OUT) {
      const T v = stk[--top];
#pragma unroll
      for (int q = 0; q < NPV; ++q)
        if (q == k) pv[q] = v;
    } else {
      const T r = stk[--top];
      const T l = stk[--top];
      stk[top++] = op == SP_ADD ? Arith<T>::add(l, r)
                   : op == SP_SUB ? Arith<T>::sub(l, r)
                   : op == SP_MUL ? Arith<T>::mul(l, r) : Arith<T>::div(l, r);
    }
  }
}

// Warp shuffle tree over a double-double (valid in every lane).
__device__ __forceinline__ DD warp_reduce_dd(DD v) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    DD o;
    o.hi = __shfl_xor_sync(0xffffffffu, v.hi, off);
    o.lo = __shfl_xor_sync(0xffffffffu, v.lo, off);
    v = dd_add(v, o);
  }
  return v;
}

// Collector combine (mid and large reductions; tools/c3_probe.cu,
// profiles/r02_c3_probe*.txt).  The grid is 1 + P CTAs: CTAs 1..P stream
// their tiles, reduce them in the CTA and store the partial into their slot
// with ONE plain 16-byte store — no fence, no atomic, so a streaming CTA
// frees its SM slot as soon as its loads retire.  A slot holds the two
// words of the partial XOR kSlotMask, so zero memory means "not written
// yet": kSlotMask's words are signalling-NaN patterns, which no arithmetic
// result (all partials are sums) can be.  Each 8-byte word is written once
// and read whole (aligned 64-bit accesses are single-copy atomic; stores and
// loads of the slots are volatile, i.e. relaxed at system scope, so the
// slots are never the target of a weak racing access), so a reader that
// sees both words non-zero has the value.
// CTA 0's first a.collect_warps warps are the collector: thread t folds
// slots t, t + C, t + 2C, ... (C = 32 * collect_warps) IN ORDER as they appear,
// polling up to kCollectBatch of its slots per round trip (volatile loads),
// and zeroes each slot it has consumed (the next launch is stream-ordered
// after this one); a shuffle tree per warp and the warps' totals in warp
// order give the total — a fixed order, so the bits depend only on n.
// C x kCollectBatch slots per round trip keep the collector ahead of the
// streaming CTAs (they complete up to ~100 slots per microsecond): one
// warp x 4 slots fell behind at 2^28; 2 warps x 4 (the default) matched
// 1 x 8 and 2 x 8 and beat 4 warps over 2^22-2^28 on one box
// (profiles/r02_collector_ab.txt) without the registers 8 slots cost.  Whatever
// order the CTAs are scheduled in, nothing waits on the collector, so it
// cannot deadlock; the collector only waits for stores that are certain to
// come.
constexpr unsigned long long kSlotMask = 0x7ff4000000000001ull;
// (a bigger batch costs the streaming path registers: the collector shares
// the kernel's register allocation — 8 took f32 nrm2 from 48 to 64)
#ifndef SALT_COLLECT_BATCH
#define SALT_COLLECT_BATCH 4
#endif
constexpr int kCollectBatch = SALT_COLLECT_BATCH;
constexpr int kCollectWarpsMax = 8;

template <class T, int BLOCK>
__device__ __forceinline__ void collect_epilogue(DD mine, const Args<T>& a, DD* smem) {
  static_assert(BLOCK >= 32 * kCollectWarpsMax, "collector warps");
  const unsigned np = gridDim.x - 1;
  if (blockIdx.x != 0) {
    DD part = block_reduce_dd<BLOCK>(mine, smem);
    if (threadIdx.x == 0) {
      const unsigned long long h = (unsigned long long)__double_as_longlong(part.hi) ^ kSlotMask;
      const unsigned long long l = (unsigned long long)__double_as_longlong(part.lo) ^ kSlotMask;
      asm volatile("st.volatile.global.v2.u64 [%0], {%1,%2};" ::"l"(a.slots + 2 * (blockIdx.x - 1)), "l"(h), "l"(l)
                   : "memory");
    }
    return;
  }
  const int nw = a.collect_warps;  // 1 .. kCollectWarpsMax
  const unsigned C = 32u * nw;
  if (threadIdx.x >= C) return;
  DD v; v.hi = 0.0; v.lo = 0.0;
  unsigned q = threadIdx.x;  // this thread's next slot
  // The loop condition is warp-uniform: a lane that has folded its last slot
  // (or has none: np is rarely a multiple of C) idles in the loop until
  // every lane of its warp is done.  Lanes that left early used to wait at
  // the shuffle tree below while the others spun on their slots, and a warp
  // split that way polled far slower: 5.0-5.6 us instead of 2.8-3.4 us for
  // 3-48 streaming CTAs unless np was a multiple of 32
  // (profiles/r02_collector_small_grids.txt).
  while (__any_sync(0xffffffffu, q < np)) {
    unsigned long long h[kCollectBatch], l[kCollectBatch];
#pragma unroll
    for (int i = 0; i < kCollectBatch; ++i) {
      const unsigned s = q + C * i;
      if (s < np)
        asm volatile("ld.volatile.global.v2.u64 {%0,%1}, [%2];" : "=l"(h[i]), "=l"(l[i]) : "l"(a.slots + 2 * s));
      else
        h[i] = l[i] = 0ull;
    }
#pragma unroll
    for (int i = 0; i < kCollectBatch; ++i) {
      if (q >= np || h[i] == 0ull || l[i] == 0ull) break;
      DD p;
      p.hi = __longlong_as_double((long long)(h[i] ^ kSlotMask));
      p.lo = __longlong_as_double((long long)(l[i] ^ kSlotMask));
      v = dd_add(v, p);
      asm volatile("st.volatile.global.v2.u64 [%0], {%1,%2};" ::"l"(a.slots + 2 * q), "l"(0ull), "l"(0ull) : "memory");
      q += C;
    }
  }
  v = warp_reduce_dd(v);
  const unsigned warp = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) smem[warp] = v;
  if (nw > 1) asm volatile("bar.sync 1, %0;" ::"r"(C) : "memory");  // the collector warps only
  if (threadIdx.x == 0) {
    DD tot = v;
    for (int w = 1; w < nw; ++w) tot = dd_add(tot, smem[w]);
    if (a.xchg.world > 0) tot = exchange_dd(tot, a.xchg);
    finish_result<T>(tot, a);
  }
}

// Round a double-double total to the element type, optional sqrt, store.
template <class T> __device__ __forceinline__ void finish_store(DD tot, int flags, void* out) {
  if (flags & FLAG_PARTIAL) {
    *(DD*)out = dd_norm(tot);
    return;
  }
  T r = (T)(finite(tot.hi) ? __dadd_rn(tot.hi, tot.lo) : tot.hi);
  if (flags & FLAG_SQRT) r = Arith<T>::sqrt_rn(r);
  *(T*)out = r;
}

template <class EA, int R, int N>
template <class T, class E>
__device__ __forceinline__ void AssignRoots<EA, R, N>::vec(E& e, T* const* dst, i64 off) {
  typedef typename Roots<EA>::template At<R>::type Root;
  constexpr int V = sizeof(e.d[R]) / sizeof(T);
#pragma unroll
  for (int k = 0; k < V; ++k) e.d[R][k] = Root::ev(e, k);
  VecIO<T, V>::store(dst[R] + off, e.d[R]);
  AssignRoots<EA, R + 1, N>::template vec<T>(e, dst, off);
}
template <class EA, int R, int N>
template <class T, class E>
__device__ __forceinline__ void AssignRoots<EA, R, N>::one(E& e, T* const* dst, i64 i) {
  typedef typename Roots<EA>::template At<R>::type Root;
  e.d[R][0] = Root::ev(e, 0);
  dst[R][i] = e.d[R][0];
  AssignRoots<EA, R + 1, N>::template one<T>(e, dst, i);
}

// The reduction epilogue shared by the fused kernel and the interpreter:
// `mine` is this thread's partial; the CTA reduces it and the grid combines
// the CTA partials (see below).  Every thread of the CTA must call it.
template <class T, int BLOCK>
__device__ __forceinline__ void reduce_epilogue(DD mine, const Args<T>& a) {
  // Two-level deterministic combine.  Every CTA publishes its partial; the
  // last CTA to arrive in its group of a.group consecutive CTAs (GROUP, or
  // the whole grid when it is a single group) folds the
  // group's partials (thread t takes CTA t of the group, then a fixed
  // shuffle/shared-memory tree); the last group to finish folds the group
  // partials in group order.  Which CTA does the folding never changes
  // the order, so the result depends only on n — not on scheduling, SM
  // count or occupancy.
  static_assert(MAX_ONE_GROUP % BLOCK == 0 && GROUP <= MAX_ONE_GROUP, "group fold layout");
  __shared__ DD smem[BLOCK];
  __shared__ int stage;  // 0 done, 1 group finisher, 2 group + final finisher
  if (a.first) {
    collect_epilogue<T, BLOCK>(mine, a, smem);
    return;
  }
  DD part = block_reduce_dd<BLOCK>(mine, smem);
  if (gridDim.x == 1) {  // small n: no partials, no tickets, no fences
    if (threadIdx.x == 0) {
      if (a.xchg.world > 0) part = exchange_dd(part, a.xchg);
      finish_result<T>(part, a);
    }
    return;
  }
  if (a.cluster) {
    // Small n: the whole grid is one cluster (<= 16 CTAs).  Partials meet
    // in distributed shared memory behind one cluster barrier instead of
    // global partials + ticket atomics.  CTA 0 folds them exactly like the
    // single-group ticket path below (thread t takes CTA t, then the same
    // block tree), so both paths give the same bits.
    __shared__ DD cpart;
    if (threadIdx.x == 0) cpart = part;
    cluster_barrier();
    DD v; v.hi = 0.0; v.lo = 0.0;
    if (blockIdx.x == 0 && threadIdx.x < gridDim.x) {
      DD p;
      p.hi = ld_dsmem(&cpart.hi, threadIdx.x);
      p.lo = ld_dsmem(&cpart.lo, threadIdx.x);
      v = dd_add(v, p);
    }
    cluster_barrier();  // every CTA's shared memory stays alive until read
    if (blockIdx.x != 0) return;
    DD q = block_reduce_dd<BLOCK>(v, smem);
    if (threadIdx.x == 0) {
      if (a.xchg.world > 0) q = exchange_dd(q, a.xchg);
      finish_result<T>(q, a);
    }
    return;
  }
  const unsigned int G = (unsigned int)a.group;
  const unsigned int g = blockIdx.x / G;
  const unsigned int ngroups = (gridDim.x + G - 1) / G;
  const unsigned int gsize = min(G, gridDim.x - g * G);
  if (threadIdx.x == 0) {
    a.partials[blockIdx.x] = part;
    stage = ticket_add(&a.group_tickets[g]) == gsize - 1 ? 1 : 0;
  }
  __syncthreads();
  if (stage == 0) return;
  // Thread t folds CTAs t, t + BLOCK, ... of the group in that order (a
  // group has at most MAX_ONE_GROUP = 4 * BLOCK CTAs); the loads (L2:
  // other CTAs wrote these during this launch) are issued before the
  // first add so they overlap.
  DD v; v.hi = 0.0; v.lo = 0.0;
  {
    DD p[MAX_ONE_GROUP / BLOCK];
#pragma unroll
    for (int i = 0; i < MAX_ONE_GROUP / BLOCK; ++i) {
      const unsigned int b = threadIdx.x + i * BLOCK;
      if (b < gsize) {
        p[i].hi = __ldcg(&a.partials[g * G + b].hi);
        p[i].lo = __ldcg(&a.partials[g * G + b].lo);
      }
    }
#pragma unroll
    for (int i = 0; i < MAX_ONE_GROUP / BLOCK; ++i)
      if (threadIdx.x + i * BLOCK < gsize) v = dd_add(v, p[i]);
  }
  __syncthreads();
  DD q = block_reduce_dd<BLOCK>(v, smem);
  if (ngroups == 1) {  // one group: its finisher holds the total
    if (threadIdx.x == 0) {
      a.group_tickets[g] = 0u;
      if (a.xchg.world > 0) q = exchange_dd(q, a.xchg);
      finish_result<T>(q, a);
    }
    return;
  }
  if (threadIdx.x == 0) {
    a.group_partials[g] = q;
    a.group_tickets[g] = 0u;  // every CTA of the group has arrived
    stage = ticket_add(a.ticket) == ngroups - 1 ? 2 : 1;
  }
  __syncthreads();
  if (stage != 2) return;
  DD w; w.hi = 0.0; w.lo = 0.0;
  for (unsigned int b = threadIdx.x; b < ngroups; b += BLOCK) {
    DD p;
    p.hi = __ldcg(&a.group_partials[b].hi);
    p.lo = __ldcg(&a.group_partials[b].lo);
    w = dd_add(w, p);
  }
  __syncthreads();
  DD tot = block_reduce_dd<BLOCK>(w, smem);
  if (threadIdx.x == 0) {
    *a.ticket = 0u;  // ready for the next launch on this workspace
    // Sharded reduction: trade this rank's total with the other ranks over
    // NVLink peer memory inside this same kernel — no separate collective.
    if (a.xchg.world > 0) tot = exchange_dd(tot, a.xchg);
    finish_result<T>(tot, a);
  }
}

// Device-observed trace (-DSALT_TRACE, NVRTC builds only): thread 0 of the
// first streaming CTA appends (kind, element index, slot) to a.trace.
#ifdef SALT_TRACE
template <class T>
__device__ __forceinline__ void trace_event(const Args<T>& a, int kind, i64 idx, int slot) {
  if (!a.trace || blockIdx.x != (unsigned)a.first || threadIdx.x != 0) return;
  const long long k = a.trace[0];
  if (1 + 3 * (k + 1) > a.trace_cap) return;
  a.trace[1 + 3 * k] = kind;
  a.trace[2 + 3 * k] = idx;
  a.trace[3 + 3 * k] = slot;
  a.trace[0] = k + 1;
}
#define SALT_TRACE_EVENT(kind, idx, slot) trace_event(a, kind, idx, slot)
#else
#define SALT_TRACE_EVENT(kind, idx, slot) ((void)0)
#endif

// ---------------------------------------------------------------- the kernel
// MODE_ASSIGN:        dst[i] = EA(i)
// MODE_REDUCE:        out    = sum_i ER(i)
// MODE_ASSIGN_REDUCE: dst[i] = EA(i); out = sum_i ER(i, D = dst[i])   (one pass)
//
// Layout of the index space: [0, head) scalar, then nvec aligned vectors of
// V lanes, then the scalar tail.  The vectors are cut into tiles of
// BLOCK*UNR; CTA b owns tiles [b*K, b*K + K) (K = tiles_per_cta: 1, or more
// once a reduction would need more than 65,536 streaming CTAs).  Per tile a
// thread issues all UNR x NL 256-bit loads before any arithmetic: the GPU
// form of the reference's load burst / vector_op burst / store burst
// (engine.py:209-225).  UNR: 2 for assignments (1 up to 2^20 vectors), 4 / 2
// for reductions (salt_abi.cu unroll_for), 8 / 16 elements when V == 1.
template <class T, class EA, class ER, int MODE, int V, int UNR, int BLOCK>
// SALT_MIN_BLOCKS (tuning: SALT_JIT_MINB JIT-builds with it) caps registers
// for that many CTAs per SM.  Left undefined on purpose: an explicit
// minimum of 1 lets ptxas spend more registers (ddot 56 -> 78) and costs
// ~10 % bandwidth (profiles/r01_launch_bounds.txt).
#ifdef SALT_MIN_BLOCKS
#define SALT_BOUNDS(B) __launch_bounds__(B, SALT_MIN_BLOCKS)
#else
#define SALT_BOUNDS(B) __launch_bounds__(B)
#endif
__global__ void SALT_BOUNDS(BLOCK) fused_kernel(Args<T> a) {
  constexpr int NL = cmax(EA::NL, ER::NL);
  constexpr int NS = cmax(EA::NS, ER::NS);
  constexpr int NP = cmax(EA::NP, ER::NP);
  constexpr bool ASSIGN = MODE != MODE_REDUCE;
  constexpr bool REDUCE = MODE != MODE_ASSIGN;
  typedef Env<T, NL, NS, NP, Roots<EA>::N, V> E1;
  typedef Env<T, NL, NS, NP, Roots<EA>::N, 1> ES;
  // Programmatic dependent launch: the host launches fused kernels with
  // programmatic stream serialization, so this grid may be scheduled while
  // the previous kernel on the stream is still finishing.  Nothing in global
  // memory is touched before this wait returns (it returns once every
  // prerequisite grid has completed and its writes are visible; without the
  // launch attribute it is a no-op).  B200, 400 back-to-back axpy launches
  // (tools/pdl_probe.cu): 2^20 f64 4.74 -> 2.87 us per launch eager,
  // 2.97 -> 2.71 us in a CUDA graph.
  asm volatile("griddepcontrol.wait;" ::: "memory");
  T pv[NP > 0 ? NP : 1];  // device scalars, loaded (or computed) once per thread
  if (NP > 0) load_pscalars(a, pv, NP);

  Acc<T> acc;
  constexpr int ND = Roots<EA>::N;
  // streaming CTA index (the collector CTA, if any, is blockIdx 0: cta < 0)
  const i64 cta = (i64)blockIdx.x - a.first;
  const i64 nthreads = ((i64)gridDim.x - a.first) * BLOCK;
  const i64 gtid = cta * BLOCK + threadIdx.x;

  // ---- scalar head + tail (at most 2*(V-1) elements, or all of them if V == 1)
  if (cta >= 0) {
    const i64 tail0 = a.head + a.nvec * V;
    const i64 nscalar = a.head + (a.n - tail0);
    for (i64 t = gtid; t < nscalar; t += nthreads) {
      const i64 i = t < a.head ? t : tail0 + (t - a.head);
      ES e;
#pragma unroll
      for (int l = 0; l < NL; ++l) e.x[l][0] = a.leaf[l][i];
#pragma unroll
      for (int s = 0; s < NS; ++s) e.s[s] = a.sc[s];
#pragma unroll
      for (int q = 0; q < NP; ++q) e.p[q] = pv[q];
      if (ASSIGN) AssignRoots<EA, 0, ND>::template one<T>(e, a.dst, i);
      if (REDUCE) acc.add(ER::ev(e, 0));
      SALT_TRACE_EVENT(3, i, -1);
    }
  }

  // ---- vector body: this CTA's run of consecutive tiles of BLOCK*UNR vectors
  const i64 tile0 = cta * a.tiles_per_cta;
  const i64 ntiles = (a.nvec + (i64)BLOCK * UNR - 1) / ((i64)BLOCK * UNR);
  const i64 tile1 = tile0 + a.tiles_per_cta < ntiles ? tile0 + a.tiles_per_cta : ntiles;
  // V == 1 (operands that do not share one misalignment): the host cuts nvec
  // to whole tiles (the ragged end joins the scalar tail above), so no slot
  // needs a bounds predicate — a V == 1 tile has 8-16 slots and only 7
  // predicate registers, and the predicated form issued its last loads only
  // after the first had returned.
  for (i64 t = cta < 0 ? tile1 : tile0; t < tile1; ++t) {
    const i64 base = t * BLOCK * UNR + threadIdx.x;
    E1 e[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const i64 j = base + (i64)u * BLOCK;
      if (V == 1 || j < a.nvec) {
        const i64 off = a.head + j * V;
#pragma unroll
        for (int l = 0; l < NL; ++l) VecIO<T, V>::load(e[u].x[l], a.leaf[l] + off);
        SALT_TRACE_EVENT(0, off, u);
      }
    }
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const i64 j = base + (i64)u * BLOCK;
      if (V == 1 || j < a.nvec) {
#pragma unroll
        for (int s = 0; s < NS; ++s) e[u].s[s] = a.sc[s];
#pragma unroll
        for (int q = 0; q < NP; ++q) e[u].p[q] = pv[q];
        SALT_TRACE_EVENT(1, a.head + j * V, u);
        if (ASSIGN) AssignRoots<EA, 0, ND>::template vec<T>(e[u], a.dst, a.head + j * V);
        if (ASSIGN) SALT_TRACE_EVENT(2, a.head + j * V, u);
        if (REDUCE) {
#pragma unroll
          for (int k = 0; k < V; ++k) acc.add(ER::ev(e[u], k));
        }
      }
    }
  }

  if (REDUCE) {
    SALT_TRACE_EVENT(4, -1, -1);
    reduce_epilogue<T, BLOCK>(acc.get(), a);
  }
}

// ---------------------------------------------------------------- batches
// Many independent assignments of ONE tree shape (different vectors,
// scalars and lengths) in ONE launch — for launch-bound sizes, where a
// launch per tree costs more than its work.  The problem table travels in
// the kernel parameters (CUDA >= 12.1 allows 32 KiB).  Problem q owns the
// global tiles [tile0, tile0 + nst + vector tiles): its first nst tiles are
// its head / tail elements (BLOCK per tile, scalar; all of it when its
// operands do not share one 32-byte alignment), the rest BLOCK*UNR-vector
// tiles exactly as in fused_kernel.  Same arithmetic per element, so the
// same bits as one fused_kernel launch per problem.
enum { BATCH_MAX = 96, BATCH_LEAVES = 8, BATCH_SCALARS = 8 };
template <class T> struct BatchProblem {
  T* dst;
  const T* leaf[BATCH_LEAVES];
  T sc[BATCH_SCALARS];
  i64 n, head, nvec;  // as Args
  i64 tile0;          // first global tile
  i64 nst;            // scalar tiles
};
template <class T> struct BatchArgs {
  int count;
  BatchProblem<T> p[BATCH_MAX];
};

template <class T, class EA, int V, int UNR, int BLOCK>
__global__ void SALT_BOUNDS(BLOCK) batch_kernel(BatchArgs<T> a) {
  asm volatile("griddepcontrol.wait;" ::: "memory");  // see fused_kernel
  constexpr int NL = EA::NL, NS = EA::NS;
  static_assert(NL <= BATCH_LEAVES && NS <= BATCH_SCALARS && EA::NP == 0, "batch tree limits");
  typedef Env<T, NL, NS, 0, 1, V> E1;
  typedef Env<T, NL, NS, 0, 1, 1> ES;
  int lo = 0, hi = a.count - 1;  // the problem owning this CTA: last tile0 <= blockIdx.x
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (a.p[mid].tile0 <= (i64)blockIdx.x) lo = mid;
    else hi = mid - 1;
  }
  const BatchProblem<T>& P = a.p[lo];
  T* const dst[1] = {P.dst};
  const i64 local = (i64)blockIdx.x - P.tile0;
  if (local < P.nst) {  // head / tail elements of this problem
    const i64 tail0 = P.head + P.nvec * V;
    const i64 nscalar = P.head + (P.n - tail0);
    const i64 t = local * BLOCK + threadIdx.x;
    if (t < nscalar) {
      const i64 i = t < P.head ? t : tail0 + (t - P.head);
      ES e;
#pragma unroll
      for (int l = 0; l < NL; ++l) e.x[l][0] = P.leaf[l][i];
#pragma unroll
      for (int s = 0; s < NS; ++s) e.s[s] = P.sc[s];
      AssignRoots<EA, 0, 1>::template one<T>(e, dst, i);
    }
    return;
  }
  const i64 base = (local - P.nst) * BLOCK * UNR + threadIdx.x;
  E1 e[UNR];
#pragma unroll
  for (int u = 0; u < UNR; ++u) {
    const i64 j = base + (i64)u * BLOCK;
    if (j < P.nvec) {
#pragma unroll
      for (int l = 0; l < NL; ++l) VecIO<T, V>::load(e[u].x[l], P.leaf[l] + P.head + j * V);
    }
  }
#pragma unroll
  for (int u = 0; u < UNR; ++u) {
    const i64 j = base + (i64)u * BLOCK;
    if (j < P.nvec) {
#pragma unroll
      for (int s = 0; s < NS; ++s) e[u].s[s] = P.sc[s];
      AssignRoots<EA, 0, 1>::template vec<T>(e[u], dst, P.head + j * V);
    }
  }
}

// Batched small reductions: CTA q sums problem q entirely — its head/tail
// elements, then its <= 2 tiles in order — and rounds it (flags: sqrt,
// partial) into P.dst, exactly the order of a one-CTA fused_kernel launch
// (which every reduction of <= 2 tiles is), so each result has the bits of
// its own salt_reduce.  Problems with more tiles are not batched.
template <class T, class ER, int V, int UNR, int BLOCK>
__global__ void SALT_BOUNDS(BLOCK) batch_reduce_kernel(BatchArgs<T> a, int flags) {
  asm volatile("griddepcontrol.wait;" ::: "memory");  // see fused_kernel
  constexpr int NL = ER::NL, NS = ER::NS;
  static_assert(NL <= BATCH_LEAVES && NS <= BATCH_SCALARS && ER::NP == 0, "batch tree limits");
  typedef Env<T, NL, NS, 0, 1, V> E1;
  typedef Env<T, NL, NS, 0, 1, 1> ES;
  const BatchProblem<T>& P = a.p[blockIdx.x];
  Acc<T> acc;
  {
    const i64 tail0 = P.head + P.nvec * V;
    const i64 nscalar = P.head + (P.n - tail0);
    for (i64 t = threadIdx.x; t < nscalar; t += BLOCK) {
      const i64 i = t < P.head ? t : tail0 + (t - P.head);
      ES e;
#pragma unroll
      for (int l = 0; l < NL; ++l) e.x[l][0] = P.leaf[l][i];
#pragma unroll
      for (int s = 0; s < NS; ++s) e.s[s] = P.sc[s];
      acc.add(ER::ev(e, 0));
    }
  }
  const i64 ntiles = (P.nvec + (i64)BLOCK * UNR - 1) / ((i64)BLOCK * UNR);
  for (i64 t = 0; t < ntiles; ++t) {
    const i64 base = t * BLOCK * UNR + threadIdx.x;
    E1 e[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const i64 j = base + (i64)u * BLOCK;
      if (j < P.nvec) {
#pragma unroll
        for (int l = 0; l < NL; ++l) VecIO<T, V>::load(e[u].x[l], P.leaf[l] + P.head + j * V);
      }
    }
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const i64 j = base + (i64)u * BLOCK;
      if (j < P.nvec) {
#pragma unroll
        for (int s = 0; s < NS; ++s) e[u].s[s] = P.sc[s];
#pragma unroll
        for (int k = 0; k < V; ++k) acc.add(ER::ev(e[u], k));
      }
    }
  }
  __shared__ DD smem[BLOCK];
  DD part = block_reduce_dd<BLOCK>(acc.get(), smem);
  if (threadIdx.x == 0) finish_store<T>(part, flags, P.dst);
}

// Combine `count` partials (all-gathered per-device DD values, rank order).
// Up to XCHG_MAX_RANKS partials are folded sequentially in rank order — the
// same arithmetic as exchange_dd, so the NCCL all-gather path and the NVLink
// exchange path give identical bits.
template <class T, int BLOCK>
__global__ void __launch_bounds__(BLOCK) finish_kernel(const DD* parts, int count, int flags, void* out) {
  __shared__ DD smem[BLOCK];
  if (count <= XCHG_MAX_RANKS) {
    if (threadIdx.x == 0) {
      DD v; v.hi = 0.0; v.lo = 0.0;
      for (int b = 0; b < count; ++b) v = dd_add(v, parts[b]);
      finish_store<T>(v, flags, out);
    }
    return;
  }
  DD v; v.hi = 0.0; v.lo = 0.0;
  for (int b = threadIdx.x; b < count; b += BLOCK) v = dd_add(v, parts[b]);
  DD tot = block_reduce_dd<BLOCK>(v, smem);
  if (threadIdx.x == 0) finish_store<T>(tot, flags, out);
}

// Single-GPU emulation of the exchange protocol for testing: block r plays
// rank r (all `world` blocks are co-resident: cooperative launch), with
// per-rank buffers in one allocation; `rounds` consecutive epochs reuse the
// buffers exactly like consecutive sharded reductions do.
__global__ void exchange_emulate_kernel(const DD* totals, DD* results, DD* slots,
                                        unsigned long long* flags, int world, int rounds,
                                        unsigned long long epoch0) {
  if (threadIdx.x != 0) return;
  Xchg x;
  x.rank = blockIdx.x;
  x.world = world;
  x.timeout_ns = 10000000000ull;
  x.error = nullptr;
  for (int p = 0; p < world; ++p) {
    x.slots[p] = slots + p * 2 * XCHG_MAX_RANKS;
    x.flags[p] = flags + p * XCHG_MAX_RANKS;
  }
  for (int r = 0; r < rounds; ++r) {
    x.epoch = epoch0 + r;
    results[r * world + x.rank] = exchange_dd(totals[r * world + x.rank], x);
  }
}

}  // namespace salt
