// salt_interp.cuh — postfix-interpreter kernel: the fallback for trees that
// are not in the compiled-in table when NVRTC is unavailable (or forced by
// salt_set_force_interp for testing).  Compiled ahead of time only; the
// NVRTC source (salt_expr.cuh) does not include it.
//
// Same semantics as fused_kernel, bit for bit on elementwise results: every
// node is one IEEE op in the element type through Arith<T> (left operand
// first, no FMA), assignment roots are evaluated in order and a later root
// reads an earlier root's value (D<r>), and reductions go through the same
// compensated accumulator and the same deterministic CTA / group combine
// (reduce_epilogue), over the same tiles of BLOCK*UNR vectors with the same
// UNR as the compiled kernel of that tree: a thread adds its values in the
// compiled kernel's order (head/tail elements, then per tile slot u = 0..UNR-1
// lane by lane), so reductions are bit-identical to the compiled kernels too
// — whichever kernel runs, a tree gives the same bits.
//
// The program comes in the kernel parameters (uniform across threads); the
// evaluation stack and the loaded leaf vectors live in shared memory, one
// column per thread ([slot][lane][thread], conflict-free), with the top of
// the stack in registers.  All of a vector's leaf loads are issued before
// the program runs (the load burst), four at a time.
#pragma once
#include "salt_expr.cuh"

namespace salt {

enum { OP_LEAF = 0, OP_SCALAR, OP_PSCALAR, OP_D, OP_ADD, OP_SUB, OP_MUL, OP_STORE, OP_ACC };
enum { MAX_PROG = 252 };

struct Prog {
  int len;       // tokens
  int nl;        // distinct leaves (loaded up front)
  int slots;     // stack slots in shared memory
  int nroots;    // assignment roots (OP_STORE targets)
  int reduce;    // 1: the program ends with OP_ACC
  unsigned char op[MAX_PROG];
  unsigned char arg[MAX_PROG];
};

template <class T> struct InterpArgs {
  Args<T> a;
  Prog pg;
};

// Shared-memory bytes one CTA needs for `pg` with V lanes per vector.
__host__ __device__ inline int interp_smem_bytes(const Prog& pg, int V, int block, int esz) {
  return (pg.nl + pg.slots + pg.nroots) * V * block * esz;
}

template <class T, int W, int BLOCK>
__device__ __forceinline__ void interp_eval(const Prog& pg, const Args<T>& a, const T* pv, T* sm,
                                            i64 off, Acc<T>& acc) {
  const int tid = threadIdx.x;
  T* X = sm;                                   // [nl][W][BLOCK]
  T* STK = sm + pg.nl * W * BLOCK;             // [slots][W][BLOCK]
  T* DV = STK + pg.slots * W * BLOCK;          // [nroots][W][BLOCK]
  // load burst: up to 4 leaves' vectors in flight per thread before any use
  for (int l0 = 0; l0 < pg.nl; l0 += 4) {
    T r[4][W];
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if (l0 + i < pg.nl) VecIO<T, W>::load(r[i], a.leaf[l0 + i] + off);
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if (l0 + i < pg.nl) {
#pragma unroll
        for (int w = 0; w < W; ++w) X[((l0 + i) * W + w) * BLOCK + tid] = r[i][w];
      }
  }
  T tos[W];
#pragma unroll
  for (int w = 0; w < W; ++w) tos[w] = T(0);
  int sp = 0;
  for (int i = 0; i < pg.len; ++i) {
    const int op = pg.op[i], k = pg.arg[i];
    if (op <= OP_D) {  // push: the old top goes to shared memory
#pragma unroll
      for (int w = 0; w < W; ++w) STK[(sp * W + w) * BLOCK + tid] = tos[w];
      ++sp;
      if (op == OP_LEAF) {
#pragma unroll
        for (int w = 0; w < W; ++w) tos[w] = X[(k * W + w) * BLOCK + tid];
      } else if (op == OP_SCALAR) {
        const T s = a.sc[k];
#pragma unroll
        for (int w = 0; w < W; ++w) tos[w] = s;
      } else if (op == OP_PSCALAR) {
        const T s = pv[k];
#pragma unroll
        for (int w = 0; w < W; ++w) tos[w] = s;
      } else {
#pragma unroll
        for (int w = 0; w < W; ++w) tos[w] = DV[(k * W + w) * BLOCK + tid];
      }
    } else if (op <= OP_MUL) {  // binary node: left = the slot below, right = top
      --sp;
#pragma unroll
      for (int w = 0; w < W; ++w) {
        const T l = STK[(sp * W + w) * BLOCK + tid];
        tos[w] = op == OP_ADD ? Arith<T>::add(l, tos[w])
                 : op == OP_SUB ? Arith<T>::sub(l, tos[w]) : Arith<T>::mul(l, tos[w]);
      }
    } else if (op == OP_STORE) {  // assignment root k: keep its value for D<k>, store it
#pragma unroll
      for (int w = 0; w < W; ++w) DV[(k * W + w) * BLOCK + tid] = tos[w];
      VecIO<T, W>::store(a.dst[k] + off, tos);
      sp = 0;
    } else {  // OP_ACC: the reduction tree's value joins the sum, lane by lane
#pragma unroll
      for (int w = 0; w < W; ++w) acc.add(tos[w]);
      sp = 0;
    }
  }
}

template <class T, int V, int UNR, int BLOCK>
__global__ void __launch_bounds__(BLOCK) interp_kernel(InterpArgs<T> ia) {
  asm volatile("griddepcontrol.wait;" ::: "memory");  // see fused_kernel
  const Args<T>& a = ia.a;
  const Prog& pg = ia.pg;
  extern __shared__ __align__(16) unsigned char interp_smem[];
  T* sm = (T*)interp_smem;
  Acc<T> acc;
  T pv[MAX_PSCALARS];  // device scalars (loaded or computed once per thread)
  load_pscalars(a, pv, a.nps);
  const i64 cta = (i64)blockIdx.x - a.first;  // < 0: the collector CTA
  const i64 nthreads = ((i64)gridDim.x - a.first) * BLOCK;
  const i64 gtid = cta * BLOCK + threadIdx.x;
  if (cta >= 0) {  // scalar head + tail, as fused_kernel
    const i64 tail0 = a.head + a.nvec * V;
    const i64 nscalar = a.head + (a.n - tail0);
    for (i64 t = gtid; t < nscalar; t += nthreads) {
      const i64 i = t < a.head ? t : tail0 + (t - a.head);
      interp_eval<T, 1, BLOCK>(pg, a, pv, sm, i, acc);
    }
  }
  const i64 ntiles = (a.nvec + (i64)BLOCK * UNR - 1) / ((i64)BLOCK * UNR);
  const i64 tile0 = cta * a.tiles_per_cta;
  const i64 tile1 = tile0 + a.tiles_per_cta < ntiles ? tile0 + a.tiles_per_cta : ntiles;
  for (i64 t = cta < 0 ? tile1 : tile0; t < tile1; ++t) {
    const i64 base = t * BLOCK * UNR + threadIdx.x;
    for (int u = 0; u < UNR; ++u) {
      const i64 j = base + (i64)u * BLOCK;
      if (j < a.nvec) interp_eval<T, V, BLOCK>(pg, a, pv, sm, a.head + j * V, acc);
    }
  }
  if (pg.reduce) reduce_epilogue<T, BLOCK>(acc.get(), a);
}

}  // namespace salt
