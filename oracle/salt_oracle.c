/*
 * salt_oracle.c — TEST INFRASTRUCTURE ONLY (parity checker / CPU baseline).
 *
 * A plain-C restatement of the reference's evaluation of BLAS-1 expression
 * trees (pkg/src/lanevec), used by tests/ to check libsalt.so, and by
 * bench.py's cpu_baseline / --impl reference leg as the CPU timing of the
 * reference algorithm.  Never linked into or called by the product.
 *
 * What it restates:
 *   - _BinaryNode.block_op (expressions.py:248-249): left op right, one
 *     IEEE op in the element type per node; ScaleNode.block_op (:319-320):
 *     alpha * child with alpha in the element type.  Evaluated tile by tile
 *     (a tile is the C analogue of the engine's U*W block, engine.py:253-255)
 *     with -ffp-contract=off so no FMA is formed.
 *   - _run_block_reduce (engine.py:267-292): a flat accumulator of B = U*W
 *     lanes in the element type, acc[j] += value[i] for i = j mod B over the
 *     masked main loop, a scalar remainder accumulator over the tail
 *     (SumNode.single_op, expressions.py:449-452), then combine_partials
 *     (expressions.py:470-480): rows in slot order, each folded left to right
 *     (horizontal_sum, lanes.py:160-170), the remainder added last.
 *
 * Signatures are the same postfix strings libsalt.so takes (include/salt.h).
 * Build: make -C oracle  (gcc -O2 -ffp-contract=off -fno-fast-math).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OR_MAX_PROG 256
#define OR_MAX_LEAVES 64
#define OR_MAX_SCALARS 64
#define OR_TILE 2048 /* multiple of every U*W (<= 128) */

enum { OP_LEAF, OP_SCALAR, OP_D, OP_ADD, OP_SUB, OP_MUL };

typedef struct {
  int op[OR_MAX_PROG];
  int arg[OR_MAX_PROG];
  int len;
  int max_depth;
} prog_t;

static int parse(const char* s, prog_t* p, int nleaves, int nscalars, int allow_d) {
  int depth = 0;
  p->len = 0;
  p->max_depth = 0;
  while (*s) {
    while (*s == ' ') ++s;
    if (!*s) break;
    const char* t = s;
    while (*s && *s != ' ') ++s;
    int tl = (int)(s - t);
    if (p->len >= OR_MAX_PROG) return -1;
    int op, arg = 0;
    if (tl == 1 && (*t == '+' || *t == '-' || *t == '*')) {
      op = *t == '+' ? OP_ADD : *t == '-' ? OP_SUB : OP_MUL;
      if (depth < 2) return -1;
      depth -= 1;
    } else if (tl == 1 && *t == 'D') {
      if (!allow_d) return -1;
      op = OP_D;
      depth += 1;
    } else if (tl >= 2 && (*t == 'L' || *t == 'S')) {
      for (int i = 1; i < tl; ++i) {
        if (t[i] < '0' || t[i] > '9') return -1;
        arg = arg * 10 + (t[i] - '0');
      }
      op = *t == 'L' ? OP_LEAF : OP_SCALAR;
      if (op == OP_LEAF && (arg >= nleaves || arg >= OR_MAX_LEAVES)) return -1;
      if (op == OP_SCALAR && (arg >= nscalars || arg >= OR_MAX_SCALARS)) return -1;
      depth += 1;
    } else {
      return -1;
    }
    p->op[p->len] = op;
    p->arg[p->len] = arg;
    p->len++;
    if (depth > p->max_depth) p->max_depth = depth;
  }
  return depth == 1 ? 0 : -1;
}

/* ---- one element type at a time: T, SUFFIX ---- */
#define DEFINE_FOR(T, SFX)                                                                  \
  /* Evaluate tile [t0, t0+m) of the tree; result pointer returned (may point into a      \
     leaf when the tree is a bare leaf).  bufs: (max_depth) scratch tiles. */              \
  static const T* eval_tile_##SFX(const prog_t* p, const T* const* leaves, const T* sc,    \
                                   const T* dval, int64_t t0, int m, T (*bufs)[OR_TILE]) {  \
    const T* vec[OR_MAX_PROG];                                                              \
    T scal[OR_MAX_PROG];                                                                    \
    int is_vec[OR_MAX_PROG];                                                                \
    int sp = 0;                                                                             \
    for (int i = 0; i < p->len; ++i) {                                                      \
      int op = p->op[i];                                                                    \
      if (op == OP_LEAF) { vec[sp] = leaves[p->arg[i]] + t0; is_vec[sp++] = 1; continue; }  \
      if (op == OP_D) { vec[sp] = dval; is_vec[sp++] = 1; continue; }                       \
      if (op == OP_SCALAR) { scal[sp] = sc[p->arg[i]]; is_vec[sp++] = 0; continue; }        \
      int ia = sp - 2, ib = sp - 1;                                                         \
      if (!is_vec[ia] && !is_vec[ib]) {                                                     \
        T a = scal[ia], b = scal[ib];                                                       \
        scal[ia] = op == OP_ADD ? (T)(a + b) : op == OP_SUB ? (T)(a - b) : (T)(a * b);      \
        sp = ib;                                                                            \
        continue;                                                                           \
      }                                                                                     \
      T* r = bufs[ia];                                                                      \
      const T* A = vec[ia];                                                                 \
      const T* B = vec[ib];                                                                 \
      T sa = scal[ia], sb = scal[ib];                                                       \
      if (is_vec[ia] && is_vec[ib]) {                                                       \
        if (op == OP_ADD) for (int k = 0; k < m; ++k) r[k] = A[k] + B[k];                   \
        else if (op == OP_SUB) for (int k = 0; k < m; ++k) r[k] = A[k] - B[k];              \
        else for (int k = 0; k < m; ++k) r[k] = A[k] * B[k];                                \
      } else if (is_vec[ib]) {                                                              \
        if (op == OP_ADD) for (int k = 0; k < m; ++k) r[k] = sa + B[k];                     \
        else if (op == OP_SUB) for (int k = 0; k < m; ++k) r[k] = sa - B[k];                \
        else for (int k = 0; k < m; ++k) r[k] = sa * B[k];                                  \
      } else {                                                                              \
        if (op == OP_ADD) for (int k = 0; k < m; ++k) r[k] = A[k] + sb;                     \
        else if (op == OP_SUB) for (int k = 0; k < m; ++k) r[k] = A[k] - sb;                \
        else for (int k = 0; k < m; ++k) r[k] = A[k] * sb;                                  \
      }                                                                                     \
      vec[ia] = r;                                                                          \
      is_vec[ia] = 1;                                                                       \
      sp = ib;                                                                              \
    }                                                                                       \
    if (!is_vec[0]) { /* constant tree: broadcast */                                        \
      for (int k = 0; k < m; ++k) bufs[0][k] = scal[0];                                     \
      return bufs[0];                                                                       \
    }                                                                                       \
    return vec[0];                                                                          \
  }                                                                                         \
                                                                                            \
  typedef struct {                                                                          \
    const prog_t* p;                                                                        \
    const prog_t* pr;                                                                       \
    T* dst;                                                                                 \
    const T* const* leaves;                                                                 \
    const T* sc;                                                                            \
    int64_t lo, hi;                                                                         \
    int unroll, width;                                                                      \
    T result;                                                                               \
    int rc;                                                                                 \
  } job_##SFX;                                                                              \
                                                                                            \
  static void* assign_worker_##SFX(void* arg) {                                             \
    job_##SFX* j = (job_##SFX*)arg;                                                         \
    T(*bufs)[OR_TILE] = malloc(sizeof(T) * OR_TILE * (j->p->max_depth + 1));                \
    if (!bufs) { j->rc = -2; return NULL; }                                                 \
    for (int64_t t0 = j->lo; t0 < j->hi; t0 += OR_TILE) {                                   \
      int m = (int)(j->hi - t0 < OR_TILE ? j->hi - t0 : OR_TILE);                           \
      const T* v = eval_tile_##SFX(j->p, j->leaves, j->sc, NULL, t0, m, bufs);              \
      /* whole tile materialised before the store: exact aliasing is safe               \
         (AssignNode.block_commit, expressions.py:392-395) */                              \
      memmove(j->dst + t0, v, sizeof(T) * (size_t)m);                                       \
    }                                                                                       \
    free(bufs);                                                                             \
    return NULL;                                                                            \
  }                                                                                         \
                                                                                            \
  /* _run_block_reduce over [lo, hi) with B = U*W lanes; hi-lo's tail is the remainder. */ \
  static void* reduce_worker_##SFX(void* arg) {                                             \
    job_##SFX* j = (job_##SFX*)arg;                                                         \
    const int B = j->unroll * j->width;                                                     \
    int nb = j->pr->max_depth;                                                              \
    if (j->p && j->p->max_depth > nb) nb = j->p->max_depth;                                 \
    T(*bufs)[OR_TILE] = malloc(sizeof(T) * OR_TILE * (nb + 2));                             \
    T* acc = calloc((size_t)B, sizeof(T));                                                  \
    T* dv = (j->p && bufs) ? bufs[nb + 1] : NULL;                                           \
    if (!bufs || !acc) { free(bufs); free(acc); j->rc = -2; return NULL; }                 \
    const int64_t len = j->hi - j->lo;                                                      \
    const int64_t nm = len & ~(int64_t)(B - 1);                                             \
    T rem = (T)0;                                                                           \
    for (int64_t t0 = j->lo; t0 < j->hi; t0 += OR_TILE) {                                   \
      int m = (int)(j->hi - t0 < OR_TILE ? j->hi - t0 : OR_TILE);                           \
      if (j->p) { /* fused assign + reduce: D = the value just assigned */                  \
        const T* a = eval_tile_##SFX(j->p, j->leaves, j->sc, NULL, t0, m, bufs);            \
        memcpy(dv, a, sizeof(T) * (size_t)m);                                               \
        memcpy(j->dst + t0, dv, sizeof(T) * (size_t)m);                                     \
      }                                                                                     \
      const T* v = eval_tile_##SFX(j->pr, j->leaves, j->sc, dv, t0, m, bufs);               \
      for (int k = 0; k < m; ++k) {                                                         \
        int64_t i = t0 + k - j->lo;                                                         \
        if (i < nm) acc[i % B] = acc[i % B] + v[k];                                         \
        else rem = rem + v[k];                                                              \
      }                                                                                     \
    }                                                                                       \
    /* combine_partials: slot rows ascending, lanes left to right, remainder last */        \
    T total = (T)0;                                                                         \
    int have = 0;                                                                           \
    for (int s = 0; s < j->unroll && nm > 0; ++s) {                                         \
      T h = acc[s * j->width];                                                              \
      for (int k = 1; k < j->width; ++k) h = h + acc[s * j->width + k];                     \
      total = have ? (T)(total + h) : h;                                                    \
      have = 1;                                                                             \
    }                                                                                       \
    j->result = have ? (T)(total + rem) : rem;                                              \
    free(bufs);                                                                             \
    free(acc);                                                                              \
    return NULL;                                                                            \
  }

DEFINE_FOR(float, f32)
DEFINE_FOR(double, f64)

static int run_threads(void* (*fn)(void*), void* jobs, size_t job_size, int nt) {
  pthread_t th[256];
  if (nt == 1) {
    fn(jobs);
    return 0;
  }
  for (int t = 0; t < nt; ++t)
    if (pthread_create(&th[t], NULL, fn, (char*)jobs + job_size * t)) return -3;
  for (int t = 0; t < nt; ++t) pthread_join(th[t], NULL);
  return 0;
}

/* dst[i] = tree(i), tiles split over nthreads contiguous ranges. */
int oracle_assign(int dtype, const char* sig, void* dst, const void* const* leaves, int nleaves,
                  const double* scalars, int nscalars, int64_t n, int nthreads) {
  prog_t p;
  if (parse(sig, &p, nleaves, nscalars, 0)) return -1;
  if (nthreads < 1) nthreads = 1;
  if (nthreads > 256) nthreads = 256;
  int64_t per = (n + nthreads - 1) / nthreads;
  per = (per + OR_TILE - 1) / OR_TILE * OR_TILE;
  if (dtype == 0) {
    float sc[OR_MAX_SCALARS];
    for (int s = 0; s < nscalars && s < OR_MAX_SCALARS; ++s) sc[s] = (float)scalars[s];
    job_f32 jobs[256];
    for (int t = 0; t < nthreads; ++t) {
      int64_t lo = t * per < n ? t * per : n, hi = lo + per < n ? lo + per : n;
      jobs[t] = (job_f32){&p, NULL, (float*)dst, (const float* const*)leaves, sc, lo, hi, 1, 1, 0, 0};
    }
    return run_threads(assign_worker_f32, jobs, sizeof(job_f32), nthreads);
  } else {
    double sc[OR_MAX_SCALARS];
    for (int s = 0; s < nscalars && s < OR_MAX_SCALARS; ++s) sc[s] = scalars[s];
    job_f64 jobs[256];
    for (int t = 0; t < nthreads; ++t) {
      int64_t lo = t * per < n ? t * per : n, hi = lo + per < n ? lo + per : n;
      jobs[t] = (job_f64){&p, NULL, (double*)dst, (const double* const*)leaves, sc, lo, hi, 1, 1, 0, 0};
    }
    return run_threads(assign_worker_f64, jobs, sizeof(job_f64), nthreads);
  }
}

/* Reduction.  nthreads == 1 reproduces the reference engine bit for bit for
 * plan (unroll, width).  nthreads > 1 applies the same algorithm to
 * contiguous chunks and adds the chunk results in order (CPU baseline timing
 * only; not order-identical to the reference).  assign_sig may be NULL; if
 * given, dst receives the assigned values and `D` in reduce_sig reads them
 * (fused axpy -> dot).  out receives one element of the dtype. */
int oracle_reduce(int dtype, const char* assign_sig, const char* reduce_sig, void* dst,
                  const void* const* leaves, int nleaves, const double* scalars, int nscalars,
                  int64_t n, int unroll, int width, int nthreads, void* out) {
  prog_t pa, pr;
  if (assign_sig && parse(assign_sig, &pa, nleaves, nscalars, 0)) return -1;
  if (parse(reduce_sig, &pr, nleaves, nscalars, assign_sig != NULL)) return -1;
  if (unroll < 1 || width < 1 || ((unroll * width) & (unroll * width - 1)) ||
      unroll * width > 128)
    return -1;
  if (nthreads < 1) nthreads = 1;
  if (nthreads > 256) nthreads = 256;
  const int B = unroll * width;
  int64_t per = (n + nthreads - 1) / nthreads;
  per = (per + OR_TILE - 1) / OR_TILE * OR_TILE; /* chunk bases stay multiples of B */
  (void)B;
  if (dtype == 0) {
    float sc[OR_MAX_SCALARS];
    for (int s = 0; s < nscalars && s < OR_MAX_SCALARS; ++s) sc[s] = (float)scalars[s];
    job_f32 jobs[256];
    for (int t = 0; t < nthreads; ++t) {
      int64_t lo = t * per < n ? t * per : n, hi = lo + per < n ? lo + per : n;
      jobs[t] = (job_f32){assign_sig ? &pa : NULL, &pr, (float*)dst, (const float* const*)leaves,
                          sc, lo, hi, unroll, width, 0, 0};
    }
    int rc = run_threads(reduce_worker_f32, jobs, sizeof(job_f32), nthreads);
    if (rc) return rc;
    float total = jobs[0].result;
    for (int t = 1; t < nthreads; ++t) total = total + jobs[t].result;
    for (int t = 0; t < nthreads; ++t) if (jobs[t].rc) return jobs[t].rc;
    *(float*)out = total;
  } else {
    double sc[OR_MAX_SCALARS];
    for (int s = 0; s < nscalars && s < OR_MAX_SCALARS; ++s) sc[s] = scalars[s];
    job_f64 jobs[256];
    for (int t = 0; t < nthreads; ++t) {
      int64_t lo = t * per < n ? t * per : n, hi = lo + per < n ? lo + per : n;
      jobs[t] = (job_f64){assign_sig ? &pa : NULL, &pr, (double*)dst,
                          (const double* const*)leaves, sc, lo, hi, unroll, width, 0, 0};
    }
    int rc = run_threads(reduce_worker_f64, jobs, sizeof(job_f64), nthreads);
    if (rc) return rc;
    double total = jobs[0].result;
    for (int t = 1; t < nthreads; ++t) total = total + jobs[t].result;
    for (int t = 0; t < nthreads; ++t) if (jobs[t].rc) return jobs[t].rc;
    *(double*)out = total;
  }
  return 0;
}

/* ---- near-exact reduction: the acceptance oracle at sizes where math.fsum
 * over Python lists is too slow.  Element-typed tree values (as
 * test_acceptance.py:95-100 forms them) are accumulated in binary128
 * (__float128, 113-bit significand) per thread and the thread sums are added
 * in binary128: the error is ~n * 2^-113 relative to the largest partial
 * sum, i.e. ~1e-26 relative even at n = 2^31, far below the 1e-12 / 1e-5
 * tolerances being checked.  out = the sum rounded to double. */
typedef struct {
  const prog_t* p;
  const prog_t* pa;
  int dtype;
  const void* const* leaves;
  const double* scalars;
  int nscalars;
  int64_t lo, hi;
  __float128 acc;
  int rc;
} qjob_t;

static void* quad_worker(void* arg) {
  qjob_t* j = (qjob_t*)arg;
  int nb = j->p->max_depth + 2;
  if (j->pa && j->pa->max_depth + 2 > nb) nb = j->pa->max_depth + 2;
  __float128 acc = 0;
  if (j->dtype == 0) {
    float sc[OR_MAX_SCALARS];
    for (int s = 0; s < j->nscalars && s < OR_MAX_SCALARS; ++s) sc[s] = (float)j->scalars[s];
    float(*bufs)[OR_TILE] = malloc(sizeof(float) * OR_TILE * (nb + 1));
    if (!bufs) { j->rc = -2; return NULL; }
    for (int64_t t0 = j->lo; t0 < j->hi; t0 += OR_TILE) {
      int m = (int)(j->hi - t0 < OR_TILE ? j->hi - t0 : OR_TILE);
      const float* dv = NULL;
      if (j->pa) {
        const float* a = eval_tile_f32(j->pa, (const float* const*)j->leaves, sc, NULL, t0, m, bufs);
        memcpy(bufs[nb], a, sizeof(float) * (size_t)m);
        dv = bufs[nb];
      }
      const float* v = eval_tile_f32(j->p, (const float* const*)j->leaves, sc, dv, t0, m, bufs);
      for (int k = 0; k < m; ++k) acc += (__float128)v[k];
    }
    free(bufs);
  } else {
    double(*bufs)[OR_TILE] = malloc(sizeof(double) * OR_TILE * (nb + 1));
    if (!bufs) { j->rc = -2; return NULL; }
    for (int64_t t0 = j->lo; t0 < j->hi; t0 += OR_TILE) {
      int m = (int)(j->hi - t0 < OR_TILE ? j->hi - t0 : OR_TILE);
      const double* dv = NULL;
      if (j->pa) {
        const double* a = eval_tile_f64(j->pa, (const double* const*)j->leaves, j->scalars, NULL, t0, m, bufs);
        memcpy(bufs[nb], a, sizeof(double) * (size_t)m);
        dv = bufs[nb];
      }
      const double* v = eval_tile_f64(j->p, (const double* const*)j->leaves, j->scalars, dv, t0, m, bufs);
      for (int k = 0; k < m; ++k) acc += (__float128)v[k];
    }
    free(bufs);
  }
  j->acc = acc;
  return NULL;
}

/* Sum of the element-typed values of reduce_sig (optionally after the
 * assign tree, whose value `D` reads; the assignment is NOT stored). */
int oracle_reduce_exact(int dtype, const char* assign_sig, const char* reduce_sig,
                        const void* const* leaves, int nleaves, const double* scalars,
                        int nscalars, int64_t n, int nthreads, double* out) {
  prog_t pa, pr;
  if (assign_sig && parse(assign_sig, &pa, nleaves, nscalars, 0)) return -1;
  if (parse(reduce_sig, &pr, nleaves, nscalars, assign_sig != NULL)) return -1;
  if (nthreads < 1) nthreads = 1;
  if (nthreads > 256) nthreads = 256;
  int64_t per = (n + nthreads - 1) / nthreads;
  per = (per + OR_TILE - 1) / OR_TILE * OR_TILE;
  qjob_t jobs[256];
  for (int t = 0; t < nthreads; ++t) {
    int64_t lo = t * per < n ? t * per : n, hi = lo + per < n ? lo + per : n;
    jobs[t] = (qjob_t){&pr, assign_sig ? &pa : NULL, dtype, leaves, scalars, nscalars, lo, hi, 0, 0};
  }
  int rc = run_threads(quad_worker, jobs, sizeof(qjob_t), nthreads);
  if (rc) return rc;
  __float128 tot = 0;
  for (int t = 0; t < nthreads; ++t) {
    if (jobs[t].rc) return jobs[t].rc;
    tot += jobs[t].acc;
  }
  *out = (double)tot;
  return 0;
}
