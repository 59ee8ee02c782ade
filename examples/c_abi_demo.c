/*
 * c_abi_demo.c — the drop-in boundary used from plain C, no Python.
 *
 * What a non-Python host (a cgo / JNI / N-API binding, or a C solver) does
 * with libsalt.so: device vectors from cudaMalloc, one call per fused tree.
 *
 *   1. d = alpha*a + beta*(b - c)        salt_assign   (one kernel)
 *   2. r = dot(d, a)                     salt_reduce   (one kernel, device workspace)
 *   3. y = y + alpha*x ; r = dot(y, z)   salt_assign_reduce (one pass)
 *   4. the same axpy on HOST buffers     salt_assign_host (chunked PCIe pipeline)
 *   5. 64 small independent axpys         salt_assign_batch (one launch)
 *
 * Elementwise results are compared bit for bit with a plain C loop in the
 * reference's operation order (expressions.py:248-249, :320: left operand
 * first, alpha on the left, one rounding per operation); reductions with a
 * relative tolerance of 1e-12 against a long-double sum.  Exit code 0 = all
 * checks passed.
 *
 * Build (examples/Makefile, also run by tests/test_gpu_c_abi.py):
 *   gcc -O2 -ffp-contract=off c_abi_demo.c -I../include -L.. -lsalt -lcudart
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <cuda_runtime_api.h>

#include "salt.h"

#define CK(x)                                                                         \
  do {                                                                                \
    cudaError_t e_ = (x);                                                             \
    if (e_ != cudaSuccess) {                                                          \
      fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
      return 2;                                                                       \
    }                                                                                 \
  } while (0)
#define SK(x)                                                                         \
  do {                                                                                \
    int r_ = (x);                                                                     \
    if (r_ != SALT_OK) {                                                              \
      fprintf(stderr, "%s:%d %s -> %d: %s\n", __FILE__, __LINE__, #x, r_,             \
              salt_last_error());                                                     \
      return 3;                                                                       \
    }                                                                                 \
  } while (0)

static uint64_t rng = 0x1109126411091264ull;
static double uniform(void) { /* xorshift64*, U[-1, 1) */
  rng ^= rng >> 12;
  rng ^= rng << 25;
  rng ^= rng >> 27;
  return (double)((rng * 2685821657736338717ull) >> 11) / 4503599627370496.0 - 1.0;
}

static int same_bits(const double* x, const double* y, int64_t n, const char* what) {
  if (memcmp(x, y, (size_t)n * sizeof(double)) != 0) {
    for (int64_t i = 0; i < n; ++i)
      if (memcmp(&x[i], &y[i], sizeof(double))) {
        fprintf(stderr, "%s: element %lld differs: %.17g vs %.17g\n", what, (long long)i, x[i], y[i]);
        break;
      }
    return 0;
  }
  printf("%-44s bit-exact (%lld elements)\n", what, (long long)n);
  return 1;
}

static int close_to(double got, long double want, const char* what) {
  double rel = (double)fabsl(((long double)got - want) / want);
  printf("%-44s %.17g  rel.err %.2e\n", what, got, rel);
  return rel <= 1e-12;
}

int main(int argc, char** argv) {
  const int64_t n = argc > 1 ? atoll(argv[1]) : (1 << 22) + 3; /* ragged tail on purpose */
  const size_t bytes = (size_t)n * sizeof(double);
  printf("libsalt ABI %d, n = %lld\n", salt_abi_version(), (long long)n);

  double *ha = malloc(bytes), *hb = malloc(bytes), *hc = malloc(bytes), *hd = malloc(bytes),
         *want = malloc(bytes);
  for (int64_t i = 0; i < n; ++i) {
    ha[i] = uniform();
    hb[i] = uniform();
    hc[i] = uniform();
  }
  const double alpha = 1.25, beta = -0.5;

  double *a, *b, *c, *d;
  CK(cudaMalloc((void**)&a, bytes));
  CK(cudaMalloc((void**)&b, bytes));
  CK(cudaMalloc((void**)&c, bytes));
  CK(cudaMalloc((void**)&d, bytes));
  CK(cudaMemcpy(a, ha, bytes, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(b, hb, bytes, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(c, hc, bytes, cudaMemcpyHostToDevice));
  cudaStream_t s;
  CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  int ok = 1;

  /* 1. d = alpha*a + beta*(b - c) */
  const void* abc[3] = {a, b, c};
  const double ab[2] = {alpha, beta};
  SK(salt_assign(SALT_F64, "S0 L0 * S1 L1 L2 - * +", d, abc, 3, ab, 2, n, s));
  CK(cudaMemcpyAsync(hd, d, bytes, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  for (int64_t i = 0; i < n; ++i) {
    volatile double t1 = alpha * ha[i], t2 = hb[i] - hc[i];
    volatile double t3 = beta * t2;
    want[i] = t1 + t3;
  }
  ok &= same_bits(hd, want, n, "salt_assign  d = alpha*a + beta*(b-c)");

  /* 2. r = dot(d, a): device workspace, result copied to the host */
  const size_t wsb = salt_reduce_workspace_bytes();
  void* ws;
  CK(cudaMalloc(&ws, wsb));
  CK(cudaMemsetAsync(ws, 0, SALT_WORKSPACE_TICKET_BYTES, s));
  double* out;
  CK(cudaMalloc((void**)&out, 64));
  const void* da[2] = {d, a};
  double r = 0.0;
  SK(salt_reduce(SALT_F64, "L0 L1 *", da, 2, NULL, 0, n, 0, ws, wsb, out, &r, s));
  long double ref = 0.0L;
  for (int64_t i = 0; i < n; ++i) ref += (long double)(want[i] * ha[i]);
  ok &= close_to(r, ref, "salt_reduce  dot(d, a)");

  /* 3. fused axpy -> dot: b = b + alpha*a ; r = dot(b_new, c), one pass */
  const void* bac[3] = {b, a, c};
  SK(salt_assign_reduce(SALT_F64, "L0 S0 L1 * +", "D L2 *", b, bac, 3, &alpha, 1, n, 0, ws, wsb,
                        out, &r, s));
  CK(cudaMemcpyAsync(hd, b, bytes, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  ref = 0.0L;
  for (int64_t i = 0; i < n; ++i) {
    volatile double t = alpha * ha[i];
    want[i] = hb[i] + t;
    ref += (long double)(want[i] * hc[i]);
  }
  ok &= same_bits(hd, want, n, "salt_assign_reduce  b += alpha*a (b)");
  ok &= close_to(r, ref, "salt_assign_reduce  dot(b_new, c)");

  /* 4. host buffers: the library streams chunks through device staging */
  double *pa, *pb;
  CK(cudaMallocHost((void**)&pa, bytes));
  CK(cudaMallocHost((void**)&pb, bytes));
  memcpy(pa, ha, bytes);
  memcpy(pb, hb, bytes);
  const size_t staging_bytes = (size_t)96 << 20;
  void* staging;
  CK(cudaMalloc(&staging, staging_bytes));
  cudaStream_t st[3];
  for (int i = 0; i < 3; ++i) CK(cudaStreamCreateWithFlags(&st[i], cudaStreamNonBlocking));
  const void* hba[2] = {pb, pa};
  SK(salt_assign_host(SALT_F64, "L0 S0 L1 * +", pb, hba, 2, &alpha, 1, n, staging, staging_bytes,
                      (void* const*)st));
  ok &= same_bits(pb, want, n, "salt_assign_host  y += alpha*x (pinned)");

  /* 5. 64 independent axpys y_k += alpha_k * x_k of ragged small lengths,
   *    one batched launch; each must equal its own salt_assign */
  {
    enum { M = 64 };
    int64_t ns[M], off[M + 1];
    off[0] = 0;
    for (int k = 0; k < M; ++k) {
      ns[k] = 100 + 97 * k;
      off[k + 1] = off[k] + ns[k] + 3; /* +3: later problems start misaligned */
    }
    const size_t tb = (size_t)off[M] * sizeof(double);
    double *hx = malloc(tb), *hy = malloc(tb), *hy1 = malloc(tb), *hy2 = malloc(tb);
    for (int64_t i = 0; i < off[M]; ++i) {
      hx[i] = uniform();
      hy[i] = uniform();
    }
    double *x, *y1, *y2;
    CK(cudaMalloc((void**)&x, tb));
    CK(cudaMalloc((void**)&y1, tb));
    CK(cudaMalloc((void**)&y2, tb));
    CK(cudaMemcpy(x, hx, tb, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(y1, hy, tb, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(y2, hy, tb, cudaMemcpyHostToDevice));
    void* dsts[M];
    const void* lv[2 * M];
    double sc[M];
    for (int k = 0; k < M; ++k) {
      dsts[k] = y1 + off[k];
      lv[2 * k] = y1 + off[k];
      lv[2 * k + 1] = x + off[k];
      sc[k] = 0.125 * (k + 1);
    }
    SK(salt_assign_batch(SALT_F64, "L0 S0 L1 * +", M, dsts, lv, 2, sc, 1, ns, s));
    for (int k = 0; k < M; ++k) {
      const void* l2[2] = {y2 + off[k], x + off[k]};
      SK(salt_assign(SALT_F64, "L0 S0 L1 * +", y2 + off[k], l2, 2, &sc[k], 1, ns[k], s));
    }
    CK(cudaMemcpyAsync(hy1, y1, tb, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(hy2, y2, tb, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    ok &= same_bits(hy1, hy2, off[M], "salt_assign_batch  64 axpys == 64 salt_assign");
    free(hx); free(hy); free(hy1); free(hy2);
  }

  /* error path: a bad signature is refused before any launch */
  int rc = salt_assign(SALT_F64, "L0 +", d, abc, 3, NULL, 0, n, s);
  printf("%-44s rc=%d (%s)\n", "bad signature", rc, salt_last_error());
  ok &= rc == SALT_EINVAL;

  printf("%s\n", ok ? "ALL OK" : "FAILED");
  return ok ? 0 : 1;
}
