// Design-space probe for the fused streaming kernel on B200 (not product
// code): d = alpha*a + beta*(b - c), f64, n = 2^28, timed with CUDA events.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//        -o tools/stream_variants tools/stream_variants.cu && tools/stream_variants
//
// Variants: LDG/STG vector width (128/256 bit), unroll, CTAs per SM, store
// cache hint, and a TMA (cp.async.bulk) producer/consumer pipeline that
// stages each leaf tile in shared memory through an mbarrier ring.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1);} } while (0)

typedef long long i64;

__device__ __forceinline__ void ld4(double (&r)[4], const double* p) {
  asm volatile("ld.global.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];"
               : "=d"(r[0]), "=d"(r[1]), "=d"(r[2]), "=d"(r[3]) : "l"(p));
}
__device__ __forceinline__ void ld4_ef(double (&r)[4], const double* p) {
  asm volatile("ld.global.L1::no_allocate.L2::evict_first.v4.f64 {%0,%1,%2,%3}, [%4];"
               : "=d"(r[0]), "=d"(r[1]), "=d"(r[2]), "=d"(r[3]) : "l"(p));
}
__device__ __forceinline__ void ld4_pf(double (&r)[4], const double* p) {
  asm volatile("ld.global.L1::no_allocate.L2::256B.v4.f64 {%0,%1,%2,%3}, [%4];"
               : "=d"(r[0]), "=d"(r[1]), "=d"(r[2]), "=d"(r[3]) : "l"(p));
}
__device__ __forceinline__ void ld4_nc(double (&r)[4], const double* p) {
  asm volatile("ld.global.nc.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];"
               : "=d"(r[0]), "=d"(r[1]), "=d"(r[2]), "=d"(r[3]) : "l"(p));
}
__device__ __forceinline__ void st4(double* p, const double (&r)[4]) {
  asm volatile("st.global.L1::no_allocate.v4.f64 [%0], {%1,%2,%3,%4};"
               :: "l"(p), "d"(r[0]), "d"(r[1]), "d"(r[2]), "d"(r[3]) : "memory");
}
__device__ __forceinline__ void st4_cs(double* p, const double (&r)[4]) {
  asm volatile("st.global.cs.v4.f64 [%0], {%1,%2,%3,%4};"
               :: "l"(p), "d"(r[0]), "d"(r[1]), "d"(r[2]), "d"(r[3]) : "memory");
}
__device__ __forceinline__ void ld2(double (&r)[2], const double* p) {
  asm volatile("ld.global.L1::no_allocate.v2.f64 {%0,%1}, [%2];" : "=d"(r[0]), "=d"(r[1]) : "l"(p));
}
__device__ __forceinline__ void st2(double* p, const double (&r)[2]) {
  asm volatile("st.global.L1::no_allocate.v2.f64 [%0], {%1,%2};" :: "l"(p), "d"(r[0]), "d"(r[1]) : "memory");
}

__device__ __forceinline__ double f(double a, double b, double c, double al, double be) {
  return __dadd_rn(__dmul_rn(al, a), __dmul_rn(be, __dsub_rn(b, c)));
}

// Variant A: grid-stride, V4 (256-bit), UNR vectors per leaf per thread.
template <int UNR, int BLOCK, int MINB, int HINT>
__global__ void __launch_bounds__(BLOCK, MINB) kA(double* d, const double* a, const double* b,
                                                  const double* c, double al, double be, i64 nvec) {
  const i64 nthreads = (i64)gridDim.x * BLOCK;
  for (i64 base = (i64)blockIdx.x * BLOCK * UNR + threadIdx.x; base < nvec; base += nthreads * UNR) {
    double x[UNR][4], y[UNR][4], z[UNR][4];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      i64 j = base + (i64)u * BLOCK;
      if (j < nvec) {
        if (HINT == 1) { ld4_ef(x[u], a + 4 * j); ld4_ef(y[u], b + 4 * j); ld4_ef(z[u], c + 4 * j); }
        else { ld4(x[u], a + 4 * j); ld4(y[u], b + 4 * j); ld4(z[u], c + 4 * j); }
      }
    }
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      i64 j = base + (i64)u * BLOCK;
      if (j < nvec) {
        double r[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) r[k] = f(x[u][k], y[u][k], z[u][k], al, be);
        if (HINT == 2) st4_cs(d + 4 * j, r); else st4(d + 4 * j, r);
      }
    }
  }
}

// Variant B: 128-bit accesses.
template <int UNR, int BLOCK>
__global__ void __launch_bounds__(BLOCK) kB(double* d, const double* a, const double* b,
                                            const double* c, double al, double be, i64 nvec2) {
  const i64 nthreads = (i64)gridDim.x * BLOCK;
  for (i64 base = (i64)blockIdx.x * BLOCK * UNR + threadIdx.x; base < nvec2; base += nthreads * UNR) {
    double x[UNR][2], y[UNR][2], z[UNR][2];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      i64 j = base + (i64)u * BLOCK;
      if (j < nvec2) { ld2(x[u], a + 2 * j); ld2(y[u], b + 2 * j); ld2(z[u], c + 2 * j); }
    }
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      i64 j = base + (i64)u * BLOCK;
      if (j < nvec2) {
        double r[2];
        r[0] = f(x[u][0], y[u][0], z[u][0], al, be);
        r[1] = f(x[u][1], y[u][1], z[u][1], al, be);
        st2(d + 2 * j, r);
      }
    }
  }
}

// Variant C: non-persistent, one tile per CTA (no grid-stride loop).
template <int UNR, int BLOCK>
__global__ void __launch_bounds__(BLOCK) kC(double* d, const double* a, const double* b,
                                            const double* c, double al, double be, i64 nvec) {
  i64 base = (i64)blockIdx.x * BLOCK * UNR + threadIdx.x;
  double x[UNR][4], y[UNR][4], z[UNR][4];
#pragma unroll
  for (int u = 0; u < UNR; ++u) {
    i64 j = base + (i64)u * BLOCK;
    if (j < nvec) { ld4(x[u], a + 4 * j); ld4(y[u], b + 4 * j); ld4(z[u], c + 4 * j); }
  }
#pragma unroll
  for (int u = 0; u < UNR; ++u) {
    i64 j = base + (i64)u * BLOCK;
    if (j < nvec) {
      double r[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) r[k] = f(x[u][k], y[u][k], z[u][k], al, be);
      st4(d + 4 * j, r);
    }
  }
}

// Variant E: variant C with a load hint: 1 = L2::256B prefetch, 2 = ld.global.nc.
template <int UNR, int BLOCK, int LH>
__global__ void __launch_bounds__(BLOCK) kE(double* d, const double* a, const double* b,
                                            const double* c, double al, double be, i64 nvec) {
  i64 base = (i64)blockIdx.x * BLOCK * UNR + threadIdx.x;
  double x[UNR][4], y[UNR][4], z[UNR][4];
#pragma unroll
  for (int u = 0; u < UNR; ++u) {
    i64 j = base + (i64)u * BLOCK;
    if (j < nvec) {
      if (LH == 1) { ld4_pf(x[u], a + 4 * j); ld4_pf(y[u], b + 4 * j); ld4_pf(z[u], c + 4 * j); }
      else { ld4_nc(x[u], a + 4 * j); ld4_nc(y[u], b + 4 * j); ld4_nc(z[u], c + 4 * j); }
    }
  }
#pragma unroll
  for (int u = 0; u < UNR; ++u) {
    i64 j = base + (i64)u * BLOCK;
    if (j < nvec) {
      double r[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) r[k] = f(x[u][k], y[u][k], z[u][k], al, be);
      st4(d + 4 * j, r);
    }
  }
}

// Variant D: persistent grid-stride with a register double buffer: the
// loads of iteration i+1 are issued before iteration i is computed/stored.
template <int UNR, int BLOCK>
__global__ void __launch_bounds__(BLOCK) kD(double* d, const double* a, const double* b,
                                            const double* c, double al, double be, i64 nvec) {
  const i64 nthreads = (i64)gridDim.x * BLOCK;
  i64 base = (i64)blockIdx.x * BLOCK * UNR + threadIdx.x;
  double x[UNR][4], y[UNR][4], z[UNR][4];
  auto load = [&](i64 bs) {
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      i64 j = bs + (i64)u * BLOCK;
      if (j < nvec) { ld4(x[u], a + 4 * j); ld4(y[u], b + 4 * j); ld4(z[u], c + 4 * j); }
    }
  };
  if (base < nvec) load(base);
  for (; base < nvec; base += nthreads * UNR) {
    double r[UNR][4];
#pragma unroll
    for (int u = 0; u < UNR; ++u)
#pragma unroll
      for (int k = 0; k < 4; ++k) r[u][k] = f(x[u][k], y[u][k], z[u][k], al, be);
    const i64 next = base + nthreads * UNR;
    if (next < nvec) load(next);
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      i64 j = base + (i64)u * BLOCK;
      if (j < nvec) st4(d + 4 * j, r[u]);
    }
  }
}

// Reduction probes: dot(a, b) f64 with TwoSum per term.
__device__ __forceinline__ void two_sum(double a, double b, double& s, double& e) {
  s = __dadd_rn(a, b);
  double bp = __dsub_rn(s, a);
  double ap = __dsub_rn(s, bp);
  e = __dadd_rn(__dsub_rn(a, ap), __dsub_rn(b, bp));
}
template <int UNR, int BLOCK, bool PREFETCH>
__global__ void __launch_bounds__(BLOCK) kR(const double* a, const double* b, i64 nvec, double* part) {
  const i64 nthreads = (i64)gridDim.x * BLOCK;
  double hi = 0, lo = 0;
  i64 base = (i64)blockIdx.x * BLOCK * UNR + threadIdx.x;
  double x[UNR][4], y[UNR][4];
  auto load = [&](i64 bs) {
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      i64 j = bs + (i64)u * BLOCK;
      if (j < nvec) { ld4(x[u], a + 4 * j); ld4(y[u], b + 4 * j); }
      else { for (int k = 0; k < 4; ++k) x[u][k] = y[u][k] = 0; }
    }
  };
  if (PREFETCH && base < nvec) load(base);
  for (; base < nvec; base += nthreads * UNR) {
    if (!PREFETCH) load(base);
    double p[UNR][4];
#pragma unroll
    for (int u = 0; u < UNR; ++u)
#pragma unroll
      for (int k = 0; k < 4; ++k) p[u][k] = __dmul_rn(x[u][k], y[u][k]);
    if (PREFETCH && base + nthreads * UNR < nvec) load(base + nthreads * UNR);
#pragma unroll
    for (int u = 0; u < UNR; ++u)
#pragma unroll
      for (int k = 0; k < 4; ++k) { double s, e; two_sum(hi, p[u][k], s, e); hi = s; lo += e; }
  }
  // crude block partial (probe only)
  for (int off = 16; off; off >>= 1) { hi += __shfl_xor_sync(~0u, hi, off); lo += __shfl_xor_sync(~0u, lo, off); }
  if ((threadIdx.x & 31) == 0) atomicAdd(part, hi + lo);
}

// Variant T: TMA bulk copies (cp.async.bulk.shared::cluster.global) into a
// STAGES-deep smem ring per CTA; one elected thread issues the copies for the
// 3 leaves of a tile and arms the stage's mbarrier with the byte count; all
// threads wait on the barrier, compute from smem and store with STG.256.
template <int STAGES, int TILE_BYTES, int BLOCK>
__global__ void __launch_bounds__(BLOCK) kT(double* d, const double* a, const double* b,
                                            const double* c, double al, double be, i64 ntiles) {
  extern __shared__ __align__(128) unsigned char smem[];
  constexpr int TE = TILE_BYTES / 8;  // doubles per leaf tile
  double* buf = (double*)smem;        // [STAGES][3][TE]
  uint64_t* bar = (uint64_t*)(smem + (size_t)STAGES * 3 * TILE_BYTES);
  const double* src[3] = {a, b, c};
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      uint32_t ba = (uint32_t)__cvta_generic_to_shared(&bar[s]);
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(ba));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](i64 tile, int s) {
    uint32_t ba = (uint32_t)__cvta_generic_to_shared(&bar[s]);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(ba), "r"(3 * TILE_BYTES) : "memory");
    for (int l = 0; l < 3; ++l) {
      uint32_t dst = (uint32_t)__cvta_generic_to_shared(buf + ((size_t)s * 3 + l) * TE);
      const double* g = src[l] + tile * TE;
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   :: "r"(dst), "l"(g), "r"(TILE_BYTES), "r"(ba) : "memory");
    }
  };
  const i64 first = blockIdx.x, stride = gridDim.x;
  const i64 mine = first < ntiles ? (ntiles - first + stride - 1) / stride : 0;
  if (threadIdx.x == 0)
    for (int s = 0; s < STAGES && s < mine; ++s) issue(first + s * stride, s);
  for (i64 k = 0; k < mine; ++k) {
    const int s = (int)(k % STAGES);
    const uint32_t phase = (uint32_t)((k / STAGES) & 1);
    uint32_t ba = (uint32_t)__cvta_generic_to_shared(&bar[s]);
    asm volatile("{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}"
                 :: "r"(ba), "r"(phase) : "memory");
    const i64 tile = first + k * stride;
    const double* x = buf + ((size_t)s * 3 + 0) * TE;
    const double* y = buf + ((size_t)s * 3 + 1) * TE;
    const double* z = buf + ((size_t)s * 3 + 2) * TE;
    for (int e = threadIdx.x * 4; e < TE; e += BLOCK * 4) {
      double r[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) r[q] = f(x[e + q], y[e + q], z[e + q], al, be);
      st4(d + tile * TE + e, r);
    }
    __syncthreads();  // everyone done reading stage s
    if (threadIdx.x == 0 && k + STAGES < mine) issue(first + (k + STAGES) * stride, s);
  }
}

int main() {
  const i64 n = i64(1) << 28;
  double *a, *b, *c, *d;
  CK(cudaMalloc(&a, n * 8)); CK(cudaMalloc(&b, n * 8)); CK(cudaMalloc(&c, n * 8)); CK(cudaMalloc(&d, n * 8));
  CK(cudaMemset(a, 0, n * 8)); CK(cudaMemset(b, 0, n * 8)); CK(cudaMemset(c, 0, n * 8));
  int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  const double bytes = 32.0 * n;
  auto run = [&](const char* name, auto launch) {
    for (int i = 0; i < 3; ++i) launch();
    CK(cudaDeviceSynchronize());
    std::vector<float> ts;
    for (int i = 0; i < 20; ++i) {
      CK(cudaEventRecord(e0)); launch(); CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
      float ms; CK(cudaEventElapsedTime(&ms, e0, e1)); ts.push_back(ms);
    }
    CK(cudaGetLastError());
    std::sort(ts.begin(), ts.end());
    printf("%-40s best %.4f ms  median %.4f ms  %.1f GB/s\n", name, ts[0], ts[ts.size() / 2], bytes / ts[0] / 1e6);
  };
  const i64 nvec = n / 4;
  auto occ = [&](const void* k, int block, size_t sm) { int o; CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, k, block, sm)); return o; };
#define RUN_A(U, B, M, H) { auto k = kA<U, B, M, H>; int o = occ((const void*)k, B, 0); int g = sms * o; \
    char nm[96]; snprintf(nm, 96, "A unr%d blk%d minb%d hint%d occ%d", U, B, M, H, o); \
    run(nm, [&] { k<<<g, B>>>(d, a, b, c, 1.25, -0.75, nvec); }); }
  RUN_A(2, 256, 1, 0); RUN_A(1, 256, 1, 0); RUN_A(4, 256, 1, 0); RUN_A(2, 256, 4, 0);
  RUN_A(2, 512, 1, 0); RUN_A(2, 128, 1, 0); RUN_A(2, 256, 1, 1); RUN_A(2, 256, 1, 2);
  RUN_A(1, 256, 8, 0); RUN_A(4, 128, 1, 0);
  { auto k = kB<4, 256>; int g = sms * occ((const void*)k, 256, 0);
    run("B 128-bit unr4 blk256", [&] { k<<<g, 256>>>(d, a, b, c, 1.25, -0.75, n / 2); }); }
  { auto k = kC<2, 256>; i64 g = (nvec + 511) / 512;
    run("C one-tile-per-CTA unr2 blk256", [&] { k<<<(unsigned)g, 256>>>(d, a, b, c, 1.25, -0.75, nvec); }); }
  { auto k = kC<1, 256>; i64 g = (nvec + 255) / 256;
    run("C one-tile-per-CTA unr1 blk256", [&] { k<<<(unsigned)g, 256>>>(d, a, b, c, 1.25, -0.75, nvec); }); }
  { auto k = kE<2, 256, 1>; i64 g = (nvec + 511) / 512;
    run("E one-tile unr2 L2::256B prefetch", [&] { k<<<(unsigned)g, 256>>>(d, a, b, c, 1.25, -0.75, nvec); }); }
  { auto k = kE<2, 256, 2>; i64 g = (nvec + 511) / 512;
    run("E one-tile unr2 ld.global.nc", [&] { k<<<(unsigned)g, 256>>>(d, a, b, c, 1.25, -0.75, nvec); }); }
  { auto k = kC<2, 512>; i64 g = (nvec + 1023) / 1024;
    run("C one-tile-per-CTA unr2 blk512", [&] { k<<<(unsigned)g, 512>>>(d, a, b, c, 1.25, -0.75, nvec); }); }
  { auto k = kC<4, 128>; i64 g = (nvec + 511) / 512;
    run("C one-tile-per-CTA unr4 blk128", [&] { k<<<(unsigned)g, 128>>>(d, a, b, c, 1.25, -0.75, nvec); }); }
  { auto k = kD<2, 256>; int o = occ((const void*)k, 256, 0); int g = sms * o; char nm[96];
    snprintf(nm, 96, "D persistent+prefetch unr2 occ%d", o);
    run(nm, [&] { k<<<g, 256>>>(d, a, b, c, 1.25, -0.75, nvec); }); }
  { auto k = kD<1, 256>; int o = occ((const void*)k, 256, 0); int g = sms * o; char nm[96];
    snprintf(nm, 96, "D persistent+prefetch unr1 occ%d", o);
    run(nm, [&] { k<<<g, 256>>>(d, a, b, c, 1.25, -0.75, nvec); }); }
  {
    double* part; CK(cudaMalloc(&part, 8));
    const double rb = 16.0 * n;
    auto runr = [&](const char* name, auto launch) {
      for (int i = 0; i < 3; ++i) launch();
      CK(cudaDeviceSynchronize());
      std::vector<float> ts;
      for (int i = 0; i < 20; ++i) {
        CK(cudaEventRecord(e0)); launch(); CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
        float ms; CK(cudaEventElapsedTime(&ms, e0, e1)); ts.push_back(ms);
      }
      std::sort(ts.begin(), ts.end());
      printf("%-40s best %.4f ms  median %.4f ms  %.1f GB/s\n", name, ts[0], ts[ts.size() / 2], rb / ts[0] / 1e6);
    };
#define RUN_R(U, P, M) { auto k = kR<U, 256, P>; int o = occ((const void*)k, 256, 0); \
      long long g = M == 0 ? (long long)sms * o : (nvec + 256 * U - 1) / (256 * U); char nm[96]; \
      snprintf(nm, 96, "R dot unr%d prefetch%d %s occ%d", U, (int)P, M == 0 ? "persistent" : "one-tile", o); \
      runr(nm, [&] { k<<<(unsigned)g, 256>>>(a, b, nvec, part); }); }
    RUN_R(2, false, 0); RUN_R(2, true, 0); RUN_R(4, false, 0); RUN_R(4, true, 0); RUN_R(1, false, 1); RUN_R(2, false, 1);
  }
#define RUN_T(ST, TB, B) { auto k = kT<ST, TB, B>; size_t sm = (size_t)ST * 3 * TB + 64; \
    CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm)); \
    int o = occ((const void*)k, B, sm); int g = sms * o; i64 nt = n * 8 / TB; \
    char nm[96]; snprintf(nm, 96, "TMA stages%d tile%dB blk%d occ%d", ST, TB, B, o); \
    run(nm, [&] { k<<<g, B, sm>>>(d, a, b, c, 1.25, -0.75, nt); }); }
  RUN_T(4, 8192, 256); RUN_T(3, 16384, 256); RUN_T(6, 8192, 256); RUN_T(2, 16384, 512); RUN_T(4, 4096, 128);
  // copy reference
  { run("cudaMemcpy D2D (2 x 2 GiB moved)", [&] { CK(cudaMemcpyAsync(d, a, n * 8, cudaMemcpyDeviceToDevice)); }); }
  return 0;
}
