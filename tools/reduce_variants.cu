// Design-space probe for the fused assign+reduce kernel (BASELINE config 5:
// y = y + alpha*x; r = dot(y, z), f64, n = 2^28) on B200.  Not product code.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//        -o tools/reduce_variants tools/reduce_variants.cu && tools/reduce_variants
//
// P: persistent grid-stride (SMs x occupancy CTAs), one partial per CTA,
//    last-CTA combine (the round-1 product scheme), UNR in {1, 2}.
// H: TPC tiles of UNR*BLOCK vectors per CTA (non-persistent), per-CTA partial,
//    hierarchical deterministic combine: the last CTA of each group of GS CTAs
//    folds the group, the last group folds the groups (2 ticket levels).
// S: semi-persistent: K tiles per CTA (grid = ceil(tiles / K)), same
//    hierarchical combine.
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdio>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1);} } while (0)
typedef long long i64;
struct DD { double hi, lo; };

__device__ __forceinline__ void ld4(double (&r)[4], const double* p) {
  asm volatile("ld.global.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];"
               : "=d"(r[0]), "=d"(r[1]), "=d"(r[2]), "=d"(r[3]) : "l"(p));
}
__device__ __forceinline__ void st4(double* p, const double (&r)[4]) {
  asm volatile("st.global.L1::no_allocate.v4.f64 [%0], {%1,%2,%3,%4};"
               :: "l"(p), "d"(r[0]), "d"(r[1]), "d"(r[2]), "d"(r[3]) : "memory");
}
__device__ __forceinline__ void two_sum(double a, double b, double& s, double& e) {
  s = __dadd_rn(a, b);
  double bp = __dsub_rn(s, a), ap = __dsub_rn(s, bp);
  e = __dadd_rn(__dsub_rn(a, ap), __dsub_rn(b, bp));
}
__device__ __forceinline__ DD dd_add(DD a, DD b) {
  double s, e;
  two_sum(a.hi, b.hi, s, e);
  e = __dadd_rn(e, __dadd_rn(a.lo, b.lo));
  DD r;
  two_sum(s, e, r.hi, r.lo);
  return r;
}
template <int BLOCK> __device__ DD block_dd(DD v, DD* sm) {
  for (int o = 16; o; o >>= 1) {
    DD w; w.hi = __shfl_xor_sync(~0u, v.hi, o); w.lo = __shfl_xor_sync(~0u, v.lo, o);
    v = dd_add(v, w);
  }
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    DD z{0, 0};
    v = threadIdx.x < BLOCK / 32 ? sm[threadIdx.x] : z;
    for (int o = 16; o; o >>= 1) {
      DD w; w.hi = __shfl_xor_sync(~0u, v.hi, o); w.lo = __shfl_xor_sync(~0u, v.lo, o);
      v = dd_add(v, w);
    }
  }
  return v;
}

// body over [t0, t1) tiles of BLOCK*UNR vectors, grid-stride by `stride` tiles
template <int UNR, int BLOCK>
__device__ void body(double* y, const double* x, const double* z, double al, i64 nvec,
                     i64 first_tile, i64 last_tile, i64 stride, double& hi, double& lo) {
  for (i64 t = first_tile; t < last_tile; t += stride) {
    const i64 base = t * BLOCK * UNR + threadIdx.x;
    double a[UNR][4], b[UNR][4], c[UNR][4];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      i64 j = base + (i64)u * BLOCK;
      if (j < nvec) { ld4(a[u], y + 4 * j); ld4(b[u], x + 4 * j); ld4(c[u], z + 4 * j); }
    }
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      i64 j = base + (i64)u * BLOCK;
      if (j < nvec) {
        double r[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          r[k] = __dadd_rn(a[u][k], __dmul_rn(al, b[u][k]));
          double p = __dmul_rn(r[k], c[u][k]), s, e;
          two_sum(hi, p, s, e);
          hi = s;
          lo = __dadd_rn(lo, e);
        }
        st4(y + 4 * j, r);
      }
    }
  }
}

// P: persistent, one ticket.
template <int UNR, int BLOCK>
__global__ void __launch_bounds__(BLOCK) kP(double* y, const double* x, const double* z, double al,
                                            i64 nvec, DD* parts, unsigned* ticket, double* out) {
  __shared__ DD sm[BLOCK / 32];
  __shared__ bool last;
  double hi = 0, lo = 0;
  const i64 ntiles = (nvec + BLOCK * UNR - 1) / (BLOCK * UNR);
  body<UNR, BLOCK>(y, x, z, al, nvec, blockIdx.x, ntiles, gridDim.x, hi, lo);
  DD v = block_dd<BLOCK>(DD{hi, lo}, sm);
  if (threadIdx.x == 0) {
    parts[blockIdx.x] = v;
    __threadfence();
    last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (last) {
    __threadfence();
    DD a{0, 0};
    for (int b = threadIdx.x; b < (int)gridDim.x; b += BLOCK) {
      DD p; p.hi = __ldcg(&parts[b].hi); p.lo = __ldcg(&parts[b].lo);
      a = dd_add(a, p);
    }
    __syncthreads();
    DD t = block_dd<BLOCK>(a, sm);
    if (threadIdx.x == 0) { *out = t.hi + t.lo; *ticket = 0; }
  }
}

// H / S: K tiles per CTA (contiguous), two-level deterministic tickets.
template <int UNR, int BLOCK, int K, int GS>
__global__ void __launch_bounds__(BLOCK) kH(double* y, const double* x, const double* z, double al,
                                            i64 nvec, DD* parts, DD* gparts, unsigned* gticket,
                                            unsigned* top, double* out) {
  __shared__ DD sm[BLOCK / 32];
  __shared__ int stage;  // 0: nothing, 1: group finisher, 2: group + final finisher
  double hi = 0, lo = 0;
  const i64 ntiles = (nvec + BLOCK * UNR - 1) / (BLOCK * UNR);
  const i64 t0 = (i64)blockIdx.x * K;
  const i64 t1 = t0 + K < ntiles ? t0 + K : ntiles;
  body<UNR, BLOCK>(y, x, z, al, nvec, t0, t1, 1, hi, lo);
  DD v = block_dd<BLOCK>(DD{hi, lo}, sm);
  const unsigned g = blockIdx.x / GS;
  const unsigned ngroups = (gridDim.x + GS - 1) / GS;
  const unsigned gsize = min((unsigned)GS, gridDim.x - g * GS);
  if (threadIdx.x == 0) {
    parts[blockIdx.x] = v;
    __threadfence();
    stage = atomicAdd(&gticket[g], 1u) == gsize - 1 ? 1 : 0;
  }
  __syncthreads();
  if (stage == 0) return;
  __threadfence();
  DD a{0, 0};
  if (threadIdx.x < gsize) { a.hi = __ldcg(&parts[g * GS + threadIdx.x].hi); a.lo = __ldcg(&parts[g * GS + threadIdx.x].lo); }
  __syncthreads();
  DD q = block_dd<BLOCK>(a, sm);
  if (threadIdx.x == 0) {
    gparts[g] = q;
    gticket[g] = 0;
    __threadfence();
    stage = atomicAdd(top, 1u) == ngroups - 1 ? 2 : 1;
  }
  __syncthreads();
  if (stage != 2) return;
  __threadfence();
  DD b{0, 0};
  for (unsigned i = threadIdx.x; i < ngroups; i += BLOCK) {
    DD p; p.hi = __ldcg(&gparts[i].hi); p.lo = __ldcg(&gparts[i].lo);
    b = dd_add(b, p);
  }
  __syncthreads();
  DD t = block_dd<BLOCK>(b, sm);
  if (threadIdx.x == 0) { *out = t.hi + t.lo; *top = 0; }
}

int main() {
  const i64 n = i64(1) << 28, nvec = n / 4;
  double *x, *y, *z, *out;
  CK(cudaMalloc(&x, n * 8)); CK(cudaMalloc(&y, n * 8)); CK(cudaMalloc(&z, n * 8)); CK(cudaMalloc(&out, 8));
  CK(cudaMemset(x, 0, n * 8)); CK(cudaMemset(y, 0, n * 8)); CK(cudaMemset(z, 0, n * 8));
  DD *parts, *gparts; unsigned *tick, *top;
  CK(cudaMalloc(&parts, (1 << 20) * sizeof(DD))); CK(cudaMalloc(&gparts, (1 << 14) * sizeof(DD)));
  CK(cudaMalloc(&tick, (1 << 14) * 4)); CK(cudaMalloc(&top, 4));
  CK(cudaMemset(tick, 0, (1 << 14) * 4)); CK(cudaMemset(top, 0, 4));
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
    printf("%-44s best %.4f ms  median %.4f ms  %.1f GB/s\n", name, ts[0], ts[ts.size() / 2], bytes / ts[0] / 1e6);
  };
  auto occ = [&](const void* k) { int o; CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, k, 256, 0)); return o; };
#define RUN_P(U) { auto k = kP<U, 256>; int o = occ((const void*)k); int g = sms * o; char nm[96]; \
    snprintf(nm, 96, "P persistent unr%d occ%d grid%d", U, o, g); \
    run(nm, [&] { k<<<g, 256>>>(y, x, z, 0.5, nvec, parts, tick, out); }); }
  RUN_P(1); RUN_P(2);
#define RUN_H(U, K, GS) { auto k = kH<U, 256, K, GS>; i64 tiles = (nvec + 256 * U - 1) / (256 * U); \
    i64 g = (tiles + K - 1) / K; int o = occ((const void*)k); char nm[96]; \
    snprintf(nm, 96, "H unr%d tiles/CTA %d group%d grid%lld occ%d", U, K, GS, g, o); \
    run(nm, [&] { k<<<(unsigned)g, 256>>>(y, x, z, 0.5, nvec, parts, gparts, tick, top, out); }); }
  RUN_H(2, 1, 256); RUN_H(1, 1, 256); RUN_H(2, 2, 256); RUN_H(2, 4, 256); RUN_H(2, 8, 128);
  RUN_H(1, 4, 256); RUN_H(2, 16, 64); RUN_H(1, 16, 64);
  return 0;
}
