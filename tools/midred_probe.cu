// Design-space probe for MID-SIZE pure reductions (BASELINE config 3 at
// n = 2^24: ddot/dnrm2, f32/f64; 2^22..2^26 around the 126 MB L2) on B200.
// Not product code.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -fmad=false \
//        -o tools/midred_probe tools/midred_probe.cu && tools/midred_probe
//
// Every variant computes the same compensated double-double sum as the
// product (TwoSum per f64 term / exact f64 sum of f32 terms) and is checked
// against variant "cur".  Timing: CUDA events around one launch, preceded
// by an L2 sweep — "clean" (a 512 MiB read sweep: L2 full of clean lines) or
// "dirty" (a 512 MiB memset: L2 full of dirty lines, config_sweep's flush).
//
// Variants (K = tiles of BLOCK*UNR vectors per CTA, GS = CTAs per group):
//   floor   K=1, per-CTA partial only, no combine (bandwidth floor)
//   cur     the product geometry: <= 16*256 tiles -> one group of <= 256
//           CTAs with K = ceil(tiles/256), else K = 2 (dot) / 4 (nrm2),
//           groups of 256, two ticket levels
//   pipe    cur + software pipeline: the next tile's loads are issued
//           before the current tile is accumulated
//   wideK   K fixed (1, 2, 4), one group of the whole grid (last CTA folds
//           every partial, strided) up to 4096 CTAs, else groups of 1024
#include <cuda_runtime.h>
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1);} } while (0)
typedef long long i64;
struct DD { double hi, lo; };
constexpr int BLOCK = 256;

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
__device__ DD block_dd(DD v, DD* sm) {
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
__device__ __forceinline__ unsigned ticket_add(unsigned* p) {
  unsigned old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(p) : "memory");
  return old;
}

template <class T> struct Vec;
template <> struct Vec<double> {
  double v[4];
  __device__ __forceinline__ void load(const double* p) {
    asm volatile("ld.global.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];"
                 : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3]) : "l"(p));
  }
  static constexpr int W = 4;
};
template <> struct Vec<float> {
  float v[8];
  __device__ __forceinline__ void load(const float* p) {
    asm volatile("ld.global.L1::no_allocate.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7])
                 : "l"(p));
  }
  static constexpr int W = 8;
};
template <class T> struct Acc;
template <> struct Acc<double> {
  double hi = 0, lo = 0;
  __device__ __forceinline__ void add(double x) { double s, e; two_sum(hi, x, s, e); hi = s; lo = __dadd_rn(lo, e); }
  __device__ __forceinline__ DD get() const { DD r; two_sum(hi, lo, r.hi, r.lo); return r; }
};
template <> struct Acc<float> {
  double hi = 0;
  __device__ __forceinline__ void add(float x) { hi = __dadd_rn(hi, (double)x); }
  __device__ __forceinline__ DD get() const { return DD{hi, 0.0}; }
};
template <class T> __device__ __forceinline__ T mul_rn(T a, T b);
template <> __device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
template <> __device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }

struct Args {
  const void* x; const void* y;  // y == x for nrm2 (one leaf)
  i64 nvec;                      // vectors of 32 bytes
  i64 K;                         // tiles per CTA
  int GS;                        // CTAs per group
  int combine;                   // 0: partials only
  DD* partials; DD* gpart; unsigned* gticket; unsigned* ticket; DD* out;
};

template <class T, int NL, int UNR>
__device__ __forceinline__ void consume(Acc<T>& acc, const Vec<T> (&a)[UNR], const Vec<T> (&b)[UNR], i64 base, i64 nvec) {
#pragma unroll
  for (int u = 0; u < UNR; ++u)
    if (base + (i64)u * BLOCK < nvec) {
#pragma unroll
      for (int k = 0; k < Vec<T>::W; ++k) acc.add(mul_rn(a[u].v[k], NL == 1 ? a[u].v[k] : b[u].v[k]));
    }
}
template <class T, int NL, int UNR>
__device__ __forceinline__ void issue(Vec<T> (&a)[UNR], Vec<T> (&b)[UNR], const T* x, const T* y, i64 base, i64 nvec) {
#pragma unroll
  for (int u = 0; u < UNR; ++u) {
    const i64 j = base + (i64)u * BLOCK;
    if (j < nvec) {
      a[u].load(x + j * Vec<T>::W);
      if (NL == 2) b[u].load(y + j * Vec<T>::W);
    }
  }
}

template <class T, int NL, int UNR, bool PIPE>
__global__ void __launch_bounds__(BLOCK) red_kernel(Args a) {
  const T* x = (const T*)a.x;
  const T* y = (const T*)a.y;
  Acc<T> acc;
  const i64 per = (i64)BLOCK * UNR;
  const i64 ntiles = (a.nvec + per - 1) / per;
  const i64 t0 = (i64)blockIdx.x * a.K;
  const i64 t1 = min(t0 + a.K, ntiles);
  if (!PIPE) {
    for (i64 t = t0; t < t1; ++t) {
      Vec<T> va[UNR], vb[UNR];
      const i64 base = t * per + threadIdx.x;
      issue<T, NL, UNR>(va, vb, x, y, base, a.nvec);
      consume<T, NL, UNR>(acc, va, vb, base, a.nvec);
    }
  } else if (t0 < t1) {
    Vec<T> va[UNR], vb[UNR], na[UNR], nb[UNR];
    i64 base = t0 * per + threadIdx.x;
    issue<T, NL, UNR>(va, vb, x, y, base, a.nvec);
    for (i64 t = t0; t < t1; ++t) {
      const i64 nbase = base + per;
      if (t + 1 < t1) issue<T, NL, UNR>(na, nb, x, y, nbase, a.nvec);
      consume<T, NL, UNR>(acc, va, vb, base, a.nvec);
#pragma unroll
      for (int u = 0; u < UNR; ++u) { va[u] = na[u]; vb[u] = nb[u]; }
      base = nbase;
    }
  }
  __shared__ DD sm[BLOCK / 32];
  __shared__ int stage;
  DD part = block_dd(acc.get(), sm);
  if (!a.combine) {
    if (threadIdx.x == 0) a.partials[blockIdx.x] = part;
    return;
  }
  const unsigned GS = a.GS;
  const unsigned g = blockIdx.x / GS, ng = (gridDim.x + GS - 1) / GS;
  const unsigned gsize = min(GS, gridDim.x - g * GS);
  if (threadIdx.x == 0) {
    a.partials[blockIdx.x] = part;
    stage = ticket_add(&a.gticket[g]) == gsize - 1;
  }
  __syncthreads();
  if (!stage) return;
  DD v{0, 0};
  {  // up to 4 partials per thread: issue the loads, then fold in CTA order
    DD p[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const unsigned b = threadIdx.x + i * BLOCK;
      if (b < gsize) { p[i].hi = __ldcg(&a.partials[g * GS + b].hi); p[i].lo = __ldcg(&a.partials[g * GS + b].lo); }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if (threadIdx.x + i * BLOCK < gsize) v = dd_add(v, p[i]);
    for (unsigned b = threadIdx.x + 4 * BLOCK; b < gsize; b += BLOCK) {
      DD q; q.hi = __ldcg(&a.partials[g * GS + b].hi); q.lo = __ldcg(&a.partials[g * GS + b].lo);
      v = dd_add(v, q);
    }
  }
  __syncthreads();
  DD q = block_dd(v, sm);
  if (ng == 1) {
    if (threadIdx.x == 0) { a.gticket[g] = 0; *a.out = q; }
    return;
  }
  if (threadIdx.x == 0) {
    a.gpart[g] = q;
    a.gticket[g] = 0;
    stage = ticket_add(a.ticket) == ng - 1 ? 2 : 0;
  }
  __syncthreads();
  if (stage != 2) return;
  DD w{0, 0};
  for (unsigned b = threadIdx.x; b < ng; b += BLOCK) {
    DD p; p.hi = __ldcg(&a.gpart[b].hi); p.lo = __ldcg(&a.gpart[b].lo);
    w = dd_add(w, p);
  }
  __syncthreads();
  DD tot = block_dd(w, sm);
  if (threadIdx.x == 0) { *a.ticket = 0; *a.out = tot; }
}

__global__ void sweep_read(const double4* p, i64 n, double* sink) {
  double s = 0;
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) {
    double4 v = p[i];
    s += v.x + v.w;
  }
  if (s == 12345.678) *sink = s;
}

struct Variant { std::string name; int unr; bool pipe; int K; int GS; int combine; };

template <class T, int NL, int UNR, bool PIPE> void launch(int grid, const Args& a) {
  red_kernel<T, NL, UNR, PIPE><<<grid, BLOCK>>>(a);
}
template <class T, int NL> void dispatch(int unr, bool pipe, int grid, const Args& a) {
  if (unr == 2) pipe ? launch<T, NL, 2, true>(grid, a) : launch<T, NL, 2, false>(grid, a);
  else if (unr == 4) pipe ? launch<T, NL, 4, true>(grid, a) : launch<T, NL, 4, false>(grid, a);
  else pipe ? launch<T, NL, 8, true>(grid, a) : launch<T, NL, 8, false>(grid, a);
}

int main(int argc, char** argv) {
  int reps = argc > 1 ? atoi(argv[1]) : 15;
  const i64 maxn = i64(1) << 27;
  void *x, *y;
  CK(cudaMalloc(&x, maxn * 8));
  CK(cudaMalloc(&y, maxn * 8));
  {  // fill with 0.5-ish values (no NaN/inf); exact values do not matter for timing
    std::vector<double> h(maxn);
    for (i64 i = 0; i < maxn; ++i) h[i] = std::ldexp((double)((i * 2654435761ull) % 1000003) - 500001.0, -20);
    CK(cudaMemcpy(x, h.data(), maxn * 8, cudaMemcpyHostToDevice));
    for (i64 i = 0; i < maxn; ++i) h[i] = std::ldexp((double)((i * 40503ull) % 999983) - 499991.0, -20);
    CK(cudaMemcpy(y, h.data(), maxn * 8, cudaMemcpyHostToDevice));
  }
  const i64 sweep_bytes = i64(512) << 20;
  void* sw; double* sink;
  CK(cudaMalloc(&sw, sweep_bytes));
  CK(cudaMemset(sw, 1, sweep_bytes));
  CK(cudaMalloc(&sink, 8));
  DD *parts, *gpart, *out;
  unsigned *gt, *tk;
  CK(cudaMalloc(&parts, 16 << 20));
  CK(cudaMalloc(&gpart, 16 << 16));
  CK(cudaMalloc(&gt, 4 << 16));
  CK(cudaMalloc(&tk, 256));
  CK(cudaMemset(gt, 0, 4 << 16));
  CK(cudaMemset(tk, 0, 256));
  CK(cudaMalloc(&out, 16));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  printf("# midred_probe: %d SMs, reps %d; us per launch (median / best) after an L2 sweep\n", sms, reps);

  const char* ops[4] = {"nrm2_f64", "dot_f64", "nrm2_f32", "dot_f32"};
  for (int op = 0; op < 4; ++op) {
    const bool f64 = op < 2;
    const int NL = (op & 1) ? 2 : 1;
    const int es = f64 ? 8 : 4;
    const char* set = getenv("PROBE_SET");
    const bool rules = set && !strcmp(set, "rules");
    for (int lg = rules ? 20 : 22; lg <= (rules ? 27 : 26); ++lg) {
      const i64 n = i64(1) << lg;
      const i64 nvec = n * es / 32;
      const double bytes = (double)n * es * NL;
      std::vector<Variant> vs;
      const int ucur = (!f64 || NL == 1) ? 4 : 2;
      vs.push_back({"floor", ucur, false, 1, 1 << 30, 0});
      vs.push_back({"cur", ucur, false, -1, 256, 1});
      if (rules) {
        vs.push_back({"new_nl", ucur, false, -2, 0, 1});
        vs.push_back({"new_512", ucur, false, -3, 0, 1});
        vs.push_back({"new_nl16", ucur, false, -4, 0, 1});
      } else
      vs.push_back({"pipe", ucur, true, -1, 256, 1});
      if (!rules)
      for (int K : {1, 2, 4, 8, 16})
        for (int u : {2, 4})
          vs.push_back({"wide_U" + std::to_string(u) + "_K" + std::to_string(K), u, false, K, -4096, 1});
      double ref = NAN;
      for (const Variant& v : vs) {
        const i64 per = (i64)BLOCK * v.unr;
        const i64 ntiles = (nvec + per - 1) / per;
        i64 K = v.K;
        int GS = v.GS;
        if (K == -1) {  // the product geometry
          if (ntiles <= 16 * 256) K = (ntiles + 255) / 256;
          else K = NL == 1 ? 4 : 2;
        } else if (K < -1) {  // candidate: one group of <= cap CTAs up to 32 tiles per CTA
          const i64 cap = K == -3 ? 512 : (NL == 1 ? 512 : 256);
          if (ntiles <= (K == -4 ? 16 : 32) * cap) { K = (ntiles + cap - 1) / cap; GS = 4096; }
          else { K = NL == 1 ? 4 : 2; GS = 256; }
        }
        const i64 grid = (ntiles + K - 1) / K;
        if (GS < 0) GS = grid <= -GS ? (int)grid : 1024;
        if (grid > (1 << 20)) continue;
        Args a{x, NL == 2 ? y : x, nvec, K, GS, v.combine, parts, gpart, gt, tk, out};
        auto sweep = [&](int mode, int r) {
          if (mode == 0) sweep_read<<<sms * 8, 256>>>((const double4*)sw, sweep_bytes / 32, sink);
          else CK(cudaMemsetAsync(sw, r & 0xff, sweep_bytes));
        };
        auto kern = [&]() {
          if (f64) (NL == 1 ? dispatch<double, 1>(v.unr, v.pipe, grid, a) : dispatch<double, 2>(v.unr, v.pipe, grid, a));
          else (NL == 1 ? dispatch<float, 1>(v.unr, v.pipe, grid, a) : dispatch<float, 2>(v.unr, v.pipe, grid, a));
        };
        for (int mode = 0; mode < 2; ++mode) {
          // differential: R x (sweep + kernel) minus R x sweep, 3 trials, min
          // (the event clock ticks in ~2 us steps on this box)
          double best = 1e30;
          for (int trial = 0; trial < 3; ++trial) {
            float ms_pair, ms_sweep;
            sweep(mode, 0); kern();
            CK(cudaEventRecord(e0));
            for (int r = 0; r < reps; ++r) { sweep(mode, r); kern(); }
            CK(cudaEventRecord(e1));
            CK(cudaEventSynchronize(e1));
            CK(cudaEventElapsedTime(&ms_pair, e0, e1));
            CK(cudaEventRecord(e0));
            for (int r = 0; r < reps; ++r) sweep(mode, r);
            CK(cudaEventRecord(e1));
            CK(cudaEventSynchronize(e1));
            CK(cudaEventElapsedTime(&ms_sweep, e0, e1));
            best = std::min(best, (double)(ms_pair - ms_sweep) * 1000.0 / reps);
          }
          CK(cudaGetLastError());
          if (v.combine && mode == 0) {
            DD h;
            CK(cudaMemcpy(&h, out, 16, cudaMemcpyDeviceToHost));
            if (std::isnan(ref)) ref = h.hi;
            else if (std::fabs(h.hi - ref) > 1e-12 * std::fabs(ref)) printf("MISMATCH %s %.17g vs %.17g\n", v.name.c_str(), h.hi, ref);
          }
          printf("%-9s 2^%d %-5s %-14s grid %7lld K %2lld GS %5d: %8.2f us  %6.0f GB/s\n", ops[op], lg,
                 mode ? "dirty" : "clean", v.name.c_str(), (long long)grid, (long long)K, GS, best, bytes / best / 1e3);
        }
      }
    }
  }
  return 0;
}
