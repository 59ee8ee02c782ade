// Probe: does programmatic dependent launch (PDL) shorten back-to-back
// launch-bound fused kernels on B200?  Not product code.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/pdl_probe tools/pdl_probe.cu
//
// Kernel: y = y + a*x (f64, one BLOCK*UNR tile of 256-bit vectors per CTA,
// like the product's assignment kernel), n = 2^12 .. 2^22, 400 launches
// back to back on one stream, eager and as a CUDA graph.
//   plain   ordinary launches
//   pdl     launch attribute programmaticStreamSerialization, kernel waits
//           (griddepcontrol.wait) before touching memory
//   pdl+tr  the same, and every CTA triggers its dependents
//           (griddepcontrol.launch_dependents) right after its loads
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1);} } while (0)
typedef long long i64;

template <int MODE>
__global__ void __launch_bounds__(256) axpy(double* y, const double* x, double a, i64 nvec) {
  if (MODE >= 1) asm volatile("griddepcontrol.wait;" ::: "memory");
  const i64 base = (i64)blockIdx.x * 512 + threadIdx.x;
  double xv[2][4], yv[2][4];
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const i64 j = base + u * 256;
    if (j < nvec) {
      asm volatile("ld.global.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];"
                   : "=d"(xv[u][0]), "=d"(xv[u][1]), "=d"(xv[u][2]), "=d"(xv[u][3]) : "l"(x + 4 * j));
      asm volatile("ld.global.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];"
                   : "=d"(yv[u][0]), "=d"(yv[u][1]), "=d"(yv[u][2]), "=d"(yv[u][3]) : "l"(y + 4 * j));
    }
  }
  if (MODE == 2) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const i64 j = base + u * 256;
    if (j < nvec) {
      double r[4];
      for (int k = 0; k < 4; ++k) r[k] = __dadd_rn(yv[u][k], __dmul_rn(a, xv[u][k]));
      asm volatile("st.global.L1::no_allocate.v4.f64 [%0], {%1,%2,%3,%4};"
                   :: "l"(y + 4 * j), "d"(r[0]), "d"(r[1]), "d"(r[2]), "d"(r[3]) : "memory");
    }
  }
}

template <int MODE> void launch(cudaStream_t st, double* y, const double* x, i64 nvec) {
  const int grid = (int)((nvec + 511) / 512);
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(256);
  cfg.stream = st;
  cfg.attrs = attr;
  cfg.numAttrs = MODE >= 1 ? 1 : 0;
  double a = 1e-9;
  CK(cudaLaunchKernelEx(&cfg, axpy<MODE>, y, x, a, nvec));
}

int main() {
  const i64 maxn = i64(1) << 22;
  double *x, *y;
  CK(cudaMalloc(&x, maxn * 8));
  CK(cudaMalloc(&y, maxn * 8));
  CK(cudaMemset(x, 0, maxn * 8));
  CK(cudaMemset(y, 0, maxn * 8));
  cudaStream_t st;
  CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  const int L = 400;
  const char* names[3] = {"plain", "pdl", "pdl+tr"};
  printf("# us per launch, %d back-to-back launches of y = y + a*x (f64), best of 5\n", L);
  for (int lg = 12; lg <= 22; lg += 2) {
    const i64 n = i64(1) << lg, nvec = n / 4;
    for (int graph = 0; graph < 2; ++graph) {
      printf("n=2^%-2d %-6s", lg, graph ? "graph" : "eager");
      for (int mode = 0; mode < 3; ++mode) {
        auto body = [&]() {
          for (int i = 0; i < L; ++i) {
            if (mode == 0) launch<0>(st, y, x, nvec);
            else if (mode == 1) launch<1>(st, y, x, nvec);
            else launch<2>(st, y, x, nvec);
          }
        };
        cudaGraphExec_t exec = nullptr;
        if (graph) {
          cudaGraph_t g;
          CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
          body();
          CK(cudaStreamEndCapture(st, &g));
          CK(cudaGraphInstantiate(&exec, g, 0));
          CK(cudaGraphDestroy(g));
        }
        float best = 1e30f;
        for (int r = 0; r < 6; ++r) {
          CK(cudaEventRecord(e0, st));
          if (graph) CK(cudaGraphLaunch(exec, st));
          else body();
          CK(cudaEventRecord(e1, st));
          CK(cudaEventSynchronize(e1));
          float ms;
          CK(cudaEventElapsedTime(&ms, e0, e1));
          if (r) best = ms < best ? ms : best;
        }
        if (exec) CK(cudaGraphExecDestroy(exec));
        printf("  %s %6.2f", names[mode], best * 1000.f / L);
      }
      printf("\n");
    }
  }
  return 0;
}
