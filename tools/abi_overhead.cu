// Host cost of one C-ABI call, without Python: back-to-back salt_assign /
// salt_reduce calls on n = 1024 (launch-bound), against a bare
// cudaLaunchKernel of an empty kernel and of an empty kernel taking a
// parameter block the size of salt::Args<double>.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/abi_overhead tools/abi_overhead.cu \
//        -Iinclude -Lpaper_1109_1264_b200 -lsalt -Xlinker -rpath,'$ORIGIN/../paper_1109_1264_b200'
//   ./tools/abi_overhead
#include <chrono>
#include <cstdio>
#include <cuda_runtime.h>

#include "salt.h"

struct Big {
  char bytes[720];
};
__global__ void empty_kernel() {}
__global__ void big_kernel(Big b) {
  if (b.bytes[0] == 42 && threadIdx.x == 1023) printf("x");
}

template <class F> double per_call_us(F f, int calls) {
  for (int i = 0; i < 200; ++i) f();
  cudaDeviceSynchronize();
  auto t0 = std::chrono::steady_clock::now();
  for (int i = 0; i < calls; ++i) f();
  auto t1 = std::chrono::steady_clock::now();
  cudaDeviceSynchronize();
  return std::chrono::duration<double, std::micro>(t1 - t0).count() / calls;
}

int main() {
  const int n = 1024, calls = 20000;
  double *a, *b, *c, *d, *out;
  cudaMalloc(&a, n * 8);
  cudaMalloc(&b, n * 8);
  cudaMalloc(&c, n * 8);
  cudaMalloc(&d, n * 8);
  cudaMalloc(&out, 256);
  cudaMemset(a, 0, n * 8);
  cudaMemset(b, 0, n * 8);
  cudaMemset(c, 0, n * 8);
  size_t wsb = salt_reduce_workspace_bytes();
  void* ws;
  cudaMalloc(&ws, wsb);
  cudaMemset(ws, 0, wsb);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  const void* leaves[3] = {a, b, c};
  const double sc[2] = {1.25, -0.5};
  Big big = {};
  printf("{\n");
  printf(" \"empty cudaLaunchKernel\": %.3f,\n",
         per_call_us([&] { empty_kernel<<<1, 256, 0, s>>>(); }, calls));
  printf(" \"empty kernel with a 720-byte parameter block\": %.3f,\n",
         per_call_us([&] { big_kernel<<<1, 256, 0, s>>>(big); }, calls));
  {
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.gridDim = dim3(1);
    cfg.blockDim = dim3(256);
    cfg.stream = s;
    cfg.attrs = attr;
    void* params[] = {&big};
    cfg.numAttrs = 0;
    printf(" \"720-byte kernel via cudaLaunchKernelExC, no attribute\": %.3f,\n",
           per_call_us([&] { cudaLaunchKernelExC(&cfg, (const void*)big_kernel, params); }, calls));
    cfg.numAttrs = 1;
    printf(" \"720-byte kernel via cudaLaunchKernelExC, PDL attribute\": %.3f,\n",
           per_call_us([&] { cudaLaunchKernelExC(&cfg, (const void*)big_kernel, params); }, calls));
  }
  printf(" \"salt_assign T2 n=1024\": %.3f,\n",
         per_call_us([&] { salt_assign(SALT_F64, "S0 L0 * S1 L1 L2 - * +", d, leaves, 3, sc, 2, n, s); },
                     calls));
  printf(" \"salt_assign axpy n=1024\": %.3f,\n",
         per_call_us([&] { salt_assign(SALT_F64, "L0 S0 L1 * +", b, leaves, 2, sc, 1, n, s); }, calls));
  printf(" \"salt_reduce dot n=1024 (device result)\": %.3f,\n",
         per_call_us([&] { salt_reduce(SALT_F64, "L0 L1 *", leaves, 2, nullptr, 0, n, 0, ws, wsb, out,
                                       nullptr, s); }, calls));
  printf(" \"unit\": \"us of host time per call (20000 back-to-back calls, no synchronisation)\"\n}\n");
  return 0;
}
