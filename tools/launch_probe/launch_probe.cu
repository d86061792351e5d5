// Launch-overhead probe (developer tool): event-timed launches of an empty
// persistent-shaped kernel, varying the kernel-parameter size, dynamic shared
// memory and an interleaved L2-flush kernel.  nvcc -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cuda_runtime.h>

template <int BYTES>
struct Blob { char b[BYTES]; };

template <int BYTES>
__global__ void __launch_bounds__(1024, 1) k_empty(const __grid_constant__ Blob<BYTES> a, int* out) {
  extern __shared__ char s[];
  if (threadIdx.x == 0 && a.b[blockIdx.x % BYTES] == 7) out[blockIdx.x] = s[0];
}

__global__ void k_flush(double4* buf, size_t n) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    buf[i] = make_double4(1, 2, 3, 4);
}

template <int BYTES>
void run(const char* name, int smem, bool flush, double4* fb, size_t fn, int* out, int block = 544) {
  Blob<BYTES> a = {};
  auto fn_ = k_empty<BYTES>;
  cudaFuncSetAttribute(fn_, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(fn_, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  float tot = 0;
  const int iters = 200;
  for (int i = 0; i < iters + 10; ++i) {
    if (flush) k_flush<<<1184, 512, 0>>>(fb, fn);
    cudaEventRecord(e0);
    fn_<<<148, block, smem>>>(a, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    if (i >= 10) tot += ms;
  }
  printf("%-28s params %5d B  smem %6d  block %4d flush %d : %.2f us/launch\n", name, BYTES, smem, block, (int)flush, 1e3 * tot / iters);
}

int main() {
  size_t fn = (512u << 20) / sizeof(double4);
  double4* fb; cudaMalloc(&fb, fn * sizeof(double4));
  int* out; cudaMalloc(&out, 4096);
  cudaFuncSetAttribute(k_flush, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  for (int f = 0; f < 2; ++f) {
    run<64>("small params", 0, f, fb, fn, out);
    run<64>("small params + smem", 113 * 1024, f, fb, fn, out);
    run<5632>("5.6KB params", 0, f, fb, fn, out);
    run<5632>("5.6KB params + smem", 113 * 1024, f, fb, fn, out);
    run<3584>("3.5KB params + 200KB smem", 200 * 1024, f, fb, fn, out, 544);
    run<3584>("3.5KB, 200KB, 288 thr", 200 * 1024, f, fb, fn, out, 288);
    run<3584>("3.5KB, 200KB, 128 thr", 200 * 1024, f, fb, fn, out, 128);
    run<3584>("3.5KB, 100KB, 544 thr", 100 * 1024, f, fb, fn, out, 544);
    run<512>("0.5KB, 200KB, 544 thr", 200 * 1024, f, fb, fn, out, 544);
  }
  return 0;
}
