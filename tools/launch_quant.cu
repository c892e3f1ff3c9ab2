// Kernel-boundary granularity probe: back-to-back launches of a kernel that
// spins for D ns (per CTA, %globaltimer), with and without a TMEM
// allocation, 148 CTAs; prints the mean launch-to-launch time per D.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/bin/launch_quant tools/launch_quant.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
template <bool TMEM>
__global__ void spin(long long ns) {
  __shared__ unsigned slot;
  if (TMEM && threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(
        (unsigned)__cvta_generic_to_shared(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  __syncthreads();
  const unsigned long long t0 = gtime();
  while ((long long)(gtime() - t0) < ns) {
  }
  __syncthreads();
  if (TMEM && threadIdx.x < 32)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(slot));
}
__global__ void sleep_kernel(long long ns) {
  const unsigned long long t0 = gtime();
  while ((long long)(gtime() - t0) < ns) {
  }
}

int main() {
  cudaStream_t s;
  cudaStreamCreate(&s);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int n = 300;
  printf("D_ns  plain_us  tmem_us\n");
  for (long long d = 0; d <= 6000; d += 250) {
    float r[2];
    for (int k = 0; k < 2; ++k) {
      sleep_kernel<<<1, 1, 0, s>>>(200000000);  // keep the queue full
      for (int w = 0; w < 10; ++w) {
        if (k) spin<true><<<148, 128, 0, s>>>(d); else spin<false><<<148, 128, 0, s>>>(d);
      }
      cudaEventRecord(a, s);
      for (int i = 0; i < n; ++i) {
        if (k) spin<true><<<148, 128, 0, s>>>(d); else spin<false><<<148, 128, 0, s>>>(d);
      }
      cudaEventRecord(b, s);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      r[k] = ms * 1e3f / n;
    }
    printf("%5lld  %7.3f  %7.3f\n", d, r[0], r[1]);
  }
  // the same in a CUDA graph (the engine's execution mode)
  for (long long d : {0LL, 1000LL, 2500LL, 4000LL}) {
    cudaGraph_t g;
    cudaGraphExec_t ge;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
    for (int i = 0; i < n; ++i) spin<false><<<148, 128, 0, s>>>(d);
    cudaStreamEndCapture(s, &g);
    cudaGraphInstantiate(&ge, g, 0);
    cudaGraphLaunch(ge, s);
    cudaStreamSynchronize(s);
    cudaEventRecord(a, s);
    cudaGraphLaunch(ge, s);
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("graph D=%lld  %7.3f us/kernel\n", d, ms * 1e3f / n);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
