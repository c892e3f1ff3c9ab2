// Microbenchmark of the tcgen05 issue loop's building blocks (one CTA, one
// issuing thread, clock64 per iteration): how many SM cycles do
//   (1) 4 x tcgen05.mma (128x256x16) + commit,  (2) 4 x mma without commit,
//   (3) commit alone, (4) mbarrier wait on an already-completed phase + fence
// cost per iteration?  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3
// tools/umma_probe.cu -o umma_probe
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t su32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint64_t desc(uint32_t saddr) {
  uint64_t d = (saddr >> 4) & 0x3FFF;
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)64 << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

__global__ void probe(int mode, int iters, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&bar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&slot)), "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((256u >> 3) << 17) | ((128u >> 4) << 24);
    const uint32_t sa = su32(sm), sb = sa + 16384;
    // complete phase 0 once so parity-1 waits return immediately
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&bar)) : "memory");
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      if (mode == 0 || mode == 1) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n"
                       ::"r"(tmem), "l"(desc(sa + 32 * k)), "l"(desc(sb + 32 * k)), "r"(idesc), "r"(1));
        }
      }
      if (mode == 0 || mode == 2)
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
      if (mode == 3) {
        asm volatile("{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W;\n}\n" ::"r"(su32(&bar)), "r"(0) : "memory");
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      }
      if (mode == 4 || mode == 5) {
        // round trip: (4 MMAs +) commit, then wait for the commit's arrival
        if (mode == 4) {
#pragma unroll
          for (int k = 0; k < 4; ++k)
            asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n"
                         ::"r"(tmem), "l"(desc(sa + 32 * k)), "l"(desc(sb + 32 * k)), "r"(idesc), "r"(1));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
        const uint32_t par = (i + 1) & 1;  // phase 0 was completed before the loop
        asm volatile("{\n.reg .pred P1;\nW2:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W2;\n}\n" ::"r"(su32(&bar)), "r"(par) : "memory");
      }
    }
    long long t1 = clock64();
    out[mode] = (t1 - t0) / iters;
  }
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
}

int main() {
  long long* d;
  cudaMalloc(&d, 8 * sizeof(long long));
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  const char* names[] = {"4 mma + commit", "4 mma only", "commit only", "wait(done)+fence",
                         "4mma+commit+wait rt", "commit+wait rt"};
  for (int mode = 0; mode < 6; ++mode) {
    probe<<<1, 128, 64 * 1024>>>(mode, 4000, d);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[8];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("%-20s %6lld cycles/iter  (%s)\n", names[mode], h[mode], cudaGetErrorString(e));
  }
  return 0;
}
