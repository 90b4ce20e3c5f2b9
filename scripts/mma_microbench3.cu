// Microbenchmark 3: cost of tcgen05.commit / mbarrier waits between small MMA groups
// (the emulated GEMM issues 4 MMAs per pipeline stage, then commits).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {
  uint64_t d = (uint64_t)((saddr & 0x3FFFFu) >> 4);
  d |= (uint64_t)1 << 16; d |= (uint64_t)(1024 >> 4) << 32; d |= (uint64_t)1 << 46; d |= (uint64_t)2 << 61;
  return d;
}
// mode 0: 4 MMAs + commit (no wait) per group; mode 1: + try_wait(completed barrier) + fence per group
// mode 2: 8 MMAs + commit per group; mode 3: 16 MMAs + commit per group
__global__ void __launch_bounds__(128, 1) mb(int groups, int mode, long long* cycles) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar[4];
  __shared__ uint32_t tslot;
  uint8_t* A = sm; uint8_t* B = sm + 16384;
  for (int i = threadIdx.x; i < 32768 / 4; i += blockDim.x) ((uint32_t*)sm)[i] = 0x01010101u;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;");
    // complete phase 0 of bar[2] so waits on parity 0 succeed immediately
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&bar[2])));
  }
  if (warp == 0) { asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot))); asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;"); }
  asm volatile("fence.proxy.async.shared::cta;"); asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads(); asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tslot;
  const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(128 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  if (threadIdx.x == 0) {
    const int per = mode == 2 ? 8 : (mode == 3 ? 16 : 4);
    long long t0 = clock64();
    for (int g = 0; g < groups; ++g) {
      if (mode == 1) {
        asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W_%=;\n}" ::"r"(smem_u32(&bar[2])));
        asm volatile("tcgen05.fence::after_thread_sync;");
      }
      for (int i = 0; i < per; ++i)
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}"
                     ::"r"(tmem + (uint32_t)((g & 3) * 128)), "l"(sdesc(smem_u32(A) + (i & 3) * 32)), "l"(sdesc(smem_u32(B) + (i & 3) * 32)), "r"(idesc), "r"(1u));
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar[g & 1])));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar[3])));
    asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W_%=;\n}" ::"r"(smem_u32(&bar[3])));
    cycles[blockIdx.x] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  long long* d; cudaMalloc(&d, sizeof(long long) * sms); long long h[256];
  cudaFuncSetAttribute(mb, cudaFuncAttributeMaxDynamicSharedMemorySize, 40 * 1024);
  for (int mode = 0; mode < 4; ++mode) {
    const int per = mode == 2 ? 8 : (mode == 3 ? 16 : 4);
    const int groups = 64000 / per;
    mb<<<sms, 128, 40 * 1024>>>(groups, mode, d);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
    double avg = 0; for (int i = 0; i < sms; ++i) avg += h[i]; avg /= sms;
    printf("mode %d (%d mma/commit%s): %s %.0f MAC/clk/SM\n", mode, per, mode == 1 ? " + wait+fence" : "",
           cudaGetErrorString(e), (double)groups * per * 128 * 128 * 32 / avg);
  }
  return 0;
}
