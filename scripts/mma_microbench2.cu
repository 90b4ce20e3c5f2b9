// Microbenchmark 2: (a) 1-CTA int8 MMA with concurrent st.shared traffic
// (is the SMEM port shared with the tensor-core operand reads?) and
// (b) cta_group::2 (CTA pair) M=256 MMAs.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {
  uint64_t d = (uint64_t)((saddr & 0x3FFFFu) >> 4);
  d |= (uint64_t)1 << 16; d |= (uint64_t)(1024 >> 4) << 32; d |= (uint64_t)1 << 46; d |= (uint64_t)2 << 61;
  return d;
}
__device__ __forceinline__ uint32_t cluster_rank() { uint32_t r; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r)); return r; }
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// (a) st.shared stress: warps 1..3 store 16B/lane continuously while warp 0 issues MMAs
__global__ void __launch_bounds__(128, 1) mma_with_stores(int groups, int stress, long long* cycles, int* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  __shared__ volatile int stop;
  uint8_t* A = sm; uint8_t* B = sm + 16384; uint8_t* S = sm + 32768;  // S: 64 KB store target
  for (int i = threadIdx.x; i < 32768 / 4; i += blockDim.x) ((uint32_t*)sm)[i] = 0x01010101u;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) { stop = 0; asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar))); asm volatile("fence.mbarrier_init.release.cluster;"); }
  if (warp == 0) { asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot))); asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;"); }
  asm volatile("fence.proxy.async.shared::cta;"); asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads(); asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tslot;
  const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(128 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  if (warp == 0) {
    if (lane == 0) {
      uint32_t phase = 0;
      long long t0 = clock64();
      for (int g = 0; g < groups; ++g) {
        for (int i = 0; i < 64; ++i)
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}"
                       ::"r"(tmem), "l"(sdesc(smem_u32(A) + (i & 3) * 32)), "l"(sdesc(smem_u32(B) + (i & 3) * 32)), "r"(idesc), "r"(1u));
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
        asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}" ::"r"(smem_u32(&bar)), "r"(phase));
        phase ^= 1;
      }
      cycles[blockIdx.x * 2] = clock64() - t0;
      stop = 1;
    }
  } else if (stress) {
    long long t0 = clock64(); long long n = 0;
    uint4 v = make_uint4(threadIdx.x, 1, 2, 3);
    const uint32_t base = smem_u32(S) + (((warp - 1) * 32 + lane) * 16);
    while (!stop) {
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(base + (i & 7) * 1536), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w));
      }
      n += 16;
    }
    if (lane == 0 && warp == 1) { cycles[blockIdx.x * 2 + 1] = (n * 16 * 32 * 3) * 1000 / (clock64() - t0); }
  }
  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  if (threadIdx.x == 0) sink[blockIdx.x] = 0;
}

// (b) CTA-pair MMA, M=256, N in {128, 256}; A: 128 rows per CTA, B: N/2 rows per CTA
template <int N>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) mma_pair(int groups, long long* cycles) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tslot;
  uint8_t* A = sm; uint8_t* B = sm + 16384;
  for (int i = threadIdx.x; i < (16384 + (N / 2) * 128) / 4; i += blockDim.x) ((uint32_t*)sm)[i] = 0x01010101u;
  const int warp = threadIdx.x >> 5;
  const uint32_t rank = cluster_rank();
  if (threadIdx.x == 0) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar))); asm volatile("fence.mbarrier_init.release.cluster;"); }
  if (warp == 0) { asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot))); asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;"); }
  asm volatile("fence.proxy.async.shared::cta;"); asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads(); cluster_sync();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tslot;
  const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
  if (threadIdx.x == 0) {
    uint32_t phase = 0;
    long long t0 = clock64();
    for (int g = 0; g < groups; ++g) {
      if (rank == 0) {
        for (int i = 0; i < 64; ++i)
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}"
                       ::"r"(tmem), "l"(sdesc(smem_u32(A) + (i & 3) * 32)), "l"(sdesc(smem_u32(B) + (i & 3) * 32)), "r"(idesc), "r"(1u));
        asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                     ::"r"(smem_u32(&bar)), "h"((uint16_t)3));
      }
      asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}" ::"r"(smem_u32(&bar)), "r"(phase));
      phase ^= 1;
    }
    cycles[blockIdx.x] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads(); cluster_sync();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  long long* d; int* sink; cudaMalloc(&d, 2 * sizeof(long long) * sms); cudaMalloc(&sink, 4 * sms);
  long long h[512];
  const int groups = 1000;
  cudaFuncSetAttribute(mma_with_stores, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  for (int stress = 0; stress < 2; ++stress) {
    cudaMemset(d, 0, 2 * sizeof(long long) * sms);
    mma_with_stores<<<sms, 128, 100 * 1024>>>(groups, stress, d, sink);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, 2 * sizeof(long long) * sms, cudaMemcpyDeviceToHost);
    double avg = 0, st = 0; for (int i = 0; i < sms; ++i) { avg += h[2 * i]; st += h[2 * i + 1]; } avg /= sms; st /= sms;
    printf("1cta N=128 stress=%d: %s %.0f MAC/clk/SM, st.shared %.1f B/clk\n", stress, cudaGetErrorString(e),
           (double)groups * 64 * 128 * 128 * 32 / avg, st / 1000.0);
  }
  {
    const int smem = 16384 + 128 * 128 + 1024;
    cudaFuncSetAttribute(mma_pair<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    mma_pair<256><<<sms, 128, smem>>>(groups, d);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
    double avg = 0; for (int i = 0; i < sms; ++i) avg += h[i]; avg /= sms;
    printf("2cta M=256 N=256: %s %.0f MAC/clk/SM\n", cudaGetErrorString(e), (double)groups * 64 * 256 * 256 * 32 / 2 / avg);
  }
  {
    const int smem = 16384 + 64 * 128 + 1024;
    cudaFuncSetAttribute(mma_pair<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    mma_pair<128><<<sms, 128, smem>>>(groups, d);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
    double avg = 0; for (int i = 0; i < sms; ++i) avg += h[i]; avg /= sms;
    printf("2cta M=256 N=128: %s %.0f MAC/clk/SM\n", cudaGetErrorString(e), (double)groups * 64 * 256 * 128 * 32 / 2 / avg);
  }
  return 0;
}
