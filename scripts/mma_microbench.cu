// Microbenchmark: tcgen05.mma kind::i8 throughput for cta_group::1 tiles,
// operands resident in shared memory (no TMA), measured with clock64.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_mb mma_microbench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {
  uint64_t d = (uint64_t)((saddr & 0x3FFFFu) >> 4);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

template <int N, int MMAS_PER_GROUP>
__global__ void __launch_bounds__(128, 1) mma_loop(int groups, long long* cycles) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  uint8_t* A = sm;
  uint8_t* B = sm + 128 * 128;
  for (int i = threadIdx.x; i < (128 + N) * 128 / 4; i += blockDim.x) ((uint32_t*)sm)[i] = 0x01010101u;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tslot;
  const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  long long t0 = 0, t1 = 0;
  if (threadIdx.x == 0) {
    uint32_t phase = 0;
    t0 = clock64();
    for (int g = 0; g < groups; ++g) {
      for (int i = 0; i < MMAS_PER_GROUP; ++i) {
        const int kk = i & 3;
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}"
                     ::"r"(tmem + (uint32_t)((g & 1) * N)), "l"(sdesc(smem_u32(A) + kk * 32)),
                       "l"(sdesc(smem_u32(B) + kk * 32)), "r"(idesc), "r"(1u));
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
      asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}" ::"r"(smem_u32(&bar)), "r"(phase));
      phase ^= 1;
    }
    t1 = clock64();
    cycles[blockIdx.x] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

template <int N, int G>
void run(int sms) {
  long long* d;
  cudaMalloc(&d, sizeof(long long) * sms);
  const int smem = (128 + N) * 128 + 1024;
  cudaFuncSetAttribute(mma_loop<N, G>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int groups = 2000;
  mma_loop<N, G><<<sms, 128, smem>>>(groups, d);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  mma_loop<N, G><<<sms, 128, smem>>>(groups, d);
  cudaEventRecord(e1);
  cudaError_t err = cudaDeviceSynchronize();
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  long long h[256]; cudaMemcpy(h, d, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
  double avg = 0; for (int i = 0; i < sms; ++i) avg += h[i]; avg /= sms;
  const double macs = (double)groups * G * 128.0 * N * 32.0;
  printf("N=%d mmas/commit=%d: %s  %.1f cycles/mma  %.0f MAC/clk/SM  %.3f POPS (event %.3f ms)\n", N, G,
         cudaGetErrorString(err), avg / (groups * G), macs / avg, 2 * macs * sms / (ms / 1e3) / 1e15, ms);
  cudaFree(d);
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<128, 4>(sms);
  run<128, 16>(sms);
  run<128, 64>(sms);
  run<256, 4>(sms);
  run<256, 16>(sms);
  run<256, 64>(sms);
  run<64, 16>(sms);
  return 0;
}
