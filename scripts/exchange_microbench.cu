// Per-step candidate exchange inside one thread-block cluster, three ways:
//  0: record in own SMEM, barrier.cluster arrive/wait, headers + winner row
//     read through DSMEM (the round-1 panel leaf);
//  1: push: every CTA copies its whole record (header + row, 544 B) into every
//     CTA's SMEM with cp.async.bulk (shared::cta -> shared::cluster, mbarrier
//     complete_tx), then waits on its own mbarrier and reduces locally;
//  2: push headers only (st.async 16 B per destination, mbarrier complete_tx),
//     winner row read through DSMEM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o exch scripts/exchange_microbench.cu
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int REC = 68;  // doubles per record: [0] |v|, [1] pos, [2] row, [4..68) values
constexpr int MAXG = 16;

__device__ __forceinline__ unsigned cluster_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ unsigned mapa(unsigned a, unsigned rank) {
  unsigned r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
__device__ __forceinline__ double ld_dsmem(unsigned addr) {
  double v;
  asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(addr) : "memory");
  return v;
}
__device__ __forceinline__ void cl_arrive() { asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory"); }
__device__ __forceinline__ void cl_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory"); }
__device__ __forceinline__ void mbar_init(unsigned bar, unsigned cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(cnt) : "memory");
}
__device__ __forceinline__ void mbar_expect(unsigned bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra W;\n\t}" ::"r"(bar), "r"(parity)
      : "memory");
}

template <int MODE>
__global__ void k(int steps, double* out) {
  __shared__ __align__(128) double mine[2][REC];         // own record (source of the push)
  __shared__ __align__(128) double recs[2][MAXG][REC];   // everyone's records (push modes)
  __shared__ __align__(8) uint64_t bar[2];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const unsigned me = cluster_rank(), G = gridDim.x;
  double acc = 0;
  if (threadIdx.x == 0) {
    mbar_init(smem_u32(&bar[0]), 1);
    mbar_init(smem_u32(&bar[1]), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  cl_arrive();
  cl_wait();
  unsigned ph[2] = {0, 0};
  for (int t = 0; t < steps; ++t) {
    const int b = t & 1;
    if (wid == 0) {
      // candidate record of this CTA (header + row values)
      mine[b][4 + lane] = t + lane;
      mine[b][36 + lane] = t;
      if (lane == 0) {
        mine[b][0] = (double)((me * 7 + t) % G);
        mine[b][1] = (double)me;
        mine[b][2] = 0;
        mine[b][3] = 0;
      }
      __syncwarp();
      if (MODE == 0) {
        // publish through own SMEM; everyone reads it after the barrier
      } else if (MODE == 1) {
        if (lane == 0) mbar_expect(smem_u32(&bar[b]), G * REC * 8);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane < (int)G) {
          const unsigned dst = mapa(smem_u32(&recs[b][me][0]), lane);
          const unsigned mb = mapa(smem_u32(&bar[b]), lane);
          asm volatile(
              "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
              ::"r"(dst), "r"(smem_u32(&mine[b][0])), "r"(REC * 8), "r"(mb)
              : "memory");
        }
      } else if (MODE == 3) {
        // st.async of the whole record: 34 16-byte chunks per destination
        if (lane == 0) mbar_expect(smem_u32(&bar[b]), G * REC * 8);
        __syncwarp();
        for (unsigned d = 0; d < G; ++d) {
          const unsigned mb = mapa(smem_u32(&bar[b]), d);
          for (int c = lane; c < REC / 2; c += 32) {
            const unsigned dst = mapa(smem_u32(&recs[b][me][2 * c]), d);
            const double v0 = mine[b][2 * c], v1 = mine[b][2 * c + 1];
            asm volatile(
                "st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];"
                ::"r"(dst), "d"(v0), "d"(v1), "r"(mb)
                : "memory");
          }
        }
      } else if (MODE == 4) {
        // no exchange at all (G = 1 work of a step)
      } else {
        if (lane == 0) mbar_expect(smem_u32(&bar[b]), G * 16);
        __syncwarp();
        if (lane < (int)G) {
          const unsigned dst = mapa(smem_u32(&recs[b][me][0]), lane);
          const unsigned mb = mapa(smem_u32(&bar[b]), lane);
          const double h0 = mine[b][0], h1 = mine[b][1];
          asm volatile(
              "st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];"
              ::"r"(dst), "d"(h0), "d"(h1), "r"(mb)
              : "memory");
        }
      }
    }
    if (MODE == 0) {
      cl_arrive();
      cl_wait();
    }
    if (wid == 0) {
      if (MODE != 0 && MODE != 4) {
        mbar_wait(smem_u32(&bar[b]), ph[b]);
        ph[b] ^= 1;
      }
      double v;
      if (MODE == 4)
        v = lane < (int)G ? mine[b][0] + lane : -1.0;
      else if (MODE == 0)
        v = lane < (int)G ? ld_dsmem(mapa(smem_u32(&mine[b][0]), lane)) : -1.0;
      else
        v = lane < (int)G ? recs[b][lane][0] : -1.0;
      int g = lane;
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, v, o);
        const int og = __shfl_xor_sync(0xffffffffu, g, o);
        if (ov > v || (ov == v && og < g)) { v = ov; g = og; }
      }
      if (MODE == 4)
        acc += mine[b][4 + lane] + mine[b][36 + lane] + g;
      else if (MODE == 1 || MODE == 3)
        acc += recs[b][g][4 + lane] + recs[b][g][36 + lane];
      else
        acc += ld_dsmem(mapa(smem_u32(&mine[b][4 + lane]), g)) +
               ld_dsmem(mapa(smem_u32(&mine[b][36 + lane]), g));
    }
    __syncthreads();
    if (MODE == 2) {
      // the DSMEM reads of mine[b] by other CTAs must finish before step t+2
      // rewrites it: the push of step t+1 proves every CTA passed step t
    }
  }
  cl_arrive();
  cl_wait();
  if (threadIdx.x == 0) out[blockIdx.x] = acc;
}

template <int MODE>
float run(int G, int steps) {
  double* out;
  cudaMalloc(&out, 64 * sizeof(double));
  cudaFuncSetAttribute(k<MODE>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(k<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 150 * 1024);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(G);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = 150 * 1024;  // one CTA per SM, like the panel
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = G;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaLaunchKernelEx(&cfg, k<MODE>, steps, out);
  cudaEventRecord(e0);
  cudaLaunchKernelEx(&cfg, k<MODE>, steps, out);
  cudaEventRecord(e1);
  cudaError_t err = cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  if (err != cudaSuccess || cudaGetLastError() != cudaSuccess) {
    printf("error %s\n", cudaGetErrorString(err));
    return -1;
  }
  double h[64];
  cudaMemcpy(h, out, G * sizeof(double), cudaMemcpyDeviceToHost);
  cudaFree(out);
  return ms * 1e3f / steps;
}

int main() {
  const int steps = getenv("EXCH_STEPS") ? atoi(getenv("EXCH_STEPS")) : 20000;
  for (int G : {2, 4, 8, 16}) {
    printf("G=%2d  barrier+DSMEM reads %.3f us  bulk push of records %.3f us  "
           "st.async headers + DSMEM row %.3f us  st.async records %.3f us  no exchange %.3f us\n",
           G, run<0>(G, steps), run<1>(G, steps), run<2>(G, steps), run<3>(G, steps),
           run<4>(G, steps));
  }
  return 0;
}
