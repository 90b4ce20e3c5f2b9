// Per-step exchange latency inside one thread-block cluster (the candidate
// exchange a cluster-resident panel kernel would use): every CTA writes a
// record to its own shared memory, barrier.cluster arrive.release /
// wait.acquire, then warp 0 reads all G records' headers (DSMEM) and the
// winner's row.  Compare with gridsync_microbench (global-memory exchange).
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned cluster_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ unsigned mapa(const void* p, unsigned rank) {
  unsigned a = (unsigned)__cvta_generic_to_shared(p), r;
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

template <int MODE>
__global__ void k(int steps, double* out) {
  __shared__ double rec[2][68];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const unsigned me = cluster_rank(), G = gridDim.x;
  double acc = 0;
  cl_arrive();
  cl_wait();
  for (int t = 0; t < steps; ++t) {
    const int b = t & 1;
    if (wid == 0) {
      rec[b][4 + lane] = t + lane;
      rec[b][36 + lane] = t;
      if (lane == 0) rec[b][0] = (double)((me * 7 + t) % G);
    }
    cl_arrive();
    cl_wait();
    if (MODE >= 1 && wid == 0) {
      double v = lane < (int)G ? ld_dsmem(mapa(&rec[b][0], lane)) : -1.0;
      int g = lane;
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, v, o);
        const int og = __shfl_xor_sync(0xffffffffu, g, o);
        if (ov > v || (ov == v && og < g)) { v = ov; g = og; }
      }
      if (MODE >= 2) acc += ld_dsmem(mapa(&rec[b][4 + lane], g)) + ld_dsmem(mapa(&rec[b][36 + lane], g));
      else acc += v;
    }
    __syncthreads();
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
  cudaFuncSetAttribute(k<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(G);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = 200 * 1024;  // one CTA per SM, like the panel
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
  if (err != cudaSuccess || cudaGetLastError() != cudaSuccess) return -1;
  cudaFree(out);
  return ms * 1e3f / steps;
}

int main() {
  const int steps = 20000;
  for (int G : {2, 4, 8, 16}) {
    int n = 0;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(G);
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = 200 * 1024;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = G; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaFuncSetAttribute(k<2>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(k<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaOccupancyMaxActiveClusters(&n, (void*)k<2>, &cfg);
    printf("G=%2d  max active clusters %3d  barrier only %.3f us  +headers %.3f us  +winner row %.3f us\n",
           G, n, run<0>(G, steps), run<1>(G, steps), run<2>(G, steps));
  }
  return 0;
}
