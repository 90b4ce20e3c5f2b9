// Grid-wide step exchange latency on B200 (the panel kernel's per-column
// pattern): G co-resident CTAs; per step every CTA (lane 0 of warp 0)
// optionally writes a record, release-adds a counter and spins (acquire)
// until all G arrived, then optionally reads all records' headers.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void red_release_add(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
template <int MODE>
__global__ void k(unsigned* ctr, double* rec, int steps, double* out) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double acc = 0;
  for (int t = 0; t < steps; ++t) {
    if (wid == 0) {
      double* my = rec + ((size_t)(t & 1) * gridDim.x + blockIdx.x) * 68;
      double2* hdr = reinterpret_cast<double2*>(rec + 2 * 160 * 68) + (size_t)(t & 1) * gridDim.x;
      if (MODE >= 1) {  // record: 2 values per lane + header
        my[4 + lane] = t + lane;
        my[36 + lane] = t;
        if (lane == 0) my[0] = blockIdx.x * 1.0;
        if (MODE >= 4 && lane == 0) hdr[blockIdx.x] = make_double2(blockIdx.x * 1.0, t);
      }
      __syncwarp();
      if (lane == 0) {
        red_release_add(ctr, 1u);
        const unsigned target = gridDim.x * (unsigned)(t + 1);
        while (ld_acquire(ctr) < target) {
          if (MODE >= 10) __nanosleep(MODE == 10 ? 32 : 128);
        }
      }
      __syncwarp();
      if (MODE >= 2) {  // read all headers (5 per lane), then a winner row
        double best = -1;
        int bg = 0;
        for (int i = 0; i < 5; ++i) {
          const int g = lane + 32 * i;
          if (g < (int)gridDim.x) {
            const double v = MODE >= 10 ? __ldcg(rec + ((size_t)(t & 1) * gridDim.x + g) * 68)
                           : MODE == 8 ? rec[((size_t)(t & 1) * gridDim.x + g) * 68]  // weak ld (L1 path)
                           : MODE == 9 ? *(volatile double*)&rec[((size_t)(t & 1) * gridDim.x + g) * 68]
                           : MODE == 6 ? __ldcg(rec + 2 * 160 * 68 + 2 * 160 * 2 + g * 16)  // never written
                           : MODE == 7 ? __ldcg(rec + ((size_t)(t & 1) * gridDim.x + blockIdx.x) * 68 + i)  // own record
                           : MODE >= 4 ? __ldcg(&hdr[g]).x
                                       : __ldcg(rec + ((size_t)(t & 1) * gridDim.x + g) * 68);
            if (v > best) { best = v; bg = g; }
          }
        }
        for (int o = 16; o > 0; o >>= 1) {
          const double ob = __shfl_xor_sync(~0u, best, o);
          const int og = __shfl_xor_sync(~0u, bg, o);
          if (ob > best) { best = ob; bg = og; }
        }
        if (MODE == 3 || MODE == 5) acc += __ldcg(rec + ((size_t)(t & 1) * gridDim.x + bg) * 68 + 4 + lane);
        acc += best;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0 && acc == 1.2345) out[0] = acc;
}
int main() {
  unsigned* ctr;
  double *rec, *out;
  cudaMalloc(&ctr, 4);
  cudaMalloc(&rec, 2 * 160 * 68 * 8 + 2 * 160 * 16 + 160 * 16 * 8);
  cudaMemset(rec, 0, 2 * 160 * 68 * 8 + 2 * 160 * 16 + 160 * 16 * 8);
  cudaMalloc(&out, 8);
  const int steps = 2000;
  for (int mode : {0, 2, 10, 11})
    for (int G : {8, 32, 64, 128, 148}) {
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      for (int rep = 0; rep < 2; ++rep) {
        cudaMemset(ctr, 0, 4);
        void* args[] = {&ctr, &rec, (void*)&steps, &out};
        void* fn = mode == 0 ? (void*)k<0> : mode == 2 ? (void*)k<2> : mode == 10 ? (void*)k<10> : (void*)k<11>;
        cudaEventRecord(e0);
        cudaLaunchCooperativeKernel(fn, dim3(G), dim3(256), args, 0, 0);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
      }
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      printf("mode=%d (%s) G=%3d: %.2f us per step\n", mode,
             mode == 0 ? "counter only" : mode == 2 ? "ld.cg headers" : mode == 10 ? "headers, 32ns backoff" : "headers, 128ns backoff",
             G, ms * 1e3 / steps);
    }
  return 0;
}
