// FP64 vector pipe throughput on B200: independent DFMA / DADD chains,
// 148 CTAs x 256 threads, CUDA-event timed.  Prints DP ops per clock per SM.
#include <cstdio>
#include <cuda_runtime.h>
template <int OP>
__global__ void k(double* out, int iters, double s) {
  double a[8];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) a[i] = fma(a[i], s, 1e-9);
      else if (OP == 1) a[i] = a[i] + s;
      else a[i] = __int2double_rn((int)a[i]) * s;  // I2F + DMUL
    }
  }
  double t = 0;
  for (int i = 0; i < 8; ++i) t += a[i];
  if (t == 123.456) out[0] = t;
}
int main() {
  double* o;
  cudaMalloc(&o, 8);
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int iters = 20000;
  for (int op = 0; op < 3; ++op) {
    for (int threads : {128, 256, 512}) {
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      auto launch = [&]() {
        if (op == 0) k<0><<<sms, threads>>>(o, iters, 0.999999);
        if (op == 1) k<1><<<sms, threads>>>(o, iters, 0.999999);
        if (op == 2) k<2><<<sms, threads>>>(o, iters, 0.999999);
      };
      launch();
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      double ops = (double)sms * threads * iters * 8;
      double per_clk_sm = ops / (ms * 1e-3) / (clk * 1e3) / sms;
      printf("op=%s threads=%d: %.3f ms, %.1f ops/clk/SM (at %d MHz nominal), %.2f Tops/s\n",
             op == 0 ? "DFMA" : op == 1 ? "DADD" : "I2F+DMUL", threads, ms, per_clk_sm, clk / 1000,
             ops / (ms * 1e-3) / 1e12);
    }
  }
  return 0;
}
