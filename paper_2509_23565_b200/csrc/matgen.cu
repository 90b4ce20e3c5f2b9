// matgen.cu — K13 of SURVEY §2.2: the matrix generators on the device,
// bit-identical with numpy's default_rng(seed).random((n, n)).
//
// Reference: /root/reference/pkg/src/ozemu/matgen.py
//   parawilk            :133-146  1 on the diagonal, -1 on subdiagonals 1..d,
//                                 alpha in columns c = b, 2b, ... for rows < c
//   parawilk_randomized :149-161  zero pattern entries <- 2.0*u*u
//   hpl_uniform         :164-171  u - 0.5
// Element (i, j) consumes stream position i*n + j (row-major draw order,
// matgen.py:4-6).  numpy's PCG64 step is state = state*M + inc followed by the
// XSL-RR output of the NEW state; random() = (x >> 11) * 2^-53.  Threads jump
// ahead with the O(log n) LCG advance and then step sequentially.
#include "common.cuh"

namespace oz {
namespace {

typedef unsigned __int128 u128;

__device__ __forceinline__ u128 pcg_mult() {
  return ((u128)0x2360ED051FC65DA4ull << 64) | (u128)0x4385DF649FCCF645ull;
}

__device__ __forceinline__ u128 pcg_advance(u128 state, u128 inc, unsigned long long delta) {
  u128 acc_m = 1, acc_p = 0, cm = pcg_mult(), cp = inc;
  while (delta > 0) {
    if (delta & 1) {
      acc_m *= cm;
      acc_p = acc_p * cm + cp;
    }
    cp = (cm + 1) * cp;
    cm *= cm;
    delta >>= 1;
  }
  return acc_m * state + acc_p;
}

__device__ __forceinline__ double pcg_double(u128 s) {
  const unsigned long long hi = (unsigned long long)(s >> 64);
  const unsigned long long lo = (unsigned long long)s;
  const unsigned long long x = hi ^ lo;
  const unsigned rot = (unsigned)(hi >> 58);
  const unsigned long long r = (x >> rot) | (x << ((64u - rot) & 63u));
  return (double)(r >> 11) * 0x1.0p-53;
}

__device__ __forceinline__ double pattern(int64_t i, int64_t j, int64_t d, int64_t blk,
                                          double alpha) {
  if (i == j) return 1.0;
  const int64_t diff = i - j;
  if (diff >= 1 && diff <= d) return -1.0;
  if (j >= blk && j % blk == 0 && i < j) return alpha;
  return 0.0;
}

__device__ __forceinline__ double element(int kind, int64_t i, int64_t j, double u, int64_t d,
                                          int64_t blk, double alpha) {
  if (kind == OZ_GEN_UNIFORM) return __dsub_rn(u, 0.5);
  const double base = pattern(i, j, d, blk, alpha);
  if (kind == OZ_GEN_PARAWILK || base != 0.0) return base;
  return __dmul_rn(__dmul_rn(2.0, u), u);
}

constexpr int RUN = 64;

// column-major friendly: thread = (row i, column run [j0, j0+RUN)); a warp covers 32
// consecutive rows so every store instruction writes 32 consecutive rows of one column.
__global__ void gen_rowruns_kernel(int kind, int64_t n, int64_t d, int64_t blk, double alpha,
                                   unsigned long long st_hi, unsigned long long st_lo,
                                   unsigned long long inc_hi, unsigned long long inc_lo,
                                   double* __restrict__ out, int64_t rs, int64_t cs) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t j0 = (int64_t)blockIdx.y * RUN;
  if (i >= n) return;
  const int64_t j1 = min(n, j0 + RUN);
  if (kind == OZ_GEN_PARAWILK) {
    for (int64_t j = j0; j < j1; ++j) out[i * rs + j * cs] = pattern(i, j, d, blk, alpha);
    return;
  }
  const u128 inc = ((u128)inc_hi << 64) | inc_lo;
  u128 s = pcg_advance(((u128)st_hi << 64) | st_lo, inc, (unsigned long long)(i * n + j0));
  const u128 m = pcg_mult();
  for (int64_t j = j0; j < j1; ++j) {
    s = s * m + inc;
    out[i * rs + j * cs] = element(kind, i, j, pcg_double(s), d, blk, alpha);
  }
}

// row-major friendly: lane l of a warp produces stream positions base+l, base+l+32, ...
__global__ void gen_interleaved_kernel(int kind, int64_t n, int64_t d, int64_t blk, double alpha,
                                       unsigned long long st_hi, unsigned long long st_lo,
                                       unsigned long long inc_hi, unsigned long long inc_lo,
                                       double* __restrict__ out, int64_t rs, int64_t cs,
                                       int64_t per_warp) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t total = n * n;
  const int64_t base = warp * per_warp;
  if (base >= total) return;
  const int64_t end = min(total, base + per_warp);
  const u128 inc = ((u128)inc_hi << 64) | inc_lo;
  const u128 s0 = ((u128)st_hi << 64) | st_lo;
  u128 s = pcg_advance(s0, inc, (unsigned long long)(base + lane + 1));
  // 32-step jump constants: s_{k+32} = M32 * s_k + C32
  u128 m32 = 1, c32 = 0;
  {
    const u128 m = pcg_mult();
    for (int k = 0; k < 32; ++k) {
      m32 *= m;
      c32 = c32 * m + inc;
    }
  }
  for (int64_t idx = base + lane; idx < end; idx += 32) {
    const int64_t i = idx / n, j = idx - (idx / n) * n;
    out[i * rs + j * cs] =
        kind == OZ_GEN_PARAWILK ? pattern(i, j, d, blk, alpha)
                                : element(kind, i, j, pcg_double(s), d, blk, alpha);
    s = m32 * s + c32;
  }
}

// 1 x Q block-cyclic column slab: local column lc of process column q holds
// global column ((lc / nb) * Q + q) * nb + lc % nb; output column-major (ldo).
// Same element values as the full generator (stream position i*n + j).
__global__ void gen_cyclic_kernel(int kind, int64_t n, int64_t d, int64_t blk, double alpha,
                                  unsigned long long st_hi, unsigned long long st_lo,
                                  unsigned long long inc_hi, unsigned long long inc_lo,
                                  int64_t nb, int64_t P, int64_t p, int64_t mloc,
                                  int64_t Q, int64_t q, int64_t ncols,
                                  double* __restrict__ out, int64_t ldo) {
  const int64_t li = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t lc0 = (int64_t)blockIdx.y * RUN;
  if (li >= mloc) return;
  const int64_t i = ((li / nb) * P + p) * nb + li % nb;
  const int64_t lc1 = min(ncols, lc0 + RUN);
  const u128 inc = ((u128)inc_hi << 64) | inc_lo;
  const u128 s0 = ((u128)st_hi << 64) | st_lo;
  const u128 m = pcg_mult();
  u128 s = 0;
  for (int64_t lc = lc0; lc < lc1; ++lc) {
    const int64_t j = ((lc / nb) * Q + q) * nb + lc % nb;
    if (kind == OZ_GEN_PARAWILK) {
      out[li + lc * ldo] = pattern(i, j, d, blk, alpha);
      continue;
    }
    if (lc == lc0 || lc % nb == 0) s = pcg_advance(s0, inc, (unsigned long long)(i * n + j));
    s = s * m + inc;
    out[li + lc * ldo] = element(kind, i, j, pcg_double(s), d, blk, alpha);
  }
}

}  // namespace
}  // namespace oz

extern "C" int oz_generate_block_cyclic(int kind, int64_t n, int64_t depth, int64_t block,
                                        double alpha, uint64_t state_hi, uint64_t state_lo,
                                        uint64_t inc_hi, uint64_t inc_lo, int64_t nb, int64_t P,
                                        int64_t p, int64_t mloc, int64_t Q, int64_t q,
                                        int64_t ncols, double* out, int64_t ldo, void* stream) {
  using namespace oz;
  OZ_REQUIRE(kind >= 0 && kind <= 2, OZ_INVALID_PARAMS, "bad generator kind %d", kind);
  OZ_REQUIRE(n >= 1 && nb >= 1 && P >= 1 && p >= 0 && p < P && Q >= 1 && q >= 0 && q < Q &&
                 mloc >= 0 && ldo >= mloc,
             OZ_INVALID_PARAMS, "bad block-cyclic generator shape");
  if (ncols <= 0 || mloc <= 0) return OZ_OK;
  const int64_t d = depth > n - 1 ? n - 1 : depth;
  dim3 grid((unsigned)ceil_div(mloc, 128), (unsigned)ceil_div(ncols, RUN));
  gen_cyclic_kernel<<<grid, 128, 0, as_stream(stream)>>>(kind, n, d, block, alpha, state_hi,
                                                        state_lo, inc_hi, inc_lo, nb, P, p, mloc,
                                                        Q, q, ncols, out, ldo);
  OZ_CHECK_LAUNCH();
  return OZ_OK;
}

extern "C" int oz_generate_cyclic(int kind, int64_t n, int64_t depth, int64_t block,
                                  double alpha, uint64_t state_hi, uint64_t state_lo,
                                  uint64_t inc_hi, uint64_t inc_lo, int64_t nb, int64_t Q,
                                  int64_t q, int64_t ncols, double* out, int64_t ldo,
                                  void* stream) {
  return oz_generate_block_cyclic(kind, n, depth, block, alpha, state_hi, state_lo, inc_hi,
                                  inc_lo, nb, 1, 0, n, Q, q, ncols, out, ldo, stream);
}

extern "C" int oz_generate(int kind, int64_t n, int64_t depth, int64_t block, double alpha,
                           uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo,
                           double* out, int64_t row_stride, int64_t col_stride, void* stream) {
  using namespace oz;
  OZ_REQUIRE(kind >= 0 && kind <= 2, OZ_INVALID_PARAMS, "bad generator kind %d", kind);
  OZ_REQUIRE(n >= 1, OZ_INVALID_PARAMS, "n must be >= 1");
  cudaStream_t st = as_stream(stream);
  const int64_t d = depth > n - 1 ? n - 1 : depth;
  if (col_stride == 1 && row_stride != 1) {
    const int64_t per_warp = 32 * 64;
    const int64_t warps = ceil_div(n * n, per_warp);
    gen_interleaved_kernel<<<(unsigned)ceil_div(warps * 32, 256), 256, 0, st>>>(
        kind, n, d, block, alpha, state_hi, state_lo, inc_hi, inc_lo, out, row_stride, col_stride,
        per_warp);
  } else {
    dim3 grid((unsigned)ceil_div(n, 128), (unsigned)ceil_div(n, RUN));
    gen_rowruns_kernel<<<grid, 128, 0, st>>>(kind, n, d, block, alpha, state_hi, state_lo, inc_hi,
                                             inc_lo, out, row_stride, col_stride);
  }
  OZ_CHECK_LAUNCH();
  return OZ_OK;
}
