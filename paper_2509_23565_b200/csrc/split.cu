// split.cu — K1/K2 of SURVEY §2.2: error-free split of an FP64 matrix into
// k signed q-bit slices under one power-of-two exponent per vector.
//
// Reference semantics: /root/reference/pkg/src/ozemu/split.py:109-160
//   e_v = frexp(max_t |a[v,t]|).exp      (0 for an all-zero vector)   :131-138
//   x   = ldexp(a, -e_v)                                                 :142
//   repeat k times: y = x*2^q; s = trunc(y); slice = s; x = y - s        :147-151
// Every step is exact in FP64, so the GPU result is bit-identical.
//
// Layout: "vector" v carries the exponent (rows when ROW_SCALED, columns when
// COL_SCALED), t is the inner (GEMM-K) index.  Element (v,t) of the source is
// src[v*vs + t*ts].  Output slices are K-major int8: slices[s*sstride + v*ld + t].
// For q = 8..10 (int16 slices, split.py:144) each slice is written as two int8
// planes, plane 2s = floor(slice / 128) and plane 2s+1 = slice mod 128, so the
// tensor cores multiply int8 planes and the GEMM recombines the slice product
// exactly (gemm_emu.cu, kWide).
//
// Two kernels: (1) exponent pass = warp-shuffle max reduction per vector plus
// NaN/Inf detection; (2) slice emission.  Each has a fast path for the
// K-contiguous case (ts == 1: 128-bit loads, one warp per vector, 16-byte
// stores per slice) and a tiled shared-memory transpose path for the
// vector-contiguous case (vs == 1, e.g. the LU's A21 panel in column-major).
#include "common.cuh"

namespace oz {
namespace {

struct SplitAux {
  int32_t nonfinite;
  int32_t pad;
  unsigned long long global_maxbits;  // IEEE bits of the global max |x|
};

__device__ __forceinline__ void note_value(double v, double& mx, bool& bad) {
  double a = fabs(v);
  if (!isfinite(v)) bad = true;
  mx = fmax(mx, a);
}

// ---- exponent pass, K contiguous: one warp per vector ----------------------
__global__ void exps_kcontig_kernel(const double* __restrict__ src, int64_t nvec, int64_t K,
                                    int64_t vs, int mode, int32_t* __restrict__ exps,
                                    SplitAux* aux) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  bool any_bad = false;
  double gmax = 0.0;
  for (int64_t v = warp; v < nvec; v += nwarps) {
    const double* p = src + v * vs;
    double mx = 0.0;
    bool bad = false;
    const bool vec2 = ((reinterpret_cast<uintptr_t>(p) & 15) == 0);
    if (vec2) {
      const double2* p2 = reinterpret_cast<const double2*>(p);
      const int64_t K2 = K >> 1;
      for (int64_t t = lane; t < K2; t += 32) {
        double2 w = __ldg(p2 + t);
        note_value(w.x, mx, bad);
        note_value(w.y, mx, bad);
      }
      if ((K & 1) && lane == 0) note_value(__ldg(p + K - 1), mx, bad);
    } else {
      for (int64_t t = lane; t < K; t += 32) note_value(__ldg(p + t), mx, bad);
    }
    mx = warp_max(mx);
    bad = __any_sync(0xffffffffu, bad);
    if (lane == 0) exps[v] = (mx == 0.0 || bad) ? 0 : frexp_exp(mx);
    any_bad |= bad;
    gmax = fmax(gmax, mx);
  }
  if (lane == 0) {
    if (any_bad) aux->nonfinite = 1;
    if (mode == OZ_GLOBAL && gmax > 0.0)
      atomicMax(&aux->global_maxbits, (unsigned long long)__double_as_longlong(gmax));
  }
}

// ---- exponent pass, general strides: 32 vectors x 8 row-groups per CTA ------
__global__ void exps_tiled_kernel(const double* __restrict__ src, int64_t nvec, int64_t K,
                                  int64_t vs, int64_t ts, int mode,
                                  int32_t* __restrict__ exps, SplitAux* aux) {
  __shared__ double smax[8][33];
  __shared__ int sbad;
  const int lx = threadIdx.x & 31, ly = threadIdx.x >> 5;
  if (threadIdx.x == 0) sbad = 0;
  __syncthreads();
  const int64_t v = blockIdx.x * 32ll + lx;
  double mx = 0.0;
  bool bad = false;
  if (v < nvec) {
    const double* p = src + v * vs;
    for (int64_t t = ly; t < K; t += 8) note_value(__ldg(p + t * ts), mx, bad);
  }
  smax[ly][lx] = mx;
  if (bad) sbad = 1;
  __syncthreads();
  if (ly == 0) {
    double m = smax[0][lx];
#pragma unroll
    for (int i = 1; i < 8; ++i) m = fmax(m, smax[i][lx]);
    const bool anybad = sbad != 0;
    if (v < nvec) exps[v] = (m == 0.0 || anybad) ? 0 : frexp_exp(m);
    double g = warp_max(m);
    if (lx == 0) {
      if (anybad) aux->nonfinite = 1;
      if (mode == OZ_GLOBAL && g > 0.0)
        atomicMax(&aux->global_maxbits, (unsigned long long)__double_as_longlong(g));
    }
  }
}

__device__ __forceinline__ int vector_exponent(const int32_t* exps, int64_t v, int mode,
                                               const SplitAux* aux) {
  if (mode == OZ_GLOBAL) {
    const double g = __longlong_as_double((long long)aux->global_maxbits);
    return g > 0.0 ? frexp_exp(g) : 0;
  }
  return exps[v];
}

// ---- slice emission, K contiguous: one warp per vector, 16 t per lane ------
template <int KS>
__global__ void slices_kcontig_kernel(const double* __restrict__ src, int64_t nvec, int64_t K,
                                      int64_t vs, int mode, int ksl, int q, bool wide,
                                      int8_t* __restrict__ out, int64_t ld, int64_t sstride,
                                      int32_t* __restrict__ exps, const SplitAux* aux) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const double radix = (double)(1 << q);
  for (int64_t v = warp; v < nvec; v += nwarps) {
    const int e = vector_exponent(exps, v, mode, aux);
    if (mode == OZ_GLOBAL && lane == 0) exps[v] = e;
    const double* p = src + v * vs;
    const bool vec2 = ((reinterpret_cast<uintptr_t>(p) & 15) == 0);
    for (int64_t t0 = (int64_t)lane * 16; t0 < ld; t0 += 32 * 16) {
      double x[16];
      if (t0 + 16 <= K && vec2) {
        const double2* p2 = reinterpret_cast<const double2*>(p + t0);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          double2 w = __ldg(p2 + i);
          x[2 * i] = w.x;
          x[2 * i + 1] = w.y;
        }
      } else {
#pragma unroll
        for (int i = 0; i < 16; ++i) x[i] = (t0 + i < K) ? __ldg(p + t0 + i) : 0.0;
      }
#pragma unroll
      for (int i = 0; i < 16; ++i) x[i] = ldexp_exact(x[i], -e);
      for (int s = 0; s < ksl; ++s) {
        uint32_t w[4], wl[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          uint32_t packed = 0, packed_lo = 0;
#pragma unroll
          for (int b = 0; b < 4; ++b) {
            double y = __dmul_rn(x[4 * i + b], radix);
            double tr = trunc(y);
            x[4 * i + b] = __dsub_rn(y, tr);
            const int ti = (int)tr;
            // q > 7: slice = 128 * hi + lo, hi = floor(slice / 128), lo in [0, 127]
            packed |= (uint32_t)(uint8_t)(int8_t)(wide ? (ti >> 7) : ti) << (8 * b);
            packed_lo |= (uint32_t)(uint8_t)(ti & 127) << (8 * b);
          }
          w[i] = packed;
          wl[i] = packed_lo;
        }
        // ld is a multiple of 16, so every 16-byte store is in bounds
        int8_t* dst = out + (wide ? 2 * s : s) * sstride + v * ld + t0;
        *reinterpret_cast<uint4*>(dst) = make_uint4(w[0], w[1], w[2], w[3]);
        if (wide)
          *reinterpret_cast<uint4*>(dst + sstride) = make_uint4(wl[0], wl[1], wl[2], wl[3]);
      }
    }
  }
}

// ---- slice emission, general strides: 32 vectors x 64 t tile via smem ------
__global__ void slices_tiled_kernel(const double* __restrict__ src, int64_t nvec, int64_t K,
                                    int64_t vs, int64_t ts, int mode, int ksl, int q, bool wide,
                                    int8_t* __restrict__ out, int64_t ld, int64_t sstride,
                                    int32_t* __restrict__ exps, const SplitAux* aux) {
  __shared__ double tile[64][33];
  __shared__ int sexp[32];
  const int tid = threadIdx.x;
  const int64_t v0 = blockIdx.x * 32ll;
  const int64_t t0 = blockIdx.y * 64ll;
  if (tid < 32) {
    const int64_t v = v0 + tid;
    int e = 0;
    if (v < nvec) {
      e = vector_exponent(exps, v, mode, aux);
      if (mode == OZ_GLOBAL && blockIdx.y == 0) exps[v] = e;
    }
    sexp[tid] = e;
  }
  // coalesced load along the vector index
  const int lx = tid & 31, ly = tid >> 5;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int tl = ly + 8 * j;
    const int64_t t = t0 + tl, v = v0 + lx;
    tile[tl][lx] = (v < nvec && t < K) ? __ldg(src + v * vs + t * ts) : 0.0;
  }
  __syncthreads();
  const int vl = tid >> 3;          // 0..31
  const int tc = (tid & 7) * 8;     // 0..56
  const int64_t v = v0 + vl;
  const int64_t tt = t0 + tc;
  if (v >= nvec || tt >= ld) return;
  const int e = sexp[vl];
  const double radix = (double)(1 << q);
  double x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = ldexp_exact(tile[tc + i][vl], -e);
  for (int s = 0; s < ksl; ++s) {
    uint32_t w[2], wl[2];
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      uint32_t packed = 0, packed_lo = 0;
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        double y = __dmul_rn(x[4 * i + b], radix);
        double tr = trunc(y);
        x[4 * i + b] = __dsub_rn(y, tr);
        const int ti = (int)tr;
        packed |= (uint32_t)(uint8_t)(int8_t)(wide ? (ti >> 7) : ti) << (8 * b);
        packed_lo |= (uint32_t)(uint8_t)(ti & 127) << (8 * b);
      }
      w[i] = packed;
      wl[i] = packed_lo;
    }
    int8_t* dst = out + (wide ? 2 * s : s) * sstride + v * ld + tt;
    *reinterpret_cast<uint2*>(dst) = make_uint2(w[0], w[1]);
    if (wide) *reinterpret_cast<uint2*>(dst + sstride) = make_uint2(wl[0], wl[1]);
  }
}

// ---- one pass, K contiguous (ts == 1), K <= 1024, per-vector exponents: one
// warp per vector keeps its values in registers (lane l owns t = 16 l + 512 c
// .. +15, the slice kernel's chunks), reduces the max, emits the slices — the
// source is read once.  Same per-element arithmetic as the two-pass kernels.
__global__ void split_kcontig_onepass_kernel(const double* __restrict__ src, int64_t nvec,
                                             int64_t K, int64_t vs, int ksl, int q, bool wide,
                                             int8_t* __restrict__ out, int64_t ld,
                                             int64_t sstride, int32_t* __restrict__ exps,
                                             SplitAux* aux) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const double radix = (double)(1 << q);
  bool any_bad = false;
  for (int64_t v = warp; v < nvec; v += nwarps) {
    const double* p = src + v * vs;
    const bool vec2 = ((reinterpret_cast<uintptr_t>(p) & 15) == 0);
    double x[2][16];
    double mx = 0.0;
    bool bad = false;
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const int64_t t0 = (int64_t)lane * 16 + 512 * c;
      if (t0 + 16 <= K && vec2) {
        const double2* p2 = reinterpret_cast<const double2*>(p + t0);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const double2 w = __ldg(p2 + i);
          x[c][2 * i] = w.x;
          x[c][2 * i + 1] = w.y;
        }
      } else {
#pragma unroll
        for (int i = 0; i < 16; ++i) x[c][i] = (t0 + i < K) ? __ldg(p + t0 + i) : 0.0;
      }
#pragma unroll
      for (int i = 0; i < 16; ++i) note_value(x[c][i], mx, bad);
    }
    mx = warp_max(mx);
    bad = __any_sync(0xffffffffu, bad);
    any_bad |= bad;
    const int e = (mx == 0.0 || bad) ? 0 : frexp_exp(mx);
    if (lane == 0) exps[v] = e;
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const int64_t t0 = (int64_t)lane * 16 + 512 * c;
      if (t0 >= ld) continue;
#pragma unroll
      for (int i = 0; i < 16; ++i) x[c][i] = ldexp_exact(x[c][i], -e);
      for (int s2 = 0; s2 < ksl; ++s2) {
        uint32_t w[4], wl[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          uint32_t packed = 0, packed_lo = 0;
#pragma unroll
          for (int b = 0; b < 4; ++b) {
            double y = __dmul_rn(x[c][4 * i + b], radix);
            double tr = trunc(y);
            x[c][4 * i + b] = __dsub_rn(y, tr);
            const int ti = (int)tr;
            packed |= (uint32_t)(uint8_t)(int8_t)(wide ? (ti >> 7) : ti) << (8 * b);
            packed_lo |= (uint32_t)(uint8_t)(ti & 127) << (8 * b);
          }
          w[i] = packed;
          wl[i] = packed_lo;
        }
        int8_t* dst = out + (wide ? 2 * s2 : s2) * sstride + v * ld + t0;
        *reinterpret_cast<uint4*>(dst) = make_uint4(w[0], w[1], w[2], w[3]);
        if (wide)
          *reinterpret_cast<uint4*>(dst + sstride) = make_uint4(wl[0], wl[1], wl[2], wl[3]);
      }
    }
  }
  if (lane == 0 && any_bad) aux->nonfinite = 1;
}

// ---- one pass, vector-contiguous source (vs == 1, e.g. the LU's A21 panel in
// column-major), per-vector exponents, K <= OP_K: a CTA keeps OP_R vectors x
// K values in shared memory, reduces each vector's max, then emits its slices
// from the tile — the FP64 source is read once instead of twice (exponent pass
// + slice pass).  Same per-element arithmetic as the two-pass kernels.
constexpr int OP_R = 8;      // vectors per CTA (70 KB tile: three CTAs per SM overlap load and emit)
constexpr int OP_K = 1024;   // max K
constexpr int OP_LD = OP_R + 1;  // tile row pitch (doubles)
__global__ void __launch_bounds__(256) split_onepass_kernel(
    const double* __restrict__ src, int64_t nvec, int64_t K, int64_t ts, int ksl, int q,
    bool wide, int8_t* __restrict__ out, int64_t ld, int64_t sstride, int32_t* __restrict__ exps,
    SplitAux* aux) {
  extern __shared__ double tile[];  // [OP_K][OP_LD]: tile[t * OP_LD + r]
  __shared__ double smax[8][2][32];
  __shared__ int sexp[OP_R];
  __shared__ int sbad;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int64_t v0 = (int64_t)blockIdx.x * OP_R;
  if (tid == 0) sbad = 0;
  // load: thread -> row r = tid % OP_R of columns t = tid / OP_R + (256 / OP_R) i
  constexpr int CS = 256 / OP_R;  // columns per pass
  const int r = tid & (OP_R - 1), tq = tid / OP_R;
  const int64_t v = v0 + r;
  const bool vok = v < nvec;
  double mx = 0.0;
  bool bad = false;
#pragma unroll 8
  for (int t = tq; t < K; t += CS) {
    const double x = vok ? __ldg(src + v + (int64_t)t * ts) : 0.0;
    tile[t * OP_LD + r] = x;
    note_value(x, mx, bad);
  }
  // the lanes of a warp that share a row (lane % OP_R), then across the 8
  // warps (max and the non-finite flag per row)
#pragma unroll
  for (int o = OP_R; o < 32; o <<= 1) {
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    bad = bad || __shfl_xor_sync(0xffffffffu, (int)bad, o);
  }
  if (lane < OP_R) {
    smax[wid][0][lane] = mx;
    smax[wid][1][lane] = bad ? 1.0 : 0.0;
  }
  if (bad) sbad = 1;
  __syncthreads();
  if (tid < OP_R) {
    double m = smax[0][0][tid], b = smax[0][1][tid];
#pragma unroll
    for (int w = 1; w < 8; ++w) {
      m = fmax(m, smax[w][0][tid]);
      b = fmax(b, smax[w][1][tid]);
    }
    const int e = (m == 0.0 || b != 0.0) ? 0 : frexp_exp(m);
    sexp[tid] = e;
    if (v0 + tid < nvec) exps[v0 + tid] = e;
  }
  if (tid == 0 && sbad) aux->nonfinite = 1;
  __syncthreads();
  // emit: thread -> row r, 16 consecutive t per chunk
  const double radix = (double)(1 << q);
  const int e = sexp[r];
  if (!vok) return;
  for (int64_t t0 = (int64_t)tq * 16; t0 < ld; t0 += 16 * CS) {
    double x[16];
#pragma unroll
    for (int i = 0; i < 16; ++i)
      x[i] = t0 + i < K ? ldexp_exact(tile[(t0 + i) * OP_LD + r], -e) : 0.0;
    for (int s2 = 0; s2 < ksl; ++s2) {
      uint32_t w[4], wl[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        uint32_t packed = 0, packed_lo = 0;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          double y = __dmul_rn(x[4 * i + b], radix);
          double tr = trunc(y);
          x[4 * i + b] = __dsub_rn(y, tr);
          const int ti = (int)tr;
          packed |= (uint32_t)(uint8_t)(int8_t)(wide ? (ti >> 7) : ti) << (8 * b);
          packed_lo |= (uint32_t)(uint8_t)(ti & 127) << (8 * b);
        }
        w[i] = packed;
        wl[i] = packed_lo;
      }
      int8_t* dst = out + (wide ? 2 * s2 : s2) * sstride + v * ld + t0;
      *reinterpret_cast<uint4*>(dst) = make_uint4(w[0], w[1], w[2], w[3]);
      if (wide) *reinterpret_cast<uint4*>(dst + sstride) = make_uint4(wl[0], wl[1], wl[2], wl[3]);
    }
  }
}
constexpr size_t OP_SMEM = sizeof(double) * OP_K * OP_LD;

}  // namespace

// OZ_SPLIT_ONEPASS=0: the two-pass tiled kernels for vector-contiguous sources (A/B)
bool split_onepass_enabled() {
  static const bool v = !getenv("OZ_SPLIT_ONEPASS") || atoi(getenv("OZ_SPLIT_ONEPASS"));
  return v;
}

int split_launch(const double* src, int64_t rows, int64_t cols, int64_t row_stride,
                 int64_t col_stride, int orientation, int mode, int k, int q, int8_t* slices,
                 int64_t slice_ld, int64_t slice_stride, int32_t* exps, void* aux_v,
                 cudaStream_t st) {
  OZ_REQUIRE(k >= 1, OZ_INVALID_PARAMS, "num_slices must be >= 1");
  OZ_REQUIRE(q >= 1 && q <= 10, OZ_INVALID_PARAMS, "slice_bits=%d outside 1..10", q);
  const bool wide = q > 7;  // int16 slices, emitted as (hi, lo) int8 planes
  OZ_REQUIRE(rows >= 1 && cols >= 1, OZ_INVALID_PARAMS, "empty matrices are not supported");
  OZ_REQUIRE(orientation == OZ_ROW_SCALED || orientation == OZ_COL_SCALED, OZ_INVALID_PARAMS,
             "bad orientation");
  OZ_REQUIRE(mode == OZ_PER_VECTOR || mode == OZ_GLOBAL, OZ_INVALID_PARAMS, "bad mode");
  const bool rowsc = orientation == OZ_ROW_SCALED;
  const int64_t nvec = rowsc ? rows : cols;
  const int64_t K = rowsc ? cols : rows;
  const int64_t vs = rowsc ? row_stride : col_stride;
  const int64_t ts = rowsc ? col_stride : row_stride;
  OZ_REQUIRE(slice_ld >= K && slice_ld % 16 == 0, OZ_INVALID_PARAMS,
             "slice_ld must be >= K and a multiple of 16");
  OZ_REQUIRE(slice_stride >= nvec * slice_ld, OZ_INVALID_PARAMS, "slice_stride too small");
  SplitAux* aux = reinterpret_cast<SplitAux*>(aux_v);
  OZ_CHECK_CUDA(cudaMemsetAsync(aux, 0, sizeof(SplitAux), st));
  const int sms = sm_count();
  if (ts == 1 && mode == OZ_PER_VECTOR && K <= 1024 && slice_ld <= 1024 &&
      split_onepass_enabled()) {
    const int threads = 256;
    int64_t blocks = ceil_div(nvec, threads / 32);
    blocks = blocks > (int64_t)sms * 16 ? (int64_t)sms * 16 : blocks;
    split_kcontig_onepass_kernel<<<(unsigned)blocks, threads, 0, st>>>(
        src, nvec, K, vs, k, q, wide, slices, slice_ld, slice_stride, exps, aux);
    OZ_CHECK_LAUNCH();
  } else if (ts == 1) {
    const int threads = 256;
    int64_t blocks = ceil_div(nvec, threads / 32);
    blocks = blocks > (int64_t)sms * 16 ? (int64_t)sms * 16 : blocks;
    exps_kcontig_kernel<<<(unsigned)blocks, threads, 0, st>>>(src, nvec, K, vs, mode, exps, aux);
    OZ_CHECK_LAUNCH();
    slices_kcontig_kernel<16><<<(unsigned)blocks, threads, 0, st>>>(
        src, nvec, K, vs, mode, k, q, wide, slices, slice_ld, slice_stride, exps, aux);
    OZ_CHECK_LAUNCH();
  } else if (vs == 1 && mode == OZ_PER_VECTOR && K <= OP_K && split_onepass_enabled()) {
    OZ_ONCE(cudaFuncSetAttribute(split_onepass_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)OP_SMEM));
    split_onepass_kernel<<<(unsigned)ceil_div(nvec, OP_R), 256, OP_SMEM, st>>>(
        src, nvec, K, ts, k, q, wide, slices, slice_ld, slice_stride, exps, aux);
    OZ_CHECK_LAUNCH();
  } else {
    exps_tiled_kernel<<<(unsigned)ceil_div(nvec, 32), 256, 0, st>>>(src, nvec, K, vs, ts, mode,
                                                                     exps, aux);
    OZ_CHECK_LAUNCH();
    dim3 grid((unsigned)ceil_div(nvec, 32), (unsigned)ceil_div(slice_ld, 64));
    slices_tiled_kernel<<<grid, 256, 0, st>>>(src, nvec, K, vs, ts, mode, k, q, wide, slices, slice_ld,
                                              slice_stride, exps, aux);
    OZ_CHECK_LAUNCH();
  }
  return OZ_OK;
}

}  // namespace oz

extern "C" size_t oz_split_aux_bytes(void) { return 16; }

extern "C" int oz_split(const double* src, int64_t rows, int64_t cols, int64_t row_stride,
                        int64_t col_stride, int orientation, int mode, int num_slices,
                        int slice_bits, int8_t* slices, int64_t slice_ld, int64_t slice_stride,
                        int32_t* exps, void* aux, void* stream) {
  return oz::split_launch(src, rows, cols, row_stride, col_stride, orientation, mode, num_slices,
                          slice_bits, slices, slice_ld, slice_stride, exps, aux,
                          oz::as_stream(stream));
}
