// dpanel.cu — the pieces of a P x Q (P > 1) block-cyclic HPL step that differ
// from the 1 x Q driver: the panel's rows are spread over the P ranks of a
// process column, so the pivot search of every panel column becomes a
// candidate exchange (one all-gather of small records along the process
// column, issued by the host between oz_dpanel_candidate and
// oz_dpanel_apply), and the interchanges of the other columns move rows
// between ranks (oz_gather_rows / oz_scatter_rows around a broadcast).
//
// The panel arithmetic is the reference's unblocked loop (solve.py:66-91)
// element for element: first maximum of |col| (smallest global row on ties),
// row swap, division by the pivot, and the outer-product update with
// separately rounded product and difference (np.outer then -=).
//
// Local rows of process row p are global rows ((lr / nb) * P + p) * nb + lr % nb,
// stored in increasing global order, so "global rows >= g" is a suffix of the
// local rows.
#include "common.cuh"

namespace oz {
namespace {

constexpr int DP_THREADS = 1024;
// record: [0] |v| of the local candidate (-1: no local rows), [1] its global
// row, [2] 1 if this rank owns row g, [3, 3+jb) candidate row (panel
// columns), [3+jb, 3+2jb) row g (when owned)
constexpr int REC_HDR = 3;

__device__ __forceinline__ int64_t local_to_global(int64_t lr, int64_t nb, int64_t P, int64_t p) {
  return ((lr / nb) * P + p) * nb + lr % nb;
}

__global__ void __launch_bounds__(DP_THREADS)
dpanel_candidate_kernel(const double* __restrict__ a, int64_t lda, int64_t lr0, int64_t mloc,
                        int t, int jb, int owns_g, int64_t nb, int64_t P, int64_t p,
                        double* __restrict__ rec) {
  __shared__ double sv[DP_THREADS / 32];
  __shared__ int64_t si[DP_THREADS / 32];
  __shared__ int64_t best_lr;
  const double* col = a + (int64_t)t * lda;
  double bv = -1.0;
  int64_t bi = INT64_MAX;
  for (int64_t r = lr0 + threadIdx.x; r < mloc; r += DP_THREADS) {
    const double v = fabs(col[r]);
    if (v > bv) { bv = v; bi = r; }          // rows ascend per thread: first max kept
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
    const int64_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
  }
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) { sv[w] = bv; si[w] = bi; }
  __syncthreads();
  if (w == 0) {
    bv = sv[l];
    bi = si[l];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int64_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
    }
    if (l == 0) {
      best_lr = bi;
      rec[0] = bi == INT64_MAX ? -1.0 : bv;
      rec[1] = bi == INT64_MAX ? -1.0 : (double)local_to_global(bi, nb, P, p);
      rec[2] = owns_g ? 1.0 : 0.0;
    }
  }
  __syncthreads();
  const int64_t br = best_lr;
  for (int c = threadIdx.x; c < jb; c += DP_THREADS) {
    rec[REC_HDR + c] = br == INT64_MAX ? 0.0 : a[br + (int64_t)c * lda];
    rec[REC_HDR + jb + c] = owns_g ? a[lr0 + (int64_t)c * lda] : 0.0;
  }
}

// winner over the P gathered records: largest |v|, then smallest global row
__device__ __forceinline__ int pick_winner(const double* recs, int P, int rlen) {
  int w = 0;
  for (int r = 1; r < P; ++r) {
    const double v = recs[(int64_t)r * rlen], bv = recs[(int64_t)w * rlen];
    if (v > bv || (v == bv && v >= 0.0 && recs[(int64_t)r * rlen + 1] < recs[(int64_t)w * rlen + 1]))
      w = r;
  }
  return w;
}

__device__ __forceinline__ int find_g_owner(const double* recs, int P, int rlen) {
  for (int r = 0; r < P; ++r)
    if (recs[(int64_t)r * rlen + 2] != 0.0) return r;
  return 0;
}

// swap rows g and the pivot row inside the panel columns; ipiv[t] <- pivot row
__global__ void dpanel_swap_kernel(double* __restrict__ a, int64_t lda, int64_t lr0, int t,
                                   int jb, int64_t g, int owns_g, int64_t nb, int64_t Pg,
                                   int64_t p, const double* __restrict__ recs, int P,
                                   int32_t* __restrict__ ipiv, int32_t* __restrict__ info) {
  const int rlen = REC_HDR + 2 * jb;
  const int w = pick_winner(recs, P, rlen);
  const double* rw = recs + (int64_t)w * rlen;
  const double* rg = recs + (int64_t)find_g_owner(recs, P, rlen) * rlen;
  const int64_t piv = (int64_t)rw[1];
  if (threadIdx.x == 0) {
    ipiv[t] = (int32_t)piv;
    if (rw[REC_HDR + t] == 0.0 && *info == 0) *info = (int32_t)(g + 1);
  }
  if (piv == g) return;
  const bool owns_piv = ((piv / nb) % Pg) == p;
  const int64_t lrp = ((piv / nb) / Pg) * nb + piv % nb;
  for (int c = threadIdx.x; c < jb; c += blockDim.x) {
    if (owns_g) a[lr0 + (int64_t)c * lda] = rw[REC_HDR + c];
    if (owns_piv) a[lrp + (int64_t)c * lda] = rg[REC_HDR + jb + c];
  }
}

// rows below g: l = a / pivot; a[:, c] -= l * u[c] for c in (t, jb)
__global__ void dpanel_update_kernel(double* __restrict__ a, int64_t lda, int64_t r0,
                                     int64_t mloc, int t, int jb,
                                     const double* __restrict__ recs, int P,
                                     unsigned long long* __restrict__ growth_bits) {
  const int rlen = REC_HDR + 2 * jb;
  const double* rw = recs + (int64_t)pick_winner(recs, P, rlen) * rlen;
  const double pv = rw[REC_HDR + t];
  const int64_t r = r0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  double seen = 0.0;
  if (r < mloc && pv != 0.0) {
    const double lv = a[r + (int64_t)t * lda] / pv;
    a[r + (int64_t)t * lda] = lv;
    for (int c = t + 1; c < jb; ++c) {
      const double v = __dsub_rn(a[r + (int64_t)c * lda], __dmul_rn(lv, rw[REC_HDR + c]));
      a[r + (int64_t)c * lda] = v;
      seen = fmax(seen, fabs(v));
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) seen = fmax(seen, __shfl_xor_sync(0xffffffffu, seen, o));
  if ((threadIdx.x & 31) == 0 && seen > 0.0)
    atomicMax(growth_bits, (unsigned long long)__double_as_longlong(seen));
}

__global__ void rows_copy_kernel(double* __restrict__ a, int64_t lda,
                                 const int32_t* __restrict__ rows, int64_t nrows, int64_t c0a,
                                 int64_t c1a, int64_t c0b, int64_t c1b, double* __restrict__ buf,
                                 const int32_t* __restrict__ brows, int64_t ldb, int scatter) {
  const int64_t na = c1a - c0a, ncols = na + (c1b - c0b);
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= nrows * ncols) return;
  const int64_t i = idx % nrows, cc = idx / nrows;
  const int64_t c = cc < na ? c0a + cc : c0b + (cc - na);
  double* ap = a + rows[i] + c * lda;
  double* bp = buf + (brows ? brows[i] : i) + cc * ldb;
  if (scatter) *ap = *bp; else *bp = *ap;
}

__global__ void scatter_vec_kernel(const double* __restrict__ src, int64_t lr0, int64_t cnt,
                                   int64_t nb, int64_t P, int64_t p, double* __restrict__ dst) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < cnt) dst[local_to_global(lr0 + i, nb, P, p)] = src[i];
}

// dst[i + c*ldd] = src[blk[i]*src_block + c*src_ld + row[i]]: rows picked
// from P stacked column-major blocks (the all-gathered panel slabs of a
// process column) into one matrix in global row order, or (blk = null) a
// plain row gather; one thread per element, coalesced on the dst rows.
__global__ void assemble_rows_kernel(const double* __restrict__ src, int64_t src_ld,
                                     int64_t src_block, const int32_t* __restrict__ blk,
                                     const int32_t* __restrict__ row, int64_t nrows,
                                     double* __restrict__ dst, int64_t ldd) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t c = blockIdx.y;
  if (i >= nrows) return;
  const int64_t b = blk ? blk[i] : 0;
  dst[i + c * ldd] = src[b * src_block + c * src_ld + row[i]];
}

}  // namespace
}  // namespace oz

extern "C" int oz_dpanel_candidate(const double* a, int64_t lda, int64_t lr0, int64_t mloc,
                                   int t, int jb, int owns_g, int64_t nb, int64_t P, int64_t p,
                                   double* rec, void* stream) {
  using namespace oz;
  OZ_REQUIRE(jb >= 1 && t >= 0 && t < jb && nb >= 1 && P >= 1 && p >= 0 && p < P && lr0 >= 0,
             OZ_INVALID_PARAMS, "bad distributed panel arguments");
  dpanel_candidate_kernel<<<1, DP_THREADS, 0, as_stream(stream)>>>(a, lda, lr0, mloc, t, jb,
                                                                   owns_g, nb, P, p, rec);
  OZ_CHECK_LAUNCH();
  return OZ_OK;
}

extern "C" int oz_dpanel_apply(double* a, int64_t lda, int64_t lr0, int64_t mloc, int t, int jb,
                               int64_t g, int owns_g, int64_t nb, int64_t P, int64_t p,
                               const double* recs, int32_t* ipiv, int32_t* info,
                               unsigned long long* growth_bits, void* stream) {
  using namespace oz;
  OZ_REQUIRE(jb >= 1 && t >= 0 && t < jb && nb >= 1 && P >= 1 && p >= 0 && p < P && lr0 >= 0,
             OZ_INVALID_PARAMS, "bad distributed panel arguments");
  cudaStream_t st = as_stream(stream);
  dpanel_swap_kernel<<<1, 256, 0, st>>>(a, lda, lr0, t, jb, g, owns_g, nb, P, p, recs, (int)P,
                                        ipiv, info);
  OZ_CHECK_LAUNCH();
  const int64_t r0 = lr0 + (owns_g ? 1 : 0);
  if (mloc > r0) {
    dpanel_update_kernel<<<(unsigned)ceil_div(mloc - r0, 256), 256, 0, st>>>(
        a, lda, r0, mloc, t, jb, recs, (int)P, growth_bits);
    OZ_CHECK_LAUNCH();
  }
  return OZ_OK;
}

static int rows_copy(double* a, int64_t lda, const int32_t* rows, int64_t nrows, int64_t c0a,
                     int64_t c1a, int64_t c0b, int64_t c1b, double* buf, const int32_t* brows,
                     int64_t ldb, int scatter, void* stream) {
  using namespace oz;
  OZ_REQUIRE(c0a <= c1a && c0b <= c1b && ldb >= 1, OZ_INVALID_PARAMS, "bad column ranges");
  const int64_t total = nrows * ((c1a - c0a) + (c1b - c0b));
  if (total <= 0) return OZ_OK;
  rows_copy_kernel<<<(unsigned)ceil_div(total, 256), 256, 0, as_stream(stream)>>>(
      a, lda, rows, nrows, c0a, c1a, c0b, c1b, buf, brows, ldb, scatter);
  OZ_CHECK_LAUNCH();
  return OZ_OK;
}

extern "C" int oz_gather_rows(const double* a, int64_t lda, const int32_t* rows, int64_t nrows,
                              int64_t c0a, int64_t c1a, int64_t c0b, int64_t c1b, double* buf,
                              const int32_t* buf_rows, int64_t ldb, void* stream) {
  return rows_copy(const_cast<double*>(a), lda, rows, nrows, c0a, c1a, c0b, c1b, buf, buf_rows,
                   ldb, 0, stream);
}

extern "C" int oz_scatter_rows(double* a, int64_t lda, const int32_t* rows, int64_t nrows,
                               int64_t c0a, int64_t c1a, int64_t c0b, int64_t c1b,
                               const double* buf, const int32_t* buf_rows, int64_t ldb,
                               void* stream) {
  return rows_copy(a, lda, rows, nrows, c0a, c1a, c0b, c1b, const_cast<double*>(buf), buf_rows,
                   ldb, 1, stream);
}

extern "C" int oz_scatter_vec(const double* src, int64_t lr0, int64_t count, int64_t nb,
                              int64_t P, int64_t p, double* dst, void* stream) {
  using namespace oz;
  OZ_REQUIRE(nb >= 1 && P >= 1 && p >= 0 && p < P, OZ_INVALID_PARAMS, "bad row map");
  if (count <= 0) return OZ_OK;
  scatter_vec_kernel<<<(unsigned)ceil_div(count, 256), 256, 0, as_stream(stream)>>>(
      src, lr0, count, nb, P, p, dst);
  OZ_CHECK_LAUNCH();
  return OZ_OK;
}

extern "C" int oz_assemble_rows(const double* src, int64_t src_ld, int64_t src_block,
                                const int32_t* blk, const int32_t* row, int64_t nrows,
                                int64_t ncols, double* dst, int64_t ldd, void* stream) {
  using namespace oz;
  OZ_REQUIRE(nrows >= 0 && ncols >= 0 && ncols <= 65535 && ldd >= nrows, OZ_INVALID_PARAMS,
             "bad row-assembly shape");
  if (nrows == 0 || ncols == 0) return OZ_OK;
  dim3 grid((unsigned)ceil_div(nrows, 256), (unsigned)ncols);
  assemble_rows_kernel<<<grid, 256, 0, as_stream(stream)>>>(src, src_ld, src_block, blk, row,
                                                            nrows, dst, ldd);
  OZ_CHECK_LAUNCH();
  return OZ_OK;
}
