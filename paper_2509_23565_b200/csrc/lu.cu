// lu.cu — K7..K12 of SURVEY §2.2: the FP64 side of the HPL-style LU.
//
// Reference: /root/reference/pkg/src/ozemu/solve.py
//   _panel_factor  :66-91   partial pivoting (first max wins ties), whole-row
//                           swaps, column DIVIDED by the pivot, rank-1 update
//                           as outer product then subtraction (no FMA)
//   lu_factor      :94-140  blocked right-looking: panel, trsm (unit lower),
//                           Schur update through the GEMM backend, growth
//   lu_solve       :143-156 perm gather, unit-lower then upper substitution
//   scaled_residual:181-214 ||Ax-b|| / ((||A|| ||x|| + ||b||) n eps)
//
// Storage is column-major (LAPACK/HPL order) with leading dimension lda.
//
// Panel design: the nb-wide panel is factored in windows of w <= 64 columns.
// Each window runs as ONE cooperative persistent kernel: every CTA keeps a
// slab of rows x w columns resident in shared memory for all w column steps;
// per step the CTAs publish their best pivot candidate (|value|, position,
// row data) to global memory, meet at a single grid barrier, and all reduce
// the candidates identically.  Rows never move inside the kernel — each row
// keeps a logical position, and the interchanges are applied afterwards by a
// gather (compose_swaps + laswp_gather), which turns LAPACK's sequential
// interchanges into one read-all/write-all pass per column.  The rest of the
// panel is updated with trsm + cuBLAS DGEMM; the Schur update is cuBLAS DGEMM
// (native comparator) or the Ozaki-INT8 tcgen05 GEMM (gemm_emu.cu).
#include <stdlib.h>
#include <algorithm>
#include <atomic>
#include <mutex>
#include <vector>

#include "common.cuh"

namespace oz {

// Temporary buffers of the residual / row-sum paths come from the device's
// default stream-ordered pool; keep its memory mapped between calls instead
// of returning it to the driver at every synchronization.
void keep_pool_mapped() {
  static const bool done = [] {
    int dev = 0;
    cudaMemPool_t pool;
    if (cudaGetDevice(&dev) == cudaSuccess &&
        cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t keep = ~0ull;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    cudaGetLastError();
    return true;
  }();
  (void)done;
}

}  // namespace oz

namespace oz {

int dtrsm_lunit(int64_t jb, int64_t n, const double* l, int64_t ldl, double* b, int64_t ldb,
                cudaStream_t st, int sm_target);
int dgemm(int transa, int transb, int64_t m, int64_t n, int64_t k, double alpha, const double* a,
          int64_t lda, const double* b, int64_t ldb, double beta, double* c, int64_t ldc,
          cudaStream_t st, int sm_target = 0);
int split_launch(const double* src, int64_t rows, int64_t cols, int64_t row_stride,
                 int64_t col_stride, int orientation, int mode, int k, int q, int8_t* slices,
                 int64_t slice_ld, int64_t slice_stride, int32_t* exps, void* aux_v,
                 cudaStream_t st);
int gemm_emu_launch(int64_t m, int64_t n, int64_t inner, const int8_t* a_slices, int64_t a_ld,
                    int64_t a_sstride, int a_nslices, const int32_t* a_exps,
                    const int8_t* b_slices, int64_t b_ld, int64_t b_sstride, int b_nslices,
                    const int32_t* b_exps, int npairs, const int32_t* pair_a,
                    const int32_t* pair_b, const int32_t* pair_shift, int slice_bits,
                    double alpha, double beta, double* c, int64_t ldc, int c_is_input,
                    unsigned long long* growth, cudaStream_t st, int max_ctas);

namespace {

constexpr int PANEL_W = 64;  // max window width
constexpr int PANEL_THREADS = 256;
constexpr int PANEL_WARPS = PANEL_THREADS / 32;
constexpr int CAND_STRIDE = 4 + PANEL_W;  // doubles per candidate record
constexpr int TRSM_W = 64;                // diagonal block of the blocked trsm
constexpr int SWAP_MAX = 2048;            // max entries of a composed swap list (2*nb)

// ------------------------------------------------------------------ grid barrier
struct GridBar {
  unsigned count;  // arrivals; reset before every window launch
  unsigned pad;
};

// np.argmax(|col|) order: larger magnitude wins, ties -> smaller logical position;
// NaN counts as the maximum (numpy returns the first NaN).
__device__ __forceinline__ bool better(double a1, int p1, double a2, int p2) {
  const bool n1 = isnan(a1), n2 = isnan(a2);
  if (n1 || n2) return n1 && (!n2 || p1 < p2);
  return a1 > a2 || (a1 == a2 && p1 < p2);
}

// Warp-wide argmax in better() order with integer reductions instead of a
// 5-round shuffle tree: the order-preserving bits of |v| (NaN canonical,
// "no candidate" (a < 0) as 0 with position INT_MAX), then the smallest
// position among the maxima.  Every lane returns the winner (a, p, r).
__device__ __forceinline__ void warp_argmax(double& a, int& p, int& r) {
  const unsigned long long b =
      a < 0.0 ? 0ull
              : (isnan(a) ? 0x7ff8000000000000ull : (unsigned long long)__double_as_longlong(a));
  const unsigned hi = (unsigned)(b >> 32), lo = (unsigned)b;
  const unsigned mhi = __reduce_max_sync(0xffffffffu, hi);
  const unsigned mlo = __reduce_max_sync(0xffffffffu, hi == mhi ? lo : 0u);
  const bool top = hi == mhi && lo == mlo;
  const int mp = __reduce_min_sync(0xffffffffu, top ? p : 0x7fffffff);
  const int src = __ffs(__ballot_sync(0xffffffffu, top && p == mp)) - 1;
  a = __shfl_sync(0xffffffffu, a, src);
  r = __shfl_sync(0xffffffffu, r, src);
  p = mp;
}

struct PanelArgs {
  double* a;
  int64_t lda;
  int64_t r0;    // first row (== first column of the window), relative to a's panel origin
  int64_t m;     // rows r0..r0+m-1
  int64_t base;  // global row index of the panel origin (ipiv values and info are global)
  int w;       // window width (<= PANEL_W)
  int rows_per_cta;
  int32_t* ipiv;
  unsigned long long* growth;
  int32_t* info;
  GridBar* bar;
  double* cand;  // [2][gridDim][CAND_STRIDE]
  int32_t* list_dst;  // gather list of this window's interchanges (rows outside
  int32_t* list_src;  // the window columns): new_row[dst] = old_row[src]
  int32_t* list_cnt;
  unsigned long long* dbg;  // optional per-phase cycle counters (OZ_PANEL_TIMING)
  unsigned epoch;           // grid variant: record tags of this launch are epoch + t + 1
};

__device__ __forceinline__ void st_release_u64(long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_u64(const long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
// candidate record: [0] |v| (double), [1] pos (low 32) | tag (high 32), [2] physical
// row, [4..4+w) row values.  Grid variant: data first, then the tag word by
// one release store; readers poll the tag word itself with acquire loads (no
// separate arrival counter: one round trip less per column).

constexpr int STAGE_G = 16;  // grids up to this size read every record in one round trip

struct PanelShared {
  double red_a[PANEL_WARPS];
  int red_p[PANEL_WARPS];
  int red_r[PANEL_WARPS];
  int occ[PANEL_W];
  int prow[PANEL_W];
  double urow[2][PANEL_W];  // pivot rows of steps t (buf) and t-1 (buf ^ 1)
  double stage[STAGE_G][CAND_STRIDE];
  double crec[2][CAND_STRIDE];  // cluster variant: this CTA's published record (DSMEM)
  int best;
};

unsigned long long* panel_dbg() {
  static unsigned long long* const dbg = [] {
    unsigned long long* d = nullptr;
    if (getenv("OZ_PANEL_TIMING") != nullptr) {  // tuning only
      cudaMalloc(&d, 8 * sizeof(unsigned long long));
      cudaMemset(d, 0, 8 * sizeof(unsigned long long));
    }
    return d;
  }();
  return dbg;
}

size_t panel_smem_bytes(int w, int R) {
  return (size_t)w * R * sizeof(double) + (size_t)R * sizeof(int);
}

__device__ __forceinline__ void cluster_arrive_release() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait_acquire() {
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ double ld_dsmem(const void* local, unsigned rank) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(local);
  unsigned ra;
  double v;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(rank));
  asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(ra) : "memory");
  return v;
}

// One window of the panel: solve.py:75-90 for columns r0..r0+w-1 over rows r0..
// kCluster = false: G co-resident CTAs (cooperative launch) exchange candidate
// records through global memory and a release/acquire counter; kCluster =
// true: the G CTAs form one thread-block cluster, each publishes its record in
// its own shared memory and a cluster barrier (arrive.release / wait.acquire)
// replaces the counter, so one column's exchange costs ~1 us instead of ~3.
template <bool kCluster>
__global__ void __launch_bounds__(PANEL_THREADS, 1) panel_window_kernel(PanelArgs p) {
  extern __shared__ double sm[];  // slab [w][R] column-major, then pos[R]
  __shared__ PanelShared sh;
  const int R = p.rows_per_cta;
  const int w = p.w;
  const int64_t row_lo = (int64_t)blockIdx.x * R;
  const int nloc = (int)max((int64_t)0, min((int64_t)R, p.m - row_lo));
  int* pos = reinterpret_cast<int*>(sm + (size_t)w * R);  // logical position; -1 = pivot used
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  double* abase = p.a + p.r0 * p.lda + p.r0 + row_lo;

  for (int c = 0; c < w; ++c)
    for (int r = tid; r < nloc; r += PANEL_THREADS) sm[c * R + r] = abase[c * p.lda + r];
  for (int r = tid; r < nloc; r += PANEL_THREADS) pos[r] = (int)(row_lo + r);
  for (int i = tid; i < PANEL_W; i += PANEL_THREADS) sh.occ[i] = i;
  __syncthreads();

  double gmax = 0.0;
  for (int i = tid; i < nloc * w; i += PANEL_THREADS) {
    const int c = i / nloc, r = i - c * nloc;
    gmax = fmax(gmax, fabs(sm[c * R + r]));
  }

  // thread-local candidate for the current column (values after the last update)
  double ca = -1.0;
  int cp = 0x7fffffff, cr = -1;
  for (int r = tid; r < nloc; r += PANEL_THREADS) {
    const double v = fabs(sm[r]);
    if (better(v, pos[r], ca, cp)) {
      ca = v;
      cp = pos[r];
      cr = r;
    }
  }

  if (kCluster) {  // every CTA of the cluster is running before any DSMEM access
    cluster_arrive_release();
    cluster_wait_acquire();
  }
  long long _tp = clock64();
  const bool staged = kCluster || gridDim.x <= STAGE_G;
  for (int t = 0; t < w; ++t) {
    const int buf = t & 1;
    double* urow = sh.urow[buf];
    const double* uprev = sh.urow[buf ^ 1];
    // ---- block argmax of the thread candidates (np.argmax order)
    warp_argmax(ca, cp, cr);
    if (lane == 0) {
      sh.red_a[wid] = ca;
      sh.red_p[wid] = cp;
      sh.red_r[wid] = cr;
    }
    __syncthreads();
    if (wid == 0) {
      double ba = lane < PANEL_WARPS ? sh.red_a[lane] : -2.0;
      int bp = lane < PANEL_WARPS ? sh.red_p[lane] : 0x7fffffff;
      int br = lane < PANEL_WARPS ? sh.red_r[lane] : -1;
      warp_argmax(ba, bp, br);
      // ---- publish the CTA's candidate record, then arrive on the step counter.
      // Step t-1's update of columns > t is deferred (below), so the
      // candidate row's values there are formed here with the same
      // product-then-subtract the deferred update will store.
      double* rec = kCluster ? sh.crec[buf]
                             : p.cand + ((size_t)buf * gridDim.x + blockIdx.x) * CAND_STRIDE;
      long long* irec = reinterpret_cast<long long*>(rec);
      if (br >= 0) {
        const double lp = t > 0 ? sm[(t - 1) * R + br] : 0.0;
        for (int c = t + lane; c < w; c += 32) {
          double v = sm[c * R + br];
          if (t > 0 && c > t) v = __dsub_rn(v, __dmul_rn(lp, uprev[c]));
          rec[4 + c] = v;
        }
      }
      const unsigned posw = br >= 0 ? (unsigned)pos[br] : 0x7fffffffu;
      if (lane == 0) {
        rec[0] = br >= 0 ? fabs(sm[t * R + br]) : -1.0;
        if (kCluster) irec[1] = posw;
        irec[2] = br >= 0 ? row_lo + br : -1;
      }
      // the warp's record stores are ordered before lane 0's release store of
      // the tag word by the warp barrier (one release instead of a GPU-scope
      // fence per lane)
      __syncwarp();
      if (!kCluster && lane == 0)
        st_release_u64(&irec[1], ((unsigned long long)(p.epoch + (unsigned)t + 1u) << 32) | posw);
      if (p.dbg && lane == 0) { const long long _n = clock64(); atomicAdd(p.dbg + 0, (unsigned long long)(_n - _tp)); _tp = _n; }
    }
    __syncthreads();  // the publish above read row br before the deferred update below
    if (kCluster) cluster_arrive_release();  // publishes sh.crec[buf] to the cluster
    // ---- while the other CTAs arrive: step t-1's update of columns t+1..w-1
    //      (column t was updated before the argmax).  pos[] is unchanged
    //      since that step, so the same rows are updated.
    if (t > 0) {
      for (int r = tid; r < nloc; r += PANEL_THREADS) {
        if (pos[r] < 0) continue;
        const double l = sm[(t - 1) * R + r];
        int c = t + 1;
        // batches of 8: all loads issued before the dependent math and the
        // stores (the compiler cannot reorder shared loads past shared
        // stores it cannot disambiguate), max over a shallow tree
        for (; c + 8 <= w; c += 8) {
          double x[8], u[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            x[i] = sm[(c + i) * R + r];
            u[i] = uprev[c + i];
          }
#pragma unroll
          for (int i = 0; i < 8; ++i) x[i] = __dsub_rn(x[i], __dmul_rn(l, u[i]));
#pragma unroll
          for (int i = 0; i < 8; ++i) sm[(c + i) * R + r] = x[i];
          const double m01 = fmax(fabs(x[0]), fabs(x[1])), m23 = fmax(fabs(x[2]), fabs(x[3]));
          const double m45 = fmax(fabs(x[4]), fabs(x[5])), m67 = fmax(fabs(x[6]), fabs(x[7]));
          gmax = fmax(gmax, fmax(fmax(m01, m23), fmax(m45, m67)));
        }
        for (; c < w; ++c) {
          const double x = __dsub_rn(sm[c * R + r], __dmul_rn(l, uprev[c]));
          sm[c * R + r] = x;
          gmax = fmax(gmax, fabs(x));
        }
      }
    }
    if (p.dbg && tid == 0) { const long long _n = clock64(); atomicAdd(p.dbg + 4, (unsigned long long)(_n - _tp)); _tp = _n; }
    // ---- wait for all CTAs: the cluster barrier, or (grid) every record's
    //      tag word of this step, polled by warp 0 (lane l: CTAs l, l+32, ..)
    const unsigned tag = p.epoch + (unsigned)t + 1u;
    const double* recs = p.cand + (size_t)buf * gridDim.x * CAND_STRIDE;
    if (kCluster) {
      cluster_wait_acquire();
    } else if (staged) {
      if (wid == 0 && lane < (int)gridDim.x) {
        const long long* tw = reinterpret_cast<const long long*>(recs + (size_t)lane * CAND_STRIDE) + 1;
        while ((unsigned)(ld_acquire_u64(tw) >> 32) != tag) {
        }
      }
      __syncthreads();
    }
    if (p.dbg && tid == 0) { const long long _n = clock64(); atomicAdd(p.dbg + 1, (unsigned long long)(_n - _tp)); _tp = _n; }
    if (staged) {
      // small grids: the whole record array in one round trip, all threads
      constexpr int LOADS = (STAGE_G * CAND_STRIDE + PANEL_THREADS - 1) / PANEL_THREADS;
      const int total = (int)gridDim.x * CAND_STRIDE;
      double v[LOADS];
#pragma unroll
      for (int i = 0; i < LOADS; ++i) {
        const int e = tid + i * PANEL_THREADS;
        if (kCluster) {
          const int g = e / CAND_STRIDE;
          v[i] = e < total ? ld_dsmem(&sh.crec[buf][e - g * CAND_STRIDE], (unsigned)g) : 0.0;
        } else {
          v[i] = e < total ? __ldcg(recs + e) : 0.0;
        }
      }
#pragma unroll
      for (int i = 0; i < LOADS; ++i) {
        const int e = tid + i * PANEL_THREADS;
        if (e < total) (&sh.stage[0][0])[e] = v[i];
      }
      __syncthreads();
    }
    if (wid == 0) {
      double ba = -2.0;
      int bp = 0x7fffffff;
      int bg = 0;
      if (staged) {
        if (lane < (int)gridDim.x) {
          ba = sh.stage[lane][0];
          bp = (int)reinterpret_cast<const long long*>(sh.stage[lane])[1];
          bg = lane;
        }
      } else {
        constexpr int PER = 5;  // up to 160 CTAs
        double av[PER];
        long long pk[PER];
#pragma unroll
        for (int i = 0; i < PER; ++i) {
          const int g = lane + 32 * i;
          const double* cr_ = recs + (size_t)g * CAND_STRIDE;
          unsigned long long w = 0x7fffffffull;
          if (g < (int)gridDim.x) {
            const long long* tw = reinterpret_cast<const long long*>(cr_) + 1;
            do {
              w = ld_acquire_u64(tw);
            } while ((unsigned)(w >> 32) != tag);
          }
          pk[i] = (long long)(w & 0xffffffffull);
          av[i] = g < (int)gridDim.x ? __ldcg(cr_) : -2.0;
        }
        // every lane's acquire precedes the warp's reads of the winner's row
        __syncwarp();
#pragma unroll
        for (int i = 0; i < PER; ++i) {
          if (lane + 32 * i >= (int)gridDim.x) continue;
          if (better(av[i], (int)pk[i], ba, bp)) {
            ba = av[i];
            bp = (int)pk[i];
            bg = lane + 32 * i;
          }
        }
      }
      warp_argmax(ba, bp, bg);
      if (p.dbg && lane == 0) { const long long _n = clock64(); atomicAdd(p.dbg + 2, (unsigned long long)(_n - _tp)); _tp = _n; }
      // ---- winner's row (the new U row) and interchange bookkeeping
      const double* win = staged ? sh.stage[bg] : recs + (size_t)bg * CAND_STRIDE;
      for (int c = t + lane; c < w; c += 32) urow[c] = staged ? win[4 + c] : __ldcg(win + 4 + c);
      if (lane == 0) {
        const int ppos = staged ? (int)reinterpret_cast<const long long*>(win)[1]
                                : (int)(unsigned)__ldcg(reinterpret_cast<const long long*>(win) + 1);
        const int64_t prow = staged ? reinterpret_cast<const long long*>(win)[2]
                                    : __ldcg(reinterpret_cast<const long long*>(win) + 2);
        const double pv = staged ? win[4 + t] : __ldcg(win + 4 + t);
        const int rt = sh.occ[t];  // relative physical row currently at position t
        if (blockIdx.x == 0) {
          p.ipiv[p.r0 + t] = (int32_t)(p.base + p.r0 + ppos);
          if (pv == 0.0)
            atomicCAS(reinterpret_cast<int*>(p.info), 0, (int)(p.base + p.r0 + t + 1));
          sh.prow[t] = (int)prow;
        }
        // solve.py:80-82: the pivot row is final; the row at position t takes
        // the pivot's old position
        if (prow >= row_lo && prow < row_lo + nloc) pos[prow - row_lo] = -(t + 1);
        if (rt != prow) {
          if (rt >= row_lo && rt < row_lo + nloc) pos[rt - row_lo] = ppos;
          if (ppos < PANEL_W) sh.occ[ppos] = rt;
        }
      }
      if (p.dbg && lane == 0) { const long long _n = clock64(); atomicAdd(p.dbg + 3, (unsigned long long)(_n - _tp)); _tp = _n; }
    }
    __syncthreads();
    // ---- column scaling by DIVISION (solve.py:84) and the rank-1 update
    //      (:86, np.outer then -=) of column t+1 only, tracking the next
    //      column's candidate; columns t+2.. follow after the next publish
    const double piv = urow[t];
    ca = -1.0;
    cp = 0x7fffffff;
    cr = -1;
    for (int r = tid; r < nloc; r += PANEL_THREADS) {
      const int pr = pos[r];
      if (pr < 0) continue;
      const double l = sm[t * R + r] / piv;
      sm[t * R + r] = l;
      const int c = t + 1;
      if (c < w) {
        const double x = __dsub_rn(sm[c * R + r], __dmul_rn(l, urow[c]));
        sm[c * R + r] = x;
        const double ax = fabs(x);
        gmax = fmax(gmax, ax);
        if (better(ax, pr, ca, cp)) {
          ca = ax;
          cp = pr;
          cr = r;
        }
      }
    }
    if (p.dbg && tid == 0) { const long long _n = clock64(); atomicAdd(p.dbg + 5, (unsigned long long)(_n - _tp)); _tp = _n; }
  }
  __syncthreads();
  // rows go straight to their final positions (pivot row of step t -> t,
  // displaced row -> its logical position); every moved row is listed so the
  // same interchanges can be applied to the other columns by a gather.
  double* wbase = p.a + p.r0 * p.lda + p.r0;
  for (int r = tid; r < nloc; r += PANEL_THREADS) {
    const int ps = pos[r];
    const int fin = ps < 0 ? -ps - 1 : ps;
    const int phys = (int)(row_lo + r);
    for (int c = 0; c < w; ++c) wbase[c * p.lda + fin] = sm[c * R + r];
    if (fin != phys) {
      const int slot = atomicAdd(p.list_cnt, 1);
      p.list_dst[slot] = (int32_t)(p.r0 + fin);
      p.list_src[slot] = (int32_t)(p.r0 + phys);
    }
  }
  if (p.growth) {
    gmax = warp_max(gmax);
    if (lane == 0 && gmax > 0.0) atomic_max_abs(p.growth, gmax);
  }
  if (kCluster) {  // no CTA leaves while others may still read its records
    cluster_arrive_release();
    cluster_wait_acquire();
  }
}

#include "panel_leaf.cuh"

// Apply a gather list (<= 2*PANEL_W entries) to columns [c0a,c1a) U [c0b,c1b):
// one warp per column, entries staged in registers (read all, then write).
constexpr int LIST_PER_LANE = (2 * PANEL_W + 31) / 32;
__global__ void laswp_gather_kernel(double* __restrict__ a, int64_t lda, const int32_t* dst,
                                    const int32_t* src, const int32_t* count, int64_t c0a,
                                    int64_t c1a, int64_t c0b, int64_t c1b) {
  const int cnt = *count;
  if (cnt == 0) return;
  const int lane = threadIdx.x & 31;
  int d[LIST_PER_LANE], sidx[LIST_PER_LANE];
#pragma unroll
  for (int i = 0; i < LIST_PER_LANE; ++i) {
    const int e = lane + 32 * i;
    d[i] = e < cnt ? dst[e] : -1;
    sidx[i] = e < cnt ? src[e] : 0;
  }
  const int64_t na = c1a - c0a, nbb = c1b - c0b;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t ci = warp; ci < na + nbb; ci += nwarps) {
    const int64_t col = ci < na ? c0a + ci : c0b + (ci - na);
    double* colp = a + col * lda;
    double v[LIST_PER_LANE];
#pragma unroll
    for (int i = 0; i < LIST_PER_LANE; ++i) v[i] = d[i] >= 0 ? colp[sidx[i]] : 0.0;
    __syncwarp();
#pragma unroll
    for (int i = 0; i < LIST_PER_LANE; ++i)
      if (d[i] >= 0) colp[d[i]] = v[i];
  }
}

// LAPACK-style sequential interchanges -> one gather list.  ipiv[t] (global
// row, >= k1 + t) is the row swapped with row k1 + t, applied in order
// t = 0..npiv-1 (solve.py:80-82 / dlaswp); the list holds (dst, src) pairs
// meaning new_row[dst] = old_row[src].
constexpr int COMPOSE_MAX = 1024;     // max interchanges per list (panel width)
// One thread per interchange, no serial replay (was one thread replaying the
// swaps on an index map: 80 us per panel on the critical chain, now 11 us).
// With p_t = ipiv[t] - k1 >= t: position t is final after step t and then
// holds what position p_t held just before step t.  Position q is touched
// before step t only as the far row of earlier steps, so it held
// H(s*) for the last s* < t with p_s* = q (q itself if none), where H(s) —
// the content of position s just before step s — is H(last s' < s with
// p_s' = s), or s: a chain resolved by pointer jumping.  Rows below the
// block end up with H(last s with p_s = q).
__global__ void __launch_bounds__(COMPOSE_MAX) compose_ipiv_kernel(
    const int32_t* __restrict__ ipiv, int npiv, int64_t k1, int32_t* dst, int32_t* src,
    int32_t* cnt) {
  __shared__ int32_t p[COMPOSE_MAX];
  __shared__ int32_t prev_top[COMPOSE_MAX];  // last s' < s with p_s' == s, or -1
  __shared__ int32_t hv[COMPOSE_MAX];        // H(s) once resolved
  __shared__ int32_t hp[COMPOSE_MAX];        // pointer-jumping link
  __shared__ int32_t has_next[COMPOSE_MAX];  // a later step has the same far row
  __shared__ int32_t prev_same[COMPOSE_MAX];  // last s < t with p_s == p_t, or -1
  __shared__ unsigned long long key[COMPOSE_MAX];
  __shared__ int32_t npos;
  const int t = threadIdx.x;
  if (t < npiv) {
    p[t] = (int)(ipiv[t] - k1);
    prev_top[t] = -1;
    has_next[t] = 0;
    prev_same[t] = -1;
  }
  // (p_t, t) sorted (bitonic, padded with max keys): equal rows become
  // neighbours in step order
  key[t] = t < npiv ? ((unsigned long long)(ipiv[t] - k1) << 11) | (unsigned)t : ~0ull;
  if (t == 0) npos = 0;
  // General interchanges (a row above its step, p_t < t, which getrf never
  // produces): one thread replays them on a content map instead
  if (__syncthreads_or(t < npiv && p[t] < t)) {
    if (t == 0) {
      int32_t* fpos = prev_same;  // far rows touched, and their contents
      int32_t* fval = has_next;
      int nf = 0;
      for (int i = 0; i < npiv; ++i) hv[i] = i;
      for (int s2 = 0; s2 < npiv; ++s2) {
        const int q = p[s2];
        int* cq;
        if (q >= 0 && q < npiv) {
          cq = &hv[q];
        } else {
          int f = 0;
          while (f < nf && fpos[f] != q) ++f;
          if (f == nf) {
            fpos[nf] = q;
            fval[nf++] = q;
          }
          cq = &fval[f];
        }
        const int v = hv[s2];
        hv[s2] = *cq;
        *cq = v;
      }
      int at = 0;
      for (int i = 0; i < npiv; ++i)
        if (hv[i] != i) {
          dst[at] = (int32_t)(k1 + i);
          src[at++] = (int32_t)(k1 + hv[i]);
        }
      for (int f = 0; f < nf; ++f)
        if (fval[f] != fpos[f]) {
          dst[at] = (int32_t)(k1 + fpos[f]);
          src[at++] = (int32_t)(k1 + fval[f]);
        }
      *cnt = at;
    }
    return;
  }
  if (t < npiv && p[t] < npiv && p[t] != t) atomicMax(&prev_top[p[t]], t);  // t < p_t
  for (int kk = 2; kk <= COMPOSE_MAX; kk <<= 1) {
    for (int jj = kk >> 1; jj > 0; jj >>= 1) {
      const int u = t ^ jj;
      if (u > t) {
        const unsigned long long x = key[t], y = key[u];
        if (((t & kk) == 0) == (x > y)) {
          key[t] = y;
          key[u] = x;
        }
      }
      __syncthreads();
    }
  }
  if (t > 0 && t < npiv) {
    const unsigned long long x = key[t], y = key[t - 1];
    if ((x >> 11) == (y >> 11)) {
      prev_same[(int)(x & 2047)] = (int)(y & 2047);
      has_next[(int)(y & 2047)] = 1;
    }
  }
  __syncthreads();
  const int sstar = t < npiv ? prev_same[t] : -1;
  if (t < npiv) {
    hp[t] = prev_top[t];
    hv[t] = t;
  }
  __syncthreads();
  for (int round = 0; round < 11; ++round) {  // 2^11 > COMPOSE_MAX
    int nv = 0, np = -1;
    if (t < npiv) {
      const int q = hp[t];
      nv = q >= 0 ? hv[q] : hv[t];
      np = q >= 0 ? hp[q] : -1;
    }
    __syncthreads();
    if (t < npiv) {
      hv[t] = nv;
      hp[t] = np;
    }
    __syncthreads();
  }
  if (t < npiv) {
    const int pt = p[t];
    const int f = sstar >= 0 ? hv[sstar] : pt;  // final content of position t
    if (f != t) {
      const int at = atomicAdd(&npos, 1);
      dst[at] = (int32_t)(k1 + t);
      src[at] = (int32_t)(k1 + f);
    }
    if (pt >= npiv && !has_next[t] && hv[t] != pt) {  // last step to touch row pt below
      const int at = atomicAdd(&npos, 1);
      dst[at] = (int32_t)(k1 + pt);
      src[at] = (int32_t)(k1 + hv[t]);
    }
  }
  __syncthreads();
  if (t == 0) *cnt = npos;
}

// Apply a gather list of up to 2*COMPOSE_MAX entries to columns [c0a,c1a) U
// [c0b,c1b): the list is staged once per CTA in shared memory; each warp owns
// one column at a time, reads every source row into its shared staging area,
// then writes every destination row (all reads before any write: cycles safe).
constexpr int LSWP_WARPS = 4;
constexpr int LSWP_MAX = 2 * COMPOSE_MAX;
constexpr size_t LSWP_SMEM = (size_t)LSWP_MAX * 2 * sizeof(int32_t) +
                             (size_t)LSWP_WARPS * LSWP_MAX * sizeof(double);
__global__ void __launch_bounds__(LSWP_WARPS * 32) laswp_list_kernel(
    double* __restrict__ a, int64_t lda, const int32_t* __restrict__ dst,
    const int32_t* __restrict__ src, const int32_t* __restrict__ count, int64_t c0a, int64_t c1a,
    int64_t c0b, int64_t c1b) {
  extern __shared__ uint8_t lsm[];
  int32_t* sd = reinterpret_cast<int32_t*>(lsm);
  int32_t* ss = sd + LSWP_MAX;
  const int cnt = *count;
  if (cnt == 0) return;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double* stage = reinterpret_cast<double*>(ss + LSWP_MAX) + (size_t)wid * LSWP_MAX;
  for (int e = threadIdx.x; e < cnt; e += blockDim.x) {
    sd[e] = dst[e];
    ss[e] = src[e];
  }
  __syncthreads();
  const int64_t na = c1a - c0a, nbb = c1b - c0b;
  for (int64_t ci = (int64_t)blockIdx.x * LSWP_WARPS + wid; ci < na + nbb;
       ci += (int64_t)gridDim.x * LSWP_WARPS) {
    const int64_t col = ci < na ? c0a + ci : c0b + (ci - na);
    double* colp = a + col * lda;
    // 8 independent scattered loads in flight per lane
    for (int e0 = lane; e0 < cnt; e0 += 32 * 8) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int e = e0 + 32 * u;
        v[u] = e < cnt ? colp[ss[e]] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int e = e0 + 32 * u;
        if (e < cnt) stage[e] = v[u];
      }
    }
    __syncwarp();
#pragma unroll 8
    for (int e = lane; e < cnt; e += 32) colp[sd[e]] = stage[e];
    __syncwarp();
  }
}

// Register variant: each warp holds one column's <= 2*COMPOSE_MAX source
// values in registers (64 per lane, all loads in flight at once), then writes
// the destinations.  No staging buffer, so 8 warps per CTA and one column's
// whole gather is a single memory round trip.
constexpr int LSWR_WARPS = 8;
constexpr int LSWR_PER_LANE = LSWP_MAX / 32;
__global__ void __launch_bounds__(LSWR_WARPS * 32, 1) laswp_list_reg_kernel(
    double* __restrict__ a, int64_t lda, const int32_t* __restrict__ dst,
    const int32_t* __restrict__ src, const int32_t* __restrict__ count, int64_t c0a, int64_t c1a,
    int64_t c0b, int64_t c1b) {
  __shared__ int32_t sd[LSWP_MAX];
  __shared__ int32_t ss[LSWP_MAX];
  const int cnt = *count;
  if (cnt == 0) return;
  for (int e = threadIdx.x; e < cnt; e += blockDim.x) {
    sd[e] = dst[e];
    ss[e] = src[e];
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t na = c1a - c0a, nbb = c1b - c0b;
  for (int64_t ci = (int64_t)blockIdx.x * LSWR_WARPS + wid; ci < na + nbb;
       ci += (int64_t)gridDim.x * LSWR_WARPS) {
    const int64_t col = ci < na ? c0a + ci : c0b + (ci - na);
    double* colp = a + col * lda;
    double v[LSWR_PER_LANE];
#pragma unroll
    for (int u = 0; u < LSWR_PER_LANE; ++u) {
      const int e = lane + 32 * u;
      v[u] = e < cnt ? colp[ss[e]] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < LSWR_PER_LANE; ++u) {
      const int e = lane + 32 * u;
      if (e < cnt) colp[sd[e]] = v[u];
    }
  }
}

// ---------------------------------------------------------------- small trsm
// B[0:w, c] <- L^{-1} B[0:w, c], L the unit-lower w x w block (w <= TRSM_W).
// One thread per right-hand-side column, the column held in registers, L in
// shared memory column by column (sLt[i][r] = L[r][i], so the update of rows
// i+1.. reads consecutive words: 16-byte broadcast loads, half the shared
// wavefronts of a row-major copy).  The L block and the 64 x TRSM_COLS tile of
// B arrive by cp.async (every load in flight at once; the tile is row-major
// with a one-word pad so the column-wise writes and the per-thread row reads
// are both conflict-free), and the result leaves through the same tile,
// coalesced along the columns.  Per element the order is b_r = fma(-l_ri,
// x_i, b_r) for i = 0, 1, ...: the sequential forward substitution.
constexpr int TRSM_COLS = 128;
constexpr int TRSM_LDX = TRSM_COLS + 1;
__global__ void __launch_bounds__(TRSM_COLS) trsm_unit_lower_kernel(
    const double* __restrict__ L, int64_t ldl, int w, double* __restrict__ B, int64_t ldb,
    int64_t ncols) {
  extern __shared__ double dsm[];
  double* sL = dsm;                         // [TRSM_W][TRSM_W], sL[i*W + r] = L[r][i]
  double* sX = dsm + TRSM_W * TRSM_W;       // [TRSM_W][TRSM_LDX]
  const int tid = threadIdx.x;
  const int64_t c0 = (int64_t)blockIdx.x * TRSM_COLS;
  for (int e = tid; e < TRSM_W * TRSM_W; e += TRSM_COLS) {
    const int i = e / TRSM_W, r = e - i * TRSM_W;
    if (r < w && i < w && r > i)
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(sL + e)),
                   "l"(L + (int64_t)i * ldl + r)
                   : "memory");
    else
      sL[e] = 0.0;
  }
  const int nc = (int)(ncols - c0 < TRSM_COLS ? ncols - c0 : TRSM_COLS);
  for (int e = tid; e < TRSM_W * TRSM_COLS; e += TRSM_COLS) {
    const int c = e / TRSM_W, r = e - c * TRSM_W;
    if (c < nc && r < w)
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(sX + r * TRSM_LDX + c)),
                   "l"(B + (c0 + c) * ldb + r)
                   : "memory");
    else
      sX[r * TRSM_LDX + c] = 0.0;
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();
  double x[TRSM_W];
#pragma unroll
  for (int i = 0; i < TRSM_W; ++i) x[i] = sX[i * TRSM_LDX + tid];
#pragma unroll
  for (int i = 0; i < TRSM_W - 1; ++i) {
#pragma unroll
    for (int r = i + 1; r < TRSM_W; ++r) x[r] = fma(-sL[i * TRSM_W + r], x[i], x[r]);
  }
#pragma unroll
  for (int i = 0; i < TRSM_W; ++i) sX[i * TRSM_LDX + tid] = x[i];
  __syncthreads();
  for (int e = tid; e < TRSM_W * TRSM_COLS; e += TRSM_COLS) {
    const int c = e / TRSM_W, r = e - c * TRSM_W;
    if (c < nc && r < w) B[(c0 + c) * ldb + r] = sX[r * TRSM_LDX + c];
  }
}
constexpr size_t TRSM_SMEM = sizeof(double) * (TRSM_W * TRSM_W + TRSM_W * TRSM_LDX);

// Whole-panel forward substitution in one launch: B[0:jb, c] <- L^{-1} B[0:jb, c]
// for NC columns per CTA, L unit lower jb x jb (jb <= 1024).  The CTA keeps its
// jb x NC block of B in shared memory and walks the 64-row diagonal blocks:
// a warp solves each column of the diagonal block (lanes = rows, x_k broadcast
// by shuffle), then all threads update the rows below, each row's NC values in
// registers and every L element read once per CTA.  Per element the order is
// the sequential forward substitution, b_r = fma(-l_rk, x_k, b_r) for k = 0, 1,
// ..., so the result does not depend on how the columns are partitioned.
constexpr int TRSMF_THREADS = 256;
constexpr int TRSMF_MAXJB = 1024;
constexpr int TRSMF_RPT = (TRSMF_MAXJB - 64 + TRSMF_THREADS - 1) / TRSMF_THREADS;  // rows/thread
constexpr int TRSMF_KB = 16;  // L columns per load batch
// Diagonal block at (r0, r0) of L into shared memory, column-major [64][64],
// asynchronously (cp.async, 8-byte elements: no alignment assumption on L);
// entries outside the matrix are zeroed (never read by the solve, which uses
// the strictly lower part of valid rows only)
__device__ __forceinline__ void trsmf_fetch_diag(const double* __restrict__ L, int64_t ldl, int jb,
                                                 int r0, double* dst, int tid) {
#pragma unroll 4
  for (int i = tid; i < TRSM_W * TRSM_W; i += TRSMF_THREADS) {
    const int c = i / TRSM_W, r = i - c * TRSM_W;
    if (r0 + r < jb && r0 + c < jb) {
      const double* src = L + (int64_t)(r0 + c) * ldl + r0 + r;
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst + i)), "l"(src)
                   : "memory");
    } else {
      dst[i] = 0.0;
    }
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
}

// Rows r0 + w .. jb - 1 of the CTA's block: b_r -= L[r, r0:r0+w] x[r0:r0+w]
// in k order, NQ rows per thread (each thread issues the L loads of all its
// rows per batch of TRSMF_KB columns: one L2 round trip per batch)
template <int NQ, int NC>
__device__ __forceinline__ void trsmf_rows_below(const double* __restrict__ L, int64_t ldl,
                                                 int jb, int r0, int w, double* sB, int tid) {
  double b[NQ][NC];
  int rr[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    rr[q] = r0 + w + tid + q * TRSMF_THREADS;
#pragma unroll
    for (int c = 0; c < NC; ++c) b[q][c] = rr[q] < jb ? sB[rr[q] * NC + c] : 0.0;
  }
  constexpr int KB = NQ <= 2 ? TRSM_W / NQ : TRSMF_KB;  // L loads in flight per thread: 64
  for (int k0 = 0; k0 < w; k0 += KB) {
    double l[NQ][KB];
#pragma unroll
    for (int q = 0; q < NQ; ++q)
#pragma unroll
      for (int u = 0; u < KB; ++u)
        l[q][u] = (rr[q] < jb && k0 + u < w) ? __ldg(L + (int64_t)(r0 + k0 + u) * ldl + rr[q])
                                             : 0.0;
#pragma unroll
    for (int u = 0; u < KB; ++u) {
      if (k0 + u < w) {
#pragma unroll
        for (int c = 0; c < NC; ++c) {
          const double x = sB[(r0 + k0 + u) * NC + c];
#pragma unroll
          for (int q = 0; q < NQ; ++q) b[q][c] = fma(-l[q][u], x, b[q][c]);
        }
      }
    }
  }
#pragma unroll
  for (int q = 0; q < NQ; ++q)
    if (rr[q] < jb)
#pragma unroll
      for (int c = 0; c < NC; ++c) sB[rr[q] * NC + c] = b[q][c];
}

template <int NC>
__global__ void __launch_bounds__(TRSMF_THREADS) trsm_fused_kernel(
    const double* __restrict__ L, int64_t ldl, int jb, double* __restrict__ B, int64_t ldb,
    int64_t ncols) {
  extern __shared__ double dsm[];
  double* sB = dsm;                          // [jb][NC]
  // diagonal blocks, column-major [64][64], double-buffered: block b+1 is
  // fetched (cp.async) while block b's rows below are updated
  double* sDb = dsm + (size_t)jb * NC;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  // grid-stride over column groups: a capped grid (look-ahead side stream)
  // walks every group
  for (int64_t c0 = (int64_t)blockIdx.x * NC; c0 < ncols; c0 += (int64_t)gridDim.x * NC) {
  const int nc = (int)(ncols - c0 < NC ? ncols - c0 : NC);
  trsmf_fetch_diag(L, ldl, jb, 0, sDb, tid);
  // loads batched (unrolled) so each thread keeps several L2/HBM requests in flight
#pragma unroll 8
  for (int i = tid; i < jb * NC; i += TRSMF_THREADS) {
    const int c = i / jb, r = i - c * jb;
    sB[r * NC + c] = c < nc ? B[(c0 + c) * ldb + r] : 0.0;
  }
  for (int r0 = 0; r0 < jb; r0 += TRSM_W) {
    const int w = jb - r0 < TRSM_W ? jb - r0 : TRSM_W;
    const double* sD = sDb + ((r0 / TRSM_W) & 1) * TRSM_W * TRSM_W;
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
    for (int c = wid; c < NC; c += TRSMF_THREADS / 32) {
      double v0 = lane < w ? sB[(r0 + lane) * NC + c] : 0.0;
      double v1 = lane + 32 < w ? sB[(r0 + lane + 32) * NC + c] : 0.0;
      if (w == TRSM_W) {
        // full block: static indices, the L loads leave the dependency chain
#pragma unroll
        for (int k = 0; k < 32; ++k) {
          const double xk = __shfl_sync(0xffffffffu, v0, k);
          if (lane > k) v0 = fma(-sD[k * TRSM_W + lane], xk, v0);
          v1 = fma(-sD[k * TRSM_W + lane + 32], xk, v1);
        }
#pragma unroll
        for (int k = 32; k < TRSM_W; ++k) {
          const double xk = __shfl_sync(0xffffffffu, v1, k - 32);
          if (lane + 32 > k) v1 = fma(-sD[k * TRSM_W + lane + 32], xk, v1);
        }
      } else {
        for (int k = 0; k < w; ++k) {
          const double xk = __shfl_sync(0xffffffffu, k < 32 ? v0 : v1, k & 31);
          if (lane > k) v0 = fma(-sD[k * TRSM_W + lane], xk, v0);
          if (lane + 32 > k) v1 = fma(-sD[k * TRSM_W + lane + 32], xk, v1);
        }
      }
      if (lane < w) sB[(r0 + lane) * NC + c] = v0;
      if (lane + 32 < w) sB[(r0 + lane + 32) * NC + c] = v1;
    }
    __syncthreads();
    // the next diagonal block into the other buffer (last read by block - 1)
    if (r0 + TRSM_W < jb)
      trsmf_fetch_diag(L, ldl, jb, r0 + TRSM_W, sDb + ((r0 / TRSM_W + 1) & 1) * TRSM_W * TRSM_W,
                       tid);
    // rows below the block: only as many rows per thread as there are rows
    // left (a CTA-uniform count), so no predicated-off FMA issues
    {
      const int below = jb - r0 - w;
      if (below > 2 * TRSMF_THREADS) {
        if (below > 3 * TRSMF_THREADS)
          trsmf_rows_below<4, NC>(L, ldl, jb, r0, w, sB, tid);
        else
          trsmf_rows_below<3, NC>(L, ldl, jb, r0, w, sB, tid);
      } else if (below > TRSMF_THREADS) {
        trsmf_rows_below<2, NC>(L, ldl, jb, r0, w, sB, tid);
      } else if (below > 0) {
        trsmf_rows_below<1, NC>(L, ldl, jb, r0, w, sB, tid);
      }
    }
    __syncthreads();
  }
#pragma unroll 8
  for (int i = tid; i < jb * NC; i += TRSMF_THREADS) {
    const int c = i / jb, r = i - c * jb;
    if (c < nc) B[(c0 + c) * ldb + r] = sB[r * NC + c];
  }
  __syncthreads();
  }
}
template <int NC>
constexpr size_t trsmf_smem(int jb) {
  return sizeof(double) * ((size_t)jb * NC + 2 * TRSM_W * TRSM_W);
}

// --------------------------------------------------------------- reductions
// max |a| over a contiguous block of `count` doubles (16-byte aligned):
// 128-bit loads, four in flight per thread, no index arithmetic per element
__global__ void max_abs_flat_kernel(const double2* __restrict__ a, int64_t count2,
                                    unsigned long long* out) {
  double mx[4] = {0.0, 0.0, 0.0, 0.0};
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  for (; i + 3 * stride < count2; i += 4 * stride) {
    double2 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = __ldcs(a + i + u * stride);
#pragma unroll
    for (int u = 0; u < 4; ++u) mx[u] = fmax(mx[u], fmax(fabs(v[u].x), fabs(v[u].y)));
  }
  for (; i < count2; i += stride) {
    const double2 v = __ldcs(a + i);
    mx[0] = fmax(mx[0], fmax(fabs(v.x), fabs(v.y)));
  }
  double m = warp_max(fmax(fmax(mx[0], mx[1]), fmax(mx[2], mx[3])));
  if ((threadIdx.x & 31) == 0 && m > 0.0) atomic_max_abs(out, m);
}

__global__ void max_abs_kernel(const double* __restrict__ a, int64_t m, int64_t n, int64_t rs,
                               int64_t cs, int upper_only, int64_t diag_off,
                               unsigned long long* out) {
  double mx = 0.0;
  const int64_t total = m * n;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i % m, c = i / m;
    if (upper_only && c + diag_off < r) continue;
    mx = fmax(mx, fabs(a[r * rs + c * cs]));
  }
  mx = warp_max(mx);
  if ((threadIdx.x & 31) == 0 && mx > 0.0) atomic_max_abs(out, mx);
}

// Row-chunked GEMV partials: part[chunk][i] = sum_{j in chunk} a_ij * x_j (x=null -> 1),
// apart[chunk][i] = sum |a_ij|.  Deterministic (fixed order, no atomics).
constexpr int GEMV_CHUNK = 1024;
__global__ void gemv_partial_kernel(const double* __restrict__ a, int64_t n, int64_t ncols,
                                    int64_t rs, int64_t cs, const double* __restrict__ x,
                                    double* __restrict__ part, double* __restrict__ apart) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t j0 = (int64_t)blockIdx.y * GEMV_CHUNK;
  if (i >= n) return;
  const int64_t j1 = min(ncols, j0 + GEMV_CHUNK);
  double s = 0.0, sa = 0.0;
  const double* row = a + i * rs;
  for (int64_t j = j0; j < j1; ++j) {
    const double v = row[j * cs];
    s = fma(v, x ? x[j] : 1.0, s);
    sa += fabs(v);
  }
  part[blockIdx.y * n + i] = s;
  if (apart) apart[blockIdx.y * n + i] = sa;
}

// out[i] = sum_chunks part ; residual mode: r_i = out_i - b_i, reduce max|r|, max asum
__global__ void gemv_finish_kernel(const double* __restrict__ part,
                                   const double* __restrict__ apart, int nchunks, int64_t n,
                                   const double* __restrict__ b, double* __restrict__ out,
                                   unsigned long long* rmax, unsigned long long* amax,
                                   double* __restrict__ abs_out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  double rr = 0.0, aa = 0.0;
  if (i < n) {
    double s = 0.0, sa = 0.0;
    for (int c = 0; c < nchunks; ++c) {
      s += part[c * n + i];
      if (apart) sa += apart[c * n + i];
    }
    if (out) out[i] = s;
    if (abs_out) abs_out[i] = sa;
    if (b) rr = fabs(s - b[i]);
    aa = sa;
  }
  rr = warp_max(rr);
  aa = warp_max(aa);
  if ((threadIdx.x & 31) == 0) {
    if (rmax && rr > 0.0) atomic_max_abs(rmax, rr);
    if (amax && aa > 0.0) atomic_max_abs(amax, aa);
  }
}

// ------------------------------------------------------------------ triangular solves
// Sync-free blocked triangular solve, one launch per triangle.  Row block i
// (TRSV_B rows) is owned by the CTA that draws ticket i (tickets follow the
// dependency order, so the scheme cannot deadlock).  The CTA folds in the
// contribution of every finished block j (spinning on its ready flag), then
// solves its diagonal block and publishes x_i.  Reads of A are coalesced
// (consecutive threads = consecutive rows of a column-major block).
constexpr int TRSV_B = 64;
constexpr int TRSV_G = 4;  // thread groups of TRSV_B threads splitting the j loop
__global__ void __launch_bounds__(TRSV_B * TRSV_G) trsv_syncfree_kernel(
    const double* __restrict__ a, int64_t lda, int64_t n, int upper, double* x, int* flags,
    int* ticket, int32_t* zero_diag) {
  __shared__ int s_blk;
  __shared__ double s_acc[TRSV_G][TRSV_B];
  __shared__ double s_diag[TRSV_B][TRSV_B + 1];
  const int tid = threadIdx.x, r = tid % TRSV_B, grp = tid / TRSV_B;
  const int nblk = (int)((n + TRSV_B - 1) / TRSV_B);
  if (tid == 0) s_blk = atomicAdd(ticket, 1);
  __syncthreads();
  const int order = s_blk;
  const int blk = upper ? nblk - 1 - order : order;
  const int64_t r0 = (int64_t)blk * TRSV_B;
  const int bs = (int)min((int64_t)TRSV_B, n - r0);
  // diagonal block into shared memory (independent of the other blocks)
  for (int c = grp; c < bs; c += TRSV_G)
    if (r < bs) s_diag[r][c] = a[(r0 + c) * lda + r0 + r];
  double acc = 0.0;
  for (int t = grp; t < order; t += TRSV_G) {
    const int j = upper ? nblk - 1 - t : t;
    const int64_t c0 = (int64_t)j * TRSV_B;
    const int cs = (int)min((int64_t)TRSV_B, n - c0);
    // the block of A does not depend on the solution: load it before waiting
    double av[TRSV_B];
    const double* col = a + c0 * lda + r0 + r;
#pragma unroll
    for (int c = 0; c < TRSV_B; ++c) av[c] = (c < cs && r < bs) ? col[c * lda] : 0.0;
    volatile int* f = flags + j;
    while (*f == 0) {
    }
    __threadfence();
    const double* xj = x + c0;
#pragma unroll
    for (int c = 0; c < TRSV_B; ++c) acc = fma(av[c], c < cs ? __ldcg(xj + c) : 0.0, acc);
  }
  s_acc[grp][r] = acc;
  __syncthreads();
  if (tid < 32) {
    // lane l owns rows l and l+32 of the block
    double y0 = 0.0, y1 = 0.0;
    const int ra = tid, rb = tid + 32;
    if (ra < bs) y0 = x[r0 + ra] - (s_acc[0][ra] + s_acc[1][ra] + s_acc[2][ra] + s_acc[3][ra]);
    if (rb < bs) y1 = x[r0 + rb] - (s_acc[0][rb] + s_acc[1][rb] + s_acc[2][rb] + s_acc[3][rb]);
    if (!upper) {
      for (int c = 0; c < bs; ++c) {
        const double xc = __shfl_sync(0xffffffffu, c < 32 ? y0 : y1, c & 31);
        if (ra > c && ra < bs) y0 = fma(-s_diag[ra][c], xc, y0);
        if (rb > c && rb < bs) y1 = fma(-s_diag[rb][c], xc, y1);
      }
    } else {
      for (int c = bs - 1; c >= 0; --c) {
        const double d = s_diag[c][c];
        if (d == 0.0 && tid == 0) *zero_diag = 1;
        double v = __shfl_sync(0xffffffffu, c < 32 ? y0 : y1, c & 31);
        v = v / d;
        if (c < 32 && ra == c) y0 = v;
        if (c >= 32 && rb == c) y1 = v;
        if (ra < c) y0 = fma(-s_diag[ra][c], v, y0);
        if (rb < c) y1 = fma(-s_diag[rb][c], v, y1);
      }
    }
    if (ra < bs) x[r0 + ra] = y0;
    if (rb < bs) x[r0 + rb] = y1;
    __threadfence();
    __syncwarp();
    if (tid == 0) atomicExch(flags + blk, 1);
  }
}

__global__ void gather_kernel(const double* __restrict__ b, const int64_t* __restrict__ perm,
                              int64_t n, double* __restrict__ x) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) x[i] = b[perm[i]];
}

__global__ void copy_flat_kernel(const double2* __restrict__ src, double2* __restrict__ dst,
                                 int64_t count2) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  for (; i + 3 * stride < count2; i += 4 * stride) {  // four 16-byte loads in flight
    double2 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = __ldcs(src + i + u * stride);
#pragma unroll
    for (int u = 0; u < 4; ++u) __stcs(dst + i + u * stride, v[u]);
  }
  for (; i < count2; i += stride) __stcs(dst + i, __ldcs(src + i));
}

__global__ void copy2d_kernel(const double* __restrict__ src, int64_t rows, int64_t cols,
                              int64_t srs, int64_t scs, double* __restrict__ dst, int64_t drs,
                              int64_t dcs) {
  __shared__ double tile[32][33];
  const int64_t r0 = (int64_t)blockIdx.y * 32, c0 = (int64_t)blockIdx.x * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
  const bool src_rowmajor = scs == 1;
  for (int k = ty; k < 32; k += 8) {
    // read with the contiguous source index on threadIdx.x
    const int64_t r = src_rowmajor ? r0 + k : r0 + tx;
    const int64_t c = src_rowmajor ? c0 + tx : c0 + k;
    if (r < rows && c < cols) {
      if (src_rowmajor) tile[k][tx] = src[r * srs + c * scs];
      else tile[tx][k] = src[r * srs + c * scs];
    }
  }
  __syncthreads();
  const bool dst_rowmajor = dcs == 1;
  for (int k = ty; k < 32; k += 8) {
    const int64_t r = dst_rowmajor ? r0 + k : r0 + tx;
    const int64_t c = dst_rowmajor ? c0 + tx : c0 + k;
    if (r < rows && c < cols) dst[r * drs + c * dcs] = dst_rowmajor ? tile[k][tx] : tile[tx][k];
  }
}

__global__ void finalize_stats_kernel(const unsigned long long* bits, double* stats) {
  stats[0] = __longlong_as_double((long long)bits[0]);
  stats[1] = __longlong_as_double((long long)bits[1]);
}

// ---------------------------------------------------------------- workspace
struct LuWs {
  GridBar* bar;
  double* cand;
  int32_t* swap_dst;
  int32_t* swap_src;
  int32_t* swap_cnt;
  int32_t* cdst;  // composed whole-panel gather list (compose_ipiv_kernel)
  int32_t* csrc;
  int32_t* ccnt;
  unsigned long long* bits;  // [0] observed growth, [1] max|A|
  void* split_aux;
  int32_t* expA;
  int32_t* expB;
  int8_t* slA;
  int8_t* slB;
  int64_t ldK;
};

size_t align_up(size_t v) { return (v + 255) & ~size_t(255); }

size_t lu_ws_layout(int64_t n, int64_t nb, int k, uint8_t* base, LuWs* ws) {
  size_t off = 0;
  auto take = [&](size_t bytes) {
    uint8_t* p = base ? base + off : nullptr;
    off += align_up(bytes);
    return p;
  };
  const int sms = 1024;  // upper bound on panel CTAs
  const int64_t ldK = round_up(nb, 16);
  LuWs w{};
  w.bar = reinterpret_cast<GridBar*>(take(sizeof(GridBar)));
  w.cand = reinterpret_cast<double*>(take(sizeof(double) * 2 * sms * CAND_STRIDE));
  w.swap_dst = reinterpret_cast<int32_t*>(take(sizeof(int32_t) * SWAP_MAX));
  w.swap_src = reinterpret_cast<int32_t*>(take(sizeof(int32_t) * SWAP_MAX));
  w.swap_cnt = reinterpret_cast<int32_t*>(take(sizeof(int32_t) * 4));
  w.cdst = reinterpret_cast<int32_t*>(take(sizeof(int32_t) * LSWP_MAX));
  w.csrc = reinterpret_cast<int32_t*>(take(sizeof(int32_t) * LSWP_MAX));
  w.ccnt = reinterpret_cast<int32_t*>(take(sizeof(int32_t) * 4));
  w.bits = reinterpret_cast<unsigned long long*>(take(sizeof(unsigned long long) * 4));
  w.split_aux = take(64);
  w.expA = reinterpret_cast<int32_t*>(take(sizeof(int32_t) * n));
  w.expB = reinterpret_cast<int32_t*>(take(sizeof(int32_t) * n));
  w.ldK = ldK;
  if (k > 0) {
    w.slA = reinterpret_cast<int8_t*>(take((size_t)k * n * ldK));
    w.slB = reinterpret_cast<int8_t*>(take((size_t)k * n * ldK));
  }
  if (ws) *ws = w;
  return off;
}

int max_abs(const double* a, int64_t m, int64_t n, int64_t rs, int64_t cs, int upper,
            int64_t diag_off, unsigned long long* out, cudaStream_t st) {
  if (m <= 0 || n <= 0) return OZ_OK;
  const int64_t count = m * n;
  if (!upper && rs == 1 && (cs == m || n == 1) && count % 2 == 0 &&
      (reinterpret_cast<uintptr_t>(a) & 15) == 0 && count >= (1 << 20)) {
    // one contiguous block (the LU's working copy, lda = n): flat 128-bit scan
    int64_t blocks = ceil_div(count / 2, 256);
    if (blocks > sm_count() * 8) blocks = sm_count() * 8;
    max_abs_flat_kernel<<<(unsigned)blocks, 256, 0, st>>>(reinterpret_cast<const double2*>(a),
                                                            count / 2, out);
    OZ_CHECK_LAUNCH();
    return OZ_OK;
  }
  int64_t blocks = ceil_div(m * n, 256);
  if (blocks > sm_count() * 8) blocks = sm_count() * 8;
  max_abs_kernel<<<(unsigned)blocks, 256, 0, st>>>(a, m, n, rs, cs, upper, diag_off, out);
  OZ_CHECK_LAUNCH();
  return OZ_OK;
}

int apply_list(double* a, int64_t lda, const LuWs& ws, int64_t c0a, int64_t c1a, int64_t c0b,
               int64_t c1b, cudaStream_t st, int max_ctas = 0) {
  const int64_t ncols = (c1a - c0a) + (c1b - c0b);
  if (ncols <= 0) return OZ_OK;
  struct Stop {
    int tag;
    cudaStream_t st;
    ~Stop() { prof_stop(tag, st, PROF_LASWP, 0.0); }
  } stop{prof_start(st), st};
  int64_t blocks = ceil_div(ncols, 8);
  if (blocks > sm_count() * 16) blocks = sm_count() * 16;
  if (max_ctas > 0 && blocks > max_ctas) blocks = max_ctas;
  laswp_gather_kernel<<<(unsigned)blocks, 256, 0, st>>>(a, lda, ws.swap_dst, ws.swap_src,
                                                        ws.swap_cnt, c0a, c1a, c0b, c1b);
  OZ_CHECK_LAUNCH();
  return OZ_OK;
}

// U12 <- L11^{-1} A12 for L11 (jb x jb, unit lower) at a[j,j], A12 = rows j..j+jb, ncols
template <int NC>
int trsm_fused(const double* L, int64_t lda, int64_t jb, double* b, int64_t ldb, int64_t ncols,
               cudaStream_t st, int max_ctas) {
  OZ_ONCE(cudaFuncSetAttribute(trsm_fused_kernel<NC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)trsmf_smem<NC>(TRSMF_MAXJB)));
  int64_t grid = ceil_div(ncols, NC);
  if (max_ctas > 0 && grid > max_ctas) grid = max_ctas;
  trsm_fused_kernel<NC><<<(unsigned)grid, TRSMF_THREADS, trsmf_smem<NC>((int)jb), st>>>(
      L, lda, (int)jb, b, ldb, ncols);
  OZ_CHECK_LAUNCH();
  return OZ_OK;
}

// Wide right-hand sides: recursive halving, X1 = L11^-1 B1, B2 -= L21 X1
// (one DGEMM of depth jb/2, jb/4, ... instead of jb/64 DGEMMs of depth 64),
// X2 = L22^-1 B2; 64-row diagonal blocks by trsm_unit_lower_kernel.
int trsm_rec(double* a, int64_t lda, int64_t j, int64_t jb, double* b, int64_t ldb,
             int64_t ncols, cudaStream_t st, int max_ctas) {
  if (jb <= TRSM_W) {
    const int tag = prof_start(st);
    trsm_unit_lower_kernel<<<(unsigned)ceil_div(ncols, TRSM_COLS), TRSM_COLS, TRSM_SMEM, st>>>(
        a + j * lda + j, lda, (int)jb, b, ldb, ncols);
    OZ_CHECK_LAUNCH();
    prof_stop(tag, st, PROF_TRSM, (double)jb * jb * ncols);
    return OZ_OK;
  }
  const int64_t h = ((jb / 2 + TRSM_W - 1) / TRSM_W) * TRSM_W;
  OZ_TRY(trsm_rec(a, lda, j, h, b, ldb, ncols, st, max_ctas));
  const int tag = prof_start(st);
  OZ_TRY(dgemm(0, 0, jb - h, ncols, h, -1.0, a + j * lda + (j + h), lda, b, ldb, 1.0, b + h, ldb,
               st, max_ctas));
  prof_stop(tag, st, PROF_DGEMM_TRSM, 2.0 * (jb - h) * ncols * h);
  return trsm_rec(a, lda, j + h, jb - h, b + h, ldb, ncols, st, max_ctas);
}

// max_ctas > 0 caps every grid of the call (look-ahead side stream: the
// panel must not take SMs the concurrent persistent GEMM was sized for)
int trsm_blocked(double* a, int64_t lda, int64_t j, int64_t jb, double* b, int64_t ldb,
                 int64_t ncols, cudaStream_t st, int max_ctas = 0) {
  if (ncols <= 0) return OZ_OK;
  static const bool legacy = getenv("OZ_TRSM_LEGACY") != nullptr;
  // few right-hand sides (the look-ahead's next panel, the recursion inside a
  // panel): one launch, latency-bound (~0.3 ms at jb = 1024 vs ~0.5 ms for the
  // 2*jb/64 launches below); wide updates: diagonal blocks + cuBLAS DGEMM,
  // FP64-throughput-bound (15 vs 5 TFLOP/s at 30720 columns)
  static const bool narrow_cublas = getenv("OZ_TRSM_NARROW_CUBLAS") != nullptr;  // tuning A/B
  if (narrow_cublas && ncols <= 2048) {
    const int tag = prof_start(st);
    const int s = dtrsm_lunit(jb, ncols, a + j * lda + j, lda, b, ldb, st, max_ctas);
    prof_stop(tag, st, PROF_TRSM, (double)jb * jb * ncols);
    return s;
  }
  if (!legacy && jb <= TRSMF_MAXJB && ncols <= 2048) {
    const int tag = prof_start(st);
    // 8 columns per CTA: measured faster than 4 or 2 (more CTAs) at every
    // panel-recursion shape and inside the LU (profiles/r02bm_trsm_nc_ab.log)
    // A capped grid (SMs held by a concurrent kernel) takes a few more
    // columns per CTA rather than a second wave of CTAs
    const int avail = max_ctas > 0 && max_ctas < sm_count() ? max_ctas : sm_count();
    static const bool widen = !getenv("OZ_TRSM_WIDEN") || atoi(getenv("OZ_TRSM_WIDEN"));
    const double* l11 = a + j * lda + j;
    const int s = !widen || ceil_div(ncols, (int64_t)8) <= avail
                      ? trsm_fused<8>(l11, lda, jb, b, ldb, ncols, st, max_ctas)
                  : ceil_div(ncols, (int64_t)9) <= avail
                      ? trsm_fused<9>(l11, lda, jb, b, ldb, ncols, st, max_ctas)
                  : ceil_div(ncols, (int64_t)10) <= avail
                      ? trsm_fused<10>(l11, lda, jb, b, ldb, ncols, st, max_ctas)
                      : trsm_fused<12>(l11, lda, jb, b, ldb, ncols, st, max_ctas);
    prof_stop(tag, st, PROF_TRSM, (double)jb * jb * ncols);
    return s;
  }
  static const bool use_cublas = getenv("OZ_TRSM_CUBLAS") != nullptr;  // tuning A/B
  if (use_cublas) {
    const int tag = prof_start(st);
    const int s = dtrsm_lunit(jb, ncols, a + j * lda + j, lda, b, ldb, st, max_ctas);
    prof_stop(tag, st, PROF_TRSM, (double)jb * jb * ncols);
    return s;
  }
  OZ_ONCE(cudaFuncSetAttribute(trsm_unit_lower_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)TRSM_SMEM));
  return trsm_rec(a, lda, j, jb, b, ldb, ncols, st, max_ctas);
}

// Cluster exchange for short panels: OZ_PANEL_CLUSTER = max cluster size
// (default 16, 0 = off), OZ_PANEL_CLUSTER_M = max panel rows (default 8192).
int panel_cluster_max() {
  static const int v = [] {
    const char* e = getenv("OZ_PANEL_CLUSTER");
    return e ? atoi(e) : 16;
  }();
  return v;
}
int64_t panel_cluster_rows() {
  static const int64_t v = [] {
    const char* e = getenv("OZ_PANEL_CLUSTER_M");
    return e ? (int64_t)atoll(e) : (int64_t)8192;
  }();
  return v;
}
int panel_smem_cap() {
  static const int max_smem = [] {
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    return v;
  }();
  return max_smem - (int)sizeof(PanelShared) - 1024;
}
// can a cluster of G panel CTAs (smem bytes each) be resident at all?
bool cluster_fits(int G, size_t smem) {
  static std::mutex mu;
  static std::vector<std::pair<long long, bool>> memo;
  std::lock_guard<std::mutex> lock(mu);
  const long long key = (long long)G << 32 | (long long)smem;
  for (auto& kv : memo)
    if (kv.first == key) return kv.second;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(G);
  cfg.blockDim = dim3(PANEL_THREADS);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = G;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int n = 0;
  const bool ok = cudaOccupancyMaxActiveClusters(&n, (void*)panel_window_kernel<true>, &cfg) ==
                      cudaSuccess && n > 0;
  cudaGetLastError();
  memo.push_back({key, ok});
  return ok;
}

// Record tags of the grid-exchange leaves: epoch + t + 1 (t < 128), unique per
// launch for 2^25 launches, so a record left in the candidate buffer by an
// earlier launch never matches the current step.
unsigned next_record_epoch() {
  static std::atomic<unsigned> seq{1};
  return (seq.fetch_add(1u) & 0x1ffffffu) << 7;
}

// Register-resident leaf (panel_leaf.cuh) for short panels: OZ_PANEL_LEAF=0
// disables it (tuning / A-B).  Variant = W*10 + RPT: rows per CTA 256*RPT,
// at most LEAF_MAXG CTAs in the cluster, W*RPT <= 64 doubles per thread.
bool leaf_enabled() {
  static const bool v = [] {
    const char* e = getenv("OZ_PANEL_LEAF");
    return e == nullptr || atoi(e) != 0;
  }();
  return v;
}
// Rows per thread the register leaf may use (OZ_PANEL_LEAF_RPT, tuning).
// Measured, LU factor time n = 8192 / 16384 / 32768, k = 7
// (profiles/r02_leaf_rpt_ab.txt): RPT 1 (64-column windows up to 4096 rows)
// 43.8 / 119.0 / 507 ms; RPT 2 (also 32-column windows up to 8192 rows)
// 38.9 / 114.0 / 504 ms; RPT 4 (also 16-column windows up to 16384 rows)
// 38.9 / 134.6 / 528 ms (the narrow windows double the recursion's inner
// nodes); shared-memory leaf only 49.9 / 123.7 / 508 ms.
int leaf_max_rpt() {
  static const int v = [] {
    const char* e = getenv("OZ_PANEL_LEAF_RPT");
    return e ? atoi(e) : 2;
  }();
  return v;
}
// OZ_PANEL_LEAF_GRID=0 keeps taller panels on the shared-memory grid leaf
// (tuning A/B): otherwise the register leaf with the global-memory exchange
// takes panels whose rows fit 256 (W = 64) or 512 (W = 32) per CTA on the
// SMs the caller may use.
bool leaf_grid_enabled() {
  static const bool v = [] {
    const char* e = getenv("OZ_PANEL_LEAF_GRID");
    return e == nullptr || atoi(e) != 0;
  }();
  return v;
}
// OZ_PANEL_LEAF_TALL=0: the tallest panels keep the shared-memory leaf (A/B).
// 1024 rows per CTA with 16-column windows measured 465 -> 461 ms at n =
// 32768; 2048 rows with 8-column windows (twice the recursion's inner nodes)
// lost (484 ms, profiles/r02bw_tall_leaf_ab.log) and was dropped.
bool leaf_tall_enabled() {
  static const bool v = [] {
    const char* e = getenv("OZ_PANEL_LEAF_TALL");
    return e == nullptr || atoi(e) != 0;
  }();
  return v;
}
int leaf_variant(int64_t m, int w, int max_ctas) {
  if (!leaf_enabled() || m < 1) return 0;
  const int rpt = leaf_max_rpt();
  const int cap = max_ctas > 0 && max_ctas < sm_count() ? max_ctas : sm_count();
  int v = 0, rows = 0;
  if (w <= 64 && m <= (int64_t)LEAF_MAXG * 128) {
    v = 6411;  // 128 threads x 1 row
    rows = 128;
  } else if (w <= 64 && m <= (int64_t)LEAF_MAXG * 256) {
    v = w <= 32 ? 3212 : 6412;
    rows = 256;
  } else if (rpt >= 2 && w <= 32 && m <= (int64_t)LEAF_MAXG * 512) {
    v = 3222;
    rows = 512;
  } else if (rpt >= 4 && w <= 16 && m <= (int64_t)LEAF_MAXG * 1024) {
    v = 1642;
    rows = 1024;
  }
  // the cluster must fit in the SMs the caller may use (look-ahead side stream)
  if (v != 0 && ceil_div(m, (int64_t)rows) <= cap) return v;
  if (!leaf_grid_enabled()) return 0;
  // taller: one co-resident grid, records exchanged through global memory
  if (w <= 64 && ceil_div(m, (int64_t)256) <= cap) return 64120;
  if (w <= 32 && ceil_div(m, (int64_t)512) <= cap) return 32220;
  // tallest (early look-ahead panels on few SMs): narrower windows, more rows
  // per thread, instead of the shared-memory leaf
  if (leaf_tall_enabled() && w <= 16 && ceil_div(m, (int64_t)1024) <= cap) return 16420;
  return 0;
}
// widest leaf the register variants take at this height (0: none)
int leaf_width_for(int64_t m, int max_ctas) {
  const int rpt = leaf_max_rpt();
  if (!leaf_enabled()) return 0;
  const int cap = max_ctas > 0 && max_ctas < sm_count() ? max_ctas : sm_count();
  if (m <= (int64_t)LEAF_MAXG * 256 &&
      ceil_div(m, (int64_t)(m <= (int64_t)LEAF_MAXG * 128 ? 128 : 256)) <= cap)
    return 64;
  if (rpt >= 2 && m <= (int64_t)LEAF_MAXG * 512 && ceil_div(m, (int64_t)512) <= cap) return 32;
  if (leaf_grid_enabled()) {
    if (ceil_div(m, (int64_t)256) <= cap) return 64;
    if (ceil_div(m, (int64_t)512) <= cap) return 32;
    if (leaf_tall_enabled() && ceil_div(m, (int64_t)1024) <= cap) return 16;
  }
  if (rpt >= 4 && m <= (int64_t)LEAF_MAXG * 1024 && ceil_div(m, (int64_t)1024) <= cap) return 16;
  return 0;
}

template <int W, int RPT, int NT, bool kGrid = false>
int panel_leaf_launch(PanelArgs pa, cudaStream_t st) {
  constexpr size_t smem = leaf_smem_bytes<W, RPT, NT>();
  OZ_ONCE([] {
    cudaError_t e = cudaFuncSetAttribute(panel_leaf_kernel<W, RPT, NT, kGrid>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e == cudaSuccess && !kGrid)
      e = cudaFuncSetAttribute(panel_leaf_kernel<W, RPT, NT, kGrid>,
                               cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    return e;
  }());
  const int G = (int)ceil_div(pa.m, (int64_t)NT * RPT);
  if constexpr (kGrid) {
    pa.epoch = next_record_epoch();
    void* args[] = {&pa};
    OZ_CHECK_CUDA(cudaLaunchCooperativeKernel((void*)panel_leaf_kernel<W, RPT, NT, kGrid>,
                                              dim3(G), dim3(NT), args, smem, st));
    return OZ_OK;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(G);
  cfg.blockDim = dim3(NT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = G;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  OZ_CHECK_CUDA(cudaLaunchKernelEx(&cfg, panel_leaf_kernel<W, RPT, NT, kGrid>, pa));
  return OZ_OK;
}

int panel_leaf(double* a, int64_t lda, int64_t r0, int64_t m, int w, int64_t base, int32_t* ipiv,
               int32_t* info, unsigned long long* growth, const LuWs& ws, cudaStream_t st,
               int max_ctas) {
  PanelArgs pa;
  pa.a = a;
  pa.lda = lda;
  pa.r0 = r0;
  pa.m = m;
  pa.base = base;
  pa.w = w;
  pa.rows_per_cta = 0;
  pa.ipiv = ipiv;
  pa.growth = growth;
  pa.info = info;
  pa.bar = ws.bar;
  pa.cand = ws.cand;
  pa.list_dst = ws.swap_dst;
  pa.list_src = ws.swap_src;
  pa.list_cnt = ws.swap_cnt;
  pa.dbg = panel_dbg();
  pa.epoch = 0;
  OZ_CHECK_CUDA(cudaMemsetAsync(ws.swap_cnt, 0, sizeof(int32_t), st));
  const int tag = prof_start(st);
  count_launch();
  int s = OZ_OK;
  switch (leaf_variant(m, w, max_ctas)) {
    case 6411: s = panel_leaf_launch<64, 1, 128>(pa, st); break;
    case 6412: s = panel_leaf_launch<64, 1, 256>(pa, st); break;
    case 3212: s = panel_leaf_launch<32, 1, 256>(pa, st); break;
    case 3222: s = panel_leaf_launch<32, 2, 256>(pa, st); break;
    case 1642: s = panel_leaf_launch<16, 4, 256>(pa, st); break;
    case 64120: s = panel_leaf_launch<64, 1, 256, true>(pa, st); break;
    case 32220: s = panel_leaf_launch<32, 2, 256, true>(pa, st); break;
    case 16420: s = panel_leaf_launch<16, 4, 256, true>(pa, st); break;
    default: s = OZ_UNSUPPORTED;
  }
  prof_stop(tag, st, PROF_PANEL, (double)m * w);
  return s;
}

int panel_window(double* a, int64_t lda, int64_t r0, int64_t m, int w, int64_t base,
                 int32_t* ipiv, int32_t* info, unsigned long long* growth, const LuWs& ws,
                 cudaStream_t st, int max_ctas) {
  OZ_ONCE([] {
    cudaError_t e = cudaFuncSetAttribute(panel_window_kernel<false>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         panel_smem_cap());
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(panel_window_kernel<true>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, panel_smem_cap());
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(panel_window_kernel<true>,
                               cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    return e;
  }());
  const int sms = max_ctas > 0 && max_ctas < sm_count() ? max_ctas : sm_count();
  if (leaf_variant(m, w, max_ctas) != 0)
    return panel_leaf(a, lda, r0, m, w, base, ipiv, info, growth, ws, st, max_ctas);
  const size_t cap = (size_t)panel_smem_cap();
  // cluster variant: as few CTAs as the slab allows, at most the cluster size
  const int cmax = panel_cluster_max();
  bool cluster = false;
  int G = 0, R = 0;
  if (cmax >= 2 && m <= panel_cluster_rows()) {
    const int64_t rmax = (int64_t)((cap - 0) / ((size_t)w * sizeof(double) + sizeof(int)));
    static const int64_t rows_target = [] {  // tuning: rows per CTA the cluster aims for
      const char* e = getenv("OZ_PANEL_CLUSTER_ROWS");
      return e ? (int64_t)atoll(e) : (int64_t)128;  // measured: 128 beats 256, = 64
    }();
    int g = (int)std::max<int64_t>(ceil_div(m, rmax),
                                   std::min<int64_t>(ceil_div(m, rows_target), cmax));
    if (g < 2) g = 2;
    if (g <= cmax && g <= sms) {
      const int rr = (int)ceil_div(m, g);
      g = (int)ceil_div(m, rr);
      if (g >= 2 && panel_smem_bytes(w, rr) <= cap && cluster_fits(g, panel_smem_bytes(w, rr))) {
        cluster = true;
        G = g;
        R = rr;
      }
    }
  }
  if (!cluster) {
    G = (int)ceil_div(m, 256);
    if (G > sms) G = sms;
    if (G < 1) G = 1;
    R = (int)ceil_div(m, G);
    while (panel_smem_bytes(w, R) > cap) {
      OZ_REQUIRE(G < sms, OZ_UNSUPPORTED, "panel of %lld rows x %d cols does not fit on chip",
                 (long long)m, w);
      ++G;
      R = (int)ceil_div(m, G);
    }
    G = (int)ceil_div(m, R);
  }
  PanelArgs pa;
  pa.a = a;
  pa.lda = lda;
  pa.r0 = r0;
  pa.m = m;
  pa.base = base;
  pa.w = w;
  pa.rows_per_cta = R;
  pa.ipiv = ipiv;
  pa.growth = growth;
  pa.info = info;
  pa.bar = ws.bar;
  pa.cand = ws.cand;
  pa.list_dst = ws.swap_dst;
  pa.list_src = ws.swap_src;
  pa.list_cnt = ws.swap_cnt;
  pa.dbg = panel_dbg();
  pa.epoch = next_record_epoch();
  OZ_CHECK_CUDA(cudaMemsetAsync(ws.swap_cnt, 0, sizeof(int32_t), st));
  const int tag = prof_start(st);
  count_launch();
  if (cluster) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(G);
    cfg.blockDim = dim3(PANEL_THREADS);
    cfg.dynamicSmemBytes = panel_smem_bytes(w, R);
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = G;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    OZ_CHECK_CUDA(cudaLaunchKernelEx(&cfg, panel_window_kernel<true>, pa));
  } else {
    void* args[] = {&pa};
    OZ_CHECK_CUDA(cudaLaunchCooperativeKernel((void*)panel_window_kernel<false>, dim3(G),
                                              dim3(PANEL_THREADS), args,
                                              panel_smem_bytes(w, R), st));
  }
  prof_stop(tag, st, PROF_PANEL, (double)m * w);
  return OZ_OK;
}

// Apply the sequential interchanges ipiv[0..npiv) of rows k1.. (global ipiv
// values) to columns [c0a,c1a) U [c0b,c1b) of a: compose once, gather once.
void compose_launch(const int32_t* ipiv, int npiv, int64_t k1, const LuWs& ws, cudaStream_t st) {
  compose_ipiv_kernel<<<1, COMPOSE_MAX, 0, st>>>(ipiv, npiv, k1, ws.cdst, ws.csrc, ws.ccnt);
}

int laswp_ipiv(double* a, int64_t lda, int64_t c0a, int64_t c1a, int64_t c0b, int64_t c1b,
               int64_t k1, const int32_t* ipiv, int npiv, const LuWs& ws, cudaStream_t st) {
  OZ_REQUIRE(npiv >= 0, OZ_INVALID_PARAMS, "negative interchange count");
  const int64_t ncols = (c1a - c0a) + (c1b - c0b);
  if (npiv == 0 || ncols <= 0) return OZ_OK;
  if (npiv > COMPOSE_MAX) {
    // lu_block > COMPOSE_MAX: the sequential interchanges compose chunk by
    // chunk (LAPACK dlaswp order is preserved)
    for (int off = 0; off < npiv; off += COMPOSE_MAX)
      OZ_TRY(laswp_ipiv(a, lda, c0a, c1a, c0b, c1b, k1 + off, ipiv + off,
                        std::min(COMPOSE_MAX, npiv - off), ws, st));
    return OZ_OK;
  }
  OZ_ONCE(cudaFuncSetAttribute(laswp_list_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)LSWP_SMEM));
  struct Stop {
    int tag;
    cudaStream_t st;
    ~Stop() { prof_stop(tag, st, PROF_LASWP, 0.0); }
  } stop{prof_start(st), st};
  compose_launch(ipiv, npiv, k1, ws, st);
  OZ_CHECK_LAUNCH();
  static const bool smem_variant = getenv("OZ_LASWP_SMEM") != nullptr;  // tuning
  if (smem_variant) {
    int64_t blocks = ceil_div(ncols, LSWP_WARPS);
    if (blocks > sm_count() * 2) blocks = sm_count() * 2;
    laswp_list_kernel<<<(unsigned)blocks, LSWP_WARPS * 32, LSWP_SMEM, st>>>(
        a, lda, ws.cdst, ws.csrc, ws.ccnt, c0a, c1a, c0b, c1b);
  } else {
    int64_t blocks = ceil_div(ncols, LSWR_WARPS);
    if (blocks > sm_count()) blocks = sm_count();
    laswp_list_reg_kernel<<<(unsigned)blocks, LSWR_WARPS * 32, 0, st>>>(
        a, lda, ws.cdst, ws.csrc, ws.ccnt, c0a, c1a, c0b, c1b);
  }
  OZ_CHECK_LAUNCH();
  return OZ_OK;
}

// laswp_ipiv in two parts: compose the gather list once, then apply it to
// column ranges (possibly on two streams at once; the list stays valid until
// the next compose, which the caller orders after every apply).
int compose_list(int64_t k1, const int32_t* ipiv, int npiv, const LuWs& ws, cudaStream_t st) {
  OZ_REQUIRE(npiv >= 0 && npiv <= COMPOSE_MAX, OZ_INVALID_PARAMS, "bad interchange count");
  if (npiv == 0) return OZ_OK;
  compose_launch(ipiv, npiv, k1, ws, st);
  OZ_CHECK_LAUNCH();
  return OZ_OK;
}
int apply_composed(double* a, int64_t lda, int64_t c0a, int64_t c1a, int64_t c0b, int64_t c1b,
                   int npiv, const LuWs& ws, cudaStream_t st, int max_ctas = 0) {
  const int64_t ncols = (c1a - c0a) + (c1b - c0b);
  if (npiv == 0 || ncols <= 0) return OZ_OK;
  struct Stop {
    int tag;
    cudaStream_t st;
    ~Stop() { prof_stop(tag, st, PROF_LASWP, 0.0); }
  } stop{prof_start(st), st};
  int64_t blocks = ceil_div(ncols, LSWR_WARPS);
  if (blocks > sm_count()) blocks = sm_count();
  if (max_ctas > 0 && blocks > max_ctas) blocks = max_ctas;
  laswp_list_reg_kernel<<<(unsigned)blocks, LSWR_WARPS * 32, 0, st>>>(
      a, lda, ws.cdst, ws.csrc, ws.ccnt, c0a, c1a, c0b, c1b);
  OZ_CHECK_LAUNCH();
  return OZ_OK;
}

// Factor one m x jb column panel in place (solve.py:66-91 for columns
// j..j+jb of the global matrix): `a` points at the panel's diagonal corner,
// rows keep the global numbering through `base` (= j).  Interchanges are
// applied to the panel's own columns only; ipiv[0..jb) receives the global
// pivot rows, info the first zero pivot (global column + 1), growth the max
// |entry| seen.  The caller applies ipiv to the other columns (laswp_ipiv).
// Widest window (<= PANEL_W) whose m-row slab fits in the shared memory of
// max_ctas CTAs: tall panels (distributed runs, m ~ 1e5) use narrower windows.
int panel_width_for(int64_t m, int max_ctas) {
  if (const int lw = leaf_width_for(m, max_ctas)) return lw;
  const int64_t cap = panel_smem_cap();
  // short panels go to the cluster variant (<= panel_cluster_max() CTAs):
  // the window must fit m / cmax rows per CTA
  const int cmax = panel_cluster_max();
  const int64_t ctas = cmax >= 2 && m <= panel_cluster_rows() ? std::min(cmax, max_ctas)
                                                             : max_ctas;
  const int64_t rows = ceil_div(m, ctas);
  int64_t w = (cap / rows - (int64_t)sizeof(int)) / (int64_t)sizeof(double);
  if (w > PANEL_W) w = PANEL_W;
  if (w >= 16) w &= ~7;  // keep the window a multiple of 8 columns
  return (int)w;
}

// Recursive panel factorization of panel columns [c0, c1) (rows c0..m-1 of
// the panel's local coordinates).  Leaves of at most wmax columns are one
// cooperative window kernel each, whose interchanges are applied at once to
// every other panel column; an inner node factors its left half, updates the
// right half with trsm + one DGEMM of depth (mid - c0), then factors the right
// half.  Same arithmetic class as solve.py:75-90 (bit-exact inside a leaf,
// blocked FP64 updates across leaves) but the in-panel updates are GEMMs of
// depth nb/2, nb/4, ... instead of nb/wmax rank-wmax updates.
int panel_rec(double* a, int64_t lda, int64_t m, int64_t jb, int64_t c0, int64_t c1, int wmax,
              int64_t base, int32_t* ipiv, int32_t* info, unsigned long long* growth,
              const LuWs& ws, cudaStream_t st, int ctas) {
  const int64_t w = c1 - c0;
  const int cap = ctas < sm_count() ? ctas : 0;  // side-stream panel: keep to its SMs
  if (w <= wmax) {
    OZ_TRY(panel_window(a, lda, c0, m - c0, (int)w, base, ipiv, info, growth, ws, st, ctas));
    return apply_list(a, lda, ws, 0, c0, c1, jb, st, cap);
  }
  int64_t mid = c0 + ((w / 2 + wmax - 1) / wmax) * wmax;
  if (mid >= c1) mid = c0 + wmax;
  OZ_TRY(panel_rec(a, lda, m, jb, c0, mid, wmax, base, ipiv, info, growth, ws, st, ctas));
  const int64_t kk = mid - c0, right = c1 - mid;
  OZ_TRY(trsm_blocked(a, lda, c0, kk, a + mid * lda + c0, lda, right, st, cap));
  if (m - mid > 0) {
    const int tag = prof_start(st);
    OZ_TRY(dgemm(0, 0, m - mid, right, kk, -1.0, a + c0 * lda + mid, lda, a + mid * lda + c0,
                 lda, 1.0, a + mid * lda + mid, lda, st, cap));
    prof_stop(tag, st, PROF_DGEMM_PANEL, 2.0 * (m - mid) * right * kk);
  }
  return panel_rec(a, lda, m, jb, mid, c1, wmax, base, ipiv, info, growth, ws, st, ctas);
}

// Factor one m x jb column panel in place (solve.py:66-91 for columns
// j..j+jb of the global matrix): `a` points at the panel's diagonal corner,
// rows keep the global numbering through `base` (= j).  Interchanges are
// applied to the panel's own columns only; ipiv[0..jb) receives the global
// pivot rows, info the first zero pivot (global column + 1), growth the max
// |entry| seen.  The caller applies ipiv to the other columns (laswp_ipiv).
int panel_factor(double* a, int64_t lda, int64_t m, int64_t jb, int64_t base, int32_t* ipiv,
                 int32_t* info, unsigned long long* growth, const LuWs& ws, cudaStream_t st,
                 int max_ctas = 0) {
  const int ctas = max_ctas > 0 && max_ctas < sm_count() ? max_ctas : sm_count();
  const int wmax = panel_width_for(m, ctas);
  OZ_REQUIRE(wmax >= 1, OZ_UNSUPPORTED, "a panel of %lld rows does not fit on chip",
             (long long)m);
  return panel_rec(a, lda, m, jb, 0, jb, wmax, base, ipiv, info, growth, ws, st, ctas);
}

// The Schur update A22 (m x ncols) -= A21 (m x jb) @ U12 (jb x ncols) through
// the selected backend (solve.py:130-134), growth = max |A22| after the
// update (:135).  Split once (schur_split), then update any column range
// [c0, c1) of A22 (schur_cols) — the look-ahead updates the next panel's
// columns first and the rest on fewer SMs.
struct Schur {
  int backend;
  int64_t m, ncols, jb;
  const double* a21;
  int64_t lda21;
  const double* u12;
  int64_t ldu;
  double* a22;
  int64_t lda22;
  int k, q, npairs;
  const int32_t *pa, *pb, *ps;
  unsigned long long* growth;
};

// Split A21 (row-scaled) and the U12 columns [c0, c1) (column-scaled) into the
// slice stacks; a column range of U12 can be split on its own for per-vector
// scaling (each column has its own exponent), not for GLOBAL (one exponent
// over all of U12).
int schur_split_part(const Schur& s, bool with_a, int64_t c0, int64_t c1, const LuWs& ws,
                     cudaStream_t st) {
  if (s.backend == 0 || s.m <= 0 || s.ncols <= 0) return OZ_OK;
  const int tag = prof_start(st);
  // backend 1: per-vector exponents, 2: one exponent per operand (GLOBAL, split.py:131-134)
  const int mode = s.backend == 2 ? OZ_GLOBAL : OZ_PER_VECTOR;
  if (with_a)
    OZ_TRY(split_launch(s.a21, s.m, s.jb, 1, s.lda21, OZ_ROW_SCALED, mode, s.k, s.q, ws.slA,
                        ws.ldK, s.m * ws.ldK, ws.expA, ws.split_aux, st));
  if (c1 > c0)
    OZ_TRY(split_launch(s.u12 + c0 * s.ldu, s.jb, c1 - c0, 1, s.ldu, OZ_COL_SCALED, mode, s.k,
                        s.q, ws.slB + c0 * ws.ldK, ws.ldK, s.ncols * ws.ldK, ws.expB + c0,
                        ws.split_aux, st));
  prof_stop(tag, st, PROF_SPLIT,
            (double)((with_a ? s.m : 0) + (c1 - c0)) * s.jb * (8.0 + s.k));
  return OZ_OK;
}

int schur_split(const Schur& s, const LuWs& ws, cudaStream_t st) {
  return schur_split_part(s, true, 0, s.ncols, ws, st);
}

int schur_cols(const Schur& s, int64_t c0, int64_t c1, const LuWs& ws, cudaStream_t st,
               int max_ctas = 0) {
  const int64_t nc = c1 - c0;
  if (s.m <= 0 || nc <= 0) return OZ_OK;
  double* c = s.a22 + c0 * s.lda22;
  if (s.backend == 0) {
    const int tag = prof_start(st);
    OZ_TRY(dgemm(0, 0, s.m, nc, s.jb, -1.0, s.a21, s.lda21, s.u12 + c0 * s.ldu, s.ldu, 1.0, c,
                 s.lda22, st));
    prof_stop(tag, st, PROF_DGEMM, 2.0 * s.m * nc * s.jb);
    return max_abs(c, s.m, nc, 1, s.lda22, 0, 0, s.growth, st);
  }
  const int tag = prof_start(st);
  OZ_TRY(gemm_emu_launch(s.m, nc, s.jb, ws.slA, ws.ldK, s.m * ws.ldK, s.k, ws.expA,
                         ws.slB + c0 * ws.ldK, ws.ldK, s.ncols * ws.ldK, s.k, ws.expB + c0,
                         s.npairs, s.pa, s.pb, s.ps, s.q, -1.0, 1.0, c, s.lda22, 1, s.growth,
                         st, max_ctas));
  prof_stop(tag, st, PROF_EMU_GEMM, 2.0 * s.npairs * s.m * nc * s.jb, max_ctas);
  return OZ_OK;
}

int schur_update(int backend, int64_t m, int64_t ncols, int64_t jb, const double* a21,
                 int64_t lda21, const double* u12, int64_t ldu, double* a22, int64_t lda22, int k,
                 int q, int npairs, const int32_t* pa, const int32_t* pb, const int32_t* ps,
                 unsigned long long* growth, const LuWs& ws, cudaStream_t st) {
  const Schur s{backend, m, ncols, jb, a21, lda21, u12, ldu, a22, lda22, k, q, npairs, pa, pb,
                ps, growth};
  OZ_TRY(schur_split(s, ws, st));
  return schur_cols(s, 0, ncols, ws, st);
}

// Look-ahead (depth 1): the next panel is factored on a side stream with S
// CTAs while the rest of the Schur update runs on the other SMs.
// OZ_LOOKAHEAD_SMS: 0 disables, a positive value fixes S, unset (-1) sizes S
// per step so the panel (latency floor ~3 us per column plus ~0.011 us per
// row per CTA) and the GEMM (~2.3 POPS on the full chip) take equal time.
int lookahead_sms() {
  static int v = -2;
  if (v == -2) {
    const char* e = getenv("OZ_LOOKAHEAD_SMS");
    v = e ? atoi(e) : -1;
    if (v < -1) v = -1;
    if (v > 0) v &= ~1;
  }
  return v;
}

int la_step() {  // tuning: granularity of the look-ahead SM search
  static const int v = getenv("OZ_LA_STEP") ? atoi(getenv("OZ_LA_STEP")) : 2;
  return v > 0 ? v : 2;  // measured: 2 vs 8 -> 497 vs 499-505 ms at n = 32768
}
int lookahead_split(int setting, int64_t m, int64_t nb, int npairs, int sms, int64_t ncols = -1) {
  if (setting >= 0) return setting;
  if (npairs <= 0) return 40;  // native DGEMM Schur update: fixed split (measured best)
  if (ncols < 0) ncols = m;    // single GPU: the whole trailing matrix
  const double ops = 2.0 * npairs * (double)m * (double)ncols * (double)nb;
  const double rate = 2.3e15;  // emulated INT8 ops/s on the full chip
  int best = 16;
  double best_t = 1e30;
  for (int s = 16; s <= sms / 2; s += la_step()) {
    const double tp = nb * (3e-6 + 1.1e-8 * (double)m / s);
    const double tg = ops / (rate * (double)(sms - s) / sms);
    const double t = tp > tg ? tp : tg;
    if (t < best_t) {
      best_t = t;
      best = s;
    }
  }
  return best;
}

// Two-phase look-ahead (emulated backend, single GPU): the next panel runs on S
// CTAs of a side stream while the first X columns of this step's Schur update
// run on the other sms - S; the remaining columns start once the panel is done,
// on every SM.  A tall panel is latency-bound (it speeds up far less than
// linearly in S), so a larger S for a shorter time beats a narrow S for the
// whole step.  Model (fit to OZ_LU_TRACE timelines at n = 32768, in-LU times,
// GEMM running beside the panel): panel ~ nb * (5.2 us + 0.012 us * m / S);
// GEMM at emu_rate(pairs) on all SMs; interchanges + trsm + split of the rest
// before the GEMM ~ 0.8 ms + 0.117 us per column.  OZ_LA_TWO_PHASE=0 keeps the
// single-phase split (lookahead_split).
struct LaPlan {
  int sms;         // panel CTAs
  int64_t cols1;   // columns of the rest updated beside the panel (phase 1)
};
bool la_two_phase() {
  static const bool v = [] {
    const char* e = getenv("OZ_LA_TWO_PHASE");
    return e == nullptr || atoi(e) != 0;
  }();
  return v;
}
// Emulated GEMM rate in the LU shape (K = nb = 1024, all SMs), INT8 ops/s,
// measured with scripts/probe.py kern (profiles/r02_gemm_rate_lu_shape.txt):
// few pairs leave the per-group FP64 epilogue less MMA work to hide behind.
double emu_rate(int npairs) {
  static const double scale = getenv("OZ_LA_RATE_SCALE") ? atof(getenv("OZ_LA_RATE_SCALE"))
                                                          : 1.0;  // tuning
  // measured 1.45 / 1.9 / 2.1 / 2.2 POPS, scaled by 1.09: planning with the
  // slightly optimistic rate measured faster at n = 32768, k = 7
  // (profiles/r02_la_rate_ab.txt: 485 vs 492 ms over three interleaved runs)
  const double r = npairs <= 6 ? 1.45e15 : npairs <= 10 ? 1.9e15 : npairs <= 15 ? 2.1e15 : 2.2e15;
  return r * 1.09 * scale;
}

// Modelled in-LU panel time (s) of an m x nb panel on s SMs (the fit of the
// two-phase comment above).  A model in which register-leaf panels do not
// depend on s (true standalone) picked the fewest SMs that fit the leaf and
// lost: beside a GEMM on more SMs the panel ran 1.2-1.5x slower
// (profiles/r02bt_panel_model_ab.log); the 1/s term stands in for that.
double panel_model(int64_t m, int64_t nb, int s) {
  static const double a = getenv("OZ_LA_TP_A") ? atof(getenv("OZ_LA_TP_A")) : 5.2e-6;  // tuning
  static const double b = getenv("OZ_LA_TP_B") ? atof(getenv("OZ_LA_TP_B")) : 1.2e-8;
  return (double)nb * (a + b * (double)m / s);
}

// Panel time for sizing phase 1 once S is chosen: panels on the register
// leaves finish ahead of the model the S search uses — ~20 % with 32/64-column
// windows (<= 512 rows per SM), ~10 % with the tall 16-column variant
// (OZ_LU_TRACE "p1-panel" column at n = 32768: phase 1 ran 0.6-2.5 ms past
// the panel in steps 8-27 with the plain model, the panel's SMs idle;
// profiles/r02bz_phase1_ab.log); shared-memory leaves ~6 % behind it.
double panel_time_p1(int64_t m, int64_t nb, int s) {
  static const double f = getenv("OZ_LA_P1_REG") ? atof(getenv("OZ_LA_P1_REG")) : 0.8;  // tuning
  static const double f16 = getenv("OZ_LA_P1_TALL") ? atof(getenv("OZ_LA_P1_TALL")) : 0.9;
  static const double fs = getenv("OZ_LA_P1_SMEM") ? atof(getenv("OZ_LA_P1_SMEM")) : 1.06;
  const int w = leaf_width_for(m, s);
  return panel_model(m, nb, s) * (w >= 32 ? f : w > 0 ? f16 : fs);
}

// phase-1 width for a given S: the columns sms - S SMs update while the panel runs
int64_t phase1_cols(int s, int64_t m, int64_t nb, int npairs, int sms, int64_t rest) {
  if (rest <= 0 || npairs <= 0) return rest > 0 ? rest : 0;
  const double rate = emu_rate(npairs);
  const double ops_per_col = 2.0 * npairs * (double)m * (double)nb;
  const double t_lt = 0.8e-3 + 1.17e-7 * (double)rest;
  const double tp = panel_time_p1(m, nb, s);
  const double r1 = rate * (double)(sms - s) / sms;
  double x = (tp - t_lt) * r1 / ops_per_col;
  if (x < 0) x = 0;
  if (x > (double)rest) x = (double)rest;
  return std::min<int64_t>(rest, ((int64_t)x + 127) / 128 * 128);  // whole 128-column tiles
}

LaPlan lookahead_plan(int setting, int64_t m, int64_t nb, int npairs, int sms, int64_t rest) {
  LaPlan best{lookahead_split(setting, m, nb, npairs, sms), rest};
  if (!la_two_phase() || setting >= 0 || npairs <= 0 || rest <= 0) return best;
  const double rate = emu_rate(npairs);
  const double ops_per_col = 2.0 * npairs * (double)m * (double)nb;
  const double t_lt = 0.8e-3 + 1.17e-7 * (double)rest;
  double best_t = 1e30;
  for (int s = 16; s <= sms - 16; s += 2) {
    const double tp = panel_model(m, nb, s);
    const double r1 = rate * (double)(sms - s) / sms;
    // phase-1 columns: what the reduced grid finishes while the panel runs
    double x = (tp - t_lt) * r1 / ops_per_col;
    if (x < 0) x = 0;
    if (x > (double)rest) x = (double)rest;
    const double t1 = t_lt + x * ops_per_col / r1;
    const double t = (t1 > tp ? t1 : tp) + ((double)rest - x) * ops_per_col / rate;
    if (t < best_t) {
      best_t = t;
      best.sms = s;
    }
  }
  // Tallest panels: where the search lands on a shared-memory leaf, take the
  // fewest SMs that fit the 1024-row register leaf instead (up to
  // OZ_LA_TALL_MAX): about the same SM-time, a panel ~2x shorter — which the
  // overlapped upload needs, its first steps being a chain of panels.
  static const int tall_max = getenv("OZ_LA_TALL_MAX") ? atoi(getenv("OZ_LA_TALL_MAX")) : 32;
  if (tall_max > 0 && leaf_tall_enabled() && leaf_width_for(m, best.sms) == 0) {
    const int st = (int)((ceil_div(m, (int64_t)1024) + 1) & ~1);
    if (st > best.sms && st <= tall_max && leaf_width_for(m, st) > 0) best.sms = st;
  }
  // phase 1 sized with the refined panel time at the chosen S (whole
  // 128-column GEMM tiles)
  best.cols1 = phase1_cols(best.sms, m, nb, npairs, sms, rest);
  return best;
}

// SMs of the look-ahead panel that factors columns [j, j + nb) of an m-row
// trailing matrix (m = n - j) beside the update of the step before it, whose
// other columns number m - min(nb, m).  Every driver (the right-looking loop,
// the upload phase, the distributed 1 x Q driver through oz_lookahead_sms)
// sizes a given panel the same way: the panel's leaf widths depend on its SM
// cap, so equal caps keep the factors bit-identical across the drivers.
int panel_sms(int setting, int64_t m, int64_t nb, int npairs, int sms) {
  return lookahead_plan(setting, m, nb, npairs, sms, m - std::min<int64_t>(nb, m)).sms;
}

// OZ_LU_TRACE=1: per-step event timeline of the driver on stderr (tuning only)
struct LuTrace {
  bool on = false;
  std::vector<cudaEvent_t> ev;
  std::vector<int> split;  // look-ahead SMs per step
  std::vector<cudaEvent_t> sub;  // per look-ahead step: after laswp / trsm / split of the rest
  void mark_sub(cudaStream_t st) {
    if (!on) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, st);
    sub.push_back(e);
  }
  void mark(cudaStream_t st) {
    if (!on) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, st);
    ev.push_back(e);
  }
};

struct SideStream {
  cudaStream_t st = nullptr;
  cudaEvent_t ready = nullptr, done = nullptr;
  cudaStream_t aux = nullptr;  // early steps: the rest's row interchanges
  cudaEvent_t aux_ready = nullptr, aux_done = nullptr;
  cudaStream_t step[8] = {};  // upload phase: one stream per wavefront step
};
int side_stream(SideStream** out) {
  static thread_local std::vector<SideStream> per_dev;
  int dev = 0;
  OZ_CHECK_CUDA(cudaGetDevice(&dev));
  if ((int)per_dev.size() <= dev) per_dev.resize(dev + 1);
  SideStream& s = per_dev[dev];
  if (!s.st) {
    int lo = 0, hi = 0;
    OZ_CHECK_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    const char* pr = getenv("OZ_SIDE_PRIO");  // tuning: 1 = highest priority for the panel
    OZ_CHECK_CUDA(cudaStreamCreateWithPriority(&s.st, cudaStreamNonBlocking,
                                               pr && atoi(pr) ? hi : lo));
    OZ_CHECK_CUDA(cudaEventCreateWithFlags(&s.ready, cudaEventDisableTiming));
    OZ_CHECK_CUDA(cudaEventCreateWithFlags(&s.done, cudaEventDisableTiming));
    OZ_CHECK_CUDA(cudaStreamCreateWithPriority(&s.aux, cudaStreamNonBlocking, lo));
    OZ_CHECK_CUDA(cudaEventCreateWithFlags(&s.aux_ready, cudaEventDisableTiming));
    OZ_CHECK_CUDA(cudaEventCreateWithFlags(&s.aux_done, cudaEventDisableTiming));
    for (auto& x : s.step) OZ_CHECK_CUDA(cudaStreamCreateWithPriority(&x, cudaStreamNonBlocking, lo));
  }
  *out = &s;
  return OZ_OK;
}

}  // namespace

// ------------------------------------------------------------------- LU driver
// chunk_ready (may be null): the caller is still uploading the matrix in
// column chunks of chunk_cols; event c fires once columns [c*chunk_cols,
// (c+1)*chunk_cols) are in place.  Panel 0, the update of panel 1's columns
// and panel 1 (side stream) start as soon as their chunks are in; step 0's
// update of every other column is streamed chunk by chunk behind the upload.
int lu_factor(double* a, int64_t n, int64_t lda, int64_t nb, int backend, int k, int q,
              int npairs, const int32_t* pa, const int32_t* pb, const int32_t* ps,
              int32_t* ipiv, double* stats, int32_t* info, void* workspace, size_t ws_bytes,
              cudaStream_t st, const cudaEvent_t* chunk_ready = nullptr,
              int64_t chunk_cols = 0) {
  OZ_REQUIRE(n >= 1, OZ_INVALID_PARAMS, "empty matrices are not supported");
  OZ_REQUIRE(nb >= 1 && nb <= n, OZ_INVALID_PARAMS, "lu_block must be in 1..%lld, got %lld",
             (long long)n, (long long)nb);
  OZ_REQUIRE(lda >= n, OZ_INVALID_PARAMS, "lda < n");
  OZ_REQUIRE(backend >= 0 && backend <= 2, OZ_INVALID_PARAMS, "bad backend %d", backend);
  LuWs ws;
  const int planes = backend != 0 ? (q > 7 ? 2 * k : k) : 0;  // int8 planes per slice stack
  const size_t need = lu_ws_layout(n, nb, planes, (uint8_t*)workspace, &ws);
  OZ_REQUIRE(ws_bytes >= need, OZ_INVALID_PARAMS, "workspace too small (%zu < %zu)", ws_bytes,
             need);
  OZ_CHECK_CUDA(cudaMemsetAsync(ws.bar, 0, sizeof(GridBar), st));
  OZ_CHECK_CUDA(cudaMemsetAsync(ws.cand, 0, sizeof(double) * 2 * 1024 * CAND_STRIDE, st));
  OZ_CHECK_CUDA(cudaMemsetAsync(ws.bits, 0, 4 * sizeof(unsigned long long), st));
  OZ_CHECK_CUDA(cudaMemsetAsync(info, 0, sizeof(int32_t), st));
  // columns [0, ready_cols) are in place and folded into max |A|
  int64_t ready_cols = 0;
  auto wait_until = [&](int64_t c1) -> int {
    if (c1 > n) c1 = n;
    const int64_t from = ready_cols;
    while (ready_cols < c1) {
      if (chunk_ready) {
        OZ_CHECK_CUDA(cudaStreamWaitEvent(st, chunk_ready[ready_cols / chunk_cols], 0));
        ready_cols = std::min<int64_t>(n, (ready_cols / chunk_cols + 1) * chunk_cols);
      } else {
        ready_cols = n;
      }
    }
    if (ready_cols > from)
      OZ_TRY(max_abs(a + from * lda, n, ready_cols - from, 1, lda, 0, 0, ws.bits + 1, st));
    return OZ_OK;
  };
  auto wait_cols = [&]() -> int { return wait_until(n); };
  OZ_TRY(wait_until(std::min<int64_t>(n, 2 * nb)));

  const int la_setting = lookahead_sms();
  SideStream* side = nullptr;
  if (la_setting != 0) OZ_TRY(side_stream(&side));
  // panel 0; every later panel is factored at the end of the previous step
  OZ_TRY(panel_factor(a, lda, n, nb < n ? nb : n, 0, ipiv, info, ws.bits, ws, st));
  LuTrace tr;
  tr.on = getenv("OZ_LU_TRACE") != nullptr;
  int64_t j_start = 0;
  // ---- upload phase (overlapped host input): the first S steps are applied
  // chunk by chunk as the columns arrive (left-looking over the chunks, same
  // per-column sequence of interchanges and updates as the right-looking
  // loop), panels 1..S factored on the side stream as soon as their columns
  // have received the earlier steps.  The loop below continues at step S.
  const int64_t nblk = ceil_div(n, nb);
  // measured at n = 32768, nb = 1024 with per-step streams and the tall-leaf
  // panel SMs: S = 3/4/5 -> 511/497/498 ms e2e (profiles/r02ci_upload_ab.log;
  // single stream, smem-leaf panels: 3/4/5/6 -> 567/578/585/592)
  static const int phase_env = getenv("OZ_UPLOAD_STEPS") ? atoi(getenv("OZ_UPLOAD_STEPS")) : 4;
  const int S = (int)std::min<int64_t>(phase_env, nblk - 2);
  if (chunk_ready && side != nullptr && backend != 2 && S >= 1 && ready_cols < n &&
      chunk_cols % nb == 0) {
    const size_t slab = (size_t)(backend != 0 ? (q > 7 ? 2 * k : k) : 0) * (size_t)n * ws.ldK;
    int8_t* sl_buf = nullptr;
    int32_t* ex_buf = nullptr;
    if (backend != 0) {
      keep_pool_mapped();
      OZ_CHECK_CUDA(cudaMallocAsync(&sl_buf, slab * S, st));
      OZ_CHECK_CUDA(cudaMallocAsync(&ex_buf, sizeof(int32_t) * n * S, st));
    }
    std::vector<cudaEvent_t> pdone(S + 1, nullptr);
    for (auto& e : pdone) OZ_CHECK_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    std::vector<LuWs> wss(S, ws);
    std::vector<Schur> scs;
    for (int s2 = 0; s2 < S; ++s2) {
      const int64_t j0 = s2 * nb, jbs = std::min<int64_t>(nb, n - j0), r = n - j0 - jbs;
      if (backend != 0) {
        wss[s2].slA = sl_buf + slab * s2;
        wss[s2].expA = ex_buf + (size_t)n * s2;
      }
      scs.push_back(Schur{backend, r, r, jbs, a + j0 * lda + (j0 + jbs), lda,
                          a + (j0 + jbs) * lda + j0, lda, a + (j0 + jbs) * lda + (j0 + jbs), lda,
                          k, q, npairs, pa, pb, ps, ws.bits});
    }
    // Each wavefront step runs on its own stream (OZ_UPLOAD_STREAMS=0: all on
    // the caller's stream), so a step waiting for its panel does not hold up
    // the earlier steps' updates of newly arrived blocks; block c's step s
    // follows its step s - 1 through an event.  Each step stream composes its
    // interchange lists in its own buffers.
    static const bool step_streams_env =
        !getenv("OZ_UPLOAD_STREAMS") || atoi(getenv("OZ_UPLOAD_STREAMS")) != 0;
    const bool step_streams = step_streams_env && S <= 8;
    std::vector<cudaStream_t> sst(S, st);
    int32_t* cmp_buf = nullptr;
    const int64_t nch = ceil_div(n, chunk_cols);
    std::vector<cudaEvent_t> cdone;  // [s * nch + c]: block c has received step s
    cudaEvent_t evm = nullptr;
    uint8_t* stepb_buf = nullptr;  // per step: U12 slices + exponents of one block, split scratch
    const size_t slabB = (size_t)planes * (size_t)chunk_cols * ws.ldK;
    const size_t stepb = align_up(slabB) + align_up(sizeof(int32_t) * chunk_cols) + 256;
    if (step_streams) {
      for (int s2 = 0; s2 < S; ++s2) sst[s2] = side->step[s2];
      const size_t per = 2 * LSWP_MAX + 4;
      OZ_CHECK_CUDA(cudaMallocAsync(&cmp_buf, sizeof(int32_t) * per * S, st));
      OZ_CHECK_CUDA(cudaMallocAsync(&stepb_buf, stepb * S, st));
      for (int s2 = 0; s2 < S; ++s2) {
        wss[s2].cdst = cmp_buf + per * s2;
        wss[s2].csrc = wss[s2].cdst + LSWP_MAX;
        wss[s2].ccnt = wss[s2].csrc + LSWP_MAX;
        uint8_t* b0 = stepb_buf + stepb * s2;
        wss[s2].slB = reinterpret_cast<int8_t*>(b0);
        wss[s2].expB = reinterpret_cast<int32_t*>(b0 + align_up(slabB));
        wss[s2].split_aux = b0 + align_up(slabB) + align_up(sizeof(int32_t) * chunk_cols);
      }
      cdone.resize((size_t)S * nch);
      for (auto& e : cdone) OZ_CHECK_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      OZ_CHECK_CUDA(cudaEventCreateWithFlags(&evm, cudaEventDisableTiming));
      OZ_CHECK_CUDA(cudaEventRecord(evm, st));  // allocations and memsets above
      for (int s2 = 0; s2 < S; ++s2) OZ_CHECK_CUDA(cudaStreamWaitEvent(sst[s2], evm, 0));
    }
    // OZ_LU_TRACE: timeline of the wavefront (task ends per step, panel ends)
    const bool ptrace = getenv("OZ_LU_TRACE") != nullptr;
    cudaEvent_t pt0 = nullptr;
    std::vector<std::pair<std::string, cudaEvent_t>> pev;
    auto pmark = [&](const std::string& name, cudaStream_t s3) {
      if (!ptrace) return;
      cudaEvent_t e;
      cudaEventCreate(&e);
      cudaEventRecord(e, s3);
      pev.emplace_back(name, e);
    };
    if (ptrace) {
      cudaEventCreate(&pt0);
      cudaEventRecord(pt0, st);
    }
    std::vector<bool> have(S + 1, false);  // panel s ready on its step stream (A21 split)
    auto ensure_panel = [&](int s2) -> int {
      if (have[s2]) return OZ_OK;
      if (s2 > 0) OZ_CHECK_CUDA(cudaStreamWaitEvent(sst[s2], pdone[s2], 0));
      if (s2 < S) OZ_TRY(schur_split_part(scs[s2], true, 0, 0, wss[s2], sst[s2]));
      // The interchanges of step s2 on the finished L columns [0, s2*nb) are
      // deferred to the end of the phase: they reorder the A21 rows of the
      // earlier steps, whose updates of later blocks are still pending (the
      // native backend reads A21 from the matrix itself).
      have[s2] = true;
      return OZ_OK;
    };
    // tuning: SMs of the phase's side-stream panels (default: the look-ahead
    // model; 48 measured equal, 74 slower at n = 32768)
    static const int phase_sms_env = getenv("OZ_UPLOAD_SMS") ? atoi(getenv("OZ_UPLOAD_SMS")) : 0;
    auto phase_panel_sms = [&](int64_t p0) {
      return phase_sms_env > 0 ? (phase_sms_env & ~1)
                               : panel_sms(la_setting, n - p0, nb, backend != 0 ? npairs : 0,
                                           sm_count());
    };
    const int la_sms = phase_panel_sms(nb);  // the phase's GEMM leaves panel 1's SMs free
    int next_panel = 1;
    // wavefront over (step, block): diagonal d applies step s to block d - s,
    // so step 0 keeps up with the upload while later steps wait for their
    // panels (each block still receives steps 0, 1, ... in order)
    for (int64_t d = 0; d < nch + S - 1; ++d) {
      for (int s2 = 0; s2 < S; ++s2) {
        const int64_t c = d - s2;
        if (c < 0 || c >= nch) continue;
        const int64_t c0 = c * chunk_cols, c1 = std::min<int64_t>(n, c0 + chunk_cols);
        const cudaStream_t ss = sst[s2];
        OZ_TRY(wait_until(c1));  // the block's arrival (and max |A|) on the caller's stream
        if (step_streams) {
          if (s2 == 0) {
            OZ_CHECK_CUDA(cudaEventRecord(evm, st));
            OZ_CHECK_CUDA(cudaStreamWaitEvent(ss, evm, 0));
          } else {
            OZ_CHECK_CUDA(cudaStreamWaitEvent(ss, cdone[(size_t)(s2 - 1) * nch + c], 0));
          }
        }
        const int64_t j0 = s2 * nb, t0 = j0 + std::min<int64_t>(nb, n - j0);
        const int64_t r0 = std::max(c0, t0);
        if (r0 >= c1) {  // this step's trailing columns start after the block
          if (step_streams) OZ_CHECK_CUDA(cudaEventRecord(cdone[(size_t)s2 * nch + c], ss));
          continue;
        }
        OZ_TRY(ensure_panel(s2));
        const int jbs = (int)std::min<int64_t>(nb, n - j0);
        OZ_TRY(laswp_ipiv(a, lda, r0, c1, 0, 0, j0, ipiv + j0, jbs, wss[s2], ss));
        OZ_TRY(trsm_blocked(a, lda, j0, jbs, a + r0 * lda + j0, lda, c1 - r0, ss));
        if (step_streams) {
          // this block's columns as a Schur update of their own: the U12
          // slices live in the step's block-sized buffer (steps run at once)
          Schur scc = scs[s2];
          scc.ncols = c1 - r0;
          scc.u12 = a + r0 * lda + j0;
          scc.a22 = a + r0 * lda + t0;
          OZ_TRY(schur_split_part(scc, false, 0, c1 - r0, wss[s2], ss));
          OZ_TRY(schur_cols(scc, 0, c1 - r0, wss[s2], ss, sm_count() - la_sms));
        } else {
          OZ_TRY(schur_split_part(scs[s2], false, r0 - t0, c1 - t0, wss[s2], ss));
          OZ_TRY(schur_cols(scs[s2], r0 - t0, c1 - t0, wss[s2], ss, sm_count() - la_sms));
        }
        if (step_streams) OZ_CHECK_CUDA(cudaEventRecord(cdone[(size_t)s2 * nch + c], ss));
        pmark("s" + std::to_string(s2) + "c" + std::to_string(c), ss);
        // panel s2+1 has now received steps 0..s2 if its columns are in this block
        const int64_t p0 = (int64_t)(s2 + 1) * nb;
        if (next_panel == s2 + 1 && s2 + 1 <= S && p0 >= r0 &&
            p0 + std::min<int64_t>(nb, n - p0) <= c1) {
          OZ_CHECK_CUDA(cudaEventRecord(side->ready, ss));
          OZ_CHECK_CUDA(cudaStreamWaitEvent(side->st, side->ready, 0));
          OZ_TRY(panel_factor(a + p0 * lda + p0, lda, n - p0, std::min<int64_t>(nb, n - p0), p0,
                              ipiv + p0, info, ws.bits, ws, side->st, phase_panel_sms(p0)));
          OZ_CHECK_CUDA(cudaEventRecord(pdone[s2 + 1], side->st));
          pmark("P" + std::to_string(s2 + 1), side->st);
          ++next_panel;
        }
      }
    }
    OZ_REQUIRE(next_panel == S + 1, OZ_UNSUPPORTED, "upload phase did not reach panel %d", S);
    OZ_CHECK_CUDA(cudaStreamWaitEvent(st, pdone[S], 0));
    if (ptrace) {
      // chunk arrivals: the caller's events (timing may be disabled on them)
      for (int64_t c = 0; c < nch; ++c) {
        cudaStreamWaitEvent(side->aux, chunk_ready[c], 0);
        pmark("a" + std::to_string(c), side->aux);
      }
    }
    if (step_streams) {
      for (int s2 = 0; s2 < S; ++s2) {
        OZ_CHECK_CUDA(cudaEventRecord(evm, sst[s2]));
        OZ_CHECK_CUDA(cudaStreamWaitEvent(st, evm, 0));
      }
      OZ_CHECK_CUDA(cudaFreeAsync(cmp_buf, st));
      OZ_CHECK_CUDA(cudaFreeAsync(stepb_buf, st));
      for (auto e : cdone) cudaEventDestroy(e);
      cudaEventDestroy(evm);
    }
    // the deferred interchanges of steps 1..S-1 on their L columns, in step
    // order (every A21 of those steps has been consumed by now); step S's
    // follow in the loop below, before anything reads those columns again
    for (int s2 = 1; s2 < S; ++s2)
      OZ_TRY(laswp_ipiv(a, lda, 0, s2 * nb, 0, 0, s2 * nb, ipiv + s2 * nb,
                        (int)std::min<int64_t>(nb, n - s2 * nb), ws, st));
    // finalized U rows of steps < S (step S's interchanges, the L columns
    // included, are applied by the loop below as usual)
    for (int s2 = 0; s2 < S; ++s2) {
      const int64_t j0 = s2 * nb;
      OZ_TRY(max_abs(a + j0 * lda + j0, std::min<int64_t>(nb, n - j0), n - j0, 1, lda, 1, 0,
                     ws.bits, st));
    }
    if (backend != 0) {
      OZ_CHECK_CUDA(cudaFreeAsync(sl_buf, st));
      OZ_CHECK_CUDA(cudaFreeAsync(ex_buf, st));
    }
    for (auto e : pdone) cudaEventDestroy(e);
    if (ptrace) {
      pmark("phase_end", st);
      cudaStreamSynchronize(st);
      cudaStreamSynchronize(side->aux);
      fprintf(stderr, "upload phase timeline [ms]:");
      for (auto& kv : pev) {
        float t = 0;
        cudaEventElapsedTime(&t, pt0, kv.second);
        fprintf(stderr, " %s=%.1f", kv.first.c_str(), t);
        cudaEventDestroy(kv.second);
      }
      fprintf(stderr, "\n");
      cudaEventDestroy(pt0);
    }
    j_start = (int64_t)S * nb;
  }
  for (int64_t j = j_start; j < n; j += nb) {
    const int64_t jb = nb < n - j ? nb : n - j;
    const int64_t rest = n - j - jb;
    const int64_t jb2 = nb < rest ? nb : rest;  // the next panel's width
    double* a12 = a + (j + jb) * lda + j;
    double* a21 = a + j * lda + (j + jb);
    double* a22 = a + (j + jb) * lda + (j + jb);
    const Schur sc{backend, rest, rest, jb, a21, lda, a12, lda, a22, lda, k, q, npairs, pa, pb,
                   ps, ws.bits};
    // Look-ahead with the next panel's columns on the critical path only:
    // swaps, trsm, split and Schur update of those jb2 columns, then the next
    // panel on the side stream while the rest of this step (swaps of the other
    // columns, trsm, split and update of the remaining columns) runs beside it.
    // GLOBAL scaling needs all of U12 for its one exponent: no column split.
    const bool la = side != nullptr && rest > jb2 && backend != 2;
    // Early (GEMM-bound) steps: the interchanges of every column but the next
    // panel's run on an aux stream with aux_ctas CTAs beside the serial chain
    // (the next panel's columns: interchanges, trsm, split, update on
    // sms - aux_ctas SMs).  Row swaps are DRAM-latency-bound, so a few CTAs
    // keep most of their throughput.  OZ_AUX_SWAPS_CTAS=0 disables.
    // Measured at n = 32768, k = 7 (profiles/r02_aux_swaps_ab.txt, three
    // interleaved runs each): off 488.7 ms, 16 CTAs 486.5, 24 481.8, 32 481.5,
    // 48 486.7; 32 CTAs from m >= 8192 480.6.
    static const int aux_ctas = getenv("OZ_AUX_SWAPS_CTAS") ? atoi(getenv("OZ_AUX_SWAPS_CTAS"))
                                                           : 32;
    static const int64_t aux_min_m = getenv("OZ_AUX_SWAPS_MIN_M")
                                         ? atoll(getenv("OZ_AUX_SWAPS_MIN_M"))
                                         : 8192;
    const bool aux = la && ready_cols >= n && aux_ctas > 0 && jb <= COMPOSE_MAX &&
                     rest >= aux_min_m && side->aux != nullptr;
    tr.mark(st);  // 0 step start
    // ---- the panel's interchanges: whole-row swaps (solve.py:80-82)
    if (!la) OZ_TRY(wait_cols());
    if (aux) {
      OZ_TRY(compose_list(j, ipiv + j, (int)jb, ws, st));
      OZ_CHECK_CUDA(cudaEventRecord(side->aux_ready, st));
      OZ_CHECK_CUDA(cudaStreamWaitEvent(side->aux, side->aux_ready, 0));
      OZ_TRY(apply_composed(a, lda, 0, j, j + jb + jb2, n, (int)jb, ws, side->aux, aux_ctas));
      OZ_CHECK_CUDA(cudaEventRecord(side->aux_done, side->aux));
      OZ_TRY(apply_composed(a, lda, j + jb, j + jb + jb2, 0, 0, (int)jb, ws, st));
    } else if (la)
      OZ_TRY(laswp_ipiv(a, lda, j + jb, j + jb + jb2, 0, 0, j, ipiv + j, (int)jb, ws, st));
    else
      OZ_TRY(laswp_ipiv(a, lda, 0, j, j + jb, n, j, ipiv + j, (int)jb, ws, st));
    tr.mark(st);  // 1 after laswp
    if (rest > 0) {
      // trsm U12 = L11^-1 A12 (solve.py:123-127), split, Schur update (:130-134)
      OZ_TRY(trsm_blocked(a, lda, j, jb, a12, lda, la ? jb2 : rest, st,
                          aux ? sm_count() - aux_ctas : 0));
      tr.mark(st);  // 2 after trsm
      OZ_TRY(schur_split_part(sc, true, 0, la ? jb2 : rest, ws, st));
      tr.mark(st);  // 3 after split
      OZ_TRY(schur_cols(sc, 0, jb2, ws, st, aux ? sm_count() - aux_ctas : 0));
      tr.mark(st);  // 4 after the update of the next panel's columns
      double* p2 = a + (j + jb) * lda + (j + jb);
      if (la) {
        // columns [jb2, rest) of this step: phase 1 [jb2, jb2 + cols1) beside
        // the panel on sms - S CTAs, phase 2 on every SM after it
        const LaPlan plan = lookahead_plan(la_setting, rest, jb, backend != 0 ? npairs : 0,
                                           sm_count(), rest - jb2);
        const int la_sms = plan.sms;
        const int64_t p1_end = jb2 + plan.cols1;
        if (tr.on) tr.split.push_back(la_sms);
        OZ_CHECK_CUDA(cudaEventRecord(side->ready, st));
        OZ_CHECK_CUDA(cudaStreamWaitEvent(side->st, side->ready, 0));
        OZ_TRY(panel_factor(p2, lda, rest, jb2, j + jb, ipiv + j + jb, info, ws.bits, ws,
                            side->st, la_sms));
        OZ_CHECK_CUDA(cudaEventRecord(side->done, side->st));
        tr.mark(side->st);  // 5 side stream: panel done
        if (ready_cols < n) {
          // step 0 while the upload is still running: interchanges, trsm,
          // split and update of each column chunk as soon as it is in place
          for (int64_t c0 = j + jb + jb2; c0 < n;) {
            OZ_TRY(wait_until(std::max<int64_t>(c0 + 1, ready_cols)));
            const int64_t c1 = ready_cols;
            OZ_TRY(laswp_ipiv(a, lda, c0, c1, 0, 0, j, ipiv + j, (int)jb, ws, st));
            OZ_TRY(trsm_blocked(a, lda, j, jb, a + c0 * lda + j, lda, c1 - c0, st));
            OZ_TRY(schur_split_part(sc, false, c0 - (j + jb), c1 - (j + jb), ws, st));
            OZ_TRY(schur_cols(sc, c0 - (j + jb), c1 - (j + jb), ws, st, sm_count() - la_sms));
            c0 = c1;
          }
          tr.mark_sub(st);
          tr.mark_sub(st);
          tr.mark_sub(st);
          tr.mark_sub(st);
        } else {
          if (aux)
            OZ_CHECK_CUDA(cudaStreamWaitEvent(st, side->aux_done, 0));
          else
            OZ_TRY(laswp_ipiv(a, lda, 0, j, j + jb + jb2, n, j, ipiv + j, (int)jb, ws, st));
          tr.mark_sub(st);
          OZ_TRY(trsm_blocked(a, lda, j, jb, a12 + jb2 * lda, lda, rest - jb2, st));
          tr.mark_sub(st);
          OZ_TRY(schur_split_part(sc, false, jb2, rest, ws, st));
          tr.mark_sub(st);
          OZ_TRY(schur_cols(sc, jb2, p1_end, ws, st, sm_count() - la_sms));
          tr.mark_sub(st);
          if (p1_end < rest) {
            OZ_CHECK_CUDA(cudaStreamWaitEvent(st, side->done, 0));
            OZ_TRY(schur_cols(sc, p1_end, rest, ws, st));
          }
        }
        tr.mark(st);  // 6 after the rest of the step
        OZ_CHECK_CUDA(cudaStreamWaitEvent(st, side->done, 0));
      } else {
        OZ_TRY(schur_cols(sc, jb2, rest, ws, st));
        tr.mark(st);  // 5 (no look-ahead): after the rest of the update
        OZ_TRY(panel_factor(p2, lda, rest, jb2, j + jb, ipiv + j + jb, info, ws.bits, ws, st));
        tr.mark(st);  // 6 (no look-ahead): after the next panel
      }
    }
    // finalized U rows of this panel: triu(lu[j:j+jb, j:]) (solve.py:135-137)
    OZ_TRY(max_abs(a + j * lda + j, jb, n - j, 1, lda, 1, 0, ws.bits, st));
  }
  if (tr.on) {
    cudaStreamSynchronize(st);
    // 7 marks per full step: start, laswp, trsm, split, gemm_a, side_done, gemm_b
    fprintf(stderr, "step    m  laswp  trsm  split gemm_a  panel(side) gemm_b  total [ms]  sms"
                    "  (rest: laswp trsm split gemm) p1-panel\n");
    for (size_t i = 0; i + 7 <= tr.ev.size(); i += 7) {
      float t[7];
      for (int q2 = 1; q2 < 7; ++q2) cudaEventElapsedTime(&t[q2], tr.ev[i], tr.ev[i + q2]);
      const float total = i + 7 < tr.ev.size() ? [&] { float x; cudaEventElapsedTime(&x, tr.ev[i], tr.ev[i + 7]); return x; }() : t[6];
      const size_t si = i / 7;
      float r3[4] = {0, 0, 0, 0};
      if (4 * si + 3 < tr.sub.size())
        for (int q3 = 0; q3 < 4; ++q3) cudaEventElapsedTime(&r3[q3], tr.ev[i + 4], tr.sub[4 * si + q3]);
      // p1-panel: end of phase 1 minus end of the panel (> 0: the panel's SMs
      // idled; < 0: the other SMs waited for the panel)
      fprintf(stderr, "%4zu %6lld %6.2f %5.2f %6.2f %6.2f %11.2f %6.2f %6.2f %4d  %5.2f %5.2f %5.2f %6.2f %7.2f\n",
              si, (long long)(n - (int64_t)si * nb - nb), t[1], t[2] - t[1], t[3] - t[2],
              t[4] - t[3], t[5] - t[4], t[6] - t[4], total,
              si < tr.split.size() ? tr.split[si] : 0, r3[0], r3[1] - r3[0], r3[2] - r3[1],
              t[6] - t[4] - r3[2], r3[3] - (t[5] - t[4]));
    }
    for (auto e : tr.ev) cudaEventDestroy(e);
    for (auto e : tr.sub) cudaEventDestroy(e);
  }
  if (unsigned long long* dbg = panel_dbg()) {
    // debug: per-phase cycles of the panel steps, summed over all CTAs
    cudaStreamSynchronize(st);
    unsigned long long h[8] = {0};
    cudaMemcpy(h, dbg, sizeof(h), cudaMemcpyDeviceToHost);
    fprintf(stderr, "panel phases (Mcycles summed over CTAs): publish %.1f deferred-update %.1f wait %.1f reduce %.1f urow %.1f update %.1f\n",
            h[0] / 1e6, h[4] / 1e6, h[1] / 1e6, h[2] / 1e6, h[3] / 1e6, h[5] / 1e6);
    cudaMemset(dbg, 0, sizeof(h));
  }
  finalize_stats_kernel<<<1, 1, 0, st>>>(ws.bits, stats);
  OZ_CHECK_LAUNCH();
  return OZ_OK;
}

int lu_solve(const double* lu, int64_t n, int64_t lda, const int64_t* perm, const double* b,
             double* x, int32_t* flag, int* sync, cudaStream_t st) {
  struct Stop {
    int tag;
    cudaStream_t st;
    double work;
    ~Stop() { prof_stop(tag, st, PROF_SOLVE, work); }
  } stop{prof_start(st), st, 2.0 * n * n};
  gather_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(b, perm, n, x);
  OZ_CHECK_LAUNCH();
  const int nblk = (int)ceil_div(n, TRSV_B);
  for (int upper = 0; upper < 2; ++upper) {
    OZ_CHECK_CUDA(cudaMemsetAsync(sync, 0, sizeof(int) * (nblk + 1), st));
    trsv_syncfree_kernel<<<nblk, TRSV_B * TRSV_G, 0, st>>>(lu, lda, n, upper, x, sync + 1, sync,
                                                           flag);
    OZ_CHECK_LAUNCH();
  }
  return OZ_OK;
}

int gemv_rows(const double* a, int64_t n, int64_t rs, int64_t cs, const double* x,
              const double* b, double* out, unsigned long long* rmax, unsigned long long* amax,
              double* part, cudaStream_t st, int64_t ncols = -1, double* abs_out = nullptr) {
  if (ncols < 0) ncols = n;
  const int nchunks = (int)ceil_div(ncols, GEMV_CHUNK);
  double* apart = (amax || abs_out) ? part + (size_t)nchunks * n : nullptr;
  dim3 grid((unsigned)ceil_div(n, 128), (unsigned)nchunks);
  gemv_partial_kernel<<<grid, 128, 0, st>>>(a, n, ncols, rs, cs, x, part, apart);
  OZ_CHECK_LAUNCH();
  gemv_finish_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(part, apart, nchunks, n, b, out,
                                                                 rmax, amax, abs_out);
  OZ_CHECK_LAUNCH();
  return OZ_OK;
}

}  // namespace oz

// ======================================================================= C ABI
extern "C" size_t oz_lu_workspace_bytes(int64_t n, int64_t nb, int num_slices, int slice_bits) {
  return oz::lu_ws_layout(n, nb, slice_bits > 7 ? 2 * num_slices : num_slices, nullptr, nullptr);
}

extern "C" int oz_lu_factor(double* a, int64_t n, int64_t lda, int64_t nb, int backend,
                            int num_slices, int slice_bits, int npairs, const int32_t* pair_a,
                            const int32_t* pair_b, const int32_t* pair_shift, int32_t* ipiv,
                            double* stats, int32_t* info, void* workspace, size_t ws_bytes,
                            void* stream) {
  return oz::lu_factor(a, n, lda, nb, backend, num_slices, slice_bits, npairs, pair_a, pair_b,
                       pair_shift, ipiv, stats, info, workspace, ws_bytes, oz::as_stream(stream));
}

extern "C" int oz_lu_factor_overlapped(double* a, int64_t n, int64_t lda, int64_t nb,
                                       int backend, int num_slices, int slice_bits, int npairs,
                                       const int32_t* pair_a, const int32_t* pair_b,
                                       const int32_t* pair_shift, int32_t* ipiv, double* stats,
                                       int32_t* info, void* workspace, size_t ws_bytes,
                                       void* const* chunk_events, int64_t chunk_cols,
                                       void* stream) {
  using namespace oz;
  OZ_REQUIRE(chunk_events != nullptr && chunk_cols >= 1, OZ_INVALID_PARAMS,
             "overlapped LU needs chunk events and a chunk width");
  return lu_factor(a, n, lda, nb, backend, num_slices, slice_bits, npairs, pair_a, pair_b,
                   pair_shift, ipiv, stats, info, workspace, ws_bytes, as_stream(stream),
                   reinterpret_cast<const cudaEvent_t*>(chunk_events), chunk_cols);
}

extern "C" int oz_memcpy2d_h2d(void* dst, size_t dpitch, const void* src, size_t spitch,
                               size_t width, size_t height, void* stream) {
  using namespace oz;
  OZ_CHECK_CUDA(cudaMemcpy2DAsync(dst, dpitch, src, spitch, width, height,
                                  cudaMemcpyHostToDevice, as_stream(stream)));
  return OZ_OK;
}

extern "C" size_t oz_lu_solve_workspace_bytes(int64_t n) {
  return sizeof(int) * (2 + oz::ceil_div(n, 64) + 16);
}

extern "C" int oz_lu_solve(const double* lu, int64_t n, int64_t lda, const int64_t* perm,
                           const double* b, double* x, void* workspace, size_t ws_bytes,
                           void* stream) {
  OZ_REQUIRE(ws_bytes >= oz_lu_solve_workspace_bytes(n), OZ_INVALID_PARAMS,
             "workspace too small");
  OZ_CHECK_CUDA(cudaMemsetAsync(workspace, 0, 4, oz::as_stream(stream)));
  int32_t* flag = reinterpret_cast<int32_t*>(workspace);
  return oz::lu_solve(lu, n, lda, perm, b, x, flag, reinterpret_cast<int*>(flag + 4),
                      oz::as_stream(stream));
}

extern "C" int oz_residual_norms(const double* a, int64_t n, int64_t row_stride,
                                 int64_t col_stride, const double* x, const double* b,
                                 double* out, void* stream) {
  using namespace oz;
  cudaStream_t st = as_stream(stream);
  const int nchunks = (int)ceil_div(n, GEMV_CHUNK);
  double* part = nullptr;
  unsigned long long* bits = nullptr;
  keep_pool_mapped();
  OZ_CHECK_CUDA(cudaMallocAsync(&part, sizeof(double) * 2 * nchunks * n, st));
  OZ_CHECK_CUDA(cudaMallocAsync(&bits, sizeof(unsigned long long) * 4, st));
  OZ_CHECK_CUDA(cudaMemsetAsync(bits, 0, sizeof(unsigned long long) * 4, st));
  int s = gemv_rows(a, n, row_stride, col_stride, x, b, nullptr, bits, bits + 1, part, st);
  if (s == OZ_OK) s = max_abs(x, n, 1, 1, 1, 0, 0, bits + 2, st);
  if (s == OZ_OK) s = max_abs(b, n, 1, 1, 1, 0, 0, bits + 3, st);
  if (s == OZ_OK) {
    OZ_CHECK_CUDA(cudaMemcpyAsync(out, bits, sizeof(double) * 4, cudaMemcpyDeviceToDevice, st));
  }
  cudaFreeAsync(part, st);
  cudaFreeAsync(bits, st);
  return s;
}

extern "C" int oz_row_sums(const double* a, int64_t n, int64_t row_stride, int64_t col_stride,
                           double* out, void* stream) {
  using namespace oz;
  cudaStream_t st = as_stream(stream);
  const int nchunks = (int)ceil_div(n, GEMV_CHUNK);
  double* part = nullptr;
  keep_pool_mapped();
  OZ_CHECK_CUDA(cudaMallocAsync(&part, sizeof(double) * nchunks * n, st));
  int s = gemv_rows(a, n, row_stride, col_stride, nullptr, nullptr, out, nullptr, nullptr, part,
                    st);
  cudaFreeAsync(part, st);
  return s;
}

extern "C" int oz_max_abs(const double* a, int64_t m, int64_t n, int64_t row_stride,
                          int64_t col_stride, double* out, void* stream) {
  using namespace oz;
  cudaStream_t st = as_stream(stream);
  OZ_CHECK_CUDA(cudaMemsetAsync(out, 0, sizeof(double), st));
  return max_abs(a, m, n, row_stride, col_stride, 0, 0,
                 reinterpret_cast<unsigned long long*>(out), st);
}

extern "C" int oz_copy2d(const double* src, int64_t rows, int64_t cols, int64_t src_rs,
                         int64_t src_cs, double* dst, int64_t dst_rs, int64_t dst_cs,
                         void* stream) {
  using namespace oz;
  if (rows <= 0 || cols <= 0) return OZ_OK;
  const int64_t count = rows * cols;
  const bool same_dense = (src_rs == 1 && dst_rs == 1 && src_cs == rows && dst_cs == rows) ||
                          (src_cs == 1 && dst_cs == 1 && src_rs == cols && dst_rs == cols);
  if (same_dense && count % 2 == 0 && ((reinterpret_cast<uintptr_t>(src) |
                                        reinterpret_cast<uintptr_t>(dst)) & 15) == 0) {
    // one dense block in the same layout (the LU's working copy): a flat
    // 128-bit copy, four loads in flight, instead of the transposing tiles
    int64_t blocks = ceil_div(count / 2, 256);
    if (blocks > sm_count() * 8) blocks = sm_count() * 8;
    copy_flat_kernel<<<(unsigned)blocks, 256, 0, as_stream(stream)>>>(
        reinterpret_cast<const double2*>(src), reinterpret_cast<double2*>(dst), count / 2);
    OZ_CHECK_LAUNCH();
    return OZ_OK;
  }
  dim3 grid((unsigned)ceil_div(cols, 32), (unsigned)ceil_div(rows, 32));
  copy2d_kernel<<<grid, dim3(32, 8), 0, as_stream(stream)>>>(src, rows, cols, src_rs, src_cs, dst,
                                                            dst_rs, dst_cs);
  OZ_CHECK_LAUNCH();
  return OZ_OK;
}

// ============================================================ step-level C ABI
// The blocked LU as separate steps, for drivers that own the loop (the
// distributed 1 x Q block-cyclic HPL in hpl.py).  Every call takes the LU
// workspace plus the (n, nb, num_slices) it was sized with.
namespace {
int ws_view(void* ws, size_t ws_bytes, int64_t n, int64_t nb, int k, oz::LuWs* out) {
  const size_t need = oz::lu_ws_layout(n, nb, k, (uint8_t*)ws, out);
  OZ_REQUIRE(ws != nullptr && ws_bytes >= need, OZ_INVALID_PARAMS,
             "workspace too small (%zu < %zu)", ws_bytes, need);
  return OZ_OK;
}
}  // namespace

extern "C" int oz_lu_ws_init(void* ws, size_t ws_bytes, int64_t n, int64_t nb, int num_slices,
                             void* stream) {
  using namespace oz;
  LuWs w;
  OZ_TRY(ws_view(ws, ws_bytes, n, nb, num_slices, &w));
  cudaStream_t st = as_stream(stream);
  OZ_CHECK_CUDA(cudaMemsetAsync(w.bar, 0, sizeof(GridBar), st));
  OZ_CHECK_CUDA(cudaMemsetAsync(w.cand, 0, sizeof(double) * 2 * 1024 * CAND_STRIDE, st));
  OZ_CHECK_CUDA(cudaMemsetAsync(w.bits, 0, 4 * sizeof(unsigned long long), st));
  return OZ_OK;
}

// The look-ahead SM split for a panel of m rows beside a trailing update of
// ncols columns (the single-GPU driver's model; 0 = no look-ahead).
extern "C" int64_t oz_lookahead_cols1(int64_t m, int64_t rest_cols, int64_t nb, int npairs,
                                      int panel_sms) {
  if (oz::lookahead_sms() == 0 || !oz::la_two_phase() || panel_sms <= 0) return rest_cols;
  return oz::phase1_cols(panel_sms, m, nb, npairs, oz::sm_count(), rest_cols);
}

extern "C" int oz_lookahead_sms(int64_t m, int64_t ncols, int64_t nb, int npairs) {
  const int setting = oz::lookahead_sms();
  if (setting == 0) return 0;
  // ncols = this rank's trailing columns, the next panel's included; on one
  // rank this is the single-GPU driver's panel_sms (bit-identical factors)
  (void)ncols;
  return oz::panel_sms(setting, m, nb, npairs, oz::sm_count());
}

extern "C" int oz_lu_panel(double* a, int64_t lda, int64_t m, int64_t jb, int64_t base,
                           int32_t* ipiv, int32_t* info, unsigned long long* growth_bits,
                           void* ws, size_t ws_bytes, int64_t ws_n, int64_t ws_nb,
                           int ws_slices, int max_ctas, void* stream) {
  using namespace oz;
  OZ_REQUIRE(m >= jb && jb >= 1 && jb <= COMPOSE_MAX && lda >= m, OZ_INVALID_PARAMS,
             "bad panel shape m=%lld jb=%lld lda=%lld", (long long)m, (long long)jb,
             (long long)lda);
  LuWs w;
  OZ_TRY(ws_view(ws, ws_bytes, ws_n, ws_nb, ws_slices, &w));
  return panel_factor(a, lda, m, jb, base, ipiv, info, growth_bits, w, as_stream(stream),
                      max_ctas > 0 ? max_ctas : 0);
}

extern "C" int oz_laswp(double* a, int64_t lda, int64_t c0a, int64_t c1a, int64_t c0b,
                        int64_t c1b, int64_t k1, const int32_t* ipiv, int npiv, void* ws,
                        size_t ws_bytes, int64_t ws_n, int64_t ws_nb, int ws_slices,
                        void* stream) {
  using namespace oz;
  OZ_REQUIRE(c0a <= c1a && c0b <= c1b, OZ_INVALID_PARAMS, "bad column ranges");
  LuWs w;
  OZ_TRY(ws_view(ws, ws_bytes, ws_n, ws_nb, ws_slices, &w));
  return laswp_ipiv(a, lda, c0a, c1a, c0b, c1b, k1, ipiv, npiv, w, as_stream(stream));
}

extern "C" int oz_trsm_lunit(const double* l11, int64_t ldl, int64_t jb, double* b, int64_t ldb,
                             int64_t ncols, void* stream) {
  using namespace oz;
  OZ_REQUIRE(jb >= 1 && ldl >= jb && ldb >= jb, OZ_INVALID_PARAMS, "bad trsm shape");
  return trsm_blocked(const_cast<double*>(l11), ldl, 0, jb, b, ldb, ncols, as_stream(stream));
}

extern "C" int oz_schur_update(int backend, int64_t m, int64_t ncols, int64_t jb,
                               const double* a21, int64_t lda21, const double* u12, int64_t ldu,
                               double* a22, int64_t lda22, int num_slices, int slice_bits,
                               int npairs, const int32_t* pair_a, const int32_t* pair_b,
                               const int32_t* pair_shift, unsigned long long* growth_bits,
                               void* ws, size_t ws_bytes, int64_t ws_n, int64_t ws_nb,
                               void* stream) {
  using namespace oz;
  OZ_REQUIRE(backend >= 0 && backend <= 2, OZ_INVALID_PARAMS, "bad backend %d", backend);
  OZ_REQUIRE(backend == 0 || (m <= ws_n && ncols <= ws_n && jb <= ws_nb), OZ_INVALID_PARAMS,
             "schur update larger than the workspace");
  LuWs w;
  OZ_TRY(ws_view(ws, ws_bytes, ws_n, ws_nb,
                 backend != 0 ? (slice_bits > 7 ? 2 * num_slices : num_slices) : 0, &w));
  return schur_update(backend, m, ncols, jb, a21, lda21, u12, ldu, a22, lda22, num_slices,
                      slice_bits, npairs, pair_a, pair_b, pair_shift, growth_bits, w,
                      as_stream(stream));
}

// max |a| (optionally only the upper trapezoid c >= r) folded into *bits
namespace oz {
namespace {
__global__ void nonfinite_kernel(const double* __restrict__ a, int64_t m, int64_t n, int64_t rs,
                                 int64_t cs, int32_t* flag) {
  bool bad = false;
  const int64_t total = m * n;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = i / m, r = i - c * m;  // consecutive threads: consecutive rows
    bad |= !isfinite(a[r * rs + c * cs]);
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicExch(flag, 1);
}
}  // namespace
}  // namespace oz

// *flag <- 1 if any entry of the m x n matrix is NaN or infinite (the
// reference's NonFiniteEntryError check, split.py:104-105 / solve.py:107-108).
extern "C" int oz_nonfinite_flag(const double* a, int64_t m, int64_t n, int64_t row_stride,
                                 int64_t col_stride, int32_t* flag, void* stream) {
  using namespace oz;
  if (m <= 0 || n <= 0) return OZ_OK;
  int64_t blocks = ceil_div(m * n, 256 * 8);
  if (blocks > sm_count() * 8) blocks = sm_count() * 8;
  nonfinite_kernel<<<(unsigned)blocks, 256, 0, as_stream(stream)>>>(a, m, n, row_stride,
                                                                   col_stride, flag);
  OZ_CHECK_LAUNCH();
  return OZ_OK;
}

extern "C" int oz_max_abs_bits(const double* a, int64_t m, int64_t n, int64_t row_stride,
                               int64_t col_stride, int upper, unsigned long long* bits,
                               void* stream) {
  return oz::max_abs(a, m, n, row_stride, col_stride, upper, 0, bits, oz::as_stream(stream));
}

// One diagonal block of a triangular solve, in place on x[0..nb):
// unit-lower (upper=0) or upper with division (upper=1); flag <- 1 on a zero
// diagonal.  workspace: oz_lu_solve_workspace_bytes(nb) bytes.
extern "C" int oz_trsv_block(const double* a, int64_t lda, int64_t nb, int upper, double* x,
                             int32_t* flag, void* workspace, size_t ws_bytes, void* stream) {
  using namespace oz;
  OZ_REQUIRE(ws_bytes >= oz_lu_solve_workspace_bytes(nb), OZ_INVALID_PARAMS,
             "workspace too small");
  cudaStream_t st = as_stream(stream);
  int* sync = reinterpret_cast<int*>(workspace);
  const int nblk = (int)ceil_div(nb, TRSV_B);
  OZ_CHECK_CUDA(cudaMemsetAsync(sync, 0, sizeof(int) * (nblk + 1), st));
  trsv_syncfree_kernel<<<nblk, TRSV_B * TRSV_G, 0, st>>>(a, lda, nb, upper, x, sync + 1, sync,
                                                         flag);
  OZ_CHECK_LAUNCH();
  return OZ_OK;
}

// Partial row sums over a block of columns: ax[i] = sum_j a_ij x_j (x = null:
// x_j = 1), asum[i] = sum_j |a_ij| (null: skipped).  Fixed summation order.
extern "C" int oz_gemv_partial(const double* a, int64_t rows, int64_t cols, int64_t row_stride,
                               int64_t col_stride, const double* x, double* ax, double* asum,
                               void* stream) {
  using namespace oz;
  if (rows <= 0) return OZ_OK;
  cudaStream_t st = as_stream(stream);
  if (cols <= 0) {
    OZ_CHECK_CUDA(cudaMemsetAsync(ax, 0, sizeof(double) * rows, st));
    if (asum) OZ_CHECK_CUDA(cudaMemsetAsync(asum, 0, sizeof(double) * rows, st));
    return OZ_OK;
  }
  const int nchunks = (int)ceil_div(cols, GEMV_CHUNK);
  double* part = nullptr;
  keep_pool_mapped();
  OZ_CHECK_CUDA(cudaMallocAsync(&part, sizeof(double) * 2 * nchunks * rows, st));
  int s = gemv_rows(a, rows, row_stride, col_stride, x, nullptr, ax, nullptr, nullptr, part, st,
                    cols, asum);
  cudaFreeAsync(part, st);
  return s;
}

// The Schur update in two calls (look-ahead drivers): split A21/U12 once,
// then update column ranges [c0, c1) of A22, optionally on at most max_ctas
// CTAs (0 = all SMs) so a concurrent panel or collective keeps some SMs.
extern "C" int oz_schur_split(int backend, int64_t m, int64_t ncols, int64_t jb,
                              const double* a21, int64_t lda21, const double* u12, int64_t ldu,
                              int num_slices, int slice_bits, void* ws, size_t ws_bytes,
                              int64_t ws_n, int64_t ws_nb, void* stream) {
  using namespace oz;
  OZ_REQUIRE(backend >= 0 && backend <= 2, OZ_INVALID_PARAMS, "bad backend %d", backend);
  if (backend == 0) return OZ_OK;
  OZ_REQUIRE(m <= ws_n && ncols <= ws_n && jb <= ws_nb, OZ_INVALID_PARAMS,
             "schur update larger than the workspace");
  LuWs w;
  OZ_TRY(ws_view(ws, ws_bytes, ws_n, ws_nb, slice_bits > 7 ? 2 * num_slices : num_slices, &w));
  const Schur s{backend, m, ncols, jb, a21, lda21, u12, ldu, nullptr, 0, num_slices, slice_bits,
                0, nullptr, nullptr, nullptr, nullptr};
  return schur_split(s, w, as_stream(stream));
}

extern "C" int oz_schur_cols(int backend, int64_t m, int64_t ncols, int64_t jb,
                             const double* a21, int64_t lda21, const double* u12, int64_t ldu,
                             double* a22, int64_t lda22, int num_slices, int slice_bits,
                             int npairs, const int32_t* pair_a, const int32_t* pair_b,
                             const int32_t* pair_shift, unsigned long long* growth_bits,
                             int64_t c0, int64_t c1, int max_ctas, void* ws, size_t ws_bytes,
                             int64_t ws_n, int64_t ws_nb, void* stream) {
  using namespace oz;
  OZ_REQUIRE(backend >= 0 && backend <= 2, OZ_INVALID_PARAMS, "bad backend %d", backend);
  OZ_REQUIRE(0 <= c0 && c0 <= c1 && c1 <= ncols, OZ_INVALID_PARAMS, "bad column range");
  OZ_REQUIRE(backend == 0 || (m <= ws_n && ncols <= ws_n && jb <= ws_nb), OZ_INVALID_PARAMS,
             "schur update larger than the workspace");
  LuWs w;
  OZ_TRY(ws_view(ws, ws_bytes, ws_n, ws_nb,
                 backend != 0 ? (slice_bits > 7 ? 2 * num_slices : num_slices) : 0, &w));
  const Schur s{backend, m, ncols, jb, a21, lda21, u12, ldu, a22, lda22, num_slices, slice_bits,
                npairs, pair_a, pair_b, pair_shift, growth_bits};
  return schur_cols(s, c0, c1, w, as_stream(stream), max_ctas);
}

// Tuning only (OZ_PANEL_TIMING=1): copy and clear the 8 panel debug counters.
extern "C" int oz_panel_debug_counters(unsigned long long* out8) {
  unsigned long long* d = oz::panel_dbg();
  if (d == nullptr) {
    for (int i = 0; i < 8; ++i) out8[i] = 0;
    return OZ_OK;
  }
  OZ_CHECK_CUDA(cudaDeviceSynchronize());
  OZ_CHECK_CUDA(cudaMemcpy(out8, d, 8 * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
  OZ_CHECK_CUDA(cudaMemset(d, 0, 8 * sizeof(unsigned long long)));
  return OZ_OK;
}
