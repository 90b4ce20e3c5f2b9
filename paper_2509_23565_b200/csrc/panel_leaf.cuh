// panel_leaf.cuh — register-resident panel leaf for short panels (included by
// lu.cu inside its anonymous namespace; uses PanelArgs, better(), warp_argmax()).
//
// Same arithmetic as panel_window_kernel and as solve.py:75-90 (np.argmax
// pivot order, division by the pivot, rank-1 update as a product followed by a
// subtraction), so the two leaves are bit-identical.  What changes is where
// the window lives and how the CTAs exchange their pivot candidates:
//
//  * rows in registers: thread i of CTA g owns window rows g*R + i + 256*k
//    (k < RPT, R = 256*RPT), all W columns of them in registers, in a
//    shifted layout — x[k][c] holds column t + c at step t — so the column
//    loop runs with static register indices.  The rank-1 update is
//    FP64-pipe-bound (W*R*2 ops per step) instead of shared-memory-bound;
//  * push exchange: the CTA's best candidate row is copied by ONE bulk copy
//    per destination (cp.async.bulk shared::cta -> shared::cluster, mbarrier
//    complete_tx) into every CTA of the cluster; each CTA waits on its own
//    mbarrier and reduces the G records locally.  No cluster barrier and no
//    remote loads per column (scripts/exchange_microbench.cu: 0.54-0.89 us
//    per exchange vs 0.83-1.02 us for barrier + DSMEM reads);
//  * the update of columns t+2.. for step t runs after the push of step t+1
//    (inside the exchange latency); only column t+1, which the next argmax
//    needs, is updated right after the exchange.
// Records are triple-buffered: a CTA pushes step t+3 into buffer t%3 only after
// it received every CTA's step t+2 record, which each CTA sends after it
// finished reading buffer t%3 (its deferred update of step t+1).
// L values are kept in shared memory (column-major [W][R]) and every row is
// written once, at its final position, at the end; moved rows are listed for
// the gather that applies the same interchanges to the other columns.

constexpr int LEAF_MAXG = 16;

template <int W, int NT, bool kGrid>
struct alignas(128) LeafShared {  // bulk-copy sources/destinations need 16-byte alignment
  // received records: [0] |v|, [1] pos, [2] row, [4..) values.  Cluster
  // variant: every CTA's; grid variant: the winner's, copied from global
  double rec[3][kGrid ? 1 : LEAF_MAXG][4 + W];
  double mine[3][4 + W];            // this CTA's record (source of the bulk copies)
  double raw[W];                    // the owner row's registers, before step t-1's update
  unsigned long long bar[3];
  // per-warp candidate |v|, position, row; two buffers by step parity: a warp
  // may write step t+1's candidate while another still reads step t's (the
  // cluster variant has no CTA barrier between those points)
  double wa[2][NT / 32];
  int wp[2][NT / 32];
  int wr[2][NT / 32];
  int occ[W];  // physical window row at logical position c (< W)
};

template <int W, int RPT, int NT>
constexpr size_t leaf_smem_bytes() {
  return (size_t)W * NT * RPT * sizeof(double);
}

// |v| as ordered integer bits (non-negative doubles order like their bits):
// the growth maximum runs on the integer pipe, beside the FP64 update
__device__ __forceinline__ unsigned long long abs_bits(double v) {
  return (unsigned long long)__double_as_longlong(v) & 0x7fffffffffffffffull;
}

__device__ __forceinline__ void leaf_mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void leaf_mbar_expect(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void leaf_mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tLEAF_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra LEAF_WAIT_%=;\n\t}" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ uint32_t leaf_mapa(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void leaf_push(uint32_t dst, uint32_t src, uint32_t bytes,
                                          uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, "
      "[%3];" ::"r"(dst),
      "r"(src), "r"(bytes), "r"(bar)
      : "memory");
}

// Grid variant records as tagged 8-byte words (LL protocol): each word holds
// 32 payload bits and the step's 32-bit tag, so a reader that sees the tag
// in a word has that word's payload — no fence on the writer, no ordering
// between words.  A record is 2 + W pairs of words (16-byte stores).
constexpr int LEAF_LL_STRIDE = 2 * (2 + 64);  // words per CTA slot (W <= 64)
__device__ __forceinline__ void leaf_ll_store(unsigned long long* p, unsigned lo, unsigned hi,
                                              unsigned tag) {
  const unsigned long long t = (unsigned long long)tag << 32;
  asm volatile("st.relaxed.gpu.global.v2.b64 [%0], {%1, %2};" ::"l"(p), "l"(t | lo), "l"(t | hi)
               : "memory");
}
__device__ __forceinline__ ulonglong2 leaf_ll_raw(const unsigned long long* p) {
  ulonglong2 v;
  asm volatile("ld.relaxed.gpu.global.v2.b64 {%0, %1}, [%2];" : "=l"(v.x), "=l"(v.y) : "l"(p)
               : "memory");
  return v;
}
__device__ __forceinline__ bool leaf_ll_ok(ulonglong2 v, unsigned tag) {
  return (unsigned)(v.x >> 32) == tag && (unsigned)(v.y >> 32) == tag;
}
__device__ __forceinline__ double leaf_ll_double(ulonglong2 v) {
  return __longlong_as_double((long long)((v.y << 32) | (v.x & 0xffffffffull)));
}
__device__ __forceinline__ void leaf_ll_load2(const unsigned long long* p, unsigned tag,
                                              unsigned& w0, unsigned& w1, unsigned& w2,
                                              unsigned& w3) {
  unsigned long long x, y, z, u;
  do {
    asm volatile("ld.relaxed.gpu.global.v2.b64 {%0, %1}, [%2];" : "=l"(x), "=l"(y) : "l"(p)
                 : "memory");
    asm volatile("ld.relaxed.gpu.global.v2.b64 {%0, %1}, [%2];" : "=l"(z), "=l"(u) : "l"(p + 2)
                 : "memory");
  } while ((unsigned)(x >> 32) != tag || (unsigned)(y >> 32) != tag ||
           (unsigned)(z >> 32) != tag || (unsigned)(u >> 32) != tag);
  w0 = (unsigned)x;
  w1 = (unsigned)y;
  w2 = (unsigned)z;
  w3 = (unsigned)u;
}

// OZ_PANEL_TIMING (tuning): thread 0 of CTA 0 adds per-phase clock64 deltas to
// p.dbg[0..5]; the owner thread of CTA 0 adds its record+push time to p.dbg[6]
#define LEAF_MARK(i)                                                   \
  if (trace) {                                                         \
    const long long _n = clock64();                                    \
    _acc[i] += (unsigned long long)(_n - _tp);                         \
    _tp = _n;                                                          \
  }

// kGrid = false: the G <= 16 CTAs form one cluster and push records through
// DSMEM (above).  kGrid = true: G co-resident CTAs (cooperative launch, G up
// to the SM count) publish records to global memory (triple-buffered slots of
// p.cand), each with a tag word written last by a release store; warp 0 of
// every CTA polls the G tags with acquire loads, reduces, and copies the
// winner's record to shared memory.  Same arithmetic, same bits.
template <int W, int RPT, int NT, bool kGrid>
__global__ void __launch_bounds__(NT, 1) panel_leaf_kernel(PanelArgs p) {
  constexpr int R = NT * RPT;
  static_assert(4 + W <= CAND_STRIDE, "grid record must fit a candidate slot");
  static_assert(2 * (2 + W) <= LEAF_LL_STRIDE, "grid record must fit a tagged slot");
  extern __shared__ double lbuf[];  // [W][R]: L (and, for pivot rows, U) values by window row
  __shared__ LeafShared<W, NT, kGrid> sh;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int G = (int)gridDim.x;  // CTAs of the window (one cluster unless kGrid)
  const int g = (int)blockIdx.x;
  const int w = p.w;
  const int64_t m = p.m;
  double* abase = p.a + p.r0 * p.lda + p.r0;  // window corner

  double x[RPT][W];
  int pos[RPT];  // logical position (>= 0), -(t+1) once the pivot of step t, INT_MIN if no row
  unsigned long long gmax = 0;  // bits of the largest |value| seen
#pragma unroll
  for (int k = 0; k < RPT; ++k) {
    const int64_t gr = (int64_t)g * R + tid + k * NT;
    const bool ok = gr < m;
    pos[k] = ok ? (int)gr : INT_MIN;
#pragma unroll
    for (int c = 0; c < W; ++c) {
      x[k][c] = ok && c < w ? abase[(int64_t)c * p.lda + gr] : 0.0;
      gmax = max(gmax, abs_bits(x[k][c]));
    }
  }
  if (tid < W) sh.occ[tid] = tid;
  if (!kGrid && tid == 0) {
    for (int b = 0; b < 3; ++b) leaf_mbar_init(smem_u32(&sh.bar[b]), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if constexpr (!kGrid) {
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
  }

  // candidate for column 0
  double ca = -1.0;
  int cp = 0x7fffffff, cr = -1;
#pragma unroll
  for (int k = 0; k < RPT; ++k) {
    const double v = fabs(x[k][0]);
    if (pos[k] >= 0 && better(v, pos[k], ca, cp)) {
      ca = v;
      cp = pos[k];
      cr = tid + k * NT;
    }
  }
  double lprev[RPT];
#pragma unroll
  for (int k = 0; k < RPT; ++k) lprev[k] = 0.0;
  const double* uprev = nullptr;  // previous step's winner row (shifted: [c] = column t-1+c)

  const bool trace = p.dbg != nullptr && g == 0 && tid == 0;
  long long _tp = clock64();
  unsigned long long _acc[6] = {0, 0, 0, 0, 0, 0}, _own = 0;
  for (int t = 0; t < w; ++t) {
    const int b = t % 3;
    const int nv = w - t;  // valid values in this step's records (columns t..w-1)
    // full records every step: columns >= w are zero in every row and stay
    // zero (0 - l*0), so the update below needs no per-column predicates
    constexpr uint32_t bytes = (uint32_t)((4 + W) * 8);
    const unsigned tag = p.epoch + (unsigned)t + 1u;  // kGrid record tag of this step
    if (!kGrid && tid == 0) leaf_mbar_expect(smem_u32(&sh.bar[b]), (uint32_t)G * bytes);
    // ---- CTA argmax of the thread candidates (np.argmax order)
    warp_argmax(ca, cp, cr);
    const int wb = t & 1;
    if (lane == 0) {
      sh.wa[wb][wid] = ca;
      sh.wp[wb][wid] = cp;
      sh.wr[wb][wid] = cr;
    }
    __syncthreads();
    LEAF_MARK(0)
    double ba = lane < NT / 32 ? sh.wa[wb][lane] : -2.0;
    int bp = lane < NT / 32 ? sh.wp[wb][lane] : 0x7fffffff;
    int br = lane < NT / 32 ? sh.wr[wb][lane] : -1;
    warp_argmax(ba, bp, br);  // every warp computes the same winner
    const bool none = br < 0;
    const int owner = none ? 0 : (br % NT);
    LEAF_MARK(1)
    if ((tid >> 5) == (owner >> 5)) {
      // ---- publish (the owner's warp): the winner row's values with step
      //      t-1's pending update applied, i.e. the same product-then-subtract
      //      the deferred update will store.  The owner dumps its registers
      //      (before that update, column t+c sits in x[c+1]); every lane then
      //      forms two columns.
      const long long _o = clock64();
      const int ol = owner & 31;
      const int kk = none ? 0 : br / NT;
      double* rec = sh.mine[b];
      double lo = 0.0;
      if (lane == ol) {
#pragma unroll
        for (int k = 0; k < RPT; ++k) {
          if (k != kk) continue;
          lo = lprev[k];
#pragma unroll
          for (int c = 0; c < W; c += 2)
            *reinterpret_cast<double2*>(&sh.raw[c]) = make_double2(x[k][c], x[k][c + 1]);
        }
        long long* irec = reinterpret_cast<long long*>(rec);
        rec[0] = none ? -1.0 : ba;
        irec[1] = none ? 0x7fffffff : bp;
        irec[2] = none ? -1 : (long long)g * R + br;
      }
      lo = __shfl_sync(0xffffffffu, lo, ol);
      __syncwarp();
#pragma unroll
      for (int i = 0; i < (W + 31) / 32; ++i) {
        const int c = lane + 32 * i;
        if (c < W) {
          double v;
          if (t == 0)
            v = sh.raw[c];  // no pending update yet: x[c] is column c
          else if (c == 0)
            v = sh.raw[0];  // column t was updated right after the exchange
          else
            v = c + 1 < W ? __dsub_rn(sh.raw[c + 1], __dmul_rn(lo, uprev[c + 1])) : 0.0;
          rec[4 + c] = v;
        }
      }
      if constexpr (kGrid) {
        // the record to this CTA's global slot as tagged words (no fence):
        // pair 0 = |v|, pair 1 = (pos, row), pair 2 + c = value c
        __syncwarp();
        unsigned long long* gs =
            reinterpret_cast<unsigned long long*>(p.cand) + ((size_t)b * G + g) * LEAF_LL_STRIDE;
        const long long* irec = reinterpret_cast<const long long*>(rec);
        for (int c = lane; c < 2 + W; c += 32) {
          unsigned lo, hi;
          if (c == 1) {
            lo = (unsigned)irec[1];
            hi = (unsigned)irec[2];
          } else {
            const unsigned long long v = (unsigned long long)irec[c == 0 ? 0 : c + 2];
            lo = (unsigned)v;
            hi = (unsigned)(v >> 32);
          }
          leaf_ll_store(gs + 2 * c, lo, hi, tag);
        }
      } else {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        // one bulk copy per destination CTA, issued by lane d (a single thread
        // issuing G copies serialises them, ~150 cycles each)
        if (lane < G) {
          const uint32_t dst = leaf_mapa(smem_u32(&sh.rec[b][g][0]), (uint32_t)lane);
          const uint32_t mb = leaf_mapa(smem_u32(&sh.bar[b]), (uint32_t)lane);
          leaf_push(dst, smem_u32(rec), bytes, mb);
        }
      }
      if (p.dbg != nullptr && g == 0 && lane == ol) _own += (unsigned long long)(clock64() - _o);
    }
    LEAF_MARK(2)
    // ---- deferred update of step t-1 on columns t+1..: x[c] <- x[c+1] - l*u[c+1]
    if (t > 0) {
      unsigned long long gm[4] = {0, 0, 0, 0};  // independent max chains
#pragma unroll
      for (int k = 0; k < RPT; ++k) {
        if (pos[k] < 0) continue;
        const double l = lprev[k];
#pragma unroll
        for (int c = 1; c < W - 1; ++c) {
          const double v = __dsub_rn(x[k][c + 1], __dmul_rn(l, uprev[c + 1]));
          x[k][c] = v;
          gm[c & 3] = max(gm[c & 3], abs_bits(v));
        }
        x[k][W - 1] = 0.0;
      }
      gmax = max(gmax, max(max(gm[0], gm[1]), max(gm[2], gm[3])));
    }
    LEAF_MARK(3)
    // ---- every CTA's record of step t has arrived
    double ra;
    int rp, rg;
    if constexpr (kGrid) {
      if (wid == 0) {
        // lane l polls the headers of CTAs l, l+32, ... until both pairs
        // carry this step's tag, the warp reduces, then copies the winner's
        // row (polling each pair's tags) into shared memory
        const unsigned long long* slots =
            reinterpret_cast<const unsigned long long*>(p.cand) + (size_t)b * G * LEAF_LL_STRIDE;
        double a1 = -2.0;
        int p1 = 0x7fffffff, g1 = -1;
        long long* irw = reinterpret_cast<long long*>(sh.rec[b][0]);
        for (int gg = lane; gg < G; gg += 32) {
          const unsigned long long* r = slots + (size_t)gg * LEAF_LL_STRIDE;
          unsigned a_lo, a_hi, pv, rv;
          leaf_ll_load2(r, tag, a_lo, a_hi, pv, rv);
          const double av = __longlong_as_double((long long)(((unsigned long long)a_hi << 32) | a_lo));
          if (better(av, (int)pv, a1, p1)) {
            a1 = av;
            p1 = (int)pv;
            g1 = gg;
          }
        }
        warp_argmax(a1, p1, g1);
        const unsigned long long* win = slots + (size_t)g1 * LEAF_LL_STRIDE;
        // the winner's row and position: every load issued at once, then each
        // pair re-polled only if its tags are not this step's yet (serial
        // 16-byte polls cost a round trip per 32 values: 12288 x 1024 panel,
        // 64-column windows on 100 SMs, leaves 3.48 -> 3.19 ms)
        constexpr int NP = (W + 1 + 31) / 32;
        ulonglong2 rv[NP];
#pragma unroll
        for (int i = 0; i < NP; ++i) {
          const int c = lane + 32 * i;
          if (c < 1 + W) rv[i] = leaf_ll_raw(win + 2 * (c == 0 ? 1 : c + 1));
        }
#pragma unroll
        for (int i = 0; i < NP; ++i) {
          const int c = lane + 32 * i;
          if (c < 1 + W) {
            while (!leaf_ll_ok(rv[i], tag)) rv[i] = leaf_ll_raw(win + 2 * (c == 0 ? 1 : c + 1));
            if (c == 0)
              irw[2] = (long long)(int)(unsigned)rv[i].y;
            else
              irw[3 + c] = (long long)((rv[i].y << 32) | (rv[i].x & 0xffffffffull));
          }
        }
        if (lane == 0) {
          sh.rec[b][0][0] = a1;
          irw[1] = p1;
        }
      }
      __syncthreads();
      ra = sh.rec[b][0][0];
      rp = (int)reinterpret_cast<const long long*>(sh.rec[b][0])[1];
      rg = 0;
    } else {
      leaf_mbar_wait(smem_u32(&sh.bar[b]), (uint32_t)((t / 3) & 1));
      const double(*recs)[4 + W] = sh.rec[b];
      ra = lane < G ? recs[lane][0] : -2.0;
      rp = lane < G ? (int)reinterpret_cast<const long long*>(recs[lane])[1] : 0x7fffffff;
      rg = lane < G ? lane : -1;
      warp_argmax(ra, rp, rg);
    }
    LEAF_MARK(4)
    (void)ra;
    const double* urow = sh.rec[b][rg] + 4;  // winner row: urow[c] = column t + c
    const int prow = (int)reinterpret_cast<const long long*>(sh.rec[b][rg])[2];
    const double piv = urow[0];
    const int rt = sh.occ[t];  // physical row at logical position t
    if (g == 0 && tid == 0) {
      p.ipiv[p.r0 + t] = (int32_t)(p.base + p.r0 + rp);
      if (piv == 0.0) atomicCAS(reinterpret_cast<int*>(p.info), 0, (int)(p.base + p.r0 + t + 1));
    }
    if (tid == 0 && rt != prow && rp < W) sh.occ[rp] = rt;
    // ---- interchange bookkeeping (solve.py:80-82), scaling (:84), update of
    //      column t+1 (:86) and the next candidate
    ca = -1.0;
    cp = 0x7fffffff;
    cr = -1;
#pragma unroll
    for (int k = 0; k < RPT; ++k) {
      const int lr = tid + k * NT;
      const int phys = g * R + lr;
      if (pos[k] == INT_MIN) continue;
      if (phys == prow) {
        // the pivot row is final: its current values are U row t
#pragma unroll
        for (int c = 0; c < W; ++c)
          if (t + c < W) lbuf[(t + c) * R + lr] = x[k][c];
        pos[k] = -(t + 1);
        continue;
      }
      if (pos[k] < 0) continue;
      if (phys == rt) pos[k] = rp;
      const double l = x[k][0] / piv;
      lbuf[t * R + lr] = l;
      lprev[k] = l;
      if (nv > 1) {
        const double v = __dsub_rn(x[k][1], __dmul_rn(l, urow[1]));
        x[k][0] = v;
        const double av = fabs(v);
        gmax = max(gmax, abs_bits(v));
        if (better(av, pos[k], ca, cp)) {
          ca = av;
          cp = pos[k];
          cr = lr;
        }
      }
    }
    uprev = urow;
    LEAF_MARK(5)
  }
  if (trace) {
    for (int i = 0; i < 6; ++i) p.dbg[i] += _acc[i];
    p.dbg[7] += (unsigned long long)w;
  }
  if (p.dbg != nullptr && g == 0 && _own) atomicAdd(p.dbg + 6, _own);
  __syncthreads();
  // rows go straight to their final positions; moved rows are listed so the
  // same interchanges can be applied to the other columns by a gather
#pragma unroll
  for (int k = 0; k < RPT; ++k) {
    if (pos[k] == INT_MIN) continue;
    const int lr = tid + k * NT;
    const int phys = g * R + lr;
    const int fin = pos[k] < 0 ? -pos[k] - 1 : pos[k];
    for (int c = 0; c < w; ++c) abase[(int64_t)c * p.lda + fin] = lbuf[c * R + lr];
    if (fin != phys) {
      const int slot = atomicAdd(p.list_cnt, 1);
      p.list_dst[slot] = (int32_t)(p.r0 + fin);
      p.list_src[slot] = (int32_t)(p.r0 + phys);
    }
  }
  if (p.growth) {
    const double gm = warp_max(__longlong_as_double((long long)gmax));
    if (lane == 0 && gm > 0.0) atomic_max_abs(p.growth, gm);
  }
  if constexpr (!kGrid) {
    // no CTA exits while its last record may still be copied out of its smem
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
  }
}
