// gemm_emu.cu — K3+K4+K5 of SURVEY §2.2: the Ozaki-INT8 emulated DGEMM.
//
// Reference semantics (/root/reference/pkg/src/ozemu/gemm.py):
//   pairs (i,j) with i+j <= t, ordered by (i+j, i)               :157-178
//   out = 0; for (i,j): out += ldexp(A_i @ B_j, eA+eB-(i+j)q)   :214-222
//   out = alpha*out; out = out + beta*c                          :266-270
// The integer products A_i @ B_j are exact (INT32 on the tensor cores), the
// FP64 accumulation is done per element in the reference pair order with one
// rounding per pair (fma(P, 2^-(i+j)q, acc)), and the row/column exponent is
// applied once at the end (exact power-of-two scaling) — bit-identical to the
// reference whenever no intermediate over/underflows.
//
// Kernel design (sm_100a), emu_gemm_pair_kernel:
//   * CTA pairs (__cluster_dims__(2), tcgen05.mma.cta_group::2.kind::i8,
//     M=256, N=128, K=32): each CTA stages its own 128 rows of A and half of
//     B, so B is shared across the pair; one persistent pair per two SMs walks
//     a grouped raster of 256x128 output tiles;
//   * loop order tile -> exact-level group -> pair -> K; each group's INT32
//     sum lands in one of 4 TMEM accumulators (128 columns each), so the
//     epilogue of one group overlaps the MMAs of the next;
//   * operands are K-major int8 slice tiles (128 rows x 128 bytes) staged by
//     TMA (cp.async.bulk.tensor.3d, 128B swizzle) through an 8-stage ring;
//   * warp roles: w8 TMA producer, w9 MMA issuer (leader CTA), w10 TMEM
//     allocator, w0..w7 epilogue (each owns 32 TMEM lanes x 64 columns and
//     keeps its 64 FP64 accumulators in registers for the whole pair loop);
//   * the FP64 recombine, alpha/beta epilogue (C read once, written once) and
//     the optional growth max (solve.py:135) are fused in the epilogue.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <stdlib.h>
#include <vector>

#include "common.cuh"

namespace oz {
namespace emu {

constexpr int BM = 128;   // rows of A per CTA (TMA box)
constexpr int BK = 128;   // bytes of K per stage (one 128B swizzle atom)
constexpr int NUM_ACC = 4;
constexpr int TMEM_COLS = 512;
constexpr int NUM_THREADS = 384;
constexpr int EPI_WARPS = 8;
constexpr int MAX_PAIRS = 256;
constexpr int GROUP_M = 16;


struct Params {
  int m, n, inner;
  int num_m_tiles, num_n_tiles, num_tiles;
  int nkb;
  int npairs;
  const int32_t* expA;
  const int32_t* expB;
  double* c;
  int64_t ldc;
  int c_is_input;
  double alpha, beta;
  unsigned long long* growth;
  int32_t* debug_out;  // pair-debug mode: raw INT32 product
  int64_t ldo;
  int ngroups;
  int group_m;  // raster band height in tiles
  int experiment;  // tuning only (OZ_GEMM_EXPERIMENT): 1 = skip FP64 math, 2 = also skip final pass
  int wide;        // slice_bits > 7: (hi, lo) int8 planes per slice
  int prefetch_c;  // C is read by the final pass: stage it into L2 ahead of it
  unsigned long long* starts;  // tuning only (OZ_GEMM_STARTS): per-CTA start/end globaltimer
  uint8_t pa[MAX_PAIRS];
  uint8_t pb[MAX_PAIRS];
  uint16_t gshift[MAX_PAIRS];      // (i+j)*q of the group's pairs
  uint16_t gstart[MAX_PAIRS + 1];  // group g = pairs [gstart[g], gstart[g+1])
};

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t* v) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]),
        "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]),
        "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// Warp-uniform issue helpers: the whole warp runs the issue loops (so loop
// state stays in uniform registers) and elect.sync picks the issuing lane.
__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(pred));
  return pred != 0;
}
// K-major, 128B-swizzled shared-memory matrix descriptor (8-row groups 1024B apart).
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {
  uint64_t d = (uint64_t)((saddr & 0x3FFFFu) >> 4);
  d |= (uint64_t)1 << 16;            // leading byte offset (unused for SW128 K-major)
  d |= (uint64_t)(1024 >> 4) << 32;  // stride byte offset
  d |= (uint64_t)1 << 46;            // descriptor version (sm_100)
  d |= (uint64_t)2 << 61;            // SWIZZLE_128B
  return d;
}

// exact int32 -> double: the magic-number trick (one DADD on the FP64 pipe)
// or the I2F.F64 conversion (OZ_CVT=1 build), chosen by measurement
#ifdef OZ_CVT_I2F
__device__ __forceinline__ double i32_to_f64(uint32_t v) { return __int2double_rn((int)v); }
#else
__device__ __forceinline__ double i32_to_f64(uint32_t v) {
  const double d = __hiloint2double(0x43300000, (int)(v ^ 0x80000000u));
  return __dsub_rn(d, 4503601774854144.0);  // 2^52 + 2^31
}
#endif

__device__ __forceinline__ void tile_coords(const Params& p, int t, int& mt, int& nt) {
  const int per_group = p.group_m * p.num_n_tiles;
  const int g = t / per_group;
  const int first_m = g * p.group_m;
  int gm = p.num_m_tiles - first_m;
  gm = gm < p.group_m ? gm : p.group_m;
  const int r = t - g * per_group;
  mt = first_m + r % gm;
  nt = r / gm;
}

// =====================================================================
// CTA-pair variant (cta_group::2): the pair computes a 256 x 128 tile; each
// CTA stages its own 128 rows of A and one half (64 rows) of B, the leader
// issues M=256 MMAs that read both CTAs' shared memory, and each CTA's
// epilogue owns its 128 x 128 block.  Per SM this ingests 24 KB per 256
// MMA-cycles instead of 32 KB (the single-CTA kernel is ingress-bound, see
// profiles/r01_mma_microbench.txt).
// =====================================================================
constexpr int P_BM = 256;
constexpr int P_BN = 128;
constexpr int P_STAGES = 8;
constexpr int P_SGROUP = 4;  // 16 MMAs per tcgen05.commit
constexpr int P_A_BYTES = 128 * BK;
constexpr int P_B_BYTES = (P_BN / 2) * BK;
constexpr int P_STAGE_BYTES = P_A_BYTES + P_B_BYTES;
constexpr size_t P_SMEM_BYTES = 1024 + (size_t)P_STAGES * P_STAGE_BYTES + 256;
constexpr uint32_t P_IDESC = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(P_BN >> 3) << 17) |
                             ((uint32_t)(P_BM >> 4) << 24);
constexpr int FP_CHUNK = 8;  // final-pass columns with loads in flight at once
// Warp roles.  The issue arbiter favours the highest warp id of each SMSP
// (warp w runs on SMSP w % 4), so the TMA producer and the MMA issuer take
// warps 8 and 9 — the top ids of SMSPs 0 and 1 — and are never starved by the
// epilogue warps 0-7 that share those SMSPs.
constexpr int P_PRODUCER = 8, P_MMA = 9, P_ALLOC = 10;
constexpr int P_EPI_ARRIVALS = 2 * EPI_WARPS;

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}
__device__ __forceinline__ uint32_t mapa_shared(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void mbar_arrive_remote(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
// TMA into this CTA's shared memory; the transaction bytes land on the
// leader CTA's barrier (peer bit cleared), as in CUTLASS's 2SM loads.
__device__ __forceinline__ void tma_load_3d_pair(uint32_t dst, const CUtensorMap* map,
                                                 uint32_t bar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(bar & 0xFEFFFFFFu)
      : "memory");
}
__device__ __forceinline__ void tc_commit_pair(uint32_t bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;\n\t}" ::"r"(bar),
      "h"((uint16_t)3)
      : "memory");
}
__device__ __forceinline__ void tc_mma_i8_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                               uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// One K stage (4 MMAs of K=32) of the pair kernel in a single asm block: one
// elect.sync, descriptors built from their 32-bit low words (the high word —
// stride, version, swizzle — is constant), so ptxas emits no per-MMA vote or
// 64-bit address arithmetic.
__device__ __forceinline__ void tc_mma_i8_pair_stage(uint32_t tmem_d, uint32_t a_lo, uint32_t b_lo,
                                                     uint32_t hi, uint32_t idesc,
                                                     uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t.reg .b64 da, db;\n\t.reg .b32 al, bl;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %5, 0;\n\t"
      "mov.b64 da, {%1, %3};\n\tmov.b64 db, {%2, %3};\n\t"
      "@e tcgen05.mma.cta_group::2.kind::i8 [%0], da, db, %4, p;\n\t"
      "add.u32 al, %1, 2;\n\tadd.u32 bl, %2, 2;\n\t"
      "mov.b64 da, {al, %3};\n\tmov.b64 db, {bl, %3};\n\t"
      "@e tcgen05.mma.cta_group::2.kind::i8 [%0], da, db, %4, 1;\n\t"
      "add.u32 al, %1, 4;\n\tadd.u32 bl, %2, 4;\n\t"
      "mov.b64 da, {al, %3};\n\tmov.b64 db, {bl, %3};\n\t"
      "@e tcgen05.mma.cta_group::2.kind::i8 [%0], da, db, %4, 1;\n\t"
      "add.u32 al, %1, 6;\n\tadd.u32 bl, %2, 6;\n\t"
      "mov.b64 da, {al, %3};\n\tmov.b64 db, {bl, %3};\n\t"
      "@e tcgen05.mma.cta_group::2.kind::i8 [%0], da, db, %4, 1;\n\t}" ::"r"(tmem_d),
      "r"(a_lo), "r"(b_lo), "r"(hi), "r"(idesc), "r"(accumulate)
      : "memory");
}

__device__ __forceinline__ void pair_tile_coords(const Params& p, int t, int& mt, int& nt) {
  tile_coords(p, t, mt, nt);  // same grouped raster, on pair tiles (num_m_tiles in 256 rows)
}

// kWide (slice_bits 8..10): each slice is a (hi, lo) pair of int8 planes
// (split.cu) and a slice-pair product is 16384*P(hi,hi) + 128*(P(hi,lo) +
// P(lo,hi)) + P(lo,lo).  The three INT32 parts of a group land in TMEM slots
// 0, 1, 2 and the epilogue recombines them exactly (integers < 2^53) before
// the reference-order FP64 accumulation; one group is in flight at a time.
template <bool kDebug, bool kWide>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(NUM_THREADS, 1)
    emu_gemm_pair_kernel(const __grid_constant__ CUtensorMap tmA,
                         const __grid_constant__ CUtensorMap tmB, const __grid_constant__ Params p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* smA = smem;
  uint8_t* smB = smem + P_STAGES * P_A_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + P_STAGES * P_STAGE_BYTES);
  uint64_t* full = bars;
  uint64_t* empty = bars + P_STAGES;
  uint64_t* tfull = bars + 2 * P_STAGES;
  uint64_t* tempty = bars + 2 * P_STAGES + NUM_ACC;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * P_STAGES + 2 * NUM_ACC);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;

  if (threadIdx.x == 0) {
    for (int s = 0; s < P_STAGES; ++s) {
      mbar_init(smem_u32(&full[s]), 1);
      mbar_init(smem_u32(&empty[s]), 1);
    }
    for (int b = 0; b < NUM_ACC; ++b) {
      mbar_init(smem_u32(&tfull[b]), 1);
      mbar_init(smem_u32(&tempty[b]), P_EPI_ARRIVALS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == P_PRODUCER && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
  }
  if (warp == P_ALLOC) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  if (p.starts != nullptr && threadIdx.x == 0) {
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    p.starts[blockIdx.x] = t0;
  }

  if (warp >= P_PRODUCER) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 40;");
  }
  if (warp == P_PRODUCER) {
    // ------------------------------------------------------------ TMA producer
    int stage = 0;
    uint32_t phase = 0;
    for (int t = cid; t < p.num_tiles; t += ncl) {
      int mt, nt;
      pair_tile_coords(p, t, mt, nt);
      const int arow = mt * P_BM + (int)rank * 128;
      const int brow = nt * P_BN + (int)rank * (P_BN / 2);
      for (int q = 0; q < p.npairs; ++q) {
       for (int sub = 0; sub < (kWide ? 4 : 1); ++sub) {
        // kWide sub-products: (hi,hi), (hi,lo), (lo,hi), (lo,lo) planes
        const int sa = kWide ? 2 * p.pa[q] + (sub >> 1) : p.pa[q];
        const int sb = kWide ? 2 * p.pb[q] + (sub & 1) : p.pb[q];
        for (int kb = 0; kb < p.nkb; ++kb) {
          if (stage % P_SGROUP == 0) mbar_wait(smem_u32(&empty[stage / P_SGROUP]), phase ^ 1);
          if (elect_one()) {
            const uint32_t fb = smem_u32(&full[stage]);
            if (leader) mbar_expect_tx(fb, 2 * P_STAGE_BYTES);
            const uint32_t fb_leader = mapa_shared(fb, 0);  // both CTAs signal the leader
            tma_load_3d_pair(smem_u32(smA + stage * P_A_BYTES), &tmA, fb_leader, kb * BK, arow,
                             sa);
            tma_load_3d_pair(smem_u32(smB + stage * P_B_BYTES), &tmB, fb_leader, kb * BK, brow,
                             sb);
          }
          __syncwarp();
          if (++stage == P_STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
       }
      }
    }
  } else if (warp == P_MMA) {
    // ------------------------------------------------ MMA issuer (leader CTA only)
    if (leader) {
      const uint64_t adesc0 = sdesc(smem_u32(smA));
      const uint64_t bdesc0 = sdesc(smem_u32(smB));
      const uint32_t a_lo0 = (uint32_t)adesc0, b_lo0 = (uint32_t)bdesc0;
      const uint32_t desc_hi = (uint32_t)(adesc0 >> 32);  // == bdesc0 >> 32
      int stage = 0;
      uint32_t phase = 0;
      uint32_t it = 0;
      for (int t = cid; t < p.num_tiles; t += ncl) {
        for (int g = 0; g < p.ngroups; ++g, ++it) {
          const uint32_t ring = kWide ? 1 : NUM_ACC;  // kWide: one slot triple
          const uint32_t buf = it % ring, aph = (it / ring) & 1;
          mbar_wait(smem_u32(&tempty[buf]), aph ^ 1);
          tc_fence_after();
          for (int q = p.gstart[g]; q < p.gstart[g + 1]; ++q) {
            const bool first_pair = q == p.gstart[g];
           for (int sub = 0; sub < (kWide ? 4 : 1); ++sub) {
            // kWide: (hi,hi) -> slot 0, (hi,lo) and (lo,hi) -> slot 1, (lo,lo) -> slot 2
            const uint32_t slot = kWide ? (sub == 0 ? 0u : sub == 3 ? 2u : 1u) : buf;
            const bool opens = first_pair && (!kWide || sub != 2);
            const uint32_t dtmem = tmem_base + slot * P_BN;
            for (int kb = 0; kb < p.nkb; ++kb) {
              mbar_wait(smem_u32(&full[stage]), phase);
              tc_fence_after();
              static_assert(BK / 32 == 4, "stage issue assumes 4 MMAs per stage");
              tc_mma_i8_pair_stage(dtmem, a_lo0 + (uint32_t)stage * (P_A_BYTES >> 4),
                                   b_lo0 + (uint32_t)stage * (P_B_BYTES >> 4), desc_hi, P_IDESC,
                                   (opens && kb == 0) ? 0u : 1u);
              if (stage % P_SGROUP == P_SGROUP - 1)
                tc_commit_pair(smem_u32(&empty[stage / P_SGROUP]));
              __syncwarp();
              if (++stage == P_STAGES) {
                stage = 0;
                phase ^= 1;
              }
            }
           }
          }
          tc_commit_pair(smem_u32(&tfull[buf]));
          __syncwarp();
        }
      }
    }
  } else if (warp < P_PRODUCER) {
    // --------------------------------------------------------------- epilogue
    asm volatile("setmaxnreg.inc.sync.aligned.u32 232;");
    const int quad = warp & 3;  // TMEM lane quadrant this warp may access
    const int half = warp >> 2;  // column half
    const uint32_t lane_base = (uint32_t)(quad * 32) << 16;
    // TMEM-slot releases go to the leader's barrier as plain remote arrives:
    // tcgen05.wait::ld + fence::before_thread_sync already order our reads.
    const uint32_t tempty_leader = mapa_shared(smem_u32(tempty), 0);
    double gmax = 0.0;
    uint32_t it = 0;
    for (int t = cid; t < p.num_tiles; t += ncl) {
      int mt, nt;
      pair_tile_coords(p, t, mt, nt);
      double acc[64];
#pragma unroll
      for (int i = 0; i < 64; ++i) acc[i] = 0.0;
      const int row = mt * P_BM + (int)rank * 128 + quad * 32 + lane;
      const int col0 = nt * P_BN + half * 64;
      const int pf_group = p.ngroups > 3 ? p.ngroups - 3 : 0;
      for (int q = 0; q < p.ngroups; ++q, ++it) {
        if (q == pf_group && p.prefetch_c && row < p.m) {
          // The final pass reads this thread's row of the tile's C block
          // (64 columns).  Pull those lines into L2 about three groups ahead,
          // so the read-modify-write runs at L2 rather than DRAM latency and
          // the next tile's MMAs (at most 4 TMEM slots ahead) wait less on it.
          const char* pf = reinterpret_cast<const char*>(p.c + (int64_t)col0 * p.ldc + row);
          const int pc = min(64, p.n - col0);
          for (int i = 0; i < pc; ++i)
            asm volatile("prefetch.global.L2 [%0];" ::"l"(pf + (int64_t)i * p.ldc * 8));
        }
        if constexpr (kWide) {
          // slot triple: exact 16384*hh + 128*mid + ll per element, then one
          // reference-order FMA; 16 columns at a time keeps registers in budget
          const uint32_t aph = it & 1;
          mbar_wait(smem_u32(&tfull[0]), aph);
          tc_fence_after();
          const uint32_t tb = tmem_base + lane_base + half * 64;
          const double s = pow2(-(int)p.gshift[q]);
#pragma unroll
          for (int c = 0; c < 64; c += 16) {
            uint32_t hh[16], mid[16], ll[16];
            tmem_ld16(tb + c, hh);
            tmem_ld16(tb + P_BN + c, mid);
            tmem_ld16(tb + 2 * P_BN + c, ll);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              const double t = __dadd_rn(fma(i32_to_f64(hh[i]), 16384.0,
                                             __dmul_rn(i32_to_f64(mid[i]), 128.0)),
                                         i32_to_f64(ll[i]));
              acc[c + i] = fma(t, s, acc[c + i]);
            }
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_remote(tempty_leader);
          continue;
        }
        const uint32_t buf = it % NUM_ACC, aph = (it / NUM_ACC) & 1;
        mbar_wait(smem_u32(&tfull[buf]), aph);
        tc_fence_after();
        const uint32_t taddr = tmem_base + lane_base + buf * P_BN + half * 64;
        uint32_t v[64];
        tmem_ld32(taddr, v);
        tmem_ld32(taddr + 32, v + 32);
        tmem_wait_ld();
        // the slot is free as soon as its values sit in registers
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_remote(tempty_leader + buf * 8);
        if (kDebug) {
#pragma unroll 4
          for (int i = 0; i < 64; ++i) {
            const int col = col0 + i;
            if (row < p.m && col < p.n) p.debug_out[(int64_t)col * p.ldo + row] = (int32_t)v[i];
          }
        } else if (p.experiment == 0) {
          const double s = pow2(-(int)p.gshift[q]);
#pragma unroll
          for (int i = 0; i < 64; ++i) acc[i] = fma(i32_to_f64(v[i]), s, acc[i]);
        }
      }
      if (kDebug || p.experiment >= 2) continue;
      {
        // every lane runs the loop (the exponent shuffles need the full warp);
        // rows past m only skip their loads and stores
        // final pass: out = alpha * ldexp(acc, er + eb) + beta * C, written
        // once.  FP_CHUNK columns per (rolled) iteration with the accumulator
        // registers shifted down so indices stay static; the column exponents
        // come from two coalesced loads + a warp shuffle per column; the LU's
        // alpha = -1, beta = 1 case is C - ab (bit-identical, one DADD).
        const bool row_ok = row < p.m;
        const int er = row_ok ? p.expA[row] : 0;
        const bool use_c = p.c_is_input && p.beta != 0.0;
        const bool lu_form = use_c && p.alpha == -1.0 && p.beta == 1.0;
        const int ncols = min(64, p.n - col0);
        const int64_t ldc = p.ldc;
        double* cp = p.c + (int64_t)col0 * ldc + row;
        const int eb_lo = lane < ncols ? __ldg(p.expB + col0 + lane) : 0;
        const int eb_hi = lane + 32 < ncols ? __ldg(p.expB + col0 + 32 + lane) : 0;
#pragma unroll 1
        for (int c0 = 0; c0 < ncols; c0 += FP_CHUNK) {
          double cv[FP_CHUNK];
          {
            const double* cq = cp;
#pragma unroll
            for (int i = 0; i < FP_CHUNK; ++i) {
              cv[i] = (use_c && row_ok && c0 + i < ncols) ? *cq : 0.0;
              cq += ldc;
            }
          }
#pragma unroll
          for (int i = 0; i < FP_CHUNK; ++i) {
            const int c = c0 + i;
            const int eb = __shfl_sync(0xffffffffu, c < 32 ? eb_lo : eb_hi, c & 31);
            if (row_ok && c < ncols) {
              const double ab = ldexp_exact(acc[i], er + eb);
              double out;
              if (lu_form) {
                out = __dsub_rn(cv[i], ab);
              } else {
                out = __dmul_rn(p.alpha, ab);
                if (use_c) out = __dadd_rn(out, __dmul_rn(p.beta, cv[i]));
              }
              *cp = out;
              gmax = fmax(gmax, fabs(out));
            }
            cp += ldc;
          }
#pragma unroll
          for (int i = 0; i < 64 - FP_CHUNK; ++i) acc[i] = acc[i + FP_CHUNK];
        }
      }
    }
    if (p.growth != nullptr) {
      gmax = warp_max(gmax);
      if (lane == 0 && gmax > 0.0) atomic_max_abs(p.growth, gmax);
    }
  }

  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  if (p.starts != nullptr && threadIdx.x == 0) {
    unsigned long long t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    p.starts[gridDim.x + blockIdx.x] = t1;
  }
  if (warp == P_ALLOC) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(TMEM_COLS)
                 : "memory");
  }
}

// ------------------------------------------------------------------ host side
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static const PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult qres;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &qres) ==
            cudaSuccess &&
        qres == cudaDriverEntryPointSuccess)
      return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
    return (PFN_cuTensorMapEncodeTiled_v12000) nullptr;
  }();
  return fn;
}

int make_slice_map(CUtensorMap* map, const int8_t* base, int64_t inner, int64_t rows,
                   int64_t ld, int64_t sstride, int nslices, int box_rows = BM) {
  auto fn = encode_fn();
  OZ_REQUIRE(fn != nullptr, OZ_CUDA_ERROR, "cuTensorMapEncodeTiled unavailable");
  OZ_REQUIRE((reinterpret_cast<uintptr_t>(base) & 15) == 0, OZ_INVALID_PARAMS,
             "slice buffer must be 16-byte aligned");
  OZ_REQUIRE(ld % 16 == 0 && sstride % 16 == 0, OZ_INVALID_PARAMS,
             "slice strides must be multiples of 16 bytes");
  cuuint64_t dims[3] = {(cuuint64_t)inner, (cuuint64_t)rows, (cuuint64_t)nslices};
  cuuint64_t strides[2] = {(cuuint64_t)ld, (cuuint64_t)sstride};
  cuuint32_t box[3] = {(cuuint32_t)BK, (cuuint32_t)box_rows, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<int8_t*>(base), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  OZ_REQUIRE(r == CUDA_SUCCESS, OZ_CUDA_ERROR, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return OZ_OK;
}

// Exact-level grouping.  The reference adds the scaled pair products one by one
// into an FP64 accumulator (gemm.py:218-222).  While every partial sum is
// exactly representable no rounding happens, so the pairs of such a level can
// be summed first (exactly, in INT32 on the tensor core) without changing a
// single bit.  A level qualifies when (a) its INT32 sum cannot overflow and
// (b) the running magnitude bound, in units of the level's LSB 2^-shift, stays
// below 2^53.  From the first level that fails, every pair is its own group
// and is accumulated in the reference order with one rounding per pair.
void build_groups(Params& p, const int32_t* shift, int npairs, int64_t inner, int q) {
  // max |P| of one pair: K * (2^q - 1)^2 (q > 7: int16 slices), and the INT32
  // sub-accumulators hold at most K * 127^2 per pair (int8 operands)
  const double smax = q > 7 ? (double)((1 << q) - 1) : 127.0;
  const double term = (double)inner * smax * smax;
  const double term32 = (double)inner * 127.0 * 127.0;
  double bound = 0.0;                                  // sum of max |P_p| * 2^-shift_p
  bool exact = true;
  int g = 0, i = 0;
  while (i < npairs) {
    int j = i;
    while (j < npairs && shift[j] == shift[i]) ++j;
    bool grouped = false;
    if (exact) {
      const double lvl = term * (j - i);
      const double nb = bound + ldexp(lvl, -shift[i]);
      if (term32 * (j - i) < 2147483648.0 && ldexp(nb, shift[i]) < 9007199254740992.0) {
        bound = nb;
        grouped = true;
      } else {
        exact = false;
      }
    }
    if (grouped) {
      p.gstart[g] = (uint16_t)i;
      p.gshift[g] = (uint16_t)shift[i];
      ++g;
    } else {
      for (int q = i; q < j; ++q) {
        p.gstart[g] = (uint16_t)q;
        p.gshift[g] = (uint16_t)shift[q];
        ++g;
      }
    }
    i = j;
  }
  p.gstart[g] = (uint16_t)npairs;
  p.ngroups = g;
}

struct StartLog {
  static constexpr int LAUNCHES = 256;
  unsigned long long* buf = nullptr;
  int used = 0;
  int grid[LAUNCHES], m[LAUNCHES], n[LAUNCHES];
};
StartLog& start_log() {
  static StartLog lg;
  if (!lg.buf) {
    cudaMalloc(&lg.buf, sizeof(unsigned long long) * StartLog::LAUNCHES * 2 * 512);
    cudaMemset(lg.buf, 0, sizeof(unsigned long long) * StartLog::LAUNCHES * 2 * 512);
  }
  return lg;
}

int launch_pair(const CUtensorMap& ta, const CUtensorMap& tb, Params& p, cudaStream_t st,
                int max_ctas = 0) {
  OZ_ONCE([] {
    cudaError_t e = cudaFuncSetAttribute(emu_gemm_pair_kernel<false, false>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)P_SMEM_BYTES);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(emu_gemm_pair_kernel<false, true>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, (int)P_SMEM_BYTES);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(emu_gemm_pair_kernel<true, false>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, (int)P_SMEM_BYTES);
    return e;
  }());
  p.num_m_tiles = (int)ceil_div(p.m, P_BM);
  p.num_n_tiles = (int)ceil_div(p.n, P_BN);
  p.num_tiles = p.num_m_tiles * p.num_n_tiles;
  p.nkb = (int)ceil_div(p.inner, BK);
  // raster band: long-K products (standalone DGEMM) keep only 2 m-tiles of A
  // in flight so the concurrently streamed slices stay L2-resident; the LU's
  // K = nb updates prefer wide bands (measured, scripts/sweep_groupm.sh)
  p.group_m = p.inner >= 4096 ? 2 : GROUP_M;
  if (const char* g = getenv("OZ_GEMM_GROUPM")) p.group_m = atoi(g) > 0 ? atoi(g) : p.group_m;
  if (const char* e = getenv("OZ_GEMM_EXPERIMENT")) p.experiment = atoi(e);
  p.prefetch_c = p.c_is_input && p.beta != 0.0 && p.debug_out == nullptr &&
                 getenv("OZ_GEMM_NO_PREFETCH") == nullptr;  // tuning switch
  int grid = sm_count() & ~1;
  if (const char* g = getenv("OZ_GEMM_GRID")) grid = atoi(g) > 0 ? (atoi(g) & ~1) : grid;
  if (max_ctas > 0 && grid > (max_ctas & ~1)) grid = max_ctas & ~1;
  if (grid < 2) grid = 2;
  if (grid > 2 * p.num_tiles) grid = 2 * p.num_tiles;
  p.starts = nullptr;
  if (getenv("OZ_GEMM_STARTS")) {  // tuning: CTA start/end spread of every launch
    StartLog& lg = start_log();
    if (lg.used < StartLog::LAUNCHES) {
      p.starts = lg.buf + (size_t)lg.used * 2 * 512;
      lg.grid[lg.used] = grid;
      lg.m[lg.used] = p.m;
      lg.n[lg.used] = p.n;
      ++lg.used;
    }
  }
  if (p.debug_out != nullptr)
    emu_gemm_pair_kernel<true, false><<<grid, NUM_THREADS, P_SMEM_BYTES, st>>>(ta, tb, p);
  else if (p.wide)
    emu_gemm_pair_kernel<false, true><<<grid, NUM_THREADS, P_SMEM_BYTES, st>>>(ta, tb, p);
  else
    emu_gemm_pair_kernel<false, false><<<grid, NUM_THREADS, P_SMEM_BYTES, st>>>(ta, tb, p);
  OZ_CHECK_LAUNCH();
  return OZ_OK;
}

}  // namespace emu

int gemm_emu_launch(int64_t m, int64_t n, int64_t inner, const int8_t* a_slices, int64_t a_ld,
                    int64_t a_sstride, int a_nslices, const int32_t* a_exps,
                    const int8_t* b_slices, int64_t b_ld, int64_t b_sstride, int b_nslices,
                    const int32_t* b_exps, int npairs, const int32_t* pair_a,
                    const int32_t* pair_b, const int32_t* pair_shift, int slice_bits,
                    double alpha, double beta, double* c, int64_t ldc, int c_is_input,
                    unsigned long long* growth, cudaStream_t st, int max_ctas) {
  using namespace emu;
  OZ_REQUIRE(slice_bits >= 1 && slice_bits <= 10, OZ_INVALID_PARAMS, "slice_bits outside 1..10");
  const bool wide = slice_bits > 7;  // slices are (hi, lo) int8 plane pairs
  OZ_REQUIRE(m >= 1 && n >= 1 && inner >= 1, OZ_INVALID_PARAMS, "empty GEMM");
  OZ_REQUIRE(m < (1ll << 31) && n < (1ll << 31), OZ_INVALID_PARAMS, "dimension too large");
  OZ_REQUIRE(inner * 127ll * 127ll < (1ll << 31), OZ_ACC_OVERFLOW,
             "inner dimension %lld breaks exact INT32 accumulation of int8 slices",
             (long long)inner);
  OZ_REQUIRE(npairs >= 1 && npairs <= MAX_PAIRS, OZ_INVALID_PARAMS, "npairs out of range");
  OZ_REQUIRE(ldc >= m, OZ_INVALID_PARAMS, "ldc < m");
  Params p{};
  p.m = (int)m;
  p.n = (int)n;
  p.inner = (int)inner;
  p.npairs = npairs;
  for (int i = 0; i < npairs; ++i) {
    OZ_REQUIRE(pair_a[i] >= 0 && pair_a[i] < a_nslices && pair_b[i] >= 0 &&
                   pair_b[i] < b_nslices && pair_shift[i] >= 0 && pair_shift[i] < 1000,
               OZ_INVALID_PARAMS, "bad pair table entry %d", i);
    OZ_REQUIRE(i == 0 || pair_shift[i] >= pair_shift[i - 1], OZ_INVALID_PARAMS,
               "pair table must be ordered by level");
    p.pa[i] = (uint8_t)pair_a[i];
    p.pb[i] = (uint8_t)pair_b[i];
  }
  build_groups(p, pair_shift, npairs, inner, slice_bits);
  p.wide = wide ? 1 : 0;
  p.expA = a_exps;
  p.expB = b_exps;
  p.c = c;
  p.ldc = ldc;
  p.c_is_input = c_is_input;
  p.alpha = alpha;
  p.beta = beta;
  p.growth = growth;
  CUtensorMap ta, tb;
  OZ_TRY(make_slice_map(&ta, a_slices, inner, m, a_ld, a_sstride, wide ? 2 * a_nslices : a_nslices,
                        BM));
  OZ_TRY(make_slice_map(&tb, b_slices, inner, n, b_ld, b_sstride, wide ? 2 * b_nslices : b_nslices,
                        P_BN / 2));
  return launch_pair(ta, tb, p, st, max_ctas);
}

}  // namespace oz

extern "C" int oz_gemm_emu(int64_t m, int64_t n, int64_t inner, const int8_t* a_slices,
                           int64_t a_ld, int64_t a_sstride, int a_nslices, const int32_t* a_exps,
                           const int8_t* b_slices, int64_t b_ld, int64_t b_sstride, int b_nslices,
                           const int32_t* b_exps, int npairs, const int32_t* pair_a,
                           const int32_t* pair_b, const int32_t* pair_shift, int slice_bits,
                           double alpha, double beta, double* c, int64_t ldc, int c_is_input,
                           unsigned long long* growth_max, void* stream) {
  cudaStream_t st = oz::as_stream(stream);
  const int tag = oz::prof_start(st);
  const int s = oz::gemm_emu_launch(m, n, inner, a_slices, a_ld, a_sstride, a_nslices, a_exps,
                                    b_slices, b_ld, b_sstride, b_nslices, b_exps, npairs, pair_a,
                                    pair_b, pair_shift, slice_bits, alpha, beta, c, ldc,
                                    c_is_input, growth_max, st, 0);
  oz::prof_stop(tag, st, oz::PROF_EMU_GEMM, 2.0 * npairs * (double)m * n * inner);
  return s;
}

extern "C" int oz_gemm_pair_i32(int64_t m, int64_t n, int64_t inner, const int8_t* a_slice,
                                int64_t a_ld, const int8_t* b_slice, int64_t b_ld, int32_t* out,
                                int64_t ldo, void* stream) {
  using namespace oz;
  using namespace oz::emu;
  OZ_REQUIRE(m >= 1 && n >= 1 && inner >= 1, OZ_INVALID_PARAMS, "empty GEMM");
  OZ_REQUIRE(inner * 127ll * 127ll < (1ll << 31), OZ_ACC_OVERFLOW, "inner too large");
  OZ_REQUIRE(ldo >= m, OZ_INVALID_PARAMS, "ldo < m");
  Params p{};
  p.m = (int)m;
  p.n = (int)n;
  p.inner = (int)inner;
  p.npairs = 1;
  p.ngroups = 1;
  p.gstart[0] = 0;
  p.gstart[1] = 1;
  p.gshift[0] = 0;
  p.debug_out = out;
  p.ldo = ldo;
  p.alpha = 1.0;
  CUtensorMap ta, tb;
  OZ_TRY(make_slice_map(&ta, a_slice, inner, m, a_ld, round_up(m * a_ld, 16), 1, BM));
  OZ_TRY(make_slice_map(&tb, b_slice, inner, n, b_ld, round_up(n * b_ld, 16), 1, P_BN / 2));
  return launch_pair(ta, tb, p, as_stream(stream));
}

// Host-only: expose the exact-level grouping plan (for tests / introspection).
// gstart must hold npairs+1 entries; returns the number of groups.
extern "C" int oz_plan_groups(int npairs, const int32_t* pair_shift, int64_t inner,
                              int slice_bits, int32_t* gstart, int32_t* gshift) {
  using namespace oz;
  using namespace oz::emu;
  OZ_REQUIRE(npairs >= 1 && npairs <= MAX_PAIRS, OZ_INVALID_PARAMS, "npairs out of range");
  Params p{};
  build_groups(p, pair_shift, npairs, inner, slice_bits);
  for (int g = 0; g <= p.ngroups; ++g) gstart[g] = p.gstart[g];
  for (int g = 0; g < p.ngroups; ++g) gshift[g] = p.gshift[g];
  return p.ngroups;
}

// Tuning only (OZ_GEMM_STARTS=1): per launch, the spread of CTA start times
// and of CTA end times (globaltimer, us), to spot late-starting CTAs.
extern "C" int oz_gemm_starts_dump(void) {
  using namespace oz::emu;
  StartLog& lg = start_log();
  cudaDeviceSynchronize();
  std::vector<unsigned long long> h((size_t)lg.used * 2 * 512);
  cudaMemcpy(h.data(), lg.buf, h.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
  for (int i = 0; i < lg.used; ++i) {
    const unsigned long long* s0 = h.data() + (size_t)i * 2 * 512;
    const int g = lg.grid[i];
    unsigned long long smin = ~0ull, smax = 0, emin = ~0ull, emax = 0;
    for (int b = 0; b < g; ++b) {
      smin = s0[b] < smin ? s0[b] : smin;
      smax = s0[b] > smax ? s0[b] : smax;
      emin = s0[g + b] < emin ? s0[g + b] : emin;
      emax = s0[g + b] > emax ? s0[g + b] : emax;
    }
    fprintf(stderr, "gemm %3d m=%6d n=%6d grid=%3d  start spread %8.1f us  end spread %8.1f us  "
            "duration %8.1f us\n", i, lg.m[i], lg.n[i], g, (smax - smin) / 1e3, (emax - emin) / 1e3,
            (emax - smin) / 1e3);
  }
  lg.used = 0;
  return 0;
}
