/*
 * ozb200.h — C ABI of the B200-native Ozaki-INT8 HPL hot path.
 *
 * Plain pointers, sizes and an opaque cudaStream_t (passed as void*).  No
 * torch types cross this boundary.  Every entry point returns an oz_status;
 * oz_last_error() returns a thread-local message for the most recent failure
 * on the calling thread.  The Python drop-in (paper_2509_23565_b200/_lib.py)
 * maps the codes onto the reference exception hierarchy
 * (/root/reference/pkg/src/ozemu/errors.py:4-41).
 *
 * Matrix conventions
 *   - FP64 matrices are addressed by (row_stride, col_stride) in elements, so
 *     row-major (numpy C order) and column-major (LAPACK/HPL order) views are
 *     both accepted without copies.
 *   - Slice stacks are int8, "K-major": slice s, vector v, inner index t lives
 *     at slices[s*slice_stride + v*slice_ld + t].  slice_ld is a multiple of 16
 *     bytes (TMA global-stride rule); bytes in [K, slice_ld) are written as 0.
 *   - The emulated GEMM writes its output column-major with respect to its own
 *     (m, n): out[col*ldc + row].  A row-major caller swaps the operands.
 *
 * Device pointers are CUDA global memory on the current device; `stream` is a
 * cudaStream_t (NULL = legacy default stream).
 */
#ifndef OZB200_H
#define OZB200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes (errors.py:4-41 mapping in paper_2509_23565_b200/_lib.py). */
enum oz_status {
  OZ_OK = 0,
  OZ_INVALID_PARAMS = 1,   /* InvalidParamsError      errors.py:8   */
  OZ_NON_FINITE = 2,       /* NonFiniteEntryError     errors.py:16  */
  OZ_SHAPE = 3,            /* ShapeMismatchError      errors.py:20  */
  OZ_ACC_OVERFLOW = 4,     /* AccumulatorOverflowError errors.py:28 */
  OZ_SINGULAR_PIVOT = 5,   /* SingularPivotError      errors.py:32  */
  OZ_CUDA_ERROR = 6,       /* runtime / driver / cuBLAS failure      */
  OZ_UNSUPPORTED = 7       /* configuration not supported on device  */
};

/* Orientation / ScalingMode (split.py:31-46). */
enum oz_orientation { OZ_ROW_SCALED = 0, OZ_COL_SCALED = 1 };
enum oz_scaling { OZ_PER_VECTOR = 0, OZ_GLOBAL = 1 };

/* Matrix generators (matgen.py:133-171). */
enum oz_gen_kind {
  OZ_GEN_UNIFORM = 0,            /* hpl_uniform: u - 0.5             matgen.py:164-171 */
  OZ_GEN_PARAWILK = 1,           /* deterministic pattern            matgen.py:133-146 */
  OZ_GEN_PARAWILK_RANDOMIZED = 2 /* pattern, zeros <- 2*u*u          matgen.py:149-161 */
};

const char* oz_last_error(void);
int oz_version(void);
/* Number of kernels this library has launched (process-wide, monotone). */
long long oz_launch_count(void);
/* Per-phase CUDA-event timing: enable (and clear) / read.  summary writes
 * 12 kinds x {total ms, launches, algorithmic work}; kinds: 0 emulated GEMM
 * (work = INT8 ops), 1 panel, 2 Schur cuBLAS DGEMM (flops), 3 split (bytes),
 * 4 laswp gather, 5 trsm kernel, 6 solve, 7 other, 8 swap composition,
 * 9 in-panel DGEMM, 10 trsm DGEMM. */
int oz_prof_enable(int on);
int oz_prof_summary(double* out);
/* Number of SMs of the current device (used by host-side schedulers). */
int oz_sm_count(int* out);

/* Scratch needed by oz_split (device bytes). */
size_t oz_split_aux_bytes(void);

/*
 * split_matrix (split.py:109-160): per-vector (or global) frexp exponent of
 * max|x|, then num_slices truncated slice_bits-bit signed slices.
 * Bit-exact with the reference.  `aux` is device scratch of
 * oz_split_aux_bytes() bytes; after the call aux[0] (int32) is nonzero iff a
 * NaN/Inf was seen (the Python layer raises NonFiniteEntryError).
 * slice_bits 1..7: int8 slices, plane s = slice s.  slice_bits 8..10 (the
 * reference's int16 slices, split.py:144): 2 * num_slices int8 planes,
 * plane 2s = floor(slice / 128), plane 2s+1 = slice mod 128 (slice =
 * 128 * hi + lo); oz_gemm_emu takes the same planes with the same slice_bits
 * and recombines every slice product exactly.
 */
int oz_split(const double* src, int64_t rows, int64_t cols,
             int64_t row_stride, int64_t col_stride,
             int orientation, int mode, int num_slices, int slice_bits,
             int8_t* slices, int64_t slice_ld, int64_t slice_stride,
             int32_t* exps, void* aux, void* stream);

/*
 * Emulated product + epilogue (gemm.py:190-229 and :266-270):
 *   P_p  = A_slice[pa[p]] . B_slice[pb[p]]^T        exact INT32 (tcgen05 kind::i8)
 *   acc  = sum_p P_p * 2^-(shift[p])  in the given order, one FP64 rounding per pair
 *   ab   = acc * 2^(expA[row] + expB[col])
 *   out  = alpha*ab ; if (c_is_input && beta != 0) out = out + beta*c
 * Pairs are 0-based slice indices; shift[p] = (i+j)*q with 1-based i, j.
 * Requires inner * (2^q - 1)^2 < 2^31 (exact INT32 accumulation).
 * growth_max (optional, device uint64): atomicMax of the IEEE bits of |out|.
 */
int oz_gemm_emu(int64_t m, int64_t n, int64_t inner,
                const int8_t* a_slices, int64_t a_ld, int64_t a_sstride, int a_nslices,
                const int32_t* a_exps,
                const int8_t* b_slices, int64_t b_ld, int64_t b_sstride, int b_nslices,
                const int32_t* b_exps,
                int npairs, const int32_t* pair_a, const int32_t* pair_b,
                const int32_t* pair_shift, int slice_bits,
                double alpha, double beta, double* c, int64_t ldc, int c_is_input,
                unsigned long long* growth_max, void* stream);

/* Host-only: the exact-level grouping plan oz_gemm_emu uses (see
 * csrc/gemm_emu.cu build_groups).  Returns the group count; gstart[0..G] are
 * pair offsets, gshift[0..G) the (i+j)*q of each group. */
int oz_plan_groups(int npairs, const int32_t* pair_shift, int64_t inner, int slice_bits,
                   int32_t* gstart, int32_t* gshift);

/* One slice-pair product as raw INT32 (debug/parity: test_gemm.py:218-240). */
int oz_gemm_pair_i32(int64_t m, int64_t n, int64_t inner,
                     const int8_t* a_slice, int64_t a_ld,
                     const int8_t* b_slice, int64_t b_ld,
                     int32_t* out, int64_t ldo, void* stream);

/* Native FP64 GEMM comparator (gemm.py:259-262) through cuBLAS DGEMM,
 * column-major: C = alpha*A*B + beta*C. */
int oz_dgemm(int transa, int transb, int64_t m, int64_t n, int64_t k, double alpha,
             const double* a, int64_t lda, const double* b, int64_t ldb, double beta,
             double* c, int64_t ldc, void* stream);

/* The reference's alpha/beta epilogue on a finished product (gemm.py:266-270),
 * elementwise over `count` contiguous doubles, each step rounded on its own:
 * out = ab; if alpha != 1: out = alpha*out; if use_c: out = out + beta*c.
 * (The native path computes ab with oz_dgemm(alpha=1, beta=0) first, so the
 * result equals numpy's `alpha*(a@b) + beta*c` bit for bit whenever the
 * products agree.)  ab and out may alias; c may be NULL when use_c == 0. */
int oz_axpby(int64_t count, double alpha, const double* ab, double beta, const double* c,
             int use_c, double* out, void* stream);

/*
 * Blocked right-looking LU with partial pivoting (solve.py:66-140) on a
 * column-major n x n matrix, in place.  backend 0 = native FP64 Schur update
 * (cuBLAS DGEMM), 1 = Ozaki-INT8 emulated Schur update with the given pair
 * table and per-vector exponents, 2 = the same with one exponent per operand
 * (ScalingMode.GLOBAL, split.py:131-134); the step-level entries below take
 * the same codes.  ipiv (device int32[n]) receives LAPACK-style 0-based row
 * interchanges; `stats` (device double[4]) receives {observed max, max|A|, -, -}
 * for the growth factor; `info` (device int32) = first zero-pivot column + 1 or 0.
 */
size_t oz_lu_workspace_bytes(int64_t n, int64_t nb, int num_slices, int slice_bits);
int oz_lu_factor(double* a, int64_t n, int64_t lda, int64_t nb,
                 int backend, int num_slices, int slice_bits,
                 int npairs, const int32_t* pair_a, const int32_t* pair_b,
                 const int32_t* pair_shift,
                 int32_t* ipiv, double* stats, int32_t* info,
                 void* workspace, size_t workspace_bytes, void* stream);

/* Host helper: LAPACK ipiv -> permutation vector (pivots[i] = original row). */
int oz_ipiv_to_perm(const int32_t* ipiv_host, int64_t n, int64_t* perm_host);

/* lu_solve (solve.py:143-156): x = U^-1 L^-1 b[perm] on device. */
int oz_lu_solve(const double* lu, int64_t n, int64_t lda, const int64_t* perm,
                const double* b, double* x, void* workspace, size_t workspace_bytes,
                void* stream);
size_t oz_lu_solve_workspace_bytes(int64_t n);

/* scaled_residual inputs (solve.py:181-214): out[0]=||Ax-b||_inf,
 * out[1]=||A||_inf, out[2]=||x||_inf, out[3]=||b||_inf.  A addressed by
 * strides; summation order is fixed (deterministic). */
int oz_residual_norms(const double* a, int64_t n, int64_t row_stride, int64_t col_stride,
                      const double* x, const double* b, double* out, void* stream);

/* b = A @ ones(n) (harness.py:126), A addressed by strides. */
int oz_row_sums(const double* a, int64_t n, int64_t row_stride, int64_t col_stride,
                double* out, void* stream);

/* max |A| over an m x n strided matrix into out[0] (device double). */
int oz_max_abs(const double* a, int64_t m, int64_t n, int64_t row_stride,
               int64_t col_stride, double* out, void* stream);

/*
 * Generators (matgen.py:133-171), bit-exact with numpy's PCG64
 * default_rng(seed).random((n, n)).  (state, inc) are the 128-bit PCG64 state
 * after seeding, split in hi/lo words.  Output element (i, j) is written at
 * out[i*row_stride + j*col_stride].
 */
int oz_generate(int kind, int64_t n, int64_t depth, int64_t block, double alpha,
                uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo,
                double* out, int64_t row_stride, int64_t col_stride, void* stream);

/* oz_lu_factor while the caller is still uploading the matrix in column
 * chunks: chunk_events[c] (cudaEvent_t) fires once columns [c*chunk_cols,
 * (c+1)*chunk_cols) are in place.  Panel 0, the update of panel 1's columns
 * and panel 1 start as soon as their chunks are in; step 0's update of the
 * other columns follows the upload chunk by chunk. */
int oz_lu_factor_overlapped(double* a, int64_t n, int64_t lda, int64_t nb, int backend,
                            int num_slices, int slice_bits, int npairs, const int32_t* pair_a,
                            const int32_t* pair_b, const int32_t* pair_shift, int32_t* ipiv,
                            double* stats, int32_t* info, void* workspace, size_t ws_bytes,
                            void* const* chunk_events, int64_t chunk_cols, void* stream);
/* *flag <- 1 if any entry is NaN or infinite (flag is not cleared). */
int oz_nonfinite_flag(const double* a, int64_t m, int64_t n, int64_t row_stride,
                      int64_t col_stride, int32_t* flag, void* stream);
/* cudaMemcpy2DAsync host -> device (a column block of a row-major host matrix). */
int oz_memcpy2d_h2d(void* dst, size_t dpitch, const void* src, size_t spitch, size_t width,
                    size_t height, void* stream);

/* Out-of-place strided copy (layout change), e.g. row-major -> column-major. */
int oz_copy2d(const double* src, int64_t rows, int64_t cols, int64_t src_rs, int64_t src_cs,
              double* dst, int64_t dst_rs, int64_t dst_cs, void* stream);


/*
 * Step-level LU (the loop of solve.py:94-140 owned by the caller; used by the
 * distributed block-cyclic HPL drivers, hpl.py and hpl2d.py).  All take the LU workspace
 * (oz_lu_workspace_bytes(ws_n, ws_nb, num_slices, slice_bits) bytes) and its
 * shape; ws_slices counts int8 planes (num_slices, doubled for slice_bits > 7).
 *
 * oz_lu_ws_init:  zero the workspace's barriers/tags (once per factorization).
 * oz_lu_panel:    factor the m x jb panel at `a` (its diagonal corner, rows
 *                 numbered from global row `base`) in place: partial pivoting
 *                 with np.argmax order, division, outer-product update
 *                 (solve.py:66-91); interchanges applied to the panel columns
 *                 only.  ipiv[0..jb) <- global pivot rows; info <- first zero
 *                 pivot (global column + 1); growth_bits <- max |entry| seen.
 *                 max_ctas > 0 keeps every kernel of the panel to that many
 *                 CTAs (a look-ahead panel beside a trailing update).
 * oz_laswp:       apply ipiv[0..npiv) (rows k1.., global values) as
 *                 sequential interchanges to columns [c0a,c1a) U [c0b,c1b)
 *                 (solve.py:80-82 whole-row swaps; LAPACK dlaswp); npiv <= 1024;
 *                 fastest for getrf pivots (ipiv[t] >= k1 + t).
 * oz_trsm_lunit:  B <- L11^-1 B, L11 unit lower jb x jb (solve.py:123-127).
 * oz_schur_update: A22 -= A21 @ U12 through backend 0 (cuBLAS DGEMM) or 1
 *                 (Ozaki-INT8 emulated, pair table as oz_gemm_emu), growth
 *                 folded into growth_bits (solve.py:130-135).
 * oz_max_abs_bits: max |a| (upper != 0: only c >= r) folded into *bits.
 */
int oz_lu_ws_init(void* workspace, size_t workspace_bytes, int64_t ws_n, int64_t ws_nb,
                  int ws_slices, void* stream);
int oz_lu_panel(double* a, int64_t lda, int64_t m, int64_t jb, int64_t base, int32_t* ipiv,
                int32_t* info, unsigned long long* growth_bits, void* workspace,
                size_t workspace_bytes, int64_t ws_n, int64_t ws_nb, int ws_slices,
                int max_ctas, void* stream);
/* SMs the look-ahead model gives the panel of an m-row trailing matrix
 * (0: no look-ahead); npairs = 0 for the native backend.  A function of m
 * only (ncols is accepted for ABI stability), identical in every driver, so
 * the panel's factors do not depend on how the columns are distributed. */
int oz_lookahead_sms(int64_t m, int64_t ncols, int64_t nb, int npairs);
/* Two-phase look-ahead: how many of this rank's rest_cols trailing columns
 * (the next panel's excluded) to update on sms - panel_sms SMs while the
 * panel runs; the remaining columns go on every SM once it is done. */
int64_t oz_lookahead_cols1(int64_t m, int64_t rest_cols, int64_t nb, int npairs, int panel_sms);
int oz_laswp(double* a, int64_t lda, int64_t c0a, int64_t c1a, int64_t c0b, int64_t c1b,
             int64_t k1, const int32_t* ipiv, int npiv, void* workspace,
             size_t workspace_bytes, int64_t ws_n, int64_t ws_nb, int ws_slices, void* stream);
int oz_trsm_lunit(const double* l11, int64_t ldl, int64_t jb, double* b, int64_t ldb,
                  int64_t ncols, void* stream);
int oz_schur_update(int backend, int64_t m, int64_t ncols, int64_t jb, const double* a21,
                    int64_t lda21, const double* u12, int64_t ldu, double* a22, int64_t lda22,
                    int num_slices, int slice_bits, int npairs, const int32_t* pair_a,
                    const int32_t* pair_b, const int32_t* pair_shift,
                    unsigned long long* growth_bits, void* workspace, size_t workspace_bytes,
                    int64_t ws_n, int64_t ws_nb, void* stream);
/* The same update in two calls for look-ahead drivers: oz_schur_split splits
 * A21 (row-scaled) and U12 (column-scaled) into the workspace once (backend 1;
 * a no-op for backend 0), oz_schur_cols then updates columns [c0, c1) of A22
 * on at most max_ctas CTAs (0 = all SMs). */
int oz_schur_split(int backend, int64_t m, int64_t ncols, int64_t jb, const double* a21,
                   int64_t lda21, const double* u12, int64_t ldu, int num_slices, int slice_bits,
                   void* workspace, size_t workspace_bytes, int64_t ws_n, int64_t ws_nb,
                   void* stream);
int oz_schur_cols(int backend, int64_t m, int64_t ncols, int64_t jb, const double* a21,
                  int64_t lda21, const double* u12, int64_t ldu, double* a22, int64_t lda22,
                  int num_slices, int slice_bits, int npairs, const int32_t* pair_a,
                  const int32_t* pair_b, const int32_t* pair_shift,
                  unsigned long long* growth_bits, int64_t c0, int64_t c1, int max_ctas,
                  void* workspace, size_t workspace_bytes, int64_t ws_n, int64_t ws_nb,
                  void* stream);
int oz_max_abs_bits(const double* a, int64_t m, int64_t n, int64_t row_stride,
                    int64_t col_stride, int upper, unsigned long long* bits, void* stream);

/* One diagonal block of lu_solve's triangular solves (solve.py:152-155), in
 * place on x[0..nb): unit lower (upper = 0) or upper (upper = 1, *flag <- 1
 * on a zero diagonal).  workspace: oz_lu_solve_workspace_bytes(nb) bytes. */
int oz_trsv_block(const double* a, int64_t lda, int64_t nb, int upper, double* x,
                  int32_t* flag, void* workspace, size_t workspace_bytes, void* stream);

/* Partial products over a block of columns (distributed rhs / residual,
 * harness.py:126, solve.py:195-198): ax[i] = sum_j a_ij x_j (x null -> 1),
 * asum[i] = sum_j |a_ij| (asum may be null).  Fixed summation order. */
int oz_gemv_partial(const double* a, int64_t rows, int64_t cols, int64_t row_stride,
                    int64_t col_stride, const double* x, double* ax, double* asum,
                    void* stream);

/* The generators' 1 x Q block-cyclic column slab of process column q
 * (local column lc = global column ((lc/nb)*Q + q)*nb + lc%nb), column-major
 * with leading dimension ldo; values identical to oz_generate's. */
int oz_generate_cyclic(int kind, int64_t n, int64_t depth, int64_t block, double alpha,
                       uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo,
                       int64_t nb, int64_t Q, int64_t q, int64_t ncols, double* out,
                       int64_t ldo, void* stream);

/* The same on a P x Q block-cyclic grid: local row lr of process row p is
 * global row ((lr/nb)*P + p)*nb + lr%nb; mloc local rows, ldo >= mloc. */
int oz_generate_block_cyclic(int kind, int64_t n, int64_t depth, int64_t block, double alpha,
                             uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi,
                             uint64_t inc_lo, int64_t nb, int64_t P, int64_t p, int64_t mloc,
                             int64_t Q, int64_t q, int64_t ncols, double* out, int64_t ldo,
                             void* stream);

/*
 * P x Q (P > 1) HPL steps (dpanel.cu).  The panel's rows are spread over the
 * P ranks of a process column, so each panel column's pivot search is a
 * candidate exchange: oz_dpanel_candidate writes this rank's record
 * (3 + 2*jb doubles: max |a[lr0.., t]|, its global row, whether this rank
 * owns global row g = j + t, that row and row g's panel entries), the caller
 * all-gathers the P records along the process column (NCCL), and
 * oz_dpanel_apply picks the same winner on every rank (largest |v|, then
 * smallest global row = np.argmax order), swaps rows g and the pivot row in
 * the panel columns, sets ipiv[t] (global row) and *info on a zero pivot,
 * divides the column below g by the pivot and applies the outer-product
 * update with separately rounded product and difference (solve.py:75-90).
 * a is the panel's first column on this rank (local rows, leading dim lda);
 * lr0 = first local row with global index >= g.
 *
 * oz_gather_rows / oz_scatter_rows: copy local rows rows[0..nrows) of
 * columns [c0a,c1a) U [c0b,c1b) to / from rows buf_rows[0..nrows) (null:
 * 0..nrows) of buf (column-major, leading dim ldb), for the row
 * interchanges that cross process rows.
 * oz_scatter_vec: dst[global(lr0 + i)] = src[i], i < count (row map of p).
 */
int oz_dpanel_candidate(const double* a, int64_t lda, int64_t lr0, int64_t mloc, int t, int jb,
                        int owns_g, int64_t nb, int64_t P, int64_t p, double* rec, void* stream);
int oz_dpanel_apply(double* a, int64_t lda, int64_t lr0, int64_t mloc, int t, int jb, int64_t g,
                    int owns_g, int64_t nb, int64_t P, int64_t p, const double* recs,
                    int32_t* ipiv, int32_t* info, unsigned long long* growth_bits,
                    void* stream);
int oz_gather_rows(const double* a, int64_t lda, const int32_t* rows, int64_t nrows, int64_t c0a,
                   int64_t c1a, int64_t c0b, int64_t c1b, double* buf, const int32_t* buf_rows,
                   int64_t ldb, void* stream);
int oz_scatter_rows(double* a, int64_t lda, const int32_t* rows, int64_t nrows, int64_t c0a,
                    int64_t c1a, int64_t c0b, int64_t c1b, const double* buf,
                    const int32_t* buf_rows, int64_t ldb, void* stream);
int oz_scatter_vec(const double* src, int64_t lr0, int64_t count, int64_t nb, int64_t P,
                   int64_t p, double* dst, void* stream);

/* P x Q gathered panel (hpl2d.py): dst[i + c*ldd] = src[blk[i]*src_block +
 * c*src_ld + row[i]] for i < nrows, c < ncols.  Assembles the all-gathered
 * local panel slabs of a process column (P stacked column-major blocks of
 * leading dimension src_ld) into the global panel in row order, and (blk =
 * NULL) copies a rank's own rows of the factored panel back into its slab. */
int oz_assemble_rows(const double* src, int64_t src_ld, int64_t src_block, const int32_t* blk,
                     const int32_t* row, int64_t nrows, int64_t ncols, double* dst, int64_t ldd,
                     void* stream);

/* Tuning only: with OZ_GEMM_STARTS=1 in the environment every emulated-GEMM
 * launch logs its CTAs' start/end times; this prints the spreads to stderr. */
int oz_gemm_starts_dump(void);
/* Tuning only (OZ_PANEL_TIMING=1): copy and clear the 8 panel-leaf phase
 * counters (clock64 sums of CTA 0 thread 0: argmax, reduce, push, deferred
 * update, wait, step tail; [6] owner record+push; [7] steps). */
int oz_panel_debug_counters(unsigned long long* out8);

#ifdef __cplusplus
}
#endif
#endif /* OZB200_H */
