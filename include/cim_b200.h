/*
 * cim_b200.h — C-ABI of the B200-native half-stored symmetric SpMM
 *
 *     Y = U·X + U_offᵀ·X  (= A·X for the full symmetric A)
 *
 * where U is the set of stored 64×64 tiles (R ≤ C, diagonal tiles held in
 * full) and U_off the stored tiles with R < C.  This is the hot path of the
 * eigensolver in arXiv 2110.10765 (Fig. 1 line 15) that the
 * reference package `cimotifs` approaches only through its pair-walk operator
 * `contract_observables` (pkg/src/cimotifs/pipeline.py:534-570).
 *
 * The reference has no C ABI; its operator boundary is Python over numpy
 * arrays.  Each entry point below states which reference
 * interface it replaces.  No torch types appear here: every buffer is a plain
 * device (or host, where stated) pointer plus sizes, owned by the caller.
 *
 * Storage ("HalfTiles", fragment layout v1)
 * -----------------------------------------
 *   tile_rc  int32 [n_tiles][2]  (R, C) with R ≤ C, sorted by R then C,
 *                                unique.  Replaces SparseSkeleton.tiles +
 *                                colind (pipeline.py:96-116): the reference
 *                                stores both triangles at entry granularity.
 *   units    int32 [n_units][4]  (R, t0, t1, 0): work units, a contiguous
 *                                tile range inside block row R.  Built by
 *                                cim_plan_units.
 *   vals     f32|f64 [n_tiles][4096] in fragment order: for tile t,
 *                                micro-row i∈[0,8), micro-block mb∈[0,128),
 *                                column slot j∈[0,4):
 *                                  vals[t][i][mb][j] = T[rg + 8i][cg + 16j]
 *                                with rg = (mb & 31) >> 2,
 *                                     cg = 4·(mb >> 5) + (mb & 3).
 *                                (f64: vals[t][i][h][mb][jj] with j = 2h+jj.)
 *                                Rows/cols ≥ n inside the last block are 0.
 *
 * Vectors: X and Y are row-major (n_pad, k) with n_pad = 64·ceil(n/64).
 * X rows ≥ n must be finite (they meet zero matrix entries).  Y rows ≥ n
 * receive zeros.  X must be dense (ldx == k); Y may be strided (ldy ≥ k,
 * ldy % 4 == 0 for f32, ldy % 2 == 0 for f64, 16-byte aligned base).
 *
 * Threading: every device entry point is asynchronous and stream-ordered;
 * calls are re-entrant for distinct Y.  The only global state is a per-device
 * cache (SM count, occupancy, a ring of scheduler counters).
 */
#ifndef CIM_B200_H
#define CIM_B200_H

#include <stdint.h>

#if defined(__GNUC__)
#define CIM_API __attribute__((visibility("default")))
#else
#define CIM_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* return codes */
#define CIM_OK            0
#define CIM_EINVAL        1   /* bad argument (shape, alignment, order)     */
#define CIM_ECUDA         2   /* a CUDA runtime call failed                 */
#define CIM_EUNSUPPORTED  3   /* k / dtype combination not compiled         */

/* dtypes */
#define CIM_F32 0
#define CIM_F64 1

/* cim_sym_spmm flags */
#define CIM_ACCUMULATE    1u  /* Y += A·X instead of Y = A·X                */
#define CIM_DETERMINISTIC 2u  /* no float atomics: every Y row block summed
                                 in a fixed order by one CTA (bitwise
                                 reproducible; needs the det_* tile lists;
                                 either tile layout; reads each tile
                                 twice — a validation mode)                */

/* cim_contract_tiles flags (with CIM_ACCUMULATE) */
#define CIM_CONTRACT_EXACT_F64 4u  /* products and sums in f64: contract_oracle
                                      (pipeline.py:573-589) instead of the
                                      reference's f32 products (:470-474)  */

/* value kinds for cim_fill_synthetic_values */
#define CIM_VALUES_H_XOR      0  /* h(i XOR j; seed)      pipeline.py:216-222 */
#define CIM_VALUES_OP_HASH    1  /* O_ij(k=op_k; seed)    pipeline.py:224-232 */
#define CIM_VALUES_IDENTITY   2  /* δ_ij                  pipeline.py:226-227 */

#define CIM_BLOCK 64

/* tile value layouts (cim_half_tiles.layout) */
#define CIM_LAYOUT_FRAG 0   /* fragment order v1: CUDA-core FFMA/FFMA2 kernel (f32, f64)   */
#define CIM_LAYOUT_TC   1   /* tensor-core kernels' layout (f32: tcgen05 split-TF32, f64:
                               DMMA): per tile, row-major rows whose 4-element chunks are
                               XOR-swizzled by row: element(r,c) = r·64 + (c/4 ^ r%8)·4 + c%4 */

/*
 * Sparse ("COO-in-tile") stored tiles, for 64-tiles below the dense
 * break-even fill (½ for f32, ⅔ for f64) — the ragged
 * orbital blocks of reference skeletons average 17% fill.  Per tile the
 * entries are sorted by local row, then column (row-major order); a column
 * permutation lists them column by column for the transposed product, so
 * both products are register reductions (no atomics inside a tile):
 *   tile_rc    int32  [n_tiles][2]   (R, C), R ≤ C (any order)
 *   entry_off  int64  [n_tiles+1]    first entry of each tile, a multiple of 16
 *                                    (entries rowptr[t][64] .. next tile are zero
 *                                    padding, so tiles stage with 16-byte copies)
 *   rowptr     uint16 [n_tiles][72]  per local row (first 65 used), offsets
 *                                    relative to the tile; 144-byte rows so a
 *                                    tile's pointers are one 16-B-aligned copy
 *   colptr     uint16 [n_tiles][72]  per local column (first 65 used), offsets into cperm
 *   col, row   uint8  [n_entries]    local column / row of each entry
 *   cperm      uint16 [n_entries]    tile-relative entry indices in column-major order
 *   vals       f32|f64[n_entries]
 * Bytes per entry: 4 + s (+ 296 B per tile), against 4096·s for a dense tile.
 */
typedef struct cim_sparse_tiles {
  int64_t         n_tiles;
  int64_t         n_entries;
  const int32_t  *tile_rc;
  const int64_t  *entry_off;
  const uint16_t *rowptr;
  const uint16_t *colptr;
  const uint8_t  *col;
  const uint8_t  *row;
  const uint16_t *cperm;
  const void     *vals;     /* dtype of the enclosing cim_half_tiles */
  /* Optional work split (NULL lists: derived on the fly by scanning
     entry_off): tiles with more than cim_sparse_small_max() padded entries
     (entry_off[t+1] − entry_off[t]) are staged through shared memory, the
     non-empty rest walked entry-parallel from global memory.  Each list holds
     tile indices; together they must cover every non-empty tile once. */
  const int32_t  *staged_tiles;
  int64_t         n_staged;
  const int32_t  *small_tiles;
  int64_t         n_small;
  /* Largest padded entry count among the staged tiles (0 = unknown); at
     ≤ 512 the staged kernel uses smaller shared-memory stages. */
  int64_t         staged_max_entries;
  /* Optional row-CSR of the small tiles (built by cim_sparse_csr_count /
     cim_exclusive_scan_i64 / cim_sparse_csr_fill).  When csr_ptr is set the
     small tiles are applied from it — row i's entries csr_ptr[i] ..
     csr_ptr[i+1] hold global columns csr_col and values csr_val (tile
     dtype), one reduction per row for the direct product — instead of
     entry-parallel from the tiles.  csr_rows = n_pad. */
  const int64_t  *csr_ptr;
  const int32_t  *csr_col;
  const void     *csr_val;
  int64_t         csr_rows;
  int64_t         csr_nnz;
  int64_t         csr_all;   /* 1: the CSR holds the staged tiles too (the
                                staged kernel is skipped by the SpMM) */
  int64_t         csr_symmetric; /* 1: the CSR rows hold both triangles of
                                the sparse tiles (each off-diagonal-block
                                entry also stored mirrored in its column's
                                row): the apply is a gather per row with no
                                transposed reductions — twice the CSR bytes
                                for the small tiles, no L2 atomics per entry */
} cim_sparse_tiles;

typedef struct cim_half_tiles {
  int64_t        n;        /* matrix order                                   */
  int32_t        block;    /* must be 64                                     */
  int32_t        dtype;    /* CIM_F32 | CIM_F64                              */
  int64_t        n_tiles;
  int64_t        n_units;
  const int32_t *tile_rc;  /* device, [n_tiles][2]                           */
  const int32_t *units;    /* device, [n_units][4]                           */
  const void    *vals;     /* device, [n_tiles][4096] in `layout` order      */
  int32_t        layout;   /* CIM_LAYOUT_FRAG | CIM_LAYOUT_TC                 */
  int32_t        reserved; /* 0                                               */
  const cim_sparse_tiles *sparse; /* NULL, or the sparse tiles of the same
                                     matrix (a tile is stored dense or sparse,
                                     never both); device arrays              */
  /* CIM_DETERMINISTIC only (else NULL): per block row b, the tiles with
     R == b (det_row_tiles[det_row_ptr[b] .. det_row_ptr[b+1]]) and the
     tiles with C == b, R < b (det_col_*), each list in (R, C) order.
     Entries t < n_tiles name dense tiles, n_tiles + s sparse tile s.      */
  const int64_t *det_row_ptr;   /* [nb+1] */
  const int32_t *det_row_tiles;
  const int64_t *det_col_ptr;   /* [nb+1] */
  const int32_t *det_col_tiles;
} cim_half_tiles;

/* Library version / build string (host). */
CIM_API const char *cim_version(void);

/* Last error message of the calling thread (host). */
CIM_API const char *cim_last_error(void);

/*
 * Y = A·X (or Y += A·X with CIM_ACCUMULATE) on `stream` (a cudaStream_t, may
 * be NULL for the legacy stream).  X, Y are device pointers to (n_pad, k)
 * row-major arrays of the tile dtype, 16-byte aligned (the kernels stage
 * 64-row X blocks with bulk / TMA tensor copies: f64 tensor-core tiles at
 * k = 16, 32 read X through a 2-D tensor map encoded per call).
 *
 * Replaces: contract_observables(...) (pipeline.py:534-570) as the operator
 * that walks every stored pair once per call; its validation contract
 * (ValueError before compute, pipeline.py:550-555) maps to CIM_EINVAL.
 * Supported k: f32 {1,2,4} ∪ 8ℕ (≤ 64); f64 {1,2} ∪ 4ℕ (≤ 64).
 *
 * Ownership and state: the caller owns X, Y and every array of H; the call
 * is stream-ordered and asynchronous, re-entrant for distinct Y.  Library
 * state per device: the SM count, a ring of scheduler counters, and, for
 * widths above one kernel pass (f32 k ∈ {24, 32, 48, 64}, f64 k ∈ {12, 16,
 * 32}), one grow-only scratch buffer per device for a pass-major copy of X
 * (n_pad · k elements; kept until process exit) whose users on different
 * streams are ordered by an event.  Counter slots are reused only after the
 * kernels that last used them finished (event-guarded ring), so concurrent
 * calls on any number of streams never share a live counter.
 *
 * Subnormals: a tile's products accumulate in registers (IEEE), but they land
 * in Y through red.global.add.f32, which PTX defines as flushing subnormal
 * operands and results to zero — an absolute error below 2⁻¹²⁶ per reduction,
 * visible only when partial sums of A·X fall under 1.2e-38.  CIM_DETERMINISTIC
 * (plain stores) keeps gradual underflow.
 */
CIM_API int cim_sym_spmm(const cim_half_tiles *H, const void *X, void *Y, int32_t k,
                 int64_t ldx, int64_t ldy, uint32_t flags, void *stream);

/*
 * Host-buffer batch: Y_b = A·X_b for b < n_batch, where X_host[b] / Y_host[b]
 * are HOST (n, k) row-major arrays of the tile dtype (pinned memory gives
 * asynchronous copies; pageable memory still works, without overlap).
 * Copies and kernels of consecutive blocks overlap on three internal streams
 * (H2D, compute, D2H) through a caller-owned device `workspace` of
 * cim_host_batch_workspace_bytes(H, k) bytes (2 X + 2 Y buffers).
 * Synchronous: returns once every Y_b is on the host.  The internal streams
 * first wait for all work queued on the legacy default stream (e.g. the fill
 * of H); work the caller queued on other streams must be complete (the
 * Python wrapper synchronises the current stream).
 *
 * Replaces: the reference's host-array operator boundary (numpy in, numpy
 * out; contract_observables writes inputs.accum in place, pipeline.py:569)
 * for a stream of independent vector blocks.
 */
CIM_API int cim_sym_spmm_host_batch(const cim_half_tiles *H, const void *const *X_host,
                                    void *const *Y_host, int32_t n_batch, int32_t k,
                                    void *workspace, uint64_t ws_bytes);

/* Device workspace bytes cim_sym_spmm_host_batch needs for (H, k). */
CIM_API uint64_t cim_host_batch_workspace_bytes(const cim_half_tiles *H, int32_t k);

/*
 * Device: G = Aᵀ·B in float64 for tall row-major blocks A (rows × ca, leading
 * dimension lda) and B (rows × cb, ldb) of dtype CIM_F32 or CIM_F64, with
 * 1 ≤ ca, cb ≤ 64; out is a device double[ca·cb] (row-major ca × cb).
 * Accumulates in f64 with a fixed reduction order (reproducible).  The
 * eigensolver's Gram / Rayleigh–Ritz products (lobpcg.py; BASELINE config 5).
 * workspace: cim_gram_workspace_bytes(rows, ca, cb) device bytes.
 *
 * Replaces: the reference's float64 oracle reductions over pair lists
 * (contract_oracle, pipeline.py:573-589) — here for the block products that
 * wrap the SpMM.
 */
CIM_API int cim_gram(const void *A, int64_t lda, int32_t ca, const void *B, int64_t ldb,
                     int32_t cb, int64_t rows, int32_t dtype, double *out,
                     void *workspace, uint64_t ws_bytes, void *stream);

/*
 * Device: Out = alpha·A·C + beta·Out for a tall f32 block A (rows × q, lda),
 * a small row-major f32 matrix C (q × p, device) and Out (rows × p, ldo),
 * 1 ≤ q, p ≤ 64 (beta = 0: Out is not read).  The eigensolver's block
 * updates, written straight into column slots of its work buffer.
 */
CIM_API int cim_tsmm(const float *A, int64_t lda, int32_t q, const float *C, int32_t p,
                     float alpha, float beta, float *Out, int64_t ldo, int64_t rows,
                     void *stream);

/*
 * Column-blocked variants: an operand of `cols` columns stored as blocks of
 * bw ∈ {4,8,16,32,64} columns, element (r, c) at
 * base + (c / bw)·bstride + r·ld + (c % bw)  (elements) — e.g. the eigensolver's
 * block-major work buffer [slot][row][bw], where a column slice of a wide
 * row-major buffer would waste most of every DRAM burst.
 * cim_gram_blocked's block_mask selects the 8×8 output blocks to compute
 * (bit bi·⌈cb/8⌉ + bj; 0 = all; the rest are written as 0) so a caller can
 * skip the mirror half of symmetric products; B == A is loaded once.
 */
CIM_API int cim_gram_blocked(const void *A, int64_t lda, int32_t a_bw, int64_t a_bstride, int32_t ca,
                             const void *B, int64_t ldb, int32_t b_bw, int64_t b_bstride, int32_t cb,
                             int64_t rows, int32_t dtype, double *out, void *workspace,
                             uint64_t ws_bytes, uint64_t block_mask, void *stream);
/* cim_gram_blocked with flags: CIM_GRAM_FAST (f32 operands) forms products
   and partial sums in f32 over runs of ≤ 32 rows, accumulating the runs in
   f64 — ~2⁻²⁴·32 relative error per run instead of exact products, for
   eigensolver Gram matrices of f32 blocks; without it, as cim_gram_blocked. */
#define CIM_GRAM_FAST 1u
CIM_API int cim_gram_blocked_ex(const void *A, int64_t lda, int32_t a_bw, int64_t a_bstride, int32_t ca,
                                const void *B, int64_t ldb, int32_t b_bw, int64_t b_bstride, int32_t cb,
                                int64_t rows, int32_t dtype, double *out, void *workspace,
                                uint64_t ws_bytes, uint64_t block_mask, uint32_t flags, void *stream);
CIM_API int cim_tsmm_blocked(const float *A, int64_t lda, int32_t a_bw, int64_t a_bstride, int32_t q,
                             const float *C, int32_t p, float alpha, float beta, float *Out,
                             int64_t ldo, int32_t o_bw, int64_t o_bstride, int64_t rows, void *stream);

/* cim_tsmm_blocked with C (q × p row-major f32, q·p ≤ 1024) read from HOST
   memory during the call and carried in the kernel parameters — no upload
   or staging buffer for the eigensolver's per-iteration coefficients. */
CIM_API int cim_tsmm_blocked_hc(const float *A, int64_t lda, int32_t a_bw, int64_t a_bstride, int32_t q,
                                const float *C_host, int32_t p, float alpha, float beta, float *Out,
                                int64_t ldo, int32_t o_bw, int64_t o_bstride, int64_t rows, void *stream);

/* Device: W = AX − X·diag(λ) over whole (rows × bw) row-major f32 slots
   (LOBPCG residuals; λ_j from HOST f64 lam[0..m), 0 for j ≥ m). */
CIM_API int cim_block_residual(const float *X, const float *AX, const double *lam_host, int32_t m, float *W,
                               int64_t rows, int32_t bw, void *stream);

/* Device: the LOBPCG Ritz update fused with the next residual, over bw = 8
   block-major f32 slots.  S and AS are q/8 consecutive slots each (q ∈ {8,
   16, 24, 32, 48}, slot stride bstride floats); C_host is the HOST q × 16
   row-major f32 coefficient matrix [C_p | C].  Writes five consecutive slots
   of Out (stride o_bstride): [S·C_p, S·C, AS·C − (S·C)·diag(λ), AS·C_p,
   AS·C] = [P', X', W', AP', AX'] with λ_j from HOST f64 lam[0..m), 0 for
   j ≥ m.  Out must not overlap S or AS. */
CIM_API int cim_ritz_update_b8(const float *S, const float *AS, int64_t bstride, int32_t q, const float *C_host,
                               const double *lam_host, int32_t m, float *Out, int64_t o_bstride, int64_t rows,
                               void *stream);

/*
 * Device: values on the entries of sparse tiles — vals_out[e] = value(i, j)
 * of entry e where mask[e] != 0 (mask: the pattern's own values, or NULL =
 * every entry), else 0.  Kinds as cim_fill_synthetic_values (the reference
 * hashes, pipeline.py:199-263).
 */
CIM_API int cim_fill_sparse_values(const cim_sparse_tiles *S, int64_t n, int32_t dtype, int32_t kind,
                                   uint64_t seed, int32_t op_k, const void *mask, void *vals_out,
                                   void *stream);

/*
 * Device construction of synthetic sparse tiles (count → scan → fill, the
 * reference's build_skeleton motif, pipeline.py:290-377, on the GPU).
 * cim_sparse_count_rows: rowcnt[t·64 + r] = kept entries of local row r of
 * tile t, kept(i, j) = symmetric hash(min, max; seed) < fill·2⁶⁴ (i, j < n).
 * The caller scans them into S->rowptr / S->entry_off and allocates the
 * entry arrays; cim_sparse_fill_entries then writes row-sorted columns, rows
 * and values of `kind` (as cim_fill_synthetic_values; h(i XOR j) bit-exact)
 * and cim_sparse_build_columns the column index (colptr, cperm) of any
 * row-sorted sparse tiles.
 */
CIM_API int cim_sparse_count_rows(const int32_t *tile_rc, int64_t n_tiles, int64_t n, double fill,
                                  uint64_t seed, int32_t *rowcnt, void *stream);
CIM_API int cim_sparse_fill_entries(const cim_sparse_tiles *S, int64_t n, int32_t dtype, double fill,
                                    uint64_t seed, int32_t kind, uint64_t value_seed, int32_t op_k,
                                    void *stream);
CIM_API int cim_sparse_build_columns(const cim_sparse_tiles *S, void *stream);

/*
 * Device construction from a many-body basis (the reference's two-pass
 * skeleton build, pipeline.py:290-377 / sparsity.py:131-193, into 64-tiles).
 * bits_lo: [n] packed occupancy of single-particle states 1..64; occ:
 * [n][n_particles] sorted 1-based occupied indices (mbstate.py Basis
 * arrays, grouped order).  Entry (i, j) is kept iff
 * popcount(bits_lo[i] ^ bits_lo[j]) ≤ threshold and the lockstep
 * occupation-list difference ≤ threshold (threshold = 2·rank); its value
 * is h(i XOR j; seed).  cim_basis_count_tiles: rowcnt[t·64 + r] = kept
 * entries of local row r of candidate tile t; the caller keeps the tiles with
 * entries, scans, and fills them dense (cim_basis_fill_dense, `layout`
 * order) or sparse (cim_basis_fill_sparse: rowptr / entry_off prefilled,
 * writes col, row, vals; then cim_sparse_build_columns).
 */
CIM_API int cim_basis_count_tiles(const uint64_t *bits_lo, const uint16_t *occ, int64_t n,
                                  int32_t n_particles, int32_t threshold, const int32_t *tile_rc,
                                  int64_t n_tiles, int32_t *rowcnt, void *stream);
CIM_API int cim_basis_fill_dense(const uint64_t *bits_lo, const uint16_t *occ, int64_t n,
                                 int32_t n_particles, int32_t threshold, const int32_t *tile_rc,
                                 int64_t n_tiles, int32_t dtype, int32_t layout, uint64_t seed,
                                 void *vals, void *stream);
CIM_API int cim_basis_fill_sparse(const uint64_t *bits_lo, const uint16_t *occ, int64_t n,
                                  int32_t n_particles, int32_t threshold, const cim_sparse_tiles *S,
                                  int32_t dtype, uint64_t seed, void *stream);

/* The small-tile threshold of the sparse path, in padded entries per tile
   (the staged_tiles / small_tiles split of cim_sparse_tiles). */
CIM_API int32_t cim_sparse_small_max(void);

/* Device workspace bytes cim_gram / cim_gram_blocked need. */
CIM_API uint64_t cim_gram_workspace_bytes(int64_t rows, int32_t ca, int32_t cb);

/*
 * Y += A·X with X and Y split into row chunks — the fused compute +
 * exchange step of the multi-GPU apply: chunk c holds block rows
 * [c·chunk_rows/64, (c+1)·chunk_rows/64) as (chunk_rows, k) row-major X
 * (ldx = k) and (chunk_rows, ldy) Y, and the pointers may be peer-mapped
 * memory of other GPUs (CUDA IPC / symmetric memory over NVLink): the
 * kernel bulk-copies X_C / X_R blocks from, and red.global-adds Y blocks
 * into, the owning rank's chunk directly — no all-gather of X, no
 * reduce-scatter of Y.  Always accumulates (the caller zeroes every chunk
 * and orders the ranks around the call).  n_chunks ≤ 8; dense
 * fragment-layout tiles; (dtype, k) of the wide-register kernel (f32 k ∈
 * {8,16,24,32,48,64}, f64 k ∈ {4,8,12,16,32}).
 */
CIM_API int cim_sym_spmm_chunked(const cim_half_tiles *H, const void *const *X_chunks,
                                 void *const *Y_chunks, int32_t n_chunks, int64_t chunk_rows,
                                 int32_t k, int64_t ldy, void *stream);

/* 1 if (dtype, k) has a compiled kernel for CIM_LAYOUT_FRAG tiles, else 0. */
CIM_API int cim_sym_spmm_supported(int32_t dtype, int32_t k);

/* 1 if (layout, dtype, k) has a compiled kernel, else 0.  CIM_LAYOUT_TC:
 * f32 with k ∈ {8, 16, …, 64} (tcgen05 kind::tf32, 3×TF32-split FP32 accuracy);
 * f64 with k ∈ {8, 16, 24, 32} (mma.sync DMMA m8n8k4) and k = 64 (two
 * column passes of 32 over a pass-major copy of X in a per-device scratch
 * buffer, as for the fragment layout's multi-pass widths). */
CIM_API int cim_layout_supports(int32_t layout, int32_t dtype, int32_t k);

/*
 * Host: build work units from a sorted tile list (R, C pairs, host memory).
 * Every block row's tiles are split into runs of at most `max_unit` tiles.
 * units_out must hold n_tiles*4 int32 (upper bound); *n_units_out receives
 * the count.  Also validates order (R ≤ C, sorted, unique, in range nb).
 *
 * Replaces: the per-(tile,row) segment layout CountsAndOffsets built by
 * counts_to_offsets (pipeline.py:319-330, fill.py:79-91).
 */
CIM_API int cim_plan_units(const int32_t *tile_rc_host, int64_t n_tiles, int64_t nb,
                   int32_t max_unit, int32_t *units_out, int64_t *n_units_out);

/*
 * Host: as cim_plan_units for tiles stored in column bands: tile order is
 * (C / band_cols, R, C) and units never cross a band.  Streaming the
 * matrix band by band keeps the random side of the transposed product
 * (X_C gathers, Y_C atomics) inside an L2-sized slice of X and Y.
 * band_cols ≥ nb gives the plain row-major order of cim_plan_units.
 */
CIM_API int cim_plan_units_banded(const int32_t *tile_rc_host, int64_t n_tiles, int64_t nb,
                                  int32_t max_unit, int64_t band_cols, int32_t *units_out,
                                  int64_t *n_units_out);

/*
 * Host: split units into `parts` contiguous ranges with balanced tile counts
 * (row-block sharding over GPUs).  bounds_out[parts+1].
 */
CIM_API int cim_partition_units(const int32_t *units_host, int64_t n_units,
                        int32_t parts, int64_t *bounds_out);

/*
 * Device: fill `vals` (fragment order, dtype) with synthetic symmetric
 * values for the tiles in tile_rc: kind CIM_VALUES_H_XOR gives the reference
 * matrix values h(i XOR j; seed) (pipeline.py:216-222, _h_values_np :247-249),
 * bit-exact after rounding to f32 (f64 tiles hold the same f32 values).
 * Entries with i ≥ n or j ≥ n are 0.
 */
CIM_API int cim_fill_synthetic_values(const int32_t *tile_rc, int64_t n_tiles, int64_t n,
                              int32_t dtype, int32_t layout, int32_t kind, uint64_t seed,
                              int32_t op_k, void *vals, void *stream);

/*
 * Device: operator values on a stored pattern — vals[e] = value(i,j) where
 * mask[e] != 0, else 0 (both in fragment order).  Gives the reference's
 * observable operators O_ij(k) (pipeline.py:224-232) restricted to the
 * interacting pairs, for the GPU contract_observables.
 */
CIM_API int cim_fill_masked_values(const int32_t *tile_rc, int64_t n_tiles, int64_t n,
                                   int32_t dtype, int32_t layout, int32_t kind, uint64_t seed,
                                   int32_t op_k, const void *mask, void *vals,
                                   void *stream);

/*
 * Device: the observables contraction in one tile walk (
 * replaces contract_observables' kernels, pipeline.py:461-570):
 *   accum[v*m_ops + k] (+)= Σ_(i,j) c[i*n_vec + v] · O_ij(k) · c[j*n_vec + v]
 * over the full symmetric pattern of H (its nonzero stored elements, dense and
 * sparse tiles; off-diagonal tiles count for both (i,j) and (j,i)), with
 * O_ij(k) computed on the fly: kind CIM_VALUES_OP_HASH (_op_value,
 * pipeline.py:224-232) or CIM_VALUES_IDENTITY.  c is f32 (n, n_vec)
 * row-major on the device, accum f64 (n_vec, m_ops) on the device, zeroed
 * first unless flags has CIM_ACCUMULATE.  Stream-ordered; accum is summed with
 * f64 atomics (reproducible to rounding).
 */
CIM_API int cim_contract_observables(const cim_half_tiles *H, const float *c, int32_t n_vec,
                                     int32_t m_ops, int32_t kind, uint64_t seed, double *accum,
                                     uint32_t flags, void *stream);

/*
 * Device: contract_observables / contract_oracle over the reference's own
 * ORBITAL tiles — the literal drop-in of pipeline.py:534-589 (a Tile list,
 * its Orbitals, the Basis and the InteractionRank):
 *   accum[v*m_ops + k] (+)= Σ_t Σ_(i∈[r0,r1), j∈[c0,c1), kept(i,j)) c[i*ldc+v]·O_ij(k)·c[j*ldc+v]
 * tile_ranges int32 (n_tiles, 4) on the device = (r0, r1, c0, c1) of each
 * tile's row / column orbital (0 ≤ r0 < r1 ≤ n, same for c; the caller swaps
 * them for the transposed walk, pipeline.py:446-447); kept(i, j) is the
 * count predicate of _collect_pairs (popcount(bits_lo[i] ^ bits_lo[j]) ≤
 * threshold and the lockstep occupation difference ≤ threshold,
 * pipeline.py:270-280 / sparsity.py:132-151); bits_lo uint64 (n,) and occ
 * uint16 (n, n_particles) in grouped order on the device.  c f32 (n, ldc)
 * row-major on the device.  kind CIM_VALUES_OP_HASH or CIM_VALUES_IDENTITY.
 * Products are the reference's f32 (c_vi·o)·c_vj, summed in f32 per lane and
 * f64 across lanes, or all-f64 with CIM_CONTRACT_EXACT_F64.  accum f64
 * (n_vec, m_ops) on the device, zeroed first unless CIM_ACCUMULATE.
 */
CIM_API int cim_contract_tiles(const uint64_t *bits_lo, const uint16_t *occ, int64_t n,
                               int32_t n_particles, int32_t threshold, const int32_t *tile_ranges,
                               int64_t n_tiles, const float *c, int64_t ldc, int32_t n_vec,
                               int32_t m_ops, int32_t kind, uint64_t seed, double *accum,
                               uint32_t flags, void *stream);

/*
 * Device: the row-CSR of a sparse tile set's SMALL tiles (small_tiles list),
 * for the row-walk apply (cim_sparse_tiles.csr_*).  cim_sparse_csr_count:
 * row_cnt int64 [n_pad] = small-tile entries per global row (zeroed first).
 * The caller scans it (cim_exclusive_scan_i64 → csr_ptr [n_pad+1]), then
 * cim_sparse_csr_fill copies the entries: one thread per (panel, local row)
 * walks the panel's small tiles in list order, so the entry order is
 * deterministic.  Panels: the block rows holding small tiles, panel p =
 * small_tiles[panel_ptr[p] .. panel_ptr[p+1]) all of block row panel_R[p]
 * (the list is grouped by block row).  csr_col int32 global columns,
 * csr_val in `dtype`.
 */
CIM_API int cim_sparse_csr_count(const cim_sparse_tiles *S, int64_t n_pad, int64_t *row_cnt, void *stream);
CIM_API int cim_sparse_csr_fill(const cim_sparse_tiles *S, int32_t dtype, const int32_t *panel_R,
                                const int64_t *panel_ptr, int64_t n_panels, const int64_t *csr_ptr,
                                int32_t *csr_col, void *csr_val, void *stream);

/*
 * Device: exclusive prefix sum of int64 counts — the reference's scan motif
 * (scan_serial, scan.py:131-139; CountsAndOffsets, scan.py:45-65) for the
 * count → scan → fill construction: y[i] = Σ_(j<i) x[j] for i < n and
 * y[n] = the total (so y is offsets followed by total; y has n+1 slots).
 * Reduce-then-scan in three stream-ordered launches (fixed summation order:
 * bitwise deterministic); x may alias y[0..n) only if x == y.  Scratch for
 * the per-block sums is stream-ordered (cudaMallocAsync).
 */
CIM_API int cim_exclusive_scan_i64(const int64_t *x, int64_t n, int64_t *y, void *stream);

/*
 * Device: the per-tile row scan of the sparse-tile build.  rowcnt int32
 * [n_tiles][64] (entries per local row) → rowptr int16 [n_tiles][72]
 * (rowptr[t][r] = Σ_(r'<r) rowcnt[t][r'], r ≤ 64; slots 65..71 zero),
 * counts int64 [n_tiles] (real entries per tile) and entry_off int64
 * [n_tiles+1] = exclusive scan of counts rounded up to `align` (the padded
 * tile ranges of cim_sparse_tiles), via cim_exclusive_scan_i64.
 */
CIM_API int cim_sparse_tile_offsets(const int32_t *rowcnt, int64_t n_tiles, int32_t align,
                                    int16_t *rowptr, int64_t *counts, int64_t *entry_off,
                                    void *stream);

/*
 * Device: repack row-major dense tiles src[n_tiles][64][64] into fragment
 * order dst (same dtype).  The repacking layer's device half
 * (SURVEY.md §7 step 4).
 */
CIM_API int cim_pack_tiles(const void *src_rowmajor, int64_t n_tiles, int32_t dtype,
                   int32_t layout, void *dst_fragment, void *stream);

/* Device: inverse of cim_pack_tiles (debug / export). */
CIM_API int cim_unpack_tiles(const void *src_fragment, int64_t n_tiles, int32_t dtype,
                     int32_t layout, void *dst_rowmajor, void *stream);

/*
 * Device: the reference's value hashes on explicit index arrays, for parity
 * checks of the device hash against _h_values_np / _op_values_np
 * (pipeline.py:247-263).  out is f32[count].
 */
CIM_API int cim_hash_values(const int64_t *i, const int64_t *j, int64_t count,
                    int32_t kind, uint64_t seed, int32_t op_k, float *out,
                    void *stream);

#ifdef __cplusplus
}
#endif
#endif /* CIM_B200_H */
