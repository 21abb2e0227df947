/*
 * spamm_b200.h -- C ABI of the B200-native SpAMM hot path.
 *
 * Plain pointers, sizes and opaque handles only (no torch types in the
 * signatures; the one CUDA type is spamm_stream_t, the layout of a
 * cudaStream_t, declared here without the CUDA headers).  Every entry point returns SPAMM_OK (0) or an error code
 * and records a message retrievable with spamm_last_error() (thread-local).
 * Calls are synchronous from the caller's point of view: results are ready
 * on return.  Trees are immutable after construction and safe to share
 * between concurrent readers; calls that touch the same device serialise on
 * a per-device lock.
 *
 * Reference interfaces replaced (arxiv/paper_1011_3534, pkg/src/spamm):
 *   spamm_tree_from_host      <- quadtree.from_dense          quadtree.py:218-251
 *   (+ _async / spamm_tree_wait: the same build overlapping queued work)
 *                                (+ QuadTreeMatrix.__init__    quadtree.py:116-151)
 *   spamm_tree_to_host        <- QuadTreeMatrix.to_dense      quadtree.py:184-187, :264-266
 *   spamm_tree_padded_to_host <- QuadTreeMatrix._padded       quadtree.py:145
 *   spamm_tree_pyramid_to_host<- QuadTreeMatrix._norm_sq / _occupied  quadtree.py:131-138
 *   spamm_tree_info_get       <- logical_dim/leaf_size/depth/padded_dim/dtype, norm()
 *                                                              quadtree.py:95-162, :189-191
 *   spamm_multiply            <- multiply.spamm               multiply.py:144-221
 *                                (_leaf_stage :224-257, _merge_contributions :119-141)
 *   spamm_stats               <- multiply.ProductStats        multiply.py:93-116
 *   spamm_product_boxes       <- ProductStats.boxes / PrunedBox multiply.py:77-90, :214-218
 *   spamm_tree_recompute_norms<- the fresh norms of audit_norm_cache quadtree.py:325-340
 *   spamm_tree_diff_norm      <- the dense norm in multiply_error  multiply.py:276
 *   spamm_tree_add            <- quadtree.add                 quadtree.py:280-293
 *   spamm_tree_scale          <- quadtree.scale               quadtree.py:296-299
 *   spamm_tree_filter_drop    <- quadtree.filter_drop         quadtree.py:302-316
 *   spamm_tree_diagonal       <- the diagonal of quadtree.trace quadtree.py:274-277
 *   spamm_tree_blocks_to_host <- _blocks[_leaf_nonzero]       quadtree.py:120-151
 *   (+ _async / spamm_transfer_wait: the same copy overlapping later calls)
 *   spamm_boxes_morton_order  <- the sort in write_box_log     multiply.py:306-315
 *                                (key: ordering._interleave3   ordering.py:24-34)
 *   spamm_tree_toeplitz       <- generators.gen_exponential / gen_algebraic
 *                                                              generators.py:24-43
 *   spamm_tree_tridiagonal    <- generators.gen_model_hamiltonian generators.py:76-88
 *   spamm_multiply_rows       <- (new) output block-row shard of spamm for multi-GPU
 *                                partitioning; the reference is single-process.
 *   spamm_tc2_update          <- the add/scale pair of tc2_step  purification.py:123-133
 *   spamm_tree_band_* , spamm_tree_pyramid_rebuild, spamm_tree_blocks_*_device,
 *   spamm_tree_diagonal_rows  <- (new) row bands of distributed matrices
 *   spamm_stream_wait / _signal, *_on  <- (new) stream-ordered hand-off with the
 *                                caller's CUDA streams (no device-wide synchronisation)
 */
#ifndef SPAMM_B200_H
#define SPAMM_B200_H

#include <stdint.h>

#if defined(__GNUC__)
#define SPAMM_API __attribute__((visibility("default")))
#else
#define SPAMM_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* status codes */
#define SPAMM_OK 0
#define SPAMM_ERR_VALUE 1     /* -> ValueError                       */
#define SPAMM_ERR_DIMENSION 2 /* -> DimensionMismatchError(ValueError) */
#define SPAMM_ERR_CUDA 3      /* -> RuntimeError (CUDA failure)       */
#define SPAMM_ERR_NOMEM 4     /* -> MemoryError                       */
#define SPAMM_ERR_INTERNAL 5  /* -> RuntimeError                      */

/* element storage types (quadtree.py:18 _SUPPORTED_DTYPES) */
#define SPAMM_DTYPE_F64 0
#define SPAMM_DTYPE_F32 1

/* spamm_multiply flags (SpammConfig, multiply.py:43-74) */
#define SPAMM_COLLECT_BOXES 0x1u  /* record a PrunedBox per tau-pruned call  */
#define SPAMM_COUNT_STATS 0x2u    /* maintain the ProductStats counters       */
#define SPAMM_TIER_TAU_DECAY 0x4u /* prune tier t against tau / 8**t          */
#define SPAMM_KEEP_TRIPLES 0x8u   /* keep the retained leaf (i,j,k) list      */
/* Traversal kernel selection (results are identical either way): shallow
 * trees (depth <= 6) default to the dense single-pass kernel; this flag
 * forces the tiered breadth-first kernel (testing / comparison). */
#define SPAMM_TIERED_TRAVERSAL 0x10u
/* Traversal only (the multi-GPU plan: which operand blocks a row shard's
 * retained triples touch): no leaf products and no C; *c is set to NULL.
 * Combine with SPAMM_KEEP_TRIPLES. */
#define SPAMM_TRAVERSE_ONLY 0x20u
/* Keep every tau-pruned call's (tier, i, j, k) and norm product, in reference
 * order (spamm_product_pruned): the multi-GPU budget merges the shards' lists
 * into the single-GPU order and sums them with the reference's pairwise sum. */
#define SPAMM_KEEP_PRUNED 0x40u
/* The B blocks (k, j) the retained triples read, as a bitmask over the block
 * grid (bit k * nb + j), formed on the device (spamm_product_need_blocks):
 * the multi-GPU plan without copying the retained triples off the device. */
#define SPAMM_NEED_BLOCKS 0x80u

typedef struct spamm_tree spamm_tree;
typedef struct spamm_product spamm_product;

typedef struct {
  int64_t logical_dim; /* n                                   */
  int64_t padded_dim;  /* N = leaf_size << depth              */
  int64_t block_grid;  /* N / leaf_size                       */
  int32_t leaf_size;
  int32_t depth;
  int32_t dtype;       /* SPAMM_DTYPE_*                        */
  int32_t device;      /* CUDA ordinal holding the tree        */
  double root_norm_sq; /* _norm_sq[0][0, 0]                    */
} spamm_tree_info;

typedef struct {
  int64_t leaf_matmuls;
  int64_t pruned_calls;
  int64_t pruned_volume;
  int64_t empty_skip_volume;
  int32_t max_depth_reached;
  int32_t reserved0;
  double omitted_budget;
  int64_t n_boxes;   /* number of PrunedBox records (if collected)   */
  int64_t n_triples; /* retained leaf triples (== leaf_matmuls)      */
  int64_t n_groups;  /* C blocks with at least one retained triple   */
  int64_t tier_candidates[32];
  int64_t tier_survivors[32];
  int64_t tier_pruned[32];
  /* device-event timings of the last call, milliseconds */
  float ms_cull;
  float ms_leaf;
  float ms_ctree;
  float ms_total;
  float ms_gemm;           /* the leaf-product kernel (K3) alone          */
  int32_t kernel_launches; /* kernels this call launched                  */
  /* traversal-kernel phase boundaries (device %globaltimer, us since start):
   * prefix end, barrier, grid tiers..., histogram, scan, scatter, sort */
  float traverse_phase_us[14];
} spamm_stats;

SPAMM_API const char *spamm_last_error(void);
SPAMM_API int spamm_device_count(int *count);
/* Library build identity, e.g. "spamm_b200 0.1 sm_100a". */
SPAMM_API const char *spamm_version(void);

/* -- stream ordering ------------------------------------------------------ */
/* The library works on its own CUDA stream per device.  Device data that a
 * caller's stream produces or consumes is handed over with events, never a
 * device-wide synchronisation:
 *   spamm_stream_wait(device, s)   the library's stream waits for the work
 *                                  queued on s so far (s produced the input);
 *   spamm_stream_signal(device, s) s waits for the work queued on the
 *                                  library's stream so far (s reads a result,
 *                                  or may now reuse / free an input).
 * spamm_stream_t has the layout of cudaStream_t (0 = the legacy stream). */
typedef struct CUstream_st *spamm_stream_t;
SPAMM_API int spamm_stream_wait(int32_t device, spamm_stream_t producer);
SPAMM_API int spamm_stream_signal(int32_t device, spamm_stream_t consumer);

/* -- trees ---------------------------------------------------------------- */
SPAMM_API int spamm_tree_from_host(const void *host, int64_t n, int64_t ld, int32_t leaf_size,
                         int32_t dtype, int32_t device, spamm_tree **out);
/* spamm_tree_from_host without waiting: the host->device copy and the norm
 * pyramid run on a separate copy-in stream (overlapping work already queued,
 * e.g. the previous matrix's multiplies) and the call returns at once.  Every
 * later call on the tree is ordered after the build; `host` must stay valid
 * (and should be pinned) until spamm_tree_wait(*out) or spamm_tree_free(*out)
 * returns (free waits for a pending build).  spamm_tree_info_get reports
 * root_norm_sq as NaN until spamm_tree_wait. */
SPAMM_API int spamm_tree_from_host_async(const void *host, int64_t n, int64_t ld, int32_t leaf_size,
                                         int32_t dtype, int32_t device, spamm_tree **out);
/* Block until an asynchronous build is complete (no-op for other trees). */
SPAMM_API int spamm_tree_wait(const spamm_tree *t);
/* `dev` is a device pointer on `device`; n x n with leading dimension ld. */
SPAMM_API int spamm_tree_from_device(const void *dev, int64_t n, int64_t ld, int32_t leaf_size,
                           int32_t dtype, int32_t device, spamm_tree **out);
/* spamm_tree_from_device ordered on the caller's stream: the copy starts
 * after the work queued on `stream` (which produced `dev`), and `stream`
 * waits for the copy, so the caller may reuse or free `dev` in stream order
 * (e.g. torch's caching allocator) -- the reference's from_dense boundary
 * (quadtree.py:218) for device-resident producers, without a device-wide sync. */
SPAMM_API int spamm_tree_from_device_on(const void *dev, int64_t n, int64_t ld, int32_t leaf_size,
                                        int32_t dtype, int32_t device, spamm_stream_t stream,
                                        spamm_tree **out);
/* Adopt an already padded N x N device array (copied), rebuild its pyramid. */
SPAMM_API int spamm_tree_from_padded_device(const void *dev_padded, int64_t n, int64_t padded_dim,
                                  int32_t leaf_size, int32_t dtype, int32_t device,
                                  spamm_tree **out);
SPAMM_API int spamm_tree_info_get(const spamm_tree *t, spamm_tree_info *info);
SPAMM_API int spamm_tree_to_host(const spamm_tree *t, void *host, int64_t ld);
SPAMM_API int spamm_tree_padded_to_host(const spamm_tree *t, void *host);
/* nsq: (4^(depth+1)-1)/3 doubles, occ: same count of bytes; level k
 * (2^k x 2^k row-major) starts at (4^k - 1)/3. */
SPAMM_API int spamm_tree_pyramid_to_host(const spamm_tree *t, double *nsq, uint8_t *occ);
/* Raw device pointers (borrowed) for collective plumbing (a band tree's
 * storage outside its rows is undefined; see spamm_multiply_rows). */
/* The squared-norm pyramid recomputed from the leaf data by K1 into scratch
 * storage and copied to host (same layout as spamm_tree_pyramid_to_host):
 * the fresh side of audit_norm_cache (quadtree.py:325-340). */
SPAMM_API int spamm_tree_recompute_norms(const spamm_tree *t, double *nsq_host);
SPAMM_API int spamm_tree_device_ptrs(const spamm_tree *t, void **padded, double **nsq, uint8_t **occ);
/* ||A - B||_F computed on the device (multiply_error, multiply.py:276). */
SPAMM_API int spamm_tree_diff_norm(const spamm_tree *a, const spamm_tree *b, double *out);

/* ------------------------------------------------------------ tree algebra
 * (the purification driver's element-wise operations; every result is a new
 * tree with its pyramid rebuilt, bit-identical to the reference's numpy) */
/* out = a + b; a block nonzero in only one operand is copied bit for bit
 * (quadtree.py:280-293).  Status 2 (DimensionMismatchError) if not conformable. */
SPAMM_API int spamm_tree_add(const spamm_tree *a, const spamm_tree *b, spamm_tree **out);
/* out = m * dtype(s) element-wise (quadtree.py:296-299). */
SPAMM_API int spamm_tree_scale(const spamm_tree *m, double s, spamm_tree **out);
/* Leaves with rn(sqrt(norm_sq)) < tau zeroed (quadtree.py:302-316).  When no
 * leaf drops, *dropped_any = 0 and *out = NULL: the input is the result. */
SPAMM_API int spamm_tree_filter_drop(const spamm_tree *m, double tau, spamm_tree **out,
                                     int32_t *dropped_any);
/* The listed leaves (ids: leaf indices i * block_grid + j) copied to host
 * memory as a contiguous [count][leaf][leaf] array in one transfer -- the
 * nonzero blocks of a tree (the reference's _blocks[_leaf_nonzero],
 * quadtree.py:120-151) without moving its empty blocks.  ids == NULL: every
 * nonzero leaf in ascending order (count must be their number), listed on the
 * device. */
SPAMM_API int spamm_tree_blocks_to_host(const spamm_tree *m, const int64_t *ids, int64_t count,
                                        void *host_out);
/* Asynchronous spamm_tree_blocks_to_host: the gather is ordered after every
 * earlier call on the tree's device, the copy runs on a separate copy-out
 * stream, and the call returns at once with a transfer handle.  host_out
 * should be pinned (page-locked) for the copy to overlap later calls; it must
 * stay valid until spamm_transfer_wait(*out) returns, which blocks until the
 * bytes are in host_out and releases the handle (exactly once per handle).
 * ids == NULL: every nonzero leaf in ascending order (count must be their
 * number), the list formed on the device. */
typedef struct spamm_transfer spamm_transfer;
SPAMM_API int spamm_tree_blocks_to_host_async(const spamm_tree *m, const int64_t *ids,
                                              int64_t count, void *host_out,
                                              spamm_transfer **out);
SPAMM_API int spamm_transfer_wait(spamm_transfer *t);
/* The logical diagonal (n elements of the tree's dtype) to host memory, for
 * trace = numpy add.reduce of it (quadtree.py:274-277). */
SPAMM_API int spamm_tree_diagonal(const spamm_tree *m, void *host_out);
SPAMM_API void spamm_tree_free(spamm_tree *t);

/* -- multiply --------------------------------------------------------------- */
SPAMM_API int spamm_multiply(const spamm_tree *a, const spamm_tree *b, double tau, uint32_t flags,
                   spamm_tree **c, spamm_stats *stats, spamm_product **product);
/* spamm_multiply ordered on the caller's stream: the library's stream waits
 * for the work queued on `stream` (e.g. kernels that wrote into the operands'
 * storage), and `stream` waits for the product (C is complete on return, as
 * for spamm_multiply, so the caller's later work on `stream` may read it). */
SPAMM_API int spamm_multiply_on(const spamm_tree *a, const spamm_tree *b, double tau, uint32_t flags,
                                spamm_stream_t stream, spamm_tree **c, spamm_stats *stats,
                                spamm_product **product);
/* Shard of spamm_multiply restricted to C leaf block rows [row_lo, row_hi):
 * only triples whose leaf rows intersect the range are traversed; pruned and
 * skipped calls are counted by the shard owning the call's first row, so the
 * per-shard integer stats sum exactly to the unsharded ones.  C is a band
 * tree: only the shard's rows are computed and stored; the others are zero
 * by definition (zero norms) and are zero-filled on the first whole-storage
 * read (to_host, padded_to_host, diff_norm, tree algebra) -- so a shard
 * never writes the other ranks' rows.  spamm_tree_device_ptrs hands out the
 * raw storage, where those rows are undefined until then. */
SPAMM_API int spamm_multiply_rows(const spamm_tree *a, const spamm_tree *b, double tau, uint32_t flags,
                        int64_t row_lo, int64_t row_hi, spamm_tree **c, spamm_stats *stats,
                        spamm_product **product);
/* boxes: 5 int64 per box (i_lo, j_lo, k_lo, edge, tier) in reference order. */
SPAMM_API int spamm_product_boxes(const spamm_product *p, int64_t *out, int64_t capacity);
/* triples: 3 int32 per retained leaf product (i, j, k), sorted by (i, j, k). */
SPAMM_API int spamm_product_triples(const spamm_product *p, int32_t *out, int64_t capacity);
/* pruned calls (SPAMM_KEEP_PRUNED): 4 int32 per call (tier, i, j, k) and its
 * norm product, reference order; count = spamm_product_pruned_count(p). */
SPAMM_API int spamm_product_pruned(const spamm_product *p, int32_t *tier_ijk, double *np_out,
                                   int64_t capacity);
SPAMM_API int64_t spamm_product_pruned_count(const spamm_product *p);
/* SPAMM_NEED_BLOCKS: (nb*nb + 31) / 32 words, bit k * nb + j set when a
 * retained triple (i, j, k) reads B block (k, j). */
SPAMM_API int spamm_product_need_blocks(const spamm_product *p, uint32_t *out, int64_t nwords);
SPAMM_API void spamm_product_free(spamm_product *p);

/* -- row bands of distributed matrices (multi-GPU; csrc/shard.cu) ------------
 * A distributed matrix is one tree per rank: the element storage of the
 * rank's C block rows [row_lo, row_hi) plus operand blocks fetched from other
 * ranks, and the WHOLE matrix's pyramid, whose leaf level the caller
 * all-gathers (NCCL) before spamm_tree_pyramid_rebuild.  Whole-storage reads
 * of a band tree fail (status 1): gather the bands first.  The reference is
 * single-process; these replace nothing in it. */
/* band rows (device pointer to logical row row_lo*leaf, leading dimension ld)
 * -> band tree whose pyramid is that of the band alone until rebuilt */
SPAMM_API int spamm_tree_band_from_device(const void *rows, int64_t n, int64_t ld, int32_t leaf,
                                          int32_t dtype, int64_t row_lo, int64_t row_hi,
                                          int32_t device, spamm_tree **out);
/* declare a tree (e.g. a spamm_multiply_rows product) the band [row_lo, row_hi) */
SPAMM_API int spamm_tree_band_set(spamm_tree *t, int64_t row_lo, int64_t row_hi);
/* the levels above the leaves and every nrm from the (gathered) leaf level */
SPAMM_API int spamm_tree_pyramid_rebuild(spamm_tree *t);
/* listed leaves (device ids i*block_grid+j) <-> contiguous device buffer */
SPAMM_API int spamm_tree_blocks_gather_device(const spamm_tree *t, const int64_t *ids, int64_t count,
                                              void *dev_out);
SPAMM_API int spamm_tree_blocks_scatter_device(spamm_tree *t, const int64_t *ids, int64_t count,
                                               const void *dev_in);
/* the logical diagonal of block rows [row_lo, row_hi) to host memory */
SPAMM_API int spamm_tree_diagonal_rows(const spamm_tree *t, int64_t row_lo, int64_t row_hi,
                                       void *host_out);
/* One TC2 sweep's element-wise work (purification.py:123-133 and the driver's
 * sweep displacement, :190-199) on block rows [row_lo, row_hi) in one pass:
 * *d_out = norms of D = add(X2, scale(X,-1)) (a norms-only tree: the
 * fixed-point gap); if make_y also *y_out = Y = add(scale(X,2), scale(X2,-1))
 * and *e_out = norms of add(Y, scale(X,-1)) -- with the reference's
 * pass-through of blocks nonzero in one operand only (quadtree.py:280-299),
 * bit-identical to those tree operations.  roots[0], roots[1]: the root
 * squared norms of D and E. */
SPAMM_API int spamm_tc2_update(const spamm_tree *x, const spamm_tree *x2, int32_t make_y,
                               int64_t row_lo, int64_t row_hi, spamm_tree **y_out,
                               spamm_tree **d_out, spamm_tree **e_out, double *roots);

/* -- box log ordering ------------------------------------------------------- */
/* order[r] = index of the box written r-th in a box log: boxes (5 int64 each,
 * i_lo, j_lo, k_lo, edge, tier) stably sorted on the device by the Morton key
 * of (i_lo, j_lo, k_lo), i-major bit interleave (multiply.py:306-315 with
 * ordering.py:24-34).  Coordinates must lie in [0, 2^21). */
SPAMM_API int spamm_boxes_morton_order(const int64_t *boxes, int64_t count, int32_t device,
                                       int64_t *order);

/* -- generators --------------------------------------------------------------- */
/* Tree of the n x n Toeplitz matrix element(i, j) = table[|i - j|], written
 * directly into device storage (gen_exponential: table[d] = exp(-alpha d);
 * gen_algebraic: table[d] = d^-p, table[0] = 0; generators.py:24-43). */
SPAMM_API int spamm_tree_toeplitz(const double *table, int64_t n, int32_t leaf_size, int32_t dtype,
                                  int32_t device, spamm_tree **out);
/* Tree of the symmetric tridiagonal matrix with diag[i] on (i, i) and off[i]
 * on (i, i+1) and (i+1, i) (gen_model_hamiltonian, generators.py:76-88). */
SPAMM_API int spamm_tree_tridiagonal(const double *diag, const double *off, int64_t n,
                                     int32_t leaf_size, int32_t dtype, int32_t device,
                                     spamm_tree **out);

#ifdef __cplusplus
}
#endif
#endif /* SPAMM_B200_H */
