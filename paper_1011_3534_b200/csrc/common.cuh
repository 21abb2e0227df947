// common.cuh -- shared device/host helpers for the SpAMM B200 library.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdarg>
#include <cstdio>
#include <mutex>
#include <string>
#include <vector>

#include "spamm_b200.h"
#include <nvtx3/nvToolsExt.h>

namespace spamm {

// ---------------------------------------------------------------- errors
void set_error(const char *fmt, ...);

struct Status {
  int code = SPAMM_OK;
};

#define SPAMM_CUDA_TRY(expr)                                                              \
  do {                                                                                    \
    cudaError_t _e = (expr);                                                              \
    if (_e != cudaSuccess) {                                                              \
      ::spamm::set_error("CUDA error %s (%s) at %s:%d", cudaGetErrorName(_e),             \
                         cudaGetErrorString(_e), __FILE__, __LINE__);                     \
      return _e == cudaErrorMemoryAllocation ? SPAMM_ERR_NOMEM : SPAMM_ERR_CUDA;          \
    }                                                                                     \
  } while (0)

#define SPAMM_TRY(expr)              \
  do {                               \
    int _s = (expr);                 \
    if (_s != SPAMM_OK) return _s;   \
  } while (0)

// ------------------------------------------------------------ pyramid layout
// Level k (2^k x 2^k, row-major) of the norm / occupancy pyramid starts at
// (4^k - 1) / 3 in one concatenated array (the reference keeps a Python list
// of per-level arrays, quadtree.py:131-138).
__host__ __device__ constexpr int64_t level_offset(int k) {
  return ((int64_t(1) << (2 * k)) - 1) / 3;
}
inline int64_t pyramid_size(int depth) { return level_offset(depth + 1); }

inline int depth_for(int64_t n, int32_t leaf) {
  int d = 0;
  while ((int64_t(leaf) << d) < n) ++d;
  return d;
}

// ------------------------------------------------------- triple packing
// A product-space triple (i, j, k) at any tier is kept packed as
// i << 42 | j << 21 | k (21 bits each, depth <= 21).  Its children are
// (2i+di, 2j+dj, 2k+dk) for (di,dj,dk) = 000..111 -- the reference's
// expansion order (multiply.py:35-37) -- and a tier's candidate list is
// generated parent by parent, so every list stays in the reference's order.
constexpr uint64_t TRIPLE_MASK = (uint64_t(1) << 21) - 1;
__host__ __device__ inline uint64_t pack_triple(uint64_t i, uint64_t j, uint64_t k) {
  return (i << 42) | (j << 21) | k;
}
__host__ __device__ inline void unpack_triple(uint64_t p, uint32_t &i, uint32_t &j, uint32_t &k) {
  i = (uint32_t)(p >> 42);
  j = (uint32_t)((p >> 21) & TRIPLE_MASK);
  k = (uint32_t)(p & TRIPLE_MASK);
}
// child q = di<<2 | dj<<1 | dk of packed parent p
__host__ __device__ inline uint64_t child_triple(uint64_t p, unsigned q) {
  return (p << 1) + ((uint64_t)(q >> 2) << 42) + ((uint64_t)((q >> 1) & 1) << 21) + (q & 1);
}

// ------------------------------------------------------------ device context
// One per CUDA device: a non-blocking stream, a lock serialising calls on
// that device, and grow-only scratch reused across multiplies.
struct Scratch {
  void *ptr = nullptr;
  size_t bytes = 0;
};

struct DeviceContext {
  int device = -1;
  int num_sms = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t side = nullptr;       // overlaps memory-bound fills with compute
  cudaStream_t copy_out = nullptr;   // device->host result transfers (overlap the next call)
  cudaStream_t copy_in = nullptr;    // asynchronous builds: host->device copy + K1 (overlap compute)
  cudaEvent_t fork = nullptr, join = nullptr;
  cudaEvent_t handoff = nullptr;  // stream hand-off with the caller's streams
  cudaEvent_t ev[8] = {};
  std::mutex mu;
  Scratch cull_codes[2];  // ping-pong survivor lists (packed i,j,k)
  Scratch pruned_codes;   // pruned codes, all tiers (u64)
  Scratch pruned_vals;    // pruned norm products, all tiers (f64)
  Scratch tile_status;    // decoupled look-back state
  Scratch counters;       // two alternating TraverseCounters sets
  Scratch keys[2];        // bucket counts/offsets, grouped inner indices
  Scratch group_starts;   // non-empty C blocks and their first triple
  Scratch reduce_tmp;     // misc reduction scratch
  Scratch pyr_tickets;    // pyramid hand-off counters (self-resetting, zero at rest)
  Scratch k1_ticket;      // K1's last-CTA ticket for the fused pyramid (zero at rest)
  Scratch k1_pcnt;        // K1 beside K3: finished children per leaf parent (zero at rest)
  Scratch pyr_tickets_in, k1_ticket_in;  // the same, for builds on copy_in
  Scratch dn_masks;       // dense traversal: two work sets (zero at rest)
  size_t dn_set_words = 0;  // words per dense work set
  int dense_parity = 0;     // which dense work set the next dense call uses
  Scratch dn_retained;    // dense traversal: retained leaf bitmask
  Scratch dn_np;          // dense traversal: leaf-tier pruned products
  Scratch dn_status;      // dense traversal: look-back state (zero at rest)
  int counter_parity = 0; // which traversal counter set the next call uses
  bool last_overlapped = false;  // the last product's C tree overlapped K3
  bool last_k3_pdl = false;      // the last product's K3 followed the traversal programmatically
  bool last_bitmask = false;     // the last traversal published bitmask groups (no ks lists)
  Scratch grp_done;       // per-group finished-tile counters (zero at rest)
  Scratch lpt_order;      // groups by decreasing size (K3's work order)
  Scratch pw_part;        // budget: per-tier partial sums of the split recursion
  size_t cull_capacity = 0;   // survivor capacity per ping-pong buffer (items)
  size_t pruned_capacity = 0; // pruned capacity (items, all tiers)
  void *host_pinned = nullptr;  // small pinned staging for counters
  Scratch host_stage;           // pinned staging of read_small_sync (grow-only)
  std::vector<Scratch> xfer_free;  // idle device staging buffers of async block transfers
};

int get_context(int device, DeviceContext **ctx);

// NVTX range over a host-side launch sequence (K1 builds, K2 traversal, K3
// leaf products, C's tree, the multiply): kernels a profiler traces nest
// under the range that launched them; no cost without a profiler attached.
struct NvtxRange {
  explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange &) = delete;
  NvtxRange &operator=(const NvtxRange &) = delete;
};
int ensure_scratch(Scratch &s, size_t bytes, cudaStream_t stream, bool zeroed = false);
// Zero `bytes` at `p` with a kernel (16-byte stores; any alignment).  Used on
// the multiply path instead of cudaMemsetAsync, which is carried out by a
// copy engine and so queues behind device->host copies in flight (an async
// product read-back would otherwise stall the next multiply).
int zero_async(void *p, size_t bytes, cudaStream_t st, int ctas);
// cudaMallocAsync, plus (debug: SPAMM_POISON=<byte>) the new memory filled with
// that byte, so a read of memory nothing initialised shows up as NaN / set
// occupancy / huge counts instead of the zeros a fresh allocation often holds.
cudaError_t dev_alloc(void **p, size_t bytes, cudaStream_t st);

// Small device->host reads (statistics, root norms, pyramids) without the
// copy engines: a kernel stores the bytes into pinned host memory, then the
// stream is synchronised and the bytes are copied to their destinations.  A
// cudaMemcpy would queue behind bulk device->host copies in flight on the
// copy-out stream (same engine); these stores interleave with them on PCIe.
struct SmallRead {
  void *host;
  const void *dev;
  size_t bytes;
};
int read_small_sync(DeviceContext *ctx, cudaStream_t st, const SmallRead *r, int n);

}  // namespace spamm

struct spamm_tree {
  int64_t n = 0;        // logical_dim
  int64_t N = 0;        // padded_dim
  int64_t nb = 0;       // block_grid
  int32_t leaf = 0;
  int32_t depth = 0;
  int32_t dtype = SPAMM_DTYPE_F64;
  int32_t device = 0;
  void *padded = nullptr;   // N x N row-major, element type per dtype
  double *nsq = nullptr;    // concatenated squared-norm pyramid
  uint8_t *occ = nullptr;   // concatenated occupancy pyramid
  double *nrm = nullptr;    // rn(sqrt(nsq)): the factors of the pruning test
  double root_norm_sq = 0.0;
  // Lazy empty blocks (every product): only the leaf blocks whose occupancy
  // is set were written; the others are zero by definition (their norms are
  // zero, and no multiply, norm or block read touches them) and are zero-
  // filled on the first whole-storage access (materialize()).  A row-sharded
  // product (band tree) is the same thing: blocks outside its rows are empty.
  bool lazy_empty = false;
  // Asynchronous build (spamm_tree_from_host_async): copy + K1 run on the
  // context's copy_in stream; every later use orders itself after `ready`
  // (tree_join), and root_norm_sq is fetched on the first spamm_tree_wait.
  cudaEvent_t ready = nullptr;
  bool root_pending = false;
  // Row band of a distributed matrix (multi-GPU layout, csrc/shard.cu): the
  // element storage holds block rows [band_lo, band_hi) plus any blocks
  // fetched from other ranks (halo), while the pyramid is the whole matrix's
  // (its leaf level all-gathered).  Whole-storage reads are refused.
  bool distributed = false;
  int64_t band_lo = 0, band_hi = 0;
  int64_t elem_size() const { return dtype == SPAMM_DTYPE_F64 ? 8 : 4; }
};

namespace spamm {
struct DeviceContext;
// zero-fill a lazy tree's empty blocks (stream-ordered on ctx->stream)
int materialize(DeviceContext *ctx, const spamm_tree *t);
// Leaf norms (K1) and the pyramid of `t`, stream-ordered (tree.cu).
int build_pyramid_async(DeviceContext *ctx, spamm_tree *t, cudaStream_t st, int *launches,
                        const uint32_t *list, const unsigned *list_count, int64_t list_cap,
                        unsigned *grp_done, unsigned grp_target, const int *overflow,
                        unsigned long long *t_end, const unsigned *ready = nullptr,
                        const unsigned *trav_done = nullptr, const void *fuse_src = nullptr,
                        int64_t fuse_ld = 0, const uint32_t *ne = nullptr);
// upper pyramid levels + interior nrm from the leaf level (tree.cu)
int pyramid_upper_async(DeviceContext *ctx, spamm_tree *t, cudaStream_t st, int *launches = nullptr);
// order ctx->stream after an asynchronous build of t (no-op otherwise)
int tree_join(DeviceContext *ctx, const spamm_tree *t);
}  // namespace spamm
