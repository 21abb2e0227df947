// multiply.cu -- spamm_multiply: orchestration of K2 (cull), the leaf-triple
// grouping, K3 (leaf products + merge) and K1 on the product (C's tree).
//
// Reference: spamm() multiply.py:144-221 and _leaf_stage :224-257.
//
// The whole multiply is one fixed launch sequence on the device's stream:
// every size the host must pass is static (tree geometry, buffer capacities)
// and every data-dependent count stays on the device, so the host
// synchronises exactly once, at the end, to read the statistics.  If a
// capacity turned out too small (flagged by the kernels), the call is re-run
// with larger buffers; capacities persist per device, so this happens at
// most a few times per process.
#include <algorithm>
#include <cstdlib>
#include <memory>
#include <vector>

#include "leaf.cuh"
#include "traverse.cuh"

struct spamm_product {
  std::vector<int64_t> boxes;    // 5 per box: i_lo, j_lo, k_lo, edge, tier
  std::vector<int32_t> triples;  // 3 per retained leaf product: i, j, k
  std::vector<int32_t> pruned;   // 4 per tau-pruned call: tier, i, j, k (SPAMM_KEEP_PRUNED)
  std::vector<double> pruned_np; // its norm product rn(rn(sqrt a) rn(sqrt b))
  std::vector<uint32_t> need;    // SPAMM_NEED_BLOCKS: bit k * nb + j per B block read
};

namespace spamm {

int alloc_tree(DeviceContext *ctx, int64_t n, int32_t leaf, int32_t dtype, spamm_tree **out,
               cudaStream_t st = nullptr);
void free_tree_async(spamm_tree *t, cudaStream_t st);
// (declared in common.cuh)
int finish_tree(DeviceContext *ctx, spamm_tree *t);
void k1_timeline_enable(cudaStream_t st);
void k1_timeline_dump(unsigned long long k3_end, unsigned long long k3_start);

static int check_conformable(const spamm_tree *a, const spamm_tree *b) {
  // quadtree.py:209-215
  if (!a || !b) {
    set_error("null tree");
    return SPAMM_ERR_VALUE;
  }
  if (a->n != b->n || a->leaf != b->leaf) {
    set_error("trees not conformable: (%lld, leaf %d) vs (%lld, leaf %d)", (long long)a->n,
              a->leaf, (long long)b->n, b->leaf);
    return SPAMM_ERR_DIMENSION;
  }
  if (a->dtype != b->dtype) {
    set_error("dtype mismatch: %s vs %s", a->dtype ? "float32" : "float64",
              b->dtype ? "float32" : "float64");
    return SPAMM_ERR_DIMENSION;
  }
  if (a->device != b->device) {
    set_error("operands live on different devices (%d vs %d)", a->device, b->device);
    return SPAMM_ERR_VALUE;
  }
  return SPAMM_OK;
}


#define SPAMM_CUDA_BREAK(expr)                                                          \
  {                                                                                     \
    cudaError_t _e = (expr);                                                            \
    if (_e != cudaSuccess) {                                                            \
      set_error("CUDA error %s at %s:%d", cudaGetErrorString(_e), __FILE__, __LINE__); \
      rc = _e == cudaErrorMemoryAllocation ? SPAMM_ERR_NOMEM : SPAMM_ERR_CUDA;          \
      break;                                                                            \
    }                                                                                   \
  }

// The B blocks (k, j) read by the retained triples, as a bitmask (bit
// k * nb + j) -- from the k lists (one warp per group) ...
__global__ void need_blocks_ks_kernel(const uint32_t *__restrict__ group_ids,
                                      const uint32_t *__restrict__ group_starts,
                                      const uint32_t *__restrict__ ks, unsigned ng, uint64_t m,
                                      int64_t nb, uint32_t *__restrict__ out) {
  const int lane = threadIdx.x & 31;
  for (unsigned g = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; g < ng;
       g += (gridDim.x * blockDim.x) >> 5) {
    const int64_t j = group_ids[g] % nb;
    const uint64_t s0 = group_starts[g], s1 = g + 1 < ng ? group_starts[g + 1] : m;
    for (uint64_t s = s0 + lane; s < s1; s += 32) {
      const uint64_t bit = (uint64_t)ks[s] * nb + j;
      atomicOr(out + (bit >> 5), 1u << (bit & 31));
    }
  }
}
// ... or from the dense traversal's retained-triple bitmask (Morton order)
__global__ void need_blocks_am_kernel(const uint32_t *__restrict__ am, int64_t words, int64_t nb,
                                      uint32_t *__restrict__ out) {
  for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < words;
       w += (int64_t)gridDim.x * blockDim.x) {
    uint32_t bits = am[w];
    while (bits) {
      const uint32_t x = (uint32_t)(w * 32) + (uint32_t)(__ffs(bits) - 1);
      bits &= bits - 1;
      const uint64_t j = compact3(x >> 1), k = compact3(x);
      const uint64_t bit = k * nb + j;
      atomicOr(out + (bit >> 5), 1u << (bit & 31));
    }
  }
}

static int multiply_impl(const spamm_tree *a, const spamm_tree *b, double tau, uint32_t flags,
                         int64_t row_lo, int64_t row_hi, spamm_tree **c_out, spamm_stats *stats,
                         spamm_product **product) {
  SPAMM_TRY(check_conformable(a, b));
  if (!(tau >= 0.0) || tau == __builtin_inf()) {  // multiply.py:72-74
    set_error("tau must be finite and >= 0, got %g", tau);
    return SPAMM_ERR_VALUE;
  }
  if (row_lo < 0 || row_hi > a->nb || row_lo >= row_hi) {
    set_error("row range [%lld, %lld) invalid for block grid %lld", (long long)row_lo,
              (long long)row_hi, (long long)a->nb);
    return SPAMM_ERR_VALUE;
  }
  if (a->distributed && (row_lo < a->band_lo || row_hi > a->band_hi)) {
    set_error("rows [%lld, %lld) are not in A's band [%lld, %lld) (distributed operand)",
              (long long)row_lo, (long long)row_hi, (long long)a->band_lo, (long long)a->band_hi);
    return SPAMM_ERR_VALUE;
  }
  if (!a->padded || !b->padded) {
    set_error("norms-only tree as a multiply operand");
    return SPAMM_ERR_VALUE;
  }
  if (a->depth > 21 || a->nb * a->nb >= (int64_t(1) << 31)) {
    set_error("quadtree depth %d / block grid %lld exceeds the supported range", a->depth,
              (long long)a->nb);
    return SPAMM_ERR_VALUE;
  }
  DeviceContext *ctx;
  SPAMM_TRY(get_context(a->device, &ctx));
  std::lock_guard<std::mutex> lk(ctx->mu);
  NvtxRange nvtx_mul("spamm.multiply");
  cudaStream_t st = ctx->stream;
  SPAMM_TRY(tree_join(ctx, a));
  SPAMM_TRY(tree_join(ctx, b));
  const int depth = a->depth;
  const int64_t nb = a->nb;
  const int64_t G = nb * nb;

  if (ctx->cull_capacity == 0) ctx->cull_capacity = std::max<size_t>(1 << 16, 2 * G);
  if (ctx->pruned_capacity == 0) ctx->pruned_capacity = std::max<size_t>(1 << 16, 2 * G);
  TraverseCounters *hc = (TraverseCounters *)ctx->host_pinned;
  // traversal only (the multi-GPU plan: which operand blocks a shard needs):
  // no product, no leaf products, no C tree
  const bool trav_only = (flags & SPAMM_TRAVERSE_ONLY) != 0;
  spamm_tree *c = nullptr;
  if (!trav_only) SPAMM_TRY(alloc_tree(ctx, a->n, a->leaf, a->dtype, &c));
  int rc = SPAMM_OK;
  int launches = 0;
  for (int attempt = 0;; ++attempt) {
    launches = 0;
    const size_t cap = ctx->cull_capacity, pcap = ctx->pruned_capacity;
    const size_t gcap = std::min<size_t>(cap, (size_t)G);
    const size_t st_tier = traverse_status_entries(cap), st_grp = group_status_entries(nb);
    if ((rc = ensure_scratch(ctx->cull_codes[0], cap * sizeof(uint64_t), st))) break;
    if ((rc = ensure_scratch(ctx->cull_codes[1], cap * sizeof(uint64_t), st))) break;
    if ((rc = ensure_scratch(ctx->pruned_vals, pcap * sizeof(double), st))) break;
    if ((rc = ensure_scratch(ctx->pruned_codes, pcap * sizeof(uint64_t), st))) break;
    // look-back state must start (and is left by the kernel) all-zero
    if ((rc = ensure_scratch(ctx->tile_status,
                             sizeof(unsigned long long) * (2 * st_tier + st_grp), st, true)))
      break;
    // two counter sets, alternating between calls (see TraverseCounters)
    if ((rc = ensure_scratch(ctx->counters, 2 * sizeof(TraverseCounters), st, true))) break;
    const bool dense = dense_traversal_ok(depth) && !(flags & SPAMM_TIERED_TRAVERSAL);
    if (dense) {
      // two work sets (alternating with the counter sets), zero at rest
      const size_t ww = dense_work_words(depth);
      if (ctx->dn_set_words < ww) {
        if (ctx->dn_masks.ptr) SPAMM_CUDA_BREAK(cudaFreeAsync(ctx->dn_masks.ptr, st));
        ctx->dn_masks.ptr = nullptr;
        ctx->dn_masks.bytes = 0;
        if ((rc = ensure_scratch(ctx->dn_masks, 2 * sizeof(uint32_t) * ww, st, true))) break;
        ctx->dn_set_words = ww;
      }
      if ((rc = ensure_scratch(ctx->dn_retained, sizeof(uint32_t) * dense_retained_words(depth), st)))
        break;
      if ((rc = ensure_scratch(ctx->dn_np, sizeof(double) * dense_np_entries(depth), st))) break;
    }
    if ((rc = ensure_scratch(ctx->keys[0], 2 * sizeof(uint32_t) * G, st))) break;  // counts, offsets
    if ((rc = ensure_scratch(ctx->group_starts, 2 * sizeof(uint32_t) * gcap, st))) break;
    if ((rc = ensure_scratch(ctx->keys[1], sizeof(uint32_t) * cap, st))) break;  // ks
    if ((rc = ensure_scratch(ctx->pw_part, sizeof(double) * MAX_TIERS * 128, st))) break;
    TraverseCounters *tcs = (TraverseCounters *)ctx->counters.ptr;
    TraverseCounters *dtc = tcs + ctx->counter_parity;

    SPAMM_CUDA_BREAK(cudaEventRecord(ctx->fork, st));
    // ------------------------------------------- K2 traversal + grouping
    TraverseArgs ta{};
    ta.depth = depth;
    ta.nb = nb;
    for (int t = 0; t <= depth; ++t)
      ta.tau_tier[t] = (flags & SPAMM_TIER_TAU_DECAY) ? tau * ldexp(1.0, -3 * t) : tau;
    ta.nrm_a = a->nrm;
    ta.nrm_b = b->nrm;
    ta.occ_a = a->occ;
    ta.occ_b = b->occ;
    ta.codes[0] = (uint64_t *)ctx->cull_codes[0].ptr;
    ta.codes[1] = (uint64_t *)ctx->cull_codes[1].ptr;
    ta.capacity = cap;
    ta.pruned_vals = (double *)ctx->pruned_vals.ptr;
    ta.pruned_codes = (uint64_t *)ctx->pruned_codes.ptr;
    ta.pruned_capacity = pcap;
    unsigned long long *stb = (unsigned long long *)ctx->tile_status.ptr;
    ta.status[0] = stb;
    ta.status[1] = stb + st_tier;
    ta.status[2] = stb + 2 * st_tier;
    ta.tc = dtc;
    ta.row_lo = row_lo;
    ta.row_hi = row_hi;
    ta.counts = (uint32_t *)ctx->keys[0].ptr;
    ta.offsets = ta.counts + G;
    ta.group_ids = (uint32_t *)ctx->group_starts.ptr;
    ta.group_starts = ta.group_ids + gcap;
    ta.ks = (uint32_t *)ctx->keys[1].ptr;
    ta.tc_clear = tcs + (ctx->counter_parity ^ 1);
    ta.pw_part = (double *)ctx->pw_part.ptr;
    if (dense) {
      // the work sets alternate between dense calls only (a tiered call in
      // between leaves them untouched)
      ta.dn_masks = (uint32_t *)ctx->dn_masks.ptr + ctx->dense_parity * ctx->dn_set_words;
      ta.dn_masks_clear = (uint32_t *)ctx->dn_masks.ptr + (ctx->dense_parity ^ 1) * ctx->dn_set_words;
      ta.dn_work_words = ctx->dn_set_words;
      ta.dn_retained = (uint32_t *)ctx->dn_retained.ptr;
      ta.dn_np = (double *)ctx->dn_np.ptr;
      // Longest-first order for K3 is opt-in: measured slower on the c2
      // sweep (the (i, j) order keeps A's block rows hot in L2 across CTAs)
      static const bool lpt = getenv("SPAMM_LPT") != nullptr;
      if (lpt) {
        if ((rc = ensure_scratch(ctx->lpt_order, sizeof(uint32_t) * G, st))) break;
        ta.lpt_order = (uint32_t *)ctx->lpt_order.ptr;
      }
      // Bitmask groups (default on the dense path with the FP64 tensor-core
      // leaf kernel): the traversal publishes only the non-empty C blocks;
      // K3 reads each block's k list from the retained bitmask and starts on
      // tc->groups_ready while the traversal's record and budget CTAs finish
      // (they are off K3's critical path).  SPAMM_NO_BITMASK_GROUPS: the k
      // lists (ks / group_starts) and a start on the traversal's completion.
      static const bool no_bm = getenv("SPAMM_NO_BITMASK_GROUPS") != nullptr;
      ta.bitmask_groups = !no_bm && !lpt && depth <= 6 &&
                          (trav_only || (a->dtype == SPAMM_DTYPE_F64 && a->leaf >= 32));
    }
    static const bool tv_timeline = getenv("SPAMM_TRAVERSE_TIMELINE") != nullptr;
    static unsigned long long *tv_tl = nullptr;
    if (tv_timeline) {
      if (!tv_tl) SPAMM_CUDA_BREAK(cudaMalloc(&tv_tl, sizeof(unsigned long long) * 4 * 4096));
      SPAMM_CUDA_BREAK(cudaMemsetAsync(tv_tl, 0, sizeof(unsigned long long) * 4 * 4096, st));
      ta.timeline = tv_tl;
    }
    // device timing starts at the first kernel (host-side setup excluded)
    SPAMM_CUDA_BREAK(cudaEventRecord(ctx->ev[0], st));
    if (dense && c) {
      ta.c_nsq_leaf = c->nsq + level_offset(depth);
      ta.c_nrm_leaf = c->nrm + level_offset(depth);
      ta.c_occ_leaf = c->occ + level_offset(depth);
    }
    {
      NvtxRange r("spamm.K2.traverse");
      if ((rc = dense ? launch_traverse_dense(ta, ctx->num_sms, st)
                      : launch_traverse(ta, ctx->num_sms, st)))
        break;
    }
    ctx->counter_parity ^= 1;
    if (dense) ctx->dense_parity ^= 1;
    ctx->last_bitmask = ta.bitmask_groups != 0;
    ++launches;
    if (trav_only) {
      SPAMM_CUDA_BREAK(cudaEventRecord(ctx->ev[4], st));
      const SmallRead r{hc, dtc, sizeof(TraverseCounters)};
      if ((rc = read_small_sync(ctx, st, &r, 1))) break;
      ++launches;
      ctx->last_overlapped = ctx->last_k3_pdl = false;
      if (!hc->overflow) break;
      unsigned long long need = 0, pneed = 0;
      for (int t = 0; t <= depth; ++t) {
        need = std::max(need, hc->n_active[t]);
        pneed += hc->n_pruned[t];
      }
      ctx->cull_capacity = std::max<size_t>(2 * cap, need + need / 8);
      ctx->pruned_capacity = std::max<size_t>(need > cap ? pcap : 2 * pcap, pneed + pneed / 8);
      if (attempt > 40) {
        set_error("culling capacity did not converge");
        rc = SPAMM_ERR_INTERNAL;
        break;
      }
      continue;
    }
    // C's block storage is not zero-filled: a product is a lazy tree whose
    // empty blocks (no retained triple; the same as occupancy clear) are
    // zero by definition and never read by a multiply, a norm build or a
    // nonzero-block read -- they are filled only if the whole storage is ever
    // read (materialize()).  That removes N^2 bytes of writes per multiply
    // (134 MB at c2, 34 GB at c5).  A row-sharded product (band tree) is the
    // same case: blocks outside its rows are empty.  C's leaf-level norms are
    // zeroed on the side stream under the traversal (only blocks that receive
    // products are recomputed below).
    c->lazy_empty = true;
    // dense path: C's leaf-level norms are zeroed by the traversal kernel
    // itself, and K3 follows it as a programmatic dependent (no event or
    // stream wait may sit between them; the traversal's time is then the
    // multiply's remainder after K3 and the C tree)
    static const bool no_pdl = getenv("SPAMM_NO_K3_PDL") != nullptr;
    const bool k3_pdl = dense && !no_pdl;
    if (dense) {
      if (!k3_pdl) SPAMM_CUDA_BREAK(cudaEventRecord(ctx->ev[1], st));
    } else {
      SPAMM_CUDA_BREAK(cudaStreamWaitEvent(ctx->side, ctx->fork, 0));  // (fork: before the traversal)
      if ((rc = zero_async(c->nsq + level_offset(depth), sizeof(double) * G, ctx->side, 64))) break;
      if ((rc = zero_async(c->occ + level_offset(depth), G, ctx->side, 64))) break;
      if ((rc = zero_async(c->nrm + level_offset(depth), sizeof(double) * G, ctx->side, 64))) break;
      SPAMM_CUDA_BREAK(cudaEventRecord(ctx->join, ctx->side));
      SPAMM_CUDA_BREAK(cudaEventRecord(ctx->ev[1], st));
      SPAMM_CUDA_BREAK(cudaStreamWaitEvent(st, ctx->join, 0));
    }

    // ------------------------------------------------ K3 leaf products -> C
    if (!k3_pdl) SPAMM_CUDA_BREAK(cudaEventRecord(ctx->ev[2], st));
    LeafArgs la{};
    la.a = a->padded;
    la.b = b->padded;
    la.c = c->padded;
    la.N = a->N;
    la.nb = nb;
    la.leaf = a->leaf;
    la.depth = depth;
    la.n_codes = &dtc->n_active[depth];
    la.capacity = cap;
    la.ks = ta.ks;
    la.group_ids = ta.group_ids;
    la.group_starts = ta.group_starts;
    la.order = ta.lpt_order;
    la.tc = dtc;
    la.pdl = k3_pdl;
    la.am = ta.bitmask_groups ? ta.dn_retained : nullptr;
    static const bool want_timeline = getenv("SPAMM_GEMM_TIMELINE") != nullptr;
    if (want_timeline) {
      if ((rc = ensure_scratch(ctx->reduce_tmp, sizeof(unsigned long long) * 3 * 4096, st))) break;
      SPAMM_CUDA_BREAK(cudaMemsetAsync(ctx->reduce_tmp.ptr, 0, sizeof(unsigned long long) * 3 * 4096, st));
      la.timeline = (unsigned long long *)ctx->reduce_tmp.ptr;
    }
    // per-group completion counters let C's norm kernel overlap K3
    if ((rc = ensure_scratch(ctx->grp_done, sizeof(unsigned) * G, st, /*zeroed=*/true))) break;
    la.grp_done = (unsigned *)ctx->grp_done.ptr;
    // The C tree overlaps K3's tail: K1 is a programmatic dependent launch
    // whose CTAs (one per SM) start on the SMs K3's CTAs vacate and read each
    // C block once K3 has stored it (per-group counters), instead of waiting
    // for K3's grid to complete (c2: C tree 35-37 us after K3, was 45-49).
    // Only for small block grids: the overlapped K1 runs one 8-leaf CTA per
    // SM, which suits ~1k C blocks (c2) but not 10^4-10^6 (c3, c5), where the
    // regular K1 (32 leaves per CTA, two per SM) finishes in fewer waves.
    // (SPAMM_CTREE_OVERLAP_MAX: the largest block grid whose C tree runs
    // beside K3 -- the segmented-chain kernel's 2-warp CTAs next to K3's CTA,
    // leaves taken from a ticket in completion order)
    static const bool no_overlap = getenv("SPAMM_NO_CTREE_OVERLAP") != nullptr;
    static const int64_t overlap_max =
        getenv("SPAMM_CTREE_OVERLAP_MAX") ? atoll(getenv("SPAMM_CTREE_OVERLAP_MAX")) : 4096;
    if (no_overlap || G > overlap_max) la.grp_done = nullptr;
    static const bool k1tl = getenv("SPAMM_K1_TIMELINE") != nullptr;
    if (k1tl) k1_timeline_enable(st);
    bool overlapped = false;
    {
      NvtxRange r("spamm.K3.leaf_products");
      if ((rc = launch_leaf(la, a->dtype, ctx->num_sms, st, &launches, &overlapped))) break;
    }
    if (!overlapped) SPAMM_CUDA_BREAK(cudaEventRecord(ctx->ev[3], st));

    // ------------------------------------------- C's tree (multiply.py:220)
    {
      NvtxRange r("spamm.K1.c_tree");
      const int tile = a->leaf < 64 ? a->leaf : 64;
      const unsigned subs = (unsigned)((a->leaf / tile) * (a->leaf / tile));
      const bool bm = ta.bitmask_groups != 0;
      if ((rc = build_pyramid_async(ctx, c, st, &launches, ta.group_ids, &dtc->num_groups,
                                    (int64_t)gcap, overlapped ? la.grp_done : nullptr,
                                    leaf_signals_per_tile(a->leaf) * subs,
                                    bm ? nullptr : &dtc->overflow, &dtc->k1_t1,
                                    bm ? &dtc->groups_ready : nullptr,
                                    bm ? &dtc->trav_done : nullptr, nullptr, 0,
                                    bm && overlapped ? ta.dn_masks + dense_ne_offset(depth) : nullptr)))
        break;
    }
    ctx->last_overlapped = overlapped;
    ctx->last_k3_pdl = k3_pdl;
    SPAMM_CUDA_BREAK(cudaEventRecord(ctx->ev[4], st));
    {
      const SmallRead r[2] = {{hc, dtc, sizeof(TraverseCounters)},
                              {&c->root_norm_sq, c->nsq, sizeof(double)}};
      if ((rc = read_small_sync(ctx, st, r, 2))) break;
      launches += 2;  // (the two store-to-host kernels of the read)
    }
    if (tv_timeline && ta.timeline) {
      std::vector<unsigned long long> tl(4 * 4096);
      cudaMemcpy(tl.data(), tv_tl, sizeof(unsigned long long) * 4 * 4096, cudaMemcpyDeviceToHost);
      unsigned long long t0 = ~0ull;
      int n = 0;
      for (int q = 0; q < 4096; ++q)
        if (tl[4 * q]) { t0 = std::min(t0, tl[4 * q]); ++n; }
      fprintf(stderr, "[traverse timeline] ctas=%d", n);
      for (int half = 0; half < 2; ++half) {
        fprintf(stderr, half ? "\n   Q:" : "\n   P:");
        for (int f = 0; f < 4; ++f) {
          std::vector<double> v;
          for (int q = half ? n / 2 : 0; q < (half ? n : n / 2); ++q)
            if (tl[4 * q] && tl[4 * q + f]) v.push_back((tl[4 * q + f] - t0) * 1e-3);
          std::sort(v.begin(), v.end());
          if (!v.empty())
            fprintf(stderr, " | s%d %.1f/%.1f/%.1f", f, v[0], v[v.size() / 2], v.back());
        }
      }
      fprintf(stderr, "\n");
    }
    if (k1tl) k1_timeline_dump(hc->k3_t1, ~hc->k3_t0n);
    if (!hc->overflow) break;
    unsigned long long need = 0, pneed = 0;
    for (int t = 0; t <= depth; ++t) {
      need = std::max(need, hc->n_active[t]);
      pneed += hc->n_pruned[t];
    }
    ctx->cull_capacity = std::max<size_t>(2 * cap, need + need / 8);
    ctx->pruned_capacity = std::max<size_t>(need > cap ? pcap : 2 * pcap, pneed + pneed / 8);
    if (attempt > 40) {
      set_error("culling capacity did not converge");
      rc = SPAMM_ERR_INTERNAL;
      break;
    }
  }
  if (rc) {
    free_tree_async(c, st);
    return rc;
  }
  if (getenv("SPAMM_GEMM_TIMELINE") && !trav_only) {
    std::vector<unsigned long long> tl(3 * 4096);
    cudaMemcpy(tl.data(), ctx->reduce_tmp.ptr, sizeof(unsigned long long) * 3 * 4096,
               cudaMemcpyDeviceToHost);
    unsigned long long t0 = ~0ull, t1 = 0;
    std::vector<double> ends;
    double busy = 0;
    int n = 0, items = 0;
    for (int q = 0; q < 4096; ++q)
      if (tl[3 * q]) { t0 = std::min(t0, tl[3 * q]); t1 = std::max(t1, tl[3 * q + 1]); }
    for (int q = 0; q < 4096; ++q)
      if (tl[3 * q]) {
        ends.push_back((tl[3 * q + 1] - t0) * 1e-3);
        busy += (tl[3 * q + 1] - tl[3 * q]) * 1e-3;
        items += (int)(tl[3 * q + 2] & 0xffff);
        ++n;
      }
    if (getenv("SPAMM_GEMM_TIMELINE_RAW"))
      for (int q = 0; q < 4096; ++q)
        if (tl[3 * q])
          fprintf(stderr, "[gemm cta] %d start=%.1f end=%.1f items=%llu stages=%llu\n", q,
                  (tl[3 * q] - t0) * 1e-3, (tl[3 * q + 1] - t0) * 1e-3, tl[3 * q + 2] & 0xffff,
                  tl[3 * q + 2] >> 16);
    std::sort(ends.begin(), ends.end());
    if (n)
      fprintf(stderr, "[gemm timeline] ctas=%d items=%d span=%.1fus end min/med/p90/max=%.1f/%.1f/%.1f/%.1f busy_avg=%.1fus\n",
              n, items, (t1 - t0) * 1e-3, ends[0], ends[n / 2], ends[n * 9 / 10], ends[n - 1], busy / n);
  }
  const TraverseCounters &cc = *hc;

  // --------------------------------------------------------- stats (host)
  spamm_stats s{};
  const bool counting = (flags & SPAMM_COUNT_STATS) != 0;
  int64_t total_pruned = 0;
  for (int t = 0; t <= depth; ++t) {
    s.tier_candidates[t] = (int64_t)cc.n_cand[t];
    s.tier_survivors[t] = (int64_t)cc.n_active[t];
    s.tier_pruned[t] = (int64_t)cc.n_pruned[t];
    total_pruned += (int64_t)cc.n_pruned[t];
    if (cc.n_cand[t] > 0) s.max_depth_reached = t;  // multiply.py:181
    if (counting) {
      const int64_t edge = a->N >> t;
      const int64_t vol = edge * edge * edge;
      s.pruned_calls += (int64_t)(cc.n_skip[t] + cc.n_pruned[t]);
      s.empty_skip_volume += (int64_t)cc.n_skip[t] * vol;
      s.pruned_volume += (int64_t)cc.n_pruned[t] * vol;
    }
  }
  const int64_t m = (int64_t)cc.n_active[depth];
  if (counting) {
    s.leaf_matmuls = m;
    s.omitted_budget = cc.budget;
  }
  s.n_triples = m;
  s.n_groups = hc->num_groups;
  s.n_boxes = (flags & SPAMM_COLLECT_BOXES) ? total_pruned : 0;
  s.kernel_launches = launches;
  for (int q = 1; q < 14; ++q)
    s.traverse_phase_us[q] = cc.phase_ns[q] ? (float)((double)(cc.phase_ns[q] - cc.phase_ns[0]) * 1e-3) : 0.f;
  for (int q = 2; q < 8; ++q)  // (dense traversal: durations from kernel entry, CTA 0)
    if (cc.phase_ns[q] && cc.phase_ns[q] < 1000000000ull) s.traverse_phase_us[q] = (float)(cc.phase_ns[q] * 1e-3);
  // slot 0: kernel entry -> phase 0 (negative offset of the prologue)
  s.traverse_phase_us[0] = cc.phase_ns[15] ? (float)((double)(cc.phase_ns[0] - cc.phase_ns[15]) * 1e-3) : 0.f;
  cudaEventElapsedTime(&s.ms_total, ctx->ev[0], ctx->ev[4]);
  if (trav_only) s.ms_cull = s.ms_total;
  else if (!ctx->last_k3_pdl) cudaEventElapsedTime(&s.ms_cull, ctx->ev[0], ctx->ev[1]);
  static const bool tail_dbg = getenv("SPAMM_TAIL_DEBUG") != nullptr;
  if (tail_dbg && cc.k3_t1 && cc.k1_t1)
    fprintf(stderr, "[tail] k3 span %.1f us, C tree done %.1f us after K3\n",
            (double)(cc.k3_t1 - ~cc.k3_t0n) * 1e-3, ((double)cc.k1_t1 - (double)cc.k3_t1) * 1e-3);
  if (ctx->last_overlapped && cc.k3_t0n && cc.k3_t1) {
    // K3 and the C tree overlap (no event can sit between them): K3's span
    // from its own %globaltimer stamps; the C tree's tail after it from K1's
    // stamp when the pyramid is fused into K1, else the rest of the multiply
    s.ms_gemm = (float)((double)(cc.k3_t1 - ~cc.k3_t0n) * 1e-6);
    s.ms_leaf = s.ms_gemm;
    if (cc.k1_t1 > cc.k3_t1)
      s.ms_ctree = (float)((double)(cc.k1_t1 - cc.k3_t1) * 1e-6);
    else
      s.ms_ctree = std::max(0.f, s.ms_total - s.ms_cull - s.ms_gemm);
  } else if (trav_only) {
    // (no leaf products, no C tree)
  } else if (ctx->last_k3_pdl && cc.k3_t0n && cc.k3_t1) {
    s.ms_gemm = (float)((double)(cc.k3_t1 - ~cc.k3_t0n) * 1e-6);
    s.ms_leaf = s.ms_gemm;
    cudaEventElapsedTime(&s.ms_ctree, ctx->ev[3], ctx->ev[4]);
  } else {
    cudaEventElapsedTime(&s.ms_leaf, ctx->ev[1], ctx->ev[3]);
    cudaEventElapsedTime(&s.ms_gemm, ctx->ev[2], ctx->ev[3]);
    cudaEventElapsedTime(&s.ms_ctree, ctx->ev[3], ctx->ev[4]);
  }
  // K3 launched programmatically behind the traversal: no event between
  // them; the traversal's share is the multiply's remainder
  if (ctx->last_k3_pdl && !trav_only) s.ms_cull = std::max(0.f, s.ms_total - s.ms_gemm - s.ms_ctree);
  (void)cudaGetLastError();  // (timing queries must not leave an error for the next call)

  // ------------------------------------------------------- product records
  if (product) {
    auto p = std::make_unique<spamm_product>();
    cudaError_t e = cudaSuccess;
    const bool keep_pruned = (flags & SPAMM_KEEP_PRUNED) && (flags & SPAMM_COUNT_STATS);
    if ((flags & SPAMM_COLLECT_BOXES) && total_pruned) {
      std::vector<uint64_t> codes(total_pruned);
      e = cudaMemcpy(codes.data(), ctx->pruned_codes.ptr, total_pruned * sizeof(uint64_t),
                     cudaMemcpyDeviceToHost);
      p->boxes.reserve(5 * total_pruned);
      int64_t pos = 0;
      for (int t = 0; t <= depth && e == cudaSuccess; ++t) {
        const int64_t edge = a->N >> t;
        for (unsigned long long q = 0; q < cc.n_pruned[t]; ++q, ++pos) {
          uint32_t i, j, k;
          unpack_triple(codes[pos], i, j, k);
          p->boxes.insert(p->boxes.end(),
                          {int64_t(i) * edge, int64_t(j) * edge, int64_t(k) * edge, edge, t});
        }
      }
    }
    if (keep_pruned && total_pruned && e == cudaSuccess) {
      // the pruned calls' norm products in reference order (tier-major; the
      // multi-GPU budget merges the shards' lists into this order)
      std::vector<uint64_t> codes(total_pruned);
      p->pruned_np.resize(total_pruned);
      e = cudaMemcpy(codes.data(), ctx->pruned_codes.ptr, total_pruned * sizeof(uint64_t),
                     cudaMemcpyDeviceToHost);
      if (e == cudaSuccess)
        e = cudaMemcpy(p->pruned_np.data(), ctx->pruned_vals.ptr, total_pruned * sizeof(double),
                       cudaMemcpyDeviceToHost);
      p->pruned.reserve(4 * total_pruned);
      int64_t pos = 0;
      for (int t = 0; t <= depth && e == cudaSuccess; ++t)
        for (unsigned long long q = 0; q < cc.n_pruned[t]; ++q, ++pos) {
          uint32_t i, j, k;
          unpack_triple(codes[pos], i, j, k);
          p->pruned.insert(p->pruned.end(), {(int32_t)t, (int32_t)i, (int32_t)j, (int32_t)k});
        }
    }
    if ((flags & SPAMM_KEEP_TRIPLES) && m && e == cudaSuccess && ctx->last_bitmask) {
      // bitmask groups: each group's k list is its C block's retained bits
      const int64_t ng = s.n_groups;
      std::vector<uint32_t> ids(ng), am(dense_retained_words(depth));
      e = cudaMemcpy(ids.data(), ctx->group_starts.ptr, ng * sizeof(uint32_t),
                     cudaMemcpyDeviceToHost);
      if (e == cudaSuccess)
        e = cudaMemcpy(am.data(), ctx->dn_retained.ptr, am.size() * sizeof(uint32_t),
                       cudaMemcpyDeviceToHost);
      p->triples.reserve(3 * m);
      for (int64_t q = 0; q < ng && e == cudaSuccess; ++q) {
        const uint32_t i = (uint32_t)(ids[q] / nb), j = (uint32_t)(ids[q] % nb);
        const uint32_t base = (spread3(i) << 2) | (spread3(j) << 1);
        for (uint32_t k = 0; k < (uint32_t)nb; ++k) {
          const uint32_t x = base | spread3(k);
          if ((am[x >> 5] >> (x & 31)) & 1u)
            p->triples.insert(p->triples.end(), {(int32_t)i, (int32_t)j, (int32_t)k});
        }
      }
    } else if ((flags & SPAMM_KEEP_TRIPLES) && m && e == cudaSuccess) {
      const int64_t ng = s.n_groups;
      const size_t gcap = std::min<size_t>(ctx->cull_capacity, G);
      std::vector<uint32_t> ids(ng), starts(ng), ks(m);
      e = cudaMemcpy(ids.data(), ctx->group_starts.ptr, ng * sizeof(uint32_t),
                     cudaMemcpyDeviceToHost);
      if (e == cudaSuccess)
        e = cudaMemcpy(starts.data(), (uint32_t *)ctx->group_starts.ptr + gcap,
                       ng * sizeof(uint32_t), cudaMemcpyDeviceToHost);
      if (e == cudaSuccess)
        e = cudaMemcpy(ks.data(), ctx->keys[1].ptr, m * sizeof(uint32_t), cudaMemcpyDeviceToHost);
      p->triples.reserve(3 * m);
      for (int64_t q = 0; q < ng && e == cudaSuccess; ++q) {
        const int64_t end = q + 1 < ng ? starts[q + 1] : m;
        for (int64_t x = starts[q]; x < end; ++x)
          p->triples.insert(p->triples.end(), {(int32_t)(ids[q] / nb), (int32_t)(ids[q] % nb),
                                               (int32_t)ks[x]});
      }
    }
    if ((flags & SPAMM_NEED_BLOCKS) && e == cudaSuccess) {
      // the B blocks the retained triples read, formed on the device from the
      // traversal's lists (still in the context's scratch)
      const size_t nwords = (size_t)((G + 31) / 32);
      p->need.assign(nwords, 0u);
      int zr = ensure_scratch(ctx->reduce_tmp, nwords * sizeof(uint32_t), st);
      if (!zr && m) zr = zero_async(ctx->reduce_tmp.ptr, nwords * sizeof(uint32_t), st, ctx->num_sms);
      if (zr) {
        free_tree_async(c, st);
        return zr;
      }
      uint32_t *need = (uint32_t *)ctx->reduce_tmp.ptr;
      if (m && ctx->last_bitmask) {
        const int64_t words = (int64_t)dense_retained_words(depth);
        need_blocks_am_kernel<<<(unsigned)std::min<int64_t>((words + 255) / 256, 4 * ctx->num_sms),
                                256, 0, st>>>((const uint32_t *)ctx->dn_retained.ptr, words, nb, need);
      } else if (m) {
        const size_t gcap = std::min<size_t>(ctx->cull_capacity, G);
        need_blocks_ks_kernel<<<4 * ctx->num_sms, 256, 0, st>>>(
            (const uint32_t *)ctx->group_starts.ptr, (const uint32_t *)ctx->group_starts.ptr + gcap,
            (const uint32_t *)ctx->keys[1].ptr, (unsigned)s.n_groups, (uint64_t)m, nb, need);
      }
      e = cudaGetLastError();
      if (m && e == cudaSuccess)
        e = cudaMemcpyAsync(p->need.data(), need, nwords * sizeof(uint32_t), cudaMemcpyDeviceToHost, st);
      if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    }
    if (e != cudaSuccess) {
      free_tree_async(c, st);
      set_error("copy of product records: %s", cudaGetErrorString(e));
      return SPAMM_ERR_CUDA;
    }
    *product = p.release();
  }
  if (stats) *stats = s;
  if (c && a->distributed) {  // a row band of a distributed product
    c->distributed = true;
    c->band_lo = row_lo;
    c->band_hi = row_hi;
  }
  *c_out = c;
  return SPAMM_OK;
}

}  // namespace spamm

using namespace spamm;

extern "C" {

int spamm_multiply(const spamm_tree *a, const spamm_tree *b, double tau, uint32_t flags,
                   spamm_tree **c, spamm_stats *stats, spamm_product **product) {
  if (product) *product = nullptr;
  const int64_t nb = a ? a->nb : 0;
  return multiply_impl(a, b, tau, flags, 0, nb, c, stats, product);
}

int spamm_multiply_on(const spamm_tree *a, const spamm_tree *b, double tau, uint32_t flags,
                      spamm_stream_t stream, spamm_tree **c, spamm_stats *stats,
                      spamm_product **product) {
  if (product) *product = nullptr;
  if (!a || !b) {
    set_error("null operand");
    return SPAMM_ERR_VALUE;
  }
  SPAMM_TRY(spamm_stream_wait(a->device, stream));
  SPAMM_TRY(multiply_impl(a, b, tau, flags, 0, a->nb, c, stats, product));
  return spamm_stream_signal(a->device, stream);
}

int spamm_multiply_rows(const spamm_tree *a, const spamm_tree *b, double tau, uint32_t flags,
                        int64_t row_lo, int64_t row_hi, spamm_tree **c, spamm_stats *stats,
                        spamm_product **product) {
  if (product) *product = nullptr;
  return multiply_impl(a, b, tau, flags, row_lo, row_hi, c, stats, product);
}

int spamm_product_boxes(const spamm_product *p, int64_t *out, int64_t capacity) {
  if (!p) { set_error("null product"); return SPAMM_ERR_VALUE; }
  const int64_t n = (int64_t)p->boxes.size() / 5;
  if (capacity < n) { set_error("box buffer too small"); return SPAMM_ERR_VALUE; }
  std::copy(p->boxes.begin(), p->boxes.end(), out);
  return SPAMM_OK;
}

int spamm_product_triples(const spamm_product *p, int32_t *out, int64_t capacity) {
  if (!p) { set_error("null product"); return SPAMM_ERR_VALUE; }
  const int64_t n = (int64_t)p->triples.size() / 3;
  if (capacity < n) { set_error("triple buffer too small"); return SPAMM_ERR_VALUE; }
  std::copy(p->triples.begin(), p->triples.end(), out);
  return SPAMM_OK;
}

int spamm_product_pruned(const spamm_product *p, int32_t *tier_ijk, double *np_out, int64_t capacity) {
  if (!p) { set_error("null product"); return SPAMM_ERR_VALUE; }
  const int64_t n = (int64_t)p->pruned_np.size();
  if (capacity < n) { set_error("pruned buffer too small"); return SPAMM_ERR_VALUE; }
  std::copy(p->pruned.begin(), p->pruned.end(), tier_ijk);
  std::copy(p->pruned_np.begin(), p->pruned_np.end(), np_out);
  return SPAMM_OK;
}

int64_t spamm_product_pruned_count(const spamm_product *p) {
  return p ? (int64_t)p->pruned_np.size() : 0;
}

int spamm_product_need_blocks(const spamm_product *p, uint32_t *out, int64_t nwords) {
  if (!p) { set_error("null product"); return SPAMM_ERR_VALUE; }
  if (p->need.empty()) { set_error("product kept no needed-block set (SPAMM_NEED_BLOCKS)"); return SPAMM_ERR_VALUE; }
  if (nwords < (int64_t)p->need.size()) { set_error("need buffer too small"); return SPAMM_ERR_VALUE; }
  std::copy(p->need.begin(), p->need.end(), out);
  return SPAMM_OK;
}

void spamm_product_free(spamm_product *p) { delete p; }

}  // extern "C"
