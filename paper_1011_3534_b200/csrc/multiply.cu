// multiply.cu -- spamm_multiply: orchestration of K2 (cull), the leaf-triple
// grouping, K3 (leaf products + merge) and K1 on the product (C's tree).
//
// Reference: spamm() multiply.py:144-221 and _leaf_stage :224-257.
#include <cub/cub.cuh>

#include <algorithm>
#include <memory>
#include <vector>

#include "cull.cuh"
#include "leaf.cuh"

struct spamm_product {
  std::vector<int64_t> boxes;    // 5 per box: i_lo, j_lo, k_lo, edge, tier
  std::vector<int32_t> triples;  // 3 per retained leaf product: i, j, k
};

namespace spamm {

int alloc_tree(DeviceContext *ctx, int64_t n, int32_t leaf, int32_t dtype, spamm_tree **out);
void free_tree_async(spamm_tree *t, cudaStream_t st);
int build_pyramid_async(spamm_tree *t, cudaStream_t st);
int finish_tree(DeviceContext *ctx, spamm_tree *t);

struct LeafCounters {
  int num_groups;
  int pad_;
  unsigned long long ticket;
};

// Leaf triple (Morton code at the leaf tier) -> grouping key (i*nb + j) << depth | k.
// Sorting by this key reproduces _leaf_stage's lexsort by (i, j, k) (multiply.py:231-233).
__global__ void codes_to_keys_kernel(const uint64_t *__restrict__ codes, int64_t m, int depth,
                                     int64_t nb, uint64_t *__restrict__ keys) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < m;
       p += (int64_t)gridDim.x * blockDim.x) {
    uint32_t i, j, k;
    morton_decode(codes[p], i, j, k);
    keys[p] = ((uint64_t(i) * nb + j) << depth) | k;
  }
}

__global__ void group_heads_kernel(const uint64_t *__restrict__ keys, int64_t m, int depth,
                                   uint8_t *__restrict__ flags) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < m;
       p += (int64_t)gridDim.x * blockDim.x)
    flags[p] = p == 0 || (keys[p] >> depth) != (keys[p - 1] >> depth);
}

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
  if (a->depth >= MAX_TIERS - 1 || a->depth > 21) {
    set_error("quadtree depth %d exceeds the supported 21 tiers", a->depth);
    return SPAMM_ERR_VALUE;
  }
  DeviceContext *ctx;
  SPAMM_TRY(get_context(a->device, &ctx));
  std::lock_guard<std::mutex> lk(ctx->mu);
  cudaStream_t st = ctx->stream;
  const int depth = a->depth;
  const int64_t nb = a->nb;

  SPAMM_CUDA_TRY(cudaEventRecord(ctx->ev[0], st));
  // ---------------------------------------------------------------- K2 cull
  if (ctx->cull_capacity == 0) ctx->cull_capacity = std::max<size_t>(1 << 16, 2 * nb * nb);
  if (ctx->pruned_capacity == 0) ctx->pruned_capacity = std::max<size_t>(1 << 16, 2 * nb * nb);
  CullCounters *hc = (CullCounters *)ctx->host_pinned;
  for (int attempt = 0;; ++attempt) {
    const size_t cap = ctx->cull_capacity, pcap = ctx->pruned_capacity;
    SPAMM_TRY(ensure_scratch(ctx->cull_codes[0], cap * sizeof(uint64_t), st));
    SPAMM_TRY(ensure_scratch(ctx->cull_codes[1], cap * sizeof(uint64_t), st));
    SPAMM_TRY(ensure_scratch(ctx->pruned_vals, pcap * sizeof(double), st));
    SPAMM_TRY(ensure_scratch(ctx->pruned_codes, pcap * sizeof(uint64_t), st));
    SPAMM_TRY(ensure_scratch(ctx->tile_status, tile_status_bytes(cap), st));
    SPAMM_TRY(ensure_scratch(ctx->counters, sizeof(CullCounters) + sizeof(LeafCounters), st));
    CullPlan plan{};
    plan.depth = depth;
    for (int t = 0; t <= depth; ++t)
      plan.tau_tier[t] = (flags & SPAMM_TIER_TAU_DECAY) ? tau * ldexp(1.0, -3 * t) : tau;
    plan.nsq_a = a->nsq;
    plan.nsq_b = b->nsq;
    plan.occ_a = a->occ;
    plan.occ_b = b->occ;
    plan.codes[0] = (uint64_t *)ctx->cull_codes[0].ptr;
    plan.codes[1] = (uint64_t *)ctx->cull_codes[1].ptr;
    plan.capacity = cap;
    plan.pruned_vals = (double *)ctx->pruned_vals.ptr;
    plan.pruned_codes = (uint64_t *)ctx->pruned_codes.ptr;
    plan.pruned_capacity = pcap;
    plan.tile_status = (unsigned long long *)ctx->tile_status.ptr;
    plan.counters = (CullCounters *)ctx->counters.ptr;
    plan.row_lo = row_lo;
    plan.row_hi = row_hi;
    plan.max_ctas = ctx->num_sms * 4;
    SPAMM_TRY(launch_cull(plan, st));
    SPAMM_CUDA_TRY(cudaMemcpyAsync(hc, ctx->counters.ptr, sizeof(CullCounters),
                                   cudaMemcpyDeviceToHost, st));
    SPAMM_CUDA_TRY(cudaStreamSynchronize(st));
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
      return SPAMM_ERR_INTERNAL;
    }
  }
  SPAMM_CUDA_TRY(cudaEventRecord(ctx->ev[1], st));

  // --------------------------------------------------------- stats (host)
  spamm_stats s{};
  const bool counting = (flags & SPAMM_COUNT_STATS) != 0;
  for (int t = 0; t <= depth; ++t) {
    s.tier_candidates[t] = (int64_t)hc->n_cand[t];
    s.tier_survivors[t] = (int64_t)hc->n_active[t];
    s.tier_pruned[t] = (int64_t)hc->n_pruned[t];
    if (hc->n_cand[t] > 0) s.max_depth_reached = t;  // multiply.py:181
    if (counting) {
      const int64_t edge = a->N >> t;
      const int64_t vol = edge * edge * edge;
      s.pruned_calls += (int64_t)(hc->n_skip[t] + hc->n_pruned[t]);
      s.empty_skip_volume += (int64_t)hc->n_skip[t] * vol;
      s.pruned_volume += (int64_t)hc->n_pruned[t] * vol;
    }
  }
  const int64_t m = (int64_t)hc->n_active[depth];
  if (counting) {
    s.leaf_matmuls = m;
    s.omitted_budget = hc->budget;
  }
  s.n_triples = m;
  int64_t total_pruned = 0;
  for (int t = 0; t <= depth; ++t) total_pruned += (int64_t)hc->n_pruned[t];
  s.n_boxes = (flags & SPAMM_COLLECT_BOXES) ? total_pruned : 0;

  // ----------------------------------------------------- C tree + leaf stage
  spamm_tree *c = nullptr;
  SPAMM_TRY(alloc_tree(ctx, a->n, a->leaf, a->dtype, &c));
  int rc = SPAMM_OK;
  std::vector<uint64_t> host_keys;
  do {
    cudaError_t e = cudaMemsetAsync(c->padded, 0, (size_t)(c->N * c->N * c->elem_size()), st);
    if (e != cudaSuccess) { set_error("memset C: %s", cudaGetErrorString(e)); rc = SPAMM_ERR_CUDA; break; }
    if (m > 0) {
      uint64_t *codes = (uint64_t *)ctx->cull_codes[depth & 1].ptr;
      if ((rc = ensure_scratch(ctx->keys[0], m * sizeof(uint64_t), st))) break;
      if ((rc = ensure_scratch(ctx->keys[1], m * sizeof(uint64_t), st))) break;
      if ((rc = ensure_scratch(ctx->flags, m, st))) break;
      if ((rc = ensure_scratch(ctx->group_starts, m * sizeof(int), st))) break;
      uint64_t *k0 = (uint64_t *)ctx->keys[0].ptr, *k1 = (uint64_t *)ctx->keys[1].ptr;
      const int grid = (int)std::min<int64_t>((m + 255) / 256, ctx->num_sms * 8);
      codes_to_keys_kernel<<<grid, 256, 0, st>>>(codes, m, depth, nb, k0);
      size_t sort_bytes = 0, sel_bytes = 0;
      const int end_bit = std::max(1, 3 * depth);
      cub::DeviceRadixSort::SortKeys(nullptr, sort_bytes, k0, k1, m, 0, end_bit, st);
      LeafCounters *lc = (LeafCounters *)((char *)ctx->counters.ptr + sizeof(CullCounters));
      cub::CountingInputIterator<int> ids(0);
      cub::DeviceSelect::Flagged(nullptr, sel_bytes, ids, (uint8_t *)ctx->flags.ptr,
                                 (int *)ctx->group_starts.ptr, &lc->num_groups, m, st);
      if ((rc = ensure_scratch(ctx->cub_temp, std::max(sort_bytes, sel_bytes), st))) break;
      sort_bytes = sel_bytes = ctx->cub_temp.bytes;
      e = cub::DeviceRadixSort::SortKeys(ctx->cub_temp.ptr, sort_bytes, k0, k1, m, 0, end_bit, st);
      if (e != cudaSuccess) { set_error("sort: %s", cudaGetErrorString(e)); rc = SPAMM_ERR_CUDA; break; }
      group_heads_kernel<<<grid, 256, 0, st>>>(k1, m, depth, (uint8_t *)ctx->flags.ptr);
      e = cub::DeviceSelect::Flagged(ctx->cub_temp.ptr, sel_bytes, ids, (uint8_t *)ctx->flags.ptr,
                                     (int *)ctx->group_starts.ptr, &lc->num_groups, m, st);
      if (e != cudaSuccess) { set_error("select: %s", cudaGetErrorString(e)); rc = SPAMM_ERR_CUDA; break; }
      e = cudaMemsetAsync(&lc->ticket, 0, sizeof(unsigned long long), st);
      if (e != cudaSuccess) { set_error("memset: %s", cudaGetErrorString(e)); rc = SPAMM_ERR_CUDA; break; }
      LeafArgs la{};
      la.a = a->padded;
      la.b = b->padded;
      la.c = c->padded;
      la.N = a->N;
      la.nb = nb;
      la.m = m;
      la.leaf = a->leaf;
      la.depth = depth;
      la.keys = k1;
      la.group_starts = (const int *)ctx->group_starts.ptr;
      la.num_groups = &lc->num_groups;
      la.ticket = &lc->ticket;
      if ((rc = launch_leaf(la, a->dtype, ctx->num_sms, st))) break;
      if (flags & SPAMM_KEEP_TRIPLES) {
        host_keys.resize(m);
        e = cudaMemcpyAsync(host_keys.data(), k1, m * sizeof(uint64_t), cudaMemcpyDeviceToHost, st);
        if (e != cudaSuccess) { set_error("copy: %s", cudaGetErrorString(e)); rc = SPAMM_ERR_CUDA; break; }
      }
      e = cudaMemcpyAsync(&s.n_groups, &lc->num_groups, sizeof(int), cudaMemcpyDeviceToHost, st);
      if (e != cudaSuccess) { set_error("copy: %s", cudaGetErrorString(e)); rc = SPAMM_ERR_CUDA; break; }
    }
    e = cudaEventRecord(ctx->ev[2], st);
    if (e != cudaSuccess) { set_error("event: %s", cudaGetErrorString(e)); rc = SPAMM_ERR_CUDA; break; }
    // C's tree: the reference rebuilds it with QuadTreeMatrix.__init__ (multiply.py:220)
    if ((rc = build_pyramid_async(c, st))) break;
    e = cudaEventRecord(ctx->ev[3], st);
    if (e != cudaSuccess) { set_error("event: %s", cudaGetErrorString(e)); rc = SPAMM_ERR_CUDA; break; }
    if ((rc = finish_tree(ctx, c))) break;  // syncs the stream
  } while (0);
  if (rc) {
    free_tree_async(c, st);
    return rc;
  }
  s.n_groups &= 0xffffffffll;
  cudaEventElapsedTime(&s.ms_cull, ctx->ev[0], ctx->ev[1]);
  cudaEventElapsedTime(&s.ms_leaf, ctx->ev[1], ctx->ev[2]);
  cudaEventElapsedTime(&s.ms_ctree, ctx->ev[2], ctx->ev[3]);
  cudaEventElapsedTime(&s.ms_total, ctx->ev[0], ctx->ev[3]);

  // ------------------------------------------------------- product records
  if (product) {
    auto p = std::make_unique<spamm_product>();
    if (flags & SPAMM_COLLECT_BOXES) {
      std::vector<uint64_t> codes(total_pruned);
      if (total_pruned) {
        cudaError_t e = cudaMemcpy(codes.data(), ctx->pruned_codes.ptr,
                                   total_pruned * sizeof(uint64_t), cudaMemcpyDeviceToHost);
        if (e != cudaSuccess) {
          free_tree_async(c, st);
          set_error("copy boxes: %s", cudaGetErrorString(e));
          return SPAMM_ERR_CUDA;
        }
      }
      p->boxes.reserve(5 * total_pruned);
      int64_t pos = 0;
      for (int t = 0; t <= depth; ++t) {
        const int64_t edge = a->N >> t;
        for (unsigned long long q = 0; q < hc->n_pruned[t]; ++q, ++pos) {
          uint32_t i, j, k;
          morton_decode(codes[pos], i, j, k);
          p->boxes.push_back(int64_t(i) * edge);
          p->boxes.push_back(int64_t(j) * edge);
          p->boxes.push_back(int64_t(k) * edge);
          p->boxes.push_back(edge);
          p->boxes.push_back(t);
        }
      }
    }
    if (flags & SPAMM_KEEP_TRIPLES) {
      const uint64_t kmask = (uint64_t(1) << depth) - 1;
      p->triples.reserve(3 * m);
      for (int64_t q = 0; q < m; ++q) {
        const uint64_t gid = host_keys[q] >> depth;
        p->triples.push_back((int32_t)(gid / nb));
        p->triples.push_back((int32_t)(gid % nb));
        p->triples.push_back((int32_t)(host_keys[q] & kmask));
      }
    }
    *product = p.release();
  }
  if (stats) *stats = s;
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

void spamm_product_free(spamm_product *p) { delete p; }

}  // extern "C"
