/*
 * spamm_oracle.c -- TEST INFRASTRUCTURE ONLY (the checker, never the product).
 *
 * A plain-C restatement of the reference SpAMM hot path
 * (arxiv/paper_1011_3534, package `spamm` 0.1.0, /root/reference/pkg/src/spamm).
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  The CUDA product path never
 * links or calls it.
 *
 * Pinned against the reference itself: tests/golden/make_golden.py imports
 * the reference package in the build container and records its pyramids,
 * retained leaf triples (captured from its own _leaf_stage), stats and boxes;
 * tests/test_oracle.py checks this file against those fixtures bit-for-bit
 * (integers, norms, budget) and to 1e-13 relative for C.
 *
 * Floating-point contract: compiled with -ffp-contract=off so every
 * `acc + e*e` rounds the product and the sum separately, exactly as numpy's
 * `acc += e * e` does (quadtree.py:80-87).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define DT_F64 0
#define DT_F32 1

/* quadtree.py:245-247 -- smallest depth with leaf << depth >= n. */
int oracle_depth(int64_t n, int32_t leaf) {
  int d = 0;
  while (((int64_t)leaf << d) < n) ++d;
  return d;
}

static inline int64_t level_offset(int k) { return (((int64_t)1 << (2 * k)) - 1) / 3; }

/*
 * QuadTreeMatrix.__init__ (quadtree.py:116-151) on an already padded N x N
 * row-major array:
 *   - leaf_nonzero = any(x != 0) per leaf                     (:126)
 *   - all-zero leaves rewritten as +0.0 (canonical form)      (:127-129)
 *   - leaf norm_sq: sequential row-major sum of squares in f64 (:74-87)
 *   - parents ((c11 + c12) + c21) + c22, occupancy OR          (:90-92, :134-138)
 * Levels are concatenated, level k (2^k x 2^k, row-major) at (4^k-1)/3.
 */
void oracle_build_pyramid(void *padded, int dtype, int64_t N, int32_t leaf,
                          double *nsq, uint8_t *occ) {
  const int depth = oracle_depth(N, leaf);
  const int64_t nb = N / leaf;
  double *lvl = nsq + level_offset(depth);
  uint8_t *olvl = occ + level_offset(depth);
  for (int64_t bi = 0; bi < nb; ++bi) {
    for (int64_t bj = 0; bj < nb; ++bj) {
      double acc = 0.0;
      int nz = 0;
      for (int r = 0; r < leaf; ++r) {
        const int64_t row = (bi * leaf + r) * N + bj * leaf;
        for (int c = 0; c < leaf; ++c) {
          double e = dtype == DT_F64 ? ((const double *)padded)[row + c]
                                     : (double)((const float *)padded)[row + c];
          nz |= (e != 0.0);
          acc = acc + e * e;
        }
      }
      if (!nz) {
        for (int r = 0; r < leaf; ++r) {
          const int64_t row = (bi * leaf + r) * N + bj * leaf;
          for (int c = 0; c < leaf; ++c) {
            if (dtype == DT_F64) ((double *)padded)[row + c] = 0.0;
            else ((float *)padded)[row + c] = 0.0f;
          }
        }
      }
      lvl[bi * nb + bj] = acc;
      olvl[bi * nb + bj] = (uint8_t)nz;
    }
  }
  for (int k = depth - 1; k >= 0; --k) {
    const int64_t s = (int64_t)1 << k, f = s * 2;
    const double *fine = nsq + level_offset(k + 1);
    const uint8_t *ofine = occ + level_offset(k + 1);
    double *coarse = nsq + level_offset(k);
    uint8_t *ocoarse = occ + level_offset(k);
    for (int64_t i = 0; i < s; ++i)
      for (int64_t j = 0; j < s; ++j) {
        const int64_t r0 = (2 * i) * f + 2 * j, r1 = r0 + f;
        coarse[i * s + j] = ((fine[r0] + fine[r0 + 1]) + fine[r1]) + fine[r1 + 1];
        ocoarse[i * s + j] = ofine[r0] | ofine[r0 + 1] | ofine[r1] | ofine[r1 + 1];
      }
  }
}

/*
 * numpy's pairwise summation for float64 (the algorithm behind
 * `norm_prod[pruned].sum()`, multiply.py:197): blocks of <= 128 use eight
 * interleaved accumulators, larger spans split at n/2 rounded down to a
 * multiple of 8.
 */
double oracle_pairwise_sum(const double *a, int64_t n) {
  if (n < 8) {
    double res = 0.0;
    for (int64_t i = 0; i < n; ++i) res += a[i];
    return res;
  }
  if (n <= 128) {
    double r[8];
    for (int q = 0; q < 8; ++q) r[q] = a[q];
    int64_t i;
    for (i = 8; i < n - (n % 8); i += 8)
      for (int q = 0; q < 8; ++q) r[q] += a[i + q];
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; ++i) res += a[i];
    return res;
  }
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  return oracle_pairwise_sum(a, n2) + oracle_pairwise_sum(a + n2, n - n2);
}

/* Result of one culling traversal; arrays are malloc'd, free with oracle_free. */
typedef struct {
  int64_t leaf_matmuls, pruned_calls, pruned_volume, empty_skip_volume;
  int32_t max_depth_reached, pad_;
  double omitted_budget;
  int64_t n_triples;   /* retained leaf triples, sorted by (i, j, k)        */
  int32_t *triples;    /* 3 * n_triples: i, j, k                             */
  int64_t n_boxes;     /* tau-pruned boxes, tier-major then candidate order  */
  int64_t *boxes;      /* 5 * n_boxes: i_lo, j_lo, k_lo, edge, tier          */
  int64_t tier_candidates[32], tier_survivors[32];
  double *box_np;      /* n_boxes: each box's norm product (multiply.py:185)  */
} oracle_cull_result;

void oracle_free(void *p) { free(p); }

static int cmp_triple(const void *x, const void *y) {
  const int32_t *a = (const int32_t *)x, *b = (const int32_t *)y;
  for (int q = 0; q < 3; ++q)
    if (a[q] != b[q]) return a[q] < b[q] ? -1 : 1;
  return 0;
}

/*
 * The breadth-first tier loop of spamm() (multiply.py:174-212): per tier the
 * occupancy test (:184), the norm product sqrt(a)*sqrt(b) (:185), the
 * optional tau/8^tier policy (:186), strict `< tau` pruning (:187), the
 * counters (:189-197), boxes (:198-200) and the 8-way (di,dj,dk) expansion
 * in 000..111 order (:35-37, :207-212).  Leaf survivors are returned sorted
 * by (i, j, k) like _leaf_stage's lexsort (:231-233).
 */
/*
 * Row-sharded variant (the multi-GPU layout, not in the reference): only
 * triples whose leaf rows [i << (depth-t), (i+1) << (depth-t)) intersect
 * [row_lo, row_hi) are traversed, and a pruned / skipped call is counted by
 * the shard owning its first row.  Summed over disjoint shards covering all
 * rows, every integer statistic equals the unsharded traversal's.
 */
int oracle_cull_rows(const double *nsq_a, const uint8_t *occ_a, const double *nsq_b,
                     const uint8_t *occ_b, int depth, int64_t N, double tau,
                     int tier_tau_decay, int count_stats, int collect_boxes,
                     int64_t row_lo, int64_t row_hi, oracle_cull_result *res);

int oracle_cull(const double *nsq_a, const uint8_t *occ_a, const double *nsq_b,
                const uint8_t *occ_b, int depth, int64_t N, double tau,
                int tier_tau_decay, int count_stats, int collect_boxes,
                oracle_cull_result *res) {
  return oracle_cull_rows(nsq_a, occ_a, nsq_b, occ_b, depth, N, tau, tier_tau_decay,
                          count_stats, collect_boxes, 0, (int64_t)1 << depth, res);
}

int oracle_cull_rows(const double *nsq_a, const uint8_t *occ_a, const double *nsq_b,
                     const uint8_t *occ_b, int depth, int64_t N, double tau,
                     int tier_tau_decay, int count_stats, int collect_boxes,
                     int64_t row_lo, int64_t row_hi, oracle_cull_result *res) {
  memset(res, 0, sizeof *res);
  int64_t cap = 8, n = 1;
  int32_t *cur = (int32_t *)malloc(sizeof(int32_t) * 3 * cap);
  if (!cur) return -1;
  cur[0] = cur[1] = cur[2] = 0;
  int64_t box_cap = 0;
  for (int tier = 0; tier <= depth; ++tier) {
    if (n == 0) break;
    res->max_depth_reached = tier;
    res->tier_candidates[tier] = n;
    const int64_t edge = N >> tier;
    const int64_t vol = edge * edge * edge;
    const int64_t s = (int64_t)1 << tier;
    const double *na = nsq_a + level_offset(tier), *nb_ = nsq_b + level_offset(tier);
    const uint8_t *oa = occ_a + level_offset(tier), *ob = occ_b + level_offset(tier);
    const double tau_t = tier_tau_decay ? tau * ldexp(1.0, -3 * tier) : tau;
    int32_t *act = (int32_t *)malloc(sizeof(int32_t) * 3 * (n > 0 ? n : 1));
    double *pruned_np = (double *)malloc(sizeof(double) * (n > 0 ? n : 1));
    if (!act || !pruned_np) return -1;
    int64_t n_act = 0, n_alive = 0, n_pruned = 0;
    const int shift = depth - tier;
    int64_t n_skip_owned = 0;
    for (int64_t c = 0; c < n; ++c) {
      const int32_t i = cur[3 * c], j = cur[3 * c + 1], k = cur[3 * c + 2];
      const int64_t r0 = (int64_t)i << shift, r1 = (int64_t)(i + 1) << shift;
      if (!(r1 > row_lo && r0 < row_hi)) continue;  /* another shard's rows */
      const int owned = r0 >= row_lo && r0 < row_hi;
      const int alive = oa[(int64_t)i * s + k] && ob[(int64_t)k * s + j];
      const double np_ = sqrt(na[(int64_t)i * s + k]) * sqrt(nb_[(int64_t)k * s + j]);
      const int pruned = alive && (np_ < tau_t);
      n_alive += alive;
      if (!alive && owned) ++n_skip_owned;
      if (pruned && !owned) continue;  /* counted by the owning shard */
      if (pruned) {
        pruned_np[n_pruned++] = np_;
        if (collect_boxes) {
          if (res->n_boxes == box_cap) {
            box_cap = box_cap ? 2 * box_cap : 1024;
            res->boxes = (int64_t *)realloc(res->boxes, sizeof(int64_t) * 5 * box_cap);
            res->box_np = (double *)realloc(res->box_np, sizeof(double) * box_cap);
            if (!res->boxes || !res->box_np) return -1;
          }
          res->box_np[res->n_boxes] = np_;
          int64_t *bx = res->boxes + 5 * res->n_boxes++;
          bx[0] = (int64_t)i * edge; bx[1] = (int64_t)j * edge; bx[2] = (int64_t)k * edge;
          bx[3] = edge; bx[4] = tier;
        }
      } else if (alive) {
        act[3 * n_act] = i; act[3 * n_act + 1] = j; act[3 * n_act + 2] = k;
        ++n_act;
      }
    }
    if (count_stats) {
      const int64_t n_skip = n_skip_owned;
      res->pruned_calls += n_skip + n_pruned;
      res->empty_skip_volume += n_skip * vol;
      res->pruned_volume += n_pruned * vol;
      if (n_pruned) res->omitted_budget += oracle_pairwise_sum(pruned_np, n_pruned);
    }
    free(pruned_np);
    res->tier_survivors[tier] = n_act;
    free(cur);
    if (tier == depth) {
      if (count_stats) res->leaf_matmuls += n_act;
      qsort(act, (size_t)n_act, sizeof(int32_t) * 3, cmp_triple);
      res->triples = act;
      res->n_triples = n_act;
      return 0;
    }
    cur = (int32_t *)malloc(sizeof(int32_t) * 3 * 8 * (n_act > 0 ? n_act : 1));
    if (!cur) return -1;
    for (int64_t c = 0; c < n_act; ++c)
      for (int q = 0; q < 8; ++q) {
        int32_t *o = cur + 3 * (8 * c + q);
        o[0] = 2 * act[3 * c] + (q >> 2);
        o[1] = 2 * act[3 * c + 1] + ((q >> 1) & 1);
        o[2] = 2 * act[3 * c + 2] + (q & 1);
      }
    n = 8 * n_act;
    free(act);
  }
  free(cur);
  return 0;
}

/* Leaf product P = A_ik * B_kj (b x b, row-major blocks inside N x N), leaf_gemm.c. */
void oracle_leaf_gemm_f64(const double *a, const double *b, int64_t lda, int32_t leaf, double *p);
void oracle_leaf_gemm_f32(const float *a, const float *b, int64_t lda, int32_t leaf, float *p);

/*
 * Merge of one C block's leaf products over the inner index
 * (_merge_contributions, multiply.py:119-141): an aligned binary interval
 * tree over k in [lo, hi); both halves present -> left + right, one present
 * -> passed through bit-intact.  `ks` is the sorted retained k list of the
 * group restricted to [lo, hi).
 */
static void merge_range_f64(const double *A, const double *B, int64_t N, int32_t leaf,
                            int32_t i, int32_t j, const int32_t *ks, int64_t nk,
                            int64_t lo, int64_t hi, double *out, double *scratch) {
  if (nk == 1) {
    oracle_leaf_gemm_f64(A + (int64_t)i * leaf * N + (int64_t)ks[0] * leaf,
                         B + (int64_t)ks[0] * leaf * N + (int64_t)j * leaf, N, leaf, out);
    return;
  }
  const int64_t mid = lo + (hi - lo) / 2;
  int64_t nl = 0;
  while (nl < nk && ks[nl] < mid) ++nl;
  if (nl == 0) { merge_range_f64(A, B, N, leaf, i, j, ks, nk, mid, hi, out, scratch); return; }
  if (nl == nk) { merge_range_f64(A, B, N, leaf, i, j, ks, nk, lo, mid, out, scratch); return; }
  const int64_t bb = (int64_t)leaf * leaf;
  merge_range_f64(A, B, N, leaf, i, j, ks, nl, lo, mid, out, scratch + bb);
  merge_range_f64(A, B, N, leaf, i, j, ks + nl, nk - nl, mid, hi, scratch, scratch + bb);
  for (int64_t q = 0; q < bb; ++q) out[q] = out[q] + scratch[q];
}

static void merge_range_f32(const float *A, const float *B, int64_t N, int32_t leaf,
                            int32_t i, int32_t j, const int32_t *ks, int64_t nk,
                            int64_t lo, int64_t hi, float *out, float *scratch) {
  if (nk == 1) {
    oracle_leaf_gemm_f32(A + (int64_t)i * leaf * N + (int64_t)ks[0] * leaf,
                         B + (int64_t)ks[0] * leaf * N + (int64_t)j * leaf, N, leaf, out);
    return;
  }
  const int64_t mid = lo + (hi - lo) / 2;
  int64_t nl = 0;
  while (nl < nk && ks[nl] < mid) ++nl;
  if (nl == 0) { merge_range_f32(A, B, N, leaf, i, j, ks, nk, mid, hi, out, scratch); return; }
  if (nl == nk) { merge_range_f32(A, B, N, leaf, i, j, ks, nk, lo, mid, out, scratch); return; }
  const int64_t bb = (int64_t)leaf * leaf;
  merge_range_f32(A, B, N, leaf, i, j, ks, nl, lo, mid, out, scratch + bb);
  merge_range_f32(A, B, N, leaf, i, j, ks + nl, nk - nl, mid, hi, scratch, scratch + bb);
  for (int64_t q = 0; q < bb; ++q) out[q] = out[q] + scratch[q];
}

/*
 * _leaf_stage (multiply.py:224-257): every (i, j) group of the sorted triple
 * list is multiplied and merged, then assigned into C's padded storage;
 * untouched blocks stay +0.0.  `c_padded` must be zeroed by the caller.
 * Groups are independent, so they run in parallel under OpenMP; the result
 * does not depend on the thread count.
 */
int oracle_leaf_stage(const void *a_padded, const void *b_padded, int dtype, int64_t N,
                      int32_t leaf, const int32_t *triples, int64_t n_triples,
                      void *c_padded) {
  const int depth = oracle_depth(N, leaf);
  const int64_t bb = (int64_t)leaf * leaf;
  int64_t n_groups = 0;
  int64_t *starts = (int64_t *)malloc(sizeof(int64_t) * (n_triples + 1));
  if (!starts) return -1;
  for (int64_t t = 0; t < n_triples; ++t)
    if (t == 0 || triples[3 * t] != triples[3 * t - 3] || triples[3 * t + 1] != triples[3 * t - 2])
      starts[n_groups++] = t;
  starts[n_groups] = n_triples;
  int status = 0;
#pragma omp parallel
  {
    const size_t esz = dtype == DT_F64 ? sizeof(double) : sizeof(float);
    void *blk = malloc(esz * bb * (depth + 2));
    int32_t *ks = (int32_t *)malloc(sizeof(int32_t) * (((int64_t)1 << depth) + 1));
    if (!blk || !ks) {
#pragma omp atomic write
      status = -1;
    } else {
#pragma omp for schedule(dynamic, 4)
      for (int64_t g = 0; g < n_groups; ++g) {
        const int64_t s0 = starts[g], s1 = starts[g + 1];
        const int32_t i = triples[3 * s0], j = triples[3 * s0 + 1];
        for (int64_t t = s0; t < s1; ++t) ks[t - s0] = triples[3 * t + 2];
        const int64_t nk = s1 - s0, nbk = (int64_t)1 << depth;
        if (dtype == DT_F64) {
          double *out = (double *)blk;
          merge_range_f64((const double *)a_padded, (const double *)b_padded, N, leaf, i, j,
                          ks, nk, 0, nbk, out, out + bb);
          double *dst = (double *)c_padded;
          for (int r = 0; r < leaf; ++r)
            memcpy(dst + ((int64_t)i * leaf + r) * N + (int64_t)j * leaf, out + (int64_t)r * leaf,
                   sizeof(double) * leaf);
        } else {
          float *out = (float *)blk;
          merge_range_f32((const float *)a_padded, (const float *)b_padded, N, leaf, i, j,
                          ks, nk, 0, nbk, out, out + bb);
          float *dst = (float *)c_padded;
          for (int r = 0; r < leaf; ++r)
            memcpy(dst + ((int64_t)i * leaf + r) * N + (int64_t)j * leaf, out + (int64_t)r * leaf,
                   sizeof(float) * leaf);
        }
      }
    }
    free(blk);
    free(ks);
  }
  free(starts);
  return status;
}

/*
 * Pieces of the above for trees too large to hold densely on the host (the
 * c5 / c4 checks pull only pyramids and selected blocks off the GPU):
 *
 * oracle_leaf_norms: _leaf_norm_sq (quadtree.py:74-87) and the occupancy
 * test (:126) of `count` contiguous leaf blocks ([count][leaf][leaf]).
 */
void oracle_leaf_norms(const void *blocks, int dtype, int64_t count, int32_t leaf, double *nsq,
                       uint8_t *occ) {
  const int64_t bb = (int64_t)leaf * leaf;
#pragma omp parallel for schedule(static)
  for (int64_t q = 0; q < count; ++q) {
    double acc = 0.0;
    int nz = 0;
    for (int64_t e = 0; e < bb; ++e) {
      const double x = dtype == DT_F64 ? ((const double *)blocks)[q * bb + e]
                                       : (double)((const float *)blocks)[q * bb + e];
      nz |= (x != 0.0);
      acc = acc + x * x;
    }
    nsq[q] = acc;
    occ[q] = (uint8_t)nz;
  }
}

/* The levels above the leaves (_aggregate_norm_sq, quadtree.py:90-92, and the
 * occupancy OR, :135-138) from a filled leaf level, concatenated layout. */
void oracle_pyramid_from_leaves(double *nsq, uint8_t *occ, int depth) {
  for (int k = depth - 1; k >= 0; --k) {
    const int64_t s = (int64_t)1 << k, f = s * 2;
    const double *fine = nsq + level_offset(k + 1);
    const uint8_t *ofine = occ + level_offset(k + 1);
    double *coarse = nsq + level_offset(k);
    uint8_t *ocoarse = occ + level_offset(k);
    for (int64_t i = 0; i < s; ++i)
      for (int64_t j = 0; j < s; ++j) {
        const int64_t r0 = (2 * i) * f + 2 * j, r1 = r0 + f;
        coarse[i * s + j] = ((fine[r0] + fine[r0 + 1]) + fine[r1]) + fine[r1 + 1];
        ocoarse[i * s + j] = ofine[r0] | ofine[r0 + 1] | ofine[r1] | ofine[r1 + 1];
      }
  }
}

/* One C block of _leaf_stage (multiply.py:224-257) from its operand blocks:
 * a_blocks[q] = A(i, ks[q]), b_blocks[q] = B(ks[q], j), contiguous leaf x
 * leaf, ks ascending; the products merged over the aligned binary intervals
 * of [0, 2^depth) (_merge_contributions, :119-141).  Same arithmetic as
 * oracle_leaf_stage, with the blocks gathered (lda = leaf). */
static void merge_blocks_f64(const double *A, const double *B, int32_t leaf, const int32_t *ks,
                             int64_t nk, int64_t lo, int64_t hi, double *out, double *scratch) {
  const int64_t bb = (int64_t)leaf * leaf;
  if (nk == 1) {
    oracle_leaf_gemm_f64(A, B, leaf, leaf, out);
    return;
  }
  const int64_t mid = lo + (hi - lo) / 2;
  int64_t nl = 0;
  while (nl < nk && ks[nl] < mid) ++nl;
  if (nl == 0) { merge_blocks_f64(A, B, leaf, ks, nk, mid, hi, out, scratch); return; }
  if (nl == nk) { merge_blocks_f64(A, B, leaf, ks, nk, lo, mid, out, scratch); return; }
  merge_blocks_f64(A, B, leaf, ks, nl, lo, mid, out, scratch + bb);
  merge_blocks_f64(A + nl * bb, B + nl * bb, leaf, ks + nl, nk - nl, mid, hi, scratch, scratch + bb);
  for (int64_t q = 0; q < bb; ++q) out[q] = out[q] + scratch[q];
}
static void merge_blocks_f32(const float *A, const float *B, int32_t leaf, const int32_t *ks,
                             int64_t nk, int64_t lo, int64_t hi, float *out, float *scratch) {
  const int64_t bb = (int64_t)leaf * leaf;
  if (nk == 1) {
    oracle_leaf_gemm_f32(A, B, leaf, leaf, out);
    return;
  }
  const int64_t mid = lo + (hi - lo) / 2;
  int64_t nl = 0;
  while (nl < nk && ks[nl] < mid) ++nl;
  if (nl == 0) { merge_blocks_f32(A, B, leaf, ks, nk, mid, hi, out, scratch); return; }
  if (nl == nk) { merge_blocks_f32(A, B, leaf, ks, nk, lo, mid, out, scratch); return; }
  merge_blocks_f32(A, B, leaf, ks, nl, lo, mid, out, scratch + bb);
  merge_blocks_f32(A + nl * bb, B + nl * bb, leaf, ks + nl, nk - nl, mid, hi, scratch, scratch + bb);
  for (int64_t q = 0; q < bb; ++q) out[q] = out[q] + scratch[q];
}
int oracle_group_product(const void *a_blocks, const void *b_blocks, int dtype, int32_t leaf,
                         const int32_t *ks, int64_t nk, int depth, void *out) {
  if (nk <= 0) return -1;
  const size_t esz = dtype == DT_F64 ? sizeof(double) : sizeof(float);
  void *scratch = malloc(esz * (size_t)leaf * leaf * (depth + 2));
  if (!scratch) return -1;
  if (dtype == DT_F64)
    merge_blocks_f64((const double *)a_blocks, (const double *)b_blocks, leaf, ks, nk, 0,
                     (int64_t)1 << depth, (double *)out, (double *)scratch);
  else
    merge_blocks_f32((const float *)a_blocks, (const float *)b_blocks, leaf, ks, nk, 0,
                     (int64_t)1 << depth, (float *)out, (float *)scratch);
  free(scratch);
  return 0;
}
