// traverse.cuh -- K2 interfaces: product-space traversal + leaf grouping.
#pragma once
#include "common.cuh"

namespace spamm {

constexpr int MAX_TIERS = 32;

// 3-bit interleave helpers of the dense traversal's Morton codes (10-bit
// coordinates): x = spread3(i) << 2 | spread3(j) << 1 | spread3(k).
__host__ __device__ __forceinline__ uint32_t compact3(uint32_t x) {
  x &= 0x09249249u;
  x = (x ^ (x >> 2)) & 0x030c30c3u;
  x = (x ^ (x >> 4)) & 0x0300f00fu;
  x = (x ^ (x >> 8)) & 0xff0000ffu;
  x = (x ^ (x >> 16)) & 0x000003ffu;
  return x;
}
__host__ __device__ __forceinline__ uint32_t spread3(uint32_t x) {
  x &= 0x3ffu;
  x = (x | (x << 16)) & 0xff0000ffu;
  x = (x | (x << 8)) & 0x0300f00fu;
  x = (x | (x << 4)) & 0x030c30c3u;
  x = (x | (x << 2)) & 0x09249249u;
  return x;
}

constexpr int DN_PARTS_H = 16, DN_MAXT_H = 8;  // dn_part dimensions

// Device-resident counters of one multiply.  Two sets alternate between
// calls: a call finds its set zero and clears the other (the previous call's,
// already read back by the host).
struct TraverseCounters {
  unsigned long long ticket[MAX_TIERS];      // tile tickets of the grid-wide tiers
  unsigned long long n_cand[MAX_TIERS];      // candidates generated
  unsigned long long n_alive[MAX_TIERS];     // occupancy survivors (intersecting the shard)
  unsigned long long n_active[MAX_TIERS];    // survivors (next tier's parents)
  unsigned long long n_pruned[MAX_TIERS];    // tau-pruned calls (owned by the shard)
  unsigned long long n_skip[MAX_TIERS];      // Empty-operand skips (owned)
  unsigned long long pruned_base[MAX_TIERS]; // offset of the tier's pruned list
  double tier_budget[MAX_TIERS];             // numpy-pairwise sum of the tier's pruned products
  double budget;                             // omitted_budget
  int overflow;                              // a capacity was exceeded: re-run larger
  int first_grid_tier;                       // tiers below ran in the single-CTA prefix
  unsigned num_groups;                       // non-empty C blocks
  unsigned budgets_done;                     // tiers whose pruned sum is final
  unsigned long long scan_ticket, sort_ticket, gemm_ticket, gemm_ticket2;
  unsigned groups_done, pad0;
  // grid barrier arrival counters (whole grid, subset), each on its own
  // 128-byte line so polling CTAs never contend with the counters above
  alignas(128) unsigned bar_grid;
  alignas(128) unsigned bar_sub;
  alignas(128) unsigned bar_pad;
  unsigned long long dirty_tiles[3];         // status entries to clear before the next call
  unsigned long long phase_ns[16];           // %globaltimer at phase boundaries (CTA 0)
  unsigned long long dn_part[16][8][4];      // dense traversal: per-CTA-group tier counters
  unsigned long long k3_t0n, k3_t1, k1_t1;   // %globaltimer: ~(K3 first start), K3 last end, C tree end
  unsigned lpt_hist[132];                    // dense traversal: groups per size (k count)
  unsigned pw_done[MAX_TIERS];               // budget items finished per tier
  unsigned tiers_done, pad1;                 // tiers whose budget is final
  // dense traversal, bitmask groups: set (release) once the group list and
  // num_groups are final -- the leaf products start on this, not on the
  // traversal grid's completion (its pruned-record and budget CTAs run on)
  alignas(128) unsigned groups_ready;
  unsigned exited;                           // traversal CTAs that have finished
  unsigned trav_done;                        // set (release) by the last one
};

struct TraverseArgs {
  int depth;
  int64_t nb;
  double tau_tier[MAX_TIERS];
  const double *nrm_a, *nrm_b;      // rn(sqrt(norm_sq)) pyramids (concatenated levels)
  const uint8_t *occ_a, *occ_b;
  uint64_t *codes[2];               // ping-pong survivor lists (packed i,j,k)
  unsigned long long capacity;      // items per survivor list
  double *pruned_vals;              // all tiers, reference order
  uint64_t *pruned_codes;
  unsigned long long pruned_capacity;
  unsigned long long *status[3];    // look-back state: two tier arrays + the group scan
  TraverseCounters *tc;
  int64_t row_lo, row_hi;           // C leaf block rows of this shard
  // grouping outputs
  uint32_t *counts;                 // nb^2 bucket sizes
  uint32_t *offsets;                // nb^2 bucket offsets
  uint32_t *group_ids;              // non-empty buckets, ascending i*nb + j
  uint32_t *group_starts;           // their offsets into ks
  uint32_t *ks;                     // inner indices, bucket-major, ascending per bucket
  // dense traversal (depth <= 6; the layouts are instantiated up to 7)
  uint32_t *dn_masks;               // this call's work set (DnLayout; zero at entry)
  uint32_t *dn_masks_clear;         // the previous call's work set, zeroed by this call
  unsigned long long dn_work_words; // words per work set
  uint32_t *dn_retained;            // retained leaf-triple bitmask
  double *dn_np;                    // leaf-tier pruned norm products, by Morton code
  unsigned long long *dn_status;    // look-back state: pruned scan, then (+dn_status_q) groups
  unsigned long long dn_status_q;
  TraverseCounters *tc_clear;       // the previous call's counter set, zeroed by this call
  unsigned long long *timeline;     // optional per-CTA %globaltimer stamps (4 per CTA)
  uint32_t *lpt_order;              // optional: groups by decreasing size (K3's work order)
  double *pw_part;                  // budget: per-tier top-of-recursion partial sums
  // dense traversal: zero the product's leaf-level norms (nb^2 entries each)
  // while classifying -- only the C blocks that receive products get norms
  double *c_nsq_leaf, *c_nrm_leaf;
  uint8_t *c_occ_leaf;
  // dense traversal: the groups are only the non-empty C blocks (group_ids,
  // num_groups); each block's k list is read from the retained bitmask by
  // the leaf-product kernel itself (no ks / group_starts), and readiness is
  // signalled through tc->groups_ready
  int bitmask_groups;
};

// Launch the cooperative traversal kernel (one launch per multiply).
int launch_traverse(const TraverseArgs &args, int num_sms, cudaStream_t st);
// Dense single-pass variant for shallow trees (see traverse.cu).
bool dense_traversal_ok(int depth);
size_t dense_mask_words(int depth);
size_t dense_work_words(int depth);
size_t dense_ne_offset(int depth);  // (words, within a work set)
size_t dense_retained_words(int depth);
size_t dense_pruned_tiles(int depth);
size_t dense_np_entries(int depth);
size_t dense_status_entries(int depth, int64_t nb);
int launch_traverse_dense(const TraverseArgs &args, int num_sms, cudaStream_t st);
size_t traverse_status_entries(size_t capacity);
size_t group_status_entries(int64_t nb);

}  // namespace spamm
