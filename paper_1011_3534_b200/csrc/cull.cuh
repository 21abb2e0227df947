// cull.cuh -- K2 interfaces (see cull.cu).
#pragma once
#include "common.cuh"

namespace spamm {

constexpr int MAX_TIERS = 32;

// Device-resident traversal counters, one slot per tier.
struct CullCounters {
  unsigned long long ticket[MAX_TIERS];      // tile tickets
  unsigned long long n_cand[MAX_TIERS];      // candidates generated
  unsigned long long n_alive[MAX_TIERS];     // occupancy survivors (intersecting)
  unsigned long long n_active[MAX_TIERS];    // survivors (next tier's parents)
  unsigned long long n_pruned[MAX_TIERS];    // tau-pruned calls (owned)
  unsigned long long n_skip[MAX_TIERS];      // Empty-operand skips (owned)
  unsigned long long pruned_base[MAX_TIERS]; // offset of the tier's pruned list
  double tier_budget[MAX_TIERS];             // pairwise sum of the tier's pruned products
  double budget;                             // omitted_budget
  int overflow;                              // a capacity was exceeded: re-run larger
  int pad_;
};

struct CullTierArgs {
  int tier, depth;
  double tau;
  const double *nsq_a, *nsq_b;    // level `tier` of each pyramid
  const uint8_t *occ_a, *occ_b;
  const uint64_t *prev;           // survivors of tier-1 (Morton codes)
  uint64_t *next;                 // survivors of this tier
  unsigned long long capacity;    // items per survivor buffer
  double *pruned_vals;            // all tiers, in reference order
  uint64_t *pruned_codes;
  unsigned long long pruned_capacity;
  unsigned long long *tile_status;
  CullCounters *counters;
  int64_t row_lo, row_hi;         // C leaf block rows of this shard
};

struct CullPlan {
  int depth;
  double tau_tier[MAX_TIERS];
  const double *nsq_a, *nsq_b;
  const uint8_t *occ_a, *occ_b;
  uint64_t *codes[2];
  unsigned long long capacity;
  double *pruned_vals;
  uint64_t *pruned_codes;
  unsigned long long pruned_capacity;
  unsigned long long *tile_status;
  CullCounters *counters;
  int64_t row_lo, row_hi;
  int max_ctas;
  int *launches;  // kernel launch counter (may be null)
};

int launch_cull(const CullPlan &plan, cudaStream_t st);
size_t tile_status_bytes(size_t capacity);

}  // namespace spamm
