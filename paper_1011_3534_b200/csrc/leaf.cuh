// leaf.cuh -- K3 interfaces (see leaf.cu).
#pragma once
#include "common.cuh"
#include "traverse.cuh"

namespace spamm {

struct LeafArgs {
  const void *a, *b;                  // padded operands (N x N row-major)
  void *c;                            // padded product (zeroed by the caller)
  int64_t N, nb;
  int32_t leaf, depth;
  const unsigned long long *n_codes;  // device count of retained triples
  unsigned long long capacity;        // clamp for n_codes
  const uint32_t *ks;                 // inner indices, sorted within each group
  const uint32_t *group_ids;          // C block i*nb + j of each group
  const uint32_t *group_starts;       // first triple of each group
  TraverseCounters *tc;               // num_groups + work ticket
  unsigned long long *timeline;       // optional: per-CTA [start, end, items] (%globaltimer)
  int b_map5;                         // B streamed as the conflict-free 5-D TMA box
  unsigned *grp_done;                 // optional: per-group count of finished warp tiles
  const uint32_t *order;              // optional: work order over the groups (longest first)
  int pdl;                            // launch as a programmatic dependent of the previous kernel
  // bitmask groups (dense traversal): each group's k list is the set bits of
  // the retained leaf-triple bitmask (Morton order) for its C block, and the
  // group list is ready once tc->groups_ready is set -- no ks / group_starts
  // and no wait for the traversal grid's completion
  const uint32_t *am;
  int tm_slots;                       // merge-stack slots kept in TMEM (the rest in local memory)
  int tm_sync;                        // wait for each TMEM spill to complete (debug)
  int drain_items;                    // final wave: take a ticket only with the ring drained
};

// Returns through *signals whether the launched kernel reports finished groups
// in args.grp_done (CWARPS per (sub-)tile) and lets dependents launch early.
int launch_leaf(const LeafArgs &args, int dtype, int num_sms, cudaStream_t st, int *launches,
                bool *signals = nullptr);
// consumer warps of the warp-specialised kernel per (sub-)tile at this leaf size
unsigned leaf_signals_per_tile(int leaf);

}  // namespace spamm
