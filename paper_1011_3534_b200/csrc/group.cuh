// group.cuh -- leaf-triple grouping interfaces (see group.cu).
#pragma once
#include <algorithm>

#include "common.cuh"

namespace spamm {

// Device counters of the leaf stage.
struct LeafCounters {
  unsigned num_groups;              // non-empty C blocks
  unsigned pad_;
  unsigned long long scan_ticket;
  unsigned long long sort_ticket;
  unsigned long long gemm_ticket;
};

struct GroupArgs {
  const uint64_t *codes;              // leaf-tier survivors (Morton codes)
  const unsigned long long *n_codes;  // device count of `codes`
  unsigned long long capacity;        // clamp for n_codes
  int depth;
  int64_t nb;
  uint32_t *counts;                   // nb^2 bucket sizes (zeroed here)
  uint32_t *offsets;                  // nb^2 bucket offsets
  uint32_t *group_ids;                // non-empty buckets, ascending i*nb + j
  uint32_t *group_starts;             // their offsets
  uint32_t *ks;                       // inner indices, bucket-major, sorted per bucket
  unsigned long long *tile_status;    // look-back state for the scan
  LeafCounters *lc;
};

int launch_grouping(const GroupArgs &g, int64_t capacity, int num_sms, cudaStream_t st,
                    int *launches);
size_t group_tile_status_bytes(int64_t nb);

}  // namespace spamm
