// leaf.cuh -- K3 interfaces (see leaf.cu).
#pragma once
#include "common.cuh"

namespace spamm {

struct LeafArgs {
  const void *a, *b;               // padded operands (N x N row-major)
  void *c;                         // padded product (zeroed by the caller)
  int64_t N, nb, m;                // padded dim, block grid, number of triples
  int32_t leaf, depth;
  const uint64_t *keys;            // sorted (i*nb + j) << depth | k
  const int *group_starts;         // first triple of each C block
  const int *num_groups;           // device-resident group count
  unsigned long long *ticket;      // zeroed work ticket
};

int launch_leaf(const LeafArgs &args, int dtype, int num_sms, cudaStream_t st);

}  // namespace spamm
