// group.cu -- grouping of the retained leaf triples by C block.
//
// Reference: _leaf_stage sorts the retained triples by (i, j, k)
// (np.lexsort, multiply.py:231-233) and forms groups i*nb + j (:234) so that
// each C block's products can be merged over ascending k.
//
// Here the same grouping is built without any host round trip (all sizes the
// host needs are static: nb^2 buckets; the triple count stays on the device):
//   1. count   -- atomic histogram of triples per C block
//   2. scan    -- single-pass look-back scan: bucket offsets, plus the
//                 ascending list of non-empty C blocks and its length
//   3. scatter -- each triple's k into its bucket (slot order arbitrary)
//   4. sort    -- each bucket's k list sorted ascending in shared memory
//                 (all-ascending bitonic network; distinct keys, so the
//                 result is unique and deterministic)
// The sorted buckets laid end to end are exactly the reference's lexsorted
// triple list.
#include "group.cuh"
#include "scan.cuh"

namespace spamm {

constexpr int GRP_THREADS = 256;
constexpr int GRP_ITEMS = 4;
constexpr int GRP_TILE = GRP_THREADS * GRP_ITEMS;
constexpr int SORT_THREADS = 256;
constexpr int SORT_SMEM_KEYS = 4096;

__device__ __forceinline__ unsigned long long n_triples(const GroupArgs &g) {
  unsigned long long m = *g.n_codes;
  return m < g.capacity ? m : g.capacity;
}

__global__ void group_count_kernel(GroupArgs g) {
  const unsigned long long m = n_triples(g);
  for (unsigned long long p = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; p < m;
       p += (unsigned long long)gridDim.x * blockDim.x) {
    uint32_t i, j, k;
    morton_decode(g.codes[p], i, j, k);
    atomicAdd(&g.counts[int64_t(i) * g.nb + j], 1u);
  }
}

__global__ void __launch_bounds__(GRP_THREADS) group_scan_kernel(GroupArgs g) {
  __shared__ unsigned long long s_warp[GRP_THREADS / 32];
  __shared__ unsigned long long s_excl;
  __shared__ unsigned long long s_tile;
  const int64_t G = g.nb * g.nb;
  const unsigned long long n_tiles = (G + GRP_TILE - 1) / GRP_TILE;
  for (;;) {
    if (threadIdx.x == 0) s_tile = atomicAdd(&g.lc->scan_ticket, 1ull);
    __syncthreads();
    const unsigned long long tile = s_tile;
    if (tile >= n_tiles) break;
    const int64_t base = (int64_t)tile * GRP_TILE + threadIdx.x * GRP_ITEMS;
    unsigned cnt[GRP_ITEMS], sum = 0, ne = 0;
#pragma unroll
    for (int q = 0; q < GRP_ITEMS; ++q) {
      cnt[q] = base + q < G ? g.counts[base + q] : 0u;
      sum += cnt[q];
      ne += cnt[q] != 0;
    }
    unsigned long long total;
    const unsigned long long in_tile =
        block_exclusive<GRP_THREADS>(pack2(sum, ne), s_warp, &total);
    if ((threadIdx.x >> 5) == 0) {
      const unsigned long long excl = lookback_exclusive(g.tile_status, tile, total);
      if ((threadIdx.x & 31) == 0) {
        s_excl = excl;
        atomicAdd(&g.lc->num_groups, unpack_b(total));
      }
    }
    __syncthreads();
    const unsigned long long pre = s_excl + in_tile;
    unsigned off = unpack_a(pre), slot = unpack_b(pre);
#pragma unroll
    for (int q = 0; q < GRP_ITEMS; ++q) {
      if (base + q < G) {
        g.offsets[base + q] = off;
        if (cnt[q]) {
          g.group_ids[slot] = (uint32_t)(base + q);
          g.group_starts[slot] = off;
          ++slot;
        }
        off += cnt[q];
      }
    }
    __syncthreads();
  }
}

__global__ void group_scatter_kernel(GroupArgs g) {
  const unsigned long long m = n_triples(g);
  for (unsigned long long p = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; p < m;
       p += (unsigned long long)gridDim.x * blockDim.x) {
    uint32_t i, j, k;
    morton_decode(g.codes[p], i, j, k);
    const int64_t gid = int64_t(i) * g.nb + j;
    const unsigned slot = atomicSub(&g.counts[gid], 1u) - 1u;
    g.ks[g.offsets[gid] + slot] = k;
  }
}

// All-ascending bitonic network over x[0, n) with virtual +inf padding to the
// next power of two: every comparator writes the minimum to the lower index,
// so padding never moves into the real range.
template <bool SHARED>
__device__ void bitonic_sort(uint32_t *x, int n) {
  int P = 1;
  while (P < n) P <<= 1;
  for (int k = 2; k <= P; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < P; i += blockDim.x) {
        const int p = (j == (k >> 1)) ? (i ^ (k - 1)) : (i ^ j);
        if (p > i && p < n) {
          const uint32_t a = x[i], b = x[p];
          if (a > b) {
            x[i] = b;
            x[p] = a;
          }
        }
      }
      if (SHARED) __syncthreads();
      else {
        __threadfence_block();
        __syncthreads();
      }
    }
  }
}

__global__ void __launch_bounds__(SORT_THREADS) group_sort_kernel(GroupArgs g) {
  __shared__ uint32_t s_k[SORT_SMEM_KEYS];
  __shared__ unsigned s_q;
  const unsigned long long m = n_triples(g);
  for (;;) {
    if (threadIdx.x == 0) s_q = (unsigned)atomicAdd(&g.lc->sort_ticket, 1ull);
    __syncthreads();
    const unsigned q = s_q;
    const unsigned ng = g.lc->num_groups;
    if (q >= ng) break;
    const unsigned start = g.group_starts[q];
    const unsigned end = q + 1 < ng ? g.group_starts[q + 1] : (unsigned)m;
    const int n = (int)(end - start);
    if (n > 1) {
      if (n <= SORT_SMEM_KEYS) {
        for (int e = threadIdx.x; e < n; e += SORT_THREADS) s_k[e] = g.ks[start + e];
        __syncthreads();
        bitonic_sort<true>(s_k, n);
        for (int e = threadIdx.x; e < n; e += SORT_THREADS) g.ks[start + e] = s_k[e];
      } else {
        bitonic_sort<false>(g.ks + start, n);
      }
    }
    __syncthreads();
  }
}

int launch_grouping(const GroupArgs &g, int64_t capacity, int num_sms, cudaStream_t st,
                    int *launches) {
  const int64_t G = g.nb * g.nb;
  SPAMM_CUDA_TRY(cudaMemsetAsync(g.counts, 0, sizeof(uint32_t) * G, st));
  SPAMM_CUDA_TRY(cudaMemsetAsync(g.tile_status, 0,
                                 sizeof(unsigned long long) * ((G + GRP_TILE - 1) / GRP_TILE + 1),
                                 st));
  const int64_t want = (capacity + 255) / 256;
  const int grid = (int)std::min<int64_t>(std::max<int64_t>(want, 1), (int64_t)num_sms * 8);
  group_count_kernel<<<grid, 256, 0, st>>>(g);
  const int64_t tiles = (G + GRP_TILE - 1) / GRP_TILE;
  group_scan_kernel<<<(int)std::min<int64_t>(tiles, (int64_t)num_sms * 4), GRP_THREADS, 0, st>>>(g);
  group_scatter_kernel<<<grid, 256, 0, st>>>(g);
  group_sort_kernel<<<num_sms * 4, SORT_THREADS, 0, st>>>(g);
  SPAMM_CUDA_TRY(cudaGetLastError());
  if (launches) *launches += 4;
  return SPAMM_OK;
}

size_t group_tile_status_bytes(int64_t nb) {
  return sizeof(unsigned long long) * ((nb * nb + GRP_TILE - 1) / GRP_TILE + 1);
}

}  // namespace spamm
