// cull.cu -- K2: level-synchronous product-space culling.
//
// Reference: the breadth-first tier loop of spamm(), multiply.py:174-212.
// Per tier t every candidate triple (i, j, k) is tested:
//   alive  = occA[t][i,k] & occB[t][k,j]                         (:184)
//   np     = rn(rn(sqrt nsqA[t][i,k]) * rn(sqrt nsqB[t][k,j]))    (:185)
//   pruned = alive & (np < tau_t)        strict; ties are computed (:187)
//   active = alive & ~pruned
// and active triples expand to their 8 children in (di,dj,dk) = 000..111
// order (:207-212).  Candidates are never materialised: candidate c of tier
// t is child (c & 7) of survivor (c >> 3) of tier t-1, each survivor kept as
// its Morton code, so every tier's list stays in the reference's order.
//
// One persistent kernel per tier: CTAs take 1024-candidate tiles from a
// device ticket, classify them, and compact the active codes (next tier's
// parents) and the pruned norm products / codes (budget and boxes) with an
// order-preserving single-pass scan: warp ballots/prefix sums inside the
// tile, decoupled look-back across tiles.  Counts stay on the device, so a
// whole traversal is launched without a host round trip.
#include "cull.cuh"
#include "scan.cuh"

namespace spamm {

constexpr int CULL_THREADS = 256;
constexpr int CULL_ITEMS = 4;
constexpr int CULL_TILE = CULL_THREADS * CULL_ITEMS;

__global__ void __launch_bounds__(CULL_THREADS) cull_tier_kernel(CullTierArgs args) {
  __shared__ unsigned long long s_warp[CULL_THREADS / 32];
  __shared__ unsigned long long s_excl;
  __shared__ unsigned long long s_tile;
  __shared__ unsigned s_counts[2];  // owned Empty skips, alive
  CullCounters *cc = args.counters;
  const int tier = args.tier;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;

  // parents = survivors of the previous tier (clamped to the buffer capacity;
  // an overflow is flagged there and the host re-runs with more room)
  unsigned long long n_cand;
  if (tier == 0) {
    n_cand = 1;
  } else {
    unsigned long long np_ = cc->n_active[tier - 1];
    if (np_ > args.capacity) np_ = args.capacity;
    n_cand = 8ull * np_;
  }
  const unsigned long long n_tiles = (n_cand + CULL_TILE - 1) / CULL_TILE;
  const unsigned long long pruned_base =
      tier == 0 ? 0ull : cc->pruned_base[tier - 1] + cc->n_pruned[tier - 1];
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    cc->pruned_base[tier] = pruned_base;
    cc->n_cand[tier] = n_cand;
  }
  const int shift = args.depth - tier;  // leaf rows per tier-t block row = 1 << shift
  const int64_t side = int64_t(1) << tier;

  for (;;) {
    if (threadIdx.x == 0) s_tile = atomicAdd(&cc->ticket[tier], 1ull);
    if (threadIdx.x < 2) s_counts[threadIdx.x] = 0;
    __syncthreads();
    const unsigned long long tile = s_tile;
    if (tile >= n_tiles) break;

    uint64_t code[CULL_ITEMS];
    double npv[CULL_ITEMS];
    unsigned act_mask = 0, prn_mask = 0, n_skip = 0, n_alive = 0;
#pragma unroll
    for (int q = 0; q < CULL_ITEMS; ++q) {
      const unsigned long long c = tile * CULL_TILE + threadIdx.x * CULL_ITEMS + q;
      code[q] = 0;
      npv[q] = 0.0;
      if (c < n_cand) {
        const uint64_t cd = tier == 0 ? 0ull : args.prev[c >> 3] * 8ull + (c & 7ull);
        code[q] = cd;
        uint32_t i, j, k;
        morton_decode(cd, i, j, k);
        const int64_t r0 = int64_t(i) << shift, r1 = int64_t(i + 1) << shift;
        const bool intersects = r1 > args.row_lo && r0 < args.row_hi;
        const bool owned = r0 >= args.row_lo && r0 < args.row_hi;
        if (intersects) {
          const int64_t ik = int64_t(i) * side + k, kj = int64_t(k) * side + j;
          const bool alive = args.occ_a[ik] && args.occ_b[kj];
          const double np_ = __dmul_rn(__dsqrt_rn(args.nsq_a[ik]), __dsqrt_rn(args.nsq_b[kj]));
          const bool pruned = alive && (np_ < args.tau);
          n_alive += alive;
          if (alive && !pruned) act_mask |= 1u << q;
          if (pruned && owned) {
            prn_mask |= 1u << q;
            npv[q] = np_;
          }
          if (!alive && owned) ++n_skip;
        }
      }
    }
    // integer stats: order independent
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      n_skip += __shfl_xor_sync(0xffffffffu, n_skip, o);
      n_alive += __shfl_xor_sync(0xffffffffu, n_alive, o);
    }
    if (lane == 0) {
      atomicAdd(&s_counts[0], n_skip);
      atomicAdd(&s_counts[1], n_alive);
    }
    // order-preserving compaction offsets of (active, pruned) within the tile
    unsigned long long tile_total;
    const unsigned long long in_tile =
        block_exclusive<CULL_THREADS>(pack2(__popc(act_mask), __popc(prn_mask)), s_warp,
                                      &tile_total);
    if (warp == 0) {
      const unsigned long long excl = lookback_exclusive(args.tile_status, tile, tile_total);
      if (lane == 0) {
        s_excl = excl;
        atomicAdd(&cc->n_active[tier], (unsigned long long)unpack_a(tile_total));
        atomicAdd(&cc->n_pruned[tier], (unsigned long long)unpack_b(tile_total));
        atomicAdd(&cc->n_skip[tier], (unsigned long long)s_counts[0]);
        atomicAdd(&cc->n_alive[tier], (unsigned long long)s_counts[1]);
      }
    }
    __syncthreads();
    const unsigned long long base = s_excl + in_tile;
    unsigned a_pos = unpack_a(base), p_pos = unpack_b(base);
#pragma unroll
    for (int q = 0; q < CULL_ITEMS; ++q) {
      if (act_mask & (1u << q)) {
        if (a_pos < args.capacity) args.next[a_pos] = code[q];
        else cc->overflow = 1;
        ++a_pos;
      }
      if (prn_mask & (1u << q)) {
        const unsigned long long dst = pruned_base + p_pos;
        if (dst < args.pruned_capacity) {
          args.pruned_vals[dst] = npv[q];
          args.pruned_codes[dst] = code[q];
        } else {
          cc->overflow = 1;
        }
        ++p_pos;
      }
    }
    __syncthreads();
  }
}

// --------------------------------------------------------------------------
// omitted_budget: numpy's pairwise summation, bit for bit.
//
// The reference adds `float(norm_prod[pruned].sum())` per tier
// (multiply.py:197); numpy sums a contiguous float64 array by pairwise
// recursion: n < 8 -> sequential from 0.0; n <= 128 -> eight interleaved
// accumulators combined ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) plus a
// sequential tail; else split at n2 = n/2 rounded down to a multiple of 8.
// One CTA per tier expands the recursion breadth-first to <= 1024 frontier
// nodes, each thread sums one frontier node with the same recursion, and the
// tree is folded back level by level.  The tier sums are then added in tier
// order, as the reference's Python float accumulation does.
__device__ double pw_block(const double *a, long long n) {
  if (n < 8) {
    double r = 0.0;
    for (long long i = 0; i < n; ++i) r = __dadd_rn(r, a[i]);
    return r;
  }
  double r[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) r[q] = a[q];
  long long i = 8;
  for (; i < n - (n % 8); i += 8) {
#pragma unroll
    for (int q = 0; q < 8; ++q) r[q] = __dadd_rn(r[q], a[i + q]);
  }
  double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                         __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
  for (; i < n; ++i) res = __dadd_rn(res, a[i]);
  return res;
}

// Sequential evaluation of the recursion for one subtree (explicit stack).
__device__ double pw_serial(const double *a, long long n) {
  if (n <= 128) return pw_block(a, n);
  // post-order traversal; the stack holds (start, len, state, left value)
  long long st_s[48], st_n[48];
  int st_state[48];
  double st_left[48];
  int sp = 0;
  st_s[0] = 0; st_n[0] = n; st_state[0] = 0; sp = 1;
  double ret = 0.0;
  while (sp) {
    const int top = sp - 1;
    const long long s = st_s[top], m = st_n[top];
    if (m <= 128) {
      ret = pw_block(a + s, m);
      --sp;
      continue;
    }
    long long n2 = m / 2;
    n2 -= n2 % 8;
    if (st_state[top] == 0) {
      st_state[top] = 1;
      st_s[sp] = s; st_n[sp] = n2; st_state[sp] = 0; ++sp;
    } else if (st_state[top] == 1) {
      st_left[top] = ret;
      st_state[top] = 2;
      st_s[sp] = s + n2; st_n[sp] = m - n2; st_state[sp] = 0; ++sp;
    } else {
      ret = __dadd_rn(st_left[top], ret);
      --sp;
    }
  }
  return ret;
}

constexpr int PW_THREADS = 1024;
constexpr int PW_NODES = 1024;

__global__ void __launch_bounds__(PW_THREADS) tier_budget_kernel(const double *__restrict__ vals,
                                                                 CullCounters *cc) {
  __shared__ long long s_start[PW_NODES], s_len[PW_NODES];
  __shared__ int s_left[PW_NODES];
  __shared__ double s_val[PW_NODES];
  __shared__ int s_lvl_begin[24];
  __shared__ int s_nlevels, s_count;
  const int tier = blockIdx.x;
  const unsigned long long n = cc->n_pruned[tier];
  const double *a = vals + cc->pruned_base[tier];
  if (n == 0) {
    if (threadIdx.x == 0) cc->tier_budget[tier] = 0.0;
    return;
  }
  if (threadIdx.x == 0) {
    // breadth-first expansion of the recursion
    s_start[0] = 0; s_len[0] = (long long)n; s_left[0] = -1;
    int count = 1, lb = 0, le = 1, nl = 0;
    s_lvl_begin[nl++] = 0;
    for (;;) {
      int add = 0;
      for (int x = lb; x < le; ++x) add += s_len[x] > 128 ? 2 : 0;
      if (add == 0 || count + add > PW_NODES || add > PW_THREADS || nl >= 23) break;
      for (int x = lb; x < le; ++x) {
        if (s_len[x] > 128) {
          long long n2 = s_len[x] / 2;
          n2 -= n2 % 8;
          s_left[x] = count;
          s_start[count] = s_start[x]; s_len[count] = n2; s_left[count] = -1; ++count;
          s_start[count] = s_start[x] + n2; s_len[count] = s_len[x] - n2; s_left[count] = -1; ++count;
        }
      }
      lb = le; le = count;
      s_lvl_begin[nl++] = lb;
    }
    s_lvl_begin[nl] = count;
    s_nlevels = nl;
    s_count = count;
  }
  __syncthreads();
  const int count = s_count;
  // frontier nodes (no children) evaluated in parallel
  for (int x = threadIdx.x; x < count; x += PW_THREADS)
    if (s_left[x] < 0) s_val[x] = pw_serial(a + s_start[x], s_len[x]);
  __syncthreads();
  // fold internal nodes bottom-up, one level at a time
  for (int l = s_nlevels - 1; l >= 0; --l) {
    for (int x = s_lvl_begin[l] + threadIdx.x; x < s_lvl_begin[l + 1]; x += PW_THREADS)
      if (s_left[x] >= 0) s_val[x] = __dadd_rn(s_val[s_left[x]], s_val[s_left[x] + 1]);
    __syncthreads();
  }
  if (threadIdx.x == 0) cc->tier_budget[tier] = s_val[0];
}

__global__ void budget_total_kernel(CullCounters *cc, int tiers) {
  double b = 0.0;
  for (int t = 0; t < tiers; ++t)
    if (cc->n_pruned[t]) b = __dadd_rn(b, cc->tier_budget[t]);
  cc->budget = b;
}

int launch_cull(const CullPlan &plan, cudaStream_t st) {
  CullTierArgs args{};
  args.counters = plan.counters;
  args.tile_status = plan.tile_status;
  args.capacity = plan.capacity;
  args.pruned_capacity = plan.pruned_capacity;
  args.pruned_vals = plan.pruned_vals;
  args.pruned_codes = plan.pruned_codes;
  args.depth = plan.depth;
  args.row_lo = plan.row_lo;
  args.row_hi = plan.row_hi;
  SPAMM_CUDA_TRY(cudaMemsetAsync(plan.counters, 0, sizeof(CullCounters), st));
  for (int t = 0; t <= plan.depth; ++t) {
    args.tier = t;
    args.tau = plan.tau_tier[t];
    args.nsq_a = plan.nsq_a + level_offset(t);
    args.occ_a = plan.occ_a + level_offset(t);
    args.nsq_b = plan.nsq_b + level_offset(t);
    args.occ_b = plan.occ_b + level_offset(t);
    args.prev = plan.codes[(t + 1) & 1];
    args.next = plan.codes[t & 1];
    // tiles this tier can have at most
    unsigned long long max_cand = 1;
    for (int q = 0; q < t && max_cand < (1ull << 40); ++q) max_cand *= 8;
    if (t > 0 && max_cand > 8ull * plan.capacity) max_cand = 8ull * plan.capacity;
    const unsigned long long max_tiles = (max_cand + CULL_TILE - 1) / CULL_TILE;
    SPAMM_CUDA_TRY(cudaMemsetAsync(plan.tile_status, 0, sizeof(unsigned long long) * max_tiles, st));
    unsigned grid = (unsigned)(max_tiles < (unsigned long long)plan.max_ctas ? max_tiles
                                                                             : plan.max_ctas);
    if (grid == 0) grid = 1;
    cull_tier_kernel<<<grid, CULL_THREADS, 0, st>>>(args);
    SPAMM_CUDA_TRY(cudaGetLastError());
    if (plan.launches) ++*plan.launches;
  }
  tier_budget_kernel<<<plan.depth + 1, PW_THREADS, 0, st>>>(plan.pruned_vals, plan.counters);
  budget_total_kernel<<<1, 1, 0, st>>>(plan.counters, plan.depth + 1);
  SPAMM_CUDA_TRY(cudaGetLastError());
  if (plan.launches) *plan.launches += 2;
  return SPAMM_OK;
}

size_t tile_status_bytes(size_t capacity) {
  return sizeof(unsigned long long) * ((8 * capacity + CULL_TILE - 1) / CULL_TILE + 2);
}

}  // namespace spamm
