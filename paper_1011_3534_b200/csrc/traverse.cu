// traverse.cu -- K2: the whole product-space traversal and the grouping of
// the retained leaf triples, in ONE cooperative persistent kernel.
//
// Reference: the breadth-first tier loop of spamm() (multiply.py:174-212)
// and the lexsort/grouping of _leaf_stage (multiply.py:231-234).
//
// Per tier t every candidate triple (i, j, k) is tested exactly like the
// reference:
//   alive  = occA[t][i,k] & occB[t][k,j]                         (:184)
//   np     = rn(rn(sqrt nsqA[t][i,k]) * rn(sqrt nsqB[t][k,j]))    (:185)
//            (the square roots are precomputed per tree node, bit-identical)
//   pruned = alive & (np < tau_t)        strict; ties are computed (:187)
//   active = alive & ~pruned
// and active triples expand to their 8 children in (di,dj,dk) = 000..111
// order (:207-212).  Candidates are never materialised: candidate c of tier
// t is child (c & 7) of survivor (c >> 3) of tier t-1 (survivors kept as
// packed (i, j, k), see common.cuh), so each tier's list stays in the
// reference's order and
// the pruned list (budget, boxes) comes out in exactly the reference's order.
//
// Phases of the kernel (grid barriers between them):
//   prefix  CTA 0 alone walks the first tiers while they are small (<= 8
//           tiles); the other CTAs meanwhile clear the grouping buckets.
//   tiers   every later tier: 1024-candidate tiles from a ticket, warp
//           ballots + block scan inside a tile, decoupled look-back across
//           tiles (order-preserving compaction of survivors and pruned calls)
//   budget  per tier, numpy's pairwise summation of the pruned products,
//           bit-for-bit (multiply.py:197), then summed in tier order
//   group   histogram of the leaf triples per C block, look-back scan of the
//           nb^2 buckets (offsets + the ascending list of non-empty blocks),
//           scatter of k, and a per-bucket bitonic sort -> the reference's
//           lexsorted (i, j, k) list, bucket by bucket.
#include <cuda/atomic>
#include <cstdlib>

#include "scan.cuh"
#include "traverse.cuh"

namespace spamm {

constexpr int TV_THREADS = 256;
constexpr int TV_ITEMS = 4;
constexpr int TV_TILE = TV_THREADS * TV_ITEMS;
constexpr unsigned long long PREFIX_MAX_CAND = 8 * TV_TILE;
constexpr int PW_NODES = 512;
constexpr int PW_SMEM_VALS = 4096;
constexpr int PREFIX_LIST = 1024;               // prefix survivor lists kept in smem
constexpr int SORT_WARP_KEYS = 512;             // per-warp shared sort buffer
constexpr int PREFIX_LEVELS = 5;                // pyramid levels 0..5 cached for the prefix
constexpr int PREFIX_ENTRIES = 1365;            // (4^6 - 1) / 3

struct TvShared {
  unsigned long long warp[TV_THREADS / 32];
  unsigned long long excl;
  unsigned long long tile;
  unsigned counts[2];                   // owned Empty skips, alive (per tile)
  unsigned long long run_act, run_prn;  // prefix: running offsets of the tier
  unsigned long long tier_cnt[4];       // prefix: active, pruned, skip, alive of the tier
  unsigned long long prev_active;       // prefix: survivors of the previous tier
  unsigned warp_item[TV_THREADS / 32];
  int pw_lvl[24];
  int pw_nlevels, pw_count;
  union {
    struct {  // prefix: the top of both pyramids + the small survivor lists
      double nrm_a[PREFIX_ENTRIES], nrm_b[PREFIX_ENTRIES];
      uint64_t list[2][PREFIX_LIST];
      uint8_t occ_a[PREFIX_ENTRIES], occ_b[PREFIX_ENTRIES];
    } top;
    struct {  // budget
      long long start[PW_NODES], len[PW_NODES];
      int left[PW_NODES];
      double val[PW_NODES];
      double vals[PW_SMEM_VALS];
    } pw;
    uint32_t keys[TV_THREADS / 32][SORT_WARP_KEYS];  // sort
  } u;
};

// ------------------------------------------------------------- grid barrier
__device__ void grid_sync(unsigned *bar, unsigned nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    cuda::atomic_ref<unsigned, cuda::thread_scope_device> cnt(bar[0]), gen(bar[1]);
    const unsigned g = gen.load(cuda::memory_order_acquire);
    __threadfence();
    if (cnt.fetch_add(1u, cuda::memory_order_acq_rel) == nblocks - 1) {
      cnt.store(0u, cuda::memory_order_relaxed);
      gen.fetch_add(1u, cuda::memory_order_release);
    } else {
      while (gen.load(cuda::memory_order_acquire) == g) __nanosleep(32);
    }
    __threadfence();
  }
  __syncthreads();
}

// ------------------------------------------------------------- one tile
// Classifies candidates [tile*TV_TILE, +TV_TILE) of `tier` and writes the
// survivors / pruned records at their order-preserving positions.  With
// `grid_mode` the tile's prefix comes from the look-back over `status`,
// otherwise from the running offsets of the single prefix CTA.
__device__ void process_tile(const TraverseArgs &a, TvShared &sh, int tier, unsigned long long tile,
                             unsigned long long n_cand, unsigned long long pruned_base,
                             bool grid_mode, unsigned long long *status) {
  TraverseCounters *tc = a.tc;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int shift = a.depth - tier;
  const int64_t side = int64_t(1) << tier;
  const int64_t loff = level_offset(tier);
  const uint64_t *prev = a.codes[(tier + 1) & 1];
  uint64_t *next = a.codes[tier & 1];
  const double tau = a.tau_tier[tier];
  const bool cached = !grid_mode && tier <= PREFIX_LEVELS;
  if (threadIdx.x < 2) sh.counts[threadIdx.x] = 0;

  uint64_t code[TV_ITEMS];
  double npv[TV_ITEMS];
  unsigned act_mask = 0, prn_mask = 0, n_skip = 0, n_alive = 0;
#pragma unroll
  for (int q = 0; q < TV_ITEMS; ++q) {
    const unsigned long long c = tile * TV_TILE + threadIdx.x * TV_ITEMS + q;
    code[q] = 0;
    npv[q] = 0.0;
    if (c < n_cand) {
      const uint64_t pc = tier == 0 ? 0ull : (!grid_mode ? sh.u.top.list[(tier + 1) & 1][c >> 3]
                                                         : prev[c >> 3]);
      const uint64_t cd = tier == 0 ? 0ull : child_triple(pc, (unsigned)(c & 7ull));
      code[q] = cd;
      uint32_t i, j, k;
      unpack_triple(cd, i, j, k);
      const int64_t r0 = int64_t(i) << shift, r1 = int64_t(i + 1) << shift;
      const bool intersects = r1 > a.row_lo && r0 < a.row_hi;
      const bool owned = r0 >= a.row_lo && r0 < a.row_hi;
      if (intersects) {
        const int64_t ik = loff + int64_t(i) * side + k, kj = loff + int64_t(k) * side + j;
        bool alive;
        double na, nb_;
        if (cached) {
          alive = sh.u.top.occ_a[ik] && sh.u.top.occ_b[kj];
          na = sh.u.top.nrm_a[ik];
          nb_ = sh.u.top.nrm_b[kj];
        } else {
          alive = a.occ_a[ik] && a.occ_b[kj];
          na = a.nrm_a[ik];
          nb_ = a.nrm_b[kj];
        }
        const double np_ = __dmul_rn(na, nb_);
        const bool pruned = alive && (np_ < tau);
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
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    n_skip += __shfl_xor_sync(0xffffffffu, n_skip, o);
    n_alive += __shfl_xor_sync(0xffffffffu, n_alive, o);
  }
  if (lane == 0) {
    atomicAdd(&sh.counts[0], n_skip);
    atomicAdd(&sh.counts[1], n_alive);
  }
  unsigned long long tile_total;
  const unsigned long long in_tile = block_exclusive<TV_THREADS>(
      pack2(__popc(act_mask), __popc(prn_mask)), sh.warp, &tile_total);
  if (warp == 0) {
    unsigned long long excl;
    if (grid_mode) {
      excl = lookback_exclusive(status, tile, tile_total);
    } else {
      excl = pack2((unsigned)sh.run_act, (unsigned)sh.run_prn);
    }
    if (lane == 0) {
      sh.excl = excl;
      if (!grid_mode) {
        sh.run_act += unpack_a(tile_total);
        sh.run_prn += unpack_b(tile_total);
        sh.tier_cnt[0] += unpack_a(tile_total);
        sh.tier_cnt[1] += unpack_b(tile_total);
        sh.tier_cnt[2] += sh.counts[0];
        sh.tier_cnt[3] += sh.counts[1];
      } else {
        atomicAdd(&tc->n_active[tier], (unsigned long long)unpack_a(tile_total));
        atomicAdd(&tc->n_pruned[tier], (unsigned long long)unpack_b(tile_total));
        atomicAdd(&tc->n_skip[tier], (unsigned long long)sh.counts[0]);
        atomicAdd(&tc->n_alive[tier], (unsigned long long)sh.counts[1]);
      }
    }
  }
  __syncthreads();
  const unsigned long long base = sh.excl + in_tile;
  unsigned a_pos = unpack_a(base), p_pos = unpack_b(base);
#pragma unroll
  for (int q = 0; q < TV_ITEMS; ++q) {
    if (act_mask & (1u << q)) {
      if (a_pos < a.capacity) next[a_pos] = code[q];
      else tc->overflow = 1;
      if (!grid_mode && a_pos < PREFIX_LIST) sh.u.top.list[tier & 1][a_pos] = code[q];
      ++a_pos;
    }
    if (prn_mask & (1u << q)) {
      const unsigned long long dst = pruned_base + p_pos;
      if (dst < a.pruned_capacity) {
        a.pruned_vals[dst] = npv[q];
        a.pruned_codes[dst] = code[q];
      } else {
        tc->overflow = 1;
      }
      ++p_pos;
    }
  }
  __syncthreads();
}

__device__ __forceinline__ unsigned long long tier_candidates(const TraverseArgs &a, int tier) {
  if (tier == 0) return 1;
  unsigned long long np_ = a.tc->n_active[tier - 1];
  if (np_ > a.capacity) np_ = a.capacity;
  return 8ull * np_;
}

// ------------------------------------------------------- pairwise budget
// numpy's pairwise summation for float64: n < 8 sequential from 0.0; n <= 128
// eight interleaved accumulators combined ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7))
// plus a sequential tail; else split at n/2 rounded down to a multiple of 8.
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
#pragma unroll 4
  for (; i < n - (n % 8); i += 8) {
#pragma unroll
    for (int q = 0; q < 8; ++q) r[q] = __dadd_rn(r[q], a[i + q]);
  }
  double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                         __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
  for (; i < n; ++i) res = __dadd_rn(res, a[i]);
  return res;
}

__device__ double pw_serial(const double *a, long long n) {
  if (n <= 128) return pw_block(a, n);
  long long st_s[48], st_n[48];
  int st_state[48];
  double st_left[48];
  int sp = 1;
  st_s[0] = 0;
  st_n[0] = n;
  st_state[0] = 0;
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

// One CTA: the recursion expanded breadth-first to <= PW_NODES nodes, the
// frontier summed in parallel, the tree folded back level by level.
__device__ double pairwise_cta(TvShared &sh, const double *a, long long n) {
  if (threadIdx.x == 0) {
    sh.u.pw.start[0] = 0;
    sh.u.pw.len[0] = n;
    sh.u.pw.left[0] = -1;
    int count = 1, lb = 0, le = 1, nl = 0;
    sh.pw_lvl[nl++] = 0;
    for (;;) {
      int add = 0;
      for (int x = lb; x < le; ++x) add += sh.u.pw.len[x] > 128 ? 2 : 0;
      if (add == 0 || count + add > PW_NODES || nl >= 22) break;
      for (int x = lb; x < le; ++x) {
        if (sh.u.pw.len[x] > 128) {
          long long n2 = sh.u.pw.len[x] / 2;
          n2 -= n2 % 8;
          sh.u.pw.left[x] = count;
          sh.u.pw.start[count] = sh.u.pw.start[x]; sh.u.pw.len[count] = n2; sh.u.pw.left[count] = -1; ++count;
          sh.u.pw.start[count] = sh.u.pw.start[x] + n2; sh.u.pw.len[count] = sh.u.pw.len[x] - n2;
          sh.u.pw.left[count] = -1; ++count;
        }
      }
      lb = le;
      le = count;
      sh.pw_lvl[nl++] = lb;
    }
    sh.pw_lvl[nl] = count;
    sh.pw_nlevels = nl;
    sh.pw_count = count;
  }
  __syncthreads();
  const int count = sh.pw_count;
  for (int x = threadIdx.x; x < count; x += TV_THREADS)
    if (sh.u.pw.left[x] < 0) sh.u.pw.val[x] = pw_serial(a + sh.u.pw.start[x], sh.u.pw.len[x]);
  __syncthreads();
  for (int l = sh.pw_nlevels - 1; l >= 0; --l) {
    for (int x = sh.pw_lvl[l] + threadIdx.x; x < sh.pw_lvl[l + 1]; x += TV_THREADS)
      if (sh.u.pw.left[x] >= 0) sh.u.pw.val[x] = __dadd_rn(sh.u.pw.val[sh.u.pw.left[x]], sh.u.pw.val[sh.u.pw.left[x] + 1]);
    __syncthreads();
  }
  const double r = sh.u.pw.val[0];
  __syncthreads();
  return r;
}

// All-ascending bitonic network (min to the lower index at every comparator;
// the first step of each merge compares mirror positions), so +inf padding
// past n never moves into the real range.  Distinct keys -> unique result.
__device__ __forceinline__ void warp_sort32(uint32_t &v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      const int p = (j == (k >> 1)) ? (lane ^ (k - 1)) : (lane ^ j);
      const uint32_t o = __shfl_sync(0xffffffffu, v, p);
      v = p > lane ? min(v, o) : max(v, o);
    }
  }
}

__device__ void warp_bitonic(uint32_t *x, int n) {
  const int lane = threadIdx.x & 31;
  int P = 1;
  while (P < n) P <<= 1;
  for (int k = 2; k <= P; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = lane; i < P; i += 32) {
        const int p = (j == (k >> 1)) ? (i ^ (k - 1)) : (i ^ j);
        if (p > i && p < n) {
          const uint32_t u = x[i], v = x[p];
          if (u > v) {
            x[i] = v;
            x[p] = u;
          }
        }
      }
      __syncwarp();
      __threadfence_block();
    }
  }
}

__device__ void clear_status_part(unsigned long long *st, unsigned long long n, unsigned part,
                                  unsigned parts) {
  for (unsigned long long i = (unsigned long long)part * TV_THREADS + threadIdx.x; i < n;
       i += (unsigned long long)parts * TV_THREADS)
    st[i] = 0ull;
}

__device__ void clear_status(unsigned long long *st, unsigned long long n) {
  for (unsigned long long i = (unsigned long long)blockIdx.x * TV_THREADS + threadIdx.x; i < n;
       i += (unsigned long long)gridDim.x * TV_THREADS)
    st[i] = 0ull;
}

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define PHASE(ix) \
  if (blockIdx.x == 0 && threadIdx.x == 0) tc->phase_ns[ix] = globaltimer();

// ================================================================= kernel
__global__ void __launch_bounds__(TV_THREADS) traverse_kernel(TraverseArgs a) {
  __shared__ TvShared sh;
  TraverseCounters *tc = a.tc;
  const unsigned nblocks = gridDim.x;
  const int depth = a.depth;
  const int64_t G = a.nb * a.nb;

  // ---------------- prefix (CTA 0) || clear the buckets (other CTAs)
  if (blockIdx.x == 0) {
    const unsigned long long t_entry = globaltimer();
    for (int x = threadIdx.x; x < (int)(sizeof(TraverseCounters) / 8); x += TV_THREADS)
      reinterpret_cast<unsigned long long *>(tc)[x] = 0ull;
    __syncthreads();
    if (threadIdx.x == 0) tc->phase_ns[15] = t_entry;
    // one parallel load of the pyramid tops; the prefix tiers then hit smem
    const int top_entries = (int)level_offset((depth < PREFIX_LEVELS ? depth : PREFIX_LEVELS) + 1);
    for (int x = threadIdx.x; x < top_entries; x += TV_THREADS) {
      sh.u.top.nrm_a[x] = a.nrm_a[x];
      sh.u.top.nrm_b[x] = a.nrm_b[x];
      sh.u.top.occ_a[x] = a.occ_a[x];
      sh.u.top.occ_b[x] = a.occ_b[x];
    }
    if (threadIdx.x == 0) sh.prev_active = 0;
    __syncthreads();
    PHASE(0)
    int t = 0;
    unsigned long long pbase = 0;
    for (; t <= depth; ++t) {
      unsigned long long n_cand = 1;
      if (t > 0) n_cand = 8ull * (sh.prev_active < a.capacity ? sh.prev_active : a.capacity);
      // the prefix serialises tiles on one CTA: only worth it while the
      // pyramid level is cached in shared memory and the tier is small
      if (t > PREFIX_LEVELS || n_cand > PREFIX_MAX_CAND || (t > 0 && sh.prev_active > PREFIX_LIST))
        break;
      if (threadIdx.x == 0) {
        sh.run_act = sh.run_prn = 0;
        sh.tier_cnt[0] = sh.tier_cnt[1] = sh.tier_cnt[2] = sh.tier_cnt[3] = 0;
      }
      __syncthreads();
      const unsigned long long tiles = (n_cand + TV_TILE - 1) / TV_TILE;
      for (unsigned long long tile = 0; tile < tiles; ++tile)
        process_tile(a, sh, t, tile, n_cand, pbase, false, nullptr);
      if (threadIdx.x == 0) {
        tc->pruned_base[t] = pbase;
        tc->n_cand[t] = n_cand;
        tc->n_active[t] = sh.tier_cnt[0];
        tc->n_pruned[t] = sh.tier_cnt[1];
        tc->n_skip[t] = sh.tier_cnt[2];
        tc->n_alive[t] = sh.tier_cnt[3];
        sh.prev_active = sh.tier_cnt[0];
      }
      pbase += sh.tier_cnt[1];
      __syncthreads();
    }
    if (threadIdx.x == 0) tc->first_grid_tier = t;
    PHASE(1)
  } else {
    for (int64_t x = (int64_t)(blockIdx.x - 1) * TV_THREADS + threadIdx.x; x < G;
         x += (int64_t)(nblocks - 1) * TV_THREADS)
      a.counts[x] = 0u;
  }
  grid_sync(a.barrier, nblocks);
  PHASE(2)

  // ---------------- grid-wide tiers
  const int t0 = tc->first_grid_tier;
  unsigned long long prev_tiles = 0;
  for (int t = t0; t <= depth; ++t) {
    const unsigned long long n_cand = tier_candidates(a, t);
    const unsigned long long pbase = t == 0 ? 0ull : tc->pruned_base[t - 1] + tc->n_pruned[t - 1];
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      tc->pruned_base[t] = pbase;
      tc->n_cand[t] = n_cand;
    }
    // the other status array was used by tier t-1 and is reused by t+1
    if (t > t0) clear_status(a.status[(t + 1) & 1], prev_tiles);
    const unsigned long long tiles = (n_cand + TV_TILE - 1) / TV_TILE;
    for (;;) {
      if (threadIdx.x == 0) sh.tile = atomicAdd(&tc->ticket[t], 1ull);
      __syncthreads();
      const unsigned long long tile = sh.tile;
      __syncthreads();
      if (tile >= tiles) break;
      process_tile(a, sh, t, tile, n_cand, pbase, true, a.status[t & 1]);
    }
    prev_tiles = tiles;
    grid_sync(a.barrier, nblocks);
    PHASE(3 + (t - t0 < 5 ? t - t0 : 4))
  }
  if (blockIdx.x == 0 && threadIdx.x == 0 && depth >= t0)
    tc->dirty_tiles[depth & 1] = prev_tiles;

  unsigned long long m = tc->n_active[depth];
  if (m > a.capacity) m = a.capacity;
  const uint64_t *leaf_codes = a.codes[depth & 1];
  const int nbud = depth + 1;  // CTAs 0..depth compute the budget, then leave

  // ---------------- omitted_budget: one CTA per tier, concurrent with the
  // grouping below (those CTAs never meet the later barriers); the last tier
  // to finish adds the tier sums in tier order, as the reference's Python
  // float does.
  if ((int)blockIdx.x < nbud) {
    const int t = blockIdx.x;
    const unsigned long long np_ = tc->n_pruned[t];
    double s = 0.0;
    if (np_ && tc->pruned_base[t] + np_ <= a.pruned_capacity) {
      const double *src = a.pruned_vals + tc->pruned_base[t];
      if (np_ <= PW_SMEM_VALS) {
        for (unsigned x = threadIdx.x; x < np_; x += TV_THREADS) sh.u.pw.vals[x] = src[x];
        __syncthreads();
        src = sh.u.pw.vals;
      }
      s = pairwise_cta(sh, src, (long long)np_);
    }
    if (threadIdx.x == 0) {
      tc->tier_budget[t] = s;
      __threadfence();
      if (atomicAdd(&tc->budgets_done, 1u) == (unsigned)depth) {
        __threadfence();
        tc->phase_ns[12] = globaltimer();
        double b = 0.0;
        for (int u = 0; u <= depth; ++u)
          if (tc->n_pruned[u]) b = __dadd_rn(b, ((volatile double *)tc->tier_budget)[u]);
        tc->budget = b;
      }
      atomicMax(&tc->phase_ns[13], globaltimer());
    }
    return;
  }
  const unsigned gi = blockIdx.x - nbud, gn = nblocks - nbud;  // grouping CTAs
#define GPHASE(ix) \
  if (gi == 0 && threadIdx.x == 0) tc->phase_ns[ix] = globaltimer();

  // ---------------- bucket histogram
  for (unsigned long long p = (unsigned long long)gi * TV_THREADS + threadIdx.x; p < m;
       p += (unsigned long long)gn * TV_THREADS) {
    uint32_t i, j, k;
    unpack_triple(leaf_codes[p], i, j, k);
    atomicAdd(&a.counts[int64_t(i) * a.nb + j], 1u);
  }
  grid_sync(a.barrier, gn);
  GPHASE(8)

  // ---------------- bucket scan: offsets + non-empty block list
  {
    const unsigned long long tiles = (G + TV_TILE - 1) / TV_TILE;
    for (;;) {
      if (threadIdx.x == 0) sh.tile = atomicAdd(&tc->scan_ticket, 1ull);
      __syncthreads();
      const unsigned long long tile = sh.tile;
      __syncthreads();
      if (tile >= tiles) break;
      const int64_t base = (int64_t)tile * TV_TILE + threadIdx.x * TV_ITEMS;
      unsigned cnt[TV_ITEMS], sum = 0, ne = 0;
#pragma unroll
      for (int q = 0; q < TV_ITEMS; ++q) {
        cnt[q] = base + q < G ? a.counts[base + q] : 0u;
        sum += cnt[q];
        ne += cnt[q] != 0;
      }
      unsigned long long total;
      const unsigned long long in_tile = block_exclusive<TV_THREADS>(pack2(sum, ne), sh.warp, &total);
      if ((threadIdx.x >> 5) == 0) {
        const unsigned long long excl = lookback_exclusive(a.status[2], tile, total);
        if ((threadIdx.x & 31) == 0) {
          sh.excl = excl;
          atomicAdd(&tc->num_groups, unpack_b(total));
        }
      }
      __syncthreads();
      const unsigned long long pre = sh.excl + in_tile;
      unsigned off = unpack_a(pre), slot = unpack_b(pre);
#pragma unroll
      for (int q = 0; q < TV_ITEMS; ++q) {
        if (base + q < G) {
          a.offsets[base + q] = off;
          if (cnt[q]) {
            a.group_ids[slot] = (uint32_t)(base + q);
            a.group_starts[slot] = off;
            ++slot;
          }
          off += cnt[q];
        }
      }
      __syncthreads();
    }
  }
  grid_sync(a.barrier, gn);
  GPHASE(9)

  // ---------------- scatter k into the buckets; clear look-back state
  for (unsigned long long p = (unsigned long long)gi * TV_THREADS + threadIdx.x; p < m;
       p += (unsigned long long)gn * TV_THREADS) {
    uint32_t i, j, k;
    unpack_triple(leaf_codes[p], i, j, k);
    const int64_t gid = int64_t(i) * a.nb + j;
    const unsigned slot = atomicSub(&a.counts[gid], 1u) - 1u;
    a.ks[a.offsets[gid] + slot] = k;
  }
  // (tier depth-1's status array was already cleared during tier depth)
  if (depth >= t0) clear_status_part(a.status[depth & 1], tc->dirty_tiles[depth & 1], gi, gn);
  clear_status_part(a.status[2], (G + TV_TILE - 1) / TV_TILE, gi, gn);
  grid_sync(a.barrier, gn);
  GPHASE(10)

  // ---------------- sort every bucket's k list ascending (one warp per bucket)
  {
    const unsigned ng = tc->num_groups;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint32_t *wkeys = sh.u.keys[wid];
    for (;;) {
      unsigned q = 0;
      if (lane == 0) q = (unsigned)atomicAdd(&tc->sort_ticket, 1ull);
      q = __shfl_sync(0xffffffffu, q, 0);
      if (q >= ng) break;
      const unsigned start = a.group_starts[q];
      const unsigned end = q + 1 < ng ? a.group_starts[q + 1] : (unsigned)m;
      const int n = (int)(end - start);
      if (n <= 1) continue;
      if (n <= 32) {
        uint32_t v = lane < n ? a.ks[start + lane] : 0xffffffffu;
        warp_sort32(v);
        if (lane < n) a.ks[start + lane] = v;
      } else if (n <= SORT_WARP_KEYS) {
        for (int e = lane; e < n; e += 32) wkeys[e] = a.ks[start + e];
        __syncwarp();
        warp_bitonic(wkeys, n);
        for (int e = lane; e < n; e += 32) a.ks[start + e] = wkeys[e];
        __syncwarp();
      } else {
        warp_bitonic(a.ks + start, n);
      }
    }
  }
  GPHASE(11)
  if (threadIdx.x == 0) atomicMax(&tc->phase_ns[13], globaltimer());  // last CTA out
#undef GPHASE
}

int launch_traverse(const TraverseArgs &args, int num_sms, cudaStream_t st) {
  static int per_sm = 0;
  if (per_sm == 0) {
    // every library kernel asks for the maximum shared-memory carveout, so
    // consecutive launches never pay for an L1/shared reconfiguration
    SPAMM_CUDA_TRY(cudaFuncSetAttribute(traverse_kernel,
                                        cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    SPAMM_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, traverse_kernel,
                                                                 TV_THREADS, 0));
    if (per_sm < 1) {
      set_error("traverse kernel cannot be resident");
      return SPAMM_ERR_INTERNAL;
    }
  }
  const int grid = num_sms * (per_sm < 2 ? per_sm : 2);
  void *kargs[] = {(void *)&args};
  SPAMM_CUDA_TRY(cudaLaunchCooperativeKernel((const void *)traverse_kernel, grid, TV_THREADS,
                                             kargs, 0, st));
  return SPAMM_OK;
}

size_t traverse_status_entries(size_t capacity) { return (8 * capacity + TV_TILE - 1) / TV_TILE + 2; }
size_t group_status_entries(int64_t nb) { return (size_t)((nb * nb + TV_TILE - 1) / TV_TILE + 2); }

}  // namespace spamm
