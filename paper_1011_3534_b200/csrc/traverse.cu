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
  union {
    struct {  // prefix: the top of both pyramids + the small survivor lists
      double nrm_a[PREFIX_ENTRIES], nrm_b[PREFIX_ENTRIES];
      uint64_t list[2][PREFIX_LIST];
      uint8_t occ_a[PREFIX_ENTRIES], occ_b[PREFIX_ENTRIES];
    } top;
    struct {  // budget: the values, then numpy's recursion tree (heap order)
      double vals[PW_SMEM_VALS];
      double val[2 * PW_NODES];
      uint8_t split[2 * PW_NODES];
    } pw;
    uint32_t keys[TV_THREADS / 32][SORT_WARP_KEYS];  // sort
    uint16_t qks[16384];                              // dense grouping: a tile's k lists
  } u;
};

// ------------------------------------------------------------- grid barrier
// One arrival counter per barrier group, zero at the start of the call (it
// lives in the call's counter set, cleared by the previous call) and never
// reset: the k-th barrier of a group of n CTAs completes when the counter
// reaches k*n.  One release-add per CTA, relaxed polling of the same word
// and one acquire fence (measured ~1.2 us on B200 for 296 CTAs vs 2.5 us for
// a count + generation pair with full fences; tools/gridsync_probe.cu).
__device__ void grid_sync(unsigned *ctr, unsigned nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned old;
    asm volatile("atom.add.release.gpu.u32 %0, [%1], 1;" : "=r"(old) : "l"(ctr) : "memory");
    const unsigned target = (old / nblocks + 1) * nblocks;
    unsigned cur;
    for (;;) {  // relaxed polling (an acquire per poll would invalidate L1 each time),
                // backed off so waiting CTAs do not flood the counter's L2 slice
      asm volatile("ld.relaxed.gpu.u32 %0, [%1];" : "=r"(cur) : "l"(ctr) : "memory");
      if (cur >= target) break;
      __nanosleep(100);
    }
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
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

// Copy n doubles global -> shared, eight loads in flight per thread.
template <int NT>
__device__ __forceinline__ void stage_values(double *dst, const double *__restrict__ src,
                                             unsigned long long n) {
  for (unsigned long long x0 = threadIdx.x; x0 < n; x0 += 8ull * NT) {
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const unsigned long long x = x0 + (unsigned long long)u * NT;
      v[u] = x < n ? __ldcg(src + x) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const unsigned long long x = x0 + (unsigned long long)u * NT;
      if (x < n) dst[x] = v[u];
    }
  }
}

// One CTA: numpy's recursion tree, PW_LOG levels deep at most, built in
// parallel -- thread p follows the left/right path spelled by its bits, the
// first thread under each node records whether the node splits (n > 128)
// and the leaves are summed serially (numpy's 8-accumulator blocks) -- then
// folded back level by level, left + right, exactly as the recursion adds.
constexpr int PW_LOG = 9;  // 2^PW_LOG = PW_NODES leaves at most
__device__ double pairwise_cta(TvShared &sh, const double *a, long long n) {
  int L = 0;
  for (long long m = n; m > 128 && L < PW_LOG; m = (m + 1) / 2) ++L;
  const int paths = 1 << L;
  for (int p = threadIdx.x; p < paths; p += TV_THREADS) {
    long long st = 0, len = n;
    int d = 0;
    for (; d < L && len > 128; ++d) {
      sh.u.pw.split[(1 << d) - 1 + (p >> (L - d))] = 1;  // every thread below writes the same 1
      long long n2 = len / 2;
      n2 -= n2 % 8;
      if ((p >> (L - 1 - d)) & 1) {
        st += n2;
        len -= n2;
      } else {
        len = n2;
      }
    }
    if ((p & ((1 << (L - d)) - 1)) == 0) {  // first path through this leaf
      const int node = (1 << d) - 1 + (p >> (L - d));
      sh.u.pw.split[node] = 0;
      sh.u.pw.val[node] = len <= 128 ? pw_block(a + st, len) : pw_serial(a + st, len);
    }
  }
  __syncthreads();
  for (int d = L - 1; d >= 0; --d) {
    for (int id = threadIdx.x; id < (1 << d); id += TV_THREADS) {
      const int node = (1 << d) - 1 + id;
      // nodes under a leaf hold stale flags but are never read
      if (sh.u.pw.split[node]) {
        const int c0 = (1 << (d + 1)) - 1 + 2 * id;
        sh.u.pw.val[node] = __dadd_rn(sh.u.pw.val[c0], sh.u.pw.val[c0 + 1]);
      }
    }
    __syncthreads();
  }
  const double r = sh.u.pw.val[0];
  __syncthreads();
  return r;
}

// ---------------------------------------------------- multi-CTA budget
// A tier with more pruned calls than one CTA can stage is split along the
// top of numpy's recursion: its 2^L subtrees (L = pw_top_depth) are summed
// by different CTAs with pairwise_cta, and the last of them folds the top
// tree, left + right at every split node, exactly as the recursion adds.
constexpr int PW_TOP_MAX = 6;  // at most 64 subtrees per tier
constexpr int PW_PART = 128;   // heap slots per tier for the top tree

__device__ __forceinline__ int pw_top_depth(long long n) {
  int L = 0;
  for (long long m = n; m > PW_SMEM_VALS && L < PW_TOP_MAX; m = (m + 1) / 2) ++L;
  return L;
}

// Path s of 2^L through the top of the recursion over n values: the node's
// range, and the depth at which it became a leaf (<= 128 values) or L.
__device__ __forceinline__ int pw_subtree(long long n, int L, int s, long long &st, long long &len) {
  st = 0;
  len = n;
  int d = 0;
  for (; d < L && len > 128; ++d) {
    long long n2 = len / 2;
    n2 -= n2 % 8;
    if ((s >> (L - 1 - d)) & 1) {
      st += n2;
      len -= n2;
    } else {
      len = n2;
    }
  }
  return d;
}

// Budget work item s of tier t (the whole CTA).  vals: the tier's pruned
// products in reference order.  Returns true to the thread that completed the
// tier's sum (tc->tier_budget[t] is final).
template <int NT>
__device__ bool budget_item(TvShared &sh, TraverseCounters *tc, double *part, const double *vals,
                            long long np_, int t, int s) {
  const int L = pw_top_depth(np_);
  long long st, len;
  const int d = pw_subtree(np_, L, s, st, len);
  const bool rep = (s & ((1 << (L - d)) - 1)) == 0;
  if (rep && np_) {
    const double *src = vals + st;
    if (len <= PW_SMEM_VALS) {
      stage_values<NT>(sh.u.pw.vals, src, (unsigned long long)len);
      __syncthreads();
      src = sh.u.pw.vals;
    }
    const double v = pairwise_cta(sh, src, len);
    if (threadIdx.x == 0) part[t * PW_PART + (1 << d) - 1 + (s >> (L - d))] = v;
  }
  bool done = false;
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(&tc->pw_done[t], 1u) == (1u << L) - 1) {  // last item of the tier: fold
      __threadfence();
      double r = 0.0;
      if (np_) {
        if (L == 0) {
          r = __ldcg(&part[t * PW_PART]);
        } else {
          // nodes split iff their range has > 128 values (and depth < L)
          for (int dd = L - 1; dd >= 0; --dd)
            for (int id = 0; id < (1 << dd); ++id) {
              long long st2, len2;
              const int dl = pw_subtree(np_, dd, id, st2, len2);
              if (dl < dd || len2 <= 128) continue;  // a leaf (or under one)
              const int node = (1 << dd) - 1 + id, c0 = (1 << (dd + 1)) - 1 + 2 * id;
              part[t * PW_PART + node] =
                  __dadd_rn(__ldcg(&part[t * PW_PART + c0]), __ldcg(&part[t * PW_PART + c0 + 1]));
            }
          r = __ldcg(&part[t * PW_PART]);
        }
      }
      tc->tier_budget[t] = r;
      done = true;
    }
  }
  return done;
}

// Items of all tiers, tier by tier: item -> (tier, subtree).
__device__ __forceinline__ bool budget_item_of(const unsigned long long *np_t, int ntiers, int item,
                                               int &t, int &s) {
  for (t = 0; t < ntiers; ++t) {
    const int k = 1 << pw_top_depth((long long)np_t[t]);
    if (item < k) {
      s = item;
      return true;
    }
    item -= k;
  }
  return false;
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
  // this call's counters were zeroed by the previous call; clear that one's
  for (int x = blockIdx.x * TV_THREADS + threadIdx.x; x < (int)(sizeof(TraverseCounters) / 8);
       x += nblocks * TV_THREADS)
    reinterpret_cast<unsigned long long *>(a.tc_clear)[x] = 0ull;
  if (blockIdx.x == 0) {
    const unsigned long long t_entry = globaltimer();
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
  grid_sync(&tc->bar_grid, nblocks);
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
    grid_sync(&tc->bar_grid, nblocks);
    PHASE(3 + (t - t0 < 5 ? t - t0 : 4))
  }
  if (blockIdx.x == 0 && threadIdx.x == 0 && depth >= t0)
    tc->dirty_tiles[depth & 1] = prev_tiles;

  unsigned long long m = tc->n_active[depth];
  if (m > a.capacity) m = a.capacity;
  const uint64_t *leaf_codes = a.codes[depth & 1];
  // CTAs 0..nbud-1 compute the budget, then leave
  const int nbud = (int)((depth + 1) * 8 < (int)nblocks / 2 ? (depth + 1) * 8 : (int)nblocks / 2);

  // ---------------- omitted_budget: the first nbud CTAs, concurrent with the
  // grouping below (those CTAs never meet the later barriers): numpy's
  // pairwise sum per tier, large tiers split over several CTAs; the last tier
  // to finish adds the tier sums in tier order, as the reference's Python
  // float does.
  if ((int)blockIdx.x < nbud) {
    const int ntiers = depth + 1;
    int total = 0;
    for (int t = 0; t < ntiers; ++t) total += 1 << pw_top_depth((long long)tc->n_pruned[t]);
    for (int item = blockIdx.x; item < total; item += nbud) {
      int t, sub;
      budget_item_of(tc->n_pruned, ntiers, item, t, sub);
      const unsigned long long np_ = tc->n_pruned[t];
      const bool ok = tc->pruned_base[t] + np_ <= a.pruned_capacity;
      const bool done = budget_item<TV_THREADS>(sh, tc, a.pw_part, a.pruned_vals + tc->pruned_base[t],
                                                ok ? (long long)np_ : 0, t, sub);
      if (done && atomicAdd(&tc->tiers_done, 1u) == (unsigned)depth) {
        __threadfence();
        tc->phase_ns[12] = globaltimer();
        double b = 0.0;
        for (int u = 0; u <= depth; ++u)
          if (tc->n_pruned[u]) b = __dadd_rn(b, __ldcg(&tc->tier_budget[u]));
        tc->budget = b;
      }
      __syncthreads();
    }
    if (threadIdx.x == 0) atomicMax(&tc->phase_ns[13], globaltimer());
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
  grid_sync(&tc->bar_sub, gn);
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
  grid_sync(&tc->bar_sub, gn);
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
  grid_sync(&tc->bar_sub, gn);
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

// ======================================================= dense traversal
//
// For shallow trees (8^depth leaf triples fit comfortably) the tier-by-tier
// compaction is replaced by one dense pass.  Thread x owns the leaf-level
// triple whose Morton code is x -- the 3-bit digits (di,dj,dk) of every
// level, the root's first -- so thread order IS the reference's
// breadth-first order at every tier: a tier-t triple sits at x >> 3(depth-t)
// and its candidates appear in the order survivors expand (multiply.py:
// 207-212).  Each thread re-derives its ancestors' verdicts top-down
// (candidate = parent active; the same alive / strict `< tau` tests as the
// tiered kernel), so no survivor list is ever materialised:
//   * tier-t counters come from the representative threads (low 3(depth-t)
//     bits zero), CTA-reduced;
//   * pruned calls owned by the shard set bits in per-tier Morton bitmasks
//     (tier depth: one ballot per warp; shallower tiers: atomicOr);
//   * retained leaf triples set bits in the leaf tier's Morton bitmask.
// After one grid barrier, half the CTAs scan the pruned bitmasks (tier-major,
// so the scan position IS the reference's pruned-list position), rebuild
// each record and then run the per-tier pairwise budgets; the other half
// walk every C block (i, j) over k ascending through the retained bitmask:
// the block's k list comes out already sorted, so there is no histogram,
// scatter or sort.  Both scans are single-pass decoupled look-backs whose
// last tile clears the look-back state.
constexpr int DN_THREADS = 256;
constexpr int DN_MAX_DEPTH = 7;
static_assert(DN_PARTS_H == 16 && DN_MAXT_H == DN_MAX_DEPTH + 1, "TraverseCounters::dn_part layout");
constexpr int DN_PARTS = DN_PARTS_H;
constexpr int DN_PW = 64;   // pruned-bitmask words per scan tile

__host__ __device__ constexpr uint64_t dn_words(int t) {  // bitmask words of tier t
  return ((uint64_t(1) << (3 * t)) + 31) >> 5;
}
__host__ __device__ constexpr uint64_t dn_base(int t) {  // first word of tier t
  uint64_t b = 0;
  for (int s = 0; s < t; ++s) b += dn_words(s);
  return b;
}

// Per-tier counters are accumulated per warp in registers (ballot + popc over
// the representatives), then per CTA in shared memory, then once per CTA in
// global memory.
//
// Work-set layout (one of two parity sets, zero at rest: a call uses set p and
// clears set p^1, which the previous call used):
//   pm  [TOTAL_WORDS]   pruned-call bitmasks, tier-major, Morton order
//   ptc [P_TILES]       pruned calls per 64-word scan tile
//   qtc [Q_TILES]       retained leaf triples per 256-block grouping tile
//   ne  [NE_WORDS]      non-empty C blocks (bit g = i * nb + j)
//   tdn [D + 1]         scan tiles finished per tier (the budget waits on it)
// All of them are filled during classification, so after the one grid barrier
// every scan tile finds its output offset by summing its predecessors' counts
// (one parallel read) -- no look-back chain.
template <int D>
struct DnLayout {
  static constexpr uint64_t TOTAL_WORDS = dn_base(D + 1);
  static constexpr uint64_t P_TILES = (TOTAL_WORDS + DN_PW - 1) / DN_PW;
  static constexpr int NB = 1 << D;
  static constexpr uint64_t G = uint64_t(NB) * NB;
  static constexpr uint64_t Q_TILES = (G + DN_THREADS - 1) / DN_THREADS;
  static constexpr uint64_t NE_WORDS = (G + 31) / 32;
  static constexpr uint64_t PM = 0, PTC = TOTAL_WORDS, QTC = PTC + P_TILES, NE = QTC + Q_TILES,
                            TDN = NE + NE_WORDS, WORDS = TDN + D + 1;
};
size_t dense_work_words(int depth);

template <int D>
__global__ void __launch_bounds__(DN_THREADS) traverse_dense_kernel(TraverseArgs a) {
  using LY = DnLayout<D>;
  constexpr int NB = LY::NB;
  constexpr uint64_t G = LY::G;
  __shared__ TvShared sh;
  __shared__ unsigned s_cnt[D + 1][4];  // alive, active, pruned(owned), skip(owned)
  __shared__ unsigned long long s_red[DN_THREADS / 32];
  TraverseCounters *tc = a.tc;
  const unsigned nblocks = gridDim.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned long long t_entry = globaltimer();
  // the leaf-product kernel may launch now: its CTAs take SMs as this grid's
  // CTAs retire and wait (griddepcontrol.wait) for this grid's results
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  if (a.c_nsq_leaf) {  // the product's leaf-level norms (and their parents') start at zero
    const uint64_t P = D >= 1 ? G / 4 : 0;  // the parent level precedes the leaf level
    for (uint64_t e = (uint64_t)blockIdx.x * DN_THREADS + threadIdx.x; e < G + P;
         e += (uint64_t)nblocks * DN_THREADS) {
      a.c_nsq_leaf[(int64_t)e - (int64_t)P] = 0.0;
      a.c_nrm_leaf[(int64_t)e - (int64_t)P] = 0.0;
      a.c_occ_leaf[(int64_t)e - (int64_t)P] = 0;
    }
  }
  uint32_t *ws = a.dn_masks;                     // this call's work set
  uint32_t *pm = ws + LY::PM, *ptc = ws + LY::PTC, *qtc = ws + LY::QTC, *ne = ws + LY::NE,
           *tdn = ws + LY::TDN;
  uint32_t *am = a.dn_retained;                  // retained leaf triples (rewritten every call)
  double *npd = a.dn_np;                         // leaf-tier pruned products by Morton code
  constexpr uint64_t N_X = uint64_t(1) << (3 * D);
  constexpr uint64_t N_X32 = (N_X + 31) & ~uint64_t(31);
  const double *__restrict__ nrm_a = a.nrm_a;
  const double *__restrict__ nrm_b = a.nrm_b;
  const uint8_t *__restrict__ occ_a = a.occ_a;
  const uint8_t *__restrict__ occ_b = a.occ_b;

  constexpr int U = D >= 2 ? D - 2 : -1;  // tiers <= U are warp-uniform (see phase 1)
  // Per-lane tiers T0..D read the operands' lower pyramid levels from L2;
  // those loads do not depend on the verdicts, so the next x's are issued
  // before this x is classified (one memory round trip per thread, not one
  // per x: a thread has 3-4 x at c2).
  constexpr int T0 = U + 1;
  constexpr int NPL = D + 1 - T0;
  struct LaneOps {
    double na[NPL], nb[NPL];
    bool oc[NPL];
  };
  auto load_lane = [&](uint64_t x, LaneOps &o) {
    const uint32_t xe = x < N_X ? (uint32_t)x : 0u;
    const uint32_t ix = compact3(xe >> 2), jx = compact3(xe >> 1), kx = compact3(xe);
#pragma unroll
    for (int t = T0; t <= D; ++t) {
      const uint32_t I = ix >> (D - t), J = jx >> (D - t), K = kx >> (D - t);
      const int64_t ik = level_offset(t) + (int64_t(I) << t) + K;
      const int64_t kj = level_offset(t) + (int64_t(K) << t) + J;
      o.oc[t - T0] = __ldg(occ_a + ik) & __ldg(occ_b + kj);
      o.na[t - T0] = __ldg(nrm_a + ik);
      o.nb[t - T0] = __ldg(nrm_b + kj);
    }
  };
  const uint64_t x_stride = (uint64_t)nblocks * DN_THREADS;
  LaneOps cur;
  uint64_t x = (uint64_t)blockIdx.x * DN_THREADS + threadIdx.x;
  // the first x's operand loads go out before anything else: their DRAM
  // latency (the L2 is cold after a flush) overlaps the clears and the
  // staging of the pyramid tops below
  if (x < N_X32) load_lane(x, cur);

  // the previous call's counters and work set were read back / consumed
  // already: leave them zero for the call after this one
  for (int x = blockIdx.x * DN_THREADS + threadIdx.x; x < (int)(sizeof(TraverseCounters) / 8);
       x += nblocks * DN_THREADS)
    reinterpret_cast<unsigned long long *>(a.tc_clear)[x] = 0ull;
  for (uint64_t x = (uint64_t)blockIdx.x * DN_THREADS + threadIdx.x; x < a.dn_work_words;
       x += (uint64_t)nblocks * DN_THREADS)
    a.dn_masks_clear[x] = 0u;
  for (int x = threadIdx.x; x < (D + 1) * 4; x += DN_THREADS) (&s_cnt[0][0])[x] = 0u;
  // the operands' pyramid tops (levels 0..U: the warp-uniform tiers), staged
  // once per CTA -- those tiers' verdicts then cost shared-memory reads
  constexpr int TOPN = U >= 0 ? (int)level_offset(U + 1) : 1;
  static_assert(TOPN <= PREFIX_ENTRIES, "pyramid top exceeds the staging area");
  double *s_top_na = sh.u.top.nrm_a, *s_top_nb = sh.u.top.nrm_b;  // (sh.u is free until the barrier)
  uint8_t *s_top_oa = sh.u.top.occ_a, *s_top_ob = sh.u.top.occ_b;
  if (U >= 0)
    for (int e = threadIdx.x; e < TOPN; e += DN_THREADS) {
      s_top_na[e] = __ldg(nrm_a + e);
      s_top_nb[e] = __ldg(nrm_b + e);
      s_top_oa[e] = __ldg(occ_a + e);
      s_top_ob[e] = __ldg(occ_b + e);
    }
  __syncthreads();
  if (blockIdx.x == 0 && threadIdx.x == 0) tc->phase_ns[2] = globaltimer() - t_entry;  // (durations)

  // ---------------- phase 1: classify every leaf triple and its ancestors
  // Tiers t <= U have one ancestor per 64 consecutive x, so a warp's 32
  // lanes share it: those verdicts are warp-uniform and a warp whose tier-U
  // ancestor is not active leaves after them.
  unsigned wc[D + 1][4];
#pragma unroll
  for (int t = 0; t <= D; ++t) wc[t][0] = wc[t][1] = wc[t][2] = wc[t][3] = 0u;
  for (; x < N_X32; x += x_stride) {
    LaneOps nxt;
    if (x + x_stride < N_X32) load_lane(x + x_stride, nxt);
    const bool valid = x < N_X;
    const uint32_t xe = valid ? (uint32_t)x : 0u;  // lanes past the end read triple 0
    const uint32_t ix = compact3(xe >> 2), jx = compact3(xe >> 1), kx = compact3(xe);
    const uint64_t xw = x - lane;  // the warp's first x
    bool cand = valid;
#pragma unroll
    for (int t = 0; t <= U; ++t) {  // warp-uniform tiers (operands staged in shared memory)
      const int sh_t = D - t;
      const uint32_t I = ix >> sh_t, J = jx >> sh_t, K = kx >> sh_t;
      const int ik = (int)level_offset(t) + (int)(I << t) + (int)K;
      const int kj = (int)level_offset(t) + (int)(K << t) + (int)J;
      const int64_t r0 = int64_t(I) << sh_t, r1 = int64_t(I + 1) << sh_t;
      const bool intersects = r1 > a.row_lo && r0 < a.row_hi;
      const bool owned = r0 >= a.row_lo && r0 < a.row_hi;
      const bool oc = s_top_oa[ik] & s_top_ob[kj];
      const double np_ = __dmul_rn(s_top_na[ik], s_top_nb[kj]);
      const bool alive = cand && intersects && oc;
      const bool pruned = alive && np_ < a.tau_tier[t];
      const bool active = alive && !pruned;
      // the tier-t representative is lane 0 of the warp starting its block
      if (lane == 0 && (xw & ((uint64_t(1) << (3 * sh_t)) - 1)) == 0) {
        wc[t][0] += alive;
        wc[t][1] += active;
        wc[t][2] += pruned && owned;
        wc[t][3] += cand && intersects && !oc && owned;
        if (pruned && owned) {
          const uint64_t m = x >> (3 * sh_t);
          const uint64_t w = dn_base(t) + (m >> 5);
          atomicOr(&pm[w], 1u << (m & 31));
          atomicAdd(&ptc[w / DN_PW], 1u);
        }
      }
      cand = active;
    }
    if (U >= 0 && !__any_sync(0xffffffffu, cand)) {  // nothing below survives
      if (lane == 0) am[x >> 5] = 0u;  // (pm's leaf words are zero at rest)
    } else {
      bool pruned_leaf = false, active_leaf = false;
      double np_leaf = 0.0;
#pragma unroll
      for (int t = T0; t <= D; ++t) {
        const int sh_t = D - t;
        const uint32_t I = ix >> sh_t;
        const bool rep = valid && (x & ((uint64_t(1) << (3 * sh_t)) - 1)) == 0;
        const int64_t r0 = int64_t(I) << sh_t, r1 = int64_t(I + 1) << sh_t;
        const bool intersects = r1 > a.row_lo && r0 < a.row_hi;
        const bool owned = r0 >= a.row_lo && r0 < a.row_hi;
        const double np_ = __dmul_rn(cur.na[t - T0], cur.nb[t - T0]);
        const bool alive = cand && intersects && cur.oc[t - T0];
        const bool pruned = alive && np_ < a.tau_tier[t];
        const bool active = alive && !pruned;
        const bool p_own = pruned && owned;
        const bool skip = cand && intersects && !cur.oc[t - T0] && owned;
        wc[t][0] += __popc(__ballot_sync(0xffffffffu, rep && alive));
        wc[t][1] += __popc(__ballot_sync(0xffffffffu, rep && active));
        wc[t][2] += __popc(__ballot_sync(0xffffffffu, rep && p_own));
        wc[t][3] += __popc(__ballot_sync(0xffffffffu, rep && skip));
        if (t < D) {
          if (rep && p_own) {
            const uint64_t m = x >> (3 * sh_t);
            const uint64_t w = dn_base(t) + (m >> 5);
            atomicOr(&pm[w], 1u << (m & 31));
            atomicAdd(&ptc[w / DN_PW], 1u);
          }
        } else {
          pruned_leaf = p_own;
          active_leaf = active;
          np_leaf = np_;
        }
        cand = active;
      }
      const unsigned bp = __ballot_sync(0xffffffffu, pruned_leaf);
      const unsigned bv = __ballot_sync(0xffffffffu, active_leaf);
      if (pruned_leaf) npd[x] = np_leaf;
      // C block of this lane's triple; a warp's blocks all lie in one grouping tile
      const uint64_t g = (uint64_t)ix * NB + jx;
      const unsigned same = __match_any_sync(0xffffffffu, g);
      if (bv && lane == __ffs(same) - 1 && (bv & same)) atomicOr(&ne[g >> 5], 1u << (g & 31));
      if (lane == 0) {
        const uint64_t w = dn_base(D) + (x >> 5);
        if (bp) {
          pm[w] = bp;
          atomicAdd(&ptc[w / DN_PW], (unsigned)__popc(bp));
        }
        am[x >> 5] = bv;
        if (bv && !a.bitmask_groups) atomicAdd(&qtc[g / DN_THREADS], (unsigned)__popc(bv));
      }
    }
    cur = nxt;
    if (blockIdx.x == 0 && threadIdx.x == 0 && x < 4 * x_stride) tc->phase_ns[3 + x / x_stride] = globaltimer() - t_entry;
  }
  // per-warp counters (lane 0 holds them) -> shared memory, then one thread
  // per counter sums the warps (no shared atomics in a chain)
  __shared__ unsigned s_wc[DN_THREADS / 32][(D + 1) * 4];
  if (lane == 0) {
#pragma unroll
    for (int t = 0; t <= D; ++t)
#pragma unroll
      for (int f = 0; f < 4; ++f) s_wc[warp][t * 4 + f] = wc[t][f];
  }
  __syncthreads();
  // CTA totals into one of DN_PARTS copies (spreads the global atomics)
  for (int x = threadIdx.x; x < (D + 1) * 4; x += DN_THREADS) {
    unsigned v = 0;
#pragma unroll
    for (int w = 0; w < DN_THREADS / 32; ++w) v += s_wc[w][x];
    if (v) atomicAdd(&tc->dn_part[blockIdx.x % DN_PARTS][x / 4][x % 4], (unsigned long long)v);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    tc->phase_ns[15] = t_entry;
    tc->phase_ns[0] = globaltimer();
  }
  if (a.timeline && threadIdx.x == 0) {
    a.timeline[4 * blockIdx.x] = t_entry;
    a.timeline[4 * blockIdx.x + 1] = globaltimer();
  }
  grid_sync(&tc->bar_grid, nblocks);
  if (blockIdx.x == 0 && threadIdx.x == 0) tc->phase_ns[1] = globaltimer();

  // sum of ptr[u] over u in [lo, hi) (and popc when `bits`), by the whole CTA
  auto cta_sum = [&](const uint32_t *ptr, uint64_t lo, uint64_t hi, bool bits) -> unsigned long long {
    unsigned long long v = 0;
    for (uint64_t u = lo + threadIdx.x; u < hi; u += DN_THREADS) {
      const uint32_t w = __ldcg(ptr + u);
      v += bits ? (unsigned long long)__popc(w) : (unsigned long long)w;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) s_red[warp] = v;
    __syncthreads();
    unsigned long long r = 0;
#pragma unroll
    for (int q = 0; q < DN_THREADS / 32; ++q) r += s_red[q];
    __syncthreads();
    return r;
  };

  // roles after the barrier: budget CTAs (one per tier), grouping CTAs, scan CTAs
  // one budget CTA per tier plus a few for the subtrees of large tiers
  const unsigned n_b = (D + 1) + 8 < nblocks / 4 ? (D + 1) + 8 : nblocks / 4;
  const unsigned n_q = a.bitmask_groups ? 1u
      : (unsigned)(LY::Q_TILES < (nblocks - n_b) / 4 ? LY::Q_TILES : (nblocks - n_b) / 4 > 0 ? (nblocks - n_b) / 4 : 1);
  // every CTA reports its exit; the last one sets tc->trav_done (release), so
  // that a kernel which starts on tc->groups_ready can still tell when the
  // whole traversal -- pruned records, budget, statistics -- is final
  auto signal_exit = [&]() {
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      if (atomicAdd(&tc->exited, 1u) == nblocks - 1) {
        __threadfence();
        asm volatile("st.release.gpu.u32 [%0], %1;" ::"l"(&tc->trav_done), "r"(1u) : "memory");
      }
    }
  };
  const unsigned n_p = nblocks - n_b - n_q;

  if (blockIdx.x < n_p) {
    // ---------------- phase 2P: pruned records, tier-major Morton order
    // Tiles of DN_PW words; the scan position of a set bit IS its place in
    // the reference's pruned list.  The tile's records are dealt out one per
    // thread (word by binary search over the word prefixes, bit by __fns), so
    // the work follows the records, not the words, and the stores coalesce.
    __shared__ unsigned s_wpre[DN_PW + 1], s_bits[DN_PW];
    for (unsigned long long tile = blockIdx.x; tile < LY::P_TILES; tile += n_p) {
      const unsigned long long base = cta_sum(ptc, 0, tile, false);
      const uint64_t w = tile * DN_PW + threadIdx.x;
      uint32_t bits = 0;
      if (threadIdx.x < DN_PW && w < LY::TOTAL_WORDS) bits = __ldcg(pm + w);
      unsigned long long tile_total;
      const unsigned long long in_tile =
          block_exclusive<DN_THREADS>(pack2(0u, (unsigned)__popc(bits)), sh.warp, &tile_total);
      if (threadIdx.x < DN_PW) {
        s_wpre[threadIdx.x] = unpack_b(in_tile);
        s_bits[threadIdx.x] = bits;
      }
      __syncthreads();
      const unsigned B = unpack_b(tile_total);
#pragma unroll 4
      for (unsigned e = threadIdx.x; e < B; e += DN_THREADS) {
        int lo = 0, hi = DN_PW - 1;  // last word whose prefix <= e
        while (lo < hi) {
          const int mid = (lo + hi + 1) >> 1;
          if (s_wpre[mid] <= e) lo = mid; else hi = mid - 1;
        }
        const unsigned bit = __fns(s_bits[lo], 0, (int)(e - s_wpre[lo]) + 1);
        const uint64_t wq = tile * DN_PW + lo;
        int t = D;
        uint32_t m;
        if (wq >= dn_base(D)) {
          m = (uint32_t)(((wq - dn_base(D)) << 5) + bit);
        } else {
          t = 0;
#pragma unroll
          for (int s2 = 1; s2 < D; ++s2) t += wq >= dn_base(s2);
          m = (uint32_t)(((wq - dn_base(t)) << 5) + bit);
        }
        const uint32_t I = compact3(m >> 2), J = compact3(m >> 1), K = compact3(m);
        double v;
        if (t == D) {
          v = npd[m];  // leaf tier: product saved by phase 1
        } else {
          const int64_t ik = level_offset(t) + (int64_t(I) << t) + K;
          const int64_t kj = level_offset(t) + (int64_t(K) << t) + J;
          v = __dmul_rn(nrm_a[ik], nrm_b[kj]);
        }
        const unsigned long long pos = base + e;
        if (pos < a.pruned_capacity) {
          a.pruned_vals[pos] = v;
          a.pruned_codes[pos] = pack_triple(I, J, K);
        } else {
          tc->overflow = 1;
        }
      }
      __syncthreads();
      if (threadIdx.x == 0) {  // tell the budget CTAs of the tiers this tile covers
        __threadfence();
        const uint64_t w0 = tile * DN_PW, w1 = w0 + DN_PW - 1;
#pragma unroll
        for (int t = 0; t <= D; ++t)
          if (w0 < dn_base(t + 1) && w1 >= dn_base(t)) atomicAdd(&tdn[t], 1u);
      }
    }
    if (a.timeline && threadIdx.x == 0) a.timeline[4 * blockIdx.x + 3] = globaltimer();
    signal_exit();
    return;
  }

  if (blockIdx.x >= nblocks - n_b) {
    // ---------------- budget: numpy pairwise per tier (large tiers split over
    // several CTAs), summed in tier order
    const int bj = (int)(blockIdx.x - (nblocks - n_b));
    __shared__ unsigned long long s_tot[D + 1][4];
    __shared__ unsigned long long s_np[D + 1];
    for (int x = threadIdx.x; x < (D + 1) * 4; x += DN_THREADS) (&s_tot[0][0])[x] = 0ull;
    __syncthreads();
    for (int x = threadIdx.x; x < DN_PARTS * (D + 1) * 4; x += DN_THREADS) {
      const int q = x / ((D + 1) * 4), f = x - q * ((D + 1) * 4);
      const unsigned long long v = __ldcg(&tc->dn_part[q][0][0] + f);
      if (v) atomicAdd(&(&s_tot[0][0])[f], v);
    }
    __syncthreads();
    unsigned long long pbase[D + 2];
    pbase[0] = 0;
#pragma unroll
    for (int u = 0; u <= D; ++u) pbase[u + 1] = pbase[u] + s_tot[u][2];
    if (threadIdx.x <= D) s_np[threadIdx.x] = s_tot[threadIdx.x][2];
    if (bj == 0 && threadIdx.x == 0) {  // publish the tier statistics
      for (int u = 0; u <= D; ++u) {
        tc->n_alive[u] = s_tot[u][0];
        tc->n_active[u] = s_tot[u][1];
        tc->n_pruned[u] = s_tot[u][2];
        tc->n_skip[u] = s_tot[u][3];
        tc->pruned_base[u] = pbase[u];
      }
      tc->n_cand[0] = 1;
      for (int u = 1; u <= D; ++u) tc->n_cand[u] = 8ull * s_tot[u - 1][1];
      tc->first_grid_tier = D + 1;
      if (pbase[D + 1] > a.pruned_capacity) tc->overflow = 1;
    }
    __syncthreads();
    int total = 0;
    for (int u = 0; u <= D; ++u) total += 1 << pw_top_depth((long long)s_np[u]);
    for (int item = bj; item < total; item += n_b) {
      int t, sub;
      budget_item_of(s_np, D + 1, item, t, sub);
      const unsigned long long np_ = s_np[t];
      const bool ok = pbase[t + 1] <= a.pruned_capacity;
      if (np_ && ok) {
        // wait until every scan tile covering tier t has written its records
        const unsigned need = (unsigned)((dn_base(t + 1) - 1) / DN_PW - dn_base(t) / DN_PW + 1);
        if (threadIdx.x == 0) {
          for (;;) {
            unsigned v;
            asm volatile("ld.relaxed.gpu.u32 %0, [%1];" : "=r"(v) : "l"(tdn + t) : "memory");
            if (v >= need) break;
            __nanosleep(64);
          }
          asm volatile("fence.acq_rel.gpu;" ::: "memory");
        }
        __syncthreads();
      }
      const bool done = budget_item<DN_THREADS>(sh, tc, a.pw_part, a.pruned_vals + pbase[t],
                                                ok ? (long long)np_ : 0, t, sub);
      if (done && atomicAdd(&tc->tiers_done, 1u) == (unsigned)D) {
        __threadfence();
        double tb[D + 1];
#pragma unroll
        for (int u = 0; u <= D; ++u) tb[u] = __ldcg(&tc->tier_budget[u]);
        double b = 0.0;
#pragma unroll
        for (int u = 0; u <= D; ++u)
          if (pbase[u + 1] > pbase[u]) b = __dadd_rn(b, tb[u]);
        tc->budget = b;
        tc->phase_ns[12] = globaltimer();
      }
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      atomicMax(&tc->phase_ns[13], globaltimer());
      if (a.timeline) a.timeline[4 * blockIdx.x + 3] = globaltimer();
    }
    signal_exit();
    return;
  }

  if (a.bitmask_groups) {
    // ---------------- phase 2Q (bitmask groups): one CTA compacts the
    // non-empty C blocks, ascending i * nb + j; the leaf-product kernel reads
    // each block's k list from the retained bitmask and starts as soon as
    // this is published (the record / budget CTAs are still running)
    unsigned long long base = 0;
    for (uint64_t w0 = 0; w0 < LY::NE_WORDS; w0 += DN_THREADS) {
      const uint64_t w = w0 + threadIdx.x;
      uint32_t bits = w < LY::NE_WORDS ? __ldcg(ne + w) : 0u;
      unsigned long long tot;
      const unsigned long long ex =
          block_exclusive<DN_THREADS>(pack2(0u, (unsigned)__popc(bits)), sh.warp, &tot);
      unsigned pos = (unsigned)(base + unpack_b(ex));
      while (bits) {
        const int q = __ffs(bits) - 1;
        bits &= bits - 1;
        a.group_ids[pos++] = (uint32_t)(w * 32 + q);
      }
      base += unpack_b(tot);
      __syncthreads();  // (sh.warp is reused by the next chunk's scan)
    }
    if (threadIdx.x == 0) {
      tc->num_groups = (unsigned)base;
      __threadfence();
      asm volatile("st.release.gpu.u32 [%0], %1;" ::"l"(&tc->groups_ready), "r"(1u) : "memory");
      atomicMax(&tc->phase_ns[13], globaltimer());
      tc->phase_ns[11] = globaltimer();
      if (a.timeline) a.timeline[4 * blockIdx.x + 3] = globaltimer();
    }
    signal_exit();
    return;
  }

  // ---------------- phase 2Q: C blocks in order, k lists ascending
  {
    __shared__ unsigned s_hist[NB + 1];
    for (unsigned long long tile = blockIdx.x - n_p; tile < LY::Q_TILES; tile += n_q) {
      // this tile's offsets: retained triples and non-empty blocks before it
      const unsigned long long ks_base = cta_sum(qtc, 0, tile, false);
      const unsigned long long slot_base = cta_sum(ne, 0, tile * DN_THREADS / 32, true);
      const int64_t g = (int64_t)tile * DN_THREADS + threadIdx.x;
      const uint32_t i = (uint32_t)(g >> D), j = (uint32_t)(g & (NB - 1));
      const uint32_t base = (spread3(i) << 2) | (spread3(j) << 1);
      // the block's retained bits: 4 k per word (k bits sit at x bits 0 and 3)
      constexpr int NW = NB >= 4 ? NB / 4 : 1;
      uint32_t wv[NW];
      unsigned cnt = 0;
#pragma unroll
      for (int q = 0; q < NW; ++q) {
        wv[q] = 0u;
        if (g < (int64_t)G) {
          if constexpr (NB >= 4) {
            const uint32_t x0 = base | spread3((uint32_t)(4 * q));
            wv[q] = (am[x0 >> 5] >> (x0 & 31)) & 0x303u;
          } else {
            for (int k = 0; k < NB; ++k) {
              const uint32_t x0 = base | spread3((uint32_t)k);
              wv[q] |= ((am[x0 >> 5] >> (x0 & 31)) & 1u) << k;
            }
          }
        }
        cnt += __popc(wv[q]);
      }
      if (a.lpt_order) {  // group sizes for the longest-first order of K3
        for (int x = threadIdx.x; x <= NB; x += DN_THREADS) s_hist[x] = 0u;
        __syncthreads();
        if (cnt) atomicAdd(&s_hist[cnt], 1u);
      }
      unsigned long long tile_total;
      const unsigned long long in_tile =
          block_exclusive<DN_THREADS>(pack2(cnt, cnt != 0), sh.warp, &tile_total);
      if (a.lpt_order)
        for (int x = threadIdx.x; x <= NB; x += DN_THREADS)
          if (s_hist[x]) atomicAdd(&tc->lpt_hist[x], s_hist[x]);
      if (threadIdx.x == 0) atomicAdd(&tc->num_groups, unpack_b(tile_total));
      const unsigned tile_off = (unsigned)ks_base, tile_cnt = unpack_a(tile_total);
      const bool fits = tile_off + tile_cnt <= a.capacity;
      const bool staged = tile_cnt <= 16384u;  // always for depth <= 6
      if (cnt) {  // group records are always written; k lists only within capacity
        const unsigned off = tile_off + unpack_a(in_tile);
        const unsigned slot = (unsigned)slot_base + unpack_b(in_tile);
        a.group_ids[slot] = (uint32_t)g;
        a.group_starts[slot] = off;
        if (!fits) {
          tc->overflow = 1;
        } else if (staged) {
          unsigned o = off - tile_off;
#pragma unroll
          for (int q = 0; q < NW; ++q) {
            if constexpr (NB >= 4) {
              if (wv[q] & 0x001u) sh.u.qks[o++] = (uint16_t)(4 * q);
              if (wv[q] & 0x002u) sh.u.qks[o++] = (uint16_t)(4 * q + 1);
              if (wv[q] & 0x100u) sh.u.qks[o++] = (uint16_t)(4 * q + 2);
              if (wv[q] & 0x200u) sh.u.qks[o++] = (uint16_t)(4 * q + 3);
            } else {
              for (int k = 0; k < NB; ++k)
                if ((wv[q] >> k) & 1u) sh.u.qks[o++] = (uint16_t)k;
            }
          }
        } else {
          unsigned o = off;
#pragma unroll
          for (int q = 0; q < NW; ++q) {
            if constexpr (NB >= 4) {
              if (wv[q] & 0x001u) a.ks[o++] = 4 * q;
              if (wv[q] & 0x002u) a.ks[o++] = 4 * q + 1;
              if (wv[q] & 0x100u) a.ks[o++] = 4 * q + 2;
              if (wv[q] & 0x200u) a.ks[o++] = 4 * q + 3;
            } else {
              for (int k = 0; k < NB; ++k)
                if ((wv[q] >> k) & 1u) a.ks[o++] = k;
            }
          }
        }
      }
      if (fits && staged) {  // the tile's k lists are one contiguous range of ks
        __syncthreads();
        for (unsigned e = threadIdx.x; e < tile_cnt; e += DN_THREADS)
          a.ks[tile_off + e] = sh.u.qks[e];
      }
      __syncthreads();
    }
    if (a.lpt_order) {
      // the last grouping CTA orders the groups, largest first (counting sort;
      // the order within a size class is arbitrary -- each group is one CTA's
      // work either way)
      __shared__ int s_last;
      if (threadIdx.x == 0) {
        __threadfence();
        s_last = atomicAdd(&tc->groups_done, 1u) == n_q - 1;
      }
      __syncthreads();
      if (s_last) {
        __threadfence();
        if (threadIdx.x == 0) {
          unsigned run = 0;
          for (int x = NB; x >= 1; --x) {
            s_hist[x] = run;
            run += __ldcg(&tc->lpt_hist[x]);
          }
          s_hist[0] = run;  // number of groups
        }
        __syncthreads();
        const unsigned ng = s_hist[0];
        unsigned tot = 0;
        for (int x = 1; x <= NB; ++x) tot += (unsigned)x * __ldcg(&tc->lpt_hist[x]);
        for (unsigned q = threadIdx.x; q < ng; q += DN_THREADS) {
          const unsigned st = __ldcg(&a.group_starts[q]);
          const unsigned size = (q + 1 < ng ? __ldcg(&a.group_starts[q + 1]) : tot) - st;
          const unsigned pos = atomicAdd(&s_hist[size], 1u);
          a.lpt_order[pos] = q;
        }
      }
    }
  }
  if (threadIdx.x == 0) {
    atomicMax(&tc->phase_ns[13], globaltimer());
    tc->phase_ns[11] = globaltimer();
    if (a.timeline) a.timeline[4 * blockIdx.x + 3] = globaltimer();
  }
  signal_exit();
}

template <int D>
static size_t dense_work_words_d() { return (size_t)DnLayout<D>::WORDS; }
template <int D>
static size_t dense_ne_offset_d() { return (size_t)DnLayout<D>::NE; }
// word offset of the non-empty C-block bitmask within a work set
size_t dense_ne_offset(int depth) {
  switch (depth) {
    case 0: return dense_ne_offset_d<0>();
    case 1: return dense_ne_offset_d<1>();
    case 2: return dense_ne_offset_d<2>();
    case 3: return dense_ne_offset_d<3>();
    case 4: return dense_ne_offset_d<4>();
    case 5: return dense_ne_offset_d<5>();
    case 6: return dense_ne_offset_d<6>();
    default: return dense_ne_offset_d<7>();
  }
}
size_t dense_work_words(int depth) {
  switch (depth) {
    case 0: return dense_work_words_d<0>();
    case 1: return dense_work_words_d<1>();
    case 2: return dense_work_words_d<2>();
    case 3: return dense_work_words_d<3>();
    case 4: return dense_work_words_d<4>();
    case 5: return dense_work_words_d<5>();
    case 6: return dense_work_words_d<6>();
    default: return dense_work_words_d<7>();
  }
}

// Dense for depth <= 6 (c2: 36-42 us vs 47-53 us tiered); at depth 7 the
// 2M-triple classification costs more than the tiers (c3: 109-115 vs 79-104 us).
bool dense_traversal_ok(int depth) { return depth <= 6; }
size_t dense_mask_words(int depth) { return (size_t)dn_base(depth + 1); }
size_t dense_retained_words(int depth) { return (size_t)dn_words(depth); }
size_t dense_np_entries(int depth) { return (size_t)1 << (3 * depth); }
size_t dense_pruned_tiles(int depth) { return (size_t)((dn_base(depth + 1) + DN_PW - 1) / DN_PW); }
size_t dense_status_entries(int depth, int64_t nb) {
  return dense_pruned_tiles(depth) + (size_t)((nb * nb + DN_THREADS - 1) / DN_THREADS) + 4;
}

template <int D>
static int launch_dense_d(const TraverseArgs &args, int num_sms, cudaStream_t st) {
  static int per_sm = 0;
  if (per_sm == 0) {
    SPAMM_CUDA_TRY(cudaFuncSetAttribute(traverse_dense_kernel<D>,
                                        cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    SPAMM_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, traverse_dense_kernel<D>,
                                                                 DN_THREADS, 0));
    if (per_sm < 1) {
      set_error("dense traverse kernel cannot be resident");
      return SPAMM_ERR_INTERNAL;
    }
  }
  // CTAs per SM (SPAMM_TRAVERSE_CTAS_PER_SM, default 2, capped by occupancy)
  static const int want = getenv("SPAMM_TRAVERSE_CTAS_PER_SM") ? atoi(getenv("SPAMM_TRAVERSE_CTAS_PER_SM")) : 2;
  const int grid = num_sms * (per_sm < want ? per_sm : want);
  void *kargs[] = {(void *)&args};
  // profiling aid: a plain launch (the grid still fits in one wave) so that
  // tools which skip cooperative launches can capture the kernel
  static const bool plain = getenv("SPAMM_TRAVERSE_PLAIN_LAUNCH") != nullptr;
  if (plain)
    SPAMM_CUDA_TRY(cudaLaunchKernel((const void *)traverse_dense_kernel<D>, grid, DN_THREADS,
                                    kargs, 0, st));
  else
    SPAMM_CUDA_TRY(cudaLaunchCooperativeKernel((const void *)traverse_dense_kernel<D>, grid,
                                               DN_THREADS, kargs, 0, st));
  return SPAMM_OK;
}

int launch_traverse_dense(const TraverseArgs &args, int num_sms, cudaStream_t st) {
  switch (args.depth) {
    case 0: return launch_dense_d<0>(args, num_sms, st);
    case 1: return launch_dense_d<1>(args, num_sms, st);
    case 2: return launch_dense_d<2>(args, num_sms, st);
    case 3: return launch_dense_d<3>(args, num_sms, st);
    case 4: return launch_dense_d<4>(args, num_sms, st);
    case 5: return launch_dense_d<5>(args, num_sms, st);
    case 6: return launch_dense_d<6>(args, num_sms, st);
    case 7: return launch_dense_d<7>(args, num_sms, st);
    default:
      set_error("dense traversal supports depth <= %d", DN_MAX_DEPTH);
      return SPAMM_ERR_INTERNAL;
  }
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
