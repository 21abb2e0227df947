// scan.cuh -- single-pass, order-preserving tile scan (decoupled look-back).
//
// Two 31-bit counters travel packed in one 64-bit status word per tile:
// [63:62] flag (0 = empty, 1 = tile aggregate, 2 = inclusive prefix),
// [61:31] counter A, [30:0] counter B.  Tiles are taken from a ticket in
// launch order, so a tile only ever waits for tiles that already started.
#pragma once
#include <cuda/atomic>

#include "common.cuh"

namespace spamm {

constexpr unsigned long long ST_AGG = 1ull << 62;
constexpr unsigned long long ST_PREFIX = 2ull << 62;
constexpr unsigned long long ST_FLAGS = 3ull << 62;
constexpr unsigned long long ST_VALUES = ~ST_FLAGS;

__device__ __forceinline__ unsigned long long pack2(unsigned a, unsigned b) {
  return ((unsigned long long)a << 31) | b;
}
__device__ __forceinline__ unsigned unpack_a(unsigned long long v) { return (unsigned)(v >> 31) & 0x7fffffffu; }
__device__ __forceinline__ unsigned unpack_b(unsigned long long v) { return (unsigned)(v & 0x7fffffffull); }

// Called by all 32 lanes of one warp.  Publishes the tile's aggregate,
// resolves its exclusive prefix from predecessors and publishes the
// inclusive prefix.  Returns the exclusive prefix (packed) on every lane.
// The status words carry their own values, so relaxed (L1-bypassing) loads
// and stores suffice: no fence, and no acquire -- which on sm_100 invalidates
// the SM's whole L1 on every poll and stalls co-resident CTAs.
__device__ __forceinline__ unsigned long long lookback_exclusive(unsigned long long *status,
                                                                 unsigned long long tile,
                                                                 unsigned long long tile_total) {
  const int lane = threadIdx.x & 31;
  unsigned long long excl = 0;
  if (tile == 0) {
    if (lane == 0) {
      cuda::atomic_ref<unsigned long long, cuda::thread_scope_device> st(status[0]);
      st.store(ST_PREFIX | tile_total, cuda::memory_order_relaxed);
    }
    return 0;
  }
  if (lane == 0) {
    cuda::atomic_ref<unsigned long long, cuda::thread_scope_device> st(status[tile]);
    st.store(ST_AGG | tile_total, cuda::memory_order_relaxed);
  }
  long long pred = (long long)tile - 1;
  for (;;) {
    const long long idx = pred - lane;
    unsigned long long s = ST_PREFIX;  // virtual zero prefix before tile 0
    if (idx >= 0) {
      cuda::atomic_ref<unsigned long long, cuda::thread_scope_device> st(status[idx]);
      for (;;) {
        s = st.load(cuda::memory_order_relaxed);
        if (s & ST_FLAGS) break;
        __nanosleep(20);
      }
    }
    const unsigned pmask = __ballot_sync(0xffffffffu, (s & ST_FLAGS) == ST_PREFIX);
    const int stop = pmask ? __ffs(pmask) - 1 : 31;
    unsigned long long val = lane <= stop ? (s & ST_VALUES) : 0ull;
#pragma unroll
    for (int o = 16; o; o >>= 1) val += __shfl_xor_sync(0xffffffffu, val, o);
    excl += val;
    if (pmask) break;
    pred -= 32;
  }
  if (lane == 0) {
    cuda::atomic_ref<unsigned long long, cuda::thread_scope_device> st(status[tile]);
    st.store(ST_PREFIX | (excl + tile_total), cuda::memory_order_relaxed);
  }
  return excl;
}

// Block-wide inclusive scan of one packed value per thread (blockDim = NT).
// Returns the thread's exclusive prefix within the block; *total = block sum.
template <int NT>
__device__ __forceinline__ unsigned long long block_exclusive(unsigned long long v,
                                                              unsigned long long *s_warp,
                                                              unsigned long long *total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned long long incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) s_warp[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    unsigned long long w = lane < NT / 32 ? s_warp[lane] : 0ull;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    if (lane < NT / 32) s_warp[lane] = w;
  }
  __syncthreads();
  *total = s_warp[NT / 32 - 1];
  return (warp ? s_warp[warp - 1] : 0ull) + (incl - v);
}

}  // namespace spamm
