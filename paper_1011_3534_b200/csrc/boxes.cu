// boxes.cu -- Morton (Z-curve) order of pruned product-space boxes, on the
// device: the sort behind the box log (multiply.py:306-315, keys from
// ordering.py:24-34).
//
// The reference sorts PrunedBox records with Python's stable sorted() by
// _interleave3(i_lo, j_lo, k_lo): the three element coordinates' bits
// interleaved i-major (bit b of i lands at 3b+2, of j at 3b+1, of k at 3b).
// Here every box gets that 63-bit key (coordinates < 2^21) and an LSD radix
// sort -- stable, like sorted() -- carries the box indices along, 8 key bits
// per pass and only as many passes as the largest key needs.  The result is a
// permutation; the caller reorders its records with it.
//
// Per pass: a histogram of the digit per 2048-box tile (digit-major, so one
// exclusive scan gives every tile its output offset per digit), the scan, and
// a stable scatter that ranks equal digits within a tile warp by warp
// (__match_any_sync) in input order.  All integer work; HBM-bound and far off
// the multiply's timed path.
#include <algorithm>
#include <vector>

#include "common.cuh"

namespace spamm {

constexpr int RS_THREADS = 256;
constexpr int RS_WARPS = RS_THREADS / 32;
constexpr int RS_ROUNDS = 8;
constexpr int RS_TILE = RS_THREADS * RS_ROUNDS;

__host__ __device__ inline uint64_t spread3(uint64_t x) {
  x &= 0x1fffffull;
  x = (x | x << 32) & 0x1f00000000ffffull;
  x = (x | x << 16) & 0x1f0000ff0000ffull;
  x = (x | x << 8) & 0x100f00f00f00f00full;
  x = (x | x << 4) & 0x10c30c30c30c30c3ull;
  x = (x | x << 2) & 0x1249249249249249ull;
  return x;
}

// boxes: 5 int64 per box (i_lo, j_lo, k_lo, edge, tier)
__global__ void box_keys_kernel(const int64_t *__restrict__ boxes, int64_t n,
                                uint64_t *__restrict__ keys, int64_t *__restrict__ idx) {
  for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < n;
       x += (int64_t)gridDim.x * blockDim.x) {
    const int64_t *b = boxes + 5 * x;
    keys[x] = (spread3((uint64_t)b[0]) << 2) | (spread3((uint64_t)b[1]) << 1) |
              spread3((uint64_t)b[2]);
    idx[x] = x;
  }
}

__global__ void __launch_bounds__(RS_THREADS)
rs_hist_kernel(const uint64_t *__restrict__ keys, int64_t n, int shift,
               unsigned *__restrict__ hist, int64_t ntiles) {
  __shared__ unsigned h[256];
  h[threadIdx.x] = 0;
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * RS_TILE;
#pragma unroll
  for (int r = 0; r < RS_ROUNDS; ++r) {
    const int64_t x = base + r * RS_THREADS + threadIdx.x;
    if (x < n) atomicAdd(&h[(keys[x] >> shift) & 255], 1u);
  }
  __syncthreads();
  hist[(int64_t)threadIdx.x * ntiles + blockIdx.x] = h[threadIdx.x];
}

// in-place exclusive scan of m counters by one CTA of 1024 threads, each
// owning a contiguous segment
__global__ void __launch_bounds__(1024) rs_scan_kernel(unsigned *__restrict__ v, int64_t m) {
  __shared__ unsigned long long s_warp[32];
  __shared__ unsigned long long s_seg[1024];
  const int64_t seg = (m + 1023) / 1024;
  const int64_t lo = std::min<int64_t>(m, threadIdx.x * seg), hi = std::min<int64_t>(m, lo + seg);
  unsigned long long sum = 0;
  for (int64_t i = lo; i < hi; ++i) sum += v[i];
  s_seg[threadIdx.x] = sum;
  __syncthreads();
  // block exclusive scan of the segment sums
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned long long incl = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) s_warp[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    unsigned long long w = s_warp[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    s_warp[lane] = w;
  }
  __syncthreads();
  unsigned long long run = (warp ? s_warp[warp - 1] : 0ull) + incl - sum;
  for (int64_t i = lo; i < hi; ++i) {
    const unsigned c = v[i];
    v[i] = (unsigned)run;
    run += c;
  }
}

__global__ void __launch_bounds__(RS_THREADS)
rs_scatter_kernel(const uint64_t *__restrict__ kin, const int64_t *__restrict__ vin,
                  uint64_t *__restrict__ kout, int64_t *__restrict__ vout, int64_t n, int shift,
                  const unsigned *__restrict__ hist, int64_t ntiles) {
  __shared__ unsigned run[256];
  __shared__ unsigned wc[RS_WARPS][256];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  run[threadIdx.x] = hist[(int64_t)threadIdx.x * ntiles + blockIdx.x];
  const int64_t base = (int64_t)blockIdx.x * RS_TILE;
  for (int r = 0; r < RS_ROUNDS; ++r) {
    const int64_t x0 = base + r * RS_THREADS;
    if (x0 >= n) break;  // uniform across the CTA
#pragma unroll
    for (int w = 0; w < RS_WARPS; ++w) wc[w][threadIdx.x] = 0;
    __syncthreads();
    const int64_t x = x0 + threadIdx.x;
    const bool valid = x < n;
    uint64_t key = 0;
    int64_t val = 0;
    unsigned d = 256;  // invalid lanes form their own group
    if (valid) {
      key = kin[x];
      val = vin[x];
      d = (unsigned)(key >> shift) & 255u;
    }
    const unsigned peers = __match_any_sync(0xffffffffu, d);
    const unsigned below = peers & ((1u << lane) - 1u);
    if (valid && below == 0) wc[warp][d] = __popc(peers);
    __syncthreads();
    if (valid) {
      unsigned off = run[d] + __popc(below);
      for (int w = 0; w < warp; ++w) off += wc[w][d];
      kout[off] = key;
      vout[off] = val;
    }
    __syncthreads();
    unsigned add = 0;
#pragma unroll
    for (int w = 0; w < RS_WARPS; ++w) add += wc[w][threadIdx.x];
    run[threadIdx.x] += add;
    __syncthreads();
  }
}

}  // namespace spamm

using namespace spamm;

extern "C" int spamm_boxes_morton_order(const int64_t *boxes, int64_t count, int32_t device,
                                        int64_t *order) {
  if (count < 0 || (count && (!boxes || !order))) {
    set_error("null box buffer");
    return SPAMM_ERR_VALUE;
  }
  if (count == 0) return SPAMM_OK;
  if (count > (int64_t)UINT32_MAX) {
    set_error("too many boxes (%lld)", (long long)count);
    return SPAMM_ERR_VALUE;
  }
  int64_t hi = 0;
  for (int64_t x = 0; x < count; ++x)
    for (int c = 0; c < 3; ++c) {
      const int64_t v = boxes[5 * x + c];
      if (v < 0 || v > (int64_t)TRIPLE_MASK) {
        set_error("box coordinate %lld outside [0, 2^21)", (long long)v);
        return SPAMM_ERR_VALUE;
      }
      hi |= v;
    }
  int coord_bits = 0;
  while (coord_bits < 21 && (hi >> coord_bits)) ++coord_bits;
  const int passes = (3 * coord_bits + 7) / 8;

  DeviceContext *ctx;
  SPAMM_TRY(get_context(device, &ctx));
  std::lock_guard<std::mutex> lk(ctx->mu);
  cudaStream_t st = ctx->stream;
  const int64_t ntiles = (count + RS_TILE - 1) / RS_TILE;
  const size_t bytes_boxes = (size_t)count * 5 * sizeof(int64_t);
  const size_t bytes_kv = (size_t)count * 8;
  const size_t bytes_hist = (size_t)ntiles * 256 * sizeof(unsigned);
  char *mem = nullptr;
  SPAMM_CUDA_TRY(dev_alloc((void **)&mem, bytes_boxes + 4 * bytes_kv + bytes_hist, st));
  int64_t *d_boxes = (int64_t *)mem;
  uint64_t *keys[2] = {(uint64_t *)(mem + bytes_boxes), (uint64_t *)(mem + bytes_boxes + bytes_kv)};
  int64_t *vals[2] = {(int64_t *)(mem + bytes_boxes + 2 * bytes_kv),
                      (int64_t *)(mem + bytes_boxes + 3 * bytes_kv)};
  unsigned *hist = (unsigned *)(mem + bytes_boxes + 4 * bytes_kv);
  cudaError_t e = cudaMemcpyAsync(d_boxes, boxes, bytes_boxes, cudaMemcpyHostToDevice, st);
  int cur = 0;
  if (e == cudaSuccess) {
    const int grid = (int)std::min<int64_t>((count + 255) / 256, (int64_t)ctx->num_sms * 8);
    box_keys_kernel<<<grid, 256, 0, st>>>(d_boxes, count, keys[0], vals[0]);
    for (int p = 0; p < passes; ++p) {
      rs_hist_kernel<<<(unsigned)ntiles, RS_THREADS, 0, st>>>(keys[cur], count, 8 * p, hist, ntiles);
      rs_scan_kernel<<<1, 1024, 0, st>>>(hist, ntiles * 256);
      rs_scatter_kernel<<<(unsigned)ntiles, RS_THREADS, 0, st>>>(
          keys[cur], vals[cur], keys[cur ^ 1], vals[cur ^ 1], count, 8 * p, hist, ntiles);
      cur ^= 1;
    }
    e = cudaGetLastError();
  }
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(order, vals[cur], bytes_kv, cudaMemcpyDeviceToHost, st);
  const cudaError_t ef = cudaFreeAsync(mem, st);
  if (e == cudaSuccess) e = ef;
  const cudaError_t es = cudaStreamSynchronize(st);
  if (e == cudaSuccess) e = es;
  if (e != cudaSuccess) {
    set_error("box sort: %s", cudaGetErrorString(e));
    return e == cudaErrorMemoryAllocation ? SPAMM_ERR_NOMEM : SPAMM_ERR_CUDA;
  }
  return SPAMM_OK;
}
