// shard.cu -- row-band trees for the multi-GPU layout and
// the fused TC2 update (purification.py:105-134) that works on a band.
//
// A distributed matrix is held as one tree per rank: the element storage of
// the rank's C block rows [band_lo, band_hi) (plus, for a multiply, the
// operand blocks fetched from other ranks), and the WHOLE matrix's norm /
// occupancy pyramid -- its leaf level assembled from every rank's band by an
// all-gather, the levels above rebuilt locally in the reference's fixed order
// (quadtree.py:90-92), so every rank holds bit-identical pyramids and the
// traversal of a row shard makes the single-GPU decisions.  The collectives
// themselves are the caller's (torch.distributed over NCCL, on the raw device
// pointers); this file provides the local pieces:
//
//   spamm_tree_band_from_device   a band's rows -> band tree (its own leaf norms)
//   spamm_tree_band_set           declare a tree (e.g. a row-shard product) a band
//   spamm_tree_pyramid_rebuild    leaf level (gathered) -> whole pyramid
//   spamm_tree_blocks_gather_device / _scatter_device   halo exchange buffers
//   spamm_tree_diagonal_rows      a band's part of trace()
//   spamm_tc2_update              X^2 - X leaf norms and 2X - X^2 in one pass
#include <algorithm>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "norms.cuh"

namespace spamm {

int alloc_tree(DeviceContext *ctx, int64_t n, int32_t leaf, int32_t dtype, spamm_tree **out,
               cudaStream_t st = nullptr);
void free_tree_async(spamm_tree *t, cudaStream_t st);
// (declared in common.cuh)
int finish_tree(DeviceContext *ctx, spamm_tree *t);

__global__ void iota_u32_kernel(uint32_t *__restrict__ out, uint32_t base, int64_t n,
                                unsigned *__restrict__ count) {
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n;
       q += (int64_t)gridDim.x * blockDim.x)
    out[q] = base + (uint32_t)q;
  if (blockIdx.x == 0 && threadIdx.x == 0) *count = (unsigned)n;
}

__global__ void leaf_nrm_kernel(const double *__restrict__ nsq, double *__restrict__ nrm, int64_t G) {
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < G;
       g += (int64_t)gridDim.x * blockDim.x)
    nrm[g] = __dsqrt_rn(nsq[g]);
}

// zero the leaf level (norms, nrm, occupancy) outside block rows [lo, hi)
__global__ void zero_leaf_level_outside(double *__restrict__ nsq, double *__restrict__ nrm,
                                        uint8_t *__restrict__ occ, int64_t G, int64_t g_lo,
                                        int64_t g_hi) {
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < G;
       g += (int64_t)gridDim.x * blockDim.x)
    if (g < g_lo || g >= g_hi) {
      nsq[g] = 0.0;
      nrm[g] = 0.0;
      occ[g] = 0;
    }
}

// copy a contiguous [count][b][b] buffer into the listed leaves
__global__ void scatter_blocks_kernel(unsigned char *__restrict__ padded, int64_t N, int32_t leaf,
                                      int64_t nb, int esz, const int64_t *__restrict__ ids,
                                      const unsigned char *__restrict__ in) {
  const int64_t q = blockIdx.x;
  const int64_t g = ids[q], bi = g / nb, bj = g - bi * nb;
  const int64_t row_bytes = (int64_t)leaf * esz;
  unsigned char *dst = padded + (bi * leaf) * N * esz + bj * row_bytes;
  const unsigned char *src = in + q * row_bytes * leaf;
  if (row_bytes % 16 == 0) {
    const int per_row = (int)(row_bytes / 16);
    for (int e = threadIdx.x; e < per_row * leaf; e += blockDim.x) {
      const int r = e / per_row, c = e - r * per_row;
      reinterpret_cast<uint4 *>(dst + (int64_t)r * N * esz)[c] =
          reinterpret_cast<const uint4 *>(src + r * row_bytes)[c];
    }
  } else {
    for (int64_t e = threadIdx.x; e < row_bytes * leaf; e += blockDim.x) {
      const int64_t r = e / row_bytes, c = e - r * row_bytes;
      dst[r * N * esz + c] = src[e];
    }
  }
}
__global__ void gather_blocks_dev_kernel(const unsigned char *__restrict__ padded, int64_t N,
                                         int32_t leaf, int64_t nb, int esz,
                                         const int64_t *__restrict__ ids,
                                         unsigned char *__restrict__ out) {
  const int64_t q = blockIdx.x;
  const int64_t g = ids[q], bi = g / nb, bj = g - bi * nb;
  const int64_t row_bytes = (int64_t)leaf * esz;
  const unsigned char *src = padded + (bi * leaf) * N * esz + bj * row_bytes;
  unsigned char *dst = out + q * row_bytes * leaf;
  if (row_bytes % 16 == 0) {
    const int per_row = (int)(row_bytes / 16);
    for (int e = threadIdx.x; e < per_row * leaf; e += blockDim.x) {
      const int r = e / per_row, c = e - r * per_row;
      reinterpret_cast<uint4 *>(dst + r * row_bytes)[c] =
          reinterpret_cast<const uint4 *>(src + (int64_t)r * N * esz)[c];
    }
  } else {
    for (int64_t e = threadIdx.x; e < row_bytes * leaf; e += blockDim.x) {
      const int64_t r = e / row_bytes, c = e - r * row_bytes;
      dst[e] = src[r * N * esz + c];
    }
  }
}

// ------------------------------------------------------------ fused TC2 step
// One TC2 sweep after the square (purification.py:123-133 and the sweep
// displacement of the driver loop, :190-199) forms from X and X2 = X^2:
//   D = add(X2, scale(X, -1))            its norm: the fixed-point test (and
//                                        the displacement when X2 is next)
//   Y = add(scale(X, 2), scale(X2, -1))  the next iterate when Tr(X) < n_occ
//   E = add(Y, scale(X, -1))             its norm: the displacement then
// Block by block (quadtree.py:280-293): where both operands are nonzero the
// elements are rn(x2 - x), rn(2x - x2), rn(y - x); where only one is, that
// operand's (scaled) block passes through bit for bit.  (For E the rule uses
// Y's block occupancy, known only after the block; but rn(0 - x) = -x, so
// rn(y - x) is the pass-through value whenever Y's block is all zero.)  This
// kernel writes Y's elements and forms the three leaf norms with the
// reference's chain (acc = rn(acc + rn(e^2)), row-major, quadtree.py:80-87)
// and occupancy (any e != 0; all-zero Y leaves canonicalised to +0.0) -- one
// thread per leaf running the independent chains side by side, so D's and
// E's elements never touch memory.  Leaves in block rows [lo, hi) only.
template <typename T>
__global__ void __launch_bounds__(128) tc2_band_kernel(
    const T *__restrict__ x, const T *__restrict__ x2, T *__restrict__ y, int64_t N, int32_t b,
    int64_t nb, int64_t g_lo, int64_t g_hi, const uint8_t *__restrict__ occ_x,
    const uint8_t *__restrict__ occ_x2, double *__restrict__ d_nsq, uint8_t *__restrict__ d_occ,
    double *__restrict__ y_nsq, uint8_t *__restrict__ y_occ, double *__restrict__ y_nrm,
    double *__restrict__ e_nsq, uint8_t *__restrict__ e_occ) {
  using U = typename Bits<T>::U;
  for (int64_t g = g_lo + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < g_hi;
       g += (int64_t)gridDim.x * blockDim.x) {
    const bool ox = occ_x[g], ox2 = occ_x2[g];
    if (!ox && !ox2) {  // both empty: D, Y and E empty (Y's block stays lazily zero)
      d_nsq[g] = 0.0;
      d_occ[g] = 0;
      if (y) {
        y_nsq[g] = 0.0;
        y_occ[g] = 0;
        y_nrm[g] = 0.0;
        e_nsq[g] = 0.0;
        e_occ[g] = 0;
      }
      continue;
    }
    const int64_t bi = g / nb, bj = g - bi * nb;
    const int64_t base = (bi * b) * N + bj * b;
    double dacc = 0.0, yacc = 0.0, eacc = 0.0;
    U dbits = 0, ybits = 0, ebits = 0;
    for (int r = 0; r < b; ++r) {
      const int64_t row = base + (int64_t)r * N;
      for (int c = 0; c < b; ++c) {
        const T xv = ox ? __ldg(x + row + c) : T(0);
        const T x2v = ox2 ? __ldg(x2 + row + c) : T(0);
        const T dv = (ox && ox2) ? (T)(x2v - xv) : ox ? (T)(-xv) : x2v;
        dbits |= Bits<T>::of(dv);
        const double de = (double)dv;
        dacc = __dadd_rn(dacc, __dmul_rn(de, de));
        if (y) {
          const T yv = (ox && ox2) ? (T)((T)(xv * T(2)) - x2v) : ox ? (T)(xv * T(2)) : (T)(-x2v);
          y[row + c] = yv;
          ybits |= Bits<T>::of(yv);
          const double ye = (double)yv;
          yacc = __dadd_rn(yacc, __dmul_rn(ye, ye));
          const T ev = ox ? (T)(yv - xv) : yv;
          ebits |= Bits<T>::of(ev);
          const double ee = (double)ev;
          eacc = __dadd_rn(eacc, __dmul_rn(ee, ee));
        }
      }
    }
    d_nsq[g] = dacc;
    d_occ[g] = (uint8_t)((U)(dbits << 1) != 0);
    if (y) {
      const bool nz = (U)(ybits << 1) != 0;
      if (!nz && ybits)  // all zero with some -0.0: canonical +0.0 (quadtree.py:127-129)
        for (int r = 0; r < b; ++r)
          for (int c = 0; c < b; ++c) y[base + (int64_t)r * N + c] = T(0);
      y_nsq[g] = yacc;
      y_occ[g] = (uint8_t)nz;
      y_nrm[g] = __dsqrt_rn(yacc);
      e_nsq[g] = eacc;
      e_occ[g] = (uint8_t)((U)(ebits << 1) != 0);
    }
  }
}

static int check_band(const spamm_tree *t, int64_t lo, int64_t hi) {
  if (lo < 0 || hi > t->nb || lo > hi) {
    set_error("row band [%lld, %lld) invalid for block grid %lld", (long long)lo, (long long)hi,
              (long long)t->nb);
    return SPAMM_ERR_VALUE;
  }
  return SPAMM_OK;
}

static unsigned grid_for(DeviceContext *ctx, int64_t n, int threads) {
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + threads - 1) / threads,
                                                          (int64_t)ctx->num_sms * 16));
}

// norms-only tree (no element storage): the D of a TC2 step
static int alloc_norms_only(DeviceContext *ctx, const spamm_tree *like, spamm_tree **out) {
  auto t = new spamm_tree;
  *t = spamm_tree{};
  t->n = like->n;
  t->N = like->N;
  t->nb = like->nb;
  t->leaf = like->leaf;
  t->depth = like->depth;
  t->dtype = like->dtype;
  t->device = like->device;
  const size_t P = (size_t)pyramid_size(t->depth);
  cudaError_t e = dev_alloc((void **)&t->nsq, sizeof(double) * P, ctx->stream);
  if (e == cudaSuccess) e = dev_alloc((void **)&t->occ, P, ctx->stream);
  if (e == cudaSuccess) e = dev_alloc((void **)&t->nrm, sizeof(double) * P, ctx->stream);
  if (e != cudaSuccess) {
    free_tree_async(t, ctx->stream);
    set_error("allocation: %s", cudaGetErrorString(e));
    return e == cudaErrorMemoryAllocation ? SPAMM_ERR_NOMEM : SPAMM_ERR_CUDA;
  }
  *out = t;
  return SPAMM_OK;
}

}  // namespace spamm

using namespace spamm;

extern "C" {

SPAMM_API int spamm_tree_band_from_device(const void *rows, int64_t n, int64_t ld, int32_t leaf,
                                          int32_t dtype, int64_t row_lo, int64_t row_hi,
                                          int32_t device, spamm_tree **out) {
  if (!out || leaf < 1 || (leaf & (leaf - 1)) || n < 1 || ld < n ||
      (dtype != SPAMM_DTYPE_F64 && dtype != SPAMM_DTYPE_F32)) {
    set_error("invalid band arguments");
    return SPAMM_ERR_VALUE;
  }
  DeviceContext *ctx;
  SPAMM_TRY(get_context(device, &ctx));
  std::lock_guard<std::mutex> lk(ctx->mu);
  spamm_tree *t = nullptr;
  SPAMM_TRY(alloc_tree(ctx, n, leaf, dtype, &t));
  int rc = check_band(t, row_lo, row_hi);
  const int64_t esz = t->elem_size();
  const int64_t r0 = row_lo * leaf, r1 = row_hi * leaf;        // padded rows of the band
  const int64_t lr1 = std::min<int64_t>(r1, n);                // ... that hold logical rows
  const int64_t G = t->nb * t->nb, g_lo = row_lo * t->nb, g_hi = row_hi * t->nb;
  do {
    if (rc) break;
    cudaStream_t st = ctx->stream;
    cudaError_t e = cudaSuccess;
    // the band's rows: logical part copied, padding zeroed
    if (r1 > r0) e = cudaMemsetAsync((unsigned char *)t->padded + r0 * t->N * esz, 0,
                                     (size_t)((r1 - r0) * t->N * esz), st);
    if (e == cudaSuccess && lr1 > r0)
      e = cudaMemcpy2DAsync((unsigned char *)t->padded + r0 * t->N * esz, (size_t)(t->N * esz), rows,
                            (size_t)(ld * esz), (size_t)(n * esz), (size_t)(lr1 - r0),
                            cudaMemcpyDeviceToDevice, st);
    if (e != cudaSuccess) {
      set_error("band copy: %s", cudaGetErrorString(e));
      rc = SPAMM_ERR_CUDA;
      break;
    }
    // leaf norms of the band's leaves (K1 list mode), zero elsewhere
    double *nsq_l = t->nsq + level_offset(t->depth), *nrm_l = t->nrm + level_offset(t->depth);
    uint8_t *occ_l = t->occ + level_offset(t->depth);
    zero_leaf_level_outside<<<grid_for(ctx, G, 256), 256, 0, st>>>(nsq_l, nrm_l, occ_l, G, g_lo, g_hi);
    if ((rc = ensure_scratch(ctx->reduce_tmp, sizeof(uint32_t) * (size_t)(g_hi - g_lo) + 64, st)))
      break;
    unsigned *cnt = (unsigned *)ctx->reduce_tmp.ptr;
    uint32_t *list = (uint32_t *)((unsigned char *)ctx->reduce_tmp.ptr + 64);
    iota_u32_kernel<<<grid_for(ctx, g_hi - g_lo, 256), 256, 0, st>>>(list, (uint32_t)g_lo, g_hi - g_lo,
                                                                   cnt);
    if ((e = cudaGetLastError()) != cudaSuccess) {
      set_error("band kernels: %s", cudaGetErrorString(e));
      rc = SPAMM_ERR_CUDA;
      break;
    }
    if (g_hi > g_lo &&
        (rc = build_pyramid_async(ctx, t, st, nullptr, list, cnt, g_hi - g_lo, nullptr, 0, nullptr,
                                  nullptr)))
      break;
    if (g_hi == g_lo && (rc = pyramid_upper_async(ctx, t, st))) break;
    rc = finish_tree(ctx, t);
  } while (0);
  if (rc) {
    free_tree_async(t, ctx->stream);
    return rc;
  }
  t->lazy_empty = true;  // rows outside the band are not held here
  t->distributed = true;
  t->band_lo = row_lo;
  t->band_hi = row_hi;
  *out = t;
  return SPAMM_OK;
}

SPAMM_API int spamm_tree_band_set(spamm_tree *t, int64_t row_lo, int64_t row_hi) {
  if (!t) {
    set_error("null tree");
    return SPAMM_ERR_VALUE;
  }
  SPAMM_TRY(check_band(t, row_lo, row_hi));
  t->distributed = true;
  t->lazy_empty = true;
  t->band_lo = row_lo;
  t->band_hi = row_hi;
  return SPAMM_OK;
}

SPAMM_API int spamm_tree_pyramid_rebuild(spamm_tree *t) {
  if (!t) {
    set_error("null tree");
    return SPAMM_ERR_VALUE;
  }
  DeviceContext *ctx;
  SPAMM_TRY(get_context(t->device, &ctx));
  std::lock_guard<std::mutex> lk(ctx->mu);
  SPAMM_TRY(tree_join(ctx, t));
  const int64_t G = t->nb * t->nb;
  leaf_nrm_kernel<<<grid_for(ctx, G, 256), 256, 0, ctx->stream>>>(
      t->nsq + level_offset(t->depth), t->nrm + level_offset(t->depth), G);
  SPAMM_CUDA_TRY(cudaGetLastError());
  SPAMM_TRY(pyramid_upper_async(ctx, t, ctx->stream));
  return finish_tree(ctx, t);
}

SPAMM_API int spamm_tree_blocks_gather_device(const spamm_tree *t, const int64_t *ids, int64_t count,
                                              void *dev_out) {
  if (!t || count < 0 || (count && (!ids || !dev_out)) || !t->padded) {
    set_error("invalid gather arguments");
    return SPAMM_ERR_VALUE;
  }
  if (!count) return SPAMM_OK;
  DeviceContext *ctx;
  SPAMM_TRY(get_context(t->device, &ctx));
  std::lock_guard<std::mutex> lk(ctx->mu);
  SPAMM_TRY(tree_join(ctx, t));
  const int64_t esz = t->elem_size(), blk = (int64_t)t->leaf * t->leaf * esz;
  for (int64_t q = 0; q < count; q += 65535) {
    const int64_t k = std::min<int64_t>(65535, count - q);
    gather_blocks_dev_kernel<<<(unsigned)k, 256, 0, ctx->stream>>>(
        (const unsigned char *)t->padded, t->N, t->leaf, t->nb, (int)esz, ids + q,
        (unsigned char *)dev_out + q * blk);
  }
  SPAMM_CUDA_TRY(cudaGetLastError());
  SPAMM_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  return SPAMM_OK;
}

SPAMM_API int spamm_tree_blocks_scatter_device(spamm_tree *t, const int64_t *ids, int64_t count,
                                               const void *dev_in) {
  if (!t || count < 0 || (count && (!ids || !dev_in)) || !t->padded) {
    set_error("invalid scatter arguments");
    return SPAMM_ERR_VALUE;
  }
  if (!t->distributed) {  // an ordinary tree's blocks are immutable (its norms cover them)
    set_error("blocks can be written only into a distributed band tree");
    return SPAMM_ERR_VALUE;
  }
  if (!count) return SPAMM_OK;
  DeviceContext *ctx;
  SPAMM_TRY(get_context(t->device, &ctx));
  std::lock_guard<std::mutex> lk(ctx->mu);
  SPAMM_TRY(tree_join(ctx, t));
  const int64_t esz = t->elem_size(), blk = (int64_t)t->leaf * t->leaf * esz;
  for (int64_t q = 0; q < count; q += 65535) {
    const int64_t k = std::min<int64_t>(65535, count - q);
    scatter_blocks_kernel<<<(unsigned)k, 256, 0, ctx->stream>>>(
        (unsigned char *)t->padded, t->N, t->leaf, t->nb, (int)esz, ids + q,
        (const unsigned char *)dev_in + q * blk);
  }
  SPAMM_CUDA_TRY(cudaGetLastError());
  SPAMM_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  return SPAMM_OK;
}

SPAMM_API int spamm_tree_diagonal_rows(const spamm_tree *t, int64_t row_lo, int64_t row_hi,
                                       void *host_out) {
  if (!t || !host_out || !t->padded) {
    set_error("null argument");
    return SPAMM_ERR_VALUE;
  }
  SPAMM_TRY(check_band(t, row_lo, row_hi));
  DeviceContext *ctx;
  SPAMM_TRY(get_context(t->device, &ctx));
  std::lock_guard<std::mutex> lk(ctx->mu);
  SPAMM_TRY(tree_join(ctx, t));
  const int64_t esz = t->elem_size();
  const int64_t r0 = std::min<int64_t>(row_lo * t->leaf, t->n), r1 = std::min<int64_t>(row_hi * t->leaf, t->n);
  if (r1 > r0) {
    // leaves on the diagonal that are empty are not held in storage (lazy):
    // those diagonal entries are zero
    std::vector<uint8_t> occ((size_t)t->nb);
    SPAMM_CUDA_TRY(cudaMemcpy2DAsync(occ.data(), 1, t->occ + level_offset(t->depth), (size_t)(t->nb + 1), 1,
                                     (size_t)t->nb, cudaMemcpyDeviceToHost, ctx->stream));
    SPAMM_CUDA_TRY(cudaMemcpy2DAsync(host_out, (size_t)esz,
                                     (const unsigned char *)t->padded + (r0 * (t->N + 1)) * esz,
                                     (size_t)((t->N + 1) * esz), (size_t)esz, (size_t)(r1 - r0),
                                     cudaMemcpyDeviceToHost, ctx->stream));
    SPAMM_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    for (int64_t r = r0; r < r1; ++r)
      if (!occ[(size_t)(r / t->leaf)])
        memset((unsigned char *)host_out + (r - r0) * esz, 0, (size_t)esz);
  }
  return SPAMM_OK;
}

SPAMM_API int spamm_tc2_update(const spamm_tree *x, const spamm_tree *x2, int32_t make_y,
                               int64_t row_lo, int64_t row_hi, spamm_tree **y_out,
                               spamm_tree **d_out, spamm_tree **e_out, double *roots) {
  if (!x || !x2 || !d_out || (make_y && (!y_out || !e_out))) {
    set_error("null argument");
    return SPAMM_ERR_VALUE;
  }
  if (x->n != x2->n || x->leaf != x2->leaf || x->dtype != x2->dtype || x->device != x2->device) {
    set_error("trees not conformable");
    return SPAMM_ERR_DIMENSION;
  }
  if (!x->padded || !x2->padded) {
    set_error("norms-only tree");
    return SPAMM_ERR_VALUE;
  }
  SPAMM_TRY(check_band(x, row_lo, row_hi));
  DeviceContext *ctx;
  SPAMM_TRY(get_context(x->device, &ctx));
  std::lock_guard<std::mutex> lk(ctx->mu);
  NvtxRange nvtx_tc2("spamm.tc2_update");
  SPAMM_TRY(tree_join(ctx, x));
  SPAMM_TRY(tree_join(ctx, x2));
  cudaStream_t st = ctx->stream;
  spamm_tree *y = nullptr, *d = nullptr, *e = nullptr;
  int rc = make_y ? alloc_tree(ctx, x->n, x->leaf, x->dtype, &y) : SPAMM_OK;
  if (!rc) rc = alloc_norms_only(ctx, x, &d);
  if (!rc && make_y) rc = alloc_norms_only(ctx, x, &e);
  const int64_t G = x->nb * x->nb, g_lo = row_lo * x->nb, g_hi = row_hi * x->nb;
  const int L = x->depth;
  auto leaf = [&](spamm_tree *t, int which) -> void * {  // 0 nsq, 1 nrm, 2 occ
    if (!t) return nullptr;
    return which == 0 ? (void *)(t->nsq + level_offset(L))
                      : which == 1 ? (void *)(t->nrm + level_offset(L)) : (void *)(t->occ + level_offset(L));
  };
  do {
    if (rc) break;
    for (spamm_tree *t : {d, y, e})
      if (t)
        zero_leaf_level_outside<<<grid_for(ctx, G, 256), 256, 0, st>>>(
            (double *)leaf(t, 0), (double *)leaf(t, 1), (uint8_t *)leaf(t, 2), G, g_lo, g_hi);
    const unsigned grid = grid_for(ctx, g_hi - g_lo, 128);
    if (x->dtype == SPAMM_DTYPE_F64)
      tc2_band_kernel<double><<<grid, 128, 0, st>>>(
          (const double *)x->padded, (const double *)x2->padded, y ? (double *)y->padded : nullptr,
          x->N, x->leaf, x->nb, g_lo, g_hi, x->occ + level_offset(L), x2->occ + level_offset(L),
          (double *)leaf(d, 0), (uint8_t *)leaf(d, 2), (double *)leaf(y, 0), (uint8_t *)leaf(y, 2),
          (double *)leaf(y, 1), (double *)leaf(e, 0), (uint8_t *)leaf(e, 2));
    else
      tc2_band_kernel<float><<<grid, 128, 0, st>>>(
          (const float *)x->padded, (const float *)x2->padded, y ? (float *)y->padded : nullptr,
          x->N, x->leaf, x->nb, g_lo, g_hi, x->occ + level_offset(L), x2->occ + level_offset(L),
          (double *)leaf(d, 0), (uint8_t *)leaf(d, 2), (double *)leaf(y, 0), (uint8_t *)leaf(y, 2),
          (double *)leaf(y, 1), (double *)leaf(e, 0), (uint8_t *)leaf(e, 2));
    cudaError_t err = cudaGetLastError();
    if (err != cudaSuccess) {
      set_error("tc2 kernel: %s", cudaGetErrorString(err));
      rc = SPAMM_ERR_CUDA;
      break;
    }
    for (spamm_tree *t : {d, y, e})
      if (t && (rc = pyramid_upper_async(ctx, t, st))) break;
    if (rc) break;
    if (y && (rc = finish_tree(ctx, y))) break;
    const SmallRead r[2] = {{&d->root_norm_sq, d->nsq, sizeof(double)},
                            {e ? &e->root_norm_sq : &d->root_norm_sq, e ? e->nsq : d->nsq, sizeof(double)}};
    rc = read_small_sync(ctx, st, r, 2);
  } while (0);
  if (rc) {
    free_tree_async(y, st);
    free_tree_async(d, st);
    free_tree_async(e, st);
    return rc;
  }
  // Y holds block rows [lo, hi); elsewhere it is lazily zero -- or, when the
  // band is part of a distributed matrix, not held here
  for (spamm_tree *t : {y, d, e}) {
    if (!t) continue;
    if (t == y) t->lazy_empty = true;
    if (x->distributed) {
      t->distributed = true;
      t->band_lo = row_lo;
      t->band_hi = row_hi;
    }
  }
  if (y) *y_out = y;
  *d_out = d;
  if (e_out) *e_out = e;
  if (roots) {
    roots[0] = d->root_norm_sq;
    roots[1] = e ? e->root_norm_sq : 0.0;
  }
  return SPAMM_OK;
}

}  // extern "C"
