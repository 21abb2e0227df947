// algebra.cu -- tree algebra on the device: add, scale, filter_drop and the
// diagonal for trace (quadtree.py:269-322), the element-wise building blocks
// of the purification driver (purification.py:115-142).
//
// Each result is a new tree whose pyramid is rebuilt by K1 (with the same
// canonicalisation of all-zero leaves as every tree), so results are
// bit-identical to the reference's numpy expressions:
//   add      out = a + b, except that a block nonzero in only one operand is
//            that operand's block, bit for bit (quadtree.py:283-293)
//   scale    out = padded * dtype(s)                      (quadtree.py:296-299)
//   filter   blocks with rn(sqrt(nsq)) < tau zeroed; the input itself when
//            nothing drops                               (quadtree.py:302-316)
//   trace    the diagonal, summed on the host with numpy's own add.reduce
//            (quadtree.py:274-277: pairwise order, padded dtype)
#include <algorithm>

#include "common.cuh"

namespace spamm {

int alloc_tree(DeviceContext *ctx, int64_t n, int32_t leaf, int32_t dtype, spamm_tree **out,
               cudaStream_t st = nullptr);
void free_tree_async(spamm_tree *t, cudaStream_t st);
// (declared in common.cuh)
int finish_tree(DeviceContext *ctx, spamm_tree *t);

// one row per CTA (grid-stride over rows), columns across the threads
template <typename T>
__global__ void add_kernel(const T *__restrict__ a, const T *__restrict__ b, T *__restrict__ out,
                           int64_t N, int32_t leaf, int64_t nb, const uint8_t *__restrict__ oa,
                           const uint8_t *__restrict__ ob) {
  for (int64_t r = blockIdx.x; r < N; r += gridDim.x) {
    const int64_t brow = (r / leaf) * nb;
    const T *ar = a + r * N;
    const T *br = b + r * N;
    T *orow = out + r * N;
    for (int64_t c = threadIdx.x; c < N; c += blockDim.x) {
      const int64_t g = brow + c / leaf;
      const bool na = oa[g], nbz = ob[g];
      const T x = ar[c], y = br[c];
      orow[c] = (na && !nbz) ? x : (!na && nbz) ? y : (T)(x + y);
    }
  }
}

template <typename T>
__global__ void scale_kernel(const T *__restrict__ a, T *__restrict__ out, int64_t count, T s) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = a[i] * s;
}

// leaves to drop: occupied and rn(sqrt(nsq)) < tau (the tree's cached nrm)
__global__ void drop_mark_kernel(const uint8_t *__restrict__ occ, const double *__restrict__ nrm,
                                 int64_t G, double tau, uint8_t *__restrict__ drop,
                                 unsigned *__restrict__ count) {
  unsigned local = 0;
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < G;
       g += (int64_t)gridDim.x * blockDim.x) {
    const bool d = occ[g] && nrm[g] < tau;
    drop[g] = d;
    local += d;
  }
  for (int o = 16; o; o >>= 1) local += __shfl_xor_sync(0xffffffffu, local, o);
  if ((threadIdx.x & 31) == 0 && local) atomicAdd(count, local);
}

template <typename T>
__global__ void filter_kernel(const T *__restrict__ a, T *__restrict__ out, int64_t N, int32_t leaf,
                              int64_t nb, const uint8_t *__restrict__ drop) {
  for (int64_t r = blockIdx.x; r < N; r += gridDim.x) {
    const int64_t brow = (r / leaf) * nb;
    for (int64_t c = threadIdx.x; c < N; c += blockDim.x)
      out[r * N + c] = drop[brow + c / leaf] ? T(0) : a[r * N + c];
  }
}

// copy the listed leaves into a contiguous [count][b][b] buffer
__global__ void gather_blocks_kernel(const unsigned char *__restrict__ padded, int64_t N, int32_t leaf,
                                     int64_t nb, int esz, const int64_t *__restrict__ ids,
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

// ids of the nonzero leaves (occupancy leaf level), ascending -- the device
// side of flatnonzero(_leaf_nonzero); one CTA, a contiguous chunk per thread
__global__ void __launch_bounds__(1024) occ_ids_kernel(const uint8_t *__restrict__ occ, int64_t G,
                                                       int64_t *__restrict__ ids) {
  __shared__ int64_t warp_tot[32];
  const int64_t per = (G + blockDim.x - 1) / blockDim.x;
  const int64_t lo0 = (int64_t)threadIdx.x * per;
  const int64_t lo = lo0 < G ? lo0 : G, hi = lo + per < G ? lo + per : G;
  int64_t cnt = 0;
  for (int64_t g = lo; g < hi; ++g) cnt += occ[g] != 0;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int64_t inc = cnt;
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t v = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += v;
  }
  if (lane == 31) warp_tot[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    int64_t w = lane < (int)(blockDim.x >> 5) ? warp_tot[lane] : 0;
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t v = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += v;
    }
    warp_tot[lane] = w;  // inclusive over warps
  }
  __syncthreads();
  int64_t pos = inc - cnt + (warp ? warp_tot[warp - 1] : 0);
  for (int64_t g = lo; g < hi; ++g)
    if (occ[g]) ids[pos++] = g;
}

static int grid_rows(DeviceContext *ctx, int64_t N) {
  return (int)std::min<int64_t>(N, (int64_t)ctx->num_sms * 16);
}

static int finish_new(DeviceContext *ctx, spamm_tree *t, spamm_tree **out) {
  int rc = build_pyramid_async(ctx, t, ctx->stream, nullptr, nullptr, nullptr, 0, nullptr, 0,
                               nullptr, nullptr);
  if (!rc) rc = finish_tree(ctx, t);
  if (rc) {
    free_tree_async(t, ctx->stream);
    return rc;
  }
  *out = t;
  return SPAMM_OK;
}

static int same_shape(const spamm_tree *a, const spamm_tree *b) {
  if (!a || !b) {
    set_error("null tree");
    return SPAMM_ERR_VALUE;
  }
  if (a->n != b->n || a->leaf != b->leaf) {  // quadtree.py:209-215
    set_error("trees not conformable: (%lld, leaf %d) vs (%lld, leaf %d)", (long long)a->n, a->leaf,
              (long long)b->n, b->leaf);
    return SPAMM_ERR_DIMENSION;
  }
  if (a->dtype != b->dtype || a->device != b->device) {
    set_error("trees differ in dtype or device");
    return SPAMM_ERR_VALUE;
  }
  return SPAMM_OK;
}

}  // namespace spamm

using namespace spamm;

extern "C" {

SPAMM_API int spamm_tree_add(const spamm_tree *a, const spamm_tree *b, spamm_tree **out) {
  SPAMM_TRY(same_shape(a, b));
  DeviceContext *ctx;
  SPAMM_TRY(get_context(a->device, &ctx));
  std::lock_guard<std::mutex> lk(ctx->mu);
  SPAMM_TRY(materialize(ctx, a));
  SPAMM_TRY(materialize(ctx, b));
  spamm_tree *t = nullptr;
  SPAMM_TRY(alloc_tree(ctx, a->n, a->leaf, a->dtype, &t));
  const uint8_t *oa = a->occ + level_offset(a->depth), *ob = b->occ + level_offset(b->depth);
  if (a->dtype == SPAMM_DTYPE_F64)
    add_kernel<double><<<grid_rows(ctx, a->N), 256, 0, ctx->stream>>>(
        (const double *)a->padded, (const double *)b->padded, (double *)t->padded, a->N, a->leaf,
        a->nb, oa, ob);
  else
    add_kernel<float><<<grid_rows(ctx, a->N), 256, 0, ctx->stream>>>(
        (const float *)a->padded, (const float *)b->padded, (float *)t->padded, a->N, a->leaf,
        a->nb, oa, ob);
  if (cudaGetLastError() != cudaSuccess) {
    free_tree_async(t, ctx->stream);
    set_error("add kernel launch failed");
    return SPAMM_ERR_CUDA;
  }
  return finish_new(ctx, t, out);
}

SPAMM_API int spamm_tree_scale(const spamm_tree *m, double s, spamm_tree **out) {
  if (!m) {
    set_error("null tree");
    return SPAMM_ERR_VALUE;
  }
  DeviceContext *ctx;
  SPAMM_TRY(get_context(m->device, &ctx));
  std::lock_guard<std::mutex> lk(ctx->mu);
  SPAMM_TRY(materialize(ctx, m));
  spamm_tree *t = nullptr;
  SPAMM_TRY(alloc_tree(ctx, m->n, m->leaf, m->dtype, &t));
  const int64_t count = m->N * m->N;
  const int grid = (int)std::min<int64_t>((count + 255) / 256, (int64_t)ctx->num_sms * 32);
  if (m->dtype == SPAMM_DTYPE_F64)
    scale_kernel<double><<<grid, 256, 0, ctx->stream>>>((const double *)m->padded,
                                                        (double *)t->padded, count, s);
  else
    scale_kernel<float><<<grid, 256, 0, ctx->stream>>>((const float *)m->padded, (float *)t->padded,
                                                       count, (float)s);
  if (cudaGetLastError() != cudaSuccess) {
    free_tree_async(t, ctx->stream);
    set_error("scale kernel launch failed");
    return SPAMM_ERR_CUDA;
  }
  return finish_new(ctx, t, out);
}

SPAMM_API int spamm_tree_filter_drop(const spamm_tree *m, double tau, spamm_tree **out,
                                     int32_t *dropped_any) {
  if (!m) {
    set_error("null tree");
    return SPAMM_ERR_VALUE;
  }
  if (!(tau >= 0.0)) {  // quadtree.py:309-310
    set_error("tau must be >= 0, got %g", tau);
    return SPAMM_ERR_VALUE;
  }
  DeviceContext *ctx;
  SPAMM_TRY(get_context(m->device, &ctx));
  std::lock_guard<std::mutex> lk(ctx->mu);
  SPAMM_TRY(materialize(ctx, m));
  const int64_t G = m->nb * m->nb;
  SPAMM_TRY(ensure_scratch(ctx->reduce_tmp, (size_t)G + 64, ctx->stream));
  uint8_t *drop = (uint8_t *)ctx->reduce_tmp.ptr + 64;
  unsigned *count = (unsigned *)ctx->reduce_tmp.ptr;
  SPAMM_CUDA_TRY(cudaMemsetAsync(count, 0, sizeof(unsigned), ctx->stream));
  drop_mark_kernel<<<(unsigned)std::min<int64_t>((G + 255) / 256, 4096), 256, 0, ctx->stream>>>(
      m->occ + level_offset(m->depth), m->nrm + level_offset(m->depth), G, tau, drop, count);
  unsigned *hc = (unsigned *)ctx->host_pinned;
  {
    const SmallRead r{hc, count, sizeof(unsigned)};
    SPAMM_TRY(read_small_sync(ctx, ctx->stream, &r, 1));
  }
  *dropped_any = *hc != 0;
  *out = nullptr;
  if (!*hc) return SPAMM_OK;  // nothing drops: the caller keeps the input tree
  spamm_tree *t = nullptr;
  SPAMM_TRY(alloc_tree(ctx, m->n, m->leaf, m->dtype, &t));
  if (m->dtype == SPAMM_DTYPE_F64)
    filter_kernel<double><<<grid_rows(ctx, m->N), 256, 0, ctx->stream>>>(
        (const double *)m->padded, (double *)t->padded, m->N, m->leaf, m->nb, drop);
  else
    filter_kernel<float><<<grid_rows(ctx, m->N), 256, 0, ctx->stream>>>(
        (const float *)m->padded, (float *)t->padded, m->N, m->leaf, m->nb, drop);
  return finish_new(ctx, t, out);
}

SPAMM_API int spamm_tree_blocks_to_host(const spamm_tree *m, const int64_t *ids, int64_t count,
                                        void *host_out) {
  if (!m || (count && !host_out) || count < 0) {
    set_error("null argument");
    return SPAMM_ERR_VALUE;
  }
  if (!count) return SPAMM_OK;
  DeviceContext *ctx;
  SPAMM_TRY(get_context(m->device, &ctx));
  std::lock_guard<std::mutex> lk(ctx->mu);
  SPAMM_TRY(tree_join(ctx, m));
  const int64_t esz = m->elem_size(), bytes = count * m->leaf * m->leaf * esz;
  SPAMM_TRY(ensure_scratch(ctx->reduce_tmp, (size_t)(bytes + count * 8 + 256), ctx->stream));
  int64_t *dids = (int64_t *)ctx->reduce_tmp.ptr;
  unsigned char *dbuf = (unsigned char *)ctx->reduce_tmp.ptr + ((count * 8 + 255) / 256) * 256;
  if (ids) {
    SPAMM_TRY(materialize(ctx, m));  // any block may be listed
    SPAMM_CUDA_TRY(cudaMemcpyAsync(dids, ids, count * 8, cudaMemcpyHostToDevice, ctx->stream));
  } else {  // every nonzero leaf, listed on the device
    occ_ids_kernel<<<1, 1024, 0, ctx->stream>>>(m->occ + level_offset(m->depth), m->nb * m->nb,
                                                dids);
  }
  for (int64_t q = 0; q < count; q += 65535) {
    const int64_t k = std::min<int64_t>(65535, count - q);
    gather_blocks_kernel<<<(unsigned)k, 256, 0, ctx->stream>>>(
        (const unsigned char *)m->padded, m->N, m->leaf, m->nb, (int)esz, dids + q,
        dbuf + q * m->leaf * m->leaf * esz);
  }
  SPAMM_CUDA_TRY(cudaGetLastError());
  SPAMM_CUDA_TRY(cudaMemcpyAsync(host_out, dbuf, bytes, cudaMemcpyDeviceToHost, ctx->stream));
  SPAMM_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  return SPAMM_OK;
}

// A pending device->host block transfer: the gather runs on the library's
// stream (ordered after the product that wrote the blocks), the copy on the
// context's copy-out stream, so the transfer overlaps whatever the caller
// launches next (the next multiply, or the next matrix's host->device copy:
// PCIe is full duplex).
}  // extern "C"
struct spamm_transfer {
  int device = 0;
  cudaEvent_t done = nullptr;
  spamm::Scratch staging;  // taken from / returned to the context's idle list
};
extern "C" {

SPAMM_API int spamm_tree_blocks_to_host_async(const spamm_tree *m, const int64_t *ids,
                                              int64_t count, void *host_out,
                                              spamm_transfer **out) {
  if (!m || !out || (count && !host_out) || count < 0) {
    set_error("null argument");
    return SPAMM_ERR_VALUE;
  }
  *out = nullptr;
  DeviceContext *ctx;
  SPAMM_TRY(get_context(m->device, &ctx));
  std::lock_guard<std::mutex> lk(ctx->mu);
  SPAMM_TRY(tree_join(ctx, m));
  auto *t = new spamm_transfer;
  t->device = m->device;
  const int64_t esz = m->elem_size(), bytes = count * m->leaf * m->leaf * esz;
  const int64_t id_bytes = ((count * 8 + 255) / 256) * 256;
  int rc = SPAMM_OK;
  do {
    cudaError_t e = cudaEventCreateWithFlags(&t->done, cudaEventDisableTiming);
    if (e == cudaSuccess && count) {
      // a persistent staging buffer (allocation-free in steady state)
      const size_t need = (size_t)(bytes + id_bytes);
      size_t best = ctx->xfer_free.size();
      for (size_t q = 0; q < ctx->xfer_free.size(); ++q)
        if (ctx->xfer_free[q].bytes >= need &&
            (best == ctx->xfer_free.size() || ctx->xfer_free[q].bytes < ctx->xfer_free[best].bytes))
          best = q;
      if (best < ctx->xfer_free.size()) {
        t->staging = ctx->xfer_free[best];
        ctx->xfer_free.erase(ctx->xfer_free.begin() + best);
      } else {
        e = cudaStreamSynchronize(ctx->stream);
        if (e == cudaSuccess) e = cudaMalloc(&t->staging.ptr, need);
        if (e == cudaSuccess) t->staging.bytes = need;
      }
    }
    if (e != cudaSuccess) {
      set_error("transfer setup: %s", cudaGetErrorString(e));
      rc = e == cudaErrorMemoryAllocation ? SPAMM_ERR_NOMEM : SPAMM_ERR_CUDA;
      break;
    }
    if (count) {
      int64_t *dids = (int64_t *)t->staging.ptr;
      unsigned char *dbuf = (unsigned char *)t->staging.ptr + id_bytes;
      if (ids) {
        SPAMM_TRY(materialize(ctx, m));  // any block may be listed
        e = cudaMemcpyAsync(dids, ids, count * 8, cudaMemcpyHostToDevice, ctx->stream);
      } else {
        // every nonzero leaf: ids from the occupancy pyramid on the device (no
        // host->device copy); occupied blocks are always defined
        occ_ids_kernel<<<1, 1024, 0, ctx->stream>>>(m->occ + level_offset(m->depth),
                                                    m->nb * m->nb, dids);
        e = cudaGetLastError();
      }
      for (int64_t q = 0; e == cudaSuccess && q < count; q += 65535) {
        const int64_t k = std::min<int64_t>(65535, count - q);
        gather_blocks_kernel<<<(unsigned)k, 256, 0, ctx->stream>>>(
            (const unsigned char *)m->padded, m->N, m->leaf, m->nb, (int)esz, dids + q,
            dbuf + q * m->leaf * m->leaf * esz);
        e = cudaGetLastError();
      }
      if (e == cudaSuccess) e = cudaEventRecord(ctx->join, ctx->stream);
      if (e == cudaSuccess) e = cudaStreamWaitEvent(ctx->copy_out, ctx->join, 0);
      if (e == cudaSuccess)
        e = cudaMemcpyAsync(host_out, dbuf, bytes, cudaMemcpyDeviceToHost, ctx->copy_out);
    }
    if (e == cudaSuccess) e = cudaEventRecord(t->done, count ? ctx->copy_out : ctx->stream);
    if (e != cudaSuccess) {
      set_error("transfer: %s", cudaGetErrorString(e));
      rc = SPAMM_ERR_CUDA;
    }
  } while (0);
  if (rc) {
    if (t->staging.ptr) {
      cudaStreamSynchronize(ctx->stream);
      ctx->xfer_free.push_back(t->staging);
    }
    if (t->done) cudaEventDestroy(t->done);
    delete t;
    return rc;
  }
  *out = t;
  return SPAMM_OK;
}

SPAMM_API int spamm_transfer_wait(spamm_transfer *t) {
  if (!t) {
    set_error("null transfer");
    return SPAMM_ERR_VALUE;
  }
  const cudaError_t e = cudaEventSynchronize(t->done);
  if (t->staging.ptr) {  // the copy is complete: the buffer is idle again
    DeviceContext *ctx;
    if (get_context(t->device, &ctx) == SPAMM_OK) {
      std::lock_guard<std::mutex> lk(ctx->mu);
      ctx->xfer_free.push_back(t->staging);
    }
  }
  cudaEventDestroy(t->done);
  delete t;
  if (e != cudaSuccess) {
    set_error("transfer: %s", cudaGetErrorString(e));
    return SPAMM_ERR_CUDA;
  }
  return SPAMM_OK;
}

SPAMM_API int spamm_tree_diagonal(const spamm_tree *m, void *host_out) {
  if (!m || !host_out) {
    set_error("null argument");
    return SPAMM_ERR_VALUE;
  }
  DeviceContext *ctx;
  SPAMM_TRY(get_context(m->device, &ctx));
  std::lock_guard<std::mutex> lk(ctx->mu);
  SPAMM_TRY(materialize(ctx, m));
  const int64_t esz = m->elem_size();
  SPAMM_CUDA_TRY(cudaMemcpy2DAsync(host_out, (size_t)esz, m->padded, (size_t)((m->N + 1) * esz),
                                   (size_t)esz, (size_t)m->n, cudaMemcpyDeviceToHost, ctx->stream));
  SPAMM_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  return SPAMM_OK;
}

}  // extern "C"
