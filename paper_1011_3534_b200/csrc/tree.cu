// tree.cu -- quadtree construction on the device: padding (K4), the
// bit-exact leaf norm kernel (K1) and the norm/occupancy pyramid, plus the
// tree half of the C ABI and the per-device context.
//
// Reference: quadtree.py:116-151 (QuadTreeMatrix.__init__), :74-87
// (_leaf_norm_sq), :90-92 (_aggregate_norm_sq), :218-251 (from_dense).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <vector>

#include "common.cuh"
#include "norms.cuh"

namespace spamm {

// ------------------------------------------------------------------ errors
static thread_local std::string g_last_error;

void set_error(const char *fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_last_error = buf;
}

// ----------------------------------------------------------------- contexts
static std::mutex g_ctx_mu;
static std::vector<std::unique_ptr<DeviceContext>> g_ctx;

int get_context(int device, DeviceContext **out) {
  std::lock_guard<std::mutex> lk(g_ctx_mu);
  int count = 0;
  SPAMM_CUDA_TRY(cudaGetDeviceCount(&count));
  if (device < 0 || device >= count) {
    set_error("CUDA device %d not available (%d visible)", device, count);
    return SPAMM_ERR_VALUE;
  }
  if ((int)g_ctx.size() < count) g_ctx.resize(count);
  if (!g_ctx[device]) {
    auto ctx = std::make_unique<DeviceContext>();
    ctx->device = device;
    SPAMM_CUDA_TRY(cudaSetDevice(device));
    SPAMM_CUDA_TRY(cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, device));
    SPAMM_CUDA_TRY(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
    SPAMM_CUDA_TRY(cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking));
    SPAMM_CUDA_TRY(cudaStreamCreateWithFlags(&ctx->copy_out, cudaStreamNonBlocking));
    SPAMM_CUDA_TRY(cudaStreamCreateWithFlags(&ctx->copy_in, cudaStreamNonBlocking));
    SPAMM_CUDA_TRY(cudaEventCreateWithFlags(&ctx->fork, cudaEventDisableTiming));
    SPAMM_CUDA_TRY(cudaEventCreateWithFlags(&ctx->join, cudaEventDisableTiming));
    SPAMM_CUDA_TRY(cudaEventCreateWithFlags(&ctx->handoff, cudaEventDisableTiming));
    for (auto &e : ctx->ev) SPAMM_CUDA_TRY(cudaEventCreate(&e));
    SPAMM_CUDA_TRY(cudaMallocHost(&ctx->host_pinned, 1 << 16));
    // keep freed pool memory cached between calls (stream-ordered allocator)
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
      uint64_t thresh = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thresh);
    }
    g_ctx[device] = std::move(ctx);
  }
  *out = g_ctx[device].get();
  SPAMM_CUDA_TRY(cudaSetDevice(device));
  return SPAMM_OK;
}

__global__ void zero_fill_kernel(unsigned char *__restrict__ p, size_t bytes) {
  const size_t head = (16 - ((uintptr_t)p & 15)) & 15;
  const size_t h = head < bytes ? head : bytes;
  const size_t body = (bytes - h) / 16, tail0 = h + body * 16;
  const size_t tid = (size_t)blockIdx.x * blockDim.x + threadIdx.x,
               stride = (size_t)gridDim.x * blockDim.x;
  uint4 *q = reinterpret_cast<uint4 *>(p + h);
  for (size_t i = tid; i < body; i += stride) q[i] = make_uint4(0u, 0u, 0u, 0u);
  if (tid < h) p[tid] = 0;
  if (tid < bytes - tail0) p[tail0 + tid] = 0;
}

int zero_async(void *p, size_t bytes, cudaStream_t st, int ctas) {
  if (!bytes) return SPAMM_OK;
  const size_t want = (bytes / 16 + 255) / 256 + 1;
  const unsigned grid = (unsigned)std::min<size_t>(want, (size_t)std::max(ctas, 1));
  zero_fill_kernel<<<grid, 256, 0, st>>>((unsigned char *)p, bytes);
  SPAMM_CUDA_TRY(cudaGetLastError());
  return SPAMM_OK;
}

// dst: pinned host memory (device-visible through UVA)
__global__ void store_to_host_kernel(unsigned char *__restrict__ dst,
                                     const unsigned char *__restrict__ src, size_t bytes) {
  const size_t tid = (size_t)blockIdx.x * blockDim.x + threadIdx.x,
               stride = (size_t)gridDim.x * blockDim.x;
  if ((((uintptr_t)dst | (uintptr_t)src) & 15) == 0) {
    const size_t q = bytes / 16;
    for (size_t i = tid; i < q; i += stride)
      reinterpret_cast<uint4 *>(dst)[i] = reinterpret_cast<const uint4 *>(src)[i];
    for (size_t i = q * 16 + tid; i < bytes; i += stride) dst[i] = src[i];
  } else {
    for (size_t i = tid; i < bytes; i += stride) dst[i] = src[i];
  }
}

int read_small_sync(DeviceContext *ctx, cudaStream_t st, const SmallRead *r, int n) {
  size_t total = 0;
  for (int q = 0; q < n; ++q) total += (r[q].bytes + 255) / 256 * 256;
  if (ctx->host_stage.bytes < total) {
    SPAMM_CUDA_TRY(cudaStreamSynchronize(st));  // the old stage may be in use by st
    if (ctx->host_stage.ptr) SPAMM_CUDA_TRY(cudaFreeHost(ctx->host_stage.ptr));
    ctx->host_stage.ptr = nullptr;
    ctx->host_stage.bytes = 0;
    const size_t want = std::max<size_t>(total + total / 4, 1 << 16);
    SPAMM_CUDA_TRY(cudaMallocHost(&ctx->host_stage.ptr, want));
    ctx->host_stage.bytes = want;
  }
  unsigned char *stage = (unsigned char *)ctx->host_stage.ptr;
  size_t off = 0;
  for (int q = 0; q < n; ++q) {
    if (r[q].bytes) {
      const unsigned grid = (unsigned)std::min<size_t>((r[q].bytes / 16 + 255) / 256 + 1, 64);
      store_to_host_kernel<<<grid, 256, 0, st>>>(stage + off, (const unsigned char *)r[q].dev,
                                                 r[q].bytes);
    }
    off += (r[q].bytes + 255) / 256 * 256;
  }
  SPAMM_CUDA_TRY(cudaGetLastError());
  SPAMM_CUDA_TRY(cudaStreamSynchronize(st));
  off = 0;
  for (int q = 0; q < n; ++q) {
    if (r[q].bytes && r[q].host != stage + off) memcpy(r[q].host, stage + off, r[q].bytes);
    off += (r[q].bytes + 255) / 256 * 256;
  }
  return SPAMM_OK;
}

cudaError_t dev_alloc(void **p, size_t bytes, cudaStream_t st) {
  static const int poison = getenv("SPAMM_POISON") ? (int)strtol(getenv("SPAMM_POISON"), nullptr, 0) : -1;
  cudaError_t e = cudaMallocAsync(p, bytes, st);
  if (e == cudaSuccess && poison >= 0 && bytes) e = cudaMemsetAsync(*p, poison & 0xff, bytes, st);
  return e;
}

int ensure_scratch(Scratch &s, size_t bytes, cudaStream_t stream, bool zeroed) {
  if (s.bytes >= bytes) return SPAMM_OK;
  if (s.ptr) SPAMM_CUDA_TRY(cudaFreeAsync(s.ptr, stream));
  s.ptr = nullptr;
  s.bytes = 0;
  size_t want = bytes + bytes / 4 + 256;
  SPAMM_CUDA_TRY(dev_alloc((void **)&s.ptr, want, stream));
  s.bytes = want;
  if (zeroed) SPAMM_TRY(zero_async(s.ptr, want, stream, 1024));
  return SPAMM_OK;
}

// ================================================================ K1 kernels
//
// One thread owns one leaf and accumulates its squared Frobenius norm in the
// reference's order: row-major over the leaf, acc = rn(acc + rn(x*x)), with
// no FMA contraction (quadtree.py:80-87; __dmul_rn/__dadd_rn pin the
// rounding).  The parallelism is across leaves only -- a per-leaf shuffle
// tree would change the bits the strict `< tau` tests compare.
//
// Data movement (warp-specialised): a CTA owns K1_LT (8 or 32) leaves.
//   warps 2-3  stream the leaves through a K1_STAGES-deep ring of
//              512-byte-per-leaf stages with cp.async; their copies arrive on
//              the stage's "full" mbarrier as they land;
//   warps 1-4  (f64) square every element in place, rn(x*x), and OR the
//              raw bit patterns for the occupancy / -0.0 tests (each warp a
//              quarter of every leaf's segments), then arrive on "squared";
//   warp 0     runs the 32 sequential chains acc = rn(acc + sq) -- nothing
//              else sits on the dependent-add critical path -- and releases
//              the stage on "empty".
// For f32 storage warp 0 also forms the squares (the f64 squares would not
// fit in place).  Stages carry 16 B of padding per leaf, so the per-lane
// LDS.128 reads are bank-conflict free while every global read uses whole
// 128-byte lines.
constexpr int K1_SQ_WARPS = 3;                 // squarer warps (f64): SMSPs 1-3, never the chain warp's
constexpr int K1_PRODUCERS = 64;
// (A spacer warp that keeps the producers off the chain warp's SMSP was
// measured not to matter here; K1_SPACER = 32 re-enables it.)
constexpr int K1_SPACER = 0;
constexpr int K1_THREADS = 32 * (1 + K1_SQ_WARPS) + K1_SPACER + K1_PRODUCERS;
constexpr int K1_CHUNK = 512;                  // bytes per leaf per stage
constexpr int K1_LEAF_STRIDE = K1_CHUNK + 16;  // smem bytes per leaf per stage

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count) {
  asm volatile("mbarrier.init.shared.b64 [%0], %1;\n" ::"r"((unsigned)__cvta_generic_to_shared(bar)),
               "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.shared.b64 st, [%0];\n}\n" ::"r"(
      (unsigned)__cvta_generic_to_shared(bar)));
}
// the calling thread's prior cp.async copies arrive on `bar` when they land
__device__ __forceinline__ void cp_async_mbar_arrive(uint64_t *bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared.b64 [%0];\n" ::"r"(
      (unsigned)__cvta_generic_to_shared(bar)));
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"((unsigned)__cvta_generic_to_shared(bar)),
      "r"(parity));
}

// Waits of the helper warps back off, so a helper that is far ahead never
// competes for issue slots with the chain warp on its SMSP.
__device__ __forceinline__ void mbar_wait_backoff(uint64_t *bar, unsigned parity) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  for (;;) {
    unsigned ok;
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.test_wait.parity.shared.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok) : "r"(a), "r"(parity) : "memory");
    if (ok) return;
    __nanosleep(64);
  }
}

// acc = rn(acc + rn(x*x)) in f64, the reference's per-element step; `bits`
// ORs the raw patterns: (bits << 1) != 0 <=> some element is nonzero (NaN
// included), bits != 0 with zero magnitude <=> a -0.0 was seen.
template <typename T>
__device__ __forceinline__ void accum(double &acc, typename Bits<T>::U &bits, T x) {
  bits |= Bits<T>::of(x);
  const double e = (double)x;
  acc = __dadd_rn(acc, __dmul_rn(e, e));
}

template <typename T>
__device__ void canonicalise_leaf(T *padded, int64_t N, int32_t b, int64_t bi, int64_t bj) {
  for (int r = 0; r < b; ++r) {
    T *row = padded + (bi * b + r) * N + bj * b;
    for (int c = 0; c < b; ++c) row[c] = T(0);
  }
}

// Warp-cooperative form (all 32 lanes call it): every flagged lane's leaf is
// zeroed by the whole warp with coalesced stores.  (One lane storing its own
// 4096 elements made a c5 build, where the 19 % of the leaves that hold only
// underflowed +-0.0 are rewritten, spend most of its time here.)
template <typename T>
__device__ void canonicalise_leaves_warp(T *padded, int64_t N, int32_t b, int64_t nb, bool flag,
                                         int64_t leaf) {
  unsigned m = __ballot_sync(0xffffffffu, flag);
  const int lane = threadIdx.x & 31;
  const bool vec = ((int64_t)b * sizeof(T)) % 16 == 0 && (N * sizeof(T)) % 16 == 0 &&
                   ((uintptr_t)padded & 15) == 0;
  while (m) {
    const int src = __ffs(m) - 1;
    m &= m - 1;
    const int64_t lf = __shfl_sync(0xffffffffu, leaf, src);
    const int64_t bi = lf / nb, bj = lf - bi * nb;
    T *base = padded + (bi * b) * N + bj * b;
    if (vec) {
      const int spr = b * (int)sizeof(T) / 16;  // 16-byte segments per leaf row
      for (int idx = lane; idx < b * spr; idx += 32) {
        const int r = idx / spr, c = idx - r * spr;
        reinterpret_cast<uint4 *>(base + (int64_t)r * N)[c] = make_uint4(0u, 0u, 0u, 0u);
      }
    } else {
      for (int idx = lane; idx < b * b; idx += 32) {
        const int r = idx / b, c = idx - r * b;
        base[(int64_t)r * N + c] = T(0);
      }
    }
  }
}

// Staged kernel: requires b * sizeof(T) >= 16.
__device__ unsigned long long *g_k1_tl = nullptr;

template <typename T, int K1_STAGES, int K1_LT>
__global__ void __launch_bounds__(K1_THREADS) leaf_norm_staged_kernel(T *__restrict__ padded,
                                                                      int64_t N, int32_t b,
                                                                      int64_t nb,
                                                                      double *__restrict__ nsq_leaf,
                                                                      uint8_t *__restrict__ occ_leaf,
                                                                      const uint32_t *__restrict__ list,
                                                                      const unsigned *list_count,
                                                                      PyrTail tail) {
  using U = typename Bits<T>::U;
  constexpr bool SQUARER = sizeof(T) == 8;  // warps 1-4 square in place (f64 only)
  constexpr int K1_STAGE_BYTES = K1_LT * K1_LEAF_STRIDE;
  extern __shared__ __align__(16) unsigned char k1_smem[];
  __shared__ __align__(8) uint64_t full_bar[K1_STAGES], sq_bar[K1_STAGES], empty_bar[K1_STAGES];
  __shared__ U s_bits[K1_SQ_WARPS][K1_LT];
  // dense mode: every leaf; list mode: only the listed leaves (C blocks that
  // received products -- every other leaf of C is exactly zero)
  // launched as a programmatic dependent of the leaf-product kernel: the CTA
  // may be resident before that kernel finishes; without per-group counters
  // it waits for the whole grid (and its stores) here
  if (tail.pdl_wait) asm volatile("griddepcontrol.wait;\n" ::: "memory");
  if (tail.ready) {
    if (threadIdx.x == 0) spin_acquire_nonzero(tail.ready);
    __syncthreads();
  }
  const int64_t n_leaves = list ? (int64_t)*list_count : nb * nb;
  const int64_t leaf0 = (int64_t)blockIdx.x * K1_LT;
  if (leaf0 < n_leaves) {
  unsigned long long *const k1_tl = g_k1_tl;  // optional timeline (SPAMM_K1_TIMELINE)
  if (k1_tl && threadIdx.x == 0) k1_tl[4 * blockIdx.x] = k1_gt();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t bb = (int64_t)b * b;
  const int EPC = (int)(bb < K1_CHUNK / (int)sizeof(T) ? bb : K1_CHUNK / (int)sizeof(T));
  const int CW = b < EPC ? b : EPC;      // chunk width (elements)
  const int R = EPC / CW;                // rows per chunk
  const int chunks_per_row = b / CW;     // a power of two
  const int n_chunks = (b / R) * chunks_per_row;
  const int segs = EPC * (int)sizeof(T) / 16;  // 16-byte segments per leaf chunk
  constexpr int EPS = 16 / (int)sizeof(T);     // elements per segment
  const bool mine = lane < K1_LT && leaf0 + lane < n_leaves;

  if (tid == 0) {
    for (int s = 0; s < K1_STAGES; ++s) {
      mbar_init(&full_bar[s], K1_PRODUCERS);
      mbar_init(&sq_bar[s], K1_SQ_WARPS);
      mbar_init(&empty_bar[s], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
  }
  __syncthreads();

  if (K1_SPACER && warp == 1 + K1_SQ_WARPS) {
    // spacer: nothing to do
  } else if (warp >= 1 + K1_SQ_WARPS + K1_SPACER / 32) {
    // ------------------------------------------------------------ producers
    const int p = tid - 32 * (1 + K1_SQ_WARPS) - K1_SPACER;
    const T *fsrc = SQUARER ? reinterpret_cast<const T *>(tail.fuse_src) : nullptr;
    const int64_t sld = fsrc ? tail.fuse_ld : N;  // the source's leading dimension
    constexpr int MAX_SLOTS = (K1_LT * (K1_CHUNK / 16) + K1_PRODUCERS - 1) / K1_PRODUCERS;
    const T *slot_ptr[MAX_SLOTS];
    unsigned slot_dst[MAX_SLOTS];
#pragma unroll
    for (int q = 0; q < MAX_SLOTS; ++q) {
      const int sidx = p + q * K1_PRODUCERS;
      slot_ptr[q] = nullptr;
      slot_dst[q] = 0;
      if (sidx < K1_LT * segs) {
        const int l = sidx / segs, part = sidx - l * segs;
        const int64_t lx = leaf0 + l;
        if (lx < n_leaves) {
          const int64_t leaf = list ? (int64_t)list[lx] : lx;
          const int64_t bi = leaf / nb, bj = leaf - bi * nb;
          const int e = part * EPS;
          const int rr = e / CW, cc = e - rr * CW;
          slot_ptr[q] = fsrc ? fsrc + (bi * b + rr) * sld + bj * b + cc
                             : padded + (bi * b + rr) * N + bj * b + cc;
          slot_dst[q] = l * K1_LEAF_STRIDE + part * 16;
        }
      }
    }
    const int shift_cpr = __ffs(chunks_per_row) - 1;
    if (tail.grp_done && (!tail.overflow || !*(volatile const int *)tail.overflow)) {
      // wait until the leaf-product kernel has stored each of this thread's leaves
#pragma unroll
      for (int q = 0; q < MAX_SLOTS; ++q) {
        const int sidx = p + q * K1_PRODUCERS;
        if (slot_ptr[q] && (q == 0 || sidx / segs != (sidx - K1_PRODUCERS) / segs)) {
          const unsigned *flag = tail.grp_done + leaf0 + sidx / segs;
          for (;;) {
            unsigned v;
            asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
            if (v >= tail.grp_target) break;
            __nanosleep(256);
          }
        }
      }
    }
    for (int chunk = 0; chunk < n_chunks; ++chunk) {
      const int stage = chunk % K1_STAGES;
      if (chunk >= K1_STAGES) mbar_wait_backoff(&empty_bar[stage], ((chunk / K1_STAGES) - 1) & 1);
      const int64_t off =
          (int64_t)((chunk >> shift_cpr) * R) * sld + (chunk & (chunks_per_row - 1)) * CW;
      unsigned char *base = k1_smem + stage * K1_STAGE_BYTES;
#pragma unroll
      for (int q = 0; q < MAX_SLOTS; ++q)
        if (slot_ptr[q]) cp_async16(base + slot_dst[q], slot_ptr[q] + off);
      cp_async_mbar_arrive(&full_bar[stage]);
    }
    cp_async_wait<0>();
  } else if (warp >= 1) {
    // ------------------------------------------------ squarers (f64 only)
    if (SQUARER) {
      const int sw = warp - 1;  // segments [sw*segs/4, (sw+1)*segs/4) of every leaf
      const int v0 = sw * segs / K1_SQ_WARPS, v1 = (sw + 1) * segs / K1_SQ_WARPS;
      U bits = 0;
      // fused build: this lane's leaf in the tree's storage (raw values are
      // written there as they pass through the stage)
      // fused build: this lane's leaf in the tree's storage (raw values are
      // written there as they pass through the stage, before the squaring)
      T *fdst = nullptr;
      if (tail.fuse_src && mine) {
        const int64_t leaf = list ? (int64_t)list[leaf0 + lane] : leaf0 + lane;
        const int64_t bi = leaf / nb, bj = leaf - bi * nb;
        fdst = padded + (bi * b) * N + bj * b;
      }
      for (int chunk = 0; chunk < n_chunks; ++chunk) {
        const int stage = chunk % K1_STAGES;
        mbar_wait_backoff(&full_bar[stage], (chunk / K1_STAGES) & 1);
        if (mine) {
          unsigned char *pp = k1_smem + stage * K1_STAGE_BYTES + lane * K1_LEAF_STRIDE;
          // (fused build) where piece v of this chunk goes in the tree's storage
          T *crow = fdst ? fdst + (int64_t)((chunk >> (__ffs(chunks_per_row) - 1)) * R) * N +
                               (chunk & (chunks_per_row - 1)) * CW
                         : nullptr;
          auto raw_out = [&](int v, const double2 &w) {
            const int e = v * EPS, rr = e / CW, cc = e - rr * CW;
            *reinterpret_cast<double2 *>(crow + (int64_t)rr * N + cc) = w;
          };
          int v = v0;
          for (; v + 8 <= v1; v += 8) {  // batched: loads, then squares, then stores
            double2 w[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) w[u] = *reinterpret_cast<double2 *>(pp + 16 * (v + u));
            if (crow)
#pragma unroll
              for (int u = 0; u < 8; ++u) raw_out(v + u, w[u]);
#pragma unroll
            for (int u = 0; u < 8; ++u) {
              bits |= Bits<T>::of((T)w[u].x) | Bits<T>::of((T)w[u].y);
              w[u].x = __dmul_rn(w[u].x, w[u].x);
              w[u].y = __dmul_rn(w[u].y, w[u].y);
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) *reinterpret_cast<double2 *>(pp + 16 * (v + u)) = w[u];
          }
          for (; v < v1; ++v) {
            double2 w = *reinterpret_cast<double2 *>(pp + 16 * v);
            if (crow) raw_out(v, w);
            bits |= Bits<T>::of((T)w.x) | Bits<T>::of((T)w.y);
            w.x = __dmul_rn(w.x, w.x);
            w.y = __dmul_rn(w.y, w.y);
            *reinterpret_cast<double2 *>(pp + 16 * v) = w;
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&sq_bar[stage]);
      }
      if (lane < K1_LT) s_bits[sw][lane] = bits;
      // hand the bit ORs to warp 0
      asm volatile("bar.sync 1, %0;\n" ::"n"(32 * (1 + K1_SQ_WARPS)) : "memory");
    }
  } else {
  // --------------------------------------------------------------- warp 0
  double acc = 0.0;
  U bits = 0;
  for (int chunk = 0; chunk < n_chunks; ++chunk) {
    const int stage = chunk % K1_STAGES;
    mbar_wait(SQUARER ? &sq_bar[stage] : &full_bar[stage], (chunk / K1_STAGES) & 1);
    if (k1_tl && lane == 0 && chunk == 0) k1_tl[4 * blockIdx.x + 1] = k1_gt();
    if (mine && SQUARER && segs == 32) {
      // the common case (every leaf of >= 64 elements): 4 batches of 8
      // segments, fully unrolled so the next batch's shared loads are in
      // flight under the current batch's 16 dependent adds
      const unsigned char *pp = k1_smem + stage * K1_STAGE_BYTES + lane * K1_LEAF_STRIDE;
      double2 w[32];
#pragma unroll
      for (int u = 0; u < 32; ++u) w[u] = *reinterpret_cast<const double2 *>(pp + 16 * u);
#pragma unroll
      for (int u = 0; u < 32; ++u) {
        acc = __dadd_rn(acc, w[u].x);
        acc = __dadd_rn(acc, w[u].y);
      }
    } else if (mine && SQUARER) {
      const unsigned char *pp = k1_smem + stage * K1_STAGE_BYTES + lane * K1_LEAF_STRIDE;
      for (int v = 0; v < segs; ++v) {
        const double2 w = *reinterpret_cast<const double2 *>(pp + 16 * v);
        acc = __dadd_rn(acc, w.x);
        acc = __dadd_rn(acc, w.y);
      }
    } else if (mine) {
      const unsigned char *pp = k1_smem + stage * K1_STAGE_BYTES + lane * K1_LEAF_STRIDE;
      int v = 0;
      for (; v + 8 <= segs; v += 8) {
          uint4 w[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) w[u] = *reinterpret_cast<const uint4 *>(pp + 16 * (v + u));
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            if (SQUARER) {
              const double *q2 = reinterpret_cast<const double *>(&w[u]);
              acc = __dadd_rn(acc, q2[0]);
              acc = __dadd_rn(acc, q2[1]);
            } else {
              const T *x = reinterpret_cast<const T *>(&w[u]);
#pragma unroll
              for (int e = 0; e < EPS; ++e) accum<T>(acc, bits, x[e]);
            }
          }
        }
        for (; v < segs; ++v) {
          const uint4 w = *reinterpret_cast<const uint4 *>(pp + 16 * v);
          if (SQUARER) {
            const double *q2 = reinterpret_cast<const double *>(&w);
            acc = __dadd_rn(acc, q2[0]);
            acc = __dadd_rn(acc, q2[1]);
          } else {
            const T *x = reinterpret_cast<const T *>(&w);
#pragma unroll
            for (int e = 0; e < EPS; ++e) accum<T>(acc, bits, x[e]);
          }
        }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty_bar[stage]);
  }
  if (SQUARER) {
    asm volatile("bar.sync 1, %0;\n" ::"n"(32 * (1 + K1_SQ_WARPS)) : "memory");
#pragma unroll
    for (int q = 0; q < K1_SQ_WARPS; ++q) bits |= lane < K1_LT ? s_bits[q][lane] : 0;
  }
  if (k1_tl && lane == 0) k1_tl[4 * blockIdx.x + 3] = k1_gt();
  bool canon = false;
  int64_t canon_leaf = 0;
  if (mine) {
    const int64_t lx = leaf0 + lane;
    const int64_t leaf = list ? (int64_t)list[lx] : lx;
    const bool nz = (U)(bits << 1) != 0;
    nsq_leaf[leaf] = acc;
    occ_leaf[leaf] = (uint8_t)nz;
    tail.nrm[level_offset(tail.depth) + leaf] = __dsqrt_rn(acc);
    if (tail.grp_done) tail.grp_done[lx] = 0u;  // zero at rest for the next product
    canon = !nz && bits;  // only -0.0 entries: stored as +0.0 (quadtree.py:127-129)
    canon_leaf = leaf;
  }
  __syncwarp();
  canonicalise_leaves_warp<T>(padded, N, b, nb, canon, canon_leaf);
  }  // warp 0
  }  // leaf0 < n_leaves
  if (tail.ticket) {  // the last CTA builds the pyramid
    __shared__ int s_last;
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      s_last = atomicAdd(tail.ticket, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (s_last) {
      if (tail.trav_done && threadIdx.x == 0) spin_acquire_nonzero(tail.trav_done);
      __threadfence();
      pyramid_cta(tail, k1_smem, (size_t)K1_STAGES * K1_LT * K1_LEAF_STRIDE);
      if (threadIdx.x == 0) {
        *tail.ticket = 0u;
        if (tail.t_end) *tail.t_end = k1_gt();
      }
    }
  }
}

// ------------------------------------------------ K1, dense rows (TMA-fed)
// Dense builds of large trees (leaf 64, every leaf, block rows of a multiple
// of 32 leaves) are HBM-bound: 32 KB read per leaf against one 4096-long add
// chain.  Persistent kernel, one 4-warp CTA per SM, every warp on its own
// SMSP and self-contained:
//   * a warp owns 32 adjacent leaves of a block row at a time (lane = leaf);
//     one matrix row of the group is 32 x (64 elements) contiguous in memory
//     and arrives with ONE TMA tensor load per stage into the warp's own
//     ROWS_R-stage ring (mbarrier completion).  The 4-D box {128 bytes,
//     32 leaves, 128-byte pieces of the leaf row, 1 matrix row} puts piece j
//     of leaf l in shared line j * 32 + l, and the 128-byte swizzle rotates
//     the line's 16-byte chunks by l & 7: the per-lane LDS.128 reads (lane =
//     leaf, a stride that would otherwise hit one bank group) are conflict
//     free with no padding;
//   * the lane squares and accumulates in the reference's order,
//     acc = rn(acc + rn(x * x)) (quadtree.py:80-87), ORs the raw bits
//     (occupancy, -0.0), and lane 0 re-issues the stage's next load itself --
//     no producer warp, no empty barriers, the ring carries on across groups;
//   * fused build (the source is not the tree's storage): lane 0 stores the
//     raw stage into the tree with one TMA tensor store (shared -> global,
//     the same box) while the warp runs the chains, and waits for the store's
//     read of the stage before the stage is refilled.
// Groups are dealt round-robin to the grid's warps.  (Per-lane 512-byte bulk
// copies instead of the tensor box measured 4.0 TB/s: the 32-way serialised
// UBLKCP issue, ~70 cycles each, was the limiter.)
constexpr int ROWS_WARPS = 4;
constexpr int ROWS_LEAF = 64;
// SPAMM_K1_ROWS_DEBUG: per-warp {cycles waiting for data, cycles in all, chunks}
__device__ unsigned long long *g_rows_dbg = nullptr;

__device__ __forceinline__ void tma_load_4d(unsigned smem, const CUtensorMap *map, int c0, int c1, int c2,
                                            int c3, unsigned bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
      "%3, %4, %5}], [%6];\n" ::"r"(smem),
      "l"((uint64_t)map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void tma_store_4d(const CUtensorMap *map, int c0, int c1, int c2, int c3,
                                             unsigned smem) {
  asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4}], [%5];\n" ::"l"(
                   (uint64_t)map),
               "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem)
               : "memory");
}

template <typename T, int R>
__global__ void __launch_bounds__(32 * ROWS_WARPS, 1)
    leaf_norm_rows_kernel(const __grid_constant__ CUtensorMap tm_src,
                          const __grid_constant__ CUtensorMap tm_dst, int fuse, T *padded, int64_t N,
                          int64_t nb, int gpr_shift, double *__restrict__ nsq_leaf,
                          uint8_t *__restrict__ occ_leaf, double *__restrict__ nrm_leaf) {
  using U = typename Bits<T>::U;
  constexpr int ROWB = ROWS_LEAF * (int)sizeof(T);  // bytes of one leaf row
  constexpr int PIECES = ROWB / 128;                // 128-byte pieces per leaf row
  constexpr int STAGE = 32 * ROWB;
  constexpr int EPS = 16 / (int)sizeof(T);
  extern __shared__ unsigned char rows_smem_raw[];
  __shared__ __align__(8) uint64_t rows_bar[ROWS_WARPS][R];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t G = nb << gpr_shift;    // groups in all (2^gpr_shift = nb / 32 per block row)
  const int64_t W = (int64_t)gridDim.x * ROWS_WARPS;
  const int64_t w0 = (int64_t)blockIdx.x + (int64_t)warp * gridDim.x;  // CTA-major deal
  // 1024-byte aligned stages (the swizzle pattern is a function of the address)
  const unsigned base = ((unsigned)__cvta_generic_to_shared(rows_smem_raw) + 1023u) & ~1023u;
  const unsigned ring = base + warp * R * STAGE;
  const unsigned bar0 = (unsigned)__cvta_generic_to_shared(&rows_bar[warp][0]);
  if (lane == 0) {
    for (int s = 0; s < R; ++s) mbar_init(&rows_bar[warp][s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
  }
  __syncwarp();
  if (w0 >= G) return;
  const int64_t my_groups = (G - w0 + W - 1) / W;
  const int64_t Q = my_groups * ROWS_LEAF;  // chunks (matrix rows of a group) this warp streams
  const int64_t gmask = ((int64_t)1 << gpr_shift) - 1;

  // (lane 0) chunk q = row q & 63 of this warp's group q >> 6, into stage q % R
  auto issue = [&](int64_t q) {
    const int64_t g = w0 + (q >> 6) * W;
    const int s = (int)(q % R);
    asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.expect_tx.shared.b64 st, [%0], %1;\n}\n" ::"r"(
                     bar0 + 8 * s),
                 "r"((unsigned)STAGE)
                 : "memory");
    tma_load_4d(ring + s * STAGE, &tm_src, 0, (int)((g & gmask) << 5), 0,
                (int)((g >> gpr_shift) * ROWS_LEAF + (q & 63)), bar0 + 8 * s);
  };
  if (lane == 0)
    for (int64_t q = 0; q < R && q < Q; ++q) issue(q);

  // this lane's chunk c of piece j sits at line j * 32 + lane, chunk c ^ (lane & 7)
  const unsigned lane_off = (unsigned)lane * 128u;
  const unsigned sw = (unsigned)(lane & 7);
  double acc = 0.0;
  U bits = 0;
  unsigned long long *const dbg = g_rows_dbg;
  long long t_wait = 0, t_begin = dbg ? clock64() : 0;
  for (int64_t q = 0; q < Q; ++q) {
    const int s = (int)(q % R);
    const long long tw = dbg ? clock64() : 0;
    mbar_wait(&rows_bar[warp][s], (unsigned)((q / R) & 1));
    if (dbg) t_wait += clock64() - tw;
    const int64_t g = w0 + (q >> 6) * W;
    const int64_t bi = g >> gpr_shift;
    const int bj0 = (int)((g & gmask) << 5);
    const int r = (int)(q & 63);
    if (fuse && lane == 0) {
      tma_store_4d(&tm_dst, 0, bj0, 0, (int)(bi * ROWS_LEAF + r), ring + s * STAGE);
      asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
    }
    const unsigned st = ring + s * STAGE + lane_off;
    uint4 w[PIECES * 8];
#pragma unroll
    for (int j = 0; j < PIECES; ++j)
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const unsigned a = st + j * 4096 + (((unsigned)c ^ sw) << 4);
        asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];\n"
                     : "=r"(w[j * 8 + c].x), "=r"(w[j * 8 + c].y), "=r"(w[j * 8 + c].z), "=r"(w[j * 8 + c].w)
                     : "r"(a));
      }
#pragma unroll
    for (int u = 0; u < PIECES * 8; ++u) {
      const T *x = reinterpret_cast<const T *>(&w[u]);
#pragma unroll
      for (int e = 0; e < EPS; ++e) accum<T>(acc, bits, x[e]);
    }
    if (fuse && lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
    __syncwarp();
    if (lane == 0 && q + R < Q) issue(q + R);
    if (r == 63) {  // the group's last row: publish the leaf
      const int64_t bj = bj0 + lane;
      const int64_t leaf = bi * nb + bj;
      const bool nz = (U)(bits << 1) != 0;
      nsq_leaf[leaf] = acc;
      occ_leaf[leaf] = (uint8_t)nz;
      nrm_leaf[leaf] = __dsqrt_rn(acc);
      const bool canon = !nz && bits;  // only -0.0 entries: stored as +0.0 (quadtree.py:127-129)
      if (__any_sync(0xffffffffu, canon)) {
        if (fuse) {  // the tree's copy of the leaf must have landed first
          if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
          __syncwarp();
          asm volatile("fence.proxy.async;\n" ::: "memory");
        }
        canonicalise_leaves_warp<T>(padded, N, ROWS_LEAF, nb, canon, leaf);
      }
      acc = 0.0;
      bits = 0;
    }
  }
  if (fuse && lane == 0) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
  if (dbg && lane == 0) {
    unsigned long long *d = dbg + 3 * (blockIdx.x * ROWS_WARPS + warp);
    d[0] = (unsigned long long)t_wait;
    d[1] = (unsigned long long)(clock64() - t_begin);
    d[2] = (unsigned long long)Q;
  }
}

// ------------------------------------------------ K1, segmented chains
// The reference's leaf norm is one sequential chain acc = rn(acc + s_i),
// s_i = rn(x_i^2) >= 0, over the leaf in row-major order (quadtree.py:80-87):
// b^2 dependent adds (4096 x ~8 cycles at b = 64).  For the C tree (a few
// hundred to a few thousand leaves right after the products) that latency,
// not bandwidth, bounds the multiply's tail.  This kernel gives each leaf a
// warp, splits the chain into 64 row-major segments (two per lane) and still
// reproduces the chain's bits exactly:
//
//  * While acc stays inside one binade [2^E, 2^(E+1)) every double there is
//    a multiple of u = 2^(E-52), so rn(acc + s) = acc + rnd_u(s), rnd_u =
//    nearest multiple of u -- unless s sits exactly half-way (a tie: its
//    rounding depends on acc's last bit).  A segment that stays in one
//    binade therefore adds D * u, D = sum of rnd_u(s_i) as an exact integer,
//    wherever in that binade it starts.
//  * Each lane predicts its segments' binades from a float prefix sum of the
//    s_i (relative error ~1e-12, margin 2^-30) and forms D in integers,
//    flagging ties.
//  * The segments are applied in order.  A segment is applied as acc + D*u
//    only if acc >= 2^E and acc + D*u < 2^(E+1) -- the exact condition for
//    all its (monotone) partial sums to stay in the binade -- and it had no
//    tie; otherwise (binade crossings, ties, tiny or non-finite values,
//    segment 0) its lane runs the plain chain from the exact acc.  The
//    result is the sequential chain's, bit for bit.  (On c2's products ~9 of
//    64 segments take the plain chain: ~600 dependent adds instead of 4096.)
// The leaf is staged in shared memory with coalesced 16-byte cp.async copies
// (segments padded by 16 bytes; lane l starts its passes at element l, which
// spreads the per-lane segment reads over distinct banks).  Lanes publish
// (simple, E, D) per segment in a table; lane 0 then walks the 64 segments in
// order, merging consecutive simple segments of one binade into a run
// (integer D sums: no floating-point dependency), applying each run with one
// exact add and running the plain chain over the other segments.
constexpr int SEG_WARPS = 6;

// W warps stage and norm leaves; H more warps only join the pyramid tail (the
// last CTA builds C's pyramid with all W + H warps; beside K3 a CTA has
// shared memory for two staging warps, but registers for six)
template <typename T, int LEAF, int W = SEG_WARPS, int H = 0>
__global__ void __launch_bounds__(32 * (W + H)) leaf_norm_seg_kernel(
    T *__restrict__ padded, int64_t N, int64_t nb, double *__restrict__ nsq_leaf,
    uint8_t *__restrict__ occ_leaf, const uint32_t *__restrict__ list, const unsigned *list_count,
    PyrTail tail, unsigned smem_bytes) {
  using U = typename Bits<T>::U;
  constexpr int L = LEAF * LEAF / 64;  // segment length (elements), >= 16
  constexpr int EPV = 16 / (int)sizeof(T);
  constexpr int SS = seg_stride<T, LEAF>();
  extern __shared__ __align__(16) unsigned char seg_smem[];
  __shared__ SegInfo tbl[W][64];
  if (tail.pdl_wait) asm volatile("griddepcontrol.wait;\n" ::: "memory");
  if (tail.ready) {
    if (threadIdx.x == 0) spin_acquire_nonzero(tail.ready);
    __syncthreads();
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned char *wsm = seg_smem + (size_t)warp * seg_warp_bytes<T, LEAF>();
  const int64_t n_leaves = list ? (int64_t)*list_count : nb * nb;
  const int64_t gw = (int64_t)blockIdx.x * W + warp;
  const int64_t nw = (int64_t)gridDim.x * W;
  const bool check_flags = tail.grp_done && (!tail.overflow || !*(volatile const int *)tail.overflow);
  unsigned long long *const k1_tl = g_k1_tl;  // optional per-leaf timeline (SPAMM_K1_TIMELINE)
  auto next_slot = [&](int64_t cur) -> int64_t {
    if (!tail.leaf_ticket) return cur < 0 ? gw : cur + nw;
    unsigned v = 0;
    if (lane == 0) v = atomicAdd(tail.leaf_ticket, 1u);
    return (int64_t)__shfl_sync(0xffffffffu, v, 0);
  };
  for (int64_t lx = warp < W ? next_slot(-1) : n_leaves; lx < n_leaves; lx = next_slot(lx)) {
    const int64_t leaf = list ? (int64_t)list[lx] : lx;
    const int64_t bi = leaf / nb, bj = leaf - bi * nb;
    const bool tl_on = k1_tl && lane == 0 && lx < 8192;
    if (tl_on) k1_tl[4 * lx + 3] = k1_gt();
    if (check_flags) {  // the leaf-product kernel has stored every tile of this block
      const unsigned *flag = tail.grp_done + lx;
      for (;;) {
        unsigned v;
        asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
        if (v >= tail.grp_target) break;
        __nanosleep(128);
      }
    }
    T *base = padded + (bi * LEAF) * N + bj * LEAF;
    __syncwarp();  // (the previous leaf's readers are done with the stage)
#pragma unroll 8
    for (int c = lane; c < LEAF * LEAF / EPV; c += 32) {
      const int e = c * EPV;
      const int sg = e / L, off = e % L;
      cp_async16(wsm + sg * SS + off * (int)sizeof(T), base + (int64_t)(e / LEAF) * N + (e % LEAF));
    }
    if (tl_on) k1_tl[4 * lx] = k1_gt();
    cp_async_commit();
    cp_async_wait<0>();
    __syncwarp();
    if (tl_on) k1_tl[4 * lx + 1] = k1_gt();
    U bits = 0;
    const double acc = seg_leaf_norm<T, LEAF>(wsm, tbl[warp], lane, bits);
    if (tl_on) k1_tl[4 * lx + 2] = k1_gt();
    // occupancy / -0.0 (as the staged kernel): OR of every lane's raw bits
    unsigned long long all = (unsigned long long)bits;
#pragma unroll
    for (int o = 16; o; o >>= 1) all |= __shfl_xor_sync(0xffffffffu, all, o);
    const bool nz = (U)((U)all << 1) != 0;
    if (!nz && all) {  // all zero with some -0.0: canonicalise to +0.0
      for (int e = lane; e < LEAF * LEAF; e += 32) base[(int64_t)(e / LEAF) * N + (e % LEAF)] = T(0);
    }
    if (lane == 0) {
      nsq_leaf[leaf] = acc;
      occ_leaf[leaf] = (uint8_t)nz;
      tail.nrm[level_offset(tail.depth) + leaf] = __dsqrt_rn(acc);
      if (tail.grp_done) tail.grp_done[lx] = 0u;  // zero at rest for the next product
      if (tail.pcnt) {
        // the parent once its last non-empty child is final: ((c11 + c12) + c21) + c22
        // (quadtree.py:90-92); empty children read as the zeros the traversal wrote
        const int64_t pi = bi >> 1, pj = bj >> 1, c0 = 2 * pi * nb + 2 * pj, c1 = c0 + nb;
        auto bit = [&](int64_t g) { return (int)((__ldcg(tail.ne + (g >> 5)) >> (g & 31)) & 1u); };
        const unsigned expect = (unsigned)(bit(c0) + bit(c0 + 1) + bit(c1) + bit(c1 + 1));
        const int64_t p = pi * (nb >> 1) + pj;
        __threadfence();
        if (atomicAdd(tail.pcnt + p, 1u) + 1u == expect) {
          __threadfence();
          const double v = __dadd_rn(__dadd_rn(__dadd_rn(__ldcg(nsq_leaf + c0), __ldcg(nsq_leaf + c0 + 1)),
                                               __ldcg(nsq_leaf + c1)), __ldcg(nsq_leaf + c1 + 1));
          const uint8_t o = __ldcg(occ_leaf + c0) | __ldcg(occ_leaf + c0 + 1) | __ldcg(occ_leaf + c1) |
                            __ldcg(occ_leaf + c1 + 1);
          const int64_t lo = level_offset(tail.depth - 1);
          tail.nsq[lo + p] = v;
          tail.occ[lo + p] = o;
          tail.nrm[lo + p] = __dsqrt_rn(v);
          tail.pcnt[p] = 0u;
        }
      }
    }
  }
  if (tail.ticket) {  // the last CTA builds the pyramid
    __shared__ int s_last;
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      s_last = atomicAdd(tail.ticket, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (s_last) {
      // (timeline: [8191] = last CTA decided, trav_done seen, pyramid done)
      if (k1_tl && threadIdx.x == 0) k1_tl[4 * 8191] = k1_gt();
      if (tail.trav_done && threadIdx.x == 0) spin_acquire_nonzero(tail.trav_done);
      __threadfence();
      if (k1_tl && threadIdx.x == 0) k1_tl[4 * 8191 + 1] = k1_gt();
      if (tail.skip_pyramid) {
        // (deep tree: pyramid_upper_async follows)
      } else if (tail.pcnt) {  // the leaves' parents are built: the pyramid from their level
        PyrTail up = tail;
        up.depth = tail.depth - 1;
        pyramid_cta(up, seg_smem, smem_bytes, k1_tl ? k1_tl + 4 * 8190 : nullptr);
      } else {
        pyramid_cta(tail, seg_smem, smem_bytes, k1_tl ? k1_tl + 4 * 8190 : nullptr);
      }
      if (threadIdx.x == 0) {
        *tail.ticket = 0u;
        if (tail.leaf_ticket) *tail.leaf_ticket = 0u;
        if (tail.t_end && !tail.skip_pyramid) *tail.t_end = k1_gt();
        if (k1_tl) k1_tl[4 * 8191 + 2] = k1_gt();
      }
    }
  }
}

// ------------------------------------------------ K1, streaming exact norms
// (opt-in: SPAMM_STREAM_NORMS.)  A CTA of 256 threads per C block, built to
// form each norm with one FP64 multiply per element and integer work --
// measured slower than the segmented-chain kernel above on c2 (C tree 52-78
// vs 27-33 us: ~15 us per leaf, and it cannot share an SM with K3, whose 17
// warps of 96 registers leave too few registers in one SM sub-partition).
// The norm is the reference's sequential chain acc = rn(acc + s_i), s_i =
// rn(x_i^2), row-major (quadtree.py:80-87), reproduced exactly:
//   * every thread owns EPT consecutive elements; a CTA scan of their float
//     sums estimates the chain value P_i before each element (FP32 from the
//     squares' bits, relative error < 2^-17);
//   * element i is "clean" when P_i (1 - 2^-10) and (P_i + s_i)(1 + 2^-10)
//     share a binade [2^E, 2^(E+1)) (E >= -99): then the exact chain stays
//     in that binade across it, where every value is a multiple of u =
//     2^(E-52), so rn(A + s_i) = A + rnd_u(s_i) u -- an integer add, with
//     rnd_u(s_i) formed from s_i's bits (a half-way s_i is a tie: not clean);
//   * consecutive clean elements of one binade form a run (one integer D);
//     every other element is a single rounded add; zeros are skipped (rn(A +
//     0) = A); a thread with more than SN_R records uses the plain chain;
//   * every warp merges its lanes' runs of one binade (warp-segmented sums);
//     one warp applies the segments in order, each run as one exact add
//     after checking that the exact chain value is in the binade and the sum
//     stays below 2^(E+1) (otherwise the plain chain over its elements).
constexpr int SN_THREADS = 256;
constexpr int SN_R = 3;  // records per thread (more: the thread's elements by the plain chain)
constexpr int SN_RUN = 0, SN_SINGLE = 1, SN_PLAIN = 2;
struct SnRec {
  unsigned long long D;  // run: sum of rnd_u(s_i); single: the bits of s_i
  short E;
  short kind;
  short first, last;     // element range (row-major index in the leaf)
};
static_assert(sizeof(SnRec) == 16, "record layout");
template <int LEAF>
constexpr unsigned sn_smem_bytes() {  // the staged leaf, then the records
  return (unsigned)(LEAF * LEAF * sizeof(double) + 2 * SN_THREADS * SN_R * sizeof(SnRec));
}

// float estimate of a square s >= 0 from its bits (no FP64 instruction):
// exponent rebiased, mantissa truncated; below 2^-126 -> 0, beyond -> inf
__device__ __forceinline__ float sq_est(double sq) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(sq);
  const int fe = (int)((b >> 52) & 0x7ff) - 1023 + 127;
  if (fe <= 0) return 0.f;
  if (fe >= 255) return __uint_as_float(0x7f800000u);
  return __uint_as_float(((unsigned)fe << 23) | (unsigned)((b >> 29) & 0x7fffffu));
}

template <int LEAF>
__global__ void __launch_bounds__(SN_THREADS, 2) leaf_norm_stream_kernel(
    double *__restrict__ padded, int64_t N, int64_t nb, double *__restrict__ nsq_leaf,
    uint8_t *__restrict__ occ_leaf, const uint32_t *__restrict__ list, const unsigned *list_count,
    PyrTail tail, unsigned smem_bytes) {
  constexpr int NE = LEAF * LEAF, EPT = NE / SN_THREADS;
  static_assert(EPT % 2 == 0 && LEAF % EPT == 0, "a thread's elements lie in one row");
  static_assert(NE < 32768, "element indices are 16-bit");
  extern __shared__ __align__(16) unsigned char sn_smem[];
  double *stage = reinterpret_cast<double *>(sn_smem);
  SnRec *rec = reinterpret_cast<SnRec *>(sn_smem + NE * sizeof(double));  // per warp: its records
  SnRec *seg = rec + SN_THREADS * SN_R;                                      // ... and merged segments
  constexpr int NW = SN_THREADS / 32;
  __shared__ float s_wsum[NW];
  __shared__ int s_wcnt[NW];
  __shared__ unsigned long long s_bits[NW];
  __shared__ double s_acc;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tail.pdl_wait) asm volatile("griddepcontrol.wait;\n" ::: "memory");
  if (tail.ready) {
    if (tid == 0) spin_acquire_nonzero(tail.ready);
    __syncthreads();
  }
  const int64_t n_leaves = list ? (int64_t)*list_count : nb * nb;
  const bool check_flags = tail.grp_done && (!tail.overflow || !*(volatile const int *)tail.overflow);
  unsigned long long *const k1_tl = g_k1_tl;  // optional per-leaf timeline (SPAMM_K1_TIMELINE)
  for (int64_t lx = blockIdx.x; lx < n_leaves; lx += gridDim.x) {
    const int64_t leaf = list ? (int64_t)list[lx] : lx;
    const int64_t bi = leaf / nb, bj = leaf - bi * nb;
    const bool tl_on = k1_tl && tid == 0 && lx < 8192;
    if (tl_on) k1_tl[4 * lx + 3] = k1_gt();
    if (check_flags) {  // the leaf-product kernel has stored every tile of this block
      if (tid == 0) {
        const unsigned *flag = tail.grp_done + lx;
        for (;;) {
          unsigned v;
          asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
          if (v >= tail.grp_target) break;
          __nanosleep(64);
        }
      }
      __syncthreads();
    }
    if (tl_on) k1_tl[4 * lx] = k1_gt();
    double *base = padded + (bi * LEAF) * N + bj * LEAF;
    const int e0 = tid * EPT;
    const double *src = base + (int64_t)(e0 / LEAF) * N + (e0 % LEAF);
    // pass A: raw-bit OR (occupancy, -0.0) and the chunk's estimated sum.
    // Estimates are FP32 (the FP64 pipe is K3's): each square's float value
    // from its bits (truncated mantissa), prefix error < 2^-17 relative.
    unsigned long long bits = 0;
    float csum = 0.f;
    // this thread's elements, staged for pass B: pair q/2 of thread t at
    // double2 slot (q/2) * SN_THREADS + t (bank-conflict free)
    double2 *stage2 = reinterpret_cast<double2 *>(stage);
#pragma unroll
    for (int q = 0; q < EPT; q += 2) {
      const double2 v = __ldcg(reinterpret_cast<const double2 *>(src + q));
      stage2[(q / 2) * SN_THREADS + tid] = v;
      bits |= (unsigned long long)__double_as_longlong(v.x) | (unsigned long long)__double_as_longlong(v.y);
      csum += sq_est(__dmul_rn(v.x, v.x));
      csum += sq_est(__dmul_rn(v.y, v.y));
    }
    // CTA exclusive scan of the chunk sums (estimates of the chain)
    float incl = csum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const float y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    unsigned long long wb = bits;
#pragma unroll
    for (int o = 16; o; o >>= 1) wb |= __shfl_xor_sync(0xffffffffu, wb, o);
    if (lane == 31) s_wsum[warp] = incl;
    if (lane == 0) s_bits[warp] = wb;
    __syncthreads();
    float P = incl - csum;
    for (int w = 0; w < warp; ++w) P += s_wsum[w];
    // pass B: classify the elements into runs / single adds
    SnRec lr[SN_R];
    int nr = 0;
    int runE = 0, runFirst = -1, runLast = -1;
    unsigned long long runD = 0;
    auto flush = [&]() {
      if (runFirst < 0) return;
      if (nr < SN_R) lr[nr] = SnRec{runD, (short)runE, (short)SN_RUN, (short)runFirst, (short)runLast};
      ++nr;
      runFirst = -1;
    };
    // (not unrolled: the classification body is long and one warp per SM
    // sub-partition cannot afford instruction-cache misses)
#pragma unroll 1
    for (int q = 0; q < EPT; q += 2) {
      const double2 v = stage2[(q / 2) * SN_THREADS + tid];
#pragma unroll 1
      for (int h = 0; h < 2; ++h) {
        const double x = h ? v.y : v.x;
        const double sq = __dmul_rn(x, x);
        const int e = e0 + q + h;
        if (sq == 0.0) continue;  // rn(A + 0) = A: no effect on the chain
        const unsigned long long sb = (unsigned long long)__double_as_longlong(sq);
        const float Pn = P + sq_est(sq);
        // the estimated chain before and after the element, widened by 2^-10
        const unsigned lob = __float_as_uint(P * (1.f - 0x1p-10f));
        const unsigned hib = __float_as_uint(Pn * (1.f + 0x1p-10f));
        const int elo = (int)((lob >> 23) & 0xff), ehi = (int)((hib >> 23) & 0xff);
        int es = (int)((sb >> 52) & 0x7ff);
        bool clean = elo == ehi && elo >= 28 && elo <= 253 && es < 0x7ff;
        unsigned long long r = 0;
        const int E = elo - 127;  // binade [2^E, 2^(E+1)) of the exact chain across this element
        if (clean) {  // rnd_u(sq), u = 2^(E-52), from the bits of sq
          unsigned long long M = sb & ((1ull << 52) - 1);
          if (es) M |= 1ull << 52;
          else es = 1;
          const int sh = E + 1023 - es;  // sq / u = M * 2^-sh
          if (sh <= 0) {
            clean = false;
          } else if (sh < 64) {
            const unsigned long long rem = M & ((1ull << sh) - 1), half = 1ull << (sh - 1);
            r = (M >> sh) + (rem > half ? 1ull : 0ull);
            clean = rem != half;  // a tie rounds by the chain value's last bit
          }
        }
        if (clean) {
          if (runFirst >= 0 && E == runE) {
            runD += r;
            runLast = e;
          } else {
            flush();
            runE = E;
            runD = r;
            runFirst = runLast = e;
          }
        } else {
          flush();
          if (nr < SN_R) lr[nr] = SnRec{sb, 0, (short)SN_SINGLE, (short)e, (short)e};
          ++nr;
        }
        P = Pn;
      }
    }
    flush();
    if (nr > SN_R) {  // too many records: this thread's elements by the plain chain
      nr = 1;
      lr[0] = SnRec{0, 0, (short)SN_PLAIN, (short)e0, (short)(e0 + EPT - 1)};
    }
    // Level 1 (every warp): its lanes' records in element order, consecutive
    // runs of one binade merged (warp-segmented sums) into segments
    {
      int ci = nr;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, ci, o);
        if (lane >= o) ci += y;
      }
      const int off = ci - nr, M = __shfl_sync(0xffffffffu, ci, 31);
      SnRec *wr = rec + warp * 32 * SN_R;  // this warp's records
      SnRec *ws = seg + warp * 32 * SN_R;  // ... and segments
#pragma unroll
      for (int k = 0; k < SN_R; ++k)
        if (k < nr) wr[off + k] = lr[k];
      __syncwarp();
      int nseg = 0;  // (warp-uniform)
      for (int c0 = 0; c0 < M; c0 += 32) {
        const int i = c0 + lane;
        const bool valid = i < M;
        const SnRec r = valid ? wr[i] : SnRec{0, 0, -1, 0, 0};
        const int rkind = r.kind, rE = r.E;
        const int pk = __shfl_up_sync(0xffffffffu, rkind, 1), pe = __shfl_up_sync(0xffffffffu, rE, 1);
        const bool cont = lane > 0 && valid && rkind == SN_RUN && pk == SN_RUN && pe == rE;
        const unsigned heads = __ballot_sync(0xffffffffu, valid && !cont);
        const unsigned vm = __ballot_sync(0xffffffffu, valid);
        const unsigned ends = vm & ((heads >> 1) | ~(vm >> 1) | 0x80000000u);
        unsigned long long ps = rkind == SN_RUN ? r.D : 0ull;  // inclusive prefix of run D
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const unsigned long long y = __shfl_up_sync(0xffffffffu, ps, o);
          if (lane >= o) ps += y;
        }
        const int hl = 31 - __clz((int)(heads & (0xffffffffu >> (31 - lane))));
        const unsigned long long pre = __shfl_sync(0xffffffffu, ps, hl > 0 ? hl - 1 : 0);
        const int first = __shfl_sync(0xffffffffu, (int)r.first, hl < 0 ? 0 : hl);
        // segment end lanes write their segment; a run continuing the
        // previous chunk's last segment is merged into it
        const bool is_end = (ends >> lane) & 1u;
        const bool merge0 = lane == hl && hl == 0 && c0 > 0 && rkind == SN_RUN && nseg > 0 &&
                            ws[nseg - 1].kind == SN_RUN && ws[nseg - 1].E == rE;
        const bool merge_first = __shfl_sync(0xffffffffu, merge0 ? 1 : 0, 0) != 0;
        const int before = __popc(ends & ((1u << lane) - 1));  // segments ending before this lane
        if (is_end) {
          SnRec sg;
          sg.kind = (short)rkind;
          sg.E = (short)rE;
          sg.first = (short)first;
          sg.last = r.last;
          sg.D = rkind == SN_RUN ? ps - (hl > 0 ? pre : 0ull) : r.D;
          if (hl == 0 && merge_first) {  // (the first segment of this chunk)
            ws[nseg - 1].D += sg.D;
            ws[nseg - 1].last = sg.last;
          } else {
            ws[nseg + before - (merge_first ? 1 : 0)] = sg;
          }
        }
        nseg += __popc(ends) - (merge_first ? 1 : 0);
        __syncwarp();
      }
      if (lane == 0) s_wcnt[warp] = nseg;
    }
    __syncthreads();
    if (tl_on) k1_tl[4 * lx + 1] = k1_gt();
    // Level 2 (one warp): the segments in order, each one exact add, one
    // rounded add or (rare) a plain chain
    if (warp == 0) {
      double acc = 0.0;
      int pE = 0, pFirst = -1, pLast = -1;
      unsigned long long pD = 0;
      auto replay = [&](int f, int l) {  // the plain chain over elements [f, l]
        for (int e0r = f; e0r <= l; e0r += 32) {  // squares in parallel, then the chain
          const int e = e0r + lane;
          const int et = e / EPT, eq = e - et * EPT;  // (element e of the staged layout)
          const double x = e <= l ? stage[2 * ((eq >> 1) * SN_THREADS + et) + (eq & 1)] : 0.0;
          const double sq = __dmul_rn(x, x);
          const int n = l - e0r + 1 < 32 ? l - e0r + 1 : 32;
          for (int k = 0; k < n; ++k) acc = __dadd_rn(acc, __shfl_sync(0xffffffffu, sq, k));
        }
      };
      auto flushp = [&]() {
        if (pFirst < 0) return;
        bool ok = false;
        const unsigned long long ab = (unsigned long long)__double_as_longlong(acc);
        if (pD < (1ull << 53) && (int)((ab >> 52) & 0x7ff) == pE + 1023) {
          const double v = acc + (double)pD * pow2_exact(pE - 52);  // exact below 2^(E+1)
          if (v < pow2_exact(pE + 1)) {
            acc = v;
            ok = true;
          }
        }
        if (!ok) replay(pFirst, pLast);
        pFirst = -1;
      };
      for (int w = 0; w < NW; ++w) {
        const SnRec *ws = seg + w * 32 * SN_R;
        const int n = s_wcnt[w];
        for (int k = 0; k < n; ++k) {
          const SnRec sg = ws[k];
          if (sg.kind == SN_RUN) {
            if (pFirst >= 0 && pE == sg.E) {
              pD += sg.D;
              pLast = sg.last;
            } else {
              flushp();
              pE = sg.E;
              pD = sg.D;
              pFirst = sg.first;
              pLast = sg.last;
            }
          } else if (sg.kind == SN_SINGLE) {
            flushp();
            acc = __dadd_rn(acc, __longlong_as_double((long long)sg.D));
          } else {
            flushp();
            replay(sg.first, sg.last);
          }
        }
      }
      flushp();
      if (lane == 0) s_acc = acc;
    }
    __syncthreads();
    if (tl_on) k1_tl[4 * lx + 2] = k1_gt();
    unsigned long long all = 0;
#pragma unroll
    for (int w = 0; w < NW; ++w) all |= s_bits[w];
    const bool nz = (all << 1) != 0;
    if (!nz && all) {  // all zero with some -0.0: canonicalise to +0.0
#pragma unroll
      for (int q = 0; q < EPT; ++q) const_cast<double *>(src)[q] = 0.0;
    }
    if (tid == 0) {
      const double acc = s_acc;
      nsq_leaf[leaf] = acc;
      occ_leaf[leaf] = (uint8_t)nz;
      tail.nrm[level_offset(tail.depth) + leaf] = __dsqrt_rn(acc);
      if (tail.grp_done) tail.grp_done[lx] = 0u;  // zero at rest for the next product
    }
    __syncthreads();  // (the record area and s_* are reused by the next leaf)
  }
  if (tail.ticket) {  // the last CTA builds the pyramid
    __shared__ int s_last;
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      s_last = atomicAdd(tail.ticket, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (s_last) {
      if (tail.trav_done && threadIdx.x == 0) spin_acquire_nonzero(tail.trav_done);
      __threadfence();
      pyramid_cta(tail, sn_smem, smem_bytes);
      if (threadIdx.x == 0) {
        *tail.ticket = 0u;
        if (tail.t_end) *tail.t_end = k1_gt();
      }
    }
  }
}

// Direct kernel for tiny leaves (b * b * sizeof(T) < 128): one thread per
// leaf reads its b x b elements in row-major order straight from global.
template <typename T>
__global__ void leaf_norm_direct_kernel(T *__restrict__ padded, int64_t N, int32_t b, int64_t nb,
                                        double *__restrict__ nsq_leaf,
                                        uint8_t *__restrict__ occ_leaf,
                                        const uint32_t *__restrict__ list,
                                        const unsigned *list_count) {
  const int64_t lx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (lx >= (list ? (int64_t)*list_count : nb * nb)) return;
  const int64_t leaf = list ? (int64_t)list[lx] : lx;
  const int64_t bi = leaf / nb, bj = leaf - bi * nb;
  double acc = 0.0;
  typename Bits<T>::U bits = 0;
  for (int r = 0; r < b; ++r) {
    const T *row = padded + (bi * b + r) * N + bj * b;
    for (int c = 0; c < b; ++c) accum<T>(acc, bits, row[c]);
  }
  const bool nz = (typename Bits<T>::U)(bits << 1) != 0;
  nsq_leaf[leaf] = acc;
  occ_leaf[leaf] = (uint8_t)nz;
  if (!nz && bits) canonicalise_leaf<T>(padded, N, b, bi, bj);
}

// Pyramid (one launch for every level): the levels are cut into passes of
// L <= 5 levels; a pass-p CTA reduces one 2^L x 2^L tile of its input level
// through L levels, parent = ((c11 + c12) + c21) + c22 (quadtree.py:90-92),
// occupancy OR (quadtree.py:137-138), and writes nrm = rn(sqrt(nsq)) of every
// node it produces (the factors of the reference's norm product,
// multiply.py:185, rounded exactly like np.sqrt).  The last of the 4^L'
// children of a pass-(p+1) tile to finish goes on to reduce that tile
// (ticket counters that reset themselves), so the whole pyramid is one
// launch whatever the depth.  Pass-0 CTAs also take the sqrt of the leaf
// level.
constexpr int PYR_THREADS = 256;
constexpr int PYR_MAX_PASSES = 6;

struct PyrPlan {
  int passes;
  int from[PYR_MAX_PASSES], L[PYR_MAX_PASSES];
  int64_t cnt_off[PYR_MAX_PASSES];  // ticket counters of pass p's tiles (p >= 1)
  int64_t n_counters;
};

static PyrPlan pyramid_plan(int depth) {
  PyrPlan pl{};
  int from = depth;
  int64_t off = 0;
  while (from > 0) {
    const int L = from < 5 ? from : 5;
    pl.from[pl.passes] = from;
    pl.L[pl.passes] = L;
    pl.cnt_off[pl.passes] = off;
    if (pl.passes > 0) off += int64_t(1) << (2 * (from - L));
    ++pl.passes;
    from -= L;
  }
  pl.n_counters = off;
  return pl;
}

__global__ void __launch_bounds__(PYR_THREADS) pyramid_fused_kernel(double *__restrict__ nsq,
                                                                    uint8_t *__restrict__ occ,
                                                                    double *__restrict__ nrm,
                                                                    PyrPlan pl,
                                                                    unsigned *__restrict__ tickets) {
  __shared__ double s_n[1024];
  __shared__ uint8_t s_o[1024];
  __shared__ int s_last;
  if (pl.passes == 0) {  // depth 0: the single leaf is the root
    if (threadIdx.x == 0) nrm[0] = __dsqrt_rn(nsq[0]);
    return;
  }
  int64_t tile = blockIdx.x;
  for (int p = 0; p < pl.passes; ++p) {
    const int from = pl.from[p], L = pl.L[p];
    const int tiles_per_side = 1 << (from - L);
    const int ti = (int)(tile / tiles_per_side), tj = (int)(tile % tiles_per_side);
    int side = 1 << L;
    const int64_t fine_side = int64_t(1) << from;
    const double *lvl = nsq + level_offset(from);
    const uint8_t *olvl = occ + level_offset(from);
    double *nlvl = nrm + level_offset(from);
    for (int e = threadIdx.x; e < side * side; e += PYR_THREADS) {
      const int r = e / side, c = e % side;
      const int64_t g = (int64_t(ti) * side + r) * fine_side + int64_t(tj) * side + c;
      // L1-bypassing loads: later passes read what other CTAs wrote
      const double x = __ldcg(lvl + g);
      s_n[e] = x;
      s_o[e] = __ldcg(olvl + g);
      if (p == 0) nlvl[g] = __dsqrt_rn(x);
    }
    __syncthreads();
    for (int k = from - 1; k >= from - L; --k) {
      const int ps = side >> 1;
      const int64_t coarse_side = int64_t(1) << k;
      double *clvl = nsq + level_offset(k);
      uint8_t *oclvl = occ + level_offset(k);
      double *nclvl = nrm + level_offset(k);
      double v[4];
      uint8_t o[4];
      int cnt = 0;
      for (int e = threadIdx.x; e < ps * ps; e += PYR_THREADS, ++cnt) {
        const int r = e / ps, c = e % ps;
        const int f0 = (2 * r) * side + 2 * c, f1 = f0 + side;
        v[cnt] = __dadd_rn(__dadd_rn(__dadd_rn(s_n[f0], s_n[f0 + 1]), s_n[f1]), s_n[f1 + 1]);
        o[cnt] = s_o[f0] | s_o[f0 + 1] | s_o[f1] | s_o[f1 + 1];
        const int64_t g = (int64_t(ti) * ps + r) * coarse_side + int64_t(tj) * ps + c;
        clvl[g] = v[cnt];
        oclvl[g] = o[cnt];
        nclvl[g] = __dsqrt_rn(v[cnt]);
      }
      __syncthreads();
      cnt = 0;
      for (int e = threadIdx.x; e < ps * ps; e += PYR_THREADS, ++cnt) {
        s_n[e] = v[cnt];
        s_o[e] = o[cnt];
      }
      __syncthreads();
      side = ps;
    }
    if (p + 1 == pl.passes) break;
    // hand the parent tile to the last of its children
    const int Ln = pl.L[p + 1];
    const int parent_side = 1 << (pl.from[p + 1] - Ln);
    const int64_t parent = int64_t(ti >> Ln) * parent_side + (tj >> Ln);
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned *tk = tickets + pl.cnt_off[p + 1] + parent;
      const unsigned children = 1u << (2 * Ln);
      const unsigned old = atomicAdd(tk, 1u);
      s_last = old == children - 1;
      if (s_last) *tk = 0;  // ready for the next build
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    tile = parent;
  }
}

// Launch of the staged K1.  `ov` (list mode, after the warp-specialised leaf
// kernel) makes it a programmatic dependent launch that overlaps that kernel
// and waits per C block; its ring is then only 4 stages deep so one K1 CTA
// fits beside the leaf kernel on every SM.
// 4-D view of an N-row f64/f32 matrix for the rows kernel: {128 bytes of a
// leaf row, leaf index along the matrix row, 128-byte piece of the leaf row,
// matrix row}; box {128 B, 32 leaves, all pieces, 1 row}, 128-byte swizzle.
// (The strides are not monotonic; a driver that rejects the encoding leaves
// the staged kernel in charge.)
static PFN_cuTensorMapEncodeTiled_v12000 rows_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void *p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
  }
  return fn;
}
template <typename T>
static bool rows_map(CUtensorMap *map, const void *base, int64_t nb, int64_t rows, int64_t ld) {
  auto enc = rows_map_encoder();
  if (!enc || ((uintptr_t)base & 15) || (ld * sizeof(T)) % 16) return false;
  constexpr cuuint32_t E = 128 / sizeof(T), PIECES = ROWS_LEAF * sizeof(T) / 128;
  cuuint64_t dims[4] = {E, (cuuint64_t)nb, PIECES, (cuuint64_t)rows};
  cuuint64_t strides[3] = {ROWS_LEAF * sizeof(T), 128, (cuuint64_t)(ld * sizeof(T))};
  cuuint32_t box[4] = {E, 32, PIECES, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  return enc(map, sizeof(T) == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4,
             const_cast<void *>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

struct K1Overlap {
  unsigned *grp_done;
  unsigned grp_target;
  const int *overflow;
  unsigned long long *t_end;
  bool pdl;  // programmatic dependent launch behind the leaf-product kernel
  const unsigned *ready, *trav_done;  // bitmask groups (see PyrTail)
  const void *fuse_src;               // fused build (see PyrTail)
  int64_t fuse_ld;
  const uint32_t *ne;                 // non-empty leaf blocks (see PyrTail)
};

template <typename T, int S, int LT>
static int launch_staged(spamm_tree *t, cudaStream_t st, const uint32_t *list,
                         const unsigned *list_count, int64_t n_leaves, unsigned *ticket,
                         const K1Overlap *ov, bool *fused) {
  const size_t smem = (size_t)S * LT * K1_LEAF_STRIDE;
  auto kern = leaf_norm_staged_kernel<T, S, LT>;
  SPAMM_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  SPAMM_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
  PyrTail tail{};
  tail.nsq = t->nsq;
  tail.occ = t->occ;
  tail.nrm = t->nrm;
  tail.depth = t->depth;
  if (ticket && t->depth <= PYR_TAIL_MAX_DEPTH) {
    tail.ticket = ticket;
    *fused = true;
  }
  if (ov) {
    tail.grp_done = ov->grp_done;
    tail.grp_target = ov->grp_target;
    tail.overflow = ov->overflow;
    tail.t_end = ov->t_end;
    tail.pdl_wait = ov->pdl && !ov->grp_done;
    tail.ready = ov->ready;
    tail.trav_done = ov->trav_done;
    tail.fuse_src = ov->fuse_src;
    tail.fuse_ld = ov->fuse_ld;
  }
  double *nsq_leaf = t->nsq + level_offset(t->depth);
  uint8_t *occ_leaf = t->occ + level_offset(t->depth);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)((n_leaves + LT - 1) / LT));
  cfg.blockDim = dim3(K1_THREADS);
  cfg.dynamicSmemBytes = smem;
  if (ov && ov->grp_done) {
    // one CTA per SM (the padding makes a second one not fit): the CTAs start
    // on SMs as the leaf kernel's CTAs retire and must not pile onto the
    // first ones (measured: 35-37 us vs 44-45 us with 60 KB, two per SM)
    static const size_t pad = (size_t)120 << 10;
    cfg.dynamicSmemBytes = std::max(smem, pad);
    SPAMM_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)cfg.dynamicSmemBytes));
  }
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  if (ov && (ov->grp_done || ov->pdl)) {
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
  }
  SPAMM_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, (T *)t->padded, t->N, (int32_t)t->leaf, t->nb,
                                    nsq_leaf, occ_leaf, list, list_count, tail));
  return SPAMM_OK;
}

// ring depth of the 32-leaf K1 for large trees (SPAMM_K1_STAGES; 3 by default: four CTAs
// per SM instead of two -- c5 K1 8.73 -> 8.08 ms, 3.94 -> 4.25 TB/s)
static int k1_big_stages() {
  static const int v = getenv("SPAMM_K1_STAGES") ? atoi(getenv("SPAMM_K1_STAGES")) : 3;
  return v;
}

template <typename T>
static int launch_leaf_norms(spamm_tree *t, cudaStream_t st, const uint32_t *list,
                             const unsigned *list_count, int64_t list_cap, unsigned *ticket,
                             const K1Overlap *ov, bool *fused) {
  *fused = false;
  const int64_t n_leaves = list ? std::min<int64_t>(list_cap, t->nb * t->nb) : t->nb * t->nb;
  double *nsq_leaf = t->nsq + level_offset(t->depth);
  uint8_t *occ_leaf = t->occ + level_offset(t->depth);
  if (t->leaf * sizeof(T) >= 16) {
    // The copy rate one SM sustains with cp.async is limited (outstanding
    // requests), so small trees spread their leaves thinly -- 8 per CTA over
    // as many SMs as possible with a deep ring -- and large trees use 32
    // leaves per CTA, two CTAs per SM.
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, t->device);
    // dense builds of large leaf-64 trees: the TMA-fed persistent rows kernel
    // (SPAMM_K1_ROWS=0: the staged kernel; =2/3/4: ring depth -- by default 3
    // stages of 16 KB for f64 and 4 of 8 KB for f32)
    static const int rows_env = getenv("SPAMM_K1_ROWS") ? atoi(getenv("SPAMM_K1_ROWS")) : -1;
    const int rows_r = rows_env >= 0 ? rows_env : (sizeof(T) == 4 ? 4 : 3);
    const bool rows_ok = rows_r > 0 && !list && t->leaf == ROWS_LEAF && t->nb % 32 == 0 &&
                         n_leaves >= (int64_t)64 * sms && !(ov && (ov->grp_done || ov->t_end)) &&
                         (!(ov && ov->fuse_src) || (ov->fuse_ld * sizeof(T)) % 16 == 0);
    CUtensorMap tm_src, tm_dst;
    const T *rows_src = ov && ov->fuse_src ? (const T *)ov->fuse_src : (const T *)t->padded;
    const int64_t rows_sld = ov && ov->fuse_src ? ov->fuse_ld : t->N;
    if (rows_ok && rows_map<T>(&tm_src, rows_src, t->nb, t->N, rows_sld) &&
        rows_map<T>(&tm_dst, t->padded, t->nb, t->N, t->N)) {
      int gpr_shift = 0;
      while (((int64_t)32 << gpr_shift) < t->nb) ++gpr_shift;
      const int64_t groups = t->nb << gpr_shift;
      const unsigned grid = (unsigned)std::min<int64_t>(sms, (groups + ROWS_WARPS - 1) / ROWS_WARPS);
      auto go = [&](auto kern, int R) -> int {
        const size_t smem = (size_t)ROWS_WARPS * R * 32 * ROWS_LEAF * sizeof(T) + 1024;
        SPAMM_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        kern<<<grid, 32 * ROWS_WARPS, smem, st>>>(tm_src, tm_dst, rows_src != (const T *)t->padded ? 1 : 0,
                                                  (T *)t->padded, t->N, t->nb, gpr_shift, nsq_leaf, occ_leaf,
                                                  t->nrm + level_offset(t->depth));
        return SPAMM_OK;
      };
      static const bool rows_debug = getenv("SPAMM_K1_ROWS_DEBUG") != nullptr;
      static unsigned long long *dbg_dev = nullptr;
      if (rows_debug && !dbg_dev) {
        cudaMalloc(&dbg_dev, sizeof(unsigned long long) * 3 * ROWS_WARPS * 1024);
        cudaMemcpyToSymbol(g_rows_dbg, &dbg_dev, sizeof(void *));
      }
      if (rows_r == 2) SPAMM_TRY(go(leaf_norm_rows_kernel<T, 2>, 2));
      else if (rows_r == 4 && sizeof(T) == 4) SPAMM_TRY(go(leaf_norm_rows_kernel<T, 4>, 4));
      else SPAMM_TRY(go(leaf_norm_rows_kernel<T, 3>, 3));
      if (rows_debug) {
        cudaStreamSynchronize(st);
        std::vector<unsigned long long> h(3 * ROWS_WARPS * grid);
        cudaMemcpy(h.data(), dbg_dev, h.size() * 8, cudaMemcpyDeviceToHost);
        double wt = 0, tot = 0, ch = 0;
        for (size_t i = 0; i < h.size(); i += 3) { wt += h[i]; tot += h[i + 1]; ch += h[i + 2]; }
        fprintf(stderr, "[k1 rows] warps=%zu chunks/warp %.0f: cycles per chunk %.0f, of which waiting for data %.0f\n",
                h.size() / 3, ch / (h.size() / 3), tot / ch, wt / ch);
      }
    } else if (ov && ov->grp_done)
      SPAMM_TRY((launch_staged<T, 12, 8>(t, st, list, list_count, n_leaves, ticket, ov, fused)));
    else if (n_leaves >= (int64_t)64 * sms && k1_big_stages() == 4)
      SPAMM_TRY((launch_staged<T, 4, 32>(t, st, list, list_count, n_leaves, ticket, ov, fused)));
    else if (n_leaves >= (int64_t)64 * sms && k1_big_stages() == 3)
      SPAMM_TRY((launch_staged<T, 3, 32>(t, st, list, list_count, n_leaves, ticket, ov, fused)));
    else if (n_leaves >= (int64_t)64 * sms)
      SPAMM_TRY((launch_staged<T, 6, 32>(t, st, list, list_count, n_leaves, ticket, ov, fused)));
    else
      SPAMM_TRY((launch_staged<T, 12, 8>(t, st, list, list_count, n_leaves, ticket, ov, fused)));
  } else {
    const int64_t grid = (n_leaves + 127) / 128;
    leaf_norm_direct_kernel<T><<<(unsigned)grid, 128, 0, st>>>(
        (T *)t->padded, t->N, t->leaf, t->nb, nsq_leaf, occ_leaf, list, list_count);
  }
  SPAMM_CUDA_TRY(cudaGetLastError());
  return SPAMM_OK;
}

static unsigned long long *h_k1_tl_dev = nullptr;
void k1_timeline_enable(cudaStream_t st) {
  if (!h_k1_tl_dev) {
    cudaMalloc(&h_k1_tl_dev, sizeof(unsigned long long) * 4 * 8192);
    cudaMemcpyToSymbol(g_k1_tl, &h_k1_tl_dev, sizeof(void *));
  }
  cudaMemsetAsync(h_k1_tl_dev, 0, sizeof(unsigned long long) * 4 * 8192, st);
}
void k1_timeline_dump(unsigned long long k3_end, unsigned long long k3_start) {
  std::vector<unsigned long long> tl(4 * 8192);
  cudaMemcpy(tl.data(), h_k1_tl_dev, tl.size() * 8, cudaMemcpyDeviceToHost);
  {  // segmented-chain kernel: per leaf [flag seen, staged, norm done, warp reached it]
    std::vector<std::pair<unsigned long long, int>> done;
    for (int q = 0; q < 8192; ++q)
      if (tl[4 * q + 2] && tl[4 * q + 3]) done.push_back({tl[4 * q + 2], q});
    if (!done.empty()) {
      std::sort(done.begin(), done.end());
      double norm_sum = 0;
      for (auto &d : done) norm_sum += (double)(tl[4 * d.second + 2] - tl[4 * d.second + 1]);
      int before_end = 0;
      double first_reach = 1e30;
      for (auto &d : done) {
        before_end += d.first < k3_end;
        first_reach = std::min(first_reach, ((double)tl[4 * d.second + 3] - (double)k3_end) * 1e-3);
      }
      fprintf(stderr, "[k1 seg] leaves=%zu done during K3 %d, first reach %.1f us, mean norm %.2f us; last leaves (us after K3 end): ",
              done.size(), before_end, first_reach, norm_sum / done.size() * 1e-3);
      for (size_t k = done.size() > 4 ? done.size() - 4 : 0; k < done.size(); ++k) {
        const int q = done[k].second;
        auto rel = [&](int f) { return ((double)tl[4 * q + f] - (double)k3_end) * 1e-3; };
        fprintf(stderr, " [reach %.1f flag %.1f staged %.1f done %.1f]", rel(3), rel(0), rel(1), rel(2));
      }
      if (tl[4 * 8190])
        fprintf(stderr, " | pyr start %.1f global level %.1f smem levels %.1f", ((double)tl[4 * 8190] - (double)k3_end) * 1e-3,
                ((double)tl[4 * 8190 + 1] - (double)k3_end) * 1e-3, ((double)tl[4 * 8190 + 2] - (double)k3_end) * 1e-3);
      if (tl[4 * 8191])
        fprintf(stderr, " | last CTA %.1f trav %.1f pyramid done %.1f",
                ((double)tl[4 * 8191] - (double)k3_end) * 1e-3, ((double)tl[4 * 8191 + 1] - (double)k3_end) * 1e-3,
                ((double)tl[4 * 8191 + 2] - (double)k3_end) * 1e-3);
      fprintf(stderr, "\n");
    }
  }
  unsigned long long t0 = ~0ull;
  int n = 0;
  for (int q = 0; q < 8192; ++q)
    if (tl[4 * q]) { t0 = std::min(t0, tl[4 * q]); ++n; }
  fprintf(stderr, "[k1 timeline] ctas=%d k3 start %.1f end %.1f", n, ((double)k3_start - (double)t0) * 1e-3,
          ((double)k3_end - (double)t0) * 1e-3);
  for (int f = 0; f < 4; ++f) {
    std::vector<double> v;
    for (int q = 0; q < 8192; ++q)
      if (tl[4 * q] && tl[4 * q + f]) v.push_back((tl[4 * q + f] - t0) * 1e-3);
    std::sort(v.begin(), v.end());
    if (!v.empty()) fprintf(stderr, " | s%d %.1f/%.1f/%.1f", f, v[0], v[v.size() / 2], v.back());
  }
  fprintf(stderr, "\n");
}

// (build_pyramid_async is declared in common.cuh)

// Rebuild the whole pyramid of `t` from its padded storage (canonicalising
// all-zero leaves in place).  Stream-ordered; no host sync; two launches.
int build_pyramid_async(DeviceContext *ctx, spamm_tree *t, cudaStream_t st, int *launches,
                        const uint32_t *list, const unsigned *list_count, int64_t list_cap,
                        unsigned *grp_done, unsigned grp_target, const int *overflow,
                        unsigned long long *t_end, const unsigned *ready,
                        const unsigned *trav_done, const void *fuse_src, int64_t fuse_ld,
                        const uint32_t *ne) {
  // builds on copy_in run concurrently with the main stream's: own tickets
  Scratch &k1t = st == ctx->copy_in ? ctx->k1_ticket_in : ctx->k1_ticket;
  SPAMM_TRY(ensure_scratch(k1t, 2 * sizeof(unsigned), st, /*zeroed=*/true));  // + leaf ticket
  unsigned *ticket = (unsigned *)k1t.ptr;
  bool fused = false;
  // list mode follows the leaf-product kernel: launch it programmatically so
  // its CTAs are resident (and waiting) as that kernel's CTAs retire
  K1Overlap ovs{grp_done, grp_target, overflow, t_end, list != nullptr && t_end != nullptr, ready,
                trav_done, fuse_src, fuse_ld, ne};
  const K1Overlap *ov = (grp_done || t_end || fuse_src) ? &ovs : nullptr;
  // list mode (C's tree): the segmented-chain kernel, a warp per leaf
  static const bool no_seg = getenv("SPAMM_NO_SEG_CHAIN") != nullptr;
  // (only where K1 overlaps K3's tail -- small block grids: per leaf the
  // segmented kernel is latency-short, but for 10^4-10^6 C blocks the staged
  // kernel's 32-leaf CTAs stream them faster: c3 C tree 0.13 vs 0.35 ms, c5
  // 0.30 vs 0.81 ms)
  // (SPAMM_STREAM_NORMS: the CTA-per-leaf streaming kernel instead -- exact
  // too, measured slower: DESIGN.md, K1)
  static const bool stream_norms = getenv("SPAMM_STREAM_NORMS") != nullptr;
  if (list && !no_seg && stream_norms && grp_done && t->dtype == SPAMM_DTYPE_F64 &&
      (t->leaf == 32 || t->leaf == 64)) {
    // the streaming exact-norm kernel: one small CTA per SM beside K3 (it is
    // launched programmatically behind K3 and becomes resident at once)
    PyrTail tail{};
    tail.nsq = t->nsq;
    tail.occ = t->occ;
    tail.nrm = t->nrm;
    tail.depth = t->depth;
    tail.ticket = t->depth <= PYR_TAIL_MAX_DEPTH ? ticket : nullptr;
    tail.grp_done = ov->grp_done;
    tail.grp_target = ov->grp_target;
    tail.overflow = ov->overflow;
    tail.t_end = ov->t_end;
    tail.pdl_wait = 0;
    tail.ready = ov->ready;
    tail.trav_done = ov->trav_done;
    cudaLaunchConfig_t cfg{};
    // CTAs (a leaf each at a time) fill the SMs as K3's CTAs retire: up to
    // two per SM (256 threads, 57 KB of shared memory each at leaf 64)
    static const int per_sm = getenv("SPAMM_SN_CTAS_PER_SM") ? atoi(getenv("SPAMM_SN_CTAS_PER_SM")) : 2;
    const unsigned smem = t->leaf == 64 ? sn_smem_bytes<64>() : sn_smem_bytes<32>();
    cfg.gridDim = dim3((unsigned)std::max<int64_t>(
        1, std::min<int64_t>(std::min<int64_t>(list_cap, t->nb * t->nb), (int64_t)ctx->num_sms * per_sm)));
    cfg.blockDim = dim3(SN_THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    auto go = [&](auto kern) -> int {
      SPAMM_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      // (the library's kernels all ask for the maximum shared-memory carveout)
      SPAMM_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
      SPAMM_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, (double *)t->padded, t->N, t->nb,
                                        t->nsq + level_offset(t->depth), t->occ + level_offset(t->depth),
                                        list, list_count, tail, smem));
      return SPAMM_OK;
    };
    if (t->leaf == 64) SPAMM_TRY(go(leaf_norm_stream_kernel<64>));
    else SPAMM_TRY(go(leaf_norm_stream_kernel<32>));
    fused = tail.ticket != nullptr;
  } else if (list && !no_seg && grp_done && (t->leaf == 32 || t->leaf == 64)) {
    const bool f64 = t->dtype == SPAMM_DTYPE_F64;
    PyrTail tail{};
    tail.nsq = t->nsq;
    tail.occ = t->occ;
    tail.nrm = t->nrm;
    tail.depth = t->depth;
    // (deeper trees: the ticket still elects the CTA that resets the leaf
    // ticket; the levels above the leaves are pyramid_upper_async's)
    tail.ticket = ticket;
    tail.skip_pyramid = t->depth > PYR_TAIL_MAX_DEPTH;
    if (ov) {
      tail.grp_done = ov->grp_done;
      tail.grp_target = ov->grp_target;
      tail.overflow = ov->overflow;
      tail.t_end = ov->t_end;
      tail.pdl_wait = ov->pdl && !ov->grp_done;
      tail.ready = ov->ready;
      tail.trav_done = ov->trav_done;
    }
    // shared memory: a staged leaf per warp (one CTA per SM).  Behind a
    // leaf-product kernel that signals finished groups, CTAs of 2 warps: one
    // fits beside K3's CTA on every SM (K3 on its 4-stage ring leaves ~95 KB
    // of shared memory), so C's leaves are normed while K3 still runs and
    // only the last groups' leaves remain after it (SPAMM_SEG_OVL_WARPS: 2 or
    // 6 = one 6-warp CTA per SM that starts as K3's CTAs retire)
    static const int ovl_w = getenv("SPAMM_SEG_OVL_WARPS") ? atoi(getenv("SPAMM_SEG_OVL_WARPS")) : 2;
    const int W = (ov && ov->grp_done && ovl_w == 2) ? 2 : SEG_WARPS;
    const unsigned smem = (unsigned)(W * (t->leaf == 64
        ? (f64 ? seg_warp_bytes<double, 64>() : seg_warp_bytes<float, 64>())
        : (f64 ? seg_warp_bytes<double, 32>() : seg_warp_bytes<float, 32>())));
    const int64_t cap = std::min<int64_t>(list_cap, t->nb * t->nb);
    // beside K3: warps take leaves from a ticket (the CTA per SM that joins
    // K3 works through the groups as they complete, the CTAs that start as
    // K3 retires share what is left); three 2-warp CTAs per SM in all
    const bool dyn = W == 2 && tail.ticket != nullptr;
    if (dyn) tail.leaf_ticket = ticket + 1;
    static const bool no_par = getenv("SPAMM_NO_K1_PARENTS") != nullptr;
    if (dyn && ov->ne && t->depth >= 1 && !no_par) {
      SPAMM_TRY(ensure_scratch(ctx->k1_pcnt, sizeof(unsigned) * ((size_t)1 << (2 * (t->depth - 1))), st,
                               /*zeroed=*/true));
      tail.ne = ov->ne;
      tail.pcnt = (unsigned *)ctx->k1_pcnt.ptr;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)std::max<int64_t>(
        1, std::min<int64_t>((cap + W - 1) / W, (int64_t)ctx->num_sms * (dyn ? 3 : 1))));
    // (W == 2: + SPAMM_SEG_HELPERS pyramid-only warps)
    static const int seg_helpers_env = getenv("SPAMM_SEG_HELPERS") ? atoi(getenv("SPAMM_SEG_HELPERS")) : 0;
    const int seg_helpers = seg_helpers_env == 1 || seg_helpers_env == 2 ? seg_helpers_env : 0;
    cfg.blockDim = dim3(32 * (W == 2 ? 2 + seg_helpers : W));
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    if (ov && (ov->grp_done || ov->pdl)) {
      attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
    }
    auto launch = [&](auto kern, auto *data) -> int {
      SPAMM_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      // (the same shared-memory carveout as K3: a CTA can only join an SM
      // whose L1 / shared split it accepts)
      SPAMM_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
      SPAMM_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, data, t->N, t->nb, t->nsq + level_offset(t->depth),
                                        t->occ + level_offset(t->depth), list, list_count, tail, smem));
      return SPAMM_OK;
    };
    double *pd = (double *)t->padded;
    float *pf = (float *)t->padded;
    if (W == 2) {
      if (seg_helpers == 2) {
        if (t->leaf == 64) SPAMM_TRY(f64 ? launch(leaf_norm_seg_kernel<double, 64, 2, 2>, pd) : launch(leaf_norm_seg_kernel<float, 64, 2, 2>, pf));
        else SPAMM_TRY(f64 ? launch(leaf_norm_seg_kernel<double, 32, 2, 2>, pd) : launch(leaf_norm_seg_kernel<float, 32, 2, 2>, pf));
      } else if (seg_helpers == 1) {
        if (t->leaf == 64) SPAMM_TRY(f64 ? launch(leaf_norm_seg_kernel<double, 64, 2, 1>, pd) : launch(leaf_norm_seg_kernel<float, 64, 2, 1>, pf));
        else SPAMM_TRY(f64 ? launch(leaf_norm_seg_kernel<double, 32, 2, 1>, pd) : launch(leaf_norm_seg_kernel<float, 32, 2, 1>, pf));
      } else {
        if (t->leaf == 64) SPAMM_TRY(f64 ? launch(leaf_norm_seg_kernel<double, 64, 2>, pd) : launch(leaf_norm_seg_kernel<float, 64, 2>, pf));
        else SPAMM_TRY(f64 ? launch(leaf_norm_seg_kernel<double, 32, 2>, pd) : launch(leaf_norm_seg_kernel<float, 32, 2>, pf));
      }
    } else if (t->leaf == 64) {
      SPAMM_TRY(f64 ? launch(leaf_norm_seg_kernel<double, 64>, pd) : launch(leaf_norm_seg_kernel<float, 64>, pf));
    } else {
      SPAMM_TRY(f64 ? launch(leaf_norm_seg_kernel<double, 32>, pd) : launch(leaf_norm_seg_kernel<float, 32>, pf));
    }
    fused = !tail.skip_pyramid;
  } else if (t->dtype == SPAMM_DTYPE_F64)
    SPAMM_TRY(launch_leaf_norms<double>(t, st, list, list_count, list_cap, ticket, ov, &fused));
  else
    SPAMM_TRY(launch_leaf_norms<float>(t, st, list, list_count, list_cap, ticket, ov, &fused));
  if (launches) ++*launches;
  if (fused) return SPAMM_OK;  // the last K1 CTA built the pyramid
  return pyramid_upper_async(ctx, t, st, launches);
}

// The levels above the leaves (and every interior nrm) from t's leaf level:
// parents ((c11 + c12) + c21) + c22 and occupancy OR (quadtree.py:90-92,
// :135-138).  Stream-ordered.
int pyramid_upper_async(DeviceContext *ctx, spamm_tree *t, cudaStream_t st, int *launches) {
  Scratch &pyt = st == ctx->copy_in ? ctx->pyr_tickets_in : ctx->pyr_tickets;
  static bool carve = false;
  if (!carve) {
    cudaFuncSetAttribute(pyramid_fused_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    carve = true;
  }
  const PyrPlan pl = pyramid_plan(t->depth);
  if (pl.passes == 0) {
    pyramid_fused_kernel<<<1, 32, 0, st>>>(t->nsq, t->occ, t->nrm, pl, nullptr);
  } else {
    // tickets start (and are left) at zero
    const size_t need = sizeof(unsigned) * (size_t)std::max<int64_t>(pl.n_counters, 1);
    SPAMM_TRY(ensure_scratch(pyt, need, st, /*zeroed=*/true));
    pyramid_fused_kernel<<<(unsigned)(int64_t(1) << (2 * (pl.from[0] - pl.L[0]))), PYR_THREADS, 0,
                           st>>>(t->nsq, t->occ, t->nrm, pl, (unsigned *)pyt.ptr);
  }
  SPAMM_CUDA_TRY(cudaGetLastError());
  if (launches) ++*launches;
  return SPAMM_OK;
}

int alloc_tree(DeviceContext *ctx, int64_t n, int32_t leaf, int32_t dtype, spamm_tree **out,
               cudaStream_t st = nullptr) {
  if (!st) st = ctx->stream;
  auto t = std::make_unique<spamm_tree>();
  t->n = n;
  t->leaf = leaf;
  t->depth = depth_for(n, leaf);
  t->N = int64_t(leaf) << t->depth;
  t->nb = t->N / leaf;
  t->dtype = dtype;
  t->device = ctx->device;
  const int64_t esz = t->elem_size();
  SPAMM_CUDA_TRY(dev_alloc((void **)&t->padded, (size_t)(t->N * t->N * esz), st));
  SPAMM_CUDA_TRY(dev_alloc((void **)&t->nsq, sizeof(double) * pyramid_size(t->depth),
                                 st));
  SPAMM_CUDA_TRY(dev_alloc((void **)&t->occ, pyramid_size(t->depth), st));
  SPAMM_CUDA_TRY(dev_alloc((void **)&t->nrm, sizeof(double) * pyramid_size(t->depth),
                                 st));
  *out = t.release();
  return SPAMM_OK;
}

int tree_join(DeviceContext *ctx, const spamm_tree *t) {
  if (t && t->ready) SPAMM_CUDA_TRY(cudaStreamWaitEvent(ctx->stream, t->ready, 0));
  return SPAMM_OK;
}

void free_tree_async(spamm_tree *t, cudaStream_t st) {
  if (!t) return;
  if (t->ready) {  // (st is the library's stream, which may not have joined yet)
    cudaStreamWaitEvent(st, t->ready, 0);
    cudaEventDestroy(t->ready);
  }
  if (t->padded) cudaFreeAsync(t->padded, st);
  if (t->nsq) cudaFreeAsync(t->nsq, st);
  if (t->occ) cudaFreeAsync(t->occ, st);
  if (t->nrm) cudaFreeAsync(t->nrm, st);
  delete t;
}

// zero every leaf block whose occupancy is clear (one warp per block)
__global__ void zero_unoccupied_kernel(unsigned char *__restrict__ padded, int64_t N, int32_t leaf,
                                       int64_t nb, int esz, const uint8_t *__restrict__ occ_leaf) {
  const int lane = threadIdx.x & 31;
  const int64_t G = nb * nb, row_bytes = (int64_t)leaf * esz;
  for (int64_t g = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; g < G;
       g += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    if (occ_leaf[g]) continue;  // warp-uniform
    const int64_t bi = g / nb, bj = g - bi * nb;
    unsigned char *base = padded + (bi * leaf) * N * esz + bj * row_bytes;
    if (row_bytes % 16 == 0) {
      const int per_row = (int)(row_bytes / 16);
      for (int e = lane; e < per_row * leaf; e += 32) {
        const int r = e / per_row, c = e - r * per_row;
        reinterpret_cast<uint4 *>(base + (int64_t)r * N * esz)[c] = make_uint4(0u, 0u, 0u, 0u);
      }
    } else {
      for (int64_t e = lane; e < row_bytes * leaf; e += 32) {
        const int64_t r = e / row_bytes, c = e - r * row_bytes;
        base[r * N * esz + c] = 0;
      }
    }
  }
}

int materialize(DeviceContext *ctx, const spamm_tree *tc) {
  spamm_tree *t = const_cast<spamm_tree *>(tc);  // the values (zeros) do not change
  SPAMM_TRY(tree_join(ctx, t));
  if (t->distributed || !t->padded) {
    set_error(t->distributed ? "row band [%lld, %lld) of a distributed tree: only its rows are held "
                               "here (gather the bands first)"
                             : "norms-only tree (no element storage)",
              (long long)t->band_lo, (long long)t->band_hi);
    return SPAMM_ERR_VALUE;
  }
  if (!t->lazy_empty) return SPAMM_OK;
  const int64_t G = t->nb * t->nb;
  const unsigned grid = (unsigned)std::min<int64_t>((G + 7) / 8, (int64_t)ctx->num_sms * 8);
  zero_unoccupied_kernel<<<grid, 256, 0, ctx->stream>>>((unsigned char *)t->padded, t->N, t->leaf,
                                                        t->nb, (int)t->elem_size(),
                                                        t->occ + level_offset(t->depth));
  SPAMM_CUDA_TRY(cudaGetLastError());
  t->lazy_empty = false;
  return SPAMM_OK;
}

int finish_tree(DeviceContext *ctx, spamm_tree *t) {
  const SmallRead r{&t->root_norm_sq, t->nsq, sizeof(double)};
  return read_small_sync(ctx, ctx->stream, &r, 1);
}

static int validate_shape(int64_t n, int64_t ld, int32_t leaf, int32_t dtype) {
  if (leaf < 1 || (leaf & (leaf - 1)) != 0) {
    set_error("leaf_size must be a power of two >= 1, got %d", leaf);
    return SPAMM_ERR_VALUE;
  }
  if (dtype != SPAMM_DTYPE_F64 && dtype != SPAMM_DTYPE_F32) {
    set_error("unsupported element dtype code %d", dtype);
    return SPAMM_ERR_VALUE;
  }
  if (n < 1) {
    set_error("matrix dimension must be >= 1");
    return SPAMM_ERR_VALUE;
  }
  if (ld < n) {
    set_error("leading dimension %lld < n %lld", (long long)ld, (long long)n);
    return SPAMM_ERR_VALUE;
  }
  return SPAMM_OK;
}

static int tree_from(const void *src, bool src_on_host, int64_t n, int64_t ld, int32_t leaf,
                     int32_t dtype, int32_t device, spamm_tree **out) {
  SPAMM_TRY(validate_shape(n, ld, leaf, dtype));
  DeviceContext *ctx;
  SPAMM_TRY(get_context(device, &ctx));
  std::lock_guard<std::mutex> lk(ctx->mu);
  NvtxRange nvtx_build(src_on_host ? "spamm.K1.tree_from_host" : "spamm.K1.tree_from_device");
  spamm_tree *t = nullptr;
  SPAMM_TRY(alloc_tree(ctx, n, leaf, dtype, &t));
  const int64_t esz = t->elem_size();
  int rc = SPAMM_OK;
  // Fused build (f64 device source that fills the padded matrix exactly, 16-byte
  // aligned rows): K1 reads the source once and writes the tree's storage as
  // it squares -- no separate device-to-device copy (SPAMM_NO_FUSED_BUILD: copy, then K1)
  static const bool no_fused = getenv("SPAMM_NO_FUSED_BUILD") != nullptr;
  const bool fuse = !src_on_host && !no_fused && dtype == SPAMM_DTYPE_F64 && t->N == n &&
                    leaf * esz >= 16 && ld % 2 == 0 && ((uintptr_t)src & 15) == 0;
  do {
    cudaError_t e;
    if (fuse) {
      rc = build_pyramid_async(ctx, t, ctx->stream, nullptr, nullptr, nullptr, 0, nullptr, 0, nullptr,
                               nullptr, nullptr, nullptr, src, ld);
      if (rc) break;
      rc = finish_tree(ctx, t);
      break;
    }
    if (t->N != n) {
      e = cudaMemsetAsync(t->padded, 0, (size_t)(t->N * t->N * esz), ctx->stream);
      if (e != cudaSuccess) { set_error("memset: %s", cudaGetErrorString(e)); rc = SPAMM_ERR_CUDA; break; }
    }
    e = cudaMemcpy2DAsync(t->padded, (size_t)(t->N * esz), src, (size_t)(ld * esz),
                          (size_t)(n * esz), (size_t)n,
                          src_on_host ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice,
                          ctx->stream);
    if (e != cudaSuccess) { set_error("copy: %s", cudaGetErrorString(e)); rc = SPAMM_ERR_CUDA; break; }
    rc = build_pyramid_async(ctx, t, ctx->stream, nullptr, nullptr, nullptr, 0, nullptr, 0, nullptr,
                             nullptr);
    if (rc) break;
    rc = finish_tree(ctx, t);
  } while (0);
  if (rc) {
    free_tree_async(t, ctx->stream);
    return rc;
  }
  *out = t;
  return SPAMM_OK;
}

// -------------------------------------------------------- ||A - B||_F kernel
template <typename T>
__global__ void diff_sq_kernel(const T *__restrict__ a, const T *__restrict__ b, int64_t count,
                               double *__restrict__ partial) {
  __shared__ double red[32];
  double acc = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double d = (double)a[i] - (double)b[i];
    acc = fma(d, d, acc);
  }
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    acc = threadIdx.x < blockDim.x / 32 ? red[threadIdx.x] : 0.0;
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (threadIdx.x == 0) partial[blockIdx.x] = acc;
  }
}

__global__ void sum_partials_kernel(const double *__restrict__ partial, int n, double *out) {
  __shared__ double red[32];
  double acc = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) acc += partial[i];
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    acc = threadIdx.x < blockDim.x / 32 ? red[threadIdx.x] : 0.0;
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (threadIdx.x == 0) *out = sqrt(acc);
  }
}

}  // namespace spamm

using namespace spamm;

extern "C" {

const char *spamm_last_error(void) { return g_last_error.c_str(); }

const char *spamm_version(void) { return "spamm_b200 0.1 sm_100a"; }

int spamm_device_count(int *count) {
  SPAMM_CUDA_TRY(cudaGetDeviceCount(count));
  return SPAMM_OK;
}

int spamm_tree_from_host(const void *host, int64_t n, int64_t ld, int32_t leaf, int32_t dtype,
                         int32_t device, spamm_tree **out) {
  return tree_from(host, true, n, ld, leaf, dtype, device, out);
}

int spamm_tree_from_host_async(const void *host, int64_t n, int64_t ld, int32_t leaf,
                               int32_t dtype, int32_t device, spamm_tree **out) {
  SPAMM_TRY(validate_shape(n, ld, leaf, dtype));
  if (!out) {
    set_error("null argument");
    return SPAMM_ERR_VALUE;
  }
  DeviceContext *ctx;
  SPAMM_TRY(get_context(device, &ctx));
  std::lock_guard<std::mutex> lk(ctx->mu);
  // everything on copy_in: allocation, padding, copy, K1 + pyramid (its own
  // tickets), then the `ready` event later uses wait on
  cudaStream_t st = ctx->copy_in;
  spamm_tree *t = nullptr;
  SPAMM_TRY(alloc_tree(ctx, n, leaf, dtype, &t, st));
  const int64_t esz = t->elem_size();
  int rc = SPAMM_OK;
  do {
    if (t->N != n && (rc = zero_async(t->padded, (size_t)(t->N * t->N * esz), st, 4 * ctx->num_sms)))
      break;
    cudaError_t e = cudaMemcpy2DAsync(t->padded, (size_t)(t->N * esz), host, (size_t)(ld * esz),
                                      (size_t)(n * esz), (size_t)n, cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) { set_error("copy: %s", cudaGetErrorString(e)); rc = SPAMM_ERR_CUDA; break; }
    rc = build_pyramid_async(ctx, t, st, nullptr, nullptr, nullptr, 0, nullptr, 0, nullptr, nullptr);
    if (rc) break;
    e = cudaEventCreateWithFlags(&t->ready, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventRecord(t->ready, st);
    if (e != cudaSuccess) { set_error("event: %s", cudaGetErrorString(e)); rc = SPAMM_ERR_CUDA; break; }
    t->root_pending = true;
  } while (0);
  if (rc) {
    cudaStreamSynchronize(st);
    if (t->ready) {
      cudaEventDestroy(t->ready);
      t->ready = nullptr;
    }
    free_tree_async(t, st);
    return rc;
  }
  *out = t;
  return SPAMM_OK;
}

int spamm_tree_wait(const spamm_tree *tc) {
  if (!tc) { set_error("null tree"); return SPAMM_ERR_VALUE; }
  spamm_tree *t = const_cast<spamm_tree *>(tc);  // completes a pending build; values unchanged
  DeviceContext *ctx;
  SPAMM_TRY(get_context(t->device, &ctx));
  std::lock_guard<std::mutex> lk(ctx->mu);
  if (!t->ready) return SPAMM_OK;
  SPAMM_CUDA_TRY(cudaEventSynchronize(t->ready));
  if (t->root_pending) {
    SPAMM_TRY(tree_join(ctx, t));
    const SmallRead r{&t->root_norm_sq, t->nsq, sizeof(double)};
    SPAMM_TRY(read_small_sync(ctx, ctx->stream, &r, 1));
    t->root_pending = false;
  }
  return SPAMM_OK;
}

int spamm_tree_from_device(const void *dev, int64_t n, int64_t ld, int32_t leaf, int32_t dtype,
                           int32_t device, spamm_tree **out) {
  return tree_from(dev, false, n, ld, leaf, dtype, device, out);
}

int spamm_stream_wait(int32_t device, spamm_stream_t producer) {
  DeviceContext *ctx;
  SPAMM_TRY(get_context(device, &ctx));
  std::lock_guard<std::mutex> lk(ctx->mu);
  SPAMM_CUDA_TRY(cudaEventRecord(ctx->handoff, (cudaStream_t)producer));
  SPAMM_CUDA_TRY(cudaStreamWaitEvent(ctx->stream, ctx->handoff, 0));
  return SPAMM_OK;
}

int spamm_stream_signal(int32_t device, spamm_stream_t consumer) {
  DeviceContext *ctx;
  SPAMM_TRY(get_context(device, &ctx));
  std::lock_guard<std::mutex> lk(ctx->mu);
  SPAMM_CUDA_TRY(cudaEventRecord(ctx->handoff, ctx->stream));
  SPAMM_CUDA_TRY(cudaStreamWaitEvent((cudaStream_t)consumer, ctx->handoff, 0));
  return SPAMM_OK;
}

int spamm_tree_from_device_on(const void *dev, int64_t n, int64_t ld, int32_t leaf, int32_t dtype,
                              int32_t device, spamm_stream_t stream, spamm_tree **out) {
  SPAMM_TRY(spamm_stream_wait(device, stream));
  SPAMM_TRY(tree_from(dev, false, n, ld, leaf, dtype, device, out));
  return spamm_stream_signal(device, stream);
}

int spamm_tree_from_padded_device(const void *dev_padded, int64_t n, int64_t padded_dim,
                                  int32_t leaf, int32_t dtype, int32_t device, spamm_tree **out) {
  SPAMM_TRY(validate_shape(n, n, leaf, dtype));
  if ((int64_t(leaf) << depth_for(n, leaf)) != padded_dim) {
    set_error("padded_dim %lld inconsistent with n=%lld leaf=%d", (long long)padded_dim,
              (long long)n, leaf);
    return SPAMM_ERR_DIMENSION;
  }
  SPAMM_TRY(tree_from(dev_padded, false, padded_dim, padded_dim, leaf, dtype, device, out));
  (*out)->n = n;
  return SPAMM_OK;
}

int spamm_tree_info_get(const spamm_tree *t, spamm_tree_info *info) {
  if (!t || !info) { set_error("null tree"); return SPAMM_ERR_VALUE; }
  info->logical_dim = t->n;
  info->padded_dim = t->N;
  info->block_grid = t->nb;
  info->leaf_size = t->leaf;
  info->depth = t->depth;
  info->dtype = t->dtype;
  info->device = t->device;
  info->root_norm_sq = t->root_pending ? NAN : t->root_norm_sq;  // (spamm_tree_wait fetches it)
  return SPAMM_OK;
}

int spamm_tree_to_host(const spamm_tree *t, void *host, int64_t ld) {
  if (!t) { set_error("null tree"); return SPAMM_ERR_VALUE; }
  DeviceContext *ctx;
  SPAMM_TRY(get_context(t->device, &ctx));
  std::lock_guard<std::mutex> lk(ctx->mu);
  SPAMM_TRY(materialize(ctx, t));
  const int64_t esz = t->elem_size();
  SPAMM_CUDA_TRY(cudaMemcpy2DAsync(host, (size_t)(ld * esz), t->padded, (size_t)(t->N * esz),
                                   (size_t)(t->n * esz), (size_t)t->n, cudaMemcpyDeviceToHost,
                                   ctx->stream));
  SPAMM_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  return SPAMM_OK;
}

int spamm_tree_padded_to_host(const spamm_tree *t, void *host) {
  if (!t) { set_error("null tree"); return SPAMM_ERR_VALUE; }
  DeviceContext *ctx;
  SPAMM_TRY(get_context(t->device, &ctx));
  std::lock_guard<std::mutex> lk(ctx->mu);
  SPAMM_TRY(materialize(ctx, t));
  SPAMM_CUDA_TRY(cudaMemcpyAsync(host, t->padded, (size_t)(t->N * t->N * t->elem_size()),
                                 cudaMemcpyDeviceToHost, ctx->stream));
  SPAMM_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  return SPAMM_OK;
}

int spamm_tree_pyramid_to_host(const spamm_tree *t, double *nsq, uint8_t *occ) {
  if (!t) { set_error("null tree"); return SPAMM_ERR_VALUE; }
  DeviceContext *ctx;
  SPAMM_TRY(get_context(t->device, &ctx));
  std::lock_guard<std::mutex> lk(ctx->mu);
  SPAMM_TRY(tree_join(ctx, t));
  const int64_t P = pyramid_size(t->depth);
  const SmallRead r[2] = {{nsq, t->nsq, nsq ? sizeof(double) * P : 0},
                         {occ, t->occ, occ ? (size_t)P : 0}};
  return read_small_sync(ctx, ctx->stream, r, 2);
}

int spamm_tree_recompute_norms(const spamm_tree *t, double *nsq_host) {
  if (!t || !nsq_host) { set_error("null argument"); return SPAMM_ERR_VALUE; }
  DeviceContext *ctx;
  SPAMM_TRY(get_context(t->device, &ctx));
  std::lock_guard<std::mutex> lk(ctx->mu);
  SPAMM_TRY(materialize(ctx, t));
  // a view of the same leaf data with a scratch pyramid
  spamm_tree view = *t;
  view.nsq = nullptr;
  view.occ = nullptr;
  view.nrm = nullptr;
  const int64_t P = pyramid_size(t->depth);
  int rc = SPAMM_OK;
  cudaError_t e = dev_alloc((void **)&view.nsq, sizeof(double) * P, ctx->stream);
  if (e == cudaSuccess) e = dev_alloc((void **)&view.occ, P, ctx->stream);
  if (e == cudaSuccess) e = dev_alloc((void **)&view.nrm, sizeof(double) * P, ctx->stream);
  if (e == cudaSuccess) {
    rc = build_pyramid_async(ctx, &view, ctx->stream, nullptr, nullptr, nullptr, 0, nullptr, 0,
                             nullptr, nullptr);
    if (rc == SPAMM_OK)
      e = cudaMemcpyAsync(nsq_host, view.nsq, sizeof(double) * P, cudaMemcpyDeviceToHost,
                          ctx->stream);
  }
  if (view.nsq) cudaFreeAsync(view.nsq, ctx->stream);
  if (view.occ) cudaFreeAsync(view.occ, ctx->stream);
  if (view.nrm) cudaFreeAsync(view.nrm, ctx->stream);
  const cudaError_t es = cudaStreamSynchronize(ctx->stream);
  if (rc) return rc;
  if (e == cudaSuccess) e = es;
  if (e != cudaSuccess) {
    set_error("norm recompute: %s", cudaGetErrorString(e));
    return e == cudaErrorMemoryAllocation ? SPAMM_ERR_NOMEM : SPAMM_ERR_CUDA;
  }
  return SPAMM_OK;
}

int spamm_tree_device_ptrs(const spamm_tree *t, void **padded, double **nsq, uint8_t **occ) {
  if (!t) { set_error("null tree"); return SPAMM_ERR_VALUE; }
  {
    // the caller may read any of the storage (a distributed band hands out
    // its raw storage: only its own rows and fetched blocks are defined)
    DeviceContext *ctx;
    SPAMM_TRY(get_context(t->device, &ctx));
    std::lock_guard<std::mutex> lk(ctx->mu);
    if (padded && t->lazy_empty && !t->distributed) SPAMM_TRY(materialize(ctx, t));
    else SPAMM_TRY(tree_join(ctx, t));
    SPAMM_CUDA_TRY(cudaStreamSynchronize(ctx->stream));  // (every queued write is visible)
  }
  if (padded) *padded = t->padded;
  if (nsq) *nsq = t->nsq;
  if (occ) *occ = t->occ;
  return SPAMM_OK;
}

int spamm_tree_diff_norm(const spamm_tree *a, const spamm_tree *b, double *out) {
  if (!a || !b) { set_error("null tree"); return SPAMM_ERR_VALUE; }
  if (a->N != b->N || a->dtype != b->dtype || a->device != b->device) {
    set_error("trees not conformable for difference norm");
    return SPAMM_ERR_DIMENSION;
  }
  DeviceContext *ctx;
  SPAMM_TRY(get_context(a->device, &ctx));
  std::lock_guard<std::mutex> lk(ctx->mu);
  SPAMM_TRY(materialize(ctx, a));
  SPAMM_TRY(materialize(ctx, b));
  const int blocks = ctx->num_sms * 4;
  SPAMM_TRY(ensure_scratch(ctx->reduce_tmp, sizeof(double) * (blocks + 1), ctx->stream));
  double *part = (double *)ctx->reduce_tmp.ptr;
  const int64_t count = a->N * a->N;
  if (a->dtype == SPAMM_DTYPE_F64)
    diff_sq_kernel<double><<<blocks, 256, 0, ctx->stream>>>((const double *)a->padded,
                                                             (const double *)b->padded, count, part);
  else
    diff_sq_kernel<float><<<blocks, 256, 0, ctx->stream>>>((const float *)a->padded,
                                                            (const float *)b->padded, count, part);
  sum_partials_kernel<<<1, 1024, 0, ctx->stream>>>(part, blocks, part + blocks);
  SPAMM_CUDA_TRY(cudaGetLastError());
  SPAMM_CUDA_TRY(cudaMemcpyAsync(out, part + blocks, sizeof(double), cudaMemcpyDeviceToHost,
                                 ctx->stream));
  SPAMM_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  return SPAMM_OK;
}

void spamm_tree_free(spamm_tree *t) {
  if (!t) return;
  DeviceContext *ctx;
  if (get_context(t->device, &ctx) != SPAMM_OK) return;
  std::lock_guard<std::mutex> lk(ctx->mu);
  // an asynchronous build may still be reading the caller's host array: the
  // caller may release that array once this returns
  if (t->ready) cudaEventSynchronize(t->ready);
  free_tree_async(t, ctx->stream);
}

}  // extern "C"
