// norms.cuh -- leaf-norm building blocks shared by the C-tree kernels
// (csrc/tree.cu) and the leaf-product kernel's fused norm warp (csrc/leaf.cu):
// raw-bit views, the segmented exact chain of one staged leaf, and the
// one-CTA norm/occupancy pyramid.
#pragma once
#include "common.cuh"

namespace spamm {

__device__ __forceinline__ unsigned long long k1_gt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

template <typename T>
struct Bits;
template <>
struct Bits<double> {
  using U = unsigned long long;
  __device__ static U of(double x) { return (U)__double_as_longlong(x); }
};
template <>
struct Bits<float> {
  using U = unsigned int;
  __device__ static U of(float x) { return (U)__float_as_uint(x); }
};


// Fused pyramid tail of K1 (small trees): the last CTA of the leaf-norm
// launch to finish reduces the whole pyramid in its shared memory, so C's
// tree costs one launch.  ticket == nullptr disables it.
struct PyrTail {
  unsigned *ticket;  // zero at rest; the last CTA resets it
  double *nsq;
  uint8_t *occ;
  double *nrm;
  int depth;
  // Overlap with the leaf-product kernel (list mode, programmatic dependent
  // launch): a leaf is read only once grp_done[slot] reaches grp_target
  // (every warp tile of that C block stored); its chain lane then resets the
  // counter.  Skipped when *overflow (the product is discarded and re-run).
  unsigned *grp_done;
  unsigned grp_target;
  const int *overflow;
  unsigned long long *t_end;  // %globaltimer when the C tree is complete
  int pdl_wait;               // launched programmatically without grp_done: wait for the grid
  // bitmask groups (the leaf-product kernel started on the traversal's group
  // list, not its completion): wait for *ready before reading the list, and
  // the last CTA waits for *trav_done (the traversal's statistics final)
  // before the kernel may complete
  const unsigned *ready;
  const unsigned *trav_done;
  // fused build (dense f64 tree from device memory, n == N): the producers
  // read the leaves from fuse_src (leading dimension fuse_ld) instead of the
  // tree's storage, and the squarer warps write the raw values into the
  // storage as they square them -- the source is read once, no separate copy
  const void *fuse_src;
  int64_t fuse_ld;
  // dynamic leaf assignment (segmented-chain kernel beside K3): warps take
  // list slots from this counter in completion order instead of a fixed
  // stride; zero at rest, reset by the last CTA with `ticket`
  unsigned *leaf_ticket;
  // ... and the leaves' parents built as their last listed child completes:
  // ne = the product's non-empty leaf blocks (bit i * nb + j), pcnt = finished
  // children per parent (zero at rest); the last CTA's pyramid then starts
  // one level up (the parent level is zeroed by the traversal)
  const uint32_t *ne;
  unsigned *pcnt;
  // trees deeper than PYR_TAIL_MAX_DEPTH beside K3: the last CTA only resets
  // the tickets; the pyramid above the leaves is a launch of its own
  int skip_pyramid;
};

__device__ __forceinline__ void spin_acquire_nonzero(const unsigned *flag) {
  for (;;) {
    unsigned v;
    asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
    if (v) break;
    __nanosleep(64);
  }
}

// Whole pyramid above the leaves in one CTA: parent = ((c11 + c12) + c21) +
// c22 (quadtree.py:90-92), occupancy OR, nrm = rn(sqrt(nsq)) for every
// interior node.  Levels too large for the CTA's shared memory are reduced
// straight from global memory (L2), the rest in shared memory.
// Level k nodes [e0, e0 + 4 * blockDim) of this thread from their children in
// global memory: all 16 child loads in flight before any store.
__device__ __forceinline__ void pyr_nodes_from_global(const PyrTail &pt, int k, int e0, int n,
                                                      double *sv, uint8_t *so) {
  const int ps = 1 << k, side = 2 * ps;
  const int64_t lc = level_offset(k + 1), lo = level_offset(k);
  double cn[4][4];
  uint8_t co[4][4];
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int e = e0 + u * (int)blockDim.x;
    const int ee = e < n ? e : 0;
    const int r = ee >> k, c = ee & (ps - 1);
    const int64_t f0 = lc + (int64_t)(2 * r) * side + 2 * c, f1 = f0 + side;
    cn[u][0] = __ldcg(pt.nsq + f0);
    cn[u][1] = __ldcg(pt.nsq + f0 + 1);
    cn[u][2] = __ldcg(pt.nsq + f1);
    cn[u][3] = __ldcg(pt.nsq + f1 + 1);
    co[u][0] = __ldcg(pt.occ + f0);
    co[u][1] = __ldcg(pt.occ + f0 + 1);
    co[u][2] = __ldcg(pt.occ + f1);
    co[u][3] = __ldcg(pt.occ + f1 + 1);
  }
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int e = e0 + u * (int)blockDim.x;
    if (e < n) {
      const double v = __dadd_rn(__dadd_rn(__dadd_rn(cn[u][0], cn[u][1]), cn[u][2]), cn[u][3]);
      const uint8_t o = co[u][0] | co[u][1] | co[u][2] | co[u][3];
      pt.nsq[lo + e] = v;
      pt.occ[lo + e] = o;
      pt.nrm[lo + e] = __dsqrt_rn(v);
      if (sv) {
        sv[e] = v;
        so[e] = o;
      }
    }
  }
}

__device__ inline void pyramid_cta(const PyrTail &pt, unsigned char *smem, size_t smem_bytes,
                                   unsigned long long *dbg = nullptr) {
  auto stamp = [&](int q) {
    if (dbg && threadIdx.x == 0) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
      dbg[q] = t;
    }
  };
  int k = pt.depth - 1;
  if (k < 0) return;
  // global-memory levels until one fits (with the next) in shared memory
  auto fits = [&](int kk) { return (size_t)(1u << (2 * kk)) * 9 * 5 / 4 + 16 <= smem_bytes; };
  for (; k > 0 && !fits(k); --k) {
    const int n = 1 << (2 * k);
    for (int e0 = threadIdx.x; e0 < n; e0 += 4 * blockDim.x)
      pyr_nodes_from_global(pt, k, e0, n, nullptr, nullptr);
    __syncthreads();
  }
  const int n0 = 1 << (2 * k);
  double *bufA = reinterpret_cast<double *>(smem);
  double *bufB = bufA + n0;
  uint8_t *oA = reinterpret_cast<uint8_t *>(bufB + (n0 >> 2) + 1);
  uint8_t *oB = oA + n0;
  stamp(0);
  for (int e0 = threadIdx.x; e0 < n0; e0 += 4 * blockDim.x) pyr_nodes_from_global(pt, k, e0, n0, bufA, oA);
  __syncthreads();
  stamp(1);
  int side = 1 << k;
  for (--k; k >= 0; --k) {
    const int ps = side >> 1;
    const int64_t lo = level_offset(k);
    for (int e = threadIdx.x; e < ps * ps; e += blockDim.x) {
      const int r = e / ps, c = e - r * ps;
      const int f0 = (2 * r) * side + 2 * c, f1 = f0 + side;
      const double v = __dadd_rn(__dadd_rn(__dadd_rn(bufA[f0], bufA[f0 + 1]), bufA[f1]), bufA[f1 + 1]);
      const uint8_t o = oA[f0] | oA[f0 + 1] | oA[f1] | oA[f1 + 1];
      bufB[e] = v;
      oB[e] = o;
      pt.nsq[lo + e] = v;
      pt.occ[lo + e] = o;
      pt.nrm[lo + e] = __dsqrt_rn(v);
    }
    __syncthreads();
    double *td = bufA; bufA = bufB; bufB = td;
    uint8_t *to = oA; oA = oB; oB = to;
    side = ps;
  }
  stamp(2);
}

// whole-pyramid tails are used up to this depth (one CTA: 4^depth leaves)
constexpr int PYR_TAIL_MAX_DEPTH = 6;


constexpr int SEG_PAD = 16;  // bytes after each staged segment

// 2^k for k in [-1074, 1023] (subnormal powers included), exactly
__device__ __forceinline__ double pow2_exact(int k) {
  return k >= -1022 ? __longlong_as_double((long long)(1023 + k) << 52)
                    : __longlong_as_double(1ll << (k + 1074));
}

template <typename T, int LEAF>
__host__ __device__ constexpr int seg_stride() {  // bytes per staged segment
  return LEAF * LEAF / 64 * (int)sizeof(T) + SEG_PAD;
}
template <typename T, int LEAF>
__host__ __device__ constexpr int seg_warp_bytes() {
  return 64 * seg_stride<T, LEAF>();
}

struct SegInfo {
  long long D;  // sum of rnd_u(s_i) (simple segments)
  int E;        // binade exponent (simple segments)
  int simple;
};

template <typename T, int LEAF>
__device__ __forceinline__ double seg_chain(const unsigned char *seg_base, double acc) {
  constexpr int L = LEAF * LEAF / 64;
  const T *x = reinterpret_cast<const T *>(seg_base);
#pragma unroll 16
  for (int i = 0; i < L; ++i) {
    const double v = (double)x[i];
    acc = __dadd_rn(acc, __dmul_rn(v, v));
  }
  return acc;
}


// The squared Frobenius norm of one leaf staged in shared memory as 64
// row-major segments of LEAF^2/64 elements, each followed by SEG_PAD bytes
// (`wsm`), computed by one warp exactly as the reference's sequential chain
// (see the segmented-chain notes in tree.cu).  `bits` returns this lane's OR
// of the raw element bits (OR them over the warp for the occupancy / -0.0
// tests); `tbl` is 64 SegInfo of per-warp shared scratch.
template <typename T, int LEAF>
__device__ __forceinline__ double seg_leaf_norm(const unsigned char *wsm, SegInfo *tbl, int lane,
                                                typename Bits<T>::U &bits) {
  using U = typename Bits<T>::U;
  constexpr int L = LEAF * LEAF / 64;  // segment length (elements)
  constexpr int SS = seg_stride<T, LEAF>();
  // pass 1, segments lane and lane + 32: raw-bit OR, float sum estimates
  bool finite[2];
  double est[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const T *sx = reinterpret_cast<const T *>(wsm + (lane + 32 * h) * SS);
    double p4[4] = {0.0, 0.0, 0.0, 0.0};
    bool fin = true;
#pragma unroll 16
    for (int i = 0; i < L; ++i) {
      const T x = sx[(i + lane) & (L - 1)];
      bits |= Bits<T>::of(x);
      const double sq = __dmul_rn((double)x, (double)x);
      fin &= sq <= 1.79e308;  // false for inf and NaN
      p4[i & 3] += sq;
    }
    finite[h] = fin;
    est[h] = (p4[0] + p4[1]) + (p4[2] + p4[3]);
  }
  double pre0 = est[0], pre1 = est[1];  // inclusive scans in segment order
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double y0 = __shfl_up_sync(0xffffffffu, pre0, o);
    const double y1 = __shfl_up_sync(0xffffffffu, pre1, o);
    if (lane >= o) {
      pre0 += y0;
      pre1 += y1;
    }
  }
  pre1 += __shfl_sync(0xffffffffu, pre0, 31);
  // predicted binade of each segment; D = sum of rnd_u(s_i) where it is one
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int seg = lane + 32 * h;
    const double hi_est = h ? pre1 : pre0, lo_est = hi_est - est[h];
    const double za = lo_est * (1.0 - 0x1p-30), zz = hi_est * (1.0 + 0x1p-30);
    // binade exponents (frexp's) from the bits: the estimates are normal
    // whenever they are used (za > 2^-900, zz < 2^1000)
    const int ea = (int)((__double_as_longlong(za) >> 52) & 0x7ff) - 1022;
    const int ez = (int)((__double_as_longlong(zz) >> 52) & 0x7ff) - 1022;
    bool simp = finite[h] && seg > 0 && za > 0x1p-900 && zz < 0x1p+1000 && ea == ez;
    long long d = 0;
    if (simp) {
      const T *sx = reinterpret_cast<const T *>(wsm + seg * SS);
      const double inv_u = pow2_exact(53 - ea);  // 2^-(E-52), E = ea - 1: exact power of two
      bool tie = false;
#pragma unroll 16
      for (int i = 0; i < L; ++i) {
        const double x = (double)sx[(i + lane) & (L - 1)];
        const double q = __dmul_rn(__dmul_rn(x, x), inv_u);  // exact scaling
        const double fl = floor(q), fr = q - fl;               // both exact
        tie |= fr == 0.5 || q >= 0x1p53;  // (q >= 2^53: the estimate was off)
        d += (long long)fmin(fl, 0x1p53) + (fr > 0.5 ? 1 : 0);
      }
      simp = !tie;
    }
    tbl[seg] = SegInfo{d, ea - 1, (int)simp};  // E: za in [2^E, 2^(E+1))
  }
  __syncwarp();
  // lane 0: the segments in order -- runs of simple segments of one binade
  // applied with one exact add each, everything else by the plain chain
  if (lane == 0) {
    double acc = 0.0;
    int run0 = -1, runE = 0;
    long long runD = 0;
    auto close_run = [&](int end) {
      if (run0 < 0) return;
      const double lo = pow2_exact(runE);
      const double v = acc + (double)runD * pow2_exact(runE - 52);  // exact when it applies
      if (runD < (1ll << 52) && acc >= lo && v < 2.0 * lo) {
        acc = v;  // every partial sum of the run stayed in [2^E, 2^(E+1))
      } else {
        for (int sg = run0; sg < end; ++sg) acc = seg_chain<T, LEAF>(wsm + sg * SS, acc);
      }
      run0 = -1;
    };
    for (int sg = 0; sg < 64; ++sg) {
      const SegInfo si = tbl[sg];
      if (si.simple && run0 >= 0 && si.E == runE) {
        runD += si.D;
        continue;
      }
      close_run(sg);
      if (si.simple) {
        run0 = sg;
        runE = si.E;
        runD = si.D;
      } else {
        acc = seg_chain<T, LEAF>(wsm + sg * SS, acc);
      }
    }
    close_run(64);
    tbl[0].D = __double_as_longlong(acc);
  }
  __syncwarp();
  const double acc = __longlong_as_double(tbl[0].D);
  __syncwarp();  // (the table may be reused right after)
  return acc;
}

}  // namespace spamm
