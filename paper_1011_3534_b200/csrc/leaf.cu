// leaf.cu -- K3: batched leaf-block products with the reference's
// deterministic k-reduction.
//
// Reference: _leaf_stage (multiply.py:224-257) multiplies every retained
// (i, j, k) leaf triple with np.matmul and merges the products of one C block
// with _merge_contributions (multiply.py:119-141): an aligned binary interval
// tree over k -- both halves present -> left + right, one present -> passed
// through bit-intact.
//
// B200 mapping (FP64): one work item = one C block (or a 64x64 sub-tile of
// it for leaves > 64).  Every product P_k = A_ik B_kj is accumulated from
// zero on the FP64 tensor-core path (mma.sync m16n8k16 f64, SASS DMMA) in
// ascending inner index, which is exactly the sequential FMA chain the CPU
// BLAS kernel produces (tools/dmma_order.cu proved DMMA accumulates in that
// order), and the products are merged in the reference's tree order with a
// shunting-yard stack keyed by the level of the lowest common ancestor of
// consecutive k (32 - clz(k_prev ^ k_next)).  Operand tiles stream through a
// 3-stage cp.async pipeline with padded shared-memory rows (conflict-free
// fragment loads); CTAs are persistent and take work items from a ticket.
#include <cstdio>
#include <cstdlib>

#include "leaf.cuh"

namespace spamm {

constexpr int MAXD = 22;  // deepest merge stack (depth <= 21 with 63-bit Morton codes)

__device__ __forceinline__ void cp_async16_l(void *smem, const void *gmem) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__device__ __forceinline__ void dmma16816(double (&c)[4], const double (&a)[8],
                                          const double (&b)[4]) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, "
      "{%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
      : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
        "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
}

// One DMMA.8x8x4: C(8x8) += A(8x4) B(4x8), f64, inner index ascending.  Not
// volatile, so the scheduler may interleave independent accumulators.
__device__ __forceinline__ void dmma884(double &c0, double &c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

// Level at which two distinct inner indices meet in the merge tree.
__device__ __forceinline__ int merge_level(uint32_t k0, uint32_t k1) {
  return 32 - __clz(k0 ^ k1);
}

struct WorkItem {
  int64_t start, end;  // triple range [start, end) of the group
  uint32_t i, j;       // C block
  int si, sj;          // sub-tile
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ bool fetch_work(const LeafArgs &args, int subs_side, int *s_work,
                                           WorkItem &w) {
  if (threadIdx.x == 0) *s_work = (int)atomicAdd(&args.tc->gemm_ticket, 1ull);
  __syncthreads();
  const int item = *s_work;
  const int ng = (int)args.tc->num_groups;
  const int subs = subs_side * subs_side;
  if (item >= ng * subs) return false;
  const int grp = item / subs, sub = item - grp * subs;
  w.si = sub / subs_side;
  w.sj = sub - w.si * subs_side;
  unsigned long long m = *args.n_codes;
  if (m > args.capacity) m = args.capacity;
  w.start = args.group_starts[grp];
  w.end = grp + 1 < ng ? args.group_starts[grp + 1] : (int64_t)m;
  const uint32_t gid = args.group_ids[grp];
  w.i = (uint32_t)(gid / (uint64_t)args.nb);
  w.j = (uint32_t)(gid - (uint64_t)w.i * args.nb);
  return true;
}


// ---------------------------------------------------------------- TMEM stack
// The merge stack's deeper entries live in tensor memory (unused by DMMA):
// each warp owns 32 TMEM lanes (its lane quarter) and NREG columns per stack
// slot, written with tcgen05.st / read with tcgen05.ld (tens of cycles,
// instead of local-memory round trips to L2).
template <int NREG>
__device__ __forceinline__ void tmem_store(uint32_t taddr, const uint32_t (&r)[NREG]);
template <int NREG>
__device__ __forceinline__ void tmem_load(uint32_t taddr, uint32_t (&r)[NREG]);

#define R8(o) "r"(r[o]), "r"(r[o + 1]), "r"(r[o + 2]), "r"(r[o + 3]), "r"(r[o + 4]), "r"(r[o + 5]), "r"(r[o + 6]), "r"(r[o + 7])
#define W8(o) "=r"(r[o]), "=r"(r[o + 1]), "=r"(r[o + 2]), "=r"(r[o + 3]), "=r"(r[o + 4]), "=r"(r[o + 5]), "=r"(r[o + 6]), "=r"(r[o + 7])
template <>
__device__ __forceinline__ void tmem_store<32>(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};\n" ::"r"(taddr),
      R8(0), R8(8), R8(16), R8(24)
      : "memory");
}
template <>
__device__ __forceinline__ void tmem_load<32>(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
      : W8(0), W8(8), W8(16), W8(24)
      : "r"(taddr)
      : "memory");
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
}
template <>
__device__ __forceinline__ void tmem_store<16>(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15,%16};\n" ::"r"(taddr),
      R8(0), R8(8)
      : "memory");
}
template <>
__device__ __forceinline__ void tmem_load<16>(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15}, [%16];\n"
      : W8(0), W8(8)
      : "r"(taddr)
      : "memory");
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
}
#undef R8
#undef W8

// ---------------------------------------------------------------- DMMA path
constexpr int DMMA_BK = 32;
constexpr int DMMA_STAGES = 3;
constexpr int KS_SMEM = 1024;  // group k lists up to this length are staged in smem

// Shared-memory tiles are dense (rows of 256 B for A, 512 B for B) with the
// 16-byte chunks of each 128-byte segment XOR-swizzled by (row & 3) << 1.
// That makes the m16n8k16 fragment loads (4 rows x 2 chunks per half-warp)
// hit 32 distinct banks, and keeps every 128-byte global line landing in one
// 128-byte shared segment for the cp.async copies.
__device__ __forceinline__ int swz(int row, int col) {  // element offset within a row
  const int chunk = col >> 1;
  return (((chunk & ~7) | ((chunk & 7) ^ ((row & 3) << 1))) << 1) | (col & 1);
}

template <int TILE, int WM, int WN>
struct DmmaCfg {
  static constexpr int THREADS = 32 * WM * WN;
  static constexpr int SA = DMMA_BK;      // A row length (doubles)
  static constexpr int SB = TILE;         // B row length (doubles)
  static constexpr int A_ELEMS = TILE * SA;
  static constexpr int B_ELEMS = DMMA_BK * SB;
  static constexpr int STAGE_ELEMS = A_ELEMS + B_ELEMS;
  static constexpr int WTM = TILE / WM;   // warp tile rows
  static constexpr int WTN = TILE / WN;   // warp tile cols
  static constexpr int MT = WTM / 16;     // m16 tiles per warp
  static constexpr int NT = WTN / 8;      // n8 tiles per warp
  static constexpr size_t SMEM = sizeof(double) * DMMA_STAGES * STAGE_ELEMS;
  static constexpr int NREG = MT * NT * 4 * 2;           // b32 registers per accumulator set
  static constexpr int TM_SLOTS = 4;                      // merge-stack slots kept in TMEM
  static constexpr int SLOT_COLS = NREG * ((WM * WN + 3) / 4);
  static constexpr int TM_COLS_RAW = TM_SLOTS * SLOT_COLS;
  static constexpr int TM_COLS = TM_COLS_RAW <= 32 ? 32 : TM_COLS_RAW <= 64 ? 64
                                 : TM_COLS_RAW <= 128 ? 128 : TM_COLS_RAW <= 256 ? 256 : 512;
  static_assert(MT >= 1 && NT >= 1, "warp tile too small");
  static_assert(NREG == 16 || NREG == 32, "TMEM spill width");
  static_assert((TILE * DMMA_BK / 2) % THREADS == 0 && (DMMA_BK * TILE / 2) % THREADS == 0, "");
};

template <int TILE, int WM, int WN>
__global__ void __launch_bounds__(32 * WM * WN, 2) leaf_dmma_kernel(LeafArgs args) {
  using C = DmmaCfg<TILE, WM, WN>;
  constexpr int QA = (TILE * DMMA_BK / 2) / C::THREADS;  // 16-B copies per thread, A stage
  constexpr int QB = (DMMA_BK * TILE / 2) / C::THREADS;  // 16-B copies per thread, B stage
  extern __shared__ __align__(16) double dsm[];
  __shared__ int s_work;
  __shared__ uint32_t s_ks[KS_SMEM];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp / WN, wn = warp % WN, g = lane >> 2, t = lane & 3;
  const int b = args.leaf;
  const int kchunks = b / DMMA_BK;             // a power of two
  const int kshift = __ffs(kchunks) - 1;
  const int subs_side = b / TILE;
  const int64_t N = args.N;
  const double *__restrict__ A = (const double *)args.a;
  const double *__restrict__ B = (const double *)args.b;
  double *__restrict__ Cm = (double *)args.c;

  // ---- loop-invariant shared-memory fragment offsets (elements in a stage).
  // Fragment rows of A are wm*WTM + mt*16 + 8h + g and rows of B are
  // kk + 4*s4 + t, so the swizzle key (row & 3) is g & 3 for A and t for B.
  const int a_row0 = (wm * C::WTM + g) * C::SA;
  int a_col[2][4];
#pragma unroll
  for (int kq = 0; kq < 2; ++kq)
#pragma unroll
    for (int s4 = 0; s4 < 4; ++s4) a_col[kq][s4] = swz(g, 16 * kq + 4 * s4 + t);
  int b_col[C::NT];
#pragma unroll
  for (int nt = 0; nt < C::NT; ++nt)
    b_col[nt] = C::A_ELEMS + t * C::SB + swz(t, wn * C::WTN + nt * 8 + g);
  // ---- loop-invariant copy slots (smem offset, global offset from the tile origin)
  int sA[QA], sB[QB];
  int64_t gA[QA], gB[QB];
#pragma unroll
  for (int q = 0; q < QA; ++q) {
    const int e = tid + q * C::THREADS, r = e / (DMMA_BK / 2), c2 = e % (DMMA_BK / 2);
    sA[q] = r * C::SA + swz(r, 2 * c2);
    gA[q] = (int64_t)r * N + 2 * c2;
  }
#pragma unroll
  for (int q = 0; q < QB; ++q) {
    const int e = tid + q * C::THREADS, r = e / (TILE / 2), c2 = e % (TILE / 2);
    sB[q] = C::A_ELEMS + r * C::SB + swz(r, 2 * c2);
    gB[q] = (int64_t)r * N + 2 * c2;
  }

  // Merge stack of the reference's tree order (see merge_level): pending
  // left operands are keyed by tree level; the op levels on the stack are
  // strictly decreasing from bottom to top, so they form a bit mask whose
  // lowest set bit is the top.  The top value lives in registers; deeper
  // ones in stk[level] (local memory), written back only when dirty.
  double stk[MAXD][C::MT][C::NT][4];  // only slots >= TM_SLOTS (deep stacks)
  double top[C::MT][C::NT][4];
  __shared__ uint32_t s_tmem;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                     (unsigned)__cvta_generic_to_shared(&s_tmem)),
                 "n"(C::TM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t t_my = s_tmem + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)((warp >> 2) * C::NREG);
  auto spill = [&](int slot) {
    if (slot < C::TM_SLOTS) {
      uint32_t r[C::NREG];
#pragma unroll
      for (int mt = 0; mt < C::MT; ++mt)
#pragma unroll
        for (int nt = 0; nt < C::NT; ++nt)
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int x = ((mt * C::NT + nt) * 4 + q) * 2;
            r[x] = (uint32_t)__double2loint(top[mt][nt][q]);
            r[x + 1] = (uint32_t)__double2hiint(top[mt][nt][q]);
          }
      tmem_store<C::NREG>(t_my + slot * C::SLOT_COLS, r);
    } else {
#pragma unroll
      for (int mt = 0; mt < C::MT; ++mt)
#pragma unroll
        for (int nt = 0; nt < C::NT; ++nt)
#pragma unroll
          for (int q = 0; q < 4; ++q) stk[slot][mt][nt][q] = top[mt][nt][q];
    }
  };
  auto reload = [&](int slot) {
    if (slot < C::TM_SLOTS) {
      uint32_t r[C::NREG];
      asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
      tmem_load<C::NREG>(t_my + slot * C::SLOT_COLS, r);
#pragma unroll
      for (int mt = 0; mt < C::MT; ++mt)
#pragma unroll
        for (int nt = 0; nt < C::NT; ++nt)
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int x = ((mt * C::NT + nt) * 4 + q) * 2;
            top[mt][nt][q] = __hiloint2double((int)r[x + 1], (int)r[x]);
          }
    } else {
#pragma unroll
      for (int mt = 0; mt < C::MT; ++mt)
#pragma unroll
        for (int nt = 0; nt < C::NT; ++nt)
#pragma unroll
          for (int q = 0; q < 4; ++q) top[mt][nt][q] = stk[slot][mt][nt][q];
    }
  };

  WorkItem w;
  const unsigned long long t_start = gtimer();
  unsigned items = 0;
  while (fetch_work(args, subs_side, &s_work, w)) {
    ++items;
    const int64_t nk = w.end - w.start;
    const int64_t nsteps = nk * kchunks;
    const bool ks_in_smem = nk <= KS_SMEM;
    if (ks_in_smem)
      for (int e = tid; e < nk; e += C::THREADS) s_ks[e] = args.ks[w.start + e];
    __syncthreads();
    const uint32_t *ks = ks_in_smem ? s_ks : args.ks + w.start;
    const double *a_org = A + (int64_t(w.i) * b + w.si * TILE) * N;
    const double *b_org = B + int64_t(w.j) * b + w.sj * TILE;

    auto issue = [&](int64_t step) {
      double *stg = dsm + (int)(step % DMMA_STAGES) * C::STAGE_ELEMS;
      const int64_t kcol = int64_t(ks[step >> kshift]) * b + (int)(step & (kchunks - 1)) * DMMA_BK;
      const double *asrc = a_org + kcol;
      const double *bsrc = b_org + kcol * N;
#pragma unroll
      for (int q = 0; q < QA; ++q) cp_async16_l(stg + sA[q], asrc + gA[q]);
#pragma unroll
      for (int q = 0; q < QB; ++q) cp_async16_l(stg + sB[q], bsrc + gB[q]);
    };

#pragma unroll
    for (int s = 0; s < DMMA_STAGES - 1; ++s) {
      if (s < nsteps) issue(s);
      cp_commit();
    }

    double acc[C::MT][C::NT][4];
#pragma unroll
    for (int mt = 0; mt < C::MT; ++mt)
#pragma unroll
      for (int nt = 0; nt < C::NT; ++nt)
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[mt][nt][q] = 0.0;
    uint32_t pending = 0;    // levels with a pending left operand
    bool top_dirty = false;  // top[] not yet written to stk[ctz(pending)]

    for (int64_t step = 0; step < nsteps; ++step) {
      cp_wait<DMMA_STAGES - 2>();
      __syncthreads();
      if (step + DMMA_STAGES - 1 < nsteps) issue(step + DMMA_STAGES - 1);
      cp_commit();
      const double *stg = dsm + (int)(step % DMMA_STAGES) * C::STAGE_ELEMS;
      const double *Ab = stg + a_row0;
#pragma unroll
      for (int kq = 0; kq < 2; ++kq) {
        // fragments of four k4 steps; every accumulator sees its inner index
        // in ascending order (k4 steps in order, each DMMA ascending inside)
        double af[C::MT][2][4], bf[C::NT][4];
#pragma unroll
        for (int mt = 0; mt < C::MT; ++mt)
#pragma unroll
          for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int s4 = 0; s4 < 4; ++s4)
              af[mt][h][s4] = Ab[(mt * 16 + 8 * h) * C::SA + a_col[kq][s4]];
#pragma unroll
        for (int nt = 0; nt < C::NT; ++nt)
#pragma unroll
          for (int s4 = 0; s4 < 4; ++s4)
            bf[nt][s4] = stg[(16 * kq + 4 * s4) * C::SB + b_col[nt]];
#pragma unroll
        for (int s4 = 0; s4 < 4; ++s4)
#pragma unroll
          for (int mt = 0; mt < C::MT; ++mt)
#pragma unroll
            for (int h = 0; h < 2; ++h)
#pragma unroll
              for (int nt = 0; nt < C::NT; ++nt)
                dmma884(acc[mt][nt][2 * h], acc[mt][nt][2 * h + 1], af[mt][h][s4], bf[nt][s4]);
      }
      if ((int)(step & (kchunks - 1)) == kchunks - 1) {
        // P_k complete: merge in the reference's tree order
        const int64_t s = step >> kshift;
        const uint32_t k = ks[s];
        int h = 31;
        if (s + 1 < nk) h = merge_level(k, ks[s + 1]);
        while (pending && (__ffs(pending) - 1) < h) {
#pragma unroll
          for (int mt = 0; mt < C::MT; ++mt)
#pragma unroll
            for (int nt = 0; nt < C::NT; ++nt)
#pragma unroll
              for (int q = 0; q < 4; ++q) acc[mt][nt][q] = __dadd_rn(top[mt][nt][q], acc[mt][nt][q]);
          pending &= pending - 1;
          if (pending) {  // the new top sits at stack position popcount - 1
            reload(__popc(pending) - 1);
            top_dirty = false;
          }
        }
        if (s + 1 < nk) {
          if (pending && top_dirty) spill(__popc(pending) - 1);
#pragma unroll
          for (int mt = 0; mt < C::MT; ++mt)
#pragma unroll
            for (int nt = 0; nt < C::NT; ++nt)
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                top[mt][nt][q] = acc[mt][nt][q];
                acc[mt][nt][q] = 0.0;
              }
          top_dirty = true;
          pending |= 1u << h;
        }
      }
    }
    cp_wait<0>();
    // epilogue: C block rows/cols of this sub-tile
    double *crow = Cm + (int64_t(w.i) * b + w.si * TILE + wm * C::WTM + g) * N +
                   int64_t(w.j) * b + w.sj * TILE + wn * C::WTN + 2 * t;
#pragma unroll
    for (int mt = 0; mt < C::MT; ++mt)
#pragma unroll
      for (int nt = 0; nt < C::NT; ++nt)
#pragma unroll
        for (int h2 = 0; h2 < 2; ++h2)
          *reinterpret_cast<double2 *>(crow + (int64_t)(mt * 16 + 8 * h2) * N + nt * 8) =
              make_double2(acc[mt][nt][2 * h2], acc[mt][nt][2 * h2 + 1]);
    __syncthreads();
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(s_tmem),
                 "n"(C::TM_COLS));
  if (args.timeline && threadIdx.x == 0) {
    args.timeline[3 * blockIdx.x] = t_start;
    args.timeline[3 * blockIdx.x + 1] = gtimer();
    args.timeline[3 * blockIdx.x + 2] = items;
  }
}

template <int TILE, int WM, int WN>
static int launch_dmma(const LeafArgs &args, int num_sms, cudaStream_t st) {
  using C = DmmaCfg<TILE, WM, WN>;
  auto kern = leaf_dmma_kernel<TILE, WM, WN>;
  SPAMM_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)C::SMEM));
  int per_sm = 0;
  SPAMM_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, C::THREADS, C::SMEM));
  if (getenv("SPAMM_GEMM_TIMELINE")) {
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, kern);
    fprintf(stderr, "[gemm launch] per_sm=%d regs=%d static_smem=%zu dyn=%zu maxthreads=%d\n", per_sm,
            fa.numRegs, fa.sharedSizeBytes, C::SMEM, fa.maxThreadsPerBlock);
  }
  // The occupancy query reports 1 CTA/SM for kernels that allocate TMEM; two
  // fit (registers, shared memory and 2 x TM_COLS <= 512 TMEM columns), and
  // the persistent ticket loop is correct for any grid size.
  kern<<<num_sms * (per_sm > 2 ? per_sm : 2), C::THREADS, C::SMEM, st>>>(args);
  return SPAMM_OK;
}

// ---------------------------------------------------------------- SIMT path
// Any leaf size and FP32 (and FP64 leaves < 32): one thread per C element of
// a <= 64 x 64 sub-tile, each product an FMA chain over the inner index in
// ascending order (np.matmul's order on this data), merged with the same
// LCA-keyed stack.
constexpr int SIMT_THREADS = 512;
constexpr int SIMT_MAXE = 8;

template <typename T>
__global__ void __launch_bounds__(SIMT_THREADS) leaf_simt_kernel(LeafArgs args) {
  __shared__ int s_work;
  const int b = args.leaf;
  const int TILE = b < 64 ? b : 64;
  const int subs_side = b / TILE;
  const int64_t N = args.N;
  const T *__restrict__ A = (const T *)args.a;
  const T *__restrict__ B = (const T *)args.b;
  T *__restrict__ Cm = (T *)args.c;
  const int elems = TILE * TILE;
  T stk[SIMT_MAXE][MAXD];
  int ops[MAXD];
  WorkItem w;
  while (fetch_work(args, subs_side, &s_work, w)) {
    const int64_t nk = w.end - w.start;
    T acc[SIMT_MAXE];
#pragma unroll
    for (int e = 0; e < SIMT_MAXE; ++e) acc[e] = T(0);
    int sp = 0;
    for (int64_t s = 0; s < nk; ++s) {
      const uint32_t k = args.ks[w.start + s];
#pragma unroll
      for (int e = 0; e < SIMT_MAXE; ++e) {
        const int idx = threadIdx.x + e * SIMT_THREADS;
        if (idx < elems) {
          const int r = idx / TILE, c = idx - r * TILE;
          const T *arow = A + (int64_t(w.i) * b + w.si * TILE + r) * N + int64_t(k) * b;
          const T *bcol = B + (int64_t(k) * b) * N + int64_t(w.j) * b + w.sj * TILE + c;
          T p = T(0);
          for (int q = 0; q < b; ++q) p = fma(arow[q], bcol[int64_t(q) * N], p);
          acc[e] = p;
        }
      }
      int h = 99;
      if (s + 1 < nk) h = merge_level(k, args.ks[w.start + s + 1]);
      while (sp > 0 && ops[sp - 1] < h) {
        --sp;
#pragma unroll
        for (int e = 0; e < SIMT_MAXE; ++e) acc[e] = stk[e][sp] + acc[e];
      }
      if (s + 1 < nk) {
#pragma unroll
        for (int e = 0; e < SIMT_MAXE; ++e) stk[e][sp] = acc[e];
        ops[sp] = h;
        ++sp;
      }
    }
#pragma unroll
    for (int e = 0; e < SIMT_MAXE; ++e) {
      const int idx = threadIdx.x + e * SIMT_THREADS;
      if (idx < elems) {
        const int r = idx / TILE, c = idx - r * TILE;
        Cm[(int64_t(w.i) * b + w.si * TILE + r) * N + int64_t(w.j) * b + w.sj * TILE + c] = acc[e];
      }
    }
    __syncthreads();
  }
}

int launch_leaf(const LeafArgs &args, int dtype, int num_sms, cudaStream_t st, int *launches) {
  if (dtype == SPAMM_DTYPE_F64 && args.leaf >= 32) {
    if (args.leaf == 32) SPAMM_TRY((launch_dmma<32, 2, 2>(args, num_sms, st)));
    else SPAMM_TRY((launch_dmma<64, 2, 4>(args, num_sms, st)));
  } else if (dtype == SPAMM_DTYPE_F64) {
    leaf_simt_kernel<double><<<num_sms * 2, SIMT_THREADS, 0, st>>>(args);
  } else {
    leaf_simt_kernel<float><<<num_sms * 2, SIMT_THREADS, 0, st>>>(args);
  }
  SPAMM_CUDA_TRY(cudaGetLastError());
  if (launches) ++*launches;
  return SPAMM_OK;
}

}  // namespace spamm
