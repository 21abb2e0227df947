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
// 6-stage TMA ring (mbarrier completion; swizzled A boxes, a 5-D B box laid
// out for conflict-free fragment loads) filled by a producer warp; CTAs are
// persistent and take work items from a ticket.
#include <cstdio>
#include <cstdlib>

#include <cuda.h>
#include <cudaTypedefs.h>

#include "leaf.cuh"

namespace spamm {

constexpr int MAXD = 22;  // deepest merge stack (depth <= 21: 21-bit packed coordinates)

__device__ __forceinline__ void cp_async16_l(void *smem, const void *gmem) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// One DMMA.8x8x4: C(8x8) += A(8x4) B(4x8), f64, inner index ascending.  Not
// volatile, so the scheduler may interleave independent accumulators.
__device__ __forceinline__ void dmma884(double &c0, double &c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

// One DMMA.16x8x16: C(16x8) += A(16x16) B(16x8), f64, the inner index
// ascending -- bit-identical to four chained m8n8k4 steps on both row halves
// (tools/dmma_order.cu), with an eighth of the instructions.
// Fragments: a_i = A(g + 8 (i & 1), t + 4 (i >> 1)); b_i = B(t + 4 i, g);
// c_i = C(g + 8 (i >> 1), 2 t + (i & 1)).
__device__ __forceinline__ void dmma16816(double &c0, double &c1, double &c2, double &c3,
                                          const double (&a)[8], const double (&b)[4]) {
  asm("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, "
      "{%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
      : "+d"(c0), "+d"(c1), "+d"(c2), "+d"(c3)
      : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
        "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
}

// m16n8k16 is bit-identical and verified by the parity tests, but measured
// ~3% slower in K3 than four m8n8k4 steps (its longer dependent chain per
// accumulator); kept selectable.
constexpr bool kUseM16N8K16 = false;

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
  const int ng = args.tc->overflow ? 0 : (int)args.tc->num_groups;  // overflow: result discarded, re-run
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



// ---------------------------------------------------------------- DMMA path
constexpr int DMMA_BK = 32;

// Shared-memory tiles are dense (rows of 256 B for A, TILE*8 B for B) with the
// 16-byte chunks of each 128-byte segment XOR-swizzled by (row & 3) << 1.
// That makes the DMMA fragment loads (4 rows x 2 chunks per half-warp) hit
// 32 distinct banks, and keeps every 128-byte global line landing in one
// 128-byte shared segment for the cp.async copies.
__device__ __forceinline__ int swz(int row, int col) {  // element offset within a row
  const int chunk = col >> 1;
  return (((chunk & ~7) | ((chunk & 7) ^ ((row & 3) << 1))) << 1) | (col & 1);
}

__device__ __forceinline__ void mbar_init_l(uint64_t *bar, unsigned count) {
  asm volatile("mbarrier.init.shared.b64 [%0], %1;\n" ::"r"((unsigned)__cvta_generic_to_shared(bar)),
               "r"(count));
}
__device__ __forceinline__ void mbar_arrive_l(uint64_t *bar) {
  asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.shared.b64 st, [%0];\n}\n" ::"r"(
                   (unsigned)__cvta_generic_to_shared(bar))
               : "memory");
}
__device__ __forceinline__ void cp_async_mbar_arrive_l(uint64_t *bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared.b64 [%0];\n" ::"r"(
                   (unsigned)__cvta_generic_to_shared(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait_l(uint64_t *bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"((unsigned)__cvta_generic_to_shared(bar)),
      "r"(parity)
      : "memory");
}

// try_wait with a suspend-time hint: the waiting thread is parked until the
// phase completes (or the hint elapses) instead of re-issuing the test --
// a spinning producer lane otherwise takes issue slots from the consumer
// warps on its SM sub-partition.
__device__ __forceinline__ void mbar_wait_sleep(uint64_t *bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"((unsigned)__cvta_generic_to_shared(bar)),
      "r"(parity), "r"(0x100000u)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx_l(uint64_t *bar, unsigned bytes) {
  asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.expect_tx.shared.b64 st, [%0], %1;\n}\n" ::"r"(
                   (unsigned)__cvta_generic_to_shared(bar)),
               "r"(bytes)
               : "memory");
}
// TMA: one 3-D box of the padded operand -> shared memory (128-byte swizzle),
// completion counted in bytes on `bar`.
__device__ __forceinline__ void tma_load_3d(void *smem, const CUtensorMap *map, int x, int y, int z,
                                            uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
      "%3, %4}], [%5];\n" ::"r"((unsigned)__cvta_generic_to_shared(smem)),
      "l"((uint64_t)map), "r"(x), "r"(y), "r"(z), "r"((unsigned)__cvta_generic_to_shared(bar))
      : "memory");
}

__device__ __forceinline__ void tma_load_5d(void *smem, const CUtensorMap *map, int x0, int x1, int x2,
                                            int x3, int x4, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
      "%3, %4, %5, %6}], [%7];\n" ::"r"((unsigned)__cvta_generic_to_shared(smem)),
      "l"((uint64_t)map), "r"(x0), "r"(x1), "r"(x2), "r"(x3), "r"(x4),
      "r"((unsigned)__cvta_generic_to_shared(bar))
      : "memory");
}

// Tiles land in shared memory as TMA boxes of 128-byte lines with the
// hardware 128-byte swizzle (16-byte chunk ^= line & 7).  A (TILE x 32) is
// loaded as the box {16, 2, TILE}: line = 2*row + col/16, so the four rows a
// half-warp's fragment load touches fall on XOR keys 2*(row & 3) + c -- 32
// distinct banks.  B (32 x TILE) is the box {16, TILE/16, 32}: line =
// (TILE/16)*k + n/16 (conflict-free for TILE = 32; 2-way for TILE = 64).
__device__ __forceinline__ int a_off_tma(int r, int c) {  // elements
  const int L = 2 * r + (c >> 4), ch = (c & 15) >> 1;
  return L * 16 + ((ch ^ (L & 7)) << 1) + (c & 1);
}
template <int TILE>
__device__ __forceinline__ int b_off_tma(int k, int n) {
  const int L = (TILE / 16) * k + (n >> 4), ch = (n & 15) >> 1;
  return L * 16 + ((ch ^ (L & 7)) << 1) + (n & 1);
}
// B for TILE = 64 as the 5-D box {16 n, 2 (n/16 & 1), 4 (k & 3), 2 (n/32), 8 (k/4)}:
// line = (n/16 & 1) + 2 (k & 3) + 8 (n/32) + 16 (k/4), so the XOR key of the
// four k rows of a half-warp is c + 2t -- conflict-free like A.
__device__ __forceinline__ int b_off_tma5(int k, int n) {
  const int L = ((n >> 4) & 1) + 2 * (k & 3) + 8 * (n >> 5) + 16 * (k >> 2), ch = (n & 15) >> 1;
  return L * 16 + ((ch ^ (L & 7)) << 1) + (n & 1);
}

// Per-stage metadata written by the producer: what the consumers do after
// the stage's DMMAs (the merge level of the product that just completed and
// whether the work item -- one C (sub-)tile -- ends here).
struct StageInfo {
  int flags;       // STG_MERGE | STG_END | STG_DONE
  int h;           // merge level with the next k (31 at the item's end)
  int64_t c_off;   // element offset of the C (sub-)tile's origin
  int grp;         // group (C block) of the item
  int pad;
};
constexpr int STG_MERGE = 1, STG_END = 2, STG_DONE = 4;

// Warp-specialised persistent leaf-product kernel.
//   warp 0      producer: takes work items from the ticket, and for every
//               32-wide k slice of every retained product streams the A and B
//               tiles into a STAGES-deep ring with cp.async (completion on the
//               stage's "full" mbarrier), plus the StageInfo.  It runs ahead
//               across item boundaries, so item starts cost no pipeline bubble.
//   warps 1-16  consumers: a 4 x 4 grid of warp tiles over the C tile; each
//               waits "full", runs its DMMAs, releases the stage ("empty"),
//               then merges / stores as StageInfo says.  No block-wide
//               barrier in the loop.
template <int TILE, int CW_ = 16, int WM_ = 4, int ST_ = 0>
struct WsCfg {
  static constexpr int CWARPS = CW_, WM = WM_, WN = CW_ / WM_;
  static constexpr int THREADS = 32 * (1 + CWARPS);
  static constexpr int WTM = TILE / WM, WTN = TILE / WN;  // warp tile
  static constexpr int MT8 = WTM / 8, NT8 = WTN / 8;      // m8 / n8 tiles per warp
  static constexpr int NACC = MT8 * NT8 * 2;              // accumulator doubles per thread
  static constexpr int NREG = 2 * NACC;                   // ... as b32 registers
  static constexpr int A_ELEMS = TILE * DMMA_BK, B_ELEMS = DMMA_BK * TILE;
  static constexpr int STAGE_ELEMS = A_ELEMS + B_ELEMS;
  static constexpr int STAGES = ST_ ? ST_ : TILE == 64 ? 6 : 10;
  static constexpr size_t SMEM = sizeof(double) * STAGES * STAGE_ELEMS;
  static constexpr int SLOT_COLS = NREG * (CWARPS / 4);   // TMEM columns per stack slot
  static constexpr int TM_COLS = 512;
  static constexpr int TM_SLOTS = TM_COLS / SLOT_COLS;
  static constexpr int QA = TILE * DMMA_BK / 2 / 32;      // 16-B copies per producer lane
  static constexpr int QB = DMMA_BK * TILE / 2 / 32;
};

template <int NREG>
__device__ __forceinline__ void tmem_store(uint32_t taddr, const uint32_t (&r)[NREG]);
template <int NREG>
__device__ __forceinline__ void tmem_load(uint32_t taddr, uint32_t (&r)[NREG]);
#define R4(o) "r"(r[o]), "r"(r[o + 1]), "r"(r[o + 2]), "r"(r[o + 3])
#define W4(o) "=r"(r[o]), "=r"(r[o + 1]), "=r"(r[o + 2]), "=r"(r[o + 3])
template <>
__device__ __forceinline__ void tmem_store<16>(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15,%16};\n" ::"r"(taddr),
      R4(0), R4(4), R4(8), R4(12)
      : "memory");
}
template <>
__device__ __forceinline__ void tmem_load<16>(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15}, [%16];\n"
      : W4(0), W4(4), W4(8), W4(12)
      : "r"(taddr)
      : "memory");
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
}
template <>
__device__ __forceinline__ void tmem_store<4>(uint32_t taddr, const uint32_t (&r)[4]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};\n" ::"r"(taddr), R4(0)
               : "memory");
}
template <>
__device__ __forceinline__ void tmem_load<4>(uint32_t taddr, uint32_t (&r)[4]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];\n"
               : W4(0)
               : "r"(taddr)
               : "memory");
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
}
template <>
__device__ __forceinline__ void tmem_store<32>(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};\n" ::"r"(taddr),
      R4(0), R4(4), R4(8), R4(12), R4(16), R4(20), R4(24), R4(28)
      : "memory");
}
template <>
__device__ __forceinline__ void tmem_load<32>(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
      : W4(0), W4(4), W4(8), W4(12), W4(16), W4(20), W4(24), W4(28)
      : "r"(taddr)
      : "memory");
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
}
template <>
__device__ __forceinline__ void tmem_store<64>(uint32_t taddr, const uint32_t (&r)[64]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x64.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,%47,%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63,%64};\n" ::"r"(taddr),
      R4(0), R4(4), R4(8), R4(12), R4(16), R4(20), R4(24), R4(28), R4(32), R4(36), R4(40), R4(44), R4(48), R4(52), R4(56), R4(60)
      : "memory");
}
template <>
__device__ __forceinline__ void tmem_load<64>(uint32_t taddr, uint32_t (&r)[64]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x64.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,%47,%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%64];\n"
      : W4(0), W4(4), W4(8), W4(12), W4(16), W4(20), W4(24), W4(28), W4(32), W4(36), W4(40), W4(44), W4(48), W4(52), W4(56), W4(60)
      : "r"(taddr)
      : "memory");
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
}
#undef R4
#undef W4

// Bitmask groups: the inner indices k of C block (i, j)'s retained triples
// as a bit set, read from the dense traversal's retained leaf-triple bitmask
// (bit x = Morton code spread3(i) << 2 | spread3(j) << 1 | spread3(k)).  Four
// k per 32-bit word (k's two low bits sit at x bits 0 and 3); nb <= 64.
__device__ __noinline__ uint64_t retained_kmask(const uint32_t *__restrict__ am, uint32_t i,
                                                   uint32_t j, int nb) {
  const uint32_t base = (spread3(i) << 2) | (spread3(j) << 1);
  uint64_t m = 0;
  if (nb >= 4) {
#pragma unroll 4
    for (int q = 0; q < 16; ++q) {
      const uint32_t x0 = base | spread3((uint32_t)(4 * q));
      const uint32_t w = 4 * q < nb ? __ldcg(am + (x0 >> 5)) >> (x0 & 31) : 0u;
      m |= ((uint64_t)(w & 3u) | ((uint64_t)((w >> 8) & 3u) << 2)) << (4 * q);
    }
  } else {
    for (int k = 0; k < nb; ++k) {
      const uint32_t x = base | spread3((uint32_t)k);
      m |= (uint64_t)((__ldcg(am + (x >> 5)) >> (x & 31)) & 1u) << k;
    }
  }
  return m;
}

template <int TILE, int CW = 16, int WMv = 4, int ST = 0>
__global__ void __launch_bounds__(WsCfg<TILE, CW, WMv, ST>::THREADS, 1)
    leaf_dmma_ws_kernel(LeafArgs args, const __grid_constant__ CUtensorMap tmA,
                        const __grid_constant__ CUtensorMap tmB) {
  using C = WsCfg<TILE, CW, WMv, ST>;
  extern __shared__ __align__(1024) unsigned char dsm_raw[];
  // TMA 128-byte swizzle needs 1024-byte aligned tiles (offset arithmetic on
  // the shared array: an integer round-trip of the pointer would lose its
  // address space and turn every fragment load into a generic LD)
  double *dsm = reinterpret_cast<double *>(
      dsm_raw + ((1024u - ((unsigned)__cvta_generic_to_shared(dsm_raw) & 1023u)) & 1023u));
  __shared__ __align__(8) uint64_t full_bar[C::STAGES], empty_bar[C::STAGES];
  __shared__ StageInfo info[C::STAGES];
  __shared__ uint32_t s_tmem;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int b = args.leaf;
  const int kchunks = b / DMMA_BK;
  const int subs_side = b / TILE;
  const int64_t N = args.N;
  const unsigned long long t_start = gtimer();

  if (tid == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init_l(&full_bar[s], 1);        // the producer's arrive (+ TMA transaction bytes)
      mbar_init_l(&empty_bar[s], C::CWARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                     (unsigned)__cvta_generic_to_shared(&s_tmem)),
                 "n"(C::TM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");

  unsigned items = 0, stages_total = 0;
  if (warp == 0) {
    // ============================================================ producer
    if (args.am && lane != 0) asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];\n" ::"l"((uint64_t)&tmA) : "memory");
      asm volatile("prefetch.tensormap [%0];\n" ::"l"((uint64_t)&tmB) : "memory");
      // launched as a programmatic dependent of the traversal: its outputs
      // (group lists, counts) are complete and visible after this (a no-op
      // for a plain launch).  Bitmask groups: the traversal publishes the
      // group list before its record / budget CTAs finish; start on that.
      if (args.am) {
        const unsigned *rdy = &args.tc->groups_ready;
        for (;;) {
          unsigned v;
          asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(v) : "l"(rdy) : "memory");
          if (v) break;
          __nanosleep(32);
        }
      } else {
        asm volatile("griddepcontrol.wait;\n" ::: "memory");
      }
      // the traversal is complete: a programmatic dependent (C's norm kernel,
      // which waits on args.grp_done) may start now and overlap this kernel.
      // Not earlier: it reads the traversal's group list and count.
      asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
      // K3's span starts when its inputs are ready (its prologue may have
      // overlapped the traversal's tail)
      atomicMax(&args.tc->k3_t0n, ~gtimer());
      unsigned long long m = *args.n_codes;
      if (m > args.capacity) m = args.capacity;
      // overflow: result discarded, re-run (bitmask groups never overflow:
      // the group list holds every C block; a pruned-record overflow set
      // later by the traversal does not concern the products)
      const int ng = args.am ? (int)args.tc->num_groups
                             : args.tc->overflow ? 0 : (int)args.tc->num_groups;
      const int subs = subs_side * subs_side;
      int stage = 0;
      unsigned phase = 0;
      long long gstep = 0;  // ring position
      auto acquire = [&]() {  // wait until the stage is free again
        if (gstep >= C::STAGES) mbar_wait_l(&empty_bar[stage], phase ^ 1);
      };
      auto advance = [&]() {
        ++gstep;
        if (++stage == C::STAGES) {
          stage = 0;
          phase ^= 1;
        }
      };
      for (;;) {
        // Final wave (the last drain_items tickets): take an item only once
        // the consumers have taken every stage already issued, so the last
        // items go to the CTAs that are actually free instead of those whose
        // producer runs a ring ahead of its consumers (end spread)
        if (args.drain_items && gstep > 0) {
          unsigned long long taken;
          asm volatile("ld.relaxed.gpu.u64 %0, [%1];" : "=l"(taken) : "l"(&args.tc->gemm_ticket) : "memory");
          if (taken + (unsigned long long)args.drain_items >= (unsigned long long)(ng * subs)) {
            const long long last = gstep - 1;
            mbar_wait_l(&empty_bar[last % C::STAGES], (unsigned)((last / C::STAGES) & 1));
          }
        }
        const int item = (int)atomicAdd(&args.tc->gemm_ticket, 1ull);
        if (item >= ng * subs) break;
        ++items;
        const int gi = item / subs, sub = item - gi * subs;
        const int grp = args.order ? (int)args.order[gi] : gi;
        const int si = sub / subs_side, sj = sub - si * subs_side;
        const uint32_t gid = args.group_ids[grp];
        const int64_t ci = gid / (uint64_t)args.nb, cj = gid - ci * args.nb;
        const int arow0 = (int)(ci * b + si * TILE), bcol16 = (int)((cj * b + sj * TILE) >> 4);
        const int64_t c_off = (int64_t)arow0 * N + cj * b + sj * TILE;
        // the group's inner indices, ascending: ks[start, end) or the set
        // bits of kmask (bitmask groups)
        int64_t s = 0, end = 0;
        uint64_t kmask = 0;
        uint32_t k;
        if (args.am) {
          kmask = retained_kmask(args.am, (uint32_t)ci, (uint32_t)cj, (int)args.nb);
          k = (uint32_t)(__ffsll((long long)kmask) - 1);
          kmask &= kmask - 1;
        } else {
          s = args.group_starts[grp];
          end = grp + 1 < ng ? args.group_starts[grp + 1] : (int64_t)m;
          k = args.ks[s];
        }
        for (;;) {
          const bool has_next = args.am ? kmask != 0 : s + 1 < end;
          const uint32_t knext = !has_next ? 0u
                                 : args.am ? (uint32_t)(__ffsll((long long)kmask) - 1) : args.ks[s + 1];
          for (int kc = 0; kc < kchunks; ++kc) {
            acquire();
            double *stg = dsm + stage * C::STAGE_ELEMS;
            const int kcol = (int)(k * b + kc * DMMA_BK);
            int flags = 0, h = 31;
            if (kc == kchunks - 1) {
              flags = STG_MERGE;
              if (has_next) h = merge_level(k, knext);
              else flags |= STG_END;
            }
            info[stage].flags = flags;
            info[stage].h = h;
            info[stage].c_off = c_off;
            info[stage].grp = grp;
            mbar_arrive_expect_tx_l(&full_bar[stage], (unsigned)(C::STAGE_ELEMS * sizeof(double)));
            tma_load_3d(stg, &tmA, 0, kcol >> 4, arow0, &full_bar[stage]);
            if (TILE == 64 && args.b_map5)
              tma_load_5d(stg + C::A_ELEMS, &tmB, 0, 0, 0, bcol16 >> 1, kcol >> 2, &full_bar[stage]);
            else
              tma_load_3d(stg + C::A_ELEMS, &tmB, 0, bcol16, kcol, &full_bar[stage]);
            advance();
          }
          if (!has_next) break;
          k = knext;
          if (args.am) kmask &= kmask - 1;
          else ++s;
        }
      }
      stages_total = (unsigned)gstep;
      // termination marker
      acquire();
      info[stage].flags = STG_DONE;
      info[stage].h = 31;
      info[stage].c_off = 0;
      mbar_arrive_l(&full_bar[stage]);
    }
    __syncwarp();
  } else {
    // ============================================================ consumers
    // bitmask groups: C's norm kernel waits for the group list itself, so it
    // may launch (and take its slot beside this CTA) right away; the launch
    // of dependents counts once every thread of every CTA has signalled
    if (args.am) asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
    const int cw = warp - 1;
    const int wm = cw / C::WN, wn = cw % C::WN, g = lane >> 2, t = lane & 3;
    double *__restrict__ Cm = (double *)args.c;
    // loop-invariant fragment offsets (elements) in the swizzled stage
    int a_o[2][4], b_o[2][4][C::NT8];
#pragma unroll
    for (int kq = 0; kq < 2; ++kq)
#pragma unroll
      for (int s4 = 0; s4 < 4; ++s4) {
        a_o[kq][s4] = a_off_tma(wm * C::WTM + g, 16 * kq + 4 * s4 + t);
#pragma unroll
        for (int nt = 0; nt < C::NT8; ++nt)
          b_o[kq][s4][nt] = C::A_ELEMS + (TILE == 64 && args.b_map5
                                              ? b_off_tma5(16 * kq + 4 * s4 + t, wn * C::WTN + nt * 8 + g)
                                              : b_off_tma<TILE>(16 * kq + 4 * s4 + t, wn * C::WTN + nt * 8 + g));
      }
    const uint32_t t_my = s_tmem + ((uint32_t)(32 * (warp & 3)) << 16) +
                          (uint32_t)(((cw >> 2) & 3) * C::NREG);
    double stk[MAXD][C::NACC];  // only slots >= TM_SLOTS (deep stacks)
    double acc[C::NACC], top[C::NACC];
#pragma unroll
    for (int x = 0; x < C::NACC; ++x) acc[x] = 0.0;
    uint32_t pending = 0;
    bool top_dirty = false;
    const int tm_slots = args.tm_slots < C::TM_SLOTS ? args.tm_slots : C::TM_SLOTS;
    auto spill = [&](int slot) {
      if (slot < tm_slots) {
        uint32_t r[C::NREG];
#pragma unroll
        for (int x = 0; x < C::NACC; ++x) {
          r[2 * x] = (uint32_t)__double2loint(top[x]);
          r[2 * x + 1] = (uint32_t)__double2hiint(top[x]);
        }
        tmem_store<C::NREG>(t_my + slot * C::SLOT_COLS, r);
        if (args.tm_sync) asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
      } else {
#pragma unroll
        for (int x = 0; x < C::NACC; ++x) stk[slot][x] = top[x];
      }
    };
    auto reload = [&](int slot) {
      if (slot < tm_slots) {
        uint32_t r[C::NREG];
        asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
        tmem_load<C::NREG>(t_my + slot * C::SLOT_COLS, r);
#pragma unroll
        for (int x = 0; x < C::NACC; ++x) top[x] = __hiloint2double((int)r[2 * x + 1], (int)r[2 * x]);
      } else {
#pragma unroll
        for (int x = 0; x < C::NACC; ++x) top[x] = stk[slot][x];
      }
    };
    int stage = 0;
    unsigned phase = 0;
    for (;;) {
      mbar_wait_l(&full_bar[stage], phase);
      const StageInfo si = info[stage];
      if (si.flags & STG_DONE) break;
      const double *stg = dsm + stage * C::STAGE_ELEMS;
#pragma unroll
      for (int kq = 0; kq < 2; ++kq) {
        double af[C::MT8][4], bf[C::NT8][4];
#pragma unroll
        for (int mt = 0; mt < C::MT8; ++mt)
#pragma unroll
          for (int s4 = 0; s4 < 4; ++s4) af[mt][s4] = stg[mt * 8 * DMMA_BK + a_o[kq][s4]];
#pragma unroll
        for (int nt = 0; nt < C::NT8; ++nt)
#pragma unroll
          for (int s4 = 0; s4 < 4; ++s4) bf[nt][s4] = stg[b_o[kq][s4][nt]];
        if constexpr (C::MT8 == 2 && kUseM16N8K16) {
          // 16-row warp tile: one m16n8k16 per n8 tile covers the four k4 steps
          // of both m8 halves (same fragments, same registers, same order)
          const double a16[8] = {af[0][0], af[1][0], af[0][1], af[1][1],
                                 af[0][2], af[1][2], af[0][3], af[1][3]};
#pragma unroll
          for (int nt = 0; nt < C::NT8; ++nt)
            dmma16816(acc[nt * 2], acc[nt * 2 + 1], acc[(C::NT8 + nt) * 2],
                      acc[(C::NT8 + nt) * 2 + 1], a16, bf[nt]);
        } else {
#pragma unroll
          for (int s4 = 0; s4 < 4; ++s4)
#pragma unroll
            for (int mt = 0; mt < C::MT8; ++mt)
#pragma unroll
              for (int nt = 0; nt < C::NT8; ++nt)
                dmma884(acc[(mt * C::NT8 + nt) * 2], acc[(mt * C::NT8 + nt) * 2 + 1], af[mt][s4],
                        bf[nt][s4]);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive_l(&empty_bar[stage]);
      if (++stage == C::STAGES) {
        stage = 0;
        phase ^= 1;
      }
      if (si.flags & STG_MERGE) {
        // P_k complete: merge in the reference's tree order
        const int h = si.h;
        while (pending && (__ffs(pending) - 1) < h) {
#pragma unroll
          for (int x = 0; x < C::NACC; ++x) acc[x] = __dadd_rn(top[x], acc[x]);
          pending &= pending - 1;
          if (pending) {  // the new top sits at stack position popcount - 1
            reload(__popc(pending) - 1);
            top_dirty = false;
          }
        }
        if (!(si.flags & STG_END)) {
          if (pending && top_dirty) spill(__popc(pending) - 1);
#pragma unroll
          for (int x = 0; x < C::NACC; ++x) {
            top[x] = acc[x];
            acc[x] = 0.0;
          }
          top_dirty = true;
          pending |= 1u << h;
        } else {
          // item complete: the C tile of this warp
          double *crow = Cm + si.c_off + (int64_t)(wm * C::WTM + g) * N + wn * C::WTN + 2 * t;
#pragma unroll
          for (int mt = 0; mt < C::MT8; ++mt)
#pragma unroll
            for (int nt = 0; nt < C::NT8; ++nt) {
              const int x = (mt * C::NT8 + nt) * 2;
              *reinterpret_cast<double2 *>(crow + (int64_t)(mt * 8) * N + nt * 8) =
                  make_double2(acc[x], acc[x + 1]);
            }
#pragma unroll
          for (int x = 0; x < C::NACC; ++x) acc[x] = 0.0;
          pending = 0;
          top_dirty = false;
          if (args.grp_done) {  // this warp's part of the group is in C
            __syncwarp();
            if (lane == 0)  // release reduction: no full fence stalling the warp
              asm volatile("red.release.gpu.global.add.u32 [%0], 1;\n" ::"l"(&args.grp_done[si.grp])
                           : "memory");
          }
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(s_tmem),
                 "n"(C::TM_COLS));
  if (tid == 0) atomicMax(&args.tc->k3_t1, gtimer());
  if (args.timeline && tid == 0) {
    args.timeline[3 * blockIdx.x] = t_start;
    args.timeline[3 * blockIdx.x + 1] = gtimer();
    args.timeline[3 * blockIdx.x + 2] = items | ((unsigned long long)stages_total << 16);
  }
}

static PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
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

// 3-D view {16, N/16, N} of a padded N x N f64 operand: box {16, box1, box2}.
static int make_operand_map(CUtensorMap *map, const void *base, int64_t N, int box1, int box2) {
  auto enc = tensor_map_encoder();
  if (!enc) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return SPAMM_ERR_CUDA;
  }
  cuuint64_t dims[3] = {16, (cuuint64_t)(N / 16), (cuuint64_t)N};
  cuuint64_t strides[2] = {128, (cuuint64_t)(N * 8)};
  cuuint32_t box[3] = {16, (cuuint32_t)box1, (cuuint32_t)box2};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<void *>(base), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (%d)", (int)r);
    return SPAMM_ERR_CUDA;
  }
  return SPAMM_OK;
}

// 5-D view of B for TILE = 64 (see b_off_tma5); its strides are not
// monotonic, so a driver that rejects the encoding falls back to the 3-D box.
static bool make_b_map5(CUtensorMap *map, const void *base, int64_t N) {
  auto enc = tensor_map_encoder();
  if (!enc || N < 64) return false;
  cuuint64_t dims[5] = {16, 2, 4, (cuuint64_t)(N / 32), (cuuint64_t)(N / 4)};
  cuuint64_t strides[4] = {128, (cuuint64_t)(N * 8), 256, (cuuint64_t)(4 * N * 8)};
  cuuint32_t box[5] = {16, 2, 4, 2, 8};
  cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, const_cast<void *>(base), dims, strides, box,
             estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int TILE, int CW = 16, int WMv = 4, int ST = 0>
static int launch_dmma_ws(LeafArgs args, int num_sms, cudaStream_t st) {
  using C = WsCfg<TILE, CW, WMv, ST>;
  static const int tm_env = getenv("SPAMM_K3_TM_SLOTS") ? atoi(getenv("SPAMM_K3_TM_SLOTS")) : C::TM_SLOTS;
  static const int tm_sync = getenv("SPAMM_K3_TM_SYNC") != nullptr;
  args.tm_slots = tm_env;
  args.tm_sync = tm_sync;
  // final-wave ticket policy (SPAMM_K3_DRAIN = tickets per CTA of the final wave, 0: off)
  static const int drain = getenv("SPAMM_K3_DRAIN") ? atoi(getenv("SPAMM_K3_DRAIN")) : 0;
  args.drain_items = drain * num_sms;
  CUtensorMap ma, mb;
  SPAMM_TRY(make_operand_map(&ma, args.a, args.N, 2, TILE));             // A: 32 k x TILE rows
  args.b_map5 = TILE == 64 && make_b_map5(&mb, args.b, args.N);
  if (!args.b_map5)
    SPAMM_TRY(make_operand_map(&mb, args.b, args.N, TILE / 16, DMMA_BK));  // B: TILE n x 32 k
  auto kern = leaf_dmma_ws_kernel<TILE, CW, WMv, ST>;
  SPAMM_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)(C::SMEM + 1024)));
  SPAMM_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(num_sms);
  cfg.blockDim = dim3(C::THREADS);
  cfg.dynamicSmemBytes = C::SMEM + 1024;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  if (args.pdl) {  // CTAs become resident (prologue done) as the traversal's CTAs retire
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
  }
  SPAMM_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, args, ma, mb));
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

// consumer-warp layout of the FP64 kernel at leaf >= 64 (SPAMM_K3_WARPS):
// 8 = 2 x 4 warp tiles of 32 x 16 (eight independent DMMA chains per warp;
// c5 K3 31.8 vs 29.8 TFLOP/s for 16) on a 6-stage ring, 84 = the same on 4
// stages (default: as fast, and leaves shared memory for C's norm kernel to
// run beside it), 87 = 7 stages, 16 = 4 x 4 of 16 x 16, 9 = 4 x 2 of 16 x 32,
// 4 = 2 x 2 of 32 x 32
int k3_warps() {
  static const int w = getenv("SPAMM_K3_WARPS") ? atoi(getenv("SPAMM_K3_WARPS")) : 84;
  return w;
}
unsigned leaf_signals_per_tile(int leaf) {
  if (leaf < 64) return 16;
  const int w = k3_warps();
  return w == 8 || w == 9 || w == 84 || w == 87 ? 8 : w == 4 ? 4 : 16;
}

// ----------------------------------------------------- FP32 tiled path
// FP32 leaves of 64 (and multiples): np.matmul's order on this data is one
// sequential FMA chain per output over the inner index from zero -- the same
// as the SIMT kernel -- but here a CTA of 256 threads owns a 64 x 64 C tile,
// each thread a 4 x 4 register micro-tile, and the operand tiles are staged in
// shared memory (A transposed, so a thread's four rows at one inner index are
// one 16-byte load), double-buffered through registers: 2 shared loads per
// 16 FMAs instead of 2 global loads per FMA.  Products are merged with the
// same LCA-keyed stack (per element, in f32).
constexpr int SG_APAD = 4;                       // floats of padding per transposed A row
constexpr int SG_A_FLOATS = 64 * (64 + SG_APAD);  // As[q][r]
constexpr int SG_B_FLOATS = 64 * 64;              // Bs[q][c]
constexpr size_t SG_SMEM = sizeof(float) * 2 * (SG_A_FLOATS + SG_B_FLOATS);

// TM x TN outputs per thread (64 / TN threads across, 64 / TM down).
template <int TM, int TN>
__global__ void __launch_bounds__(4096 / (TM * TN), 512 / (4096 / (TM * TN)) < 3 ? 1 : 3) leaf_sgemm_kernel(LeafArgs args) {
  constexpr int THREADS = 4096 / (TM * TN), NX = 64 / TN;
  constexpr int PER = 1024 / THREADS;  // float4 pieces per thread per operand tile
  extern __shared__ __align__(16) float sg_smem[];
  __shared__ int s_work;
  const int tid = threadIdx.x, tx = tid % NX, ty = tid / NX;
  const int b = args.leaf;
  const int subs_side = b / 64, kchunks = b / 64;
  const int64_t N = args.N;
  const float *__restrict__ A = (const float *)args.a;
  const float *__restrict__ B = (const float *)args.b;
  float *__restrict__ Cm = (float *)args.c;
  float stk[MAXD][TM * TN];
  WorkItem w;
  while (fetch_work(args, subs_side, &s_work, w)) {
    const int64_t nk = w.end - w.start;
    const int64_t steps = nk * kchunks;  // (product, inner chunk) pairs, in order
    const int64_t arow0 = (int64_t)w.i * b + w.si * 64, bcol0 = (int64_t)w.j * b + w.sj * 64;
    float4 ra[PER], rb[PER];
    // A piece u of this thread: row r, float4 column c4 -- lanes run down 8
    // rows, then across 4 columns: whole 64-byte row segments from global and
    // transposed shared stores with at most two lanes per bank
    auto a_rc = [&](int u, int &r, int &c4) {
      const int f = tid + THREADS * u, t = f >> 5, l = f & 31;
      r = 8 * (t & 7) + (l & 7);
      c4 = 4 * (4 * (t >> 3) + (l >> 3));
    };
    auto load = [&](int64_t step) {  // global -> registers
      const int64_t s = step / kchunks;
      const int kc = (int)(step - s * kchunks);
      const int64_t kcol = (int64_t)args.ks[w.start + s] * b + kc * 64;
#pragma unroll
      for (int u = 0; u < PER; ++u) {
        int r, c4;
        a_rc(u, r, c4);
        ra[u] = __ldg(reinterpret_cast<const float4 *>(A + (arow0 + r) * N + kcol + c4));
        const int f = tid + THREADS * u, rr = f >> 4, cc4 = (f & 15) * 4;
        rb[u] = __ldg(reinterpret_cast<const float4 *>(B + (kcol + rr) * N + bcol0 + cc4));
      }
    };
    auto store = [&](int buf) {  // registers -> shared (A transposed)
      float *As = sg_smem + buf * (SG_A_FLOATS + SG_B_FLOATS), *Bs = As + SG_A_FLOATS;
#pragma unroll
      for (int u = 0; u < PER; ++u) {
        int r, c4;
        a_rc(u, r, c4);
        As[(c4 + 0) * (64 + SG_APAD) + r] = ra[u].x;
        As[(c4 + 1) * (64 + SG_APAD) + r] = ra[u].y;
        As[(c4 + 2) * (64 + SG_APAD) + r] = ra[u].z;
        As[(c4 + 3) * (64 + SG_APAD) + r] = ra[u].w;
        const int f = tid + THREADS * u, rr = f >> 4, cc4 = (f & 15) * 4;
        *reinterpret_cast<float4 *>(Bs + rr * 64 + cc4) = rb[u];
      }
    };
    float acc[TM * TN];
#pragma unroll
    for (int e = 0; e < TM * TN; ++e) acc[e] = 0.f;
    uint32_t pending = 0;
    load(0);
    store(0);
    __syncthreads();
    for (int64_t step = 0; step < steps; ++step) {
      const int cur = (int)(step & 1);
      if (step + 1 < steps) load(step + 1);
      const float *As = sg_smem + cur * (SG_A_FLOATS + SG_B_FLOATS), *Bs = As + SG_A_FLOATS;
#pragma unroll 16
      for (int q = 0; q < 64; ++q) {
        float av[TM], bw[TN];
#pragma unroll
        for (int i = 0; i < TM; i += 4) {
          const float4 a = *reinterpret_cast<const float4 *>(As + q * (64 + SG_APAD) + ty * TM + i);
          av[i] = a.x;
          av[i + 1] = a.y;
          av[i + 2] = a.z;
          av[i + 3] = a.w;
        }
#pragma unroll
        for (int j = 0; j < TN; j += 4) {
          const float4 bv = *reinterpret_cast<const float4 *>(Bs + q * 64 + tx * TN + j);
          bw[j] = bv.x;
          bw[j + 1] = bv.y;
          bw[j + 2] = bv.z;
          bw[j + 3] = bv.w;
        }
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
          for (int j = 0; j < TN; ++j) acc[i * TN + j] = fmaf(av[i], bw[j], acc[i * TN + j]);
      }
      if (step + 1 < steps) store(cur ^ 1);
      __syncthreads();
      const int64_t s = step / kchunks;
      if (step - s * kchunks == kchunks - 1) {  // product P_k complete: merge in tree order
        // the stack's merge levels as a bit set (they increase downwards, so
        // the top is the lowest set bit and the depth is the popcount): no
        // local-memory level array in the pop loop's condition
        const uint32_t k = args.ks[w.start + s];
        const bool has_next = s + 1 < nk;
        const int h = has_next ? merge_level(k, args.ks[w.start + s + 1]) : 32;
        while (pending && (__ffs(pending) - 1) < h) {
          const int top = __popc(pending) - 1;
#pragma unroll
          for (int e = 0; e < TM * TN; ++e) acc[e] = stk[top][e] + acc[e];
          pending &= pending - 1;
        }
        if (has_next) {
          const int slot = __popc(pending);
#pragma unroll
          for (int e = 0; e < TM * TN; ++e) {
            stk[slot][e] = acc[e];
            acc[e] = 0.f;
          }
          pending |= 1u << h;
        }
      }
    }
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
      for (int j = 0; j < TN; j += 4)
        *reinterpret_cast<float4 *>(Cm + (arow0 + ty * TM + i) * N + bcol0 + tx * TN + j) =
            make_float4(acc[i * TN + j], acc[i * TN + j + 1], acc[i * TN + j + 2],
                        acc[i * TN + j + 3]);
  }
}

// ------------------------------------- FP32 warp-specialised TMA path
// The same per-element FMA chain as leaf_sgemm_kernel, restructured for the
// shared-memory pipe, which bounds the register-staged kernel (ncu: L1 81 %,
// eight wavefronts per inner step per warp, transposing stores 4-way
// conflicted):
//   * a producer warp streams each (product, 64-wide inner chunk) as two TMA
//     boxes into a STAGES-deep ring (mbarrier completion) -- no register
//     staging, no block-wide barrier, item boundaries without a bubble;
//   * A stays row-major: its box is 68 floats wide (the 4 extra columns are
//     never read, OOB columns zero-filled), so rows sit 272 B apart and a
//     thread reads four inner steps of one row as one 16-byte load;
//   * two consumer warps own the 64 x 64 C tile, 8 x 8 outputs per thread
//     (rows 16 u + 4 ty + r', columns 32 v + 4 tx + c'): per four inner steps
//     a thread issues 8 A loads and 8 B loads for 256 FMAs, and every
//     half-warp load touches <= 128 distinct bytes in distinct banks (one
//     wavefront).
// KW = the inner-chunk width of one stage (64 or 32): A box KW + 4 floats
// wide (rows 4 apart 16 banks apart), B box 64 x KW.
template <int KW>
struct SwCfg {
  static constexpr int AW = KW + 4;
  static constexpr int A_BYTES = 64 * AW * 4, B_BYTES = KW * 64 * 4;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;  // a multiple of 128
};
constexpr int SW_CWARPS = 2, SW_THREADS = 32 * (1 + SW_CWARPS);

__device__ __forceinline__ void tma_load_2d(void *smem, const CUtensorMap *map, int x, int y,
                                            uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
      "%3}], [%4];\n" ::"r"((unsigned)__cvta_generic_to_shared(smem)),
      "l"((uint64_t)map), "r"(x), "r"(y), "r"((unsigned)__cvta_generic_to_shared(bar))
      : "memory");
}

// MINB = CTAs per SM the register budget is sized for: 4 (168 registers, no
// spills, room for the scheduler to run the fragment loads ahead) measured
// faster than 5 (128) or 6 (96, spilling) at c5-f32 -- 45.4 vs 39.0 vs 28.2
// TFLOP/s.
template <int STAGES, int KW, int MINB = 4>
__global__ void __launch_bounds__(SW_THREADS, MINB)
    leaf_sgemm_ws_kernel(LeafArgs args, const __grid_constant__ CUtensorMap tmA,
                         const __grid_constant__ CUtensorMap tmB) {
  extern __shared__ __align__(128) unsigned char sw_raw[];
  // (offset arithmetic on the shared array keeps the loads LDS)
  unsigned char *dsm = sw_raw + ((128u - ((unsigned)__cvta_generic_to_shared(sw_raw) & 127u)) & 127u);
  __shared__ __align__(8) uint64_t full_bar[STAGES], empty_bar[STAGES];
  __shared__ StageInfo info[STAGES];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int b = args.leaf;
  using C = SwCfg<KW>;
  const int kchunks = b / KW, subs_side = b / 64;
  const int64_t N = args.N;
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init_l(&full_bar[s], 1);
      mbar_init_l(&empty_bar[s], SW_CWARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
  }
  __syncthreads();
  if (warp == 0) {
    // ============================================================ producer
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];\n" ::"l"((uint64_t)&tmA) : "memory");
      asm volatile("prefetch.tensormap [%0];\n" ::"l"((uint64_t)&tmB) : "memory");
      if (args.am) {
        const unsigned *rdy = &args.tc->groups_ready;
        for (;;) {
          unsigned v;
          asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(v) : "l"(rdy) : "memory");
          if (v) break;
          __nanosleep(32);
        }
      } else {
        asm volatile("griddepcontrol.wait;\n" ::: "memory");
      }
      asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
      atomicMax(&args.tc->k3_t0n, ~gtimer());
      unsigned long long m = *args.n_codes;
      if (m > args.capacity) m = args.capacity;
      const int ng = args.am ? (int)args.tc->num_groups
                             : args.tc->overflow ? 0 : (int)args.tc->num_groups;
      const int subs = subs_side * subs_side;
      int stage = 0;
      unsigned phase = 0;
      long long gstep = 0;
      for (;;) {
        const int item = (int)atomicAdd(&args.tc->gemm_ticket, 1ull);
        if (item >= ng * subs) break;
        const int grp = item / subs, sub = item - grp * subs;
        const int si = sub / subs_side, sj = sub - si * subs_side;
        const uint32_t gid = args.group_ids[grp];
        const int64_t ci = gid / (uint64_t)args.nb, cj = gid - ci * args.nb;
        const int arow0 = (int)(ci * b + si * 64), bcol0 = (int)(cj * b + sj * 64);
        const int64_t c_off = (int64_t)arow0 * N + bcol0;
        int64_t s = 0, end = 0;
        uint64_t kmask = 0;
        uint32_t k;
        if (args.am) {
          kmask = retained_kmask(args.am, (uint32_t)ci, (uint32_t)cj, (int)args.nb);
          k = (uint32_t)(__ffsll((long long)kmask) - 1);
          kmask &= kmask - 1;
        } else {
          s = args.group_starts[grp];
          end = grp + 1 < ng ? args.group_starts[grp + 1] : (int64_t)m;
          k = args.ks[s];
        }
        for (;;) {
          const bool has_next = args.am ? kmask != 0 : s + 1 < end;
          const uint32_t knext = !has_next ? 0u
                                 : args.am ? (uint32_t)(__ffsll((long long)kmask) - 1) : args.ks[s + 1];
          for (int kc = 0; kc < kchunks; ++kc) {
            if (gstep >= STAGES) mbar_wait_sleep(&empty_bar[stage], phase ^ 1);
            unsigned char *stg = dsm + stage * C::STAGE_BYTES;
            const int kcol = (int)(k * b + kc * KW);
            int flags = 0, h = 31;
            if (kc == kchunks - 1) {
              flags = STG_MERGE;
              if (has_next) h = merge_level(k, knext);
              else flags |= STG_END;
            }
            info[stage].flags = flags;
            info[stage].h = h;
            info[stage].c_off = c_off;
            info[stage].grp = grp;
            mbar_arrive_expect_tx_l(&full_bar[stage], (unsigned)C::STAGE_BYTES);
            tma_load_2d(stg, &tmA, kcol, arow0, &full_bar[stage]);
            tma_load_2d(stg + C::A_BYTES, &tmB, bcol0, kcol, &full_bar[stage]);
            ++gstep;
            if (++stage == STAGES) {
              stage = 0;
              phase ^= 1;
            }
          }
          if (!has_next) break;
          k = knext;
          if (args.am) kmask &= kmask - 1;
          else ++s;
        }
      }
      if (gstep >= STAGES) mbar_wait_sleep(&empty_bar[stage], phase ^ 1);
      info[stage].flags = STG_DONE;
      mbar_arrive_l(&full_bar[stage]);
    }
    __syncwarp();
  } else {
    // ============================================================ consumers
    const int cw = warp - 1, tx = lane & 7, ty = lane >> 3;
    float *__restrict__ Cm = (float *)args.c;
    // this thread's rows (relative to the tile) and the byte offsets of its
    // A row starts / B column pairs within a stage
    int a_off[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) a_off[r] = (cw * 32 + (r >> 2) * 16 + ty * 4 + (r & 3)) * C::AW * 4;
    const int b_off = C::A_BYTES + tx * 16;
    float acc[64];
#pragma unroll
    for (int e = 0; e < 64; ++e) acc[e] = 0.f;
    float stk[MAXD][64];
    uint32_t pending = 0;
    int stage = 0;
    unsigned phase = 0;
    for (;;) {
      mbar_wait_sleep(&full_bar[stage], phase);
      const StageInfo si = info[stage];
      if (si.flags & STG_DONE) break;
      const unsigned char *stg = dsm + stage * C::STAGE_BYTES;
#pragma unroll 2
      for (int q4 = 0; q4 < KW / 4; ++q4) {
        float4 a[8];
#pragma unroll
        for (int r = 0; r < 8; ++r) a[r] = *reinterpret_cast<const float4 *>(stg + a_off[r] + q4 * 16);
#pragma unroll
        for (int qq = 0; qq < 4; ++qq) {
          const unsigned char *brow = stg + b_off + (q4 * 4 + qq) * 256;
          const float4 b0 = *reinterpret_cast<const float4 *>(brow);
          const float4 b1 = *reinterpret_cast<const float4 *>(brow + 128);
          const float bv[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
          for (int r = 0; r < 8; ++r) {
            const float av = qq == 0 ? a[r].x : qq == 1 ? a[r].y : qq == 2 ? a[r].z : a[r].w;
#pragma unroll
            for (int c = 0; c < 8; ++c) acc[r * 8 + c] = fmaf(av, bv[c], acc[r * 8 + c]);
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive_l(&empty_bar[stage]);
      if (++stage == STAGES) {
        stage = 0;
        phase ^= 1;
      }
      if (si.flags & STG_MERGE) {
        const int h = si.h;
        while (pending && (__ffs(pending) - 1) < h) {
          const int top = __popc(pending) - 1;
#pragma unroll
          for (int e = 0; e < 64; ++e) acc[e] = stk[top][e] + acc[e];
          pending &= pending - 1;
        }
        if (!(si.flags & STG_END)) {
          const int slot = __popc(pending);
#pragma unroll
          for (int e = 0; e < 64; ++e) {
            stk[slot][e] = acc[e];
            acc[e] = 0.f;
          }
          pending |= 1u << h;
        } else {
#pragma unroll
          for (int r = 0; r < 8; ++r) {
            float *crow = Cm + si.c_off + (int64_t)(cw * 32 + (r >> 2) * 16 + ty * 4 + (r & 3)) * N + tx * 4;
            // (scalar stores: vector stores would pin the accumulators into
            // aligned quads whose registers share banks with the B quads)
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              crow[c] = acc[r * 8 + c];
              crow[32 + c] = acc[r * 8 + 4 + c];
            }
          }
#pragma unroll
          for (int e = 0; e < 64; ++e) acc[e] = 0.f;
          pending = 0;
          if (args.grp_done) {
            __syncwarp();
            if (lane == 0)
              asm volatile("red.release.gpu.global.add.u32 [%0], 1;\n" ::"l"(&args.grp_done[si.grp])
                           : "memory");
          }
        }
      }
    }
  }
  __syncthreads();
  if (tid == 0) atomicMax(&args.tc->k3_t1, gtimer());
}

// 2-D view {N, N} of a padded f32 operand: box {w, h}.
static int make_f32_map(CUtensorMap *map, const void *base, int64_t N, int w, int h) {
  auto enc = tensor_map_encoder();
  if (!enc) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return SPAMM_ERR_CUDA;
  }
  cuuint64_t dims[2] = {(cuuint64_t)N, (cuuint64_t)N};
  cuuint64_t strides[1] = {(cuuint64_t)(N * 4)};
  cuuint32_t box[2] = {(cuuint32_t)w, (cuuint32_t)h};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void *>(base), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled (f32) failed (%d)", (int)r);
    return SPAMM_ERR_CUDA;
  }
  return SPAMM_OK;
}

template <int STAGES, int KW, int MINB = 4>
static int launch_sgemm_ws(LeafArgs args, int num_sms, cudaStream_t st) {
  CUtensorMap ma, mb;
  SPAMM_TRY(make_f32_map(&ma, args.a, args.N, SwCfg<KW>::AW, 64));
  SPAMM_TRY(make_f32_map(&mb, args.b, args.N, 64, KW));
  auto kern = leaf_sgemm_ws_kernel<STAGES, KW, MINB>;
  const int smem = STAGES * SwCfg<KW>::STAGE_BYTES + 128;
  SPAMM_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  SPAMM_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
  int per_sm = 0;
  SPAMM_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, SW_THREADS, smem));
  if (per_sm < 1) per_sm = 1;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(num_sms * per_sm);
  cfg.blockDim = dim3(SW_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  if (args.pdl) {
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
  }
  SPAMM_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, args, ma, mb));
  return SPAMM_OK;
}

static int sgemm_ws_stages() {
  static const int v = getenv("SPAMM_SGEMM_WS_STAGES") ? atoi(getenv("SPAMM_SGEMM_WS_STAGES")) : 2;
  return v;
}

int launch_leaf(const LeafArgs &args, int dtype, int num_sms, cudaStream_t st, int *launches,
                bool *signals) {
  if (signals) *signals = false;
  if (dtype == SPAMM_DTYPE_F64 && args.leaf >= 32) {
    if (args.leaf == 32) SPAMM_TRY((launch_dmma_ws<32>(args, num_sms, st)));
    else if (k3_warps() == 8) SPAMM_TRY((launch_dmma_ws<64, 8, 2>(args, num_sms, st)));
    else if (k3_warps() == 84) SPAMM_TRY((launch_dmma_ws<64, 8, 2, 4>(args, num_sms, st)));
    else if (k3_warps() == 87) SPAMM_TRY((launch_dmma_ws<64, 8, 2, 7>(args, num_sms, st)));
    else if (k3_warps() == 9) SPAMM_TRY((launch_dmma_ws<64, 8, 4>(args, num_sms, st)));
    else if (k3_warps() == 4) SPAMM_TRY((launch_dmma_ws<64, 4, 2>(args, num_sms, st)));
    else if (k3_warps() == 5) SPAMM_TRY((launch_dmma_ws<64, 16, 4, 5>(args, num_sms, st)));
    else if (k3_warps() == 3) SPAMM_TRY((launch_dmma_ws<64, 16, 4, 4>(args, num_sms, st)));
    else SPAMM_TRY((launch_dmma_ws<64>(args, num_sms, st)));
    if (signals) *signals = args.grp_done != nullptr;
  } else {
    LeafArgs a2 = args;
    a2.grp_done = nullptr;
    a2.order = nullptr;
    static const bool no_sgemm = getenv("SPAMM_NO_SGEMM") != nullptr;
    if (dtype == SPAMM_DTYPE_F64) {
      leaf_simt_kernel<double><<<num_sms * 2, SIMT_THREADS, 0, st>>>(a2);
    } else if (args.leaf >= 64 && !no_sgemm && sgemm_ws_stages() > 0) {
      // FP32 warp-specialised TMA kernel (SPAMM_SGEMM_WS_STAGES: ring depth, 0: off)
      // SPAMM_SGEMM_WS_STAGES: 2 (default) or 3 stages of 32-wide inner
      // chunks; 64: 2 stages of 64 (3 CTAs per SM by shared memory); 5: two
      // stages at the 128-register budget (5 CTAs per SM); 0: the
      // register-staged kernel below
      switch (sgemm_ws_stages()) {
        case 3: SPAMM_TRY((launch_sgemm_ws<3, 32>(a2, num_sms, st))); break;
        case 64: SPAMM_TRY((launch_sgemm_ws<2, 64>(a2, num_sms, st))); break;
        case 5: SPAMM_TRY((launch_sgemm_ws<2, 32, 5>(a2, num_sms, st))); break;
        default: SPAMM_TRY((launch_sgemm_ws<2, 32>(a2, num_sms, st))); break;
      }
    } else if (args.leaf >= 64 && !no_sgemm) {
      // micro-tile shape (SPAMM_SGEMM_SHAPE): 84 = 8 x 4 per thread (128 threads,
      // default), 44 = 4 x 4 (256), 88 = 8 x 8 (64)
      static const int shape = getenv("SPAMM_SGEMM_SHAPE") ? atoi(getenv("SPAMM_SGEMM_SHAPE")) : 84;
      auto go = [&](auto kern, int threads) -> int {
        SPAMM_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            (int)SG_SMEM));
        kern<<<num_sms * 3, threads, SG_SMEM, st>>>(a2);
        return SPAMM_OK;
      };
      if (shape == 44) SPAMM_TRY(go(leaf_sgemm_kernel<4, 4>, 256));
      else if (shape == 88) SPAMM_TRY(go(leaf_sgemm_kernel<8, 8>, 64));
      else SPAMM_TRY(go(leaf_sgemm_kernel<8, 4>, 128));
    } else {
      leaf_simt_kernel<float><<<num_sms * 2, SIMT_THREADS, 0, st>>>(a2);
    }
  }
  SPAMM_CUDA_TRY(cudaGetLastError());
  if (launches) ++*launches;
  return SPAMM_OK;
}

}  // namespace spamm
