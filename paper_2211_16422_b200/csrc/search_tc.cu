// Tensor-core engine of the windowed Hamming top-k search (k <= 64) (sm_100a: tcgen05 + TMEM + bulk copies,
// CTA pairs / cta_group::2 from D = 2048 up).
//
// Reference semantics are those of search.cu (search.cpp:93-169): per query the candidate row with
// the largest Hamming similarity inside its precursor window, ties broken by (|q - r|, id, ordinal).
//
// The similarity of two D-bit hypervectors is an inner product once every bit b is expanded to the
// int8 value 2b - 1:   dot(x, y) = #agree - #differ = D - 2 * popcount(x ^ y)
//                      raw_score = D - popcount(x ^ y) = (D + dot) / 2        (hypervector.hpp:70-81)
// exactly, in int32.  tools/microbench.cu measured the alternatives on a B200: the XOR+POPC pipe
// tops out at 15.3 32-bit words/clk/SM (23 with a carry-save tree), mma.sync.s8 at 61 word
// equivalents, and the 5th-generation tensor core (tcgen05.mma kind::i8) at 8192 MAC/clk/SM =
// 256 word equivalents.  So the search becomes a windowed GEMM:
//
//   C[query, row] = Qx[query, :] . Lx[row, :]      Qx, Lx in {-1, +1}^D (0 in padding)
//
// * Lx is built once per library upload, Qx once per search, both in HBM as
//   [k-chunk][row][128 bytes] with the 16-byte units of every row XOR-swizzled by (row & 7): a
//   tile of R consecutive rows of one k-chunk is then ONE contiguous R*128-byte block that is
//   already in the SWIZZLE_128B K-major layout tcgen05.mma wants, so a stage of the pipeline is
//   two cp.async.bulk copies (no tensor map needed) completing on an mbarrier.  Operands are e2m1
//   nibbles (kind::mxf4 with unit block scales, 256 dimensions per row, N = 224, 5 stages); the
//   int8 encoding of round 1 (kind::i8: twice the bytes, half the rate, same results) was removed.
// * queries are sorted by window start + end (search.cu) and cut into tiles of 128 = the 128 TMEM lanes;
//   the library rows a tile needs (union of its windows) are cut into N-row MMA tiles aligned to
//   absolute multiples of N, so that different query tiles fetch identical blocks (L2 hits).
// * one CTA per SM, 6 warps: one (elected) thread of warp 0 draws work items and issues the bulk copies, one
//   thread of warp 1 issues the MMAs (4 per stage) into one of two 128 x N accumulators in TMEM, warps 2-5
//   drain the other accumulator: lane = query, column = library row; every thread keeps the running best of
//   its query with the exact 3-level key (top-k: appends the candidates above the query's floor to a buffer,
//   tc_select_kernel picks the k best exactly) and masks columns outside the query's own window.  The drain
//   overlaps with the next tile's MMAs.  From D = 2048 up two CTAs of a cluster pair up on 256-query tiles
//   (cta_group::2, TcShape<true>): each streams its own queries and half of every library tile.  At D <= 1024
//   the query tile's k-chunks stay resident in shared memory for a whole work item (TcShape<false, true>).
// * work items (query tile x strip of row tiles) are planned on the device (tc_plan_*_kernel),
//   ordered (group of query tiles, strip, tile) and handed out dynamically in that order, so that
//   the CTAs running at any moment share both query and row tiles in L2; the whole search is
//   stream-ordered, without a host round trip.
#include <algorithm>
#include <climits>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "radix.cuh"
#include "topk.cuh"

namespace hb {

constexpr int kTcM = 128;      // queries per tile == TMEM lanes
constexpr int kTcKB = 128;     // K bytes per pipeline stage == one swizzle atom
constexpr uint32_t kTcABytes = kTcM * kTcKB;  // 16 KB
constexpr int kTcThreads = 192;
constexpr uint32_t kTcBarBytes = 512;
constexpr uint32_t kTcTmemCols = 512;  // two accumulators (+ the scale-factor columns in fp4 mode)

// Operand encoding of the +-1 contraction: e2m1 nibbles (+1.0 = 0x2, -1.0 = 0xA), 256 dimensions per
// 128-byte stage row, block scale factors all 1.0 (UE8M0 0x7F), fp32 accumulate (exact: |dot| <= D <
// 2^24).  N = 224 leaves room in TMEM for the (constant) scale factors next to two accumulators and in
// shared memory for a 5-stage ring (220 KB).
struct TcMode {
#ifndef HB_TC_FP4_N
#define HB_TC_FP4_N 224      // measured: 224 rows x 5 stages beats 240 x 4 and 208 x 5 (profiles/)
#define HB_TC_FP4_STAGES 5
#endif
  static constexpr int N = HB_TC_FP4_N;            // library rows per MMA tile
  static constexpr int Stages = HB_TC_FP4_STAGES;  // depth of the smem ring
  static constexpr int kDims = 256;                // dimensions per 128-byte stage row
  static constexpr uint32_t BBytes = N * kTcKB;
  static constexpr uint32_t StageBytes = kTcABytes + BBytes;  // multiple of 1024
  static constexpr uint32_t SmemBytes = Stages * StageBytes + 1024 + kTcBarBytes;
  static constexpr uint32_t SfCol = 480;           // scale-factor columns [480, 512)
};
// Shape of one CTA's share of a pipeline stage.  Single: the CTA holds the whole 128 x N tile pair (A 16 KB +
// B 28 KB, 5 stages).  Pair (cta_group::2): two CTAs of one cluster (one TPC) work on a 256-query x N-row tile
// with M = 256; each holds its own 128 query rows and HALF of the library tile (A 16 KB + B 14 KB, 7 stages):
// a third fewer bytes from L2 per MMA and a third fewer shared-memory operand reads, which under the board's
// power cap is clock.
// kARes (single CTA, D <= 1024): the query tile's k-chunks (<= 4 x 16 KB) are loaded ONCE per work item into a
// resident area and only the library tiles stream through the ring -- at D = 1024 every row tile re-fetched the same
// four A chunks, 36 % of the operand bytes, and the kernel was bound by the L2 -> SM fills (ncu: lts throughput 82 %,
// 20 TB/s of fills, tensor pipe 75 % active).
constexpr uint32_t kTcAResChunks = 4;
template <bool kPair, bool kARes = false>
struct TcShape {
  static_assert(!(kPair && kARes), "the resident-A form is a single-CTA form");
  static constexpr int BRows = kPair ? TcMode::N / 2 : TcMode::N;
  static constexpr uint32_t BBytes = BRows * kTcKB;
  static constexpr uint32_t StageBytes = (kARes ? 0u : kTcABytes) + BBytes;  // multiple of 1024
  static constexpr uint32_t AOff = kARes ? 0u : 0u;                            // A inside a stage (streamed forms)
  static constexpr uint32_t BOff = kARes ? 0u : kTcABytes;                     // B inside a stage
  static constexpr uint32_t ResBytes = kARes ? kTcAResChunks * kTcABytes : 0u;  // resident A area in front of the ring
  static constexpr int Stages = kPair ? 7 : TcMode::Stages;
  static constexpr uint32_t SmemBytes = ResBytes + Stages * StageBytes + 1024 + kTcBarBytes;
  static constexpr uint32_t TileQ = kPair ? 2 * kTcM : kTcM;  // sorted positions per planning tile
};
static_assert(TcShape<true>::StageBytes % 1024 == 0 && TcShape<false>::StageBytes % 1024 == 0 &&
                  TcShape<false, true>::StageBytes % 1024 == 0,
              "stage alignment");
static_assert(TcShape<true>::SmemBytes <= 227 * 1024 && TcShape<false>::SmemBytes <= 227 * 1024 &&
                  TcShape<false, true>::SmemBytes <= 227 * 1024,
              "shared memory");
constexpr uint32_t kTcGroupTiles = 12;  // query tiles per L2 group, at least
constexpr int kTcMaxK = 32;             // top-k depth the drain keeps per query in ONE pass; larger k runs
                                        // ceil(k / 32) passes, each bounded below by the previous pass's last key
constexpr uint64_t kTcBatch = 64 * 1024;  // sorted slots per planning batch

struct TcItem {
  uint32_t tile;       // query tile (128 sorted positions) inside the batch
  uint32_t row_begin;  // local library rows [row_begin, row_end), row_begin % 256 == 0
  uint32_t row_end;
  uint32_t pad;
};

struct TcParams {
  const uint8_t* lib_x;
  const uint8_t* q_x;
  uint64_t lib_rows;  // rows per k-chunk plane of lib_x
  uint64_t q_rows;    // rows per k-chunk plane of q_x
  uint32_t n_kc;
  uint32_t dim;
  const TcItem* items;
  const uint32_t* n_items;  // device: number of work items (written by the planner)
  uint32_t* counter;        // device: next work item to hand out (zeroed by the planner)
  const uint64_t* keys;  // sorted (local first row << 32 | local last row), batch base applied
  const uint32_t* vals;  // sorted slot ids
  const uint32_t* subset;
  const double* q_mz;
  const double* lib_mz;
  const uint32_t* lib_rank;
  uint64_t n;  // sorted positions in this batch
  Cand* partial;  // [n_items][128][k]
  int* gbest;     // [q_rows][k] best dot seen per residue class (row % k) of a sorted position (see the drain)
  uint32_t k;     // candidates kept per query in this pass (1 .. kTcMaxK)
  uint32_t prev_col;      // pass > 0: column of `prev` holding the last key of the previous pass
  const Cand* prev;       // pass > 0: the output so far, [slot][prev_stride]; only keys strictly after
  uint32_t prev_stride;   //           prev[slot][prev_col] are candidates of this pass (nullptr: pass 0)
  uint32_t l2_hints;      // bit 0: query tiles (A) evict_last, bit 1: library tiles (B) evict_first
  // collect mode (KM == 0): candidates at or above the query's floor are appended to its buffer
  uint32_t* ccount;       // [q_rows] entries appended so far (may run past ccap: overflow, see tc_select_kernel)
  uint2* cbuf;            // [q_rows][ccap] (dot, local row)
  uint32_t ccap;
  uint32_t pad3;
};

// ---- PTX wrappers ---------------------------------------------------------------------------

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}
// A wait that can never hang the GPU: a pipeline bug traps after ~4 s instead of spinning forever.
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  if (mbar_try_wait(bar, parity)) return;
  const long long t0 = clock64();
  uint32_t spins = 0;
  while (!mbar_try_wait(bar, parity)) {
    if ((++spins & 0xFFFu) == 0 && clock64() - t0 > 8000000000ll) __trap();
  }
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}
// the same copy with an L2 eviction-priority hint (createpolicy descriptor)
__device__ __forceinline__ void bulk_g2s_hint(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(bar), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_policy_evict_normal() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
// ---- cluster (CTA pair) helpers ----
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// shared::cta address -> shared::cluster address of the same offset in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t mapa_u32(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
// Remote arrives.  The release form orders this thread's earlier stores (the FIFO entry written into the peer's
// shared memory) before the arrive; it costs a MEMBAR.ALL.GPU and is used once per work item.  The relaxed form is
// a bare arrive for the signals that publish no data of this thread: "my stage has landed" (the bytes sit in the
// signalling SM's own shared memory and are read by that SM's tensor core), "accumulator drained", "slot free".
__device__ __forceinline__ void mbar_arrive_remote(uint32_t cluster_bar) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_bar) : "memory");
}
__device__ __forceinline__ void mbar_arrive_remote_relaxed(uint32_t cluster_bar) {
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_bar) : "memory");
}
__device__ __forceinline__ void st_remote_b64(uint32_t cluster_addr, uint64_t v) {
  asm volatile("st.shared::cluster.b64 [%0], %1;" ::"r"(cluster_addr), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_shared_volatile_b64(uint32_t addr) {
  uint64_t v;
  asm volatile("ld.volatile.shared.b64 %0, [%1];" : "=l"(v) : "r"(addr) : "memory");
  return v;
}
__device__ __forceinline__ uint4 ld_shared_volatile_v4(uint32_t addr) {
  uint4 v;
  asm volatile("ld.volatile.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr) : "memory");
  return v;
}
// wait that also acquires what a thread of the OTHER CTA of the cluster published before its arrive
__device__ __forceinline__ bool mbar_try_wait_cluster(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait_cluster(uint32_t bar, uint32_t parity) {
  if (mbar_try_wait_cluster(bar, parity)) return;
  const long long t0 = clock64();
  uint32_t spins = 0;
  while (!mbar_try_wait_cluster(bar, parity)) {
    if ((++spins & 0xFFFu) == 0 && clock64() - t0 > 8000000000ll) __trap();
  }
}
// completion of every MMA issued so far by this thread, signalled to the barrier at this offset in BOTH CTAs
__device__ __forceinline__ void tc_commit_pair(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(bar),
               "h"(static_cast<uint16_t>(3))
               : "memory");
}
__device__ __forceinline__ void tc_mma_fp4_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                                uint32_t sfa, uint32_t sfb, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %6, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::mxf4.block_scale.scale_vec::2X [%0], %1, %2, %3, [%4], [%5], p;\n\t}" ::"r"(
          tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(sfa), "r"(sfb), "r"(accumulate)
      : "memory");
}
// true in exactly one lane of the (converged) warp; unlike `lane == 0` the compiler KNOWS the guarded code runs in
// a single thread and issues the uniform-datapath instructions (UBLKCP, UTCOMMA, UTCBAR) without wrapping each one
// in a loop over the distinct operand values of the active threads
__device__ __forceinline__ bool elect_one() {
#ifdef HB_TC_NO_ELECT  // A/B build: the round-1 form (profiles/r02_ab_elect.log)
  return (threadIdx.x & 31) == 0;
#endif
  uint32_t pred;
  asm volatile("{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(pred));
  return pred != 0;
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}
// D[tmem] (+)= A * B^T, e2m1 x e2m1 with per-32 UE8M0 block scales from TMEM -> fp32, K = 64
__device__ __forceinline__ void tc_mma_fp4(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                           uint32_t sfa, uint32_t sfb, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %6, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.scale_vec::2X [%0], %1, %2, %3, [%4], [%5], p;\n\t}" ::"r"(
          tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(sfa), "r"(sfb), "r"(accumulate)
      : "memory");
}
// issue a load of 32 consecutive columns of this thread's TMEM lane; v is valid after tc_ld_wait()
__device__ __forceinline__ void tc_ld32_issue(uint32_t taddr, int (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
      "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
        "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),
        "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),
        "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr)
      : "memory");
}
// wait for the outstanding TMEM loads; the registers are listed as in/out operands so that the
// compiler cannot move any use of them above the wait
__device__ __forceinline__ void tc_ld_wait(int (&v)[32]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;"
               : "+r"(v[0]), "+r"(v[1]), "+r"(v[2]), "+r"(v[3]), "+r"(v[4]), "+r"(v[5]), "+r"(v[6]), "+r"(v[7]),
                 "+r"(v[8]), "+r"(v[9]), "+r"(v[10]), "+r"(v[11]), "+r"(v[12]), "+r"(v[13]), "+r"(v[14]),
                 "+r"(v[15]), "+r"(v[16]), "+r"(v[17]), "+r"(v[18]), "+r"(v[19]), "+r"(v[20]), "+r"(v[21]),
                 "+r"(v[22]), "+r"(v[23]), "+r"(v[24]), "+r"(v[25]), "+r"(v[26]), "+r"(v[27]), "+r"(v[28]),
                 "+r"(v[29]), "+r"(v[30]), "+r"(v[31])
               :
               : "memory");
}
// fill 32 consecutive columns of this thread's TMEM lane with one word
__device__ __forceinline__ void tc_st32_fill(uint32_t taddr, uint32_t w) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, "
      "%1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1};" ::"r"(taddr),
      "r"(w)
      : "memory");
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}
// Shared-memory matrix descriptor of a K-major SWIZZLE_128B operand whose rows are 128 bytes:
// start address >> 4 in bits [0,14), leading byte offset (unused for one swizzle atom along K) in
// [16,30), stride byte offset = 1024 B between 8-row groups in [32,46), descriptor version 1 in
// [46,48), layout type 2 = SWIZZLE_128B in [61,64).
__device__ __forceinline__ uint64_t tc_smem_desc(uint32_t smem_addr) {
  const uint64_t lo = (uint64_t(smem_addr & 0x3FFFFu) >> 4) | (uint64_t(1) << 16);
  const uint64_t hi = uint64_t(1024 >> 4) | (uint64_t(1) << 14) | (uint64_t(2) << 29);
  return lo | (hi << 32);
}
// Block-scaled descriptor, kind::mxf4: A = B = E2M1 (format 1 in [7,10) and [10,13)), K-major,
// N >> 3 in [17,23), scale format UE8M0 (bit 23), M >> 4 in [24,29), scale-factor ids 0, K = 64.
constexpr uint32_t kTcIdescFp4 = (1u << 7) | (1u << 10) | (uint32_t(TcMode::N >> 3) << 17) | (1u << 23) |
                                 (uint32_t(kTcM >> 4) << 24);
constexpr uint32_t kTcIdescFp4Pair = (1u << 7) | (1u << 10) | (uint32_t(TcMode::N >> 3) << 17) | (1u << 23) |
                                     (uint32_t((2 * kTcM) >> 4) << 24);  // M = 256 over the CTA pair

// ---- expansion: packed bits -> swizzled +-1 operand image -----------------------------------

// One warp per (row, group of 4 k-chunks): lane = (k-chunk in group) * 8 + 16-byte unit.  A bit b
// becomes the e2m1 nibble +-1.0 (32 dimensions per unit); dimensions at or above dim and rows at or above n_rows become 0 so that they contribute
// nothing to any dot product.  The order of the dimensions inside a unit is irrelevant as long as
// library and queries use the same one (a dot product is invariant under a common permutation).
__global__ void tc_expand_kernel(uint64_t out_rows, uint64_t n_rows, const uint32_t* __restrict__ src_pos,
                                 const uint32_t* __restrict__ src_subset, uint64_t pos_base,
                                 const uint64_t* __restrict__ words, uint32_t stride_words, uint32_t dim,
                                 uint32_t n_kc, uint8_t* __restrict__ out) {
  constexpr uint32_t kUnitDims = 32;
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t warp = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint32_t groups = (n_kc + 3) / 4;
  const uint64_t row = warp / groups;
  const uint32_t kc = static_cast<uint32_t>(warp % groups) * 4 + (lane >> 3);
  if (row >= out_rows || kc >= n_kc) return;
  const uint32_t unit = lane & 7;
  uint4 o = make_uint4(0, 0, 0, 0);
  if (row < n_rows) {
    uint64_t src = row;
    if (src_pos) {  // queries: sorted position -> slot -> resident query
      src = src_pos[pos_base + row];
      if (src_subset) src = src_subset[src];
    }
    const uint32_t bit0 = kc * TcMode::kDims + unit * kUnitDims;
    uint32_t bits = 0;
    if (bit0 < dim)
      bits = static_cast<uint32_t>(words[src * stride_words + (bit0 >> 6)] >> (bit0 & 63));
    const uint32_t valid = dim - min(dim, bit0);  // dimensions of this unit below dim
    uint32_t w[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {  // 8 dimensions -> 8 nibbles: bit 1 -> 0x2 (+1.0), bit 0 -> 0xA (-1.0)
      const uint32_t b8 = (bits >> (8 * i)) & 0xFFu;
      uint32_t spread = 0, keep = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        spread |= ((b8 >> j) & 1u) << (4 * j + 3);
        if (uint32_t(8 * i + j) < valid) keep |= 0xFu << (4 * j);
      }
      w[i] = (0xAAAAAAAAu ^ spread) & keep;
    }
    o = make_uint4(w[0], w[1], w[2], w[3]);
  }
  uint8_t* dst = out + ((uint64_t(kc) * out_rows + row) * 128) + ((unit ^ (row & 7)) << 4);
  *reinterpret_cast<uint4*>(dst) = o;
}

// per planning tile of the batch: union [lo, hi) of the windows of its tile_q (128, CTA pair: 256) sorted positions
__global__ void tc_tile_ranges_kernel(uint64_t n, const uint64_t* __restrict__ keys, uint32_t n_tiles, uint32_t tile_q,
                                      uint2* __restrict__ ranges) {
  const uint32_t tile = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t lane = threadIdx.x & 31;
  if (tile >= n_tiles) return;
  uint32_t lo = kNone, hi = 0;
  for (uint32_t j = lane; j < tile_q; j += 32) {
    const uint64_t p = uint64_t(tile) * tile_q + j;
    if (p >= n) break;
    const uint64_t key = keys[p];
    if (key == ~0ull) continue;
    lo = min(lo, static_cast<uint32_t>(key >> 32));
    hi = max(hi, static_cast<uint32_t>(key));
  }
  for (int o = 16; o > 0; o >>= 1) {
    lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  if (lane == 0) ranges[tile] = (lo == kNone || hi <= lo) ? make_uint2(0, 0) : make_uint2(lo, hi);
}

// ---- device planner ---------------------------------------------------------------------------
// Work items = (query tile, strip of row tiles).  Strips sit at absolute multiples of `strip` row
// tiles so that different query tiles fetch identical blocks; items are ordered (query-tile group,
// strip, tile) and kept short (<= max_strip row tiles, about items_per_sm items per SM) so that the
// CTAs running at the same time stay in step and share both operands in L2 (ncu: DRAM 261 GB ->
// 30 GB per launch on config 2).  Planning on the device keeps the whole search stream-ordered:
// no host round trip between the window bounds and the search kernel.

struct TcPlanHead {
  uint32_t n_items, strip, n_pairs, n_groups;
  uint32_t counter;  // work-item queue of tc_search_kernel
};
struct TcPlanCfg {
  uint32_t n_tiles, group_tiles, max_strip, tiles_total;
  uint64_t target_items;  // items the planner aims for (SM count x items per SM)
  uint32_t item_cap;      // capacity of the item / partial arrays
  uint32_t pad;
};
// plan block layout (uint32 units after the head): see tc_plan_layout()
struct TcPlanPtrs {
  TcPlanHead* head;
  TcItem* items;
  uint32_t *tile_start, *tile_items, *tlo, *thi, *grp_item_base, *grp_pair_base, *grp_lo_strip;
};
static __host__ __device__ inline size_t tc_plan_bytes(uint32_t n_tiles, uint32_t item_cap) {
  return 64 + size_t(item_cap) * (sizeof(TcItem) + 4) + (size_t(n_tiles) * 6 + 8) * 4;
}
static __host__ __device__ inline TcPlanPtrs tc_plan_layout(void* base, uint32_t n_tiles, uint32_t item_cap) {
  TcPlanPtrs q;
  auto* b = static_cast<unsigned char*>(base);
  q.head = reinterpret_cast<TcPlanHead*>(b);
  q.items = reinterpret_cast<TcItem*>(b + 64);
  q.tile_items = reinterpret_cast<uint32_t*>(q.items + item_cap);
  q.tile_start = q.tile_items + item_cap;   // n_tiles + 1
  q.tlo = q.tile_start + n_tiles + 1;       // n_tiles
  q.thi = q.tlo + n_tiles;                  // n_tiles
  q.grp_item_base = q.thi + n_tiles;        // <= n_tiles + 1
  q.grp_pair_base = q.grp_item_base + n_tiles + 1;
  q.grp_lo_strip = q.grp_pair_base + n_tiles + 1;  // <= n_tiles
  return q;
}

constexpr int kTcPlanThreads = 512;  // >= query tiles per planning batch (kTcBatch / kTcM)

template <uint32_t kN>
__global__ void __launch_bounds__(kTcPlanThreads) tc_plan_head_kernel(TcPlanCfg c, const uint2* __restrict__ ranges,
                                                                      void* plan) {
  const TcPlanPtrs q = tc_plan_layout(plan, c.n_tiles, c.item_cap);
  __shared__ uint32_t s_lo[kTcPlanThreads], s_hi[kTcPlanThreads];  // row-tile range of every query tile
  __shared__ unsigned long long s_work;
  __shared__ uint32_t s_strip, s_total[3];
  const uint32_t t = threadIdx.x;
  uint32_t lo = 0, hi = 0;
  if (t < c.n_tiles) {
    const uint2 r = ranges[t];
    lo = r.x / kN;
    hi = r.y > r.x ? (r.y + kN - 1) / kN : lo;
    q.tlo[t] = lo;
    q.thi[t] = hi;
  }
  s_lo[t] = lo;
  s_hi[t] = hi;
  if (t == 0) s_work = 0;
  __syncthreads();
  if (hi > lo) atomicAdd(&s_work, static_cast<unsigned long long>(hi - lo));
  __syncthreads();
  if (t == 0) {
    const uint64_t work = s_work;
    uint64_t strip = (work + c.target_items - 1) / c.target_items;
    strip = strip < 1 ? 1 : (strip > c.max_strip ? c.max_strip : strip);
    // never more items than the arrays hold: items <= work / strip + 2 * n_tiles
    const uint64_t slack = 2ull * c.n_tiles + 16;
    const uint64_t fit = c.item_cap > slack ? (work + (c.item_cap - slack) - 1) / (c.item_cap - slack)
                                            : uint64_t(c.tiles_total) + 1;
    if (fit > strip) strip = fit;
    s_strip = static_cast<uint32_t>(strip < 0xffffffffull ? strip : 0xffffffffull);
  }
  __syncthreads();
  const uint32_t strip = s_strip;
  const uint32_t ns = hi > lo ? (hi + strip - 1) / strip - lo / strip : 0;  // strips this tile overlaps
  // exclusive scan of ns over the tiles (warp shuffles + one shared-memory step, radix.cuh)
  const uint32_t ns_before = block_exclusive_sum_u32<kTcPlanThreads>(ns);
  if (t < c.n_tiles) q.tile_start[t] = ns_before;
  if (t == c.n_tiles - 1) q.tile_start[c.n_tiles] = ns_before + ns;
  // groups of consecutive query tiles
  const uint32_t n_groups = (c.n_tiles + c.group_tiles - 1) / c.group_tiles;
  uint32_t g_items = 0, g_pairs = 0, g_lo_strip = 0;
  if (t < n_groups) {
    const uint32_t t0 = t * c.group_tiles, t1 = min(c.n_tiles, t0 + c.group_tiles);
    uint32_t glo = 0xffffffffu, ghi = 0;
    for (uint32_t j = t0; j < t1; ++j) {
      const uint32_t a = s_lo[j], b = s_hi[j];
      if (b > a) {
        glo = min(glo, a);
        ghi = max(ghi, b);
        g_items += (b + strip - 1) / strip - a / strip;
      }
    }
    if (glo != 0xffffffffu) {
      g_lo_strip = glo / strip;
      g_pairs = (ghi + strip - 1) / strip - g_lo_strip;
    }
    q.grp_lo_strip[t] = g_lo_strip;
  }
  // exclusive scans over the groups
  const uint32_t items_before = block_exclusive_sum_u32<kTcPlanThreads>(g_items);
  const uint32_t pairs_before = block_exclusive_sum_u32<kTcPlanThreads>(g_pairs);
  if (t < n_groups) {
    q.grp_item_base[t] = items_before;
    q.grp_pair_base[t] = pairs_before;
  }
  if (t == kTcPlanThreads - 1) {  // the last thread's exclusive sums + its own values are the totals
    s_total[0] = items_before + g_items;
    s_total[1] = pairs_before + g_pairs;
  }
  __syncthreads();
  if (t == 0) {
    q.grp_item_base[n_groups] = s_total[0];
    q.grp_pair_base[n_groups] = s_total[1];
    q.head->n_items = s_total[0];
    q.head->counter = 0;
    q.head->strip = strip;
    q.head->n_pairs = s_total[1];
    q.head->n_groups = n_groups;
  }
}

// one WARP per (group, strip) pair: its items, in tile order, and the per-tile item lists.  (One thread per pair
// walked the group's tiles twice in a chain of dependent loads: 34 us for config 2's 307 strips.)
template <uint32_t kN>
__global__ void tc_plan_items_kernel(TcPlanCfg c, void* plan) {
  const TcPlanPtrs q = tc_plan_layout(plan, c.n_tiles, c.item_cap);
  const uint32_t n_pairs = q.head->n_pairs, n_groups = q.head->n_groups, strip = q.head->strip;
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, n_warps = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t pr = warp; pr < n_pairs; pr += n_warps) {
    uint32_t g = 0, gh = n_groups;  // last group whose pair base is <= pr
    while (gh - g > 1) {
      const uint32_t mid = (g + gh) >> 1;
      if (q.grp_pair_base[mid] <= pr) g = mid;
      else gh = mid;
    }
    const uint32_t sidx = q.grp_lo_strip[g] + (pr - q.grp_pair_base[g]);
    const uint32_t t0 = g * c.group_tiles, t1 = min(c.n_tiles, t0 + c.group_tiles);
    // items of this group that come before strip sidx: per tile, its strips below sidx
    uint32_t before = 0;
    for (uint32_t j = t0 + lane; j < t1; j += 32) {
      const uint32_t a = q.tlo[j], b = q.thi[j];
      if (b <= a) continue;
      const uint32_t first = a / strip, cnt = (b + strip - 1) / strip - first;
      before += sidx > first ? min(sidx - first, cnt) : 0;
    }
    uint32_t idx = q.grp_item_base[g] + __reduce_add_sync(0xffffffffu, before);
    const uint64_t s_lo = uint64_t(sidx) * strip, s_hi = s_lo + strip;
    for (uint32_t j0 = t0; j0 < t1; j0 += 32) {  // 32 tiles per round, items numbered in tile order
      const uint32_t j = j0 + lane;
      uint32_t tl = 0, th = 0;
      if (j < t1) {
        tl = q.tlo[j];
        th = q.thi[j];
      }
      const uint64_t a = max(uint64_t(tl), s_lo), b = min(uint64_t(th), s_hi);
      const bool has = j < t1 && b > a;
      const uint32_t mask = __ballot_sync(0xffffffffu, has);
      if (has) {
        const uint32_t my = idx + __popc(mask & ((1u << lane) - 1u));
        q.items[my] = TcItem{j, static_cast<uint32_t>(a) * kN, static_cast<uint32_t>(b) * kN, 0};
        q.tile_items[q.tile_start[j] + (sidx - tl / strip)] = my;
      }
      idx += __popc(mask);
    }
  }
}

// ---- the search kernel ----------------------------------------------------------------------


// accumulator word -> score domain of the drain: fp32 holding exact integers
struct TcAcc {
  using T = float;
  static __device__ __forceinline__ T lowest() { return -3.0e38f; }
  static __device__ __forceinline__ T get(int raw) { return __int_as_float(raw); }
  static __device__ __forceinline__ int to_int(T v) { return __float2int_rn(v); }
  static __device__ __forceinline__ T from_int(int v) { return static_cast<float>(v); }
};

// KM = 1: plain top-1 drain; KM > 1: the drain keeps the best KM >= p.k candidates per query; KM = 0: collect.
// kPair: two CTAs of a cluster share every work item (see TcShape): the leader (cluster rank 0) draws the
// items and issues the M = 256 MMAs for both, each CTA streams its own operand share and drains its own
// 128 queries.  What crosses the pair: the item FIFO (leader -> peer, DSMEM store + remote arrive), "my stage is
// full" (peer -> leader, relayed by the peer's otherwise idle warp 1), "accumulator drained" and "item slot
// free" (peer -> leader, remote arrives); "stage free" and "accumulator complete" reach both CTAs through the
// multicast form of tcgen05.commit.
template <int KM, bool kPair, bool kARes>
__global__ void __launch_bounds__(kTcThreads, 1) tc_search_kernel(const TcParams p) {
  constexpr bool kTopK = KM > 1;      // register lists of depth KM
  constexpr bool kCollect = KM == 0;  // append candidates above the floor, select exactly afterwards
  constexpr int kList = KM > 0 ? KM : 1;
  using Mode = TcMode;
  using Shape = TcShape<kPair, kARes>;
  using Acc = TcAcc;
  using AccT = typename Acc::T;
  constexpr int kN = Mode::N;
  constexpr int kStages = Shape::Stages;
  extern __shared__ unsigned char tc_smem_raw[];
  const uint32_t raw = smem_u32(tc_smem_raw);
  const uint32_t res_base = (raw + 1023u) & ~1023u;  // SWIZZLE_128B atoms need 1024-byte alignment
  const uint32_t base = res_base + Shape::ResBytes;  // the ring; the resident A area (kARes) sits in front of it
  unsigned char* gen_base = tc_smem_raw + (base - raw);
  const uint32_t bar0 = base + kStages * Shape::StageBytes;
  // barrier block: full[S], empty[S], tfull[2], tempty[2], TMEM base address, ifull[Q], iempty[Q], pfull[S], items[Q],
  // afull, aempty (kARes: the resident A area is loaded / may be overwritten)
  auto full_bar = [&](int s) { return bar0 + 8u * s; };
  auto empty_bar = [&](int s) { return bar0 + 8u * (kStages + s); };
  auto tfull_bar = [&](int a) { return bar0 + 8u * (2 * kStages + a); };
  auto tempty_bar = [&](int a) { return bar0 + 8u * (2 * kStages + 2 + a); };
  volatile uint32_t* tmem_slot =
      reinterpret_cast<volatile uint32_t*>(gen_base + kStages * Shape::StageBytes + 8 * (2 * kStages + 4));
  // Work items are handed out dynamically, in plan order, through one device-wide counter: however
  // long a CTA's drain takes, the CTAs running at any moment work on ~gridDim consecutive items, which
  // is what keeps their operand tiles shared in L2 (with a static round-robin a delayed CTA stays
  // behind for good and drifts out of its neighbours' tiles: top-5 read 108 GB from DRAM per launch
  // instead of 29).  The producer draws the ids and passes the items to the MMA thread and the drain warps
  // through a small FIFO in shared memory (ifull / iempty barriers per slot).
  constexpr int kItemQ = 4;
  constexpr uint32_t ibar_off = 8u * (2 * kStages + 4) + 8u;
  auto ifull_bar = [&](int s) { return bar0 + ibar_off + 8u * s; };
  auto iempty_bar = [&](int s) { return bar0 + ibar_off + 8u * (kItemQ + s); };
  auto pfull_bar = [&](int s) { return bar0 + ibar_off + 8u * (2 * kItemQ + s); };  // pair: the peer's stage s is full
  constexpr uint32_t item_off = (ibar_off + 8u * (2 * kItemQ + kStages) + 15u) & ~15u;
  static_assert(item_off + 16 * kItemQ + 16 <= kTcBarBytes, "barrier block too small");
  const uint32_t afull_bar = bar0 + item_off + 16u * kItemQ, aempty_bar = afull_bar + 8u;
  volatile uint32_t* s_item = reinterpret_cast<volatile uint32_t*>(gen_base + kStages * Shape::StageBytes + item_off);
  const uint32_t s_item_addr = bar0 + item_off;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = kPair ? cluster_ctarank() : 0u;  // 0: leader (draws items, issues the MMAs)
  // consumers of an item slot: the MMA thread + 4 drain warps here; in a pair also the peer's producer, relay
  // and 4 drain warps (they arrive on the LEADER's barrier)
  constexpr uint32_t kItemConsumers = kPair ? 11 : 5;

  // no FIFO entry left over from an earlier launch may pass for a hand-out of this one (see read_item)
  if (threadIdx.x >= 32 && threadIdx.x < 32 + 4 * kItemQ) s_item[threadIdx.x - 32] = 0xFFFFFFFFu;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(full_bar(s), 1);
      mbar_init(empty_bar(s), 1);
      mbar_init(pfull_bar(s), 1);
    }
    for (int s = 0; s < kItemQ; ++s) {
      mbar_init(ifull_bar(s), 1);
      mbar_init(iempty_bar(s), kItemConsumers);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(tfull_bar(a), 1);
      mbar_init(tempty_bar(a), kPair ? 8 : 4);  // one arrival per drain warp (of both CTAs)
    }
    mbar_init(afull_bar, 1);
    mbar_init(aempty_bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    if constexpr (kPair) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(const_cast<uint32_t*>(tmem_slot))),
                   "r"(kTcTmemCols)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(const_cast<uint32_t*>(tmem_slot))),
                   "r"(kTcTmemCols)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (kPair) cluster_sync_all();  // the peer's barriers are initialised before anything arrives on them
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // every block scale is 1.0 = UE8M0 0x7F: fill all 32 scale-factor columns of all 128 lanes once,
  // so whatever bytes the MMA reads for A or B rows it reads 1.0
  if (warp >= 2) tc_st32_fill(tmem_base + (uint32_t((warp & 3) * 32) << 16) + Mode::SfCol, 0x7F7F7F7Fu);
  tc_fence_before();
  __syncthreads();
  if constexpr (kPair) cluster_sync_all();  // both CTAs' scale factors are in place before the first MMA
  tc_fence_after();

  const uint32_t n_kc = p.n_kc;
  const uint32_t n_items = __ldg(p.n_items);
  // an item slot is released to the leader's producer
  auto release_item_slot = [&](int s) {
    if (kPair && rank != 0) mbar_arrive_remote_relaxed(mapa_u32(iempty_bar(s), 0));
    else mbar_arrive(iempty_bar(s));
  };
  // One FIFO entry = 16 bytes {item id or kNone, tile, row_begin, row_end}: ordinary shared memory behind an
  // mbarrier in the CTA that draws the items.  The PEER's copy of the FIFO carries 8 bytes per slot, {item id,
  // hand-out number}, written through DSMEM with ONE 64-bit store (single-copy atomic) followed by a relaxed remote
  // arrive -- no cluster-scope fence on either side (a release / acquire pair at cluster scope is a
  // MEMBAR.ALL.GPU plus an L1 invalidate per item and waiting thread, on the producers' critical path).  Should the
  // arrive overtake the store (it does), the reader sees the slot's previous occupant, whose hand-out number
  // differs, and re-reads until the entry of this hand-out is there; the item itself it then loads from the plan.
  auto read_item = [&](int s, uint32_t parity, uint32_t seq, uint32_t& item, TcItem& it) {
    mbar_wait(ifull_bar(s), parity);
    if (kPair && rank != 0) {
      uint64_t e = ld_shared_volatile_b64(s_item_addr + 16u * s);
      while (static_cast<uint32_t>(e >> 32) != seq) e = ld_shared_volatile_b64(s_item_addr + 16u * s);
      item = static_cast<uint32_t>(e);
      it = item != kNone ? p.items[item] : TcItem{0, 0, 0, 0};
    } else {
      const uint4 e = ld_shared_volatile_v4(s_item_addr + 16u * s);
      item = e.x;
      it.tile = e.y;
      it.row_begin = e.z;
      it.row_end = e.w;
      it.pad = 0;
    }
  };

  if (warp == 0) {
    // ===== producer: two bulk copies per stage =====
    if (elect_one()) {
      uint32_t stage = 0, phase = 0, qslot = 0, qphase = 0;
      // L2 residency: a library strip (B) is read by the group's query tiles within one short window and is
      // then dead, while the group's query tiles (A) are re-read for every strip of the sweep.  Fetching B with
      // evict_first kept the streaming strips from pushing A out and paid 1.7 ... 3.7 % with the single-CTA kernel
      // of early round 2; with CTA pairs and lean issue threads it no longer changes the time (+-0.3 % on configs
      // 2, 3 and D = 1024 ... 16384) but costs DRAM traffic (strips evicted before the slowest pair has read them:
      // 9.0 vs 6.0 GB per launch on config 2, 240 vs 183 GB on the config-3 prefix), so both hints are off by
      // default (profiles/r02_ab_l2_hints_pair.log; HOMS_B200_TC_L2_HINTS bit 0 = A evict_last, bit 1 = B evict_first).
      const uint64_t pol_a = (p.l2_hints & 1u) ? l2_policy_evict_last() : l2_policy_evict_normal();
      const uint64_t pol_b = (p.l2_hints & 2u) ? l2_policy_evict_first() : l2_policy_evict_normal();
      // everything the inner loop needs lives in registers: no parameter reloads, no 64-bit multiplies per stage
      const uint64_t a_step = p.q_rows * kTcKB, b_step = p.lib_rows * kTcKB;  // bytes between k-chunk planes
      const uint8_t* const q_x = p.q_x;
      const uint8_t* const lib_x = p.lib_x;
      uint32_t next = rank == 0 ? atomicAdd(p.counter, 1u) : 0u;
      uint32_t iseq = 0;
      for (;;) {
        TcItem it{0, 0, 0, 0};
        uint32_t item;
        if (rank == 0) {
          item = next;
          mbar_wait(iempty_bar(qslot), qphase ^ 1u);
          if (item < n_items) it = p.items[item];
          const uint32_t id = item < n_items ? item : kNone;
          volatile uint32_t* e = s_item + 4 * qslot;
          e[0] = id;
          e[1] = it.tile;
          e[2] = it.row_begin;
          e[3] = it.row_end;
          mbar_arrive(ifull_bar(qslot));
          if constexpr (kPair) {
            st_remote_b64(mapa_u32(s_item_addr + 16u * qslot, 1), (uint64_t(iseq) << 32) | id);
            mbar_arrive_remote_relaxed(mapa_u32(ifull_bar(qslot), 1));
          }
        } else {  // the pair's second CTA follows the leader's FIFO
          read_item(qslot, qphase, iseq, item, it);
          release_item_slot(qslot);
          if (item == kNone) item = n_items;
        }
        ++iseq;
        if (++qslot == kItemQ) {
          qslot = 0;
          qphase ^= 1u;
        }
        if (item >= n_items) break;
        if (rank == 0) next = atomicAdd(p.counter, 1u);  // the next id arrives while this item streams
        const uint32_t n_nt = (it.row_end - it.row_begin + kN - 1) / kN;
        // own query rows: tile it.tile (single) or half `rank` of the 256-query tile it.tile (pair)
        const uint8_t* a_src = q_x + (uint64_t(it.tile) * Shape::TileQ + uint64_t(rank) * kTcM) * kTcKB;
        // own library rows: the whole N-row tile (single) or half `rank` of it (pair)
        const uint8_t* b_src = lib_x + (uint64_t(it.row_begin) + uint64_t(rank) * Shape::BRows) * kTcKB;
        // (An L2 prefetch of the next row tile's library block, cp.async.bulk.prefetch.L2 one k-chunk per stage by
        // every query tile or by one in eight, was measured 11-16 % SLOWER: profiles/r02_ab_l2_prefetch.log.)
        if constexpr (kARes) {  // the item's query chunks, once: when the previous item's MMAs have read theirs
          mbar_wait(aempty_bar, iseq & 1u);  // iseq = item number + 1: passes at once for the first item
          mbar_expect_tx(afull_bar, n_kc * kTcABytes);
          const uint8_t* ap = a_src;
          for (uint32_t kc = 0; kc < n_kc; ++kc, ap += a_step)
            bulk_g2s_hint(res_base + kc * kTcABytes, ap, kTcABytes, afull_bar, pol_a);
        }
        for (uint32_t nt = 0; nt < n_nt; ++nt, b_src += uint64_t(kN) * kTcKB) {
          const uint8_t* ap = a_src;
          const uint8_t* bp = b_src;
          for (uint32_t kc = 0; kc < n_kc; ++kc, ap += a_step, bp += b_step) {
            mbar_wait(empty_bar(stage), phase ^ 1u);
            const uint32_t sa = base + stage * Shape::StageBytes;
            const uint32_t fb = full_bar(stage);
            mbar_expect_tx(fb, Shape::StageBytes);
            if constexpr (!kARes) bulk_g2s_hint(sa, ap, kTcABytes, fb, pol_a);
            bulk_g2s_hint(sa + Shape::BOff, bp, Shape::BBytes, fb, pol_b);
            if (++stage == kStages) {
              stage = 0;
              phase ^= 1u;
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ===== MMA issuer: one thread (of the leader); in the peer the same thread relays "stage full" =====
    if (elect_one()) {
      uint32_t stage = 0, phase = 0, acc = 0, aphase = 0;  // aphase: one parity bit per accumulator
      uint32_t qslot = 0, qphase = 0, iseq = 0;
      for (;;) {
        uint32_t item;
        TcItem mit;
        read_item(qslot, qphase, iseq, item, mit);
        ++iseq;
        const uint32_t row_begin = mit.row_begin, row_end = mit.row_end;
        release_item_slot(qslot);
        if (++qslot == kItemQ) {
          qslot = 0;
          qphase ^= 1u;
        }
        if (item == kNone) break;
        const uint32_t n_nt = (row_end - row_begin + kN - 1) / kN;
        if (kPair && rank != 0) {  // relay: my share of stage s has landed -> the leader's pfull[s]
          for (uint32_t i = 0; i < n_nt * n_kc; ++i) {
            mbar_wait(full_bar(stage), phase);
            mbar_arrive_remote_relaxed(mapa_u32(pfull_bar(stage), 0));
            if (++stage == kStages) {
              stage = 0;
              phase ^= 1u;
            }
          }
          continue;
        }
        if constexpr (kARes) mbar_wait(afull_bar, (iseq & 1u) ^ 1u);  // this item's query chunks have landed
        for (uint32_t nt = 0; nt < n_nt; ++nt) {
          mbar_wait(tempty_bar(acc), ((aphase >> acc) & 1u) ^ 1u);  // drain warps released this accumulator
          aphase ^= 1u << acc;
          tc_fence_after();
          const uint32_t tmem_d = tmem_base + acc * kN;
          for (uint32_t kc = 0; kc < n_kc; ++kc) {
            mbar_wait(full_bar(stage), phase);
            if constexpr (kPair) mbar_wait(pfull_bar(stage), phase);  // the peer's share has landed in ITS shared memory
            tc_fence_after();
            const uint32_t sa = base + stage * Shape::StageBytes;
            const uint64_t adesc = tc_smem_desc(kARes ? res_base + kc * kTcABytes : sa);
            const uint64_t bdesc = tc_smem_desc(sa + Shape::BOff);
#pragma unroll
            for (uint32_t k = 0; k < kTcKB / 32; ++k) {  // +32 bytes along K inside the swizzle atom
              if constexpr (kPair)
                tc_mma_fp4_pair(tmem_d, adesc + 2 * k, bdesc + 2 * k, kTcIdescFp4Pair, tmem_base + Mode::SfCol,
                                tmem_base + Mode::SfCol + 16, (kc | k) != 0u);
              else
                tc_mma_fp4(tmem_d, adesc + 2 * k, bdesc + 2 * k, kTcIdescFp4, tmem_base + Mode::SfCol,
                           tmem_base + Mode::SfCol + 16, (kc | k) != 0u);
            }
            // stage reusable (in both CTAs) once these MMAs have read it
            if constexpr (kPair) tc_commit_pair(empty_bar(stage));
            else tc_commit(empty_bar(stage));
            if (++stage == kStages) {
              stage = 0;
              phase ^= 1u;
            }
          }
          // accumulator complete (in both CTAs)
          if constexpr (kPair) tc_commit_pair(tfull_bar(acc));
          else tc_commit(tfull_bar(acc));
          acc ^= 1u;
        }
        if constexpr (kARes) tc_commit(aempty_bar);  // the resident query chunks may be replaced
      }
    }
  } else {
    // ===== drain warps 2..5: TMEM -> running best per query =====
    // One pass over the accumulator, 32 columns per TMEM load, the next load in flight while the
    // current chunk is reduced.  Per chunk a thread takes the maximum of its query's valid columns
    // (1 MNMX per element); only when that maximum reaches `bar` -- the larger of the item's own
    // running best and `floor`, a lower bound of the query's final score published by work items
    // that finished earlier (gbest) -- does it look for the columns that hold it and apply the
    // exact tie-break.  Candidates below `floor` can never win, ties with it must be kept.
    const int quarter = warp & 3;  // a warp may only touch TMEM lanes [32 * (warp % 4), +32)
    const int qrow = quarter * 32 + lane;
    constexpr int kChunks = (kN + 31) / 32;
    uint32_t acc = 0, tphase = 0, qslot = 0, qphase = 0, iseq = 0;
    for (;;) {
      uint32_t item;
      TcItem it;
      read_item(qslot, qphase, iseq, item, it);
      ++iseq;
      __syncwarp();
      if (lane == 0) release_item_slot(qslot);
      if (++qslot == kItemQ) {
        qslot = 0;
        qphase ^= 1u;
      }
      if (item == kNone) break;
      const uint32_t n_nt = (it.row_end - it.row_begin + kN - 1) / kN;
      const uint64_t pos = uint64_t(it.tile) * Shape::TileQ + uint64_t(rank) * kTcM + qrow;
      uint32_t lf = 0, ll = 0;
      double qmz = 0.0;
      int floor_i = INT_MIN;
      if (pos < p.n) {
        const uint64_t key = p.keys[pos];
        if (key != ~0ull) {
          lf = static_cast<uint32_t>(key >> 32);
          ll = static_cast<uint32_t>(key);
        }
        const uint32_t slot = p.vals[pos];
        qmz = p.q_mz[p.subset ? p.subset[slot] : slot];
        if constexpr (kTopK || kCollect) {  // k dots of distinct candidates: the smallest bounds the final k-th best
          floor_i = INT_MAX;
          for (uint32_t j = 0; j < p.k; ++j) floor_i = min(floor_i, __ldcg(p.gbest + pos * p.k + j));
        } else {
          floor_i = __ldcg(p.gbest + pos);
        }
      }
      // pass > 0 of a deep top-k: everything up to and including the previous pass's last key is taken
      bool has_prev = false;
      int prev_dot = 0;
      uint64_t prev_ad = 0;
      uint32_t prev_rk = 0;
      if constexpr (kTopK) {
        if (p.prev != nullptr && pos < p.n) {
          const Cand pv = p.prev[uint64_t(p.vals[pos]) * p.prev_stride + p.prev_col];
          if (pv.d == kNone) {
            lf = ll = 0;  // the previous pass already ran out of candidates for this query
          } else {
            has_prev = true;
            prev_dot = static_cast<int>(p.dim) - 2 * static_cast<int>(pv.d);
            prev_ad = pv.ad;
            prev_rk = pv.rk;
          }
        }
      }
      AccT bar = Acc::from_int(floor_i);
      AccT best_dot = Acc::lowest();
      uint32_t best_row = kNone, best_rk = 0;
      uint64_t best_ad = 0;
      bool have_key = false;
      TcTopK<kList> topk;  // kTopK only
#pragma unroll
      for (int i = 0; i < kList; ++i) {
        topk.dot[i] = kTcNoDot;
        topk.row[i] = kNone;
      }
      uint32_t fresh = 0;  // kCollect: candidates appended since the floor was last read

      for (uint32_t nt = 0; nt < n_nt; ++nt) {
        const uint32_t row0 = it.row_begin + nt * kN;
        // this query's valid columns [c0, c1) of the tile
        int c0 = lf > row0 ? static_cast<int>(min(lf - row0, uint32_t(kN))) : 0;
        int c1 = ll > row0 ? static_cast<int>(min(ll - row0, uint32_t(kN))) : 0;
        if (c1 <= c0) c0 = c1 = 0;

        mbar_wait(tfull_bar(acc), (tphase >> acc) & 1u);
        tphase ^= 1u << acc;
        tc_fence_after();
        const uint32_t taddr = tmem_base + (uint32_t(quarter * 32) << 16) + acc * kN;

        auto reduce_chunk = [&](const int (&v)[32], int cb) {
          if constexpr (kCollect) {
            // While the floor is still weak a thread appends most of what it sees (the first tile of a query's
            // first item would append all 224 rows, and two or three of its items start at once: measured mean
            // 620 entries per query at k = 5, of which ~90 are needed).  Its own appends (and those of items
            // running elsewhere) have raised the class slots meanwhile: read them again, per chunk.
            if (fresh >= 4) {
              int f = INT_MAX;
              for (uint32_t j = 0; j < p.k; ++j) f = min(f, __ldcg(p.gbest + pos * p.k + j));
              bar = max(bar, Acc::from_int(f));
              fresh = 0;
            }
          }
          AccT cm = Acc::lowest();
          if (c0 <= cb && cb + 32 <= c1) {
#pragma unroll
            for (int j = 0; j < 32; ++j) cm = max(cm, Acc::get(v[j]));
          } else if (cb < c1 && cb + 32 > c0) {
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (cb + j >= c0 && cb + j < c1) cm = max(cm, Acc::get(v[j]));
          } else {
            return;
          }
          if (cm < bar) return;
          if constexpr (kCollect) {
            // Every valid column at or above the floor goes to the query's buffer; nothing else happens
            // here: no list, no tie-break loads, a few instructions per candidate.  The floor is the
            // smallest of k class maxima (class = row mod k), i.e. a dot that k DISTINCT rows of this
            // query's window reach, so the final k-th best dot can never be below it and every row
            // that ties with or beats the final k-th best is appended.  tc_select_kernel picks the exact
            // k best (full reference key) out of the buffer.
            uint32_t hits = 0;
#pragma unroll
            for (int j = 0; j < 32; ++j) hits |= (Acc::get(v[j]) >= bar ? 1u : 0u) << j;
            const int lo = max(c0 - cb, 0), hi = min(c1 - cb, 32);  // 0 <= lo < hi <= 32 here
            hits &= (hi >= 32 ? 0xffffffffu : (1u << hi) - 1u) & ~((1u << lo) - 1u);
            while (hits) {
              const int jj = __ffs(hits) - 1;
              hits &= hits - 1;
              AccT vj = Acc::lowest();
#pragma unroll
              for (int j = 0; j < 32; ++j)
                if (j == jj) vj = Acc::get(v[j]);
              const int dot = Acc::to_int(vj);
              const uint32_t r = row0 + cb + jj;
              const uint32_t idx = atomicAdd(p.ccount + pos, 1u);
              if (idx < p.ccap) p.cbuf[pos * p.ccap + idx] = make_uint2(static_cast<uint32_t>(dot), r);
              atomicMax(p.gbest + pos * p.k + r % p.k, dot);
              ++fresh;
            }
            return;
          }
          if constexpr (kTopK) {
            // every valid column at or above the bar is a candidate for the k best; the bar rises
            // to the list's k-th dot as soon as the list is full (ties with it must still be looked at)
            uint32_t hits = 0;
#pragma unroll
            for (int j = 0; j < 32; ++j) hits |= (Acc::get(v[j]) >= bar ? 1u : 0u) << j;
            const int lo = max(c0 - cb, 0), hi = min(c1 - cb, 32);  // 0 <= lo < hi <= 32 here
            hits &= (hi >= 32 ? 0xffffffffu : (1u << hi) - 1u) & ~((1u << lo) - 1u);
            while (hits) {
              const int jj = __ffs(hits) - 1;
              hits &= hits - 1;
              AccT vj = Acc::lowest();
#pragma unroll
              for (int j = 0; j < 32; ++j)
                if (j == jj) vj = Acc::get(v[j]);
              if (vj < bar) continue;  // the bar rose since the mask was taken
              if (has_prev) {
                const int dj = Acc::to_int(vj);
                if (dj > prev_dot) continue;  // ranked before the previous pass's last key: already reported
                if (dj == prev_dot) {
                  const uint32_t r = row0 + cb + jj;
                  const uint64_t ad = static_cast<uint64_t>(__double_as_longlong(fabs(qmz - p.lib_mz[r])));
                  if (!key_less(prev_ad, prev_rk, ad, p.lib_rank[r])) continue;
                }
              }
              tc_topk_insert<kList>(topk, p.lib_mz, p.lib_rank, qmz, Acc::to_int(vj), row0 + cb + jj);
              bar = max(bar, Acc::from_int(tc_topk_kth<kList>(topk, p.k)));
            }
            return;
          }
          uint32_t hits = 0;  // the columns that hold the chunk maximum
#pragma unroll
          for (int j = 0; j < 32; ++j) hits |= (Acc::get(v[j]) == cm ? 1u : 0u) << j;
          while (hits) {
            const int c = cb + __ffs(hits) - 1;
            hits &= hits - 1;
            if (c < c0 || c >= c1) continue;
            const uint32_t r = row0 + c;
            if (best_row == kNone || cm > best_dot) {
              best_dot = cm;
              best_row = r;
              have_key = false;
            } else {  // tie on score: |mass diff|, then id, then ordinal (search.cpp:137-145)
              if (!have_key) {
                best_ad = static_cast<uint64_t>(__double_as_longlong(fabs(qmz - p.lib_mz[best_row])));
                best_rk = p.lib_rank[best_row];
                have_key = true;
              }
              const uint64_t ad = static_cast<uint64_t>(__double_as_longlong(fabs(qmz - p.lib_mz[r])));
              const uint32_t rk = p.lib_rank[r];
              if (key_less(ad, rk, best_ad, best_rk)) {
                best_row = r;
                best_ad = ad;
                best_rk = rk;
              }
            }
          }
          if (best_row != kNone) bar = best_dot;
        };

        int va[32], vb[32];
        tc_ld32_issue(taddr, va);
        tc_ld_wait(va);
#pragma unroll 1
        for (int ch = 0; ch < kChunks; ch += 2) {
          if (ch + 1 < kChunks) tc_ld32_issue(taddr + (ch + 1) * 32, vb);
          reduce_chunk(va, ch * 32);
          if (ch + 1 < kChunks) {
            tc_ld_wait(vb);
            if (ch + 2 < kChunks) tc_ld32_issue(taddr + (ch + 2) * 32, va);
            reduce_chunk(vb, (ch + 1) * 32);
            if (ch + 2 < kChunks) tc_ld_wait(va);
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {  // the accumulator is released to the (leader's) MMA thread
          if (kPair && rank != 0) mbar_arrive_remote_relaxed(mapa_u32(tempty_bar(acc), 0));
          else mbar_arrive(tempty_bar(acc));
        }
        acc ^= 1u;
      }

      if constexpr (kCollect) continue;  // everything this item found is already in the query's buffer
      if constexpr (kTopK) {
        const uint32_t k = p.k;
        Cand* dst = p.partial + (uint64_t(item) * Shape::TileQ + rank * kTcM + qrow) * k;
#pragma unroll
        for (int j = 0; j < KM; ++j) {
          if (uint32_t(j) < k) {
            Cand out{kNone, kNone, ~0ull};
            const uint32_t r = topk.row[j];
            if (r != kNone) {
              out.d = static_cast<uint32_t>(static_cast<int>(p.dim) - topk.dot[j]) >> 1;  // dot = dim - 2 * distance
              out.rk = p.lib_rank[r];
              out.ad = static_cast<uint64_t>(__double_as_longlong(fabs(qmz - p.lib_mz[r])));
              // Publish: slot (row % k) of the query holds the best dot seen among the rows of that
              // residue class.  Classes are disjoint, so the k slots are dots of k distinct real
              // candidates and min(slots) can never exceed the final k-th best dot, under any
              // interleaving of the (fire-and-forget) atomicMax of concurrent items.
              if (topk.dot[j] > floor_i) atomicMax(p.gbest + pos * k + r % k, topk.dot[j]);
            }
            dst[j] = out;
          }
        }
        continue;
      }

      Cand out{kNone, kNone, ~0ull};
      if (best_row != kNone) {
        if (!have_key) {
          best_ad = static_cast<uint64_t>(__double_as_longlong(fabs(qmz - p.lib_mz[best_row])));
          best_rk = p.lib_rank[best_row];
        }
        const int dot = Acc::to_int(best_dot);
        if (dot > floor_i) atomicMax(p.gbest + pos, dot);  // raise the floor for later items
        // dot = dim - 2 * distance
        out.d = static_cast<uint32_t>(static_cast<int>(p.dim) - dot) >> 1;
        out.rk = best_rk;
        out.ad = best_ad;
      }
      p.partial[uint64_t(item) * Shape::TileQ + rank * kTcM + qrow] = out;
    }
  }

  tc_fence_before();
  __syncthreads();
  if constexpr (kPair) cluster_sync_all();  // no remote arrive or MMA of the pair is still under way
  if (warp == 1) {
    tc_fence_after();
    if constexpr (kPair)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(kTcTmemCols) : "memory");
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(kTcTmemCols) : "memory");
  }
}

// per sorted position: minimum over the items of its query tile.  One CTA per query tile,
// 128 positions x 8 item slices (a tile has a few hundred items), then a shared-memory fold.
constexpr int kTcReduceSlices = 8;
__global__ void __launch_bounds__(kTcM * kTcReduceSlices)
tc_reduce_kernel(uint64_t n, const uint32_t* __restrict__ vals, const uint32_t* __restrict__ tile_item_start,
                 const uint32_t* __restrict__ tile_items, const Cand* __restrict__ partial,
                 Cand* __restrict__ out, uint32_t k_stride, uint32_t tile_shift) {
  __shared__ Cand s_best[kTcReduceSlices][kTcM];
  const uint32_t t = blockIdx.x, r = threadIdx.x, slice = threadIdx.y;
  // planning tile (128 << tile_shift positions) and this block's 128-position part of it
  const uint32_t pt = t >> tile_shift, part = (t & ((1u << tile_shift) - 1u)) * kTcM;
  Cand best{kNone, kNone, ~0ull};
  // four records in flight per thread: the loop is a chain of dependent L2 round trips otherwise (53 us per
  // 16 000 queries, a quarter of everything a step does outside the search kernel)
  const uint32_t i_end = tile_item_start[pt + 1];
  for (uint32_t i = tile_item_start[pt] + slice; i < i_end; i += 4 * kTcReduceSlices) {
    Cand c[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint32_t iu = i + u * kTcReduceSlices;
      c[u] = iu < i_end ? partial[(uint64_t(tile_items[iu]) << tile_shift) * kTcM + part + r] : Cand{kNone, kNone, ~0ull};
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (c[u].d != best.d ? c[u].d < best.d : key_less(c[u].ad, c[u].rk, best.ad, best.rk)) best = c[u];
  }
  s_best[slice][r] = best;
  __syncthreads();
  const uint64_t pos = uint64_t(t) * kTcM + r;
  if (slice != 0 || pos >= n) return;
  for (int sl = 1; sl < kTcReduceSlices; ++sl) {
    const Cand c = s_best[sl][r];
    if (c.d != best.d ? c.d < best.d : key_less(c.ad, c.rk, best.ad, best.rk)) best = c;
  }
  out[uint64_t(vals[pos]) * k_stride] = best;
}

// top-k: per sorted position the k best of the (sorted) lists its query tile's items left
__global__ void tc_reduce_topk_kernel(uint64_t n, const uint32_t* __restrict__ vals,
                                      const uint32_t* __restrict__ tile_item_start,
                                      const uint32_t* __restrict__ tile_items, const Cand* __restrict__ partial,
                                      Cand* __restrict__ out, uint32_t k, uint32_t k_stride,
                                      const uint8_t* __restrict__ only, uint32_t tile_q) {
  const uint64_t pos = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (pos >= n) return;
  if (only != nullptr && !only[pos]) return;  // fix-up pass: this query already has its exact answer
  const uint32_t t = static_cast<uint32_t>(pos / tile_q), r = static_cast<uint32_t>(pos % tile_q);
  Cand best[kTcMaxK];  // k <= kTcMaxK per pass
  uint32_t count = 0;
  for (uint32_t i = tile_item_start[t]; i < tile_item_start[t + 1]; ++i) {
    const Cand* src = partial + (uint64_t(tile_items[i]) * tile_q + r) * k;
    for (uint32_t j = 0; j < k; ++j) {
      const Cand c = src[j];
      if (c.d == kNone) break;  // lists are sorted, empty entries last
      uint32_t m = count;
      if (m == k) {
        const Cand& w = best[k - 1];
        if (!(c.d != w.d ? c.d < w.d : key_less(c.ad, c.rk, w.ad, w.rk))) break;  // nor can the rest of this list
        --m;
      }
      uint32_t q = m;
      while (q > 0) {
        const Cand& b = best[q - 1];
        if (b.d != c.d ? b.d < c.d : key_less(b.ad, b.rk, c.ad, c.rk)) break;
        best[q] = b;
        --q;
      }
      best[q] = c;
      count = m + 1;
    }
  }
  Cand* dst = out + uint64_t(vals[pos]) * k_stride;
  for (uint32_t j = 0; j < k; ++j) dst[j] = j < count ? best[j] : Cand{kNone, kNone, ~0ull};
}

// ---- collect mode: exact selection ------------------------------------------------------------
// One warp per sorted position: the k best, by the full reference key, of the candidates the drain appended.
//   1. T = the k-th largest dot in the buffer (binary search on the value, counting with the whole warp);
//      everything below T is out, everything above it is in, rows with dot == T compete on (|dm|, id_rank).
//   2. the survivors (dot >= T; k plus the ties at T) are expanded to full 16-byte keys once, in shared
//      memory, and the k smallest are extracted in order.  A buffer with more survivors than the staging
//      area (degenerate libraries: thousands of equal scores) is extracted straight from global memory.
// A query whose buffer overflowed (ccount > ccap) is flagged and left to the fix-up pass of the caller.
constexpr int kSelWarps = 4;
constexpr uint32_t kSelStage = 256;  // survivors staged per warp (16 B each)
__global__ void __launch_bounds__(kSelWarps * 32)
tc_select_kernel(uint64_t n, const uint32_t* __restrict__ vals, const uint32_t* __restrict__ subset,
                 const uint32_t* __restrict__ ccount, const uint2* __restrict__ cbuf, uint32_t ccap, uint32_t k,
                 uint32_t k_stride, uint32_t dim, const double* __restrict__ q_mz,
                 const double* __restrict__ lib_mz, const uint32_t* __restrict__ lib_rank, Cand* __restrict__ out,
                 uint8_t* __restrict__ overflow) {
  __shared__ Cand s_stage[kSelWarps][kSelStage];
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t pos = uint64_t(blockIdx.x) * kSelWarps + warp;
  if (pos >= n) return;
  const uint32_t cnt = ccount[pos];
  if (cnt > ccap) {
    if (lane == 0) overflow[pos] = 1;
    return;
  }
  if (lane == 0) overflow[pos] = 0;
  const uint32_t slot = vals[pos];
  const double qmz = q_mz[subset ? subset[slot] : slot];
  const uint2* e = cbuf + pos * ccap;
  Cand* dst = out + uint64_t(slot) * k_stride;

  // 1. T
  int T = INT_MIN;
  if (cnt > k) {
    int lo = INT_MAX, hi = INT_MIN;
    for (uint32_t i = lane; i < cnt; i += 32) {
      const int d = static_cast<int>(e[i].x);
      lo = min(lo, d);
      hi = max(hi, d);
    }
    for (int o = 16; o > 0; o >>= 1) {
      lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
      hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    while (lo < hi) {  // largest v with count(dot >= v) >= k
      const int mid = lo + (hi - lo + 1) / 2;
      uint32_t c = 0;
      for (uint32_t i = lane; i < cnt; i += 32) c += static_cast<int>(e[i].x) >= mid ? 1u : 0u;
      c = __reduce_add_sync(0xffffffffu, c);
      if (c >= k) lo = mid;
      else hi = mid - 1;
    }
    T = lo;
  }
  // 2. survivors
  uint32_t m = 0;
  for (uint32_t i0 = 0; i0 < cnt; i0 += 32) {
    const uint32_t i = i0 + lane;
    const bool keep = i < cnt && static_cast<int>(e[i].x) >= T;
    const uint32_t mask = __ballot_sync(0xffffffffu, keep);
    if (keep) {
      const uint32_t at = m + __popc(mask & ((1u << lane) - 1u));
      if (at < kSelStage) {
        const uint32_t row = e[i].y;
        s_stage[warp][at] = Cand{static_cast<uint32_t>(static_cast<int>(dim) - static_cast<int>(e[i].x)) >> 1,
                                 lib_rank[row], static_cast<uint64_t>(__double_as_longlong(fabs(qmz - lib_mz[row])))};
      }
    }
    m += __popc(mask);
  }
  __syncwarp();
  Cand last{0, 0, 0};
  bool have_last = false;
  for (uint32_t j = 0; j < k; ++j) {
    Cand best{kNone, kNone, ~0ull};
    if (m <= kSelStage) {
      for (uint32_t i = lane; i < m; i += 32) {
        const Cand c = s_stage[warp][i];
        if (have_last && !(last.d != c.d ? last.d < c.d : key_less(last.ad, last.rk, c.ad, c.rk))) continue;
        if (c.d != best.d ? c.d < best.d : key_less(c.ad, c.rk, best.ad, best.rk)) best = c;
      }
    } else {  // too many survivors to stage: straight from the buffer, keys rebuilt on demand
      for (uint32_t i = lane; i < cnt; i += 32) {
        const int dot = static_cast<int>(e[i].x);
        if (dot < T) continue;
        const uint32_t d = static_cast<uint32_t>(static_cast<int>(dim) - dot) >> 1;
        if ((have_last && d < last.d) || d > best.d) continue;
        const uint32_t row = e[i].y;
        const Cand c{d, lib_rank[row], static_cast<uint64_t>(__double_as_longlong(fabs(qmz - lib_mz[row])))};
        if (have_last && !(last.d != c.d ? last.d < c.d : key_less(last.ad, last.rk, c.ad, c.rk))) continue;
        if (c.d != best.d ? c.d < best.d : key_less(c.ad, c.rk, best.ad, best.rk)) best = c;
      }
    }
    for (int o = 16; o > 0; o >>= 1) {
      Cand c;
      c.d = __shfl_xor_sync(0xffffffffu, best.d, o);
      c.rk = __shfl_xor_sync(0xffffffffu, best.rk, o);
      c.ad = __shfl_xor_sync(0xffffffffu, best.ad, o);
      if (c.d != best.d ? c.d < best.d : key_less(c.ad, c.rk, best.ad, best.rk)) best = c;
    }
    if (lane == 0) dst[j] = best;
    if (best.d == kNone) {  // fewer than k candidates: the rest is empty
      for (uint32_t jj = j + 1 + lane; jj < k; jj += 32) dst[jj] = Cand{kNone, kNone, ~0ull};
      break;
    }
    last = best;
    have_last = true;
  }
}

// fix-up pass of collect mode: only the flagged queries keep their window
__global__ void tc_mask_keys_kernel(uint64_t n, const uint64_t* __restrict__ keys, const uint8_t* __restrict__ flag,
                                    uint64_t* __restrict__ out) {
  const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) out[i] = flag[i] ? keys[i] : ~0ull;
}

// ---- host side --------------------------------------------------------------------------------

bool tc_available(const homs_b200_ctx* ctx) { return ctx->lib.d_x.p != nullptr && ctx->lib.x_rows > 0; }

static int expand_launch(homs_b200_ctx* ctx, uint64_t out_rows, uint64_t n_rows, const uint32_t* src_pos,
                         const uint32_t* src_subset, uint64_t pos_base, const uint64_t* words,
                         uint32_t stride_words, uint32_t dim, uint32_t n_kc, uint8_t* out) {
  const uint32_t groups = (n_kc + 3) / 4;
  const uint64_t warps = out_rows * groups;
  tc_expand_kernel<<<static_cast<unsigned>((warps * 32 + 255) / 256), 256, 0, ctx->stream>>>(
      out_rows, n_rows, src_pos, src_subset, pos_base, words, stride_words, dim, n_kc, out);
  HB_LAUNCHED(ctx);
  return HOMS_B200_OK;
}

int tc_expand_library(homs_b200_ctx* ctx) {
  Library& lib = ctx->lib;
  const uint32_t tile_n = TcMode::N;
  lib.n_kc = (lib.dim + TcMode::kDims - 1) / TcMode::kDims;
  lib.x_rows = (lib.n_local + tile_n - 1) / tile_n * tile_n + tile_n;
  HB_TRY(ensure(ctx, lib.d_x, size_t(lib.n_kc) * lib.x_rows * kTcKB));
  return expand_launch(ctx, lib.x_rows, lib.n_local, nullptr, nullptr, 0, lib.d_words.as<uint64_t>(), lib.S,
                       lib.dim, lib.n_kc, lib.d_x.as<uint8_t>());
}

// One planning batch (<= 64 Ki sorted slots): union windows, device plan, expanded queries.  Shared by
// every pass of a deep top-k over the batch.
struct TcBatch {
  uint64_t b0 = 0, nb = 0, q_rows = 0;
  uint32_t n_tiles = 0;  // planning tiles: 128 sorted positions each, 256 when CTA pairs run the search
  bool pair = false;
  bool ares = false;  // single CTAs with the query tile's k-chunks resident in shared memory (D <= 1024)
  TcPlanPtrs pp{};
};

// CTA pairs (TcShape<true>, cta_group::2) or one CTA per SM?  A pair moves a third fewer operand bytes per MMA
// (L2 -> shared memory and shared memory -> tensor core), which under the board's power cap is SM clock (+5 %), and
// its ring is 7 stages deep instead of 5 (ncu: tensor pipe 99.6 % active against 95.7 %); it pays with cross-CTA
// hand-offs per work item and row tile.  Interleaved A/B on one box (profiles/r02_ab_cta_pair_v2.log,
// r02_ab_cta_pair_threshold.log): D = 16384 -4.7 %, config-3 prefix -3.4 % (-7 % at D = 2048), config 2 -1.5 ... -2.3 %,
// D = 4096 -2 ... -6 %, D = 2048 -4 %, D = 1024 +4.8 % -- so pairs serve D >= 2048 when the device co-schedules a
// 2-CTA cluster on every SM pair (HOMS_B200_TC_PAIR=0 / 1 forces either form).
static bool tc_use_pair(const homs_b200_ctx* ctx);
constexpr uint32_t kTcPairMinKc = 8;  // k-chunks of 256 dimensions: D >= 2048
bool tc_uses_pairs(const homs_b200_ctx* ctx) { return tc_use_pair(ctx); }
static bool tc_use_pair(const homs_b200_ctx* ctx) {
  if (ctx->knobs.pair == 0 || ctx->tc_pair_ctas < 2) return false;
  if (ctx->knobs.pair == 1) return true;
  return ctx->lib.n_kc >= kTcPairMinKc && ctx->tc_pair_ctas + 1 >= ctx->sm_count;
}

// k_partial: list depth the per-item partial block is sized for (0: none, collect mode); reuse_qx: the
// expanded queries of this very batch are already in place (fix-up pass)
static int tc_prepare_batch(homs_b200_ctx* ctx, const uint32_t* d_subset, const uint64_t* d_keys,
                            const uint32_t* d_vals, uint64_t b0, uint64_t nb, uint32_t k_pass, uint32_t k_partial,
                            bool reuse_qx, TcBatch* out) {
  constexpr uint32_t kN = TcMode::N;
  const Library& lib = ctx->lib;
  const Queries& q = ctx->q;
  const TcKnobs& knobs = ctx->knobs;  // development knobs, read from the environment at ctx_create
  const bool pair = tc_use_pair(ctx);
  const uint32_t tile_q = pair ? TcShape<true>::TileQ : TcShape<false>::TileQ;
  const uint32_t n_tiles = static_cast<uint32_t>((nb + tile_q - 1) / tile_q);
  const uint64_t q_rows = uint64_t(n_tiles) * tile_q;

  // 1. union window of every query tile
  HB_TRY(ensure(ctx, ctx->scratch[kScrTcTiles], size_t(n_tiles) * sizeof(uint2)));
  auto* d_ranges = ctx->scratch[kScrTcTiles].as<uint2>();
  tc_tile_ranges_kernel<<<(n_tiles * 32 + 255) / 256, 256, 0, ctx->stream>>>(nb, d_keys + b0, n_tiles, tile_q, d_ranges);
  HB_LAUNCHED(ctx);

  // 2. plan on the device (see the planner above).  Capacity of the item arrays from what the
  //    host knows: every tile's window is at most the whole local library.
  TcPlanCfg pc;
  pc.n_tiles = n_tiles;
  // Query tiles per group.  A group's A operand (tiles x n_kc x 16 KB) is re-read for every strip of the
  // sweep, so it has to stay in L2 while the library strips stream through (fetched with an evict_first
  // hint, see the producer): 32 MB groups in general; when ALL query tiles of the batch fit in 64 MB they
  // form one group and every library strip is fetched from DRAM exactly once (config 2: 125 tiles = 62.5 MB,
  // DRAM 8.4 -> 5.9 GB per launch = 1.19x the compulsory bytes, 22.4 -> 21.6 ms; 64 MB groups on longer
  // query sets -- several groups, each sweeping the whole library -- measured 8 % slower than 32 MB:
  // profiles/r02_sweep_l2_hints_group.log)
  const uint64_t a_tile = uint64_t(tile_q) * lib.n_kc * kTcKB;
  uint64_t a_budget = uint64_t(n_tiles) * a_tile <= (64ull << 20) ? 64ull << 20 : 32ull << 20;
  if (knobs.group_mb) a_budget = uint64_t(knobs.group_mb) << 20;
  pc.group_tiles = static_cast<uint32_t>(std::max<uint64_t>(kTcGroupTiles, a_budget / a_tile));
  // Work-item length: about 400 items per SM of at most 8 row tiles keep co-running CTAs on neighbouring
  // tiles (L2 sharing) and the tail short.  An item also costs its drain warps 2-3 us of dependent global
  // loads (window, precursor, floor) before the first accumulator can be released; two 8.6 us row tiles hide
  // that at D = 8192, 1.1 us row tiles at D <= 1024 do not, so there items are 4x longer (interleaved A/B on
  // one box, profiles/r02_ab_item_sizing.log: D = 1024 3.18 -> 3.03 ms; D = 2048 and 4096 no gain, left alone).
  const bool short_k = lib.n_kc <= 4;
  pc.max_strip = short_k ? 32 : 8;
  uint32_t items_per_sm = short_k ? 100 : 400;
  if (knobs.group_tiles) pc.group_tiles = knobs.group_tiles;
  if (knobs.items_per_sm) items_per_sm = knobs.items_per_sm;
  if (knobs.max_strip) pc.max_strip = knobs.max_strip;
  pc.tiles_total = static_cast<uint32_t>((lib.n_local + kN - 1) / kN + 1);
  pc.target_items = uint64_t(pair ? ctx->tc_pair_ctas / 2 : ctx->sm_count) * items_per_sm;  // per CTA (pair)
  const uint64_t slack = 2ull * n_tiles + 16;
  const uint64_t by_shape =
      std::max<uint64_t>(pc.target_items, (uint64_t(n_tiles) * pc.tiles_total + pc.max_strip - 1) / pc.max_strip) + slack;
  const uint64_t by_memory = std::max<uint64_t>(
      (4ull << 30) / (size_t(tile_q) * std::max(1u, k_partial) * sizeof(Cand)), slack + 4ull * ctx->sm_count);
  pc.item_cap = static_cast<uint32_t>(std::min<uint64_t>(std::min(by_shape, by_memory), 0x7fffffffull));
  if (knobs.item_cap)  // development / test knob: force the capacity-bound plan
    pc.item_cap = static_cast<uint32_t>(std::min<uint64_t>(pc.item_cap, std::max<uint64_t>(slack + 1, knobs.item_cap)));
  pc.pad = 0;
  HB_TRY(ensure(ctx, ctx->scratch[kScrTcPlan], tc_plan_bytes(n_tiles, pc.item_cap)));
  void* d_plan = ctx->scratch[kScrTcPlan].p;
  static_assert(kTcBatch / kTcM <= kTcPlanThreads, "one planner thread per query tile");
  tc_plan_head_kernel<kN><<<1, kTcPlanThreads, 0, ctx->stream>>>(pc, d_ranges, d_plan);
  HB_LAUNCHED(ctx);
  tc_plan_items_kernel<kN><<<ctx->sm_count, 256, 0, ctx->stream>>>(pc, d_plan);
  HB_LAUNCHED(ctx);

  // 3. expand the batch's queries in sorted order
  if (!reuse_qx) {
    HB_TRY(ensure(ctx, ctx->scratch[kScrTcQx], size_t(lib.n_kc) * q_rows * kTcKB));
    HB_TRY(expand_launch(ctx, q_rows, nb, d_vals, d_subset, b0, q.d_words.as<uint64_t>(), stride_for(q.dim), q.dim,
                         lib.n_kc, ctx->scratch[kScrTcQx].as<uint8_t>()));
  }
  if (k_partial) HB_TRY(ensure(ctx, ctx->scratch[kScrTcPartial], size_t(pc.item_cap) * tile_q * k_partial * sizeof(Cand)));
  HB_TRY(ensure(ctx, ctx->scratch[kScrTcBest], q_rows * k_pass * sizeof(int)));
  out->b0 = b0;
  out->nb = nb;
  out->q_rows = q_rows;
  out->n_tiles = n_tiles;
  out->pair = pair;
  out->ares = !pair && lib.n_kc <= kTcAResChunks && ctx->knobs.ares != 0;
  out->pp = tc_plan_layout(d_plan, n_tiles, pc.item_cap);
  return HOMS_B200_OK;
}

// the search kernel over a prepared batch: one CTA per SM, or one 2-CTA cluster per SM pair
// HB_TC_PAIR = 0 compiles the CTA-pair form of the search kernel (TcShape<true>) out.
#ifndef HB_TC_PAIR
#define HB_TC_PAIR 1
#endif

template <int KM>
static int tc_launch_search(homs_b200_ctx* ctx, const TcBatch& tb, const TcParams& tp) {
  KernelTimer timer(ctx, HOMS_B200_KERNEL_SEARCH);
#if HB_TC_PAIR
  if (tb.pair) {
    using Shape = TcShape<true>;
    HB_CUDA(ctx, cudaFuncSetAttribute(tc_search_kernel<KM, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(Shape::SmemBytes)));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(ctx->tc_pair_ctas);
    cfg.blockDim = dim3(kTcThreads);
    cfg.dynamicSmemBytes = Shape::SmemBytes;
    cfg.stream = ctx->stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    HB_CUDA(ctx, cudaLaunchKernelEx(&cfg, tc_search_kernel<KM, true, false>, tp));
    return HOMS_B200_OK;
  }
#endif
  if (tb.ares) {
    using Shape = TcShape<false, true>;
    HB_CUDA(ctx, cudaFuncSetAttribute(tc_search_kernel<KM, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(Shape::SmemBytes)));
    tc_search_kernel<KM, false, true><<<ctx->sm_count, kTcThreads, Shape::SmemBytes, ctx->stream>>>(tp);
  } else {
    using Shape = TcShape<false>;
    HB_CUDA(ctx, cudaFuncSetAttribute(tc_search_kernel<KM, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(Shape::SmemBytes)));
    tc_search_kernel<KM, false, false><<<ctx->sm_count, kTcThreads, Shape::SmemBytes, ctx->stream>>>(tp);
  }
  return HOMS_B200_OK;
}

// co-resident 2-CTA clusters of the search kernel x 2 (0: pairs cannot be scheduled); asked once per context
int tc_query_pair_ctas(homs_b200_ctx* ctx) {
#if !HB_TC_PAIR
  (void)ctx;
  return 0;
#else
  using Shape = TcShape<true>;
  if (cudaFuncSetAttribute(tc_search_kernel<1, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(Shape::SmemBytes)) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(ctx->sm_count / 2 * 2);
  cfg.blockDim = dim3(kTcThreads);
  cfg.dynamicSmemBytes = Shape::SmemBytes;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int clusters = 0;
  if (cudaOccupancyMaxActiveClusters(&clusters, tc_search_kernel<1, true, false>, &cfg) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return std::min(clusters, ctx->sm_count / 2) * 2;
#endif
}

// One pass over a prepared batch: the k best per query (k <= KM) -- after the key in column prev_col of
// the output when prev_col != kNone -- into columns [col0, col0 + k) of d_out_full.
template <int KM>
static int tc_run_pass(homs_b200_ctx* ctx, const TcBatch& tb, const uint32_t* d_subset, const uint64_t* d_keys,
                       const uint32_t* d_vals, Cand* d_out_full, uint32_t k_stride, uint32_t col0, uint32_t k,
                       uint32_t prev_col, const uint8_t* d_only = nullptr) {
  using Mode = TcMode;
  const Library& lib = ctx->lib;
  const Queries& q = ctx->q;
  const TcPlanPtrs& pp = tb.pp;
  if (prev_col != kNone)  // a later pass over the same plan: hand the work items out again
    HB_CUDA(ctx, cudaMemsetAsync(&pp.head->counter, 0, sizeof(uint32_t), ctx->stream));
  // every byte 0x80: a dot no candidate can be below
  HB_CUDA(ctx, cudaMemsetAsync(ctx->scratch[kScrTcBest].p, 0x80, tb.q_rows * k * sizeof(int), ctx->stream));

  // 4. search + reduce
  TcParams tp;
  tp.lib_x = lib.d_x.as<uint8_t>();
  tp.q_x = ctx->scratch[kScrTcQx].as<uint8_t>();
  tp.lib_rows = lib.x_rows;
  tp.q_rows = tb.q_rows;
  tp.n_kc = lib.n_kc;
  tp.dim = lib.dim;
  tp.items = pp.items;
  tp.n_items = &pp.head->n_items;
  tp.counter = &pp.head->counter;
  tp.keys = d_keys + tb.b0;
  tp.vals = d_vals + tb.b0;
  tp.subset = d_subset;
  tp.q_mz = q.d_mz.as<double>();
  tp.lib_mz = lib.d_mz_local.as<double>();
  tp.lib_rank = lib.d_id_rank_local.as<uint32_t>();
  tp.n = tb.nb;
  tp.partial = ctx->scratch[kScrTcPartial].as<Cand>();
  tp.gbest = ctx->scratch[kScrTcBest].as<int>();
  tp.k = k;
  tp.prev = prev_col != kNone ? d_out_full : nullptr;
  tp.prev_stride = k_stride;
  tp.prev_col = prev_col;
  tp.l2_hints = ctx->knobs.l2_hints;
  tp.ccount = nullptr;
  tp.cbuf = nullptr;
  tp.ccap = 0;
  tp.pad3 = 0;
  HB_TRY(tc_launch_search<KM>(ctx, tb, tp));
  HB_LAUNCHED(ctx);
  if constexpr (KM > 1)
    tc_reduce_topk_kernel<<<static_cast<unsigned>((tb.nb + 127) / 128), 128, 0, ctx->stream>>>(
        tb.nb, d_vals + tb.b0, pp.tile_start, pp.tile_items, ctx->scratch[kScrTcPartial].as<Cand>(), d_out_full + col0,
        k, k_stride, d_only, tb.pair ? TcShape<true>::TileQ : TcShape<false>::TileQ);
  else
    tc_reduce_kernel<<<static_cast<unsigned>((tb.nb + kTcM - 1) / kTcM), dim3(kTcM, kTcReduceSlices), 0, ctx->stream>>>(
        tb.nb, d_vals + tb.b0, pp.tile_start, pp.tile_items, ctx->scratch[kScrTcPartial].as<Cand>(), d_out_full + col0,
        k_stride, tb.pair ? 1u : 0u);
  HB_LAUNCHED(ctx);
  return HOMS_B200_OK;
}

uint32_t tc_max_topk() { return HOMS_B200_MAX_TOPK; }  // any k the ABI allows

// The register-list passes: ceil(k / 32) passes of up to 32 candidates per query over a prepared batch.
static int tc_list_passes(homs_b200_ctx* ctx, const TcBatch& tb, const uint32_t* d_subset, const uint64_t* d_keys,
                          const uint32_t* d_vals, Cand* d_out, uint32_t k, uint32_t k_stride, const uint8_t* d_only) {
  for (uint32_t col0 = 0; col0 < k; col0 += kTcMaxK) {
    const uint32_t kr = std::min<uint32_t>(kTcMaxK, k - col0);
    const uint32_t prev_col = col0 ? col0 - 1 : kNone;
    // a later pass needs the top-k drain (it is the one that knows about the lower bound), even for kr = 1
    if (kr == 1 && col0 == 0) HB_TRY(tc_run_pass<1>(ctx, tb, d_subset, d_keys, d_vals, d_out, k_stride, col0, kr, prev_col));
    else if (kr <= 4) HB_TRY(tc_run_pass<4>(ctx, tb, d_subset, d_keys, d_vals, d_out, k_stride, col0, kr, prev_col, d_only));
    else if (kr <= 8) HB_TRY(tc_run_pass<8>(ctx, tb, d_subset, d_keys, d_vals, d_out, k_stride, col0, kr, prev_col, d_only));
    else if (kr <= 16) HB_TRY(tc_run_pass<16>(ctx, tb, d_subset, d_keys, d_vals, d_out, k_stride, col0, kr, prev_col, d_only));
    else HB_TRY(tc_run_pass<kTcMaxK>(ctx, tb, d_subset, d_keys, d_vals, d_out, k_stride, col0, kr, prev_col, d_only));
  }
  return HOMS_B200_OK;
}

// Collect mode (k >= 2): ONE pass whose drain only appends the candidates at or above each query's floor to
// a per-query buffer, tc_select_kernel for the exact k best, then a fix-up run of the list passes restricted
// to the queries whose buffer overflowed (none, unless thousands of rows tie at the top of a window: the
// fix-up plan is then empty and its kernels return at once).  Everything stays stream-ordered.
static int tc_collect_batch(homs_b200_ctx* ctx, const uint32_t* d_subset, const uint64_t* d_keys,
                            const uint32_t* d_vals, uint64_t* d_keys_fix, uint64_t b0, uint64_t nb, Cand* d_out,
                            uint32_t k, uint32_t k_stride, uint32_t ccap) {
  using Mode = TcMode;
  const Library& lib = ctx->lib;
  const Queries& q = ctx->q;
  TcBatch tb;
  HB_TRY(tc_prepare_batch(ctx, d_subset, d_keys, d_vals, b0, nb, k, 0, false, &tb));
  HB_TRY(ensure(ctx, ctx->scratch[kScrTcCount], tb.q_rows * sizeof(uint32_t)));
  HB_TRY(ensure(ctx, ctx->scratch[kScrTcBuf], tb.q_rows * size_t(ccap) * sizeof(uint2)));
  HB_TRY(ensure(ctx, ctx->scratch[kScrTcOverflow], tb.q_rows));
  HB_CUDA(ctx, cudaMemsetAsync(ctx->scratch[kScrTcCount].p, 0, tb.q_rows * sizeof(uint32_t), ctx->stream));
  HB_CUDA(ctx, cudaMemsetAsync(ctx->scratch[kScrTcBest].p, 0x80, tb.q_rows * k * sizeof(int), ctx->stream));
  TcParams tp{};
  tp.lib_x = lib.d_x.as<uint8_t>();
  tp.q_x = ctx->scratch[kScrTcQx].as<uint8_t>();
  tp.lib_rows = lib.x_rows;
  tp.q_rows = tb.q_rows;
  tp.n_kc = lib.n_kc;
  tp.dim = lib.dim;
  tp.items = tb.pp.items;
  tp.n_items = &tb.pp.head->n_items;
  tp.counter = &tb.pp.head->counter;
  tp.keys = d_keys + b0;
  tp.vals = d_vals + b0;
  tp.subset = d_subset;
  tp.q_mz = q.d_mz.as<double>();
  tp.lib_mz = lib.d_mz_local.as<double>();
  tp.lib_rank = lib.d_id_rank_local.as<uint32_t>();
  tp.n = nb;
  tp.partial = nullptr;
  tp.gbest = ctx->scratch[kScrTcBest].as<int>();
  tp.k = k;
  tp.prev = nullptr;
  tp.prev_stride = k_stride;
  tp.prev_col = kNone;
  tp.l2_hints = ctx->knobs.l2_hints;
  tp.ccount = ctx->scratch[kScrTcCount].as<uint32_t>();
  tp.cbuf = ctx->scratch[kScrTcBuf].as<uint2>();
  tp.ccap = ccap;
  tp.pad3 = 0;
  HB_TRY(tc_launch_search<0>(ctx, tb, tp));
  HB_LAUNCHED(ctx);
  if (ctx->knobs.debug) {  // development: how full did the candidate buffers get?
    std::vector<uint32_t> h(nb);
    cudaMemcpyAsync(h.data(), tp.ccount, nb * sizeof(uint32_t), cudaMemcpyDeviceToHost, ctx->stream);
    cudaStreamSynchronize(ctx->stream);
    uint64_t sum = 0, over = 0;
    uint32_t mx = 0;
    for (uint32_t c : h) {
      sum += c;
      mx = std::max(mx, c);
      over += c > ccap;
    }
    std::sort(h.begin(), h.end());
    fprintf(stderr, "[tc collect] k=%u ccap=%u queries=%llu mean=%.1f p50=%u p99=%u max=%u overflowed=%llu\n", k, ccap,
            (unsigned long long)nb, double(sum) / double(nb), h[nb / 2], h[nb - 1 - nb / 100], mx, (unsigned long long)over);
  }
  auto* d_over = ctx->scratch[kScrTcOverflow].as<uint8_t>();
  tc_select_kernel<<<static_cast<unsigned>((nb + kSelWarps - 1) / kSelWarps), kSelWarps * 32, 0, ctx->stream>>>(
      nb, d_vals + b0, d_subset, tp.ccount, tp.cbuf, ccap, k, k_stride, lib.dim, q.d_mz.as<double>(),
      lib.d_mz_local.as<double>(), lib.d_id_rank_local.as<uint32_t>(), d_out, d_over);
  HB_LAUNCHED(ctx);
  // fix-up: the exact list passes over the flagged queries only (their windows survive in d_keys_fix)
  tc_mask_keys_kernel<<<static_cast<unsigned>((nb + 255) / 256), 256, 0, ctx->stream>>>(nb, d_keys + b0, d_over,
                                                                                      d_keys_fix + b0);
  HB_LAUNCHED(ctx);
  TcBatch fix;
  HB_TRY(tc_prepare_batch(ctx, d_subset, d_keys_fix, d_vals, b0, nb, std::min<uint32_t>(k, kTcMaxK),
                          std::min<uint32_t>(k, kTcMaxK), true, &fix));
  return tc_list_passes(ctx, fix, d_subset, d_keys_fix, d_vals, d_out, k, k_stride, d_over);
}

int tc_search_sorted(homs_b200_ctx* ctx, const uint32_t* d_subset, uint64_t n, const uint64_t* d_keys,
                     const uint32_t* d_vals, Cand* d_out, uint32_t k, uint32_t k_stride) {
  HB_REQUIRE(ctx, k >= 1 && k <= HOMS_B200_MAX_TOPK, HOMS_B200_ERR_ARGUMENT, "tensor engine: k out of range");
  // Collect + select serves every k >= 2 (one pass; interleaved A/B against the register-list passes on config 2,
  // ms per 16 000-query step, lists -> collect: k = 2: 22.8 -> 22.5, k = 5: 24.4 -> 23.3, k = 8: 25.4 -> 23.2,
  // k = 16: 28.3 -> 24.1, k = 64: 113.8 -> 31.6; profiles/r02_ab_topk_collect_vs_lists_v2.log).  The register
  // lists remain as the fix-up for overflowed buffers and behind HOMS_B200_TC_TOPK=lists.
  const bool collect = k >= 2 && ctx->knobs.topk_lists != 1;
  if (collect) {
    // buffer capacity per query: the floor admits about k x H(k) x ln(window / strip) candidates plus what the
    // first, floor-less items append (measured counts: DESIGN.md K4a); batches sized for <= 1 GB of buffers
    const uint32_t ccap = ctx->knobs.ccap ? ctx->knobs.ccap : std::min(8192u, std::max(2048u, 128u * k));
    uint64_t batch = std::max<uint64_t>(kTcM, ((1ull << 30) / (uint64_t(ccap) * sizeof(uint2))) / kTcM * kTcM);
    batch = std::min<uint64_t>(batch, kTcBatch);
    HB_TRY(ensure(ctx, ctx->scratch[kScrTcKeysFix], n * sizeof(uint64_t)));
    for (uint64_t b0 = 0; b0 < n; b0 += batch)
      HB_TRY(tc_collect_batch(ctx, d_subset, d_keys, d_vals, ctx->scratch[kScrTcKeysFix].as<uint64_t>(), b0,
                              std::min<uint64_t>(batch, n - b0), d_out, k, k_stride, ccap));
    return HOMS_B200_OK;
  }
  const uint32_t k_pass = std::min<uint32_t>(k, kTcMaxK);
  for (uint64_t b0 = 0; b0 < n; b0 += kTcBatch) {
    TcBatch tb;
    HB_TRY(tc_prepare_batch(ctx, d_subset, d_keys, d_vals, b0, std::min<uint64_t>(kTcBatch, n - b0), k_pass, k_pass,
                            false, &tb));
    HB_TRY(tc_list_passes(ctx, tb, d_subset, d_keys, d_vals, d_out, k, k_stride, nullptr));
    // the next batch reuses the plan / operand / partial blocks: stream order keeps that safe
  }
  return HOMS_B200_OK;
}

// ---- tensor-pipe ceiling probe ----------------------------------------------------------------
// The issue loop of tc_search_kernel with everything else removed: one thread per SM issues the same
// MMA shape back to back on whatever bytes shared memory holds (no global traffic, no drain), in
// groups of 4 per commit with `depth` groups in flight.  bench.py times it on the same box in the same run and
// reports the search kernel against it: MEASURED_PEAKS.json holds a bf16 figure only, and the
// sustained rate of the 4-bit kind under the power cap is not a fixed multiple of it.
__global__ void __launch_bounds__(kTcThreads, 1) tc_peak_kernel(uint32_t groups) {
  using Mode = TcMode;
  constexpr int kN = Mode::N;
  constexpr int kDepth = 4;
  extern __shared__ unsigned char tc_smem_raw[];
  const uint32_t raw = smem_u32(tc_smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  unsigned char* gen_base = tc_smem_raw + (base - raw);
  const uint32_t bar0 = base + Mode::Stages * Mode::StageBytes;
  volatile uint32_t* tmem_slot =
      reinterpret_cast<volatile uint32_t*>(gen_base + Mode::Stages * Mode::StageBytes + 8 * kDepth);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // operands: any finite pattern will do; e2m1 has no NaN or Inf encodings
  for (uint32_t i = threadIdx.x; i < Mode::StageBytes / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(gen_base)[i] = make_uint4(0x2A2A2A2Au, 0xA2A2A2A2u, 0x22AA22AAu, 0xAAAA2222u);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x == 0) {
    for (int s = 0; s < kDepth; ++s) mbar_init(bar0 + 8u * s, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(const_cast<uint32_t*>(tmem_slot))),
                 "r"(kTcTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (warp >= 2) tc_st32_fill(tmem_base + (uint32_t((warp & 3) * 32) << 16) + Mode::SfCol, 0x7F7F7F7Fu);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1 && elect_one()) {
    const uint64_t adesc = tc_smem_desc(base);
    const uint64_t bdesc = tc_smem_desc(base + kTcABytes);
    for (uint32_t g = 0; g < groups; ++g) {
      const uint32_t slot = g % kDepth;
      if (g >= kDepth) mbar_wait(bar0 + 8u * slot, ((g / kDepth) - 1u) & 1u);
      const uint32_t tmem_d = tmem_base + (g & 1u) * kN;
#pragma unroll
      for (uint32_t k = 0; k < kTcKB / 32; ++k)
        tc_mma_fp4(tmem_d, adesc + 2 * k, bdesc + 2 * k, kTcIdescFp4, tmem_base + Mode::SfCol,
                   tmem_base + Mode::SfCol + 16, 1u);
      tc_commit(bar0 + 8u * slot);
    }
    for (uint32_t g = groups > kDepth ? groups - kDepth : 0; g < groups; ++g)
      mbar_wait(bar0 + 8u * (g % kDepth), (g / kDepth) & 1u);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(kTcTmemCols)
                 : "memory");
  }
}

int tc_peak_probe(homs_b200_ctx* ctx, double seconds, double* out_ops_per_s, double* out_ms) {
  using Mode = TcMode;
  HB_CUDA(ctx, cudaFuncSetAttribute(tc_peak_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(Mode::SmemBytes)));
  cudaEvent_t e0, e1;
  HB_CUDA(ctx, cudaEventCreate(&e0));
  HB_CUDA(ctx, cudaEventCreate(&e1));
  // ops of one group: 4 MMAs of M128 x N x (32 bytes of K)
  const double ops_group = 2.0 * kTcM * Mode::N * Mode::kDims;
  uint32_t groups = 1u << 14;
  float ms = 0.f;
  for (int pass = 0; pass < 3; ++pass) {  // calibrate, warm (reach the power-capped clock), measure
    HB_CUDA(ctx, cudaEventRecord(e0, ctx->stream));
    tc_peak_kernel<<<ctx->sm_count, kTcThreads, Mode::SmemBytes, ctx->stream>>>(groups);
    HB_LAUNCHED(ctx);
    HB_CUDA(ctx, cudaEventRecord(e1, ctx->stream));
    HB_CUDA(ctx, cudaEventSynchronize(e1));
    HB_CUDA(ctx, cudaEventElapsedTime(&ms, e0, e1));
    if (pass == 0) {
      const double want = seconds * 1e3 / std::max(1e-3f, ms) * groups;
      groups = static_cast<uint32_t>(std::min(want, 4.0e9));
      groups = std::max(groups, 1u << 10);
    }
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  *out_ops_per_s = ops_group * groups * ctx->sm_count / (ms * 1e-3);
  if (out_ms) *out_ms = ms;
  return HOMS_B200_OK;
}

}  // namespace hb
