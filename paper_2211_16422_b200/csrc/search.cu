// Windowed Hamming top-k search for sm_100a.
//
// Reference semantics (paths under /root/reference/proj/core/):
//   Tolerance::window_at/accepts  include/homs/search.hpp:23-30
//   select_candidates             src/search.cpp:62-89
//   row_similarity / search_one   src/search.cpp:93-169
//   search_batch                  src/search.cpp:171-183
//   run_stage / cascade_search    src/search.cpp:188-248
//
// Pipeline of one search call (all on the context's stream, no host round trip):
//   1. bounds_kernel      K3: per query, two binary searches of the exact fp64 predicates
//                         (q - r > w) and (r - q > w) over the bucket's sorted precursor m/z.
//   2. radix sort         queries ordered by window start + end (= by precursor m/z inside a bucket), so
//                         neighbours share reference rows and a tile of queries has a tight union window.
//   3. plan_*_kernel      groups QB consecutive queries into a block, takes the union of their
//                         windows, cuts it into row chunks -> work items (device-side, no sync).
//   4. search_kernel      K4: persistent CTAs pull work items from an atomic counter.  A CTA
//                         streams its row chunk through a 4-stage cp.async ring of 256-row x
//                         64-byte tiles (XOR-swizzled, conflict-free LDS.128), one thread per
//                         reference row; the QB query vectors sit in shared memory and are read
//                         as warp broadcasts; distances accumulate with XOR + POPC.  Each thread
//                         keeps the best row per query (exact 3-level key), the CTA reduces with
//                         warp shuffles and writes one 16-byte candidate per query.
//   5. reduce_kernel      per query lexicographic minimum over the work items of its block.
// Top-k (k > 1) repeats 4-5 with the previous round's key as an exclusive lower bound, which
// yields exactly the k smallest keys in order.

#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>

#include "common.cuh"
#include "radix.cuh"
#include "topk.cuh"

namespace hb {

constexpr int kTileRows = 256;    // threads per CTA == reference rows per tile
constexpr int kChunkBytes = 64;   // bytes of every row per pipeline stage
constexpr int kStages = 4;
constexpr int kStageBytes = kTileRows * kChunkBytes;

__device__ __forceinline__ bool cand_less(uint32_t d1, uint64_t ad1, uint32_t rk1, uint32_t d2,
                                          uint64_t ad2, uint32_t rk2) {
  if (d1 != d2) return d1 < d2;
  if (ad1 != ad2) return ad1 < ad2;
  return rk1 < rk2;
}

__device__ __forceinline__ uint64_t abs_diff_bits(double q, double r) {
  return static_cast<uint64_t>(__double_as_longlong(fabs(q - r)));  // search.cpp:127
}

// ------------------------------------------------------------------------------------------
// K3: candidate windows
// ------------------------------------------------------------------------------------------

__global__ void bounds_kernel(uint64_t n, const uint32_t* __restrict__ subset,
                              const double* __restrict__ q_mz, const uint8_t* __restrict__ q_charge,
                              uint32_t tol_kind, double tol_value, const double* __restrict__ lib_mz,
                              const BucketDev* __restrict__ buckets,
                              const int32_t* __restrict__ bucket_of_charge,
                              uint64_t* __restrict__ out_first, uint64_t* __restrict__ out_last,
                              uint8_t* __restrict__ out_has, uint64_t* __restrict__ keys,
                              uint32_t* __restrict__ vals) {
  const uint64_t s = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (s >= n) return;
  const uint64_t qi = subset ? subset[s] : s;
  const double q = q_mz[qi];
  const uint8_t c = q_charge[qi];
  const int32_t bi = c == 0 ? -1 : bucket_of_charge[c];  // search.cpp:65-67
  uint64_t first = 0, last = 0;
  uint64_t key = ~0ull;
  if (bi >= 0) {
    const BucketDev b = buckets[bi];
    const double* mzs = lib_mz + b.begin;
    const double w = tol_kind == HOMS_B200_TOL_PPM ? tol_value * q * 1e-6 : tol_value;  // search.hpp:24
    uint64_t lo = b.size, hi = b.size;
    if (q == q && w == w) {  // a NaN on either side accepts nothing (search.hpp:29)
      // accepts(q, r) <=> !(q - r > w) && !(r - q > w); both predicates are monotone along the
      // sorted bucket, so the accepted rows are exactly [lo, hi) -- the run search.cpp:77-83
      // arrives at by extend/trim.
      uint64_t a = 0, len = b.size;
      while (len > 0) {
        const uint64_t half = len >> 1;
        if (q - mzs[a + half] > w) {
          a += half + 1;
          len -= half + 1;
        } else {
          len = half;
        }
      }
      lo = a;
      len = b.size - lo;
      while (len > 0) {
        const uint64_t half = len >> 1;
        if (mzs[a + half] - q > w) {
          len = half;
        } else {
          a += half + 1;
          len -= half + 1;
        }
      }
      hi = a;
    }
    first = lo;
    last = hi;
    const uint64_t cl = min(max(lo, b.shard_begin), b.shard_end);
    const uint64_t ch = min(max(hi, b.shard_begin), b.shard_end);
    if (ch > cl) {
      const uint64_t lf = cl - b.shard_begin + b.local_offset;
      const uint64_t ll = ch - b.shard_begin + b.local_offset;
      key = (lf << 32) | ll;
    }
  }
  if (out_first) out_first[s] = first;
  if (out_last) out_last[s] = last;
  if (out_has) out_has[s] = bi >= 0;
  keys[s] = key;
  vals[s] = static_cast<uint32_t>(s);
}

// ------------------------------------------------------------------------------------------
// planning
// ------------------------------------------------------------------------------------------

struct PlanHeader {
  uint32_t chunk_rows;
  uint32_t n_items;
  uint32_t counter;
  uint32_t pad;
};

__global__ void plan_blocks_kernel(uint64_t n, uint32_t qb, const uint64_t* __restrict__ keys,
                                   uint32_t n_blocks, uint32_t* __restrict__ blk_lo,
                                   uint32_t* __restrict__ blk_rows) {
  const uint32_t b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= n_blocks) return;
  uint32_t lo = kNone, hi = 0;
  for (uint32_t j = 0; j < qb; ++j) {
    const uint64_t p = uint64_t(b) * qb + j;
    if (p >= n) break;
    const uint64_t key = keys[p];
    if (key == ~0ull) continue;
    lo = min(lo, static_cast<uint32_t>(key >> 32));
    hi = max(hi, static_cast<uint32_t>(key));
  }
  blk_lo[b] = lo == kNone ? 0 : lo;
  blk_rows[b] = hi > lo && lo != kNone ? hi - lo : 0;
}

// single CTA: chunk size, items per block, exclusive scan
__global__ void __launch_bounds__(1024)
plan_items_kernel(uint32_t n_blocks, uint32_t target_items, const uint32_t* __restrict__ blk_rows,
                  uint32_t* __restrict__ item_start, PlanHeader* __restrict__ hdr) {
  __shared__ unsigned long long s_total;
  __shared__ uint32_t s_scan[1024];
  __shared__ uint32_t s_carry;
  const uint32_t tid = threadIdx.x;
  if (tid == 0) {
    s_total = 0;
    s_carry = 0;
  }
  __syncthreads();
  unsigned long long local = 0;
  for (uint32_t b = tid; b < n_blocks; b += blockDim.x) local += blk_rows[b];
  atomicAdd(&s_total, local);
  __syncthreads();
  const unsigned long long total = s_total;
  unsigned long long chunk = (total + target_items - 1) / target_items;
  chunk = (chunk + kTileRows - 1) / kTileRows * kTileRows;
  if (chunk < 4 * kTileRows) chunk = 4 * kTileRows;
  if (chunk > 0x40000000ull) chunk = 0x40000000ull;
  const uint32_t chunk_rows = static_cast<uint32_t>(chunk);

  for (uint32_t base = 0; base < n_blocks; base += blockDim.x) {
    const uint32_t b = base + tid;
    const uint32_t items = b < n_blocks ? (blk_rows[b] + chunk_rows - 1) / chunk_rows : 0;
    s_scan[tid] = items;
    __syncthreads();
    for (uint32_t off = 1; off < blockDim.x; off <<= 1) {  // Hillis-Steele inclusive scan
      const uint32_t v = tid >= off ? s_scan[tid - off] : 0;
      __syncthreads();
      s_scan[tid] += v;
      __syncthreads();
    }
    const uint32_t carry = s_carry;
    if (b < n_blocks) item_start[b] = carry + s_scan[tid] - items;
    __syncthreads();
    if (tid == blockDim.x - 1) s_carry = carry + s_scan[tid];
    __syncthreads();
  }
  if (tid == 0) {
    item_start[n_blocks] = s_carry;
    hdr->chunk_rows = chunk_rows;
    hdr->n_items = s_carry;
    hdr->counter = 0;
  }
}

__global__ void reset_counter_kernel(PlanHeader* hdr) { hdr->counter = 0; }

// ------------------------------------------------------------------------------------------
// K4: the search kernel
// ------------------------------------------------------------------------------------------

__device__ __forceinline__ void cp_async16(uint32_t smem_addr, const void* gptr) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_addr), "l"(gptr));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

struct SearchParams {
  const uint64_t* lib_words;      // local rows, padded stride
  const double* lib_mz;           // local rows
  const uint32_t* lib_rank;       // local rows
  const uint64_t* q_words;        // resident queries, padded stride
  const double* q_mz;
  const uint32_t* subset;         // nullable
  const uint64_t* keys;           // sorted (lf << 32 | ll)
  const uint32_t* vals;           // sorted slot indices
  const uint32_t* blk_lo;
  const uint32_t* blk_rows;
  const uint32_t* item_start;
  PlanHeader* hdr;
  const Cand* prev;               // [n][k] output so far; round r reads entry r-1 (nullable)
  Cand* partial;                  // [n_items][QB]
  uint64_t n;                     // slots
  uint32_t n_blocks;
  uint32_t row_bytes;             // padded row size in bytes (multiple of 128)
  uint32_t k, round;
};

template <int QB>
__global__ void __launch_bounds__(kTileRows, 2) search_kernel(const SearchParams p) {
  extern __shared__ __align__(128) unsigned char smem[];
  unsigned char* s_ref = smem;                                   // kStages * kStageBytes
  unsigned char* s_q = smem + kStages * kStageBytes;             // QB * row_bytes
  unsigned char* s_meta = s_q + size_t(QB) * p.row_bytes;
  uint32_t* s_lf = reinterpret_cast<uint32_t*>(s_meta);          // [QB]
  uint32_t* s_ll = s_lf + QB;                                    // [QB]
  uint32_t* s_qi = s_ll + QB;                                    // [QB] resident query index
  uint32_t* s_pd = s_qi + QB;                                    // [QB] prev distance
  uint32_t* s_prk = s_pd + QB;                                   // [QB] prev id_rank
  uint32_t* s_flag = s_prk + QB;                                 // [QB] 1: has prev
  double* s_qmz = reinterpret_cast<double*>(s_flag + QB);        // [QB]
  uint64_t* s_pad = reinterpret_cast<uint64_t*>(s_qmz + QB);     // [QB] prev abs diff
  Cand* s_red = reinterpret_cast<Cand*>(s_pad + QB);             // [8 warps][QB]
  __shared__ uint32_t s_item;

  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const uint32_t row_bytes = p.row_bytes;
  const uint32_t row_u4 = row_bytes / 16;
  const uint32_t kch = row_bytes / kChunkBytes;
  const uint32_t s_ref_addr = static_cast<uint32_t>(__cvta_generic_to_shared(s_ref));
  const uint32_t s_q_addr = static_cast<uint32_t>(__cvta_generic_to_shared(s_q));
  const unsigned char* lib_bytes = reinterpret_cast<const unsigned char*>(p.lib_words);
  const unsigned char* q_bytes = reinterpret_cast<const unsigned char*>(p.q_words);
  const uint32_t chunk_rows = p.hdr->chunk_rows;
  const uint32_t n_items = p.hdr->n_items;

  for (;;) {
    __syncthreads();  // previous item fully retired (smem reuse, s_item)
    if (tid == 0) s_item = atomicAdd(&p.hdr->counter, 1u);
    __syncthreads();
    const uint32_t item = s_item;
    if (item >= n_items) break;

    // item -> (query block, chunk): last block whose item_start <= item
    uint32_t lo_b = 0, hi_b = p.n_blocks;
    while (hi_b - lo_b > 1) {
      const uint32_t mid = (lo_b + hi_b) >> 1;
      if (p.item_start[mid] <= item) lo_b = mid;
      else hi_b = mid;
    }
    const uint32_t blk = lo_b;
    const uint32_t row_lo = p.blk_lo[blk] + (item - p.item_start[blk]) * chunk_rows;
    const uint32_t row_hi = min(row_lo + chunk_rows, p.blk_lo[blk] + p.blk_rows[blk]);

    if (tid < QB) {
      const uint64_t pos = uint64_t(blk) * QB + tid;
      uint32_t lf = 0, ll = 0, qi = 0, flag = 0, pd = 0, prk = 0;
      uint64_t pad = 0;
      double qmz = 0.0;
      if (pos < p.n) {
        const uint64_t key = p.keys[pos];
        const uint32_t slot = p.vals[pos];
        qi = p.subset ? p.subset[slot] : slot;
        qmz = p.q_mz[qi];
        if (key != ~0ull) {
          lf = static_cast<uint32_t>(key >> 32);
          ll = static_cast<uint32_t>(key);
        }
        if (p.round > 0) {
          const Cand pv = p.prev[uint64_t(slot) * p.k + (p.round - 1)];
          flag = 1;
          pd = pv.d;
          prk = pv.rk;
          pad = pv.ad;
          if (pv.d == kNone) ll = lf;  // nothing left for this query
        }
      }
      s_lf[tid] = lf;
      s_ll[tid] = ll;
      s_qi[tid] = qi;
      s_pd[tid] = pd;
      s_prk[tid] = prk;
      s_flag[tid] = flag;
      s_qmz[tid] = qmz;
      s_pad[tid] = pad;
    }
    __syncthreads();

    // query vectors -> shared memory (joins the first cp.async group)
    for (uint32_t idx = tid; idx < QB * row_u4; idx += kTileRows) {
      const uint32_t qq = idx / row_u4, u = idx - qq * row_u4;
      if (s_ll[qq] > s_lf[qq])
        cp_async16(s_q_addr + idx * 16, q_bytes + size_t(s_qi[qq]) * row_bytes + size_t(u) * 16);
    }

    const uint32_t n_rows = row_hi - row_lo;
    const uint32_t n_tiles = (n_rows + kTileRows - 1) / kTileRows;
    const uint32_t total = n_tiles * kch;

    auto load_stage = [&](uint32_t s) {
      const uint32_t t = s / kch, kc = s - t * kch;
      const uint32_t row0 = row_lo + t * kTileRows;
      const uint32_t buf = s_ref_addr + (s % kStages) * kStageBytes;
#pragma unroll
      for (int i = 0; i < kChunkBytes / 16; ++i) {
        const uint32_t idx = tid + i * kTileRows;
        const uint32_t r = idx >> 2, c = idx & 3;
        const uint32_t grow = min(row0 + r, row_hi - 1);
        cp_async16(buf + r * kChunkBytes + ((c ^ ((r >> 1) & 3)) << 4),
                   lib_bytes + size_t(grow) * row_bytes + size_t(kc) * kChunkBytes + c * 16);
      }
    };

    uint32_t acc[QB], best_d[QB], best_row[QB];
#pragma unroll
    for (int q = 0; q < QB; ++q) {
      acc[q] = 0;
      best_d[q] = kNone;
      best_row[q] = kNone;
    }

#pragma unroll
    for (int s = 0; s < kStages - 1; ++s) {
      if (static_cast<uint32_t>(s) < total) load_stage(s);
      cp_async_commit();
    }

    for (uint32_t s = 0; s < total; ++s) {
      cp_async_wait<kStages - 2>();
      __syncthreads();
      if (s + kStages - 1 < total) load_stage(s + kStages - 1);
      cp_async_commit();

      const uint32_t t = s / kch, kc = s - t * kch;
      const uint4* rrow = reinterpret_cast<const uint4*>(s_ref + (s % kStages) * kStageBytes +
                                                         tid * kChunkBytes);
      const uint4* qbase = reinterpret_cast<const uint4*>(s_q) + kc * (kChunkBytes / 16);
      const int sw = (tid >> 1) & 3;
#pragma unroll
      for (int c = 0; c < kChunkBytes / 16; ++c) {
        const uint4 r = rrow[c ^ sw];
#pragma unroll
        for (int q = 0; q < QB; ++q) {
          const uint4 w = qbase[q * row_u4 + c];  // warp-uniform address: broadcast
          acc[q] += __popc(r.x ^ w.x) + __popc(r.y ^ w.y) + __popc(r.z ^ w.z) + __popc(r.w ^ w.w);
        }
      }

      if (kc == kch - 1) {  // the row's distance to every query of the block is complete
        const uint32_t row = row_lo + t * kTileRows + tid;
        const bool row_ok = row < row_hi;
#pragma unroll
        for (int q = 0; q < QB; ++q) {
          const uint32_t d = acc[q];
          acc[q] = 0;
          if (!row_ok || row < s_lf[q] || row >= s_ll[q]) continue;
          if (s_flag[q]) {  // top-k round > 0: only keys strictly above the previous pick
            const uint32_t pd = s_pd[q];
            if (d < pd) continue;
            if (d == pd) {
              const uint64_t ad = abs_diff_bits(s_qmz[q], p.lib_mz[row]);
              if (!cand_less(pd, s_pad[q], s_prk[q], d, ad, p.lib_rank[row])) continue;
            }
          }
          if (d < best_d[q]) {
            best_d[q] = d;
            best_row[q] = row;
          } else if (d == best_d[q]) {  // tie on score: |mass diff|, then id, then ordinal
            const double qm = s_qmz[q];
            const uint32_t br = best_row[q];
            if (cand_less(d, abs_diff_bits(qm, p.lib_mz[row]), p.lib_rank[row], d,
                          abs_diff_bits(qm, p.lib_mz[br]), p.lib_rank[br]))
              best_row[q] = row;
          }
        }
      }
    }
    cp_async_wait<0>();

    // CTA-wide lexicographic minimum per query
#pragma unroll
    for (int q = 0; q < QB; ++q) {
      uint32_t d = best_d[q], rk = kNone;
      uint64_t ad = ~0ull;
      if (d != kNone) {
        ad = abs_diff_bits(s_qmz[q], p.lib_mz[best_row[q]]);
        rk = p.lib_rank[best_row[q]];
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const uint32_t d2 = __shfl_xor_sync(0xffffffffu, d, o);
        const uint32_t rk2 = __shfl_xor_sync(0xffffffffu, rk, o);
        const uint64_t ad2 = __shfl_xor_sync(0xffffffffu, ad, o);
        if (cand_less(d2, ad2, rk2, d, ad, rk)) {
          d = d2;
          ad = ad2;
          rk = rk2;
        }
      }
      if (lane == 0) s_red[warp * QB + q] = Cand{d, rk, ad};
    }
    __syncthreads();
    if (tid < QB) {
      Cand best = s_red[tid];
      for (int w = 1; w < kTileRows / 32; ++w) {
        const Cand c = s_red[w * QB + tid];
        if (cand_less(c.d, c.ad, c.rk, best.d, best.ad, best.rk)) best = c;
      }
      p.partial[uint64_t(item) * QB + tid] = best;
    }
  }
}

// per query: minimum over the work items of its block
__global__ void reduce_kernel(uint64_t n, uint32_t qb, const uint32_t* __restrict__ vals,
                              const uint32_t* __restrict__ item_start, const Cand* __restrict__ partial,
                              Cand* __restrict__ out, uint32_t k, uint32_t round) {
  const uint64_t pos = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (pos >= n) return;
  const uint32_t b = static_cast<uint32_t>(pos / qb), j = static_cast<uint32_t>(pos % qb);
  Cand best{kNone, kNone, ~0ull};
  for (uint32_t it = item_start[b]; it < item_start[b + 1]; ++it) {
    const Cand c = partial[uint64_t(it) * qb + j];
    if (cand_less(c.d, c.ad, c.rk, best.d, best.ad, best.rk)) best = c;
  }
  out[uint64_t(vals[pos]) * k + round] = best;
}

// k-way merge of per-shard sorted candidate lists
__global__ void merge_kernel(uint64_t n, uint32_t k, uint32_t n_parts, const Cand* __restrict__ parts,
                             Cand* __restrict__ out) {
  const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint32_t head[64];
  for (uint32_t s = 0; s < n_parts; ++s) head[s] = 0;
  for (uint32_t j = 0; j < k; ++j) {
    Cand best{kNone, kNone, ~0ull};
    uint32_t from = kNone;
    for (uint32_t s = 0; s < n_parts; ++s) {
      if (head[s] >= k) continue;
      const Cand c = parts[(uint64_t(s) * n + i) * k + head[s]];
      if (c.d == kNone) continue;
      if (from == kNone || cand_less(c.d, c.ad, c.rk, best.d, best.ad, best.rk)) {
        best = c;
        from = s;
      }
    }
    if (from != kNone) ++head[from];
    out[i * k + j] = best;
  }
}

__global__ void decode_kernel(uint64_t total, const Cand* __restrict__ rec, uint32_t dim,
                              const uint32_t* __restrict__ ord_of_rank, uint32_t* __restrict__ score,
                              uint32_t* __restrict__ ordinal) {
  const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= total) return;
  const Cand c = rec[i];
  if (c.d == kNone) {
    score[i] = 0;
    ordinal[i] = HOMS_B200_NO_HIT;
  } else {
    score[i] = dim - c.d;  // search.cpp:100
    ordinal[i] = ord_of_rank[c.rk];
  }
}

// ------------------------------------------------------------------------------------------
// host side
// ------------------------------------------------------------------------------------------

// ------------------------------------------------------------------------------------------
// K4c: direct engine -- one warp per query, for windows of a few dozen rows
// ------------------------------------------------------------------------------------------
// The tensor engine's cost has a floor of one pass over the library image per call (every query
// tile's union window, summed over the tiles, covers the library once: 0.7 ms on config 2 however
// narrow the tolerance).  A 20 ppm window holds ~25 rows: reading exactly those rows (neighbouring
// sorted queries share them in L2) is an order of magnitude less traffic.  k <= 64 (32 per pass).

// KM = 1: running best; KM > 1: the k <= KM best in a register list every lane holds identically
// (the comparisons are warp-uniform) -- the warp-level top-k with the reference's tie-break.
constexpr uint32_t kDirectMaxK = 32;  // list depth of one pass; deeper top-k takes ceil(k / 32) passes
// LPR = 0: a row spans the warp (row_u4 lanes of every 32 at a time).  LPR = 8 / 16: rows of exactly LPR 16-byte
// slabs (D <= 1024 / D <= 2048): 32 / LPR rows side by side in the warp, so that every lane loads and four
// passes keep 16 / 8 rows in flight instead of 4 (at D = 1024 three quarters of the lanes used to idle and the
// kernel was bound by the latency of 23 dependent rounds per 90-row window).
template <int KM, int LPR>
__global__ void __launch_bounds__(256)
direct_search_kernel(uint64_t n, const uint64_t* __restrict__ keys, const uint32_t* __restrict__ vals,
                     const uint32_t* __restrict__ subset, const uint4* __restrict__ q_words,
                     const double* __restrict__ q_mz, const uint4* __restrict__ lib_words,
                     const double* __restrict__ lib_mz, const uint32_t* __restrict__ lib_rank, uint32_t row_u4,
                     Cand* __restrict__ out, uint32_t k, uint32_t k_stride, uint32_t col0, uint32_t prev_col) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t pos = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (pos >= n) return;
  const uint64_t key = keys[pos];
  const uint32_t slot = vals[pos];
  const uint32_t qi = subset ? subset[slot] : slot;
  uint32_t lf = 0, ll = 0;
  if (key != ~0ull) {
    lf = static_cast<uint32_t>(key >> 32);
    ll = static_cast<uint32_t>(key);
  }
  const double qmz = q_mz[qi];
  const uint4* q = q_words + size_t(qi) * row_u4;
  // pass > 0 of a deep top-k (KM > 1 only): keys up to and including out[slot][prev_col] are taken
  bool has_prev = false;
  uint32_t prev_d = 0, prev_rk = 0;
  uint64_t prev_ad = 0;
  if (prev_col != kNone) {
    const Cand pv = out[uint64_t(slot) * k_stride + prev_col];
    if (pv.d == kNone) {
      lf = ll = 0;  // the previous pass already ran out of candidates
    } else {
      has_prev = true;
      prev_d = pv.d;
      prev_rk = pv.rk;
      prev_ad = pv.ad;
    }
  }
  uint32_t best_d = kNone, best_rk = kNone, best_row = kNone;
  uint64_t best_ad = ~0ull;
  bool have_key = false;
  TcTopK<KM> topk;  // KM > 1 only; "dot" = -distance
  int kth = kTcNoDot;
#pragma unroll
  for (int i = 0; i < KM; ++i) {
    topk.dot[i] = kTcNoDot;
    topk.row[i] = kNone;
  }

  auto consider = [&](uint32_t row, uint32_t d) {  // warp-uniform
    if constexpr (KM > 1) {
      const int dot = -static_cast<int>(d);
      if (dot < kth) return;  // below the k-th best so far (ties with it are looked at)
      if (has_prev) {
        if (d < prev_d) return;  // ranked before the previous pass's last key: already reported
        if (d == prev_d && !key_less(prev_ad, prev_rk, abs_diff_bits(qmz, lib_mz[row]), lib_rank[row])) return;
      }
      tc_topk_insert<KM>(topk, lib_mz, lib_rank, qmz, dot, row);
      kth = tc_topk_kth<KM>(topk, k);
      return;
    }
    if (d < best_d) {
      best_d = d;
      best_row = row;
      have_key = false;
    } else if (d == best_d) {  // tie on score: |mass diff|, then id, then ordinal (search.cpp:137-145)
      if (!have_key) {
        best_ad = abs_diff_bits(qmz, lib_mz[best_row]);
        best_rk = lib_rank[best_row];
        have_key = true;
      }
      const uint64_t ad = abs_diff_bits(qmz, lib_mz[row]);
      const uint32_t rk = lib_rank[row];
      if (cand_less(d, ad, rk, d, best_ad, best_rk)) {
        best_row = row;
        best_ad = ad;
        best_rk = rk;
      }
    }
  };

  uint32_t r = lf;
  if constexpr (LPR != 0) {
    constexpr uint32_t kRpp = 32 / LPR;  // rows per pass
    const uint32_t sub = lane / LPR, sl = lane % LPR;
    const uint4 a = q[sl];
    for (; r < ll; r += 4 * kRpp) {  // four passes in flight per lane
      uint32_t c[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t row = r + j * kRpp + sub;
        uint4 x = a;  // a row past the window: distance 0, never looked at
        if (row < ll) x = __ldg(lib_words + size_t(row) * LPR + sl);
        c[j] = __popc(a.x ^ x.x) + __popc(a.y ^ x.y) + __popc(a.z ^ x.z) + __popc(a.w ^ x.w);
      }
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int o = LPR / 2; o > 0; o >>= 1) c[j] += __shfl_xor_sync(0xffffffffu, c[j], o);
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (uint32_t sb = 0; sb < kRpp; ++sb) {
          const uint32_t d = __shfl_sync(0xffffffffu, c[j], sb * LPR);
          const uint32_t row = r + j * kRpp + sb;
          if (row < ll) consider(row, d);
        }
    }
    r = ll;
  }
  for (; r + 4 <= ll; r += 4) {  // four rows in flight per lane
    uint32_t c0 = 0, c1 = 0, c2 = 0, c3 = 0;
    const uint4* b = lib_words + size_t(r) * row_u4;
    for (uint32_t u = lane; u < row_u4; u += 32) {
      const uint4 a = q[u];
      const uint4 x0 = __ldg(b + u), x1 = __ldg(b + row_u4 + u), x2 = __ldg(b + 2 * size_t(row_u4) + u),
                  x3 = __ldg(b + 3 * size_t(row_u4) + u);
      c0 += __popc(a.x ^ x0.x) + __popc(a.y ^ x0.y) + __popc(a.z ^ x0.z) + __popc(a.w ^ x0.w);
      c1 += __popc(a.x ^ x1.x) + __popc(a.y ^ x1.y) + __popc(a.z ^ x1.z) + __popc(a.w ^ x1.w);
      c2 += __popc(a.x ^ x2.x) + __popc(a.y ^ x2.y) + __popc(a.z ^ x2.z) + __popc(a.w ^ x2.w);
      c3 += __popc(a.x ^ x3.x) + __popc(a.y ^ x3.y) + __popc(a.z ^ x3.z) + __popc(a.w ^ x3.w);
    }
    consider(r, __reduce_add_sync(0xffffffffu, c0));
    consider(r + 1, __reduce_add_sync(0xffffffffu, c1));
    consider(r + 2, __reduce_add_sync(0xffffffffu, c2));
    consider(r + 3, __reduce_add_sync(0xffffffffu, c3));
  }
  for (; r < ll; ++r) {
    uint32_t c0 = 0;
    const uint4* b = lib_words + size_t(r) * row_u4;
    for (uint32_t u = lane; u < row_u4; u += 32) {
      const uint4 a = q[u];
      const uint4 x0 = __ldg(b + u);
      c0 += __popc(a.x ^ x0.x) + __popc(a.y ^ x0.y) + __popc(a.z ^ x0.z) + __popc(a.w ^ x0.w);
    }
    consider(r, __reduce_add_sync(0xffffffffu, c0));
  }
  if (lane != 0) return;
  Cand* dst = out + uint64_t(slot) * k_stride + col0;
  if constexpr (KM > 1) {
#pragma unroll
    for (int j = 0; j < KM; ++j) {
      if (uint32_t(j) < k) {
        Cand c{kNone, kNone, ~0ull};
        const uint32_t row = topk.row[j];
        if (row != kNone)
          c = Cand{static_cast<uint32_t>(-topk.dot[j]), lib_rank[row], abs_diff_bits(qmz, lib_mz[row])};
        dst[j] = c;
      }
    }
    return;
  }
  Cand c{kNone, kNone, ~0ull};
  if (best_row != kNone) {
    if (!have_key) {
      best_ad = abs_diff_bits(qmz, lib_mz[best_row]);
      best_rk = lib_rank[best_row];
    }
    c = Cand{best_d, best_rk, best_ad};
  }
  dst[0] = c;
}

// Expected candidate rows per query for this tolerance, from the library's own m/z distribution
// (queries are assumed to be distributed like the library): 16 probe points per bucket.
static double expected_window_rows(const Library& lib, const homs_b200_tolerance* tol) {
  double acc = 0.0;
  for (const BucketDev& b : lib.buckets) {
    if (b.size == 0) continue;
    const double* m = lib.h_mz.data() + b.begin;
    double rows = 0.0;
    for (int j = 0; j < 16; ++j) {
      const double c = m[b.size * (2 * j + 1) / 32];
      const double w = tol->kind == HOMS_B200_TOL_PPM ? tol->value * c * 1e-6 : tol->value;
      rows += static_cast<double>(std::upper_bound(m, m + b.size, c + w) - std::lower_bound(m, m + b.size, c - w));
    }
    acc += rows / 16.0 * static_cast<double>(b.size);
  }
  return lib.n ? acc / static_cast<double>(lib.n) : 0.0;
}

// AUTO: the direct engine when the rows it would read are far fewer bytes than the tensor engine's
// floor of one pass over the library image per planning batch (measured crossover, profiles/)
static bool direct_is_cheaper(const homs_b200_ctx* ctx, uint64_t n, const homs_b200_tolerance* tol) {
  const Library& lib = ctx->lib;
  const double share = lib.n ? static_cast<double>(lib.n_local) / static_cast<double>(lib.n) : 1.0;
  const double direct_bytes = expected_window_rows(lib, tol) * share * static_cast<double>(n) * lib.S * 8.0;
  const double batches = static_cast<double>((n + 65535) / 65536);
  const double tensor_bytes = static_cast<double>(lib.n_kc) * static_cast<double>(lib.x_rows) * 128.0 * batches;
  return direct_bytes < tensor_bytes;  // measured crossover on config 2: 4.0 M pairs 0.64 vs 0.75 ms, 27 M pairs 3.5 vs 0.72 ms
}

static int pick_qb(uint32_t row_bytes) {
  if (row_bytes <= 2048) return 16;
  if (row_bytes <= 4096) return 8;
  if (row_bytes <= 8192) return 4;
  return 0;
}

static size_t search_smem(int qb, uint32_t row_bytes) {
  return size_t(kStages) * kStageBytes + size_t(qb) * row_bytes + size_t(qb) * (6 * 4 + 2 * 8) +
         size_t(kTileRows / 32) * qb * sizeof(Cand);
}

template <int QB>
static int launch_search(homs_b200_ctx* ctx, const SearchParams& sp, int grid) {
  const size_t smem = search_smem(QB, sp.row_bytes);
  HB_CUDA(ctx, cudaFuncSetAttribute(search_kernel<QB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(smem)));
  {
    KernelTimer timer(ctx, HOMS_B200_KERNEL_SEARCH);
    search_kernel<QB><<<grid, kTileRows, smem, ctx->stream>>>(sp);
  }
  HB_LAUNCHED(ctx);
  return HOMS_B200_OK;
}

static int check_tol(homs_b200_ctx* ctx, const homs_b200_tolerance* tol) {
  HB_REQUIRE(ctx, tol != nullptr, HOMS_B200_ERR_ARGUMENT, "tolerance is null");
  HB_REQUIRE(ctx, tol->kind == HOMS_B200_TOL_PPM || tol->kind == HOMS_B200_TOL_DALTON,
             HOMS_B200_ERR_ARGUMENT, "tolerance kind must be ppm (0) or dalton (1)");
  return HOMS_B200_OK;
}

// bounds for n slots of the resident query arrays (or explicit device arrays)
static int run_bounds(homs_b200_ctx* ctx, uint64_t n, const uint32_t* d_subset, const double* d_qmz,
                      const uint8_t* d_qcharge, const homs_b200_tolerance* tol, uint64_t* d_first,
                      uint64_t* d_last, uint8_t* d_has) {
  const Library& lib = ctx->lib;
  HB_TRY(ensure(ctx, ctx->scratch[kScrKeys], n * 8));
  HB_TRY(ensure(ctx, ctx->scratch[kScrVals], n * 4));
  bounds_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, ctx->stream>>>(
      n, d_subset, d_qmz, d_qcharge, tol->kind, tol->value, lib.d_mz.as<double>(),
      lib.d_buckets.as<BucketDev>(), lib.d_bucket_of_charge.as<int32_t>(), d_first, d_last, d_has,
      ctx->scratch[kScrKeys].as<uint64_t>(), ctx->scratch[kScrVals].as<uint32_t>());
  HB_LAUNCHED(ctx);
  return HOMS_B200_OK;
}

// Full device pipeline for n slots; writes n*k candidates to d_out.
int search_dev_locked(homs_b200_ctx* ctx, const uint32_t* d_subset, uint64_t n,
                             const homs_b200_tolerance* tol, uint32_t k, Cand* d_out,
                             uint64_t* d_first, uint64_t* d_last, uint8_t* d_has) {
  const Library& lib = ctx->lib;
  const Queries& q = ctx->q;
  HB_REQUIRE(ctx, lib.ready, HOMS_B200_ERR_STATE, "search: no library uploaded");
  HB_REQUIRE(ctx, q.ready, HOMS_B200_ERR_STATE, "search: no queries resident");
  HB_TRY(check_tol(ctx, tol));
  HB_REQUIRE(ctx, k >= 1 && k <= HOMS_B200_MAX_TOPK, HOMS_B200_ERR_ARGUMENT, "search: k must be in [1, 64]");
  // search.cpp:107-109
  HB_REQUIRE(ctx, q.dim == lib.dim, HOMS_B200_ERR_INVARIANT,
             "search_one: query dimensionality does not match index");
  if (n == 0) return HOMS_B200_OK;
  HB_REQUIRE(ctx, n <= 0x7FFFFFFFull, HOMS_B200_ERR_ARGUMENT, "search: more than 2^31-1 queries in one call");
  const uint32_t row_bytes = lib.S * 8;
  const int qb = pick_qb(row_bytes);
  HB_REQUIRE(ctx, qb != 0, HOMS_B200_ERR_ARGUMENT, "search: dim above 65536 is not supported");

  HB_TRY(run_bounds(ctx, n, d_subset, q.d_mz.as<double>(), q.d_charge.as<uint8_t>(), tol, d_first,
                    d_last, d_has));

  const bool tensor_ok = ctx->engine != HOMS_B200_ENGINE_POPC && ctx->engine != HOMS_B200_ENGINE_DIRECT && tc_available(ctx);
  const bool use_direct = ctx->engine == HOMS_B200_ENGINE_DIRECT ||
                          (ctx->engine == HOMS_B200_ENGINE_AUTO && tensor_ok && direct_is_cheaper(ctx, n, tol));
  // Sort the slots by window position: neighbours then share library rows on chip.
  // The direct engine skips it when the windows are so sparse that neighbours would share nothing
  // anyway (expected rows read < rows resident: every row comes from HBM once either way).
  const bool sparse = use_direct && expected_window_rows(lib, tol) * static_cast<double>(n) < static_cast<double>(lib.n);
  const uint64_t* keys = ctx->scratch[kScrKeys].as<uint64_t>();
  const uint32_t* vals = ctx->scratch[kScrVals].as<uint32_t>();
  if (!sparse) {
    HB_TRY(ensure(ctx, ctx->scratch[kScrKeysAlt], n * 8));
    HB_TRY(ensure(ctx, ctx->scratch[kScrValsAlt], n * 4));
    // key = window start << 32 | window end; a slot without a window carries ~0.  The slots are ordered by
    // start + end: inside a charge bucket that is the order of the precursor m/z, so BOTH ends of the windows of
    // neighbouring slots are close and the union window of a query tile stays tight (ordering by the start alone
    // left the ends of all the queries whose window begins at the bucket's first row in input order: 4.2 % of the
    // tensor engine's MMA work was masked columns on config 2, 1.1 % now; 5.5 % -> 2.8 % with 256-query tiles).
    // Sums are below 2 x n_local; the all-ones key of a slot without a window sums to 2^33 - 2 and still sorts last
    // when truncated to `bits` bits, as long as 2^bits - 2 is above every real sum.
    int bits = 8;
    while (bits < 40 && ((uint64_t(1) << bits) - 2) <= 2 * lib.n_local) bits += 8;
    HB_TRY(ensure(ctx, ctx->scratch[kScrCub], radix_temp_bytes(n)));
    bool in_b = false;
    HB_TRY(radix_sort_pairs_by_half_sum(ctx, ctx->scratch[kScrKeys].as<uint64_t>(), ctx->scratch[kScrKeysAlt].as<uint64_t>(),
                                        ctx->scratch[kScrVals].as<uint32_t>(), ctx->scratch[kScrValsAlt].as<uint32_t>(), n,
                                        bits, ctx->scratch[kScrCub].p, &in_b));
    if (in_b) {
      keys = ctx->scratch[kScrKeysAlt].as<uint64_t>();
      vals = ctx->scratch[kScrValsAlt].as<uint32_t>();
    }
  }

  if (use_direct) {
    const unsigned blocks = static_cast<unsigned>((n * 32 + 255) / 256);
#define HB_DIRECT_ARGS                                                                                        \
  n, keys, vals, d_subset, q.d_words.as<uint4>(), q.d_mz.as<double>(), lib.d_words.as<uint4>(),               \
      lib.d_mz_local.as<double>(), lib.d_id_rank_local.as<uint32_t>(), lib.S / 2, d_out, kr, k, col0, prev_col
#define HB_DIRECT_LAUNCH(KM)                                                                                  \
  do {                                                                                                        \
    if (lib.S / 2 == 8) direct_search_kernel<KM, 8><<<blocks, 256, 0, ctx->stream>>>(HB_DIRECT_ARGS);         \
    else if (lib.S / 2 == 16) direct_search_kernel<KM, 16><<<blocks, 256, 0, ctx->stream>>>(HB_DIRECT_ARGS);  \
    else direct_search_kernel<KM, 0><<<blocks, 256, 0, ctx->stream>>>(HB_DIRECT_ARGS);                        \
  } while (0)
    // k > 32: passes of up to 32, each bounded below by the previous pass's last key (as on the tensor engine)
    for (uint32_t col0 = 0; col0 < k; col0 += kDirectMaxK) {
      const uint32_t kr = std::min<uint32_t>(kDirectMaxK, k - col0);
      const uint32_t prev_col = col0 ? col0 - 1 : kNone;
      {
        KernelTimer timer(ctx, HOMS_B200_KERNEL_SEARCH);
        if (kr == 1 && col0 == 0) HB_DIRECT_LAUNCH(1);
        else if (kr <= 4) HB_DIRECT_LAUNCH(4);
        else if (kr <= 8) HB_DIRECT_LAUNCH(8);
        else if (kr <= 16) HB_DIRECT_LAUNCH(16);
        else HB_DIRECT_LAUNCH(32);
      }
      HB_LAUNCHED(ctx);
    }
#undef HB_DIRECT_LAUNCH
#undef HB_DIRECT_ARGS
    ctx->last_engine = HOMS_B200_ENGINE_DIRECT;
    return HOMS_B200_OK;
  }
  if (tensor_ok) {
    ctx->last_engine = HOMS_B200_ENGINE_TENSOR_FP4;
    return tc_search_sorted(ctx, d_subset, n, keys, vals, d_out, k, k);
  }
  ctx->last_engine = HOMS_B200_ENGINE_POPC;

  const uint32_t n_blocks = static_cast<uint32_t>((n + qb - 1) / qb);
  const int grid = ctx->sm_count * 2;
  const uint32_t target_items = static_cast<uint32_t>(grid) * 8;
  const size_t plan_bytes = 256 + size_t(n_blocks) * 4 * 2 + size_t(n_blocks + 1) * 4;
  HB_TRY(ensure(ctx, ctx->scratch[kScrPlan], plan_bytes));
  auto* base = ctx->scratch[kScrPlan].as<unsigned char>();
  auto* hdr = reinterpret_cast<PlanHeader*>(base);
  auto* blk_lo = reinterpret_cast<uint32_t*>(base + 256);
  auto* blk_rows = blk_lo + n_blocks;
  auto* item_start = blk_rows + n_blocks;
  const uint64_t max_items = uint64_t(target_items) + n_blocks + 1;
  HB_TRY(ensure(ctx, ctx->scratch[kScrPartial], max_items * qb * sizeof(Cand)));

  plan_blocks_kernel<<<(n_blocks + 255) / 256, 256, 0, ctx->stream>>>(n, qb, keys, n_blocks, blk_lo, blk_rows);
  HB_LAUNCHED(ctx);
  plan_items_kernel<<<1, 1024, 0, ctx->stream>>>(n_blocks, target_items, blk_rows, item_start, hdr);
  HB_LAUNCHED(ctx);

  SearchParams sp;
  sp.lib_words = lib.d_words.as<uint64_t>();
  sp.lib_mz = lib.d_mz_local.as<double>();
  sp.lib_rank = lib.d_id_rank_local.as<uint32_t>();
  sp.q_words = q.d_words.as<uint64_t>();
  sp.q_mz = q.d_mz.as<double>();
  sp.subset = d_subset;
  sp.keys = keys;
  sp.vals = vals;
  sp.blk_lo = blk_lo;
  sp.blk_rows = blk_rows;
  sp.item_start = item_start;
  sp.hdr = hdr;
  sp.prev = d_out;
  sp.partial = ctx->scratch[kScrPartial].as<Cand>();
  sp.n = n;
  sp.n_blocks = n_blocks;
  sp.row_bytes = row_bytes;
  sp.k = k;
  for (uint32_t round = 0; round < k; ++round) {
    sp.round = round;
    if (round > 0) {
      reset_counter_kernel<<<1, 1, 0, ctx->stream>>>(hdr);
      HB_LAUNCHED(ctx);
    }
    if (qb == 16) HB_TRY(launch_search<16>(ctx, sp, grid));
    else if (qb == 8) HB_TRY(launch_search<8>(ctx, sp, grid));
    else HB_TRY(launch_search<4>(ctx, sp, grid));
    reduce_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, ctx->stream>>>(
        n, qb, vals, item_start, sp.partial, d_out, k, round);
    HB_LAUNCHED(ctx);
  }
  return HOMS_B200_OK;
}

int queries_set_locked(homs_b200_ctx* ctx, uint32_t dim, uint64_t nq, const uint64_t* words,
                       const double* mz, const uint8_t* charge, bool on_device) {
  Queries& q = ctx->q;
  q.ready = false;
  HB_REQUIRE(ctx, dim >= 1, HOMS_B200_ERR_ARGUMENT, "queries: dim must be positive");
  HB_REQUIRE(ctx, nq == 0 || (words && mz && charge), HOMS_B200_ERR_ARGUMENT, "queries: null argument");
  const uint32_t W = words_for(dim), S = stride_for(dim);
  q.dim = dim;
  q.nq = nq;
  HB_TRY(ensure(ctx, q.d_words, nq * S * 8));
  HB_TRY(ensure(ctx, q.d_mz, nq * 8));
  HB_TRY(ensure(ctx, q.d_charge, nq));
  if (nq) {
    const cudaMemcpyKind kind = on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    if (on_device) HB_TRY(repack_rows_dev(ctx, q.d_words.as<uint64_t>(), words, nq, W, S));
    else HB_TRY(upload_rows(ctx, q.d_words.as<uint64_t>(), words, nq, W, S));
    HB_CUDA(ctx, cudaMemcpyAsync(q.d_mz.p, mz, nq * 8, kind, ctx->stream));
    HB_CUDA(ctx, cudaMemcpyAsync(q.d_charge.p, charge, nq, kind, ctx->stream));
  }
  q.ready = true;
  return HOMS_B200_OK;
}

int merge_launch(homs_b200_ctx* ctx, uint64_t n, uint32_t k, uint32_t n_parts, const Cand* d_parts, Cand* d_out) {
  if (n == 0) return HOMS_B200_OK;
  merge_kernel<<<static_cast<unsigned>((n + 127) / 128), 128, 0, ctx->stream>>>(n, k, n_parts, d_parts, d_out);
  HB_LAUNCHED(ctx);
  return HOMS_B200_OK;
}

static int decode_locked(homs_b200_ctx* ctx, uint64_t total, const Cand* d_rec, uint32_t* out_score,
                         uint32_t* out_ordinal) {
  if (total == 0) return HOMS_B200_OK;
  HB_TRY(ensure(ctx, ctx->scratch[kScrDecode], total * 8));
  auto* d_score = ctx->scratch[kScrDecode].as<uint32_t>();
  auto* d_ord = d_score + total;
  decode_kernel<<<static_cast<unsigned>((total + 255) / 256), 256, 0, ctx->stream>>>(
      total, d_rec, ctx->lib.dim, ctx->lib.d_ord_of_rank.as<uint32_t>(), d_score, d_ord);
  HB_LAUNCHED(ctx);
  HB_CUDA(ctx, cudaMemcpyAsync(out_score, d_score, total * 4, cudaMemcpyDeviceToHost, ctx->stream));
  HB_CUDA(ctx, cudaMemcpyAsync(out_ordinal, d_ord, total * 4, cudaMemcpyDeviceToHost, ctx->stream));
  HB_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  return HOMS_B200_OK;
}

}  // namespace hb

using namespace hb;

extern "C" {

int homs_b200_window_bounds(homs_b200_ctx* ctx, uint64_t nq, const double* q_mz,
                            const uint8_t* q_charge, const homs_b200_tolerance* tol,
                            uint64_t* out_first, uint64_t* out_last, uint8_t* out_has_bucket) {
  if (!ctx) return HOMS_B200_ERR_ARGUMENT;
  Lock lock(ctx);
  HB_REQUIRE(ctx, ctx->lib.ready, HOMS_B200_ERR_STATE, "window_bounds: no library uploaded");
  HB_TRY(check_tol(ctx, tol));
  if (nq == 0) return HOMS_B200_OK;
  HB_REQUIRE(ctx, q_mz && q_charge && out_first && out_last, HOMS_B200_ERR_ARGUMENT,
             "window_bounds: null argument");
  HB_TRY(ensure(ctx, ctx->scratch[kScrMisc], nq * 8));
  HB_TRY(ensure(ctx, ctx->scratch[kScrMisc2], nq));
  HB_TRY(ensure(ctx, ctx->scratch[kScrQFirst], nq * 8));
  HB_TRY(ensure(ctx, ctx->scratch[kScrQLast], nq * 8));
  HB_TRY(ensure(ctx, ctx->scratch[kScrHas], nq));
  auto* d_mz = ctx->scratch[kScrMisc].as<double>();
  auto* d_ch = ctx->scratch[kScrMisc2].as<uint8_t>();
  auto* d_first = ctx->scratch[kScrQFirst].as<uint64_t>();
  auto* d_last = ctx->scratch[kScrQLast].as<uint64_t>();
  auto* d_has = ctx->scratch[kScrHas].as<uint8_t>();
  HB_CUDA(ctx, cudaMemcpyAsync(d_mz, q_mz, nq * 8, cudaMemcpyHostToDevice, ctx->stream));
  HB_CUDA(ctx, cudaMemcpyAsync(d_ch, q_charge, nq, cudaMemcpyHostToDevice, ctx->stream));
  HB_TRY(run_bounds(ctx, nq, nullptr, d_mz, d_ch, tol, d_first, d_last, d_has));
  HB_CUDA(ctx, cudaMemcpyAsync(out_first, d_first, nq * 8, cudaMemcpyDeviceToHost, ctx->stream));
  HB_CUDA(ctx, cudaMemcpyAsync(out_last, d_last, nq * 8, cudaMemcpyDeviceToHost, ctx->stream));
  if (out_has_bucket)
    HB_CUDA(ctx, cudaMemcpyAsync(out_has_bucket, d_has, nq, cudaMemcpyDeviceToHost, ctx->stream));
  HB_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  return HOMS_B200_OK;
}

int homs_b200_queries_upload(homs_b200_ctx* ctx, uint32_t query_dim, uint64_t nq,
                             const uint64_t* q_words, const double* q_mz, const uint8_t* q_charge) {
  if (!ctx) return HOMS_B200_ERR_ARGUMENT;
  Lock lock(ctx);
  HB_TRY(queries_set_any_locked(ctx, query_dim, nq, q_words, q_mz, q_charge, false));
  return sync_all_locked(ctx);  // the caller may reuse its buffers
}

int homs_b200_queries_upload_dev(homs_b200_ctx* ctx, uint32_t query_dim, uint64_t nq,
                                 const uint64_t* d_q_words, const double* d_q_mz,
                                 const uint8_t* d_q_charge) {
  if (!ctx) return HOMS_B200_ERR_ARGUMENT;
  Lock lock(ctx);
  return queries_set_any_locked(ctx, query_dim, nq, d_q_words, d_q_mz, d_q_charge, true);
}

int homs_b200_search_resident_dev(homs_b200_ctx* ctx, const uint32_t* d_subset, uint64_t n_subset,
                                  const homs_b200_tolerance* tol, uint32_t k,
                                  homs_b200_candidate* d_out) {
  if (!ctx) return HOMS_B200_ERR_ARGUMENT;
  Lock lock(ctx);
  const uint64_t n = d_subset ? n_subset : ctx->q.nq;
  HB_REQUIRE(ctx, n == 0 || d_out, HOMS_B200_ERR_ARGUMENT, "search_resident: null output");
  return search_any_locked(ctx, d_subset, n, tol, k, reinterpret_cast<Cand*>(d_out), nullptr, nullptr, nullptr);
}

int homs_b200_merge_candidates_dev(homs_b200_ctx* ctx, uint64_t n, uint32_t k, uint32_t n_parts,
                                   const homs_b200_candidate* d_parts, homs_b200_candidate* d_out) {
  if (!ctx) return HOMS_B200_ERR_ARGUMENT;
  Lock lock(ctx);
  HB_REQUIRE(ctx, k >= 1 && k <= HOMS_B200_MAX_TOPK, HOMS_B200_ERR_ARGUMENT, "merge: k must be in [1, 64]");
  HB_REQUIRE(ctx, n_parts >= 1 && n_parts <= 64, HOMS_B200_ERR_ARGUMENT, "merge: n_parts must be in [1, 64]");
  if (n == 0) return HOMS_B200_OK;
  HB_REQUIRE(ctx, d_parts && d_out, HOMS_B200_ERR_ARGUMENT, "merge: null argument");
  return merge_launch(ctx, n, k, n_parts, reinterpret_cast<const Cand*>(d_parts), reinterpret_cast<Cand*>(d_out));
}

int homs_b200_candidates_decode(homs_b200_ctx* ctx, uint64_t n, uint32_t k,
                                const homs_b200_candidate* d_records, uint32_t* out_raw_score,
                                uint32_t* out_ordinal) {
  if (!ctx) return HOMS_B200_ERR_ARGUMENT;
  Lock lock(ctx);
  HB_REQUIRE(ctx, ctx->lib.ready, HOMS_B200_ERR_STATE, "decode: no library uploaded");
  HB_REQUIRE(ctx, n == 0 || (d_records && out_raw_score && out_ordinal), HOMS_B200_ERR_ARGUMENT,
             "decode: null argument");
  return decode_locked(ctx, n * k, reinterpret_cast<const Cand*>(d_records), out_raw_score, out_ordinal);
}

int homs_b200_search_batch(homs_b200_ctx* ctx, uint32_t query_dim, uint64_t nq,
                           const uint64_t* q_words, const double* q_mz, const uint8_t* q_charge,
                           const homs_b200_tolerance* tol, uint32_t k, uint32_t* out_raw_score,
                           uint32_t* out_ordinal, uint64_t* out_first, uint64_t* out_last) {
  if (!ctx) return HOMS_B200_ERR_ARGUMENT;
  Lock lock(ctx);
  HB_REQUIRE(ctx, ctx->lib.ready, HOMS_B200_ERR_STATE, "search_batch: no library uploaded");
  HB_REQUIRE(ctx, ctx->lib.shard_count == 1 || is_group(ctx), HOMS_B200_ERR_STATE,
             "search_batch: this context holds one shard of a library split across processes; use "
             "search_resident_dev + an all-gather + merge_candidates_dev (or a multi-device context)");
  HB_REQUIRE(ctx, query_dim == ctx->lib.dim, HOMS_B200_ERR_INVARIANT,
             "search_one: query dimensionality does not match index");
  HB_TRY(check_tol(ctx, tol));
  HB_REQUIRE(ctx, k >= 1 && k <= HOMS_B200_MAX_TOPK, HOMS_B200_ERR_ARGUMENT, "search: k must be in [1, 64]");
  if (nq == 0) return HOMS_B200_OK;
  HB_REQUIRE(ctx, out_raw_score && out_ordinal, HOMS_B200_ERR_ARGUMENT, "search_batch: null output");
  HB_TRY(queries_set_any_locked(ctx, query_dim, nq, q_words, q_mz, q_charge, false));
  HB_TRY(ensure(ctx, ctx->scratch[kScrRecords], nq * k * sizeof(Cand)));
  uint64_t* d_first = nullptr;
  uint64_t* d_last = nullptr;
  if (out_first || out_last) {
    HB_TRY(ensure(ctx, ctx->scratch[kScrQFirst], nq * 8));
    HB_TRY(ensure(ctx, ctx->scratch[kScrQLast], nq * 8));
    d_first = ctx->scratch[kScrQFirst].as<uint64_t>();
    d_last = ctx->scratch[kScrQLast].as<uint64_t>();
  }
  Cand* d_rec = ctx->scratch[kScrRecords].as<Cand>();
  HB_TRY(search_any_locked(ctx, nullptr, nq, tol, k, d_rec, d_first, d_last, nullptr));
  if (out_first) HB_CUDA(ctx, cudaMemcpyAsync(out_first, d_first, nq * 8, cudaMemcpyDeviceToHost, ctx->stream));
  if (out_last) HB_CUDA(ctx, cudaMemcpyAsync(out_last, d_last, nq * 8, cudaMemcpyDeviceToHost, ctx->stream));
  return decode_locked(ctx, nq * k, d_rec, out_raw_score, out_ordinal);
}

}  // extern "C"

// cascade over the RESIDENT queries (q_words == nullptr) or over host queries uploaded first
static int cascade_locked(homs_b200_ctx* ctx, uint32_t query_dim, uint64_t nq, const uint64_t* q_words,
                          const double* q_mz, const uint8_t* q_charge, const homs_b200_tolerance* narrow,
                          const homs_b200_tolerance* wide, double fdr_q, const uint8_t* lib_is_decoy,
                          uint64_t* out_query, uint32_t* out_ordinal, uint8_t* out_stage,
                          uint32_t* out_raw_score, double* out_q_value, uint64_t* out_count) {
  const bool resident = q_words == nullptr && q_mz == nullptr && q_charge == nullptr;
  if (resident) {
    HB_REQUIRE(ctx, ctx->q.ready, HOMS_B200_ERR_STATE, "cascade_resident: no resident queries");
    query_dim = ctx->q.dim;
    nq = ctx->q.nq;
  }
  HB_REQUIRE(ctx, ctx->lib.ready, HOMS_B200_ERR_STATE, "cascade_search: no library uploaded");
  HB_REQUIRE(ctx, ctx->lib.shard_count == 1 || is_group(ctx), HOMS_B200_ERR_STATE,
             "cascade_search: this context holds one shard of a library split across processes");
  HB_TRY(check_tol(ctx, narrow));
  HB_TRY(check_tol(ctx, wide));
  // Tolerance::validate, search.cpp:13-15 via :223-224
  HB_REQUIRE(ctx, narrow->value > 0.0 && wide->value > 0.0, HOMS_B200_ERR_CONFIG,
             "tolerance value must be positive");
  HB_REQUIRE(ctx, out_count != nullptr, HOMS_B200_ERR_ARGUMENT, "cascade_search: null out_count");
  *out_count = 0;
  if (nq == 0) return HOMS_B200_OK;
  HB_REQUIRE(ctx, query_dim == ctx->lib.dim, HOMS_B200_ERR_INVARIANT,
             "search_one: query dimensionality does not match index");
  HB_REQUIRE(ctx, lib_is_decoy && out_query && out_ordinal && out_stage && out_raw_score && out_q_value,
             HOMS_B200_ERR_ARGUMENT, "cascade_search: null argument");
  if (!resident) HB_TRY(queries_set_any_locked(ctx, query_dim, nq, q_words, q_mz, q_charge, false));
  HB_TRY(ensure(ctx, ctx->scratch[kScrRecords], nq * sizeof(Cand)));
  Cand* d_rec = ctx->scratch[kScrRecords].as<Cand>();

  struct Accepted {
    bool has = false;
    uint8_t stage = 0;
    uint32_t score = 0, ordinal = 0;
    double q = 0.0;
  };
  std::vector<Accepted> accepted(nq);
  std::vector<uint32_t> todo(nq);
  std::iota(todo.begin(), todo.end(), 0u);
  std::vector<uint32_t> h_score(nq), h_ord(nq);
  const double dim_d = static_cast<double>(ctx->lib.dim);

  for (uint8_t stage = 0; stage < 2; ++stage) {  // run_stage, search.cpp:188-215
    const uint64_t n = todo.size();
    if (n == 0) continue;
    const uint32_t* d_subset = nullptr;
    if (stage == 1) {
      HB_TRY(ensure(ctx, ctx->scratch[kScrSubset], n * 4));
      HB_CUDA(ctx, cudaMemcpyAsync(ctx->scratch[kScrSubset].p, todo.data(), n * 4,
                                   cudaMemcpyHostToDevice, ctx->stream));
      d_subset = ctx->scratch[kScrSubset].as<uint32_t>();
    }
    HB_TRY(search_any_locked(ctx, d_subset, n, stage == 0 ? narrow : wide, 1, d_rec, nullptr, nullptr,
                             nullptr));
    HB_TRY(decode_locked(ctx, n, d_rec, h_score.data(), h_ord.data()));
    std::vector<double> score;
    std::vector<uint8_t> decoy;
    std::vector<uint32_t> pool;  // index into todo
    for (uint64_t i = 0; i < n; ++i) {
      if (h_ord[i] == HOMS_B200_NO_HIT) continue;
      pool.push_back(static_cast<uint32_t>(i));
      score.push_back(static_cast<double>(h_score[i]) / dim_d);  // search.cpp:165
      decoy.push_back(lib_is_decoy[h_ord[i]] != 0);
    }
    const uint64_t np = pool.size();
    std::vector<uint64_t> order(np);
    std::vector<double> fdr(np), qv(np);
    HB_TRY(homs_b200_compute_fdr_curve(np, score.data(), decoy.data(), order.data(), fdr.data(), qv.data()));
    for (uint64_t pp = 0; pp < np; ++pp) {  // search.cpp:209-214
      const uint64_t in = order[pp];
      if (!decoy[in] && qv[pp] <= fdr_q) {
        Accepted& a = accepted[todo[pool[in]]];
        a.has = true;
        a.stage = stage;
        a.score = h_score[pool[in]];
        a.ordinal = h_ord[pool[in]];
        a.q = qv[pp];
      }
    }
    if (stage == 0) {
      std::vector<uint32_t> rest;
      for (uint32_t i = 0; i < nq; ++i)
        if (!accepted[i].has) rest.push_back(i);
      todo.swap(rest);
    }
  }
  uint64_t m = 0;
  for (uint8_t stage = 0; stage < 2; ++stage)  // search.cpp:240-247
    for (uint64_t i = 0; i < nq; ++i)
      if (accepted[i].has && accepted[i].stage == stage) {
        out_query[m] = i;
        out_ordinal[m] = accepted[i].ordinal;
        out_stage[m] = stage;
        out_raw_score[m] = accepted[i].score;
        out_q_value[m] = accepted[i].q;
        ++m;
      }
  *out_count = m;
  return HOMS_B200_OK;
}

extern "C" {

int homs_b200_cascade_search(homs_b200_ctx* ctx, uint32_t query_dim, uint64_t nq,
                             const uint64_t* q_words, const double* q_mz, const uint8_t* q_charge,
                             const homs_b200_tolerance* narrow, const homs_b200_tolerance* wide,
                             double fdr_q, const uint8_t* lib_is_decoy, uint64_t* out_query,
                             uint32_t* out_ordinal, uint8_t* out_stage, uint32_t* out_raw_score,
                             double* out_q_value, uint64_t* out_count) {
  if (!ctx) return HOMS_B200_ERR_ARGUMENT;
  Lock lock(ctx);
  HB_REQUIRE(ctx, nq == 0 || (q_words && q_mz && q_charge), HOMS_B200_ERR_ARGUMENT,
             "cascade_search: null argument");
  if (nq == 0) {  // keep the validation order of the host-query form
    static const uint64_t none = 0;
    q_words = &none;
  }
  return cascade_locked(ctx, query_dim, nq, q_words, q_mz, q_charge, narrow, wide, fdr_q, lib_is_decoy, out_query,
                        out_ordinal, out_stage, out_raw_score, out_q_value, out_count);
}

int homs_b200_cascade_resident(homs_b200_ctx* ctx, const homs_b200_tolerance* narrow,
                               const homs_b200_tolerance* wide, double fdr_q, const uint8_t* lib_is_decoy,
                               uint64_t* out_query, uint32_t* out_ordinal, uint8_t* out_stage,
                               uint32_t* out_raw_score, double* out_q_value, uint64_t* out_count) {
  if (!ctx) return HOMS_B200_ERR_ARGUMENT;
  Lock lock(ctx);
  return cascade_locked(ctx, 0, 0, nullptr, nullptr, nullptr, narrow, wide, fdr_q, lib_is_decoy, out_query,
                        out_ordinal, out_stage, out_raw_score, out_q_value, out_count);
}

int homs_b200_search_resident(homs_b200_ctx* ctx, const homs_b200_tolerance* tol, uint32_t k,
                              uint32_t* out_raw_score, uint32_t* out_ordinal, uint64_t* out_first,
                              uint64_t* out_last) {
  if (!ctx) return HOMS_B200_ERR_ARGUMENT;
  Lock lock(ctx);
  HB_REQUIRE(ctx, ctx->lib.ready, HOMS_B200_ERR_STATE, "search_resident: no library uploaded");
  HB_REQUIRE(ctx, ctx->q.ready, HOMS_B200_ERR_STATE, "search_resident: no resident queries");
  HB_REQUIRE(ctx, ctx->lib.shard_count == 1 || is_group(ctx), HOMS_B200_ERR_STATE,
             "search_resident: this context holds one shard of a library split across processes; use "
             "search_resident_dev + an all-gather + merge_candidates_dev (or a multi-device context)");
  HB_REQUIRE(ctx, ctx->q.dim == ctx->lib.dim, HOMS_B200_ERR_INVARIANT,
             "search_one: query dimensionality does not match index");
  HB_TRY(check_tol(ctx, tol));
  HB_REQUIRE(ctx, k >= 1 && k <= HOMS_B200_MAX_TOPK, HOMS_B200_ERR_ARGUMENT, "search: k must be in [1, 64]");
  const uint64_t nq = ctx->q.nq;
  if (nq == 0) return HOMS_B200_OK;
  HB_REQUIRE(ctx, out_raw_score && out_ordinal, HOMS_B200_ERR_ARGUMENT, "search_resident: null output");
  HB_TRY(ensure(ctx, ctx->scratch[kScrRecords], nq * k * sizeof(Cand)));
  uint64_t* d_first = nullptr;
  uint64_t* d_last = nullptr;
  if (out_first || out_last) {
    HB_TRY(ensure(ctx, ctx->scratch[kScrQFirst], nq * 8));
    HB_TRY(ensure(ctx, ctx->scratch[kScrQLast], nq * 8));
    d_first = ctx->scratch[kScrQFirst].as<uint64_t>();
    d_last = ctx->scratch[kScrQLast].as<uint64_t>();
  }
  Cand* d_rec = ctx->scratch[kScrRecords].as<Cand>();
  HB_TRY(search_any_locked(ctx, nullptr, nq, tol, k, d_rec, d_first, d_last, nullptr));
  if (out_first) HB_CUDA(ctx, cudaMemcpyAsync(out_first, d_first, nq * 8, cudaMemcpyDeviceToHost, ctx->stream));
  if (out_last) HB_CUDA(ctx, cudaMemcpyAsync(out_last, d_last, nq * 8, cudaMemcpyDeviceToHost, ctx->stream));
  return decode_locked(ctx, nq * k, d_rec, out_raw_score, out_ordinal);
}

}  // extern "C"
