// Spectrum preprocessing (K1) and ID-level hypervector encoding (K2) for sm_100a.
//
// Reference semantics (paths under /root/reference/proj/core/):
//   refine_peaks   src/preprocess.cpp:41-75      vectorize  src/preprocess.cpp:77-110
//   quantize       src/encoder.cpp:11-17         encode     src/encoder.cpp:19-55
//   encode_spectra src/pipeline.cpp:60-85
//
// K1  one warp per spectrum, fp64 throughout (compiled with -fmad=false; every operation is a
//     single IEEE add/sub/mul/div/sqrt/floor/round exactly as in the reference), peaks staged in
//     shared memory, order-preserving ballot compaction.
// K2  one warp per spectrum, bit-sliced: lane owns one 128-bit column slab per pass; per peak the
//     lane XNORs its slab of the position row (L2 gather, LDG.128) with the level row (shared
//     memory) and feeds the 32x4 one-bit votes into a carry-save adder tree (7:3 compressors,
//     LOP3) that accumulates vertical counters; the strict majority 2*votes > n is a bit-serial
//     comparison of the counter planes against floor(n/2)+1.  Output rows are written with
//     coalesced 128-bit stores.
#include <algorithm>
#include <cstring>
#include <vector>

#include "common.cuh"

namespace hb {

// ------------------------------------------------------------------------------------------
// K1: refine_peaks + vectorize + quantize_intensity
// ------------------------------------------------------------------------------------------

// out_count marker of a spectrum on which the reference would throw InvariantError (a normalised
// intensity outside [0, 1]); encode_kernel turns it into ok flag HOMS_B200_OK_FLAG_INVARIANT
constexpr uint32_t kInvalidCount = 0xFFFFFFFFu;

struct PreParams {
  double min_mz, max_mz, bin_size, intensity_floor;
  uint32_t max_peaks, min_peaks, scaling, dims, levels;
};

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

__device__ __forceinline__ uint32_t quantize_level(double v, uint32_t levels) {
  // encoder.cpp:15-16: min(u32(round(v * Q)), Q); round() is half-away-from-zero
  const double level = round(v * static_cast<double>(levels));
  const uint32_t l = static_cast<uint32_t>(level);
  return l < levels ? l : levels;
}

// One warp per spectrum.  Shared memory per warp: max_peaks * (8 + 8 + 4) bytes.
__global__ void __launch_bounds__(256)
preprocess_kernel(PreParams p, uint64_t n, const uint64_t* __restrict__ offsets,
                  const double* __restrict__ mz, const double* __restrict__ inten,
                  uint32_t* __restrict__ out_bins, uint32_t* __restrict__ out_levels,
                  uint32_t* __restrict__ out_count, int warps_per_cta) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const uint32_t MP = p.max_peaks;
  double* s_mz = reinterpret_cast<double*>(smem_raw) + size_t(warp) * 2 * MP;
  double* s_int = s_mz + MP;
  uint32_t* s_bin = reinterpret_cast<uint32_t*>(reinterpret_cast<double*>(smem_raw) +
                                                size_t(warps_per_cta) * 2 * MP) +
                    size_t(warp) * MP;
  double* o_val = s_mz;  // reused once the bins have been computed

  for (uint64_t spec = uint64_t(blockIdx.x) * warps_per_cta + warp; spec < n;
       spec += uint64_t(gridDim.x) * warps_per_cta) {
    const uint64_t a = offsets[spec], b = offsets[spec + 1];

    // preprocess.cpp:45-49 range / positivity filter, :52-53 base peak over the filtered set
    double base = 0.0;
    for (uint64_t j = a + lane; j < b; j += 32) {
      const double m = mz[j], v = inten[j];
      if (m >= p.min_mz && m < p.max_mz && v > 0.0) base = fmax(base, v);
    }
    base = warp_max(base);
    const double floor_intensity = p.intensity_floor * base;  // :54

    // survivors of :55 (strict <), counted
    uint32_t m_surv = 0;
    for (uint64_t j = a + lane; j < b; j += 32) {
      const double m = mz[j], v = inten[j];
      m_surv += (m >= p.min_mz && m < p.max_mz && v > 0.0 && !(v < floor_intensity));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m_surv += __shfl_xor_sync(0xffffffffu, m_surv, o);
    const bool truncate = m_surv > MP;  // :58

    // :60-64 keep the max_peaks first in (intensity desc, m/z asc) order.  Selection instead of ranking: T = the
    // MP-th largest surviving intensity (positive doubles order like their bit patterns, so T is built bit by bit
    // from the top: 63 counting passes over the peaks, O(63 P / 32) per lane where the all-pairs rank took
    // O(P^2 / 32)); everything above T is kept, and of the peaks AT T the first `need_ties` by (m/z asc, position).
    // Spectra of up to 256 raw peaks hold their intensity bits in registers (8 per lane) for the counting passes.
    uint64_t thr = 0;
    uint32_t need_ties = 0;
    bool ties_all = true;
    if (truncate) {
      constexpr int kRegPeaks = 8;
      const bool in_regs = b - a <= 32ull * kRegPeaks;
      uint64_t vb[kRegPeaks];
#pragma unroll
      for (int r = 0; r < kRegPeaks; ++r) {
        vb[r] = 0;  // not a survivor: below every candidate threshold (candidates are > 0)
        const uint64_t j = a + uint64_t(r) * 32 + lane;
        if (in_regs && j < b) {
          const double m = mz[j], v = inten[j];
          if (m >= p.min_mz && m < p.max_mz && v > 0.0 && !(v < floor_intensity))
            vb[r] = static_cast<uint64_t>(__double_as_longlong(v));
        }
      }
      auto count_ge = [&](uint64_t cand) {  // survivors whose intensity bits are >= cand (cand > 0)
        uint32_t c = 0;
        if (in_regs) {
#pragma unroll
          for (int r = 0; r < kRegPeaks; ++r) c += vb[r] >= cand;
        } else {
          for (uint64_t j = a + lane; j < b; j += 32) {
            const double m = mz[j], v = inten[j];
            c += m >= p.min_mz && m < p.max_mz && v > 0.0 && !(v < floor_intensity) &&
                 static_cast<uint64_t>(__double_as_longlong(v)) >= cand;
          }
        }
        return __reduce_add_sync(0xffffffffu, c);
      };
      for (int bit = 62; bit >= 0; --bit) {
        const uint64_t cand = thr | (1ull << bit);
        if (count_ge(cand) >= MP) thr = cand;
      }
      const uint32_t n_gt = count_ge(thr + 1), n_ge = count_ge(thr);
      need_ties = MP - n_gt;               // >= 1 by the choice of thr
      ties_all = n_ge - n_gt == need_ties;  // every peak at the threshold is kept: no order among them needed
    }

    // ordered compaction of the kept peaks into shared memory
    uint32_t kept = 0;
    for (uint64_t c = a; c < b; c += 32) {
      const uint64_t j = c + lane;
      bool keep = false;
      double m = 0.0, v = 0.0;
      if (j < b) {
        m = mz[j];
        v = inten[j];
        keep = m >= p.min_mz && m < p.max_mz && v > 0.0 && !(v < floor_intensity);
      }
      if (truncate) {
        const uint64_t bits = static_cast<uint64_t>(__double_as_longlong(v));
        const bool at_thr = keep && bits == thr;
        keep = keep && bits >= thr;
        if (!ties_all && __any_sync(0xffffffffu, at_thr)) {
          // rank among the peaks at the threshold: (m/z asc, position breaks exact duplicates)
          uint32_t rank = 0;
          for (uint64_t jj = a; jj < b; ++jj) {
            const double m2 = mz[jj], v2 = inten[jj];  // warp-uniform address: broadcast load
            const bool tie2 = m2 >= p.min_mz && m2 < p.max_mz && static_cast<uint64_t>(__double_as_longlong(v2)) == thr;
            rank += tie2 && (m2 < m || (m2 == m && jj < j));
          }
          if (at_thr) keep = rank < need_ties;
        }
      }
      const uint32_t mask = __ballot_sync(0xffffffffu, keep);
      if (keep) {
        const uint32_t slot = kept + __popc(mask & ((1u << lane) - 1u));
        s_mz[slot] = m;
        s_int[slot] = v;
      }
      kept += __popc(mask);
    }
    __syncwarp();

    if (kept < p.min_peaks || kept == 0) {  // :69 (kept == 0 cannot encode; validate() forbids min_peaks 0)
      if (lane == 0) out_count[spec] = 0;
      continue;
    }

    // vectorize :91-94 bin index
    for (uint32_t s = lane; s < kept; s += 32) {
      const double q = (s_mz[s] - p.min_mz) / p.bin_size + 1e-9;
      double f = floor(q);
      const double hi = static_cast<double>(p.dims - 1);
      f = f < 0.0 ? 0.0 : (hi < f ? hi : f);  // std::clamp
      s_bin[s] = static_cast<uint32_t>(f);
    }
    __syncwarp();

    // :95-100 adjacent equal bins are summed left to right (sequential fp64 adds per run)
    uint32_t nb = 0;
    for (uint32_t c = 0; c < kept; c += 32) {
      const uint32_t s = c + lane;
      bool head = false;
      uint32_t bin = 0;
      if (s < kept) {
        bin = s_bin[s];
        head = s == 0 || s_bin[s - 1] != bin;
      }
      const uint32_t mask = __ballot_sync(0xffffffffu, head);
      double sum = 0.0;
      uint32_t slot = 0;
      if (head) {
        slot = nb + __popc(mask & ((1u << lane) - 1u));
        sum = s_int[s];
        for (uint32_t t = s + 1; t < kept && s_bin[t] == bin; ++t) sum += s_int[t];
        if (p.scaling == 1) sum = sqrt(sum);  // :103-105
      }
      // o_val aliases s_mz: all lanes of this chunk have consumed s_mz already (bins done),
      // and s_int (the source of the sums) is a different array.
      __syncwarp();
      if (head) {
        o_val[slot] = sum;
        out_bins[spec * MP + slot] = bin;
      }
      nb += __popc(mask);
    }
    __syncwarp();

    // :107-108 divide by the maximum, then encoder.cpp:11-17
    double top = 0.0;
    for (uint32_t k = lane; k < nb; k += 32) top = fmax(top, o_val[k]);
    top = warp_max(top);
    bool bad = false;  // encoder.cpp:12-14: quantize_intensity throws outside [0, 1] (inf / inf = NaN)
    for (uint32_t k = lane; k < nb; k += 32) {
      const double v = o_val[k] / top;
      bad |= !(v >= 0.0 && v <= 1.0);
      out_levels[spec * MP + k] = quantize_level(v, p.levels);
    }
    bad = __any_sync(0xffffffffu, bad);
    if (lane == 0) out_count[spec] = bad ? kInvalidCount : nb;
    __syncwarp();
  }
}

// ------------------------------------------------------------------------------------------
// K2: encode
// ------------------------------------------------------------------------------------------

struct U4 {
  uint32_t v[4];
};

__device__ __forceinline__ U4 ld_global_u4(const uint4* p) {
  const uint4 t = __ldg(p);
  return U4{{t.x, t.y, t.z, t.w}};
}

// carry-save adder on 4 independent 32-bit lanes: (a + b + c) = s + 2*k
#define HB_CSA(s, k, a, b, c)                                                 \
  _Pragma("unroll") for (int i_ = 0; i_ < 4; ++i_) {                          \
    const uint32_t a_ = (a).v[i_], b_ = (b).v[i_], c_ = (c).v[i_];            \
    (s).v[i_] = a_ ^ b_ ^ c_;                                                 \
    (k).v[i_] = (a_ & b_) | (a_ & c_) | (b_ & c_);                            \
  }

// Encodes spectra [0, n).  The (bin, level) list of spectrum i is
//   strided mode (sv_offsets == nullptr): sv_bins[i*stride .. +sv_count[i])
//   CSR mode:                              sv_bins[sv_offsets[i] .. sv_offsets[i+1])
// NP = number of vertical counter planes (counts < 2^NP).
#ifndef HB_ENC_MINB
#define HB_ENC_MINB 2   // resident CTAs per SM the register budget is sized for (A/B: profiles/)
#define HB_ENC_WARPS 8  // warps (= spectra in flight) per CTA
#endif
#ifndef HB_ENC_PIPELINED
// 1: the gathers of group t+1 are issued pairwise into the registers of group t as the carry-save tree
// consumes them (software pipelining at no extra registers).  MEASURED AND LEFT OFF: 3.31 -> 5.86 ms per
// 250 k spectra (profiles/r02_ab_encode_pipelined.log) -- with four refill points per iteration the
// refilled pairs share scoreboards with pairs still awaited, so every wait also covers loads issued a few
// instructions earlier and the L2 latency is exposed four times per group instead of once.
#define HB_ENC_PIPELINED 0
#endif
template <int NP, bool kLvlSmem>
__global__ void __launch_bounds__(HB_ENC_WARPS * 32, HB_ENC_MINB)
encode_kernel(uint64_t n, const uint64_t* __restrict__ sv_offsets, uint32_t stride,
              const uint32_t* __restrict__ sv_bins, const uint32_t* __restrict__ sv_levels,
              const uint32_t* __restrict__ sv_count, const uint4* __restrict__ pos,
              const uint4* __restrict__ lvl_global, uint32_t n_level_rows, uint32_t row_u4,
              uint32_t dim, uint32_t W, int vec_store,
              uint64_t* __restrict__ out_words,
              uint8_t* __restrict__ out_ok) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  // level rows: shared memory when they fit (LDS with a 32-bit address), else global through L1
  uint4* s_lvl = reinterpret_cast<uint4*>(smem_raw);
  if constexpr (kLvlSmem) {
    for (uint32_t i = threadIdx.x; i < (n_level_rows + 1) * row_u4; i += blockDim.x) s_lvl[i] = lvl_global[i];
    __syncthreads();
  }
  const int lane = threadIdx.x & 31;
  const int warps = blockDim.x >> 5;
  const int warp = threadIdx.x >> 5;

  for (uint64_t spec = uint64_t(blockIdx.x) * warps + warp; spec < n;
       spec += uint64_t(gridDim.x) * warps) {
    uint64_t start;
    uint32_t nb;
    if (sv_offsets) {
      start = sv_offsets[spec];
      nb = static_cast<uint32_t>(sv_offsets[spec + 1] - start);
    } else {
      start = spec * stride;
      nb = sv_count[spec];
    }
    uint64_t* out_row = out_words + spec * W;
    if (nb == 0 || nb == kInvalidCount) {  // unprocessable: zero row (pipeline.cpp:68 `continue`)
      for (uint32_t w = lane; w < W; w += 32) out_row[w] = 0;
      if (lane == 0 && out_ok) out_ok[spec] = nb == 0 ? 0 : HOMS_B200_OK_FLAG_INVARIANT;
      continue;
    }
    const uint32_t thresh = nb / 2 + 1;  // 2*votes > n  <=>  votes >= floor(n/2)+1  (encoder.cpp:52)

    for (uint32_t sb = 0; sb < row_u4; sb += 32) {
      const uint32_t u = sb + lane;
      const bool active = u < row_u4;
      U4 c[NP];
#pragma unroll
      for (int b = 0; b < NP; ++b) c[b] = U4{{0, 0, 0, 0}};

      // The (bin, level) list is staged through registers 32 entries at a time (lane j holds entry
      // c0 + j: one coalesced load per warp, the next block prefetched) and broadcast by shuffle,
      // so the position-row gathers depend on no other memory access.  Votes are summed by a
      // Harley-Seal tree: c[0..4] are carry-save accumulators of weight 1, 2, 4, 8, 16 (and, being
      // single bits per position, ARE planes 0..4 of the count); every 32 inputs emit one carry
      // of weight 32 into the half-adder chain c[5..NP).  31 CSAs + NP-5 half adders per 32 inputs.
      // Groups of 8 run in a real loop: 8 gathers in flight per lane, bounded registers.
      // Entries past the end of the list read position row 0 against the extra level row
      // (~position[0], see homs_b200_codebook_upload): XNOR = 0 everywhere, i.e. no vote and no
      // per-entry mask.  All addressing is a byte offset prepared by the staging lane, so a gather
      // costs one wide multiply-add and a level fetch one add next to the logic ops that bound the
      // kernel (ncu: ALU pipe 85 % before this change).
      const uint32_t uu = active ? u : row_u4 - 1;  // idle lanes gather a valid slab and store nothing
      const unsigned char* pos_b = reinterpret_cast<const unsigned char*>(pos + uu);
      const unsigned char* lvl_b = reinterpret_cast<const unsigned char*>((kLvlSmem ? s_lvl : lvl_global) + uu);
      const uint32_t row_bytes = row_u4 * 16;
      const uint32_t null_lev = n_level_rows * row_bytes;  // the extra row
#if HB_ENC_PIPELINED
      // Software-pipelined gathers.  A group's 8 position-row gathers land ~1000 cycles after issue
      // (L2 under load) and the XNOR + carry-save work on them is ~180 issue slots per warp; run back
      // to back (load 8, wait, compute) the two add up and the kernel sits at 0.58 of the measured
      // random-row gather ceiling (tools/l2_gather_bench).  Here the gathers of group t+1 are issued
      // pairwise into the registers of group t as soon as the carry-save tree has consumed them, so
      // every warp keeps ~8 gathers in flight WHILE it computes, at no extra registers.
      uint32_t my_bin = 0, my_lev = null_lev, nxt_bin = 0, nxt_lev = null_lev;
      if (lane < nb) {
        my_bin = sv_bins[start + lane];
        my_lev = sv_levels[start + lane] * row_bytes;
      }
      U4 x[8];
      uint32_t lev[8];
#define HB_ENC_ISSUE(j, src_bin, src_lev, kk)                                                         \
  do {                                                                                                \
    const uint32_t bin_ = __shfl_sync(0xffffffffu, (src_bin), (kk));                                  \
    lev[j] = __shfl_sync(0xffffffffu, (src_lev), (kk));                                               \
    x[j] = ld_global_u4(reinterpret_cast<const uint4*>(pos_b + uint64_t(bin_) * row_bytes));          \
  } while (0)
#define HB_ENC_XNOR(j)                                                                                \
  do {                                                                                                \
    const uint4* lp_ = reinterpret_cast<const uint4*>(lvl_b + lev[j]);                                \
    const uint4 lw4_ = kLvlSmem ? *lp_ : __ldg(lp_);                                                  \
    x[j].v[0] = ~(x[j].v[0] ^ lw4_.x); /* encoder.cpp:41 agree = ~(pos ^ lvl) */                      \
    x[j].v[1] = ~(x[j].v[1] ^ lw4_.y);                                                                \
    x[j].v[2] = ~(x[j].v[2] ^ lw4_.z);                                                                \
    x[j].v[3] = ~(x[j].v[3] ^ lw4_.w);                                                                \
  } while (0)
#pragma unroll
      for (int j = 0; j < 8; ++j) HB_ENC_ISSUE(j, my_bin, my_lev, j);  // prologue: group 0 (nb >= 1)
      for (uint32_t c0 = 0; c0 < nb; c0 += 32) {
        if (c0 + 32 + lane < nb) {  // stage the next block of 32 entries (lane j holds entry c0 + 32 + j)
          nxt_bin = sv_bins[start + c0 + 32 + lane];
          nxt_lev = sv_levels[start + c0 + 32 + lane] * row_bytes;
        } else {
          nxt_bin = 0;
          nxt_lev = null_lev;
        }
        const uint32_t cn = min(32u, nb - c0);
        const uint32_t cn_next = c0 + 32 < nb ? min(32u, nb - c0 - 32) : 0u;
        const uint32_t n_groups = 2 * ((cn + 15) / 16);  // groups of 8, an even number of them
        U4 pend8{{0, 0, 0, 0}}, pend16{{0, 0, 0, 0}};
#pragma unroll 1
        for (uint32_t g = 0; g < n_groups; ++g) {
          // the group after this one: in this block, or group 0 of the next block
          const bool in_block = g + 1 < n_groups;
          const bool has_next = in_block ? 8 * (g + 1) < cn : cn_next > 0;
          const uint32_t nb_src = in_block ? my_bin : nxt_bin, nl_src = in_block ? my_lev : nxt_lev;
          const uint32_t kb = in_block ? 8 * (g + 1) : 0;
          U4 e{{0, 0, 0, 0}};
          if (8 * g < cn) {  // a group wholly past the end of the list only completes the carry pairing
            // 8 inputs -> c[0..2] updated, one carry e of weight 8; consumed registers refill at once
            U4 ta, tb, fa, fb;
            HB_ENC_XNOR(0);
            HB_ENC_XNOR(1);
            HB_CSA(c[0], ta, c[0], x[0], x[1]);
            if (has_next) {
              HB_ENC_ISSUE(0, nb_src, nl_src, kb + 0);
              HB_ENC_ISSUE(1, nb_src, nl_src, kb + 1);
            }
            HB_ENC_XNOR(2);
            HB_ENC_XNOR(3);
            HB_CSA(c[0], tb, c[0], x[2], x[3]);
            if (has_next) {
              HB_ENC_ISSUE(2, nb_src, nl_src, kb + 2);
              HB_ENC_ISSUE(3, nb_src, nl_src, kb + 3);
            }
            HB_CSA(c[1], fa, c[1], ta, tb);
            HB_ENC_XNOR(4);
            HB_ENC_XNOR(5);
            HB_CSA(c[0], ta, c[0], x[4], x[5]);
            if (has_next) {
              HB_ENC_ISSUE(4, nb_src, nl_src, kb + 4);
              HB_ENC_ISSUE(5, nb_src, nl_src, kb + 5);
            }
            HB_ENC_XNOR(6);
            HB_ENC_XNOR(7);
            HB_CSA(c[0], tb, c[0], x[6], x[7]);
            if (has_next) {
              HB_ENC_ISSUE(6, nb_src, nl_src, kb + 6);
              HB_ENC_ISSUE(7, nb_src, nl_src, kb + 7);
            }
            HB_CSA(c[1], fb, c[1], ta, tb);
            HB_CSA(c[2], e, c[2], fa, fb);
          } else if (has_next) {
#pragma unroll
            for (int j = 0; j < 8; ++j) HB_ENC_ISSUE(j, nb_src, nl_src, kb + j);
          }
          if ((g & 1u) == 0) {
            pend8 = e;
          } else {  // the weight-8 carries of an even/odd pair meet in c[3] ...
            U4 carry;
            HB_CSA(c[3], carry, c[3], pend8, e);
            if ((g & 2u) == 0 && g + 1 < n_groups) {
              pend16 = carry;
            } else {  // ... the weight-16 carries of two pairs in c[4], and the rest ripples up
              if ((g & 2u) == 0) pend16 = U4{{0, 0, 0, 0}};  // a lone pair (at most 16 entries left)
              HB_CSA(c[4], carry, c[4], pend16, carry);
#pragma unroll
              for (int b = 5; b < NP; ++b) {
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                  const uint32_t a = c[b].v[i];
                  c[b].v[i] = a ^ carry.v[i];
                  carry.v[i] = a & carry.v[i];
                }
              }
            }
          }
        }
        my_bin = nxt_bin;
        my_lev = nxt_lev;
      }
#undef HB_ENC_ISSUE
#undef HB_ENC_XNOR
#else
      uint32_t nxt_bin = 0, nxt_lev = null_lev;
      if (lane < nb) {
        nxt_bin = sv_bins[start + lane];
        nxt_lev = sv_levels[start + lane] * row_bytes;
      }
      for (uint32_t c0 = 0; c0 < nb; c0 += 32) {
        const uint32_t my_bin = nxt_bin, my_lev = nxt_lev;
        nxt_bin = 0;
        nxt_lev = null_lev;
        if (c0 + 32 + lane < nb) {
          nxt_bin = sv_bins[start + c0 + 32 + lane];
          nxt_lev = sv_levels[start + c0 + 32 + lane] * row_bytes;
        }
        const uint32_t cn = min(32u, nb - c0);
        const uint32_t n_groups = 2 * ((cn + 15) / 16);  // groups of 8, an even number of them
        U4 pend8{{0, 0, 0, 0}}, pend16{{0, 0, 0, 0}};
#pragma unroll 1
        for (uint32_t g = 0; g < n_groups; ++g) {
          U4 e{{0, 0, 0, 0}};
          if (8 * g < cn) {  // a group wholly past the end of the list only completes the carry pairing
            U4 x[8];
            uint32_t lev[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) {  // 8 position-row gathers in flight
              const uint32_t k = 8 * g + j;
              const uint32_t bin = __shfl_sync(0xffffffffu, my_bin, k);
              lev[j] = __shfl_sync(0xffffffffu, my_lev, k);
              x[j] = ld_global_u4(reinterpret_cast<const uint4*>(pos_b + uint64_t(bin) * row_bytes));
            }
            asm volatile("" ::: "memory");  // level rows (shared memory) are fetched only as the gathers land
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const uint4* lp = reinterpret_cast<const uint4*>(lvl_b + lev[j]);
              const uint4 lw4 = kLvlSmem ? *lp : __ldg(lp);
              x[j].v[0] = ~(x[j].v[0] ^ lw4.x);  // encoder.cpp:41 agree = ~(pos ^ lvl)
              x[j].v[1] = ~(x[j].v[1] ^ lw4.y);
              x[j].v[2] = ~(x[j].v[2] ^ lw4.z);
              x[j].v[3] = ~(x[j].v[3] ^ lw4.w);
            }
            // 8 inputs -> c[0..2] updated, one carry e of weight 8
            U4 ta, tb, fa, fb;
            HB_CSA(c[0], ta, c[0], x[0], x[1]);
            HB_CSA(c[0], tb, c[0], x[2], x[3]);
            HB_CSA(c[1], fa, c[1], ta, tb);
            HB_CSA(c[0], ta, c[0], x[4], x[5]);
            HB_CSA(c[0], tb, c[0], x[6], x[7]);
            HB_CSA(c[1], fb, c[1], ta, tb);
            HB_CSA(c[2], e, c[2], fa, fb);
          }
          if ((g & 1u) == 0) {
            pend8 = e;
          } else {  // the weight-8 carries of an even/odd pair meet in c[3] ...
            U4 carry;
            HB_CSA(c[3], carry, c[3], pend8, e);
            if ((g & 2u) == 0 && g + 1 < n_groups) {
              pend16 = carry;
            } else {  // ... the weight-16 carries of two pairs in c[4], and the rest ripples up
              if ((g & 2u) == 0) pend16 = U4{{0, 0, 0, 0}};  // a lone pair (at most 16 entries left)
              HB_CSA(c[4], carry, c[4], pend16, carry);
#pragma unroll
              for (int b = 5; b < NP; ++b) {
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                  const uint32_t a = c[b].v[i];
                  c[b].v[i] = a ^ carry.v[i];
                  carry.v[i] = a & carry.v[i];
                }
              }
            }
          }
        }
      }

#endif

      // votes >= thresh, plane by plane from the top
      U4 res;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        uint32_t gt = 0, eq = 0xffffffffu;
#pragma unroll
        for (int b = NP - 1; b >= 0; --b) {
          const uint32_t cb = c[b].v[i];
          if ((thresh >> b) & 1u) {
            eq &= cb;
          } else {
            gt |= eq & cb;
            eq &= ~cb;
          }
        }
        uint32_t r = gt | eq;
        // clear tail bits >= dim (Hypervector keeps them zero, hypervector.hpp:12-15); the zero
        // padding of both codebook rows XNORs to ones and must not leak out.
        const uint32_t bit0 = (u * 4 + i) * 32;
        if (bit0 >= dim) r = 0;
        else if (bit0 + 32 > dim) r &= (1u << (dim - bit0)) - 1u;
        res.v[i] = r;
      }
      if (active) {
        const uint32_t w0 = u * 2;  // first u64 word of this slab
        const uint64_t lo = uint64_t(res.v[0]) | (uint64_t(res.v[1]) << 32);
        const uint64_t hi = uint64_t(res.v[2]) | (uint64_t(res.v[3]) << 32);
        if (vec_store) {
          if (w0 < W) *reinterpret_cast<ulonglong2*>(out_row + w0) = make_ulonglong2(lo, hi);
        } else {
          if (w0 < W) out_row[w0] = lo;
          if (w0 + 1 < W) out_row[w0 + 1] = hi;
        }
      }
    }
    if (lane == 0 && out_ok) out_ok[spec] = 1;
  }
}

// quantize host-provided SpectrumVector intensities and validate (encoder.cpp:12-14, :20-25)
__global__ void quantize_kernel(uint64_t total, const double* __restrict__ intens,
                                const uint32_t* __restrict__ bins, uint32_t levels, uint32_t n_bins,
                                uint32_t* __restrict__ out_levels, uint32_t* __restrict__ bad) {
  const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= total) return;
  const double v = intens[i];
  if (!(v >= 0.0 && v <= 1.0)) {
    atomicOr(bad, 1u);
    out_levels[i] = 0;
  } else {
    out_levels[i] = quantize_level(v, levels);
  }
  if (bins[i] >= n_bins) atomicOr(bad, 2u);
}

// hypervector.hpp:70-81: one warp per row pair
__global__ void hamming_kernel(uint64_t n, uint32_t W, uint32_t dim, const uint64_t* __restrict__ a,
                               const uint64_t* __restrict__ b, uint32_t* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const uint64_t row = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (row >= n) return;
  uint32_t diff = 0;
  for (uint32_t w = lane; w < W; w += 32) diff += __popcll(a[row * W + w] ^ b[row * W + w]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) diff += __shfl_xor_sync(0xffffffffu, diff, o);
  if (lane == 0) out[row] = dim - diff;
}

// ------------------------------------------------------------------------------------------
// host side
// ------------------------------------------------------------------------------------------

static int fill_pre_params(homs_b200_ctx* ctx, const homs_b200_preprocess_config* cfg,
                           uint32_t levels, PreParams* p) {
  HB_REQUIRE(ctx, cfg != nullptr, HOMS_B200_ERR_ARGUMENT, "preprocess config is null");
  HB_REQUIRE(ctx, cfg->max_peaks >= 1, HOMS_B200_ERR_CONFIG, "preprocess: max_peaks must be at least 1");
  HB_REQUIRE(ctx, cfg->bin_size > 0.0 && cfg->min_mz < cfg->max_mz, HOMS_B200_ERR_CONFIG,
             "preprocess: need bin_size > 0 and min_mz < max_mz");
  p->min_mz = cfg->min_mz;
  p->max_mz = cfg->max_mz;
  p->bin_size = cfg->bin_size;
  p->intensity_floor = cfg->intensity_floor;
  p->max_peaks = cfg->max_peaks;
  p->min_peaks = cfg->min_peaks;
  p->scaling = cfg->scaling;
  p->dims = homs_b200_dimension(cfg);
  p->levels = levels;
  return HOMS_B200_OK;
}

static int launch_preprocess(homs_b200_ctx* ctx, const PreParams& p, uint64_t n,
                             const uint64_t* d_off, const double* d_mz, const double* d_int,
                             uint32_t* d_bins, uint32_t* d_lev, uint32_t* d_count) {
  if (n == 0) return HOMS_B200_OK;
  const size_t per_warp = size_t(p.max_peaks) * 20;
  const size_t budget = 200 * 1024;
  int warps = static_cast<int>(std::min<size_t>(8, budget / per_warp));
  HB_REQUIRE(ctx, warps >= 1, HOMS_B200_ERR_ARGUMENT,
             "preprocess: max_peaks above 10240 is not supported by the device path");
  const size_t smem = per_warp * warps;
  HB_CUDA(ctx, cudaFuncSetAttribute(preprocess_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(smem)));
  const uint64_t want = (n + warps - 1) / warps;
  const int grid = static_cast<int>(std::min<uint64_t>(want, uint64_t(ctx->sm_count) * 16));
  {
    KernelTimer timer(ctx, HOMS_B200_KERNEL_PREPROCESS);
    preprocess_kernel<<<grid, warps * 32, smem, ctx->stream>>>(p, n, d_off, d_mz, d_int, d_bins,
                                                               d_lev, d_count, warps);
  }
  HB_LAUNCHED(ctx);
  return HOMS_B200_OK;
}

static int launch_encode(homs_b200_ctx* ctx, uint64_t n, const uint64_t* d_sv_off, uint32_t stride,
                         const uint32_t* d_bins, const uint32_t* d_lev, const uint32_t* d_count,
                         uint32_t max_count, uint64_t* d_out, uint8_t* d_ok) {
  if (n == 0) return HOMS_B200_OK;
  const Codebook& cb = ctx->cb;
  const uint32_t row_u4 = cb.S / 2;
  const size_t lvl_bytes = size_t(cb.levels + 2) * cb.S * 8;  // level rows + the no-vote row
  const int lvl_in_smem = lvl_bytes <= 96 * 1024;
  const size_t smem = lvl_in_smem ? lvl_bytes : 0;
  const int warps = HB_ENC_WARPS;
  const uint64_t want = (n + warps - 1) / warps;
  const int grid = static_cast<int>(std::min<uint64_t>(want, uint64_t(ctx->sm_count) * HB_ENC_MINB * 4));
  // 128-bit stores need an even word count and a 16-byte aligned destination
  const int vec_store = (cb.W % 2 == 0) && (reinterpret_cast<uintptr_t>(d_out) % 16 == 0);
  HB_REQUIRE(ctx, max_count <= 65535, HOMS_B200_ERR_ARGUMENT,
             "encode: more than 65535 bins per spectrum is not supported by the device path");
#define HB_ENC_LAUNCH(NP, SM)                                                                    \
  do {                                                                                           \
    HB_CUDA(ctx, cudaFuncSetAttribute(encode_kernel<NP, SM>,                                     \
                                      cudaFuncAttributeMaxDynamicSharedMemorySize,               \
                                      static_cast<int>(smem)));                                  \
    encode_kernel<NP, SM><<<grid, warps * 32, smem, ctx->stream>>>(                              \
        n, d_sv_off, stride, d_bins, d_lev, d_count, cb.d_pos.as<uint4>(), cb.d_lvl.as<uint4>(), \
        cb.levels + 1, row_u4, cb.dim, cb.W, vec_store, d_out, d_ok);                            \
  } while (0)
  {
    KernelTimer timer(ctx, HOMS_B200_KERNEL_ENCODE);
    if (max_count <= 255) {
      if (lvl_in_smem) HB_ENC_LAUNCH(8, true);
      else HB_ENC_LAUNCH(8, false);
    } else {
      if (lvl_in_smem) HB_ENC_LAUNCH(16, true);
      else HB_ENC_LAUNCH(16, false);
    }
  }
#undef HB_ENC_LAUNCH
  HB_LAUNCHED(ctx);
  return HOMS_B200_OK;
}

int encode_dev_locked(homs_b200_ctx* ctx, const homs_b200_preprocess_config* cfg, uint64_t n,
                      const uint64_t* d_off, const double* d_mz, const double* d_int,
                      uint64_t* d_out, uint8_t* d_ok) {
  HB_REQUIRE(ctx, ctx->cb.ready, HOMS_B200_ERR_STATE, "encode: no codebook uploaded");
  PreParams p;
  HB_TRY(fill_pre_params(ctx, cfg, ctx->cb.levels, &p));
  // encoder.cpp:20-22: the spectrum vector's dims must equal the codebook's spectrum_dims
  HB_REQUIRE(ctx, p.dims == ctx->cb.n_bins, HOMS_B200_ERR_INVARIANT,
             "encode: spectrum vector dims do not match codebook");
  if (n == 0) return HOMS_B200_OK;
  const size_t sv = size_t(n) * p.max_peaks * 4;
  HB_TRY(ensure(ctx, ctx->scratch[kScrSvBins], sv));
  HB_TRY(ensure(ctx, ctx->scratch[kScrSvLev], sv));
  HB_TRY(ensure(ctx, ctx->scratch[kScrSvCount], size_t(n) * 4));
  uint32_t* d_bins = ctx->scratch[kScrSvBins].as<uint32_t>();
  uint32_t* d_lev = ctx->scratch[kScrSvLev].as<uint32_t>();
  uint32_t* d_cnt = ctx->scratch[kScrSvCount].as<uint32_t>();
  HB_TRY(launch_preprocess(ctx, p, n, d_off, d_mz, d_int, d_bins, d_lev, d_cnt));
  HB_TRY(launch_encode(ctx, n, nullptr, p.max_peaks, d_bins, d_lev, d_cnt, p.max_peaks, d_out, d_ok));
  return HOMS_B200_OK;
}

// ------------------------------------------------------------------------------------------
// chunked host <-> device pipeline (pipeline.cpp:60-85 fans spectra out to threads; here chunks
// of the CSR stream through three streams so that PCIe and the kernels overlap)
// ------------------------------------------------------------------------------------------

static int pipeline_resources(homs_b200_ctx* ctx) {
  if (ctx->copy_in) return HOMS_B200_OK;
  HB_CUDA(ctx, cudaStreamCreateWithFlags(&ctx->copy_in, cudaStreamNonBlocking));
  HB_CUDA(ctx, cudaStreamCreateWithFlags(&ctx->copy_out, cudaStreamNonBlocking));
  for (int i = 0; i < 2; ++i) {
    HB_CUDA(ctx, cudaEventCreateWithFlags(&ctx->pipe_in_ready[i], cudaEventDisableTiming));
    HB_CUDA(ctx, cudaEventCreateWithFlags(&ctx->pipe_done[i], cudaEventDisableTiming));
    HB_CUDA(ctx, cudaEventCreateWithFlags(&ctx->pipe_out_free[i], cudaEventDisableTiming));
  }
  return HOMS_B200_OK;
}

int encode_pipeline(homs_b200_ctx* ctx, const homs_b200_preprocess_config* cfg, uint64_t n,
                    const uint64_t* offsets, const double* mz, const double* intensity, uint64_t* d_keep,
                    uint8_t* d_keep_ok, uint64_t* h_words, uint8_t* h_ok) {
  HB_REQUIRE(ctx, ctx->cb.ready, HOMS_B200_ERR_STATE, "encode: no codebook uploaded");
  PreParams p;
  HB_TRY(fill_pre_params(ctx, cfg, ctx->cb.levels, &p));
  HB_REQUIRE(ctx, p.dims == ctx->cb.n_bins, HOMS_B200_ERR_INVARIANT,
             "encode: spectrum vector dims do not match codebook");
  if (n == 0) return HOMS_B200_OK;
  HB_REQUIRE(ctx, offsets != nullptr, HOMS_B200_ERR_ARGUMENT, "encode: null offsets");
  const uint64_t total = offsets[n] - offsets[0];
  HB_REQUIRE(ctx, total == 0 || (mz && intensity), HOMS_B200_ERR_ARGUMENT, "encode: null peaks");
  const uint32_t W = ctx->cb.W;

  // chunks: at most 64 Ki spectra and about 4 Mi peaks (64 MB of m/z + intensity) each
  constexpr uint64_t kMaxSpectra = 64 * 1024, kMaxPeaks = 4ull << 20;
  std::vector<uint64_t> cuts{0};
  uint64_t max_n = 0, max_peaks = 0;
  for (uint64_t a = 0; a < n;) {
    uint64_t b = a + 1;
    while (b < n && b - a < kMaxSpectra && offsets[b + 1] - offsets[a] <= kMaxPeaks) ++b;
    HB_REQUIRE(ctx, offsets[b] >= offsets[a], HOMS_B200_ERR_ARGUMENT, "encode: offsets must be non-decreasing");
    max_n = std::max(max_n, b - a);
    max_peaks = std::max(max_peaks, offsets[b] - offsets[a]);
    cuts.push_back(b);
    a = b;
  }
  const bool to_host = h_words != nullptr || h_ok != nullptr;
  const bool out_slots = d_keep == nullptr;  // rows live in a slot only until they are copied out
  HB_TRY(pipeline_resources(ctx));
  const size_t in_bytes = (max_n + 1) * 8 + max_peaks * 16;
  const size_t out_bytes = out_slots ? max_n * W * 8 + max_n : (d_keep_ok ? 0 : max_n);
  for (int s = 0; s < 2; ++s) {
    HB_TRY(ensure(ctx, ctx->scratch[kScrPipeIn0 + s], in_bytes));
    if (out_bytes) HB_TRY(ensure(ctx, ctx->scratch[kScrPipeOut0 + s], out_bytes));
  }
  // sized once so that no chunk reallocates under the pipeline
  HB_TRY(ensure(ctx, ctx->scratch[kScrSvBins], size_t(max_n) * p.max_peaks * 4));
  HB_TRY(ensure(ctx, ctx->scratch[kScrSvLev], size_t(max_n) * p.max_peaks * 4));
  HB_TRY(ensure(ctx, ctx->scratch[kScrSvCount], size_t(max_n) * 4));

  cudaStream_t cs = ctx->stream, in = ctx->copy_in, out = ctx->copy_out;
  for (size_t c = 0; c + 1 < cuts.size(); ++c) {
    const int s = static_cast<int>(c & 1);
    const uint64_t a = cuts[c], b = cuts[c + 1], cn = b - a;
    const uint64_t p0 = offsets[a], np = offsets[b] - p0;
    auto* d_off = ctx->scratch[kScrPipeIn0 + s].as<uint64_t>();
    auto* d_mz = reinterpret_cast<double*>(d_off + (max_n + 1));
    auto* d_int = d_mz + max_peaks;
    if (c >= 2) HB_CUDA(ctx, cudaStreamWaitEvent(in, ctx->pipe_done[s], 0));  // slot inputs consumed
    HB_CUDA(ctx, cudaMemcpyAsync(d_off, offsets + a, (cn + 1) * 8, cudaMemcpyHostToDevice, in));
    if (np) {
      HB_CUDA(ctx, cudaMemcpyAsync(d_mz, mz + p0, np * 8, cudaMemcpyHostToDevice, in));
      HB_CUDA(ctx, cudaMemcpyAsync(d_int, intensity + p0, np * 8, cudaMemcpyHostToDevice, in));
    }
    HB_CUDA(ctx, cudaEventRecord(ctx->pipe_in_ready[s], in));

    uint64_t* d_rows;
    uint8_t* d_ok;
    if (out_slots) {
      d_rows = ctx->scratch[kScrPipeOut0 + s].as<uint64_t>();
      d_ok = reinterpret_cast<uint8_t*>(d_rows + max_n * W);
    } else {
      d_rows = d_keep + a * W;
      d_ok = d_keep_ok ? d_keep_ok + a : ctx->scratch[kScrPipeOut0 + s].as<uint8_t>();
    }
    HB_CUDA(ctx, cudaStreamWaitEvent(cs, ctx->pipe_in_ready[s], 0));
    if (to_host && c >= 2) HB_CUDA(ctx, cudaStreamWaitEvent(cs, ctx->pipe_out_free[s], 0));
    // the kernels index peaks with the absolute offsets: shift the slot pointers by -p0
    HB_TRY(encode_dev_locked(ctx, cfg, cn, d_off, d_mz - p0, d_int - p0, d_rows, d_ok));
    HB_CUDA(ctx, cudaEventRecord(ctx->pipe_done[s], cs));

    if (to_host) {
      HB_CUDA(ctx, cudaStreamWaitEvent(out, ctx->pipe_done[s], 0));
      if (h_words)
        HB_CUDA(ctx, cudaMemcpyAsync(h_words + a * W, d_rows, cn * W * 8, cudaMemcpyDeviceToHost, out));
      if (h_ok) HB_CUDA(ctx, cudaMemcpyAsync(h_ok + a, d_ok, cn, cudaMemcpyDeviceToHost, out));
      HB_CUDA(ctx, cudaEventRecord(ctx->pipe_out_free[s], out));
    }
  }
  HB_CUDA(ctx, cudaStreamSynchronize(in));
  HB_CUDA(ctx, cudaStreamSynchronize(cs));
  HB_CUDA(ctx, cudaStreamSynchronize(out));
  if (h_ok)  // the reference's encode_spectra lets quantize_intensity's exception escape (pipeline.cpp:67-72)
    for (uint64_t i = 0; i < n; ++i)
      HB_REQUIRE(ctx, h_ok[i] != HOMS_B200_OK_FLAG_INVARIANT, HOMS_B200_ERR_INVARIANT,
                 "quantize_intensity: intensity outside [0, 1]");
  return HOMS_B200_OK;
}

}  // namespace hb

using namespace hb;

extern "C" {

int homs_b200_codebook_upload(homs_b200_ctx* ctx, uint32_t dim, uint32_t n_bins, uint32_t levels,
                              const uint64_t* pos, const uint64_t* lvl) {
  if (!ctx) return HOMS_B200_ERR_ARGUMENT;
  Lock lock(ctx);
  if (is_group(ctx))  // replicas of the codebook on every device (encoding needs no collective)
    return group_for_each(ctx, [&](uint32_t, homs_b200_ctx* m) -> int {
      return codebook_upload_locked(m, dim, n_bins, levels, pos, lvl);
    });
  return codebook_upload_locked(ctx, dim, n_bins, levels, pos, lvl);
}

}  // extern "C"

int hb::codebook_upload_locked(homs_b200_ctx* ctx, uint32_t dim, uint32_t n_bins, uint32_t levels,
                               const uint64_t* pos, const uint64_t* lvl) {
  HB_REQUIRE(ctx, pos && lvl, HOMS_B200_ERR_ARGUMENT, "codebook_upload: null codebook");
  HB_REQUIRE(ctx, dim >= 1 && n_bins >= 1 && levels >= 1, HOMS_B200_ERR_ARGUMENT,
             "codebook_upload: dim, n_bins and levels must be positive");
  Codebook& cb = ctx->cb;
  cb.ready = false;
  cb.dim = dim;
  cb.n_bins = n_bins;
  cb.levels = levels;
  cb.W = words_for(dim);
  cb.S = stride_for(dim);
  HB_TRY(ensure(ctx, cb.d_pos, size_t(n_bins) * cb.S * 8));
  // one row more than the reference's table: ~position[0] (all ones in the padding), the level an
  // entry past the end of a spectrum's list is given so that it XNORs to zero votes (encode_kernel)
  HB_TRY(ensure(ctx, cb.d_lvl, size_t(levels + 2) * cb.S * 8));
  HB_TRY(upload_rows(ctx, cb.d_pos.as<uint64_t>(), pos, n_bins, cb.W, cb.S));
  HB_TRY(upload_rows(ctx, cb.d_lvl.as<uint64_t>(), lvl, levels + 1, cb.W, cb.S));
  std::vector<uint64_t> no_vote(cb.S, ~0ull);
  for (uint32_t w = 0; w < cb.W; ++w) no_vote[w] = ~pos[w];
  HB_CUDA(ctx, cudaMemcpyAsync(cb.d_lvl.as<uint64_t>() + size_t(levels + 1) * cb.S, no_vote.data(), size_t(cb.S) * 8,
                               cudaMemcpyHostToDevice, ctx->stream));
  HB_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  cb.ready = true;
  return HOMS_B200_OK;
}

extern "C" {

int homs_b200_encode_batch_dev(homs_b200_ctx* ctx, const homs_b200_preprocess_config* cfg,
                               uint64_t n, uint64_t n_peaks_total, const uint64_t* d_offsets,
                               const double* d_mz, const double* d_intensity,
                               uint64_t* d_out_words, uint8_t* d_out_ok) {
  (void)n_peaks_total;
  if (!ctx) return HOMS_B200_ERR_ARGUMENT;
  Lock lock(ctx);
  HB_REQUIRE(ctx, n == 0 || (d_offsets && d_out_words), HOMS_B200_ERR_ARGUMENT,
             "encode_batch_dev: null argument");
  return encode_dev_locked(ctx, cfg, n, d_offsets, d_mz, d_intensity, d_out_words, d_out_ok);
}

int homs_b200_encode_batch(homs_b200_ctx* ctx, const homs_b200_preprocess_config* cfg, uint64_t n,
                           const uint64_t* offsets, const double* mz, const double* intensity,
                           uint64_t* out_words, uint8_t* out_ok) {
  if (!ctx) return HOMS_B200_ERR_ARGUMENT;
  Lock lock(ctx);
  HB_REQUIRE(ctx, n == 0 || (offsets && out_words && out_ok), HOMS_B200_ERR_ARGUMENT,
             "encode_batch: null argument");
  HB_REQUIRE(ctx, n == 0 || offsets[0] == 0, HOMS_B200_ERR_ARGUMENT, "encode_batch: offsets[0] must be 0");
  if (is_group(ctx) && n >= 2 * ctx->members.size()) {
    // spectra split evenly over the devices, every member streams its slice through its own
    // three-stream pipeline (encode_spectra's thread fan-out, pipeline.cpp:66-73, across GPUs)
    const uint64_t G = ctx->members.size();
    const uint32_t W = ctx->cb.W;
    return group_for_each(ctx, [&](uint32_t g, homs_b200_ctx* m) -> int {
      const uint64_t a = n * g / G, b = n * (g + 1) / G;
      return encode_pipeline(m, cfg, b - a, offsets + a, mz, intensity, nullptr, nullptr, out_words + a * W,
                             out_ok + a);
    });
  }
  return encode_pipeline(ctx, cfg, n, offsets, mz, intensity, nullptr, nullptr, out_words, out_ok);
}

int homs_b200_preprocess_batch(homs_b200_ctx* ctx, const homs_b200_preprocess_config* cfg,
                               uint32_t levels, uint64_t n, const uint64_t* offsets,
                               const double* mz, const double* intensity, uint32_t* out_bins,
                               uint32_t* out_levels, uint32_t* out_count) {
  if (!ctx) return HOMS_B200_ERR_ARGUMENT;
  Lock lock(ctx);
  PreParams p;
  HB_TRY(fill_pre_params(ctx, cfg, levels, &p));
  if (n == 0) return HOMS_B200_OK;
  HB_REQUIRE(ctx, offsets && out_bins && out_levels && out_count, HOMS_B200_ERR_ARGUMENT,
             "preprocess_batch: null argument");
  const uint64_t total = offsets[n];
  const size_t sv = size_t(n) * p.max_peaks * 4;
  HB_TRY(ensure(ctx, ctx->scratch[kScrOffsets], (n + 1) * 8));
  HB_TRY(ensure(ctx, ctx->scratch[kScrMz], total * 8));
  HB_TRY(ensure(ctx, ctx->scratch[kScrInt], total * 8));
  HB_TRY(ensure(ctx, ctx->scratch[kScrSvBins], sv));
  HB_TRY(ensure(ctx, ctx->scratch[kScrSvLev], sv));
  HB_TRY(ensure(ctx, ctx->scratch[kScrSvCount], size_t(n) * 4));
  auto* d_off = ctx->scratch[kScrOffsets].as<uint64_t>();
  auto* d_mz = ctx->scratch[kScrMz].as<double>();
  auto* d_int = ctx->scratch[kScrInt].as<double>();
  auto* d_bins = ctx->scratch[kScrSvBins].as<uint32_t>();
  auto* d_lev = ctx->scratch[kScrSvLev].as<uint32_t>();
  auto* d_cnt = ctx->scratch[kScrSvCount].as<uint32_t>();
  HB_CUDA(ctx, cudaMemcpyAsync(d_off, offsets, (n + 1) * 8, cudaMemcpyHostToDevice, ctx->stream));
  if (total) {
    HB_CUDA(ctx, cudaMemcpyAsync(d_mz, mz, total * 8, cudaMemcpyHostToDevice, ctx->stream));
    HB_CUDA(ctx, cudaMemcpyAsync(d_int, intensity, total * 8, cudaMemcpyHostToDevice, ctx->stream));
  }
  HB_CUDA(ctx, cudaMemsetAsync(d_bins, 0, sv, ctx->stream));
  HB_CUDA(ctx, cudaMemsetAsync(d_lev, 0, sv, ctx->stream));
  HB_TRY(launch_preprocess(ctx, p, n, d_off, d_mz, d_int, d_bins, d_lev, d_cnt));
  HB_CUDA(ctx, cudaMemcpyAsync(out_bins, d_bins, sv, cudaMemcpyDeviceToHost, ctx->stream));
  HB_CUDA(ctx, cudaMemcpyAsync(out_levels, d_lev, sv, cudaMemcpyDeviceToHost, ctx->stream));
  HB_CUDA(ctx, cudaMemcpyAsync(out_count, d_cnt, size_t(n) * 4, cudaMemcpyDeviceToHost, ctx->stream));
  HB_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  for (uint64_t i = 0; i < n; ++i)
    HB_REQUIRE(ctx, out_count[i] != kInvalidCount, HOMS_B200_ERR_INVARIANT,
               "quantize_intensity: intensity outside [0, 1]");
  return HOMS_B200_OK;
}

int homs_b200_encode_vectors(homs_b200_ctx* ctx, uint64_t n, const uint64_t* sv_offsets,
                             const uint32_t* bins, const double* intensities,
                             uint64_t* out_words) {
  if (!ctx) return HOMS_B200_ERR_ARGUMENT;
  Lock lock(ctx);
  HB_REQUIRE(ctx, ctx->cb.ready, HOMS_B200_ERR_STATE, "encode: no codebook uploaded");
  if (n == 0) return HOMS_B200_OK;
  HB_REQUIRE(ctx, sv_offsets && bins && intensities && out_words, HOMS_B200_ERR_ARGUMENT,
             "encode_vectors: null argument");
  uint32_t max_count = 0;
  for (uint64_t i = 0; i < n; ++i) {
    const uint64_t c = sv_offsets[i + 1] - sv_offsets[i];
    HB_REQUIRE(ctx, c >= 1, HOMS_B200_ERR_INVARIANT, "encode: empty spectrum vector");  // encoder.cpp:23-25
    HB_REQUIRE(ctx, c <= 65535, HOMS_B200_ERR_ARGUMENT, "encode: more than 65535 bins per spectrum");
    max_count = std::max<uint32_t>(max_count, static_cast<uint32_t>(c));
  }
  const uint64_t total = sv_offsets[n];
  const uint32_t W = ctx->cb.W;
  HB_TRY(ensure(ctx, ctx->scratch[kScrOffsets], (n + 1) * 8));
  HB_TRY(ensure(ctx, ctx->scratch[kScrInt], total * 8));
  HB_TRY(ensure(ctx, ctx->scratch[kScrSvBins], total * 4));
  HB_TRY(ensure(ctx, ctx->scratch[kScrSvLev], total * 4));
  HB_TRY(ensure(ctx, ctx->scratch[kScrEncOut], n * W * 8));
  HB_TRY(ensure(ctx, ctx->scratch[kScrMisc], 16));
  auto* d_off = ctx->scratch[kScrOffsets].as<uint64_t>();
  auto* d_int = ctx->scratch[kScrInt].as<double>();
  auto* d_bins = ctx->scratch[kScrSvBins].as<uint32_t>();
  auto* d_lev = ctx->scratch[kScrSvLev].as<uint32_t>();
  auto* d_out = ctx->scratch[kScrEncOut].as<uint64_t>();
  auto* d_bad = ctx->scratch[kScrMisc].as<uint32_t>();
  HB_CUDA(ctx, cudaMemcpyAsync(d_off, sv_offsets, (n + 1) * 8, cudaMemcpyHostToDevice, ctx->stream));
  HB_CUDA(ctx, cudaMemcpyAsync(d_int, intensities, total * 8, cudaMemcpyHostToDevice, ctx->stream));
  HB_CUDA(ctx, cudaMemcpyAsync(d_bins, bins, total * 4, cudaMemcpyHostToDevice, ctx->stream));
  HB_CUDA(ctx, cudaMemsetAsync(d_bad, 0, 4, ctx->stream));
  quantize_kernel<<<static_cast<unsigned>((total + 255) / 256), 256, 0, ctx->stream>>>(
      total, d_int, d_bins, ctx->cb.levels, ctx->cb.n_bins, d_lev, d_bad);
  HB_LAUNCHED(ctx);
  uint32_t bad = 0;
  HB_CUDA(ctx, cudaMemcpyAsync(&bad, d_bad, 4, cudaMemcpyDeviceToHost, ctx->stream));
  HB_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  HB_REQUIRE(ctx, !(bad & 1u), HOMS_B200_ERR_INVARIANT, "quantize_intensity: intensity outside [0, 1]");
  HB_REQUIRE(ctx, !(bad & 2u), HOMS_B200_ERR_INVARIANT, "encode: spectrum vector dims do not match codebook");
  HB_TRY(launch_encode(ctx, n, d_off, 0, d_bins, d_lev, nullptr, max_count, d_out, nullptr));
  HB_CUDA(ctx, cudaMemcpyAsync(out_words, d_out, n * W * 8, cudaMemcpyDeviceToHost, ctx->stream));
  HB_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  return HOMS_B200_OK;
}

int homs_b200_hamming_similarity(homs_b200_ctx* ctx, uint32_t dim, uint64_t n, const uint64_t* a,
                                 const uint64_t* b, uint32_t* out) {
  if (!ctx) return HOMS_B200_ERR_ARGUMENT;
  Lock lock(ctx);
  if (n == 0) return HOMS_B200_OK;
  HB_REQUIRE(ctx, a && b && out, HOMS_B200_ERR_ARGUMENT, "hamming_similarity: null argument");
  const uint32_t W = words_for(dim);
  HB_TRY(ensure(ctx, ctx->scratch[kScrEncOut], n * W * 8));
  HB_TRY(ensure(ctx, ctx->scratch[kScrMz], n * W * 8));
  HB_TRY(ensure(ctx, ctx->scratch[kScrSvCount], n * 4));
  auto* d_a = ctx->scratch[kScrEncOut].as<uint64_t>();
  auto* d_b = ctx->scratch[kScrMz].as<uint64_t>();
  auto* d_o = ctx->scratch[kScrSvCount].as<uint32_t>();
  HB_CUDA(ctx, cudaMemcpyAsync(d_a, a, n * W * 8, cudaMemcpyHostToDevice, ctx->stream));
  HB_CUDA(ctx, cudaMemcpyAsync(d_b, b, n * W * 8, cudaMemcpyHostToDevice, ctx->stream));
  const uint64_t threads = n * 32;
  hamming_kernel<<<static_cast<unsigned>((threads + 255) / 256), 256, 0, ctx->stream>>>(n, W, dim, d_a,
                                                                                       d_b, d_o);
  HB_LAUNCHED(ctx);
  HB_CUDA(ctx, cudaMemcpyAsync(out, d_o, n * 4, cudaMemcpyDeviceToHost, ctx->stream));
  HB_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  return HOMS_B200_OK;
}

}  // extern "C"
