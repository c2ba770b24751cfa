// Register-resident top-k lists shared by the tensor engines' drain (search_tc.cu) and the direct
// engine (search.cu).  Reference order of two candidates of one query (search.cpp:133-146): score
// desc, |mass diff| asc, id asc, ordinal asc; here: dot desc (any value monotone in the score),
// then (|q - r| bits, id_rank) asc.
#pragma once
#include "common.cuh"

namespace hb {

__device__ __forceinline__ bool key_less(uint64_t ad1, uint32_t rk1, uint64_t ad2, uint32_t rk2) {
  return ad1 != ad2 ? ad1 < ad2 : rk1 < rk2;
}

// The KM best candidates of one query seen so far, ascending in the reference key
// (distance asc == dot desc, |mass diff| asc, id_rank asc), held in REGISTERS: every access is
// fully unrolled, so an insert is ~6 KM ALU operations and no memory traffic (a local-memory
// list cost several dependent L2 round trips per insert with the L1 carved down to its minimum).
// Only (dot, row) are kept; the rest of the key is fetched when two dots tie and when the list is
// written out.  Unused entries hold kTcNoDot / kNone.  The caller needs the best k <= KM only.
constexpr int kTcNoDot = -(1 << 30);  // below every real dot (|dot| <= dim <= 65536), exact in fp32
template <int KM>
struct TcTopK {
  int dot[KM];
  uint32_t row[KM];
};

// candidate row a before row b among equal dots: |mass diff|, then id, then ordinal (search.cpp:137-145)
__device__ __forceinline__ bool tc_row_before(const double* __restrict__ lib_mz, const uint32_t* __restrict__ lib_rank,
                                              double qmz, uint32_t a, uint32_t b) {
  const uint64_t ada = static_cast<uint64_t>(__double_as_longlong(fabs(qmz - lib_mz[a])));
  const uint64_t adb = static_cast<uint64_t>(__double_as_longlong(fabs(qmz - lib_mz[b])));
  return ada != adb ? ada < adb : lib_rank[a] < lib_rank[b];
}

template <int KM>
__device__ __forceinline__ void tc_topk_insert(TcTopK<KM>& l, const double* __restrict__ lib_mz,
                                               const uint32_t* __restrict__ lib_rank, double qmz, int dot,
                                               uint32_t row) {
  uint32_t ahead = 0;  // entries that stay in front of the new one (a prefix: the list is sorted)
#pragma unroll
  for (int i = 0; i < KM; ++i) {
    bool a = l.dot[i] > dot;
    if (l.dot[i] == dot) a = tc_row_before(lib_mz, lib_rank, qmz, l.row[i], row);  // rare
    ahead += a ? 1u : 0u;
  }
#pragma unroll
  for (int i = KM - 1; i >= 0; --i) {
    if (uint32_t(i) > ahead) {
      if (i > 0) {
        l.dot[i] = l.dot[i - 1];
        l.row[i] = l.row[i - 1];
      }
    } else if (uint32_t(i) == ahead) {
      l.dot[i] = dot;
      l.row[i] = row;
    }
  }
}

// dot of the k-th entry (k >= 1), kTcNoDot while the list holds fewer than k candidates
template <int KM>
__device__ __forceinline__ int tc_topk_kth(const TcTopK<KM>& l, uint32_t k) {
  int d = l.dot[0];
#pragma unroll
  for (int i = 1; i < KM; ++i) {
    int t = l.dot[i];
    asm("" : "+r"(t));  // keeps this a chain of selects: a dynamic index would move the list to local memory
    d = uint32_t(i) == k - 1 ? t : d;
  }
  return d;
}

}  // namespace hb
