// Stable LSD radix sort of (key, u32 value) pairs on the context's stream (radix.cu).
#pragma once

#include <cstddef>
#include <cstdint>

struct homs_b200_ctx;

namespace hb {

// bytes of device scratch radix_sort_pairs needs for n items
size_t radix_temp_bytes(uint64_t n);

// Sorts n pairs by key bits [begin_bit, end_bit), stable, ping-ponging between the a and b arrays
// (ceil((end_bit - begin_bit) / 8) passes).  *result_in_b tells where the sorted pairs ended up.
// first_vals_iota: the input values are 0, 1, 2, ... and vals_a need not be initialised.
// K = uint8_t, uint32_t or uint64_t.  Stream-ordered, no host synchronisation.
template <typename K>
int radix_sort_pairs(homs_b200_ctx* ctx, K* keys_a, K* keys_b, uint32_t* vals_a, uint32_t* vals_b, uint64_t n,
                     int begin_bit, int end_bit, void* d_temp, bool first_vals_iota, bool* result_in_b);

}  // namespace hb
