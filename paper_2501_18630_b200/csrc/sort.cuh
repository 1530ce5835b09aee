// Stable LSD radix sort (8-bit digits, sort.cu) shared by the depth export and the codec.
#pragma once

#include "common.cuh"

namespace bsr {

template <typename K>
struct SortArgs {
    K *keys[2];
    uint32_t *vals[2];
    const uint32_t *count;            // device element count
    const uint32_t *bias_inv;         // if non-null: bias = ~(*bias_inv) (min key)
    uint32_t *hist;                   // [passes][256], zeroed; becomes exclusive offsets
    uint32_t *plan;                   // [passes + 1]
    uint32_t *status;                 // [passes][max_parts][256], zeroed
    uint32_t *tickets;                // [passes], zeroed
    int passes;
    int items;                        // keys per thread (4 or 16), see sort_items()
    int64_t max_parts;
};

// Sorts keys[0] / vals[0] (count elements, at most cap); the result is in keys[s] /
// vals[s] with s = plan[passes] & 1 (device), see sort_plan_kernel.
template <typename K>
int launch_sort(const SortArgs<K> &a, int64_t cap, cudaStream_t st);

}  // namespace bsr
