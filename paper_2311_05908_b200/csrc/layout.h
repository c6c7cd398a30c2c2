// layout.h -- shared-memory table layouts used by both the host planner
// (which writes the tables) and the kernels (which read them).
#pragma once
#include <cstdint>

#if defined(__CUDACC__)
#define FC_HD __host__ __device__ __forceinline__
#else
#define FC_HD inline
#endif

namespace fc {

// Bank-conflict-free layout of a row-major table of 16-byte chunks read
// "one row per lane": chunk j of row r lives at chunk (j ^ (r & 7)) when a row
// has >= 8 chunks, and at the 128B-swizzled position for 4-chunk rows.
template <int CPR>
FC_HD uint32_t tab_off(uint32_t row, uint32_t j) {
  if constexpr (CPR >= 8) {
    return (row * CPR + (j ^ (row & 7u))) * 16u;
  } else {
    static_assert(CPR == 4, "rows of 4 or >= 8 chunks");
    return (row * 4u + (j ^ ((row >> 1) & 3u))) * 16u;
  }
}

FC_HD uint32_t tab_off_rt(uint32_t cpr, uint32_t row, uint32_t j) {
  return cpr >= 8 ? (row * cpr + (j ^ (row & 7u))) * 16u : (row * cpr + (j ^ ((row >> 1) & 3u))) * 16u;
}

}  // namespace fc
