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
// "one row per lane": rows are padded by one chunk, so consecutive rows start
// 4 banks apart and 8 lanes reading chunk j of 8 consecutive rows hit 8
// distinct 4-bank groups.  Chunk addresses stay base + j*16 (immediates).
FC_HD uint32_t tab_stride(uint32_t cpr) { return cpr * 16u + 16u; }
FC_HD uint32_t tab_off_rt(uint32_t cpr, uint32_t row, uint32_t j) { return row * tab_stride(cpr) + j * 16u; }
template <int CPR>
FC_HD uint32_t tab_off(uint32_t row, uint32_t j) { return row * (CPR * 16u + 16u) + j * 16u; }

}  // namespace fc
