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

// k_f block of a single-pass order-3 plan (K_f[f' + 2048 k0] / L0 -- the 1/L0
// of the outer inverse DFT folded in --, f' = k2 + 64 k1, one block per
// (head, k0)): float4 {kr(k1), kr(k1+1), ki(k1), ki(k1+1)} of
// k1 pair kp = k1 / 2 at index ((kp / 4) * 64 + k2) * 4 + kp % 4.  The
// L0 = 4 epilogue-2 thread (k2 = lane / 4 + ..., kp % 4 = lane % 4, one
// 16x256b TMEM fragment) reads one float4 per k0 and 4 k1 pairs: 8 lanes
// cover 128 contiguous bytes (conflict-free from shared memory, full lines
// from L2).  16 KB per block; blocks are tab_stride(16) * 64 bytes apart.
FC_HD uint32_t dit_kf_off(uint32_t k2, uint32_t kp) { return (((kp >> 2) * 64u + k2) * 4u + (kp & 3u)) * 16u; }

}  // namespace fc
