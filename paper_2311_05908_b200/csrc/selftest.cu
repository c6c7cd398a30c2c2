// selftest.cu -- device self-test hooks for the sm_100a primitives the fused
// FFT-conv kernels are built from (not part of the fftconv C-ABI).
//
// fcst_mma(): one CTA stages A (M x K) and B (K x N) fp16 into shared memory
// in the SWIZZLE_NONE canonical layout selected by a_mn / b_mn, issues
// K/16 tcgen05.mma.kind::f16 instructions accumulating into TMEM, and reads
// D (M x N fp32) back with tcgen05.ld.  Used by tests/test_gpu_primitives.py
// to pin the descriptor encodings against a host matmul, including the A-in-TMEM
// (ts) form and the M = 64 lane layout.
#include <cuda_runtime.h>
#include "sm100.cuh"

namespace {

__device__ uint32_t canon_off(int r, int k, int R, int K, bool mn_major) {
  // r = M (or N) index, k = K index; returns byte offset.
  if (mn_major) {
    const uint32_t sbo = 128, lbo = (R / 8) * 128;
    return (r / 8) * sbo + (k / 8) * lbo + (k % 8) * 16 + (r % 8) * 2;
  } else {
    const uint32_t lbo = 128, sbo = (K / 8) * 128;
    return (r / 8) * sbo + (k / 8) * lbo + (r % 8) * 16 + (k % 8) * 2;
  }
}

__global__ void __launch_bounds__(128, 1) mma_selftest_kernel(const __half* A, const __half* B, float* D, int M,
                                                                 int N, int K, int a_mn, int b_mn, int a_tmem,
                                                                 int d_lane) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  uint8_t* sA = smem;
  uint8_t* sB = smem + M * K * 2;
  const int tid = threadIdx.x;
  if (!a_tmem) {
    for (int i = tid; i < M * K; i += blockDim.x) {
      int m = i / K, k = i % K;
      *reinterpret_cast<__half*>(sA + canon_off(m, k, M, K, a_mn)) = A[i];
    }
  }
  for (int i = tid; i < K * N; i += blockDim.x) {
    int k = i / N, n = i % N;
    *reinterpret_cast<__half*>(sB + canon_off(n, k, N, K, b_mn)) = B[i];
  }
  if (tid == 0) {
    fc::mbar_init(&bar, 1);
    fc::fence_barrier_init();
  }
  if (tid < 32) fc::tmem_alloc<512>(&tmem_base);
  fc::fence_async_smem();
  fc::tc_fence_before();
  __syncthreads();
  fc::tc_fence_after();
  const uint32_t tbase = tmem_base;
  const int warp = tid / 32;
  const uint32_t a_col = 256;  // A operand columns when staged in TMEM
  if (a_tmem) {                // row m in lane m (M == 128), two fp16 per column
    for (int c = 0; c < K / 2; c += 4) {
      uint32_t v[4];
      for (int j = 0; j < 4; ++j) {
        __half2 h = __halves2half2(A[tid * K + 2 * (c + j)], A[tid * K + 2 * (c + j) + 1]);
        v[j] = *reinterpret_cast<uint32_t*>(&h);
      }
      fc::tmem_st4(tbase + ((uint32_t)(warp * 32) << 16) + a_col + c, v[0], v[1], v[2], v[3]);
    }
    fc::tmem_st_wait();
    fc::tc_fence_before();
    __syncthreads();
    fc::tc_fence_after();
  }
  const uint32_t dt = tbase + ((uint32_t)d_lane << 16);
  if (tid == 0) {
    const uint32_t idesc = fc::idesc_f16(M, N, a_mn, b_mn);
    const uint32_t a0 = fc::smem_u32(sA), b0 = fc::smem_u32(sB);
    for (int s = 0; s < K / 16; ++s) {
      uint64_t ad, bd;
      if (a_mn) ad = fc::smem_desc(a0 + 2 * s * (M / 8) * 128, (M / 8) * 128, 128);
      else      ad = fc::smem_desc(a0 + s * 256, 128, (K / 8) * 128);
      if (b_mn) bd = fc::smem_desc(b0 + 2 * s * (N / 8) * 128, (N / 8) * 128, 128);
      else      bd = fc::smem_desc(b0 + s * 256, 128, (K / 8) * 128);
      if (a_tmem) fc::mma_f16_ts(dt, tbase + a_col + 8 * s, bd, idesc, s > 0);
      else        fc::mma_f16_ss(dt, ad, bd, idesc, s > 0);
    }
    fc::mma_commit(&bar);
  }
  fc::mbar_wait(&bar, 0);
  fc::tc_fence_after();
  // D row r: lane r (M == 128); lane 32 (r / 16) + r % 16 + d_lane (M == 64)
  const int lane = tid % 32;
  int row = -1;
  if (M == 128) row = tid;
  else if (lane >= d_lane && lane < d_lane + 16) row = warp * 16 + lane - d_lane;
  for (int c = 0; c < N; c += 8) {
    float v[8];
    fc::tmem_ld8(tbase + ((uint32_t)(warp * 32) << 16) + c, v);
    fc::tmem_ld_wait();
    if (row >= 0)
      for (int j = 0; j < 8; ++j) D[row * N + c + j] = v[j];
  }
  fc::tc_fence_before();
  __syncthreads();
  if (tid < 32) fc::tmem_dealloc<512>(tbase);
}

}  // namespace

// M in {64, 128}; a_tmem: A staged in TMEM (M == 128 only); d_lane: TMEM lane
// offset of D (0 or 16, M == 64 only).
extern "C" int fcst_mma(const void* A, const void* B, void* D, int M, int N, int K, int a_mn, int b_mn, int a_tmem,
                        int d_lane) {
  if ((M != 128 && M != 64) || N % 16 || N < 16 || N > 256 || K % 16 || K > 128) return 1;
  if (a_tmem && (M != 128 || a_mn)) return 1;
  if (M == 128 && d_lane) return 1;
  size_t smem = (size_t)(M + N) * K * 2;
  cudaFuncSetAttribute(mma_selftest_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  mma_selftest_kernel<<<1, 128, smem>>>((const __half*)A, (const __half*)B, (float*)D, M, N, K, a_mn, b_mn, a_tmem,
                                        d_lane);
  cudaError_t e = cudaDeviceSynchronize();
  return e == cudaSuccess ? 0 : 100 + (int)e;
}

// ---------------------------------------------------------------- microbenchmarks
// (experiments: TMEM read throughput and back-to-back MMA cost)
namespace {
__global__ void __launch_bounds__(512, 1) tmem_ld_bench_kernel(int iters, int nwarps, long long* out) {
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid / 32;
  if (warp == 0) fc::tmem_alloc<512>(&tmem_base);
  fc::tc_fence_before();
  __syncthreads();
  fc::tc_fence_after();
  const uint32_t t = tmem_base + ((uint32_t)((warp & 3) * 32) << 16) + (warp >> 2) * 64;
  float acc = 0.f;
  __syncthreads();
  long long c0 = clock64();
  if (warp < nwarps) {
    for (int i = 0; i < iters; ++i) {
      float v[32];
      fc::tmem_ld16(t, v);
      fc::tmem_ld16(t + 16, v + 16);
      fc::tmem_ld_wait();
      for (int j = 0; j < 32; ++j) acc += v[j];
    }
  }
  __syncthreads();
  long long c1 = clock64();
  if (tid == 0) out[0] = c1 - c0;
  if (acc == 12345.f) out[1] = 1;
  fc::tc_fence_before();
  __syncthreads();
  if (warp == 0) fc::tmem_dealloc<512>(tmem_base);
}

__global__ void __launch_bounds__(128, 1) mma_rate_kernel(int nmma, int N, int ts, long long* out, int M = 128) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x;
  for (int i = tid; i < 16384; i += 128) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  if (tid == 0) {
    fc::mbar_init(&bar, 1);
    fc::fence_barrier_init();
  }
  if (tid < 32) fc::tmem_alloc<512>(&tmem_base);
  fc::fence_async_smem();
  fc::tc_fence_before();
  __syncthreads();
  fc::tc_fence_after();
  const uint32_t tb = fc::warp_uniform(tmem_base);
  if (tid < 32 && fc::elect_one()) {
    const uint32_t a0 = fc::smem_u32(smem), b0 = a0 + 32768;
    const uint64_t ad = fc::smem_desc(a0, 128, 256), bd = fc::smem_desc(b0, 128, 256);
    long long c0 = clock64();
    for (int r = 0; r < 2; ++r) {
      if (r == 1) c0 = clock64();
      for (int s = 0; s < nmma; ++s) {
        const uint32_t idesc = fc::idesc_f16(M, N, false, false);
        if (ts) fc::mma_f16_ts(tb, tb + 256, bd, idesc, s > 0);
        else fc::mma_f16_ss(tb, ad, bd, idesc, s > 0);
      }
      long long ci = clock64();
      fc::mma_commit(&bar);
      fc::mbar_wait(&bar, r);
      long long c1 = clock64();
      out[2 * r] = ci - c0;
      out[2 * r + 1] = c1 - c0;
    }
  }
  fc::tc_fence_before();
  __syncthreads();
  if (tid < 32) fc::tmem_dealloc<512>(tb);
}
// Cost-model constants (P:786-791 protocol, re-measured on B200).
// tau_G: "continuously applying Twiddle factors" -- every thread keeps 16
// complex values (8 f32x2 pairs) and multiplies them by a twiddle pair per
// iteration (2 FMUL2 + 2 FFMA2 = 6 real flops per complex value), the
// twiddle itself advancing by a fixed step (another 6 flops per pair).
__global__ void __launch_bounds__(256) twiddle_rate_kernel(int iters, float* sink) {
  float2 xr[8], xi[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    xr[j] = make_float2(1.0f + j, 0.5f);
    xi[j] = make_float2(0.25f, -1.0f + j);
  }
  float2 wr = make_float2(0.9999f, 0.9998f), wi = make_float2(0.0141f, 0.0200f);
  const float2 sr = make_float2(0.99999f, 0.99999f), si = make_float2(0.0045f, 0.0045f);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float2 nr = fc::fma2(xr[j], wr, fc::mul2(xi[j], make_float2(-wi.x, -wi.y)));
      const float2 ni = fc::fma2(xr[j], wi, fc::mul2(xi[j], wr));
      xr[j] = nr;
      xi[j] = ni;
    }
    const float2 nwr = fc::fma2(wr, sr, fc::mul2(wi, make_float2(-si.x, -si.y)));
    wi = fc::fma2(wr, si, fc::mul2(wi, sr));
    wr = nwr;
  }
  float acc = 0.f;
#pragma unroll
  for (int j = 0; j < 8; ++j) acc += xr[j].x + xr[j].y + xi[j].x + xi[j].y;
  if (acc == 123.456f) sink[threadIdx.x] = acc;  // keep the work
}

// sigma_S: shared-memory bandwidth of intermediate writes and reads -- each
// thread stores and reloads 16 B per step at conflict-free addresses.
__global__ void __launch_bounds__(256) smem_bw_kernel(int iters, float* sink) {
  __shared__ uint4 buf[2][256];
  uint4 v = make_uint4(threadIdx.x, 1, 2, 3);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      fc::st_shared_v4(fc::smem_u32(&buf[j & 1][threadIdx.x]), v.x, v.y, v.z, v.w);
      const uint4 r = fc::ld_shared_u4(fc::smem_u32(&buf[(j + 1) & 1][threadIdx.x ^ 1]));
      v.x += r.y;
      v.y ^= r.z;
    }
  }
  if (v.x == 0xdeadbeefu) sink[threadIdx.x] = float(v.y);
}
}  // namespace

// Chip-wide launches for the cost-model script (tools/cost_model.py); the
// caller times them with CUDA events on the current stream.
extern "C" int fcst_twiddle_rate(int blocks, int iters, void* sink, void* stream) {
  twiddle_rate_kernel<<<blocks, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(iters, static_cast<float*>(sink));
  return int(cudaGetLastError());
}
extern "C" int fcst_smem_bw(int blocks, int iters, void* sink, void* stream) {
  smem_bw_kernel<<<blocks, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(iters, static_cast<float*>(sink));
  return int(cudaGetLastError());
}

extern "C" int fcst_tmem_ld_bench(int iters, int nwarps, long long* host_out) {
  long long* d;
  cudaMalloc(&d, 16);
  tmem_ld_bench_kernel<<<1, 512>>>(iters, nwarps, d);
  cudaError_t e = cudaMemcpy(host_out, d, 8, cudaMemcpyDeviceToHost);
  cudaFree(d);
  return e == cudaSuccess ? 0 : 100 + (int)e;
}

extern "C" int fcst_mma_rate(int nmma, int N, int ts, long long* host_out) {
  long long* d;
  cudaMalloc(&d, 32);
  cudaFuncSetAttribute(mma_rate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  mma_rate_kernel<<<1, 128, 65536>>>(nmma, N, ts, d);
  cudaError_t e = cudaMemcpy(host_out, d, 32, cudaMemcpyDeviceToHost);
  cudaFree(d);
  return e == cudaSuccess ? 0 : 100 + (int)e;
}

// tcgen05.mma issue/completion cost for an M x N x 16 fp16 MMA chain
// (M = 64 or 128; ts: A from TMEM, M = 128 only)
extern "C" int fcst_mma_rate_m(int nmma, int M, int N, int ts, long long* host_out) {
  long long* d;
  cudaMalloc(&d, 32);
  cudaFuncSetAttribute(mma_rate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  mma_rate_kernel<<<1, 128, 65536>>>(nmma, N, ts, d, M);
  cudaError_t e = cudaMemcpy(host_out, d, 32, cudaMemcpyDeviceToHost);
  cudaFree(d);
  return int(e);
}

