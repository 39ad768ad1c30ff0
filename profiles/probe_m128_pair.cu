// probe_m128_pair.cu -- where does a CTA-pair (cta_group::2) BF16 MMA with M = 128 put its
// accumulator rows in TMEM, and which A rows of each CTA's shared memory does it read?
// (Needed for half-height tail tiles of the grouped GEMM: an expert's last 256-row tile with
// <= 128 valid rows.)  A[r][0] = 1 + (global row id), A[r][1] = 1; B[n][0] = 256, B[n][1] = 1 + n;
// so D = 256 * (1 + row) + (1 + n) identifies both the row and the column of every value.
// CTA c writes A rows 0..127 of its smem with ids 128 * c + r (rows >= 64 act as a probe of
// whether M = 128 reads them).  TMEM is pre-filled with a sentinel; every lane / column is dumped.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -I paper_2605_02960_b200/csrc \
//        -o probe_m128 profiles/probe_m128_pair.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#include "common.cuh"

using namespace aep;

__device__ __forceinline__ uint64_t desc(uint32_t addr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46) | ((uint64_t)layout << 61);
}

// SW128 K-major: element (r, k) of a 64-wide bf16 tile
__device__ __forceinline__ int sw128(int r, int k) {
  return (r / 8) * 1024 + (r % 8) * 128 + ((((k * 2) / 16) ^ (r % 8)) * 16) + (k * 2) % 16;
}

// back-to-back issue rate: n MMAs (K = 16 each) into one accumulator, clock64 around issue + commit wait
__global__ void __cluster_dims__(2, 1, 1) rate(int M, int n, long long* cycles) {
  __shared__ __align__(1024) uint8_t sa[128 * 128];
  __shared__ __align__(1024) uint8_t sb[128 * 128];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x;
  const uint32_t rank = cluster_ctarank();
  for (int i = tid; i < 128 * 128; i += blockDim.x) sa[i] = sb[i] = 0;
  fence_proxy_async_smem();
  if (tid < 32) tmem_alloc2(&tslot, 512);
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  if (rank == 0 && tid == 0) {
    const uint64_t a0 = desc(smem_u32(sa), 16, 1024, 2), b0 = desc(smem_u32(sb), 16, 1024, 2);
    const uint32_t id = make_idesc(M, 256, true);
    const long long c0 = clock64();
    for (int i = 0; i < n; ++i) mma_bf16_2(tslot, a0 + 2 * (i & 3), b0 + 2 * (i & 3), id, 1u);
    tc_commit2_mc(&bar, 0x3);
    mbar_wait(&bar, 0);
    cycles[blockIdx.x / 2] = clock64() - c0;
  } else {
    mbar_wait(&bar, 0);
  }
  tc_fence_before();
  cluster_sync_all();
  if (tid < 32) {
    tc_fence_after();
    tmem_dealloc2(tslot, 512);
  }
}

__global__ void __cluster_dims__(2, 1, 1) probe(int M, float* out) {
  __shared__ __align__(1024) uint8_t sa[128 * 128];
  __shared__ __align__(1024) uint8_t sb[128 * 128];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x;
  const uint32_t rank = cluster_ctarank();
  for (int i = tid; i < 128 * 128; i += blockDim.x) sa[i] = sb[i] = 0;
  __syncthreads();
  if (tid < 128) {
    const int r = tid;
    *reinterpret_cast<__nv_bfloat16*>(sa + sw128(r, 0)) = __float2bfloat16((float)(1 + 128 * rank + r));
    *reinterpret_cast<__nv_bfloat16*>(sa + sw128(r, 1)) = __float2bfloat16(1.f);
    *reinterpret_cast<__nv_bfloat16*>(sb + sw128(r, 0)) = __float2bfloat16(256.f);
    *reinterpret_cast<__nv_bfloat16*>(sb + sw128(r, 1)) = __float2bfloat16((float)(1 + 128 * rank + r));
  }
  fence_proxy_async_smem();
  if (tid < 32) tmem_alloc2(&tslot, 512);
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tm = tslot;
  if (tid < 128) {  // sentinel fill
    uint32_t s[32];
    for (int i = 0; i < 32; ++i) s[i] = 0xFFFFFFFFu;  // NaN
    for (int c = 0; c < 256; c += 32) tmem_st32(tm + ((uint32_t)((tid / 32) * 32) << 16) + c, s);
    tmem_st_wait();
  }
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  if (rank == 0 && tid == 0) {
    const uint64_t a0 = desc(smem_u32(sa), 16, 1024, 2), b0 = desc(smem_u32(sb), 16, 1024, 2);
    mma_bf16_2(tm, a0, b0, make_idesc(M, 256, true), 0u);
    tc_commit2_mc(&bar, 0x3);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  if (tid < 128) {
    const int w = tid / 32;
    for (int c = 0; c < 256; c += 32) {
      uint32_t v[32];
      tmem_ld32(tm + ((uint32_t)(w * 32) << 16) + c, v);
      tmem_ld_wait();
      for (int i = 0; i < 32; ++i) out[((128 * rank + tid) * 256) + c + i] = __uint_as_float(v[i]);
    }
  }
  tc_fence_before();
  cluster_sync_all();
  if (tid < 32) {
    tc_fence_after();
    tmem_dealloc2(tm, 512);
  }
}

int main() {
  float* d;
  cudaMalloc(&d, 256 * 256 * sizeof(float));
  static float h[256 * 256];
  for (int M : {256, 128}) {
    cudaMemset(d, 0, 256 * 256 * sizeof(float));
    probe<<<2, 128>>>(M, d);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("M %d: CUDA error %s\n", M, cudaGetErrorString(e));
      return 1;
    }
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("== M = %d: per (cta, lane): decoded A row id of column 0 / decoded n at columns 0,1,127,128,255\n", M);
    for (int cta = 0; cta < 2; ++cta)
      for (int lane = 0; lane < 128; ++lane) {
        const float* row = h + (128 * cta + lane) * 256;
        printf("cta %d lane %3d:", cta, lane);
        for (int c : {0, 1, 127, 128, 255}) {
          const float v = row[c];
          if (v != v) { printf("  [%3d] --", c); continue; }
          const long iv = (long)v;
          const long n1 = ((iv - 1) % 256) + 1, r1 = (iv - n1) / 256;
          printf("  [%3d] r%ld n%ld", c, r1 - 1, n1 - 1);
        }
        printf("\n");
      }
  }
  long long* cyc;
  cudaMalloc(&cyc, 74 * sizeof(long long));
  static long long hc[74];
  for (int M : {256, 128, 256, 128}) {
    rate<<<148, 128>>>(M, 4096, cyc);
    cudaDeviceSynchronize();
    cudaMemcpy(hc, cyc, sizeof(hc), cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < 74; ++i) avg += hc[i] / 74.0;
    printf("rate M=%d N=256 K=16 cta_group::2, 4096 MMAs on 74 pairs: %.1f cycles per MMA\n", M, avg / 4096);
  }
  return 0;
}
