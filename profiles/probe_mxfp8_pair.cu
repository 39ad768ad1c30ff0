// probe_mxfp8_pair.cu -- the CTA-pair (cta_group::2) version of probe_mxfp8.cu: M = 256 (128 rows
// per CTA), N = 256 (B rows 0-127 in CTA 0, 128-255 in CTA 1), K = 128 as 4 block-scaled MMAs.
// Measured: each CTA's TMEM holds the scale factors of ITS 128 A rows (4 columns) but of ALL 256
// B rows (8 columns: B rows 0-127 then 128-255, the 512-B chunk layout of the 1-CTA probe each),
// loaded by tcgen05.cp.cta_group::2 issued by the leader (each CTA copies from its own smem).
// (A first version with only the CTA's own B half read scale 0 = 2^-127 for the other half.)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -I paper_2605_02960_b200/csrc \
//        -o probe2 profiles/probe_mxfp8_pair.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#include "common.cuh"

using namespace aep;

__device__ __forceinline__ uint64_t desc(uint32_t addr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46) | ((uint64_t)layout << 61);
}

// exponent of the A scale of (global row r, k) and of the B scale of (global col n, k)
__host__ __device__ int ea_of(int mode, int r, int k) {
  if (mode == 0) return k == 0 ? (r % 8) : 0;
  if (mode == 1) return k == 2 ? (r / 32) % 8 : 0;
  return 0;
}
__host__ __device__ int eb_of(int mode, int n, int k) {
  if (mode == 2) return k == 1 ? (n % 8) : 0;
  if (mode == 3) return k == 3 ? (n / 32) : 0;  // distinguishes B halves (n / 32 in 0..7)
  return 0;
}

__global__ void __cluster_dims__(2, 1, 1) probe2(int mode, float* out) {
  __shared__ __align__(1024) uint8_t sa[128 * 128];
  __shared__ __align__(1024) uint8_t sb[128 * 128];
  __shared__ __align__(128) uint8_t sfa[512];
  __shared__ __align__(128) uint8_t sfb[1024];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x;
  const uint32_t rank = cluster_ctarank();
  for (int i = tid; i < 128 * 128; i += blockDim.x) sa[i] = sb[i] = 0x38;  // e4m3 1.0
  for (int i = tid; i < 512; i += blockDim.x) {
    const int m0 = i / 16, m1 = (i % 16) / 4, k = i % 4, m = m0 + 32 * m1;
    sfa[i] = (uint8_t)(127 + ea_of(mode, 128 * rank + m, k));
    sfb[i] = (uint8_t)(127 + eb_of(mode, m, k));              // B rows 0-127
    sfb[512 + i] = (uint8_t)(127 + eb_of(mode, 128 + m, k));   // B rows 128-255
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
  const uint32_t d_t = tm, sfa_t = tm + 256, sfb_t = tm + 264;
  if (rank == 0 && tid == 0) {
    const uint64_t da = desc(smem_u32(sfa), 0, 128, 0), db = desc(smem_u32(sfb), 0, 128, 0),
                   db2 = desc(smem_u32(sfb + 512), 0, 128, 0);
    asm volatile("tcgen05.cp.cta_group::2.32x128b.warpx4 [%0], %1;" ::"r"(sfa_t), "l"(da));
    asm volatile("tcgen05.cp.cta_group::2.32x128b.warpx4 [%0], %1;" ::"r"(sfb_t), "l"(db));
    asm volatile("tcgen05.cp.cta_group::2.32x128b.warpx4 [%0], %1;" ::"r"(sfb_t + 4), "l"(db2));
    const uint64_t a0 = desc(smem_u32(sa), 16, 1024, 2), b0 = desc(smem_u32(sb), 16, 1024, 2);
    for (int k = 0; k < 4; ++k) {
      const uint32_t idesc = ((uint32_t)k << 4) | ((256u >> 3) << 17) | (1u << 23) | ((256u >> 4) << 24) |
                             ((uint32_t)k << 29);
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %6, 0;\n\t"
          "tcgen05.mma.cta_group::2.kind::mxf8f6f4.block_scale [%0], %1, %2, %3, [%4], [%5], p;\n\t}" ::"r"(d_t),
          "l"(a0 + 2 * k), "l"(b0 + 2 * k), "r"(idesc), "r"(sfa_t), "r"(sfb_t), "r"((uint32_t)(k > 0))
          : "memory");
    }
    tc_commit2_mc(&bar, 0x3);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  if (tid < 128) {
    const int w = tid / 32;
    for (int c = 0; c < 256; c += 32) {
      uint32_t v[32];
      tmem_ld32(d_t + ((uint32_t)(w * 32) << 16) + c, v);
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
  int bad_total = 0;
  for (int mode = 0; mode < 4; ++mode) {
    cudaMemset(d, 0xff, 256 * 256 * sizeof(float));
    probe2<<<2, 128>>>(mode, d);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("mode %d: CUDA error %s\n", mode, cudaGetErrorString(e));
      return 1;
    }
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int r = 0; r < 256; ++r)
      for (int n = 0; n < 256; ++n) {
        double ref = 0;
        for (int k = 0; k < 4; ++k) ref += 32.0 * (double)(1 << (ea_of(mode, r, k) + eb_of(mode, n, k)));
        if (h[r * 256 + n] != (float)ref) {
          if (bad < 6) printf("mode %d r %d n %d: got %g want %g\n", mode, r, n, h[r * 256 + n], ref);
          ++bad;
        }
      }
    printf("mode %d: %d mismatches of %d\n", mode, bad, 256 * 256);
    bad_total += bad;
  }
  return bad_total ? 2 : 0;
}
