// probe_mxfp8.cu -- layout probe for MX block-scaled FP8 on sm_100a (design study for the MX
// expert path, S9): one CTA copies a 512-B scale-factor chunk smem -> TMEM with
// tcgen05.cp.32x128b.warpx4 and runs tcgen05.mma.kind::mxf8f6f4.block_scale (M=128, N=128,
// K=128 as 4 MMAs of 32, A = B = 1.0 in e4m3) with per-(row, k-step) exponents e(m, k).
// Expected D[m][n] = 32 * sum_k 2^(e_a(m,k) + e_b(n,k)).  Prints mismatches.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -o probe profiles/probe_mxfp8.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// matrix descriptor: start >> 4, LBO >> 4 at [16,30), SBO >> 4 at [32,46), version 1 at 46,
// layout (61-63): 0 = no swizzle, 2 = 128-B swizzle
__device__ __forceinline__ uint64_t desc(uint32_t addr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46) | ((uint64_t)layout << 61);
}

__global__ void probe(int mode, float* out) {
  // A, B: 128 rows x 128 e4m3 (128 B per row), 128-B swizzled K-major tiles (all bytes 0x38 = 1.0,
  // so the swizzle is irrelevant); SFA / SFB: one 512-B chunk each
  __shared__ __align__(1024) uint8_t sa[128 * 128];
  __shared__ __align__(1024) uint8_t sb[128 * 128];
  __shared__ __align__(128) uint8_t sfa[512];
  __shared__ __align__(128) uint8_t sfb[512];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x;
  for (int i = tid; i < 128 * 128; i += blockDim.x) sa[i] = sb[i] = 0x38;
  // chunk byte (m % 32) * 16 + (m / 32) * 4 + k  <->  (row m, k-step k)
  for (int i = tid; i < 512; i += blockDim.x) {
    const int m0 = i / 16, m1 = (i % 16) / 4, k = i % 4, m = m0 + 32 * m1;
    int ea = 0, eb = 0;
    if (mode == 0) ea = (k == 0) ? (m % 8) : 0;
    if (mode == 1) ea = (k == 3) ? (m % 8) : 0;
    if (mode == 2) eb = (k == 1) ? (m % 8) : 0;
    if (mode == 3) { ea = (k == 2) ? (m / 32) : 0; eb = (k == 2) ? (m % 4) : 0; }
    sfa[i] = (uint8_t)(127 + ea);
    sfb[i] = (uint8_t)(127 + eb);
  }
  __syncthreads();
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)),
                 "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = tslot;
  const uint32_t d_t = tm, sfa_t = tm + 128, sfb_t = tm + 136;
  if (tid == 0) {
    // 32 rows x 16 B, rows contiguous: 4 core matrices (8 x 16 B) along M, SBO = 128 B
    const uint64_t da = desc(smem_u32(sfa), 0, 128, 0), db = desc(smem_u32(sfb), 0, 128, 0);
    asm volatile("tcgen05.cp.cta_group::1.32x128b.warpx4 [%0], %1;" ::"r"(sfa_t), "l"(da));
    asm volatile("tcgen05.cp.cta_group::1.32x128b.warpx4 [%0], %1;" ::"r"(sfb_t), "l"(db));
    const uint64_t a0 = desc(smem_u32(sa), 16, 1024, 2), b0 = desc(smem_u32(sb), 16, 1024, 2);
    for (int k = 0; k < 4; ++k) {
      // block-scaled idesc: sf ids at [4,6) (B) and [29,31) (A), E4M3 (0) operands, K-major,
      // N >> 3 at [17,23), scale format E8M0 at bit 23, M >> 4 at [24,29)
      const uint32_t idesc = ((uint32_t)k << 4) | ((128u >> 3) << 17) | (1u << 23) | ((128u >> 4) << 24) |
                             ((uint32_t)k << 29);
      const uint32_t acc = k > 0;
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %6, 0;\n\t"
          "tcgen05.mma.cta_group::1.kind::mxf8f6f4.block_scale [%0], %1, %2, %3, [%4], [%5], p;\n\t}" ::"r"(d_t),
          "l"(a0 + 2 * k), "l"(b0 + 2 * k), "r"(idesc), "r"(sfa_t), "r"(sfb_t), "r"(acc)
          : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
        smem_u32(&bar)));
  }
  __syncwarp();
  {
    uint32_t ph = 0, done = 0;
    while (!done)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0,1,0,p;\n\t}"
                   : "=r"(done) : "r"(smem_u32(&bar)), "r"(ph));
  }
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (tid < 128) {
    const int w = tid / 32;
    uint32_t v[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(d_t + ((uint32_t)(w * 32) << 16)));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int n = 0; n < 8; ++n) out[tid * 8 + n] = __uint_as_float(v[n]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(256));
}

int main() {
  float* d;
  cudaMalloc(&d, 128 * 8 * sizeof(float));
  float h[128 * 8];
  int bad_total = 0;
  for (int mode = 0; mode < 4; ++mode) {
    probe<<<1, 128>>>(mode, d);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("mode %d: CUDA error %s\n", mode, cudaGetErrorString(e));
      return 1;
    }
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int m = 0; m < 128; ++m)
      for (int n = 0; n < 8; ++n) {
        double ref = 0;
        for (int k = 0; k < 4; ++k) {
          int ea = 0, eb = 0;
          if (mode == 0) ea = (k == 0) ? (m % 8) : 0;
          if (mode == 1) ea = (k == 3) ? (m % 8) : 0;
          if (mode == 2) eb = (k == 1) ? (n % 8) : 0;
          if (mode == 3) { ea = (k == 2) ? (m / 32) : 0; eb = (k == 2) ? (n % 4) : 0; }
          ref += 32.0 * (double)(1 << (ea + eb));
        }
        if (h[m * 8 + n] != (float)ref) {
          if (bad < 6) printf("mode %d m %d n %d: got %g want %g\n", mode, m, n, h[m * 8 + n], ref);
          ++bad;
        }
      }
    printf("mode %d: %d mismatches of %d\n", mode, bad, 128 * 8);
    bad_total += bad;
  }
  return bad_total ? 2 : 0;
}
