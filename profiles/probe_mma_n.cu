// probe_mma_n.cu -- cost of one tcgen05.mma.cta_group::2 (M = 256) as a function of N, BF16
// (kind::f16, K = 16) and FP8 (kind::f8f6f4, K = 32), operands resident in shared memory (no loads):
// the question behind the swap-AB tail tiles (weights as M = 256, r tokens as N).  Every CTA pair
// of a full grid (74 pairs) issues R MMAs back to back into one TMEM accumulator and times them
// with clock64 from the first issue to the commit's completion.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -I paper_2605_02960_b200/csrc \
//        -o probe_mma_n profiles/probe_mma_n.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#include "common.cuh"

using namespace aep;

constexpr int R = 2048;

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128) probe(int n, int fp8, long long* cyc) {
  extern __shared__ uint8_t dyn[];  // 4 stages each of A and B: 128-row x 128-B k-blocks
  uint8_t* sa = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(dyn) + 1023) & ~uintptr_t(1023));
  uint8_t* sb = sa + 4 * 128 * 128;
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x;
  const uint32_t rank = cluster_ctarank();
  for (int i = tid; i < 4 * 128 * 128 / 4; i += blockDim.x) {
    reinterpret_cast<uint32_t*>(sa)[i] = 0x38383838u;  // e4m3 1.0 / bf16 ~0.69: finite either way
    reinterpret_cast<uint32_t*>(sb)[i] = 0x38383838u;
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
  const uint32_t d = tslot;
  if (rank == 0 && tid == 0) {
    const uint32_t idesc = make_idesc(256, n, !fp8);
    const uint64_t a0 = make_smem_desc_sw128(smem_u32(sa)), b0 = make_smem_desc_sw128(smem_u32(sb));
    const long long t0 = clock64();
    for (int i = 0; i < R; ++i) {
      const int st = i & 3;
      const uint64_t ad = a0 + (uint64_t)((st * 16384) >> 4), bd = b0 + (uint64_t)((st * 16384) >> 4);
      if (fp8) mma_f8_2(d, ad + 2 * (i & 3), bd + 2 * (i & 3), idesc, i > 0);
      else mma_bf16_2(d, ad + 2 * (i & 3), bd + 2 * (i & 3), idesc, i > 0);
    }
    tc_commit2_mc(&bar, 0x3);
    mbar_wait(&bar, 0);
    cyc[blockIdx.x / 2] = clock64() - t0;
  } else if (tid == 0) {
    mbar_wait(&bar, 0);
  }
  tc_fence_before();
  cluster_sync_all();
  if (tid < 32) {
    tc_fence_after();
    tmem_dealloc2(d, 512);
  }
}

int main() {
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int pairs = sms / 2;
  long long* dc;
  cudaMalloc(&dc, pairs * sizeof(long long));
  long long* h = new long long[pairs];
  const int smem = 8 * 128 * 128 + 1024;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int fp8 = 0; fp8 < 2; ++fp8) {
    for (int n = 16; n <= 256; n += (n < 64 ? 16 : 32)) {
      probe<<<2 * pairs, 128, smem>>>(n, fp8, dc);  // warm-up
      probe<<<2 * pairs, 128, smem>>>(n, fp8, dc);
      if (cudaDeviceSynchronize() != cudaSuccess) {
        printf("CUDA error\n");
        return 1;
      }
      cudaMemcpy(h, dc, pairs * sizeof(long long), cudaMemcpyDeviceToHost);
      double avg = 0;
      for (int p = 0; p < pairs; ++p) avg += (double)h[p] / pairs;
      const double per = avg / R;
      printf("{\"dtype\": \"%s\", \"M\": 256, \"N\": %d, \"cycles_per_mma\": %.2f, \"flop_per_cycle_per_sm\": %.1f}\n",
             fp8 ? "e4m3" : "bf16", n, per, 2.0 * 256 * n * (fp8 ? 32 : 16) / per / 2);
    }
  }
  return 0;
}
