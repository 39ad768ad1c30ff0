// probe_mx_rate.cu -- issue-to-completion cost of tcgen05.mma.cta_group::2 (M = 256, K = 32 e4m3),
// kind::f8f6f4 vs kind::mxf8f6f4.block_scale (E8M0 scales in TMEM), N = 256 and 224, operands
// resident in shared memory: the MMA-rate question behind the MX down GEMM (S6).  Every CTA
// pair of a full grid issues R MMAs; tiles of 48 MMAs (12 k-blocks) alternate between two
// accumulators ([0, N) and [256, 256 + N) for N <= 224, one accumulator for N = 256); mode cp adds
// one tcgen05.cp of a 512-B scale chunk per 4 MMAs (one per k-block, as the GEMM does); mode
// 3 / 4 (f8 / mx) interleave two independent accumulators MMA by MMA ([0, N) and [256, 256 + N)).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -I paper_2605_02960_b200/csrc \
//        -o probe_mx_rate profiles/probe_mx_rate.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#include "common.cuh"

using namespace aep;

constexpr int R = 4800;

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128) probe(int n, int mode, long long* cyc) {
  extern __shared__ uint8_t dyn[];
  uint8_t* sa = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(dyn) + 1023) & ~uintptr_t(1023));
  uint8_t* sb = sa + 4 * 128 * 128;
  uint8_t* sf = sb + 4 * 128 * 128;  // 4 scale chunks of 512 B + the B chunk
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x;
  const uint32_t rank = cluster_ctarank();
  for (int i = tid; i < 4 * 128 * 128 / 4; i += blockDim.x) {
    reinterpret_cast<uint32_t*>(sa)[i] = 0x38383838u;
    reinterpret_cast<uint32_t*>(sb)[i] = 0x38383838u;
  }
  for (int i = tid; i < 5 * 128; i += blockDim.x) reinterpret_cast<uint32_t*>(sf)[i] = 0x7F7F7F7Fu;
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
  const bool mx = mode == 1 || mode == 2 || mode == 4, cp = mode == 2;
  if (rank == 0 && tid == 0) {
    const uint32_t sfb = tm + 480, sfa0 = tm + 488;
    if (mx) {
      tc_cp_sf_2(sfb, smem_u32(sf + 4 * 512));
      tc_cp_sf_2(sfb + 4, smem_u32(sf + 4 * 512));
      for (int s = 0; s < 4; ++s) tc_cp_sf_2(sfa0 + 4 * s, smem_u32(sf + s * 512));
    }
    const uint64_t a0 = make_smem_desc_sw128(smem_u32(sa)), b0 = make_smem_desc_sw128(smem_u32(sb));
    const long long t0 = clock64();
    for (int i = 0; i < R; ++i) {
      const int st = (i >> 2) & 3, k = i & 3;
      const int tile = i / 48;
      uint32_t d = tm + ((n <= 224 && (tile & 1)) ? 256u : 0u);
      uint32_t acc = (i % 48) != 0;
      if (mode >= 3) {  // two chains, alternating per MMA
        d = tm + ((i & 1) ? 256u : 0u);
        acc = (i % 96) >= 2;
      }
      const uint64_t ad = a0 + (uint64_t)((st * 16384) >> 4) + 2 * k, bd = b0 + (uint64_t)((st * 16384) >> 4) + 2 * k;
      if (mx) {
        const uint32_t sfa = sfa0 + 4 * st;
        if (cp && k == 0) tc_cp_sf_2(sfa, smem_u32(sf + st * 512));
        mma_mx_2(d, ad, bd, make_idesc_mx(256, n, k), sfa, sfb, acc);
      } else {
        mma_f8_2(d, ad, bd, make_idesc(256, n, false), acc);
      }
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
    tmem_dealloc2(tm, 512);
  }
}

int main() {
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int pairs = sms / 2;
  long long* dc;
  cudaMalloc(&dc, pairs * sizeof(long long));
  long long* h = new long long[pairs];
  const int smem = 8 * 128 * 128 + 5 * 512 + 1024;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const char* names[5] = {"f8f6f4", "mxf8f6f4", "mxf8f6f4+cp", "f8f6f4 2 chains", "mxf8f6f4 2 chains"};
  for (int n : {256, 224, 128}) {
    for (int mode = 0; mode < 5; ++mode) {
      if (mode >= 3 && n > 224) continue;
      probe<<<2 * pairs, 128, smem>>>(n, mode, dc);  // warm-up
      probe<<<2 * pairs, 128, smem>>>(n, mode, dc);
      if (cudaDeviceSynchronize() != cudaSuccess) {
        printf("CUDA error\n");
        return 1;
      }
      cudaMemcpy(h, dc, pairs * sizeof(long long), cudaMemcpyDeviceToHost);
      double avg = 0;
      for (int p = 0; p < pairs; ++p) avg += (double)h[p] / pairs;
      const double per = avg / R;
      printf("{\"kind\": \"%s\", \"M\": 256, \"N\": %d, \"cycles_per_mma\": %.2f, \"ideal\": %.1f}\n", names[mode], n,
             per, n / 2.0);
    }
  }
  return 0;
}
