// combine.cu -- step (4): weighted combine / unpermute ("... and sums their
// outputs"; reading R9 for the residual):
//     y_t = r_t + sum_{j=0..k-1} w_tj * Y_perm[dest(t, j)]     (fp32 accumulate, j order)
// One warp per token, 16-B vectors (8 bf16 per lane per step); HBM-bound.
#include "common.cuh"
#include "kernels.cuh"

namespace aep {

namespace {
template <int KMAX>
__global__ void __launch_bounds__(256) combine_kernel(const bf16* __restrict__ yperm,
                                                      const int32_t* __restrict__ dest,
                                                      const float* __restrict__ w, const bf16* residual,
                                                      bf16* y, int64_t T, int H, int k) {
  const int lane = threadIdx.x & 31;
  const int64_t t = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (t >= T) return;
  int32_t d[KMAX];
  float wj[KMAX];
#pragma unroll
  for (int j = 0; j < KMAX; ++j) {
    d[j] = (j < k) ? dest[t * k + j] : 0;
    wj[j] = (j < k) ? w[t * k + j] : 0.f;
  }
  const int nv = H / 8;
  for (int v = lane; v < nv; v += 32) {
    float acc[8];
    if (residual) {
      const uint4 r = reinterpret_cast<const uint4*>(residual + t * H)[v];
      const uint32_t u[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
      for (int q = 0; q < 4; ++q) { acc[2 * q] = bf16_lo(u[q]); acc[2 * q + 1] = bf16_hi(u[q]); }
    } else {
#pragma unroll
      for (int q = 0; q < 8; ++q) acc[q] = 0.f;
    }
    uint4 vals[KMAX];
#pragma unroll
    for (int j = 0; j < KMAX; ++j)
      if (j < k)
        asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(vals[j].x), "=r"(vals[j].y), "=r"(vals[j].z), "=r"(vals[j].w)
                     : "l"(reinterpret_cast<const uint4*>(yperm + (int64_t)d[j] * H) + v));
#pragma unroll
    for (int j = 0; j < KMAX; ++j) {
      if (j < k) {
        const uint32_t u[4] = {vals[j].x, vals[j].y, vals[j].z, vals[j].w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          acc[2 * q] = fmaf(wj[j], bf16_lo(u[q]), acc[2 * q]);
          acc[2 * q + 1] = fmaf(wj[j], bf16_hi(u[q]), acc[2 * q + 1]);
        }
      }
    }
    uint4 o;
    o.x = pack_bf16x2(acc[0], acc[1]);
    o.y = pack_bf16x2(acc[2], acc[3]);
    o.z = pack_bf16x2(acc[4], acc[5]);
    o.w = pack_bf16x2(acc[6], acc[7]);
    reinterpret_cast<uint4*>(y + t * H)[v] = o;
  }
}
__global__ void spin_ns_kernel(uint64_t ns) {
  uint64_t t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (;;) {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 >= ns) break;
    __nanosleep(1000);
  }
}

// The gather transport on SMs that the persistent GEMMs leave room on: small CTAs (128 threads,
// no shared memory, few registers) that co-reside with a GEMM CTA on every SM, so the copy
// progresses DURING the GEMMs instead of waiting for SMs to drain (the driver's D2D memcpy and
// NCCL's kernels do not fit beside a ~220 KB-smem GEMM CTA).  Streaming 16-B loads / stores
// (evict-first: the slot is read once, by the next layer); works on NVLink peer pointers too.
// Each thread keeps 8 x 16 B in flight per round (the NVLink read latency needs ~1 MB in flight
// per GPU for the link rate, so few CTAs suffice).
// min_ns > 0 (1-GPU link emulation): block 0 holds the kernel open until min_ns after it started,
// so a chunk takes max(copy, link) time, and ns_per_round > 0: every CTA paces itself -- round r of its strided share
// may start only ns_per_round * r after the kernel started -- so the copy streams smoothly at the
// emulated link rate over the whole chunk, like a remote read, instead of bursting at HBM speed.
constexpr int kCopyUnroll = 8;
__global__ void __launch_bounds__(128) gather_copy_kernel(uint4* __restrict__ dst, const uint4* __restrict__ src,
                                                          size_t n16, uint64_t ns_per_round, uint64_t min_ns) {
  uint64_t t0 = 0;
  if (ns_per_round || min_ns) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  const size_t stride = (size_t)gridDim.x * 128;
  size_t i = (size_t)blockIdx.x * 128 + threadIdx.x;
  uint64_t round = 0;
  for (; i + (kCopyUnroll - 1) * stride < n16; i += kCopyUnroll * stride) {
    if (ns_per_round) {
      for (;;) {
        uint64_t t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (t - t0 >= ns_per_round * round) break;
        __nanosleep(256);
      }
      ++round;
    }
    uint4 v[kCopyUnroll];
#pragma unroll
    for (int u = 0; u < kCopyUnroll; ++u) v[u] = __ldcs(src + i + u * stride);
#pragma unroll
    for (int u = 0; u < kCopyUnroll; ++u) __stcs(dst + i + u * stride, v[u]);
  }
  for (; i < n16; i += stride) __stcs(dst + i, __ldcs(src + i));
  if (min_ns && blockIdx.x == 0 && threadIdx.x == 0)  // the chunk takes max(copy, link) time
    for (;;) {
      uint64_t t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t - t0 >= min_ns) break;
      __nanosleep(500);
    }
}
}  // namespace

void launch_spin_ns(uint64_t ns, cudaStream_t s) { spin_ns_kernel<<<1, 1, 0, s>>>(ns); }

void launch_gather_copy(void* dst, const void* src, size_t bytes, int ctas, cudaStream_t s, uint64_t min_ns) {
  if (!bytes) return;
  const size_t n16 = bytes / 16;
  // pacing: the chunk must take min_ns; a CTA's share is split into rounds of 128 x kCopyUnroll x 16 B
  const size_t per_round = (size_t)ctas * 128 * kCopyUnroll;
  const uint64_t rounds = (n16 + per_round - 1) / per_round;
  const uint64_t ns_per_round = (min_ns && rounds) ? min_ns / rounds : 0;
  gather_copy_kernel<<<ctas, 128, 0, s>>>(static_cast<uint4*>(dst), static_cast<const uint4*>(src), n16,
                                         ns_per_round, min_ns);
}

void launch_combine(const bf16* yperm, const int32_t* dest, const float* w, const bf16* residual, bf16* y,
                    int64_t T, int H, int k, cudaStream_t s) {
  if (T <= 0) return;
  const unsigned grid = (unsigned)((T + 7) / 8);
  if (k <= 2) combine_kernel<2><<<grid, 256, 0, s>>>(yperm, dest, w, residual, y, T, H, k);
  else if (k <= 4) combine_kernel<4><<<grid, 256, 0, s>>>(yperm, dest, w, residual, y, T, H, k);
  else if (k <= 8) combine_kernel<8><<<grid, 256, 0, s>>>(yperm, dest, w, residual, y, T, H, k);
  else combine_kernel<16><<<grid, 256, 0, s>>>(yperm, dest, w, residual, y, T, H, k);
}

}  // namespace aep
