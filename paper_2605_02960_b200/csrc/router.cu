// router.cu -- step (1) of the hot path: router GEMM + softmax + top-k
// ("a lightweight router dispatches each token to its top-k experts";
//  readings R1-R3 in DESIGN.md: fp32 logits, softmax -> top-k -> renormalise,
//  descending logit with ties -> lower expert id).
//
// CUDA-core variant: a 64-token x E-expert logits tile per CTA in shared memory
// (register-blocked fp32 FMAs over H in 32-wide chunks), then one warp per token for
// the top-k (k rounds of a warp arg-max on the key (logit, -id)).
#include "common.cuh"
#include "kernels.cuh"

namespace aep {

namespace {
constexpr int RT = 64;     // tokens per CTA
constexpr int RE = 128;    // experts per inner tile
constexpr int RK = 32;     // H chunk
constexpr int RTHREADS = 256;

// Top-k of one token held in shared memory (E logits), by one warp.  Writes ids / w.
__device__ void warp_topk(const float* lg, int E, int k, int norm_topk, int32_t* ids, float* w) {
  const int lane = threadIdx.x & 31;
  constexpr int kPer = kMaxExperts / 32;
  float v[kPer];
#pragma unroll
  for (int i = 0; i < kPer; ++i) {
    const int e = lane + 32 * i;
    v[i] = (e < E) ? lg[e] : -INFINITY;
  }
  float sel_l[kMaxTopK];
  int sel_e[kMaxTopK];
  for (int j = 0; j < k; ++j) {
    float bv = -INFINITY;
    int be = 0x7fffffff;
#pragma unroll
    for (int i = 0; i < kPer; ++i) {
      const int e = lane + 32 * i;
      if (e < E && (v[i] > bv || (v[i] == bv && e < be))) { bv = v[i]; be = e; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oe = __shfl_xor_sync(0xffffffffu, be, o);
      if (ov > bv || (ov == bv && oe < be)) { bv = ov; be = oe; }
    }
    sel_l[j] = bv;
    sel_e[j] = be;
    if ((be & 31) == lane) {
#pragma unroll
      for (int i = 0; i < kPer; ++i)
        if (i == (be >> 5)) v[i] = -INFINITY;  // mark taken (stays out of later rounds)
    }
  }
  // weights: norm_topk -> softmax over the k selected logits (== softmax_E -> top-k ->
  // renormalise, R1); else the full-E softmax probability of each selected expert.
  float denom = 0.f, ref = sel_l[0];
  if (norm_topk) {
    for (int j = 0; j < k; ++j) denom += expf(sel_l[j] - ref);
  } else {
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < kPer; ++i) {
      const int e = lane + 32 * i;
      if (e < E) s += expf(lg[e] - ref);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    denom = s;
  }
  for (int j = lane; j < k; j += 32) {
    ids[j] = sel_e[j];
    w[j] = expf(sel_l[j] - ref) / denom;
  }
}

__global__ void __launch_bounds__(RTHREADS) router_simt_kernel(const bf16* __restrict__ x,
                                                               const bf16* __restrict__ wr, int64_t T, int H,
                                                               int E, int k, int norm_topk, int32_t* ids,
                                                               float* w) {
  extern __shared__ float sm[];
  float* xs = sm;                    // [RK][RT]
  float* ws = xs + RK * RT;          // [RK][RE]
  float* lg = ws + RK * RE;          // [RT][E+1]
  const int tid = threadIdx.x;
  const int64_t t0 = (int64_t)blockIdx.x * RT;
  const int tx = tid % 16, ty = tid / 16;  // 16 x 16 threads: 8 experts x 4 tokens each
  const int ldl = E + 1;

  for (int e0 = 0; e0 < E; e0 += RE) {
    float acc[4][8];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 8; ++b) acc[a][b] = 0.f;
    for (int k0 = 0; k0 < H; k0 += RK) {
      {  // x chunk: 64 tokens x 32 -> transposed fp32
        const int tok = tid / 4, kp = (tid % 4) * 8;
        const int64_t t = t0 + tok;
        uint4 v = make_uint4(0, 0, 0, 0);
        if (t < T) v = *reinterpret_cast<const uint4*>(x + t * H + k0 + kp);
        const uint32_t u[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          xs[(kp + 2 * q) * RT + tok] = bf16_lo(u[q]);
          xs[(kp + 2 * q + 1) * RT + tok] = bf16_hi(u[q]);
        }
      }
#pragma unroll
      for (int half = 0; half < 2; ++half) {  // w chunk: 128 experts x 32
        const int ex = tid / 2, kp = (tid % 2) * 16 + half * 8;
        const int e = e0 + ex;
        uint4 v = make_uint4(0, 0, 0, 0);
        if (e < E) v = *reinterpret_cast<const uint4*>(wr + (int64_t)e * H + k0 + kp);
        const uint32_t u[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          ws[(kp + 2 * q) * RE + ex] = bf16_lo(u[q]);
          ws[(kp + 2 * q + 1) * RE + ex] = bf16_hi(u[q]);
        }
      }
      __syncthreads();
#pragma unroll 8
      for (int kk = 0; kk < RK; ++kk) {
        const float4 xa = *reinterpret_cast<const float4*>(xs + kk * RT + ty * 4);
        const float4 wa = *reinterpret_cast<const float4*>(ws + kk * RE + tx * 8);
        const float4 wb = *reinterpret_cast<const float4*>(ws + kk * RE + tx * 8 + 4);
        const float xv[4] = {xa.x, xa.y, xa.z, xa.w};
        const float wv[8] = {wa.x, wa.y, wa.z, wa.w, wb.x, wb.y, wb.z, wb.w};
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 8; ++b) acc[a][b] = fmaf(xv[a], wv[b], acc[a][b]);
      }
      __syncthreads();
    }
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 8; ++b) {
        const int e = e0 + tx * 8 + b;
        if (e < E) lg[(ty * 4 + a) * ldl + e] = acc[a][b];
      }
  }
  __syncthreads();
  const int warp = tid >> 5;
  for (int tl = warp; tl < RT; tl += RTHREADS / 32) {
    const int64_t t = t0 + tl;
    if (t >= T) break;
    warp_topk(lg + tl * ldl, E, k, norm_topk, ids + t * k, w + t * k);
  }
}
}  // namespace

void launch_router_simt(const bf16* x, const bf16* wr, int64_t T, int H, int E, int k, int norm_topk,
                        int32_t* ids, float* w, cudaStream_t s) {
  if (T <= 0) return;
  const size_t smem = sizeof(float) * ((size_t)RK * RT + (size_t)RK * RE + (size_t)RT * (E + 1));
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(router_simt_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr = true;
  }
  const unsigned grid = (unsigned)((T + RT - 1) / RT);
  router_simt_kernel<<<grid, RTHREADS, smem, s>>>(x, wr, T, H, E, k, norm_topk, ids, w);
}

}  // namespace aep
