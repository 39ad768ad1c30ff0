// router.cu -- step (1) of the hot path: router GEMM + softmax + top-k
// ("a lightweight router dispatches each token to its top-k experts";
//  readings R1-R3 in DESIGN.md: fp32 logits, softmax -> top-k -> renormalise,
//  descending logit with ties -> lower expert id).
//
// CUDA-core variant: a 64-token x E-expert logits tile per CTA in shared memory
// (register-blocked fp32 FMAs over H in 32-wide chunks), then one warp per token for
// the top-k (k rounds of a warp arg-max on the key (logit, -id)).
#include <mutex>

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


// ------------------------------------------------------------------ router, experts as the MMA's M
// One 1-CTA tcgen05 tile per 256 tokens: D[128 experts x 256 tokens] = W_r[128 x H] . x[256 x H]^T
// (M = 128 lanes = experts, N = 256 columns = tokens, full MMA width; W_r rows >= E are TMA zero
// fill).  At 32K tokens that is 128 tiles, one wave over the 148 SMs, each streaming its 256 token
// rows once -- the pair-tile router needs two waves of N = 128 MMAs.  Epilogue: each of the 4
// warps moves its 32 expert lanes x 128 token columns from TMEM to a padded shared-memory
// [token][expert] block; then one thread per token runs the top-k over the E logits in increasing
// id (strict '>': ties -> lower id, R2) and the softmax over the selected (R1) or all (norm_topk
// = 0) logits -- the same arithmetic as the pair router's TMEM epilogue.
namespace {
constexpr int RS_TOK = 256;                 // tokens per tile (MMA N)
constexpr int RS_STAGES = 3;
constexpr int RS_A = 128 * 128;             // W_r k-block: 128 rows x 128 B
constexpr int RS_B = RS_TOK * 128;          // x k-block: 256 rows x 128 B
constexpr int RS_LD = 132;                  // padded logits row (floats): float4 reads conflict-free
constexpr size_t RS_SMEM = 1024 + (size_t)RS_STAGES * (RS_A + RS_B) + 128 * RS_LD * 4 + 256;

template <int KMAX>
__global__ void __launch_bounds__(256, 1)
    router_swap_kernel(const __grid_constant__ CUtensorMap map_wr, const __grid_constant__ CUtensorMap map_x,
                       int64_t T, int H, int E, int k, int norm_topk, int32_t* __restrict__ ids,
                       float* __restrict__ w) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = sA + RS_STAGES * RS_A;
  float* buf = reinterpret_cast<float*>(sB + RS_STAGES * RS_B);
  uint64_t* full = reinterpret_cast<uint64_t*>(buf + 128 * RS_LD);
  uint64_t* empty = full + RS_STAGES;
  uint64_t* tfull = empty + RS_STAGES;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(tfull + 1);
  const int warp = warp_id(), lane = lane_id();
  const int64_t tok0 = (int64_t)blockIdx.x * RS_TOK;
  const int nkb = H / 64;
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&map_wr);
    tma_prefetch_desc(&map_x);
    for (int s = 0; s < RS_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tfull, 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(tslot, 256);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int kb = 0; kb < nkb; ++kb) {
        mbar_wait(&empty[stage], phase ^ 1);
        mbar_arrive_expect_tx(&full[stage], RS_A + RS_B);
        tma_load_3d_nohint(sA + stage * RS_A, &map_wr, &full[stage], kb * 64, 0, 0);
        tma_load_2d_nohint(sB + stage * RS_B, &map_x, &full[stage], kb * 64, (int)tok0);
        if (++stage == RS_STAGES) { stage = 0; phase ^= 1; }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    const uint32_t idesc = make_idesc(128, RS_TOK, true);
    const uint64_t a0 = make_smem_desc_sw128(smem_u32(sA)), b0 = make_smem_desc_sw128(smem_u32(sB));
    int stage = 0;
    uint32_t phase = 0;
    for (int kb = 0; kb < nkb; ++kb) {
      mbar_wait(&full[stage], phase);
      tc_fence_after();
      if (elect_one()) {
#pragma unroll
        for (int q = 0; q < 4; ++q)
          mma_bf16(tmem, a0 + (uint64_t)((stage * RS_A) >> 4) + 2 * q, b0 + (uint64_t)((stage * RS_B) >> 4) + 2 * q,
                   idesc, (kb | q) != 0 ? 1u : 0u);
        tc_commit(&empty[stage]);
      }
      __syncwarp();
      if (++stage == RS_STAGES) { stage = 0; phase ^= 1; }
    }
    if (elect_one()) tc_commit(tfull);
    __syncwarp();
  } else if (warp >= 4) {
    const int quad = warp & 3;  // TMEM lanes (experts) [32 quad, 32 quad + 32)
    const int et = threadIdx.x - 128;  // 0..127: this thread's token within the half tile
    mbar_wait(tfull, 0);
    tc_fence_after();
    for (int half = 0; half < 2; ++half) {
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {  // 32 token columns per tcgen05.ld
        uint32_t r[32];
        tmem_ld32(tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(half * 128 + c * 32), r);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 32; ++i) buf[(c * 32 + i) * RS_LD + quad * 32 + lane] = __uint_as_float(r[i]);
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");
      const int64_t t = tok0 + half * 128 + et;
      if (t < T) {
        const float* lg = buf + et * RS_LD;
        float tv[KMAX];
        int ti[KMAX];
#pragma unroll
        for (int j = 0; j < KMAX; ++j) { tv[j] = -INFINITY; ti[j] = 0; }
#pragma unroll 1
        for (int e0 = 0; e0 < E; e0 += 4) {
          const float4 v4 = *reinterpret_cast<const float4*>(lg + e0);
          const float vv[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            float v = vv[i];
            if (e0 + i < E && v > tv[KMAX - 1]) {
              int e = e0 + i;
#pragma unroll
              for (int j = 0; j < KMAX; ++j) {
                if (v > tv[j]) {
                  const float sv = tv[j];
                  const int se = ti[j];
                  tv[j] = v; ti[j] = e; v = sv; e = se;
                }
              }
            }
          }
        }
        float denom = 0.f;
        const float ref = tv[0];
        if (norm_topk) {
#pragma unroll
          for (int j = 0; j < KMAX; ++j)
            if (j < k) denom += expf(tv[j] - ref);
        } else {
          for (int e = 0; e < E; ++e) denom += expf(lg[e] - ref);
        }
#pragma unroll
        for (int j = 0; j < KMAX; ++j)
          if (j < k) {
            ids[t * k + j] = ti[j];
            w[t * k + j] = expf(tv[j] - ref) / denom;
          }
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");  // the block is rewritten by the next half
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, 256);
  }
}
}  // namespace

bool router_swap_ok(int E, int H) { return E <= 128 && H % 64 == 0; }

bool launch_router_swap(const CUtensorMap& map_wr128, const bf16* x, int64_t T, int H, int E, int k, int norm_topk,
                        int32_t* ids, float* w, cudaStream_t s) {
  if (T <= 0) return true;
  CUtensorMap map_x;
  const uint64_t dims[2] = {(uint64_t)H, (uint64_t)T};
  const uint64_t strides[1] = {(uint64_t)H * 2};
  const uint32_t box[2] = {64, RS_TOK};
  if (!encode_tmap(&map_x, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, x, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B))
    return false;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaFuncSetAttribute(router_swap_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)RS_SMEM);
    cudaFuncSetAttribute(router_swap_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)RS_SMEM);
  });
  const unsigned grid = (unsigned)((T + RS_TOK - 1) / RS_TOK);
  if (k <= 8) router_swap_kernel<8><<<grid, 256, RS_SMEM, s>>>(map_wr128, map_x, T, H, E, k, norm_topk, ids, w);
  else router_swap_kernel<16><<<grid, 256, RS_SMEM, s>>>(map_wr128, map_x, T, H, E, k, norm_topk, ids, w);
  return true;
}

}  // namespace aep
