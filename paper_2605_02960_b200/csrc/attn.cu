// attn.cu -- NEXT-3: the data-parallel attention layer in front of each
// MoE layer, KV-cache-free (PAPER.md:275 "pure DP attention", :311 "after computing attention
// locally", :351-353 "disables KV storage entirely and computes attention on the fly").
// Architecture reading R19 (S3): the Qwen3-MoE block -- RMSNorm, QKV projection,
// per-head QK RMSNorm + rotate-half RoPE, causal GQA per prompt, O projection + residual,
// post-attention RMSNorm (the MoE router's input).
//
// Kernels here: rmsnorm (x -> xn), qk_rope (qkv -> q, k with norm + RoPE), v_transpose
// (qkv -> V^T per kv head, the K-major B operand of P.V), flash_attn (tcgen05), and
// residual_rmsnorm (x + attn -> x', RMSNorm(x')).  The two projections run on the tcgen05
// GEMM (gemm_tc.cu, dense mode).
//
// flash_attn: one CTA per (query head, 128-query tile of one prompt); 256 threads:
//   warp 0   TMA producer: Q tile once, then per 128-key block K_j and V^T_j into a 2-stage
//            ring (K and V released separately: K after S_j, V after PV_j)
//   warp 1   MMA issuer: S_j = Q K_j^T (M=128, N=128, K=d) into a double-buffered TMEM S,
//            one block ahead of PV_j = P_j V_j (A = P from smem, B = V^T_j) accumulated in a
//            TMEM O (accumulate flag off for j = 0)
//   warp 2   TMEM allocator (512 columns: S0, S1, O)
//   warps 4-7 softmax, thread = query row: S row from TMEM (4 x 32 columns), scale to the
//            log2 domain, causal / prompt-end mask on the diagonal block, row max, p =
//            exp2(s - m), row sum in fp32, P as bf16 into the 128-B-swizzled smem tile the
//            MMA reads.  The running max is only moved (and O rescaled in TMEM) when it grows
//            by more than 8 (log2 units): the final O / l uses the same stale max in both, so
//            the result is exact, and O is rarely touched.
// The rows of a tile past the end of its prompt are computed but never stored.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <mutex>

#include "common.cuh"
#include "kernels.cuh"

namespace aep {
namespace {

constexpr int FA_BM = 128;  // queries per tile
constexpr int FA_BN = 128;  // keys per block
constexpr int FA_D = 128;   // head dim
constexpr int FA_KB = 16 * 1024;       // one [128 rows x 128 B] swizzled k-block
constexpr int FA_TILE = 2 * FA_KB;     // a 128 x 128 bf16 operand tile (2 k-blocks of 64)
constexpr int FA_NTHREADS = 256;
constexpr float kRescaleThresh = 8.0f;  // log2 units

struct FaSmem {
  // operand tiles (each 1024-B aligned, [k-block][128 rows][128 B])
  static constexpr int Q = 0;
  static constexpr int K0 = Q + FA_TILE;
  static constexpr int V0 = K0 + 2 * FA_TILE;
  static constexpr int P = V0 + 2 * FA_TILE;
  static constexpr int BAR = P + FA_TILE;
  static constexpr int BYTES = BAR + 256;
  static constexpr int ALLOC = BYTES + 1024;  // alignment slack
};

struct FaArgs {
  const int32_t* cu;   // [B+1] prompt offsets (tokens)
  const int32_t* vcu;  // [B+1] prompt offsets in the V^T columns (multiples of 8: TMA needs a
                       // 16-B aligned start along the contiguous dimension)
  int B;
  int Hq, Hkv;
  float scale_log2;  // softmax scale * log2(e)
  __nv_bfloat16* o;  // [T, Hq, d]
};

// (prompt, q tile) of linear tile u: prompts in order, each prompt's tiles heaviest first
__device__ bool fa_tile(const int32_t* cu, int B, int u, int& b, int& tile, int& start, int& len) {
  // linear scan over the prompts (one thread per CTA)
  int acc = 0;
  for (int i = 0; i < B; ++i) {
    const int s = cu[i], L = cu[i + 1] - s;
    const int nt = (L + FA_BM - 1) / FA_BM;
    if (u < acc + nt) {
      b = i;
      start = s;
      len = L;
      tile = nt - 1 - (u - acc);
      return true;
    }
    acc += nt;
  }
  return false;
}

__global__ void __launch_bounds__(FA_NTHREADS, 1)
    flash_attn_kernel(const __grid_constant__ CUtensorMap map_q, const __grid_constant__ CUtensorMap map_k,
                      const __grid_constant__ CUtensorMap map_vt, const FaArgs p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + FaSmem::BAR);
  uint64_t* q_full = bars + 0;
  uint64_t* k_full = bars + 1;   // [2]
  uint64_t* k_empty = bars + 3;  // [2]
  uint64_t* v_full = bars + 5;   // [2]
  uint64_t* v_empty = bars + 7;  // [2]
  uint64_t* s_full = bars + 9;   // [2]
  uint64_t* s_empty = bars + 11; // [2]
  uint64_t* p_full = bars + 13;
  uint64_t* pv_done = bars + 14;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 16);
  __shared__ int s_tile[4];

  const int warp = warp_id(), lane = lane_id();
  const int head = blockIdx.x;
  if (threadIdx.x == 0) {
    int b = 0, tile = 0, start = 0, len = 0;
    const bool ok = fa_tile(p.cu, p.B, blockIdx.y, b, tile, start, len);
    s_tile[0] = ok ? tile : -1;
    s_tile[1] = start;
    s_tile[2] = len;
    s_tile[3] = ok ? p.vcu[b] : 0;
  }
  __syncthreads();
  const int tile = s_tile[0];
  if (tile < 0) return;  // past the last tile of the batch (grid is an upper bound)
  const int start = s_tile[1], len = s_tile[2], vstart = s_tile[3];
  const int q0 = tile * FA_BM;        // first query position in the prompt
  const int nblk = tile + 1;          // causal: key blocks 0..tile
  const int kvh = head / (p.Hq / p.Hkv);

  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&k_full[i], 1);
      mbar_init(&k_empty[i], 1);
      mbar_init(&v_full[i], 1);
      mbar_init(&v_empty[i], 1);
      mbar_init(&s_full[i], 1);
      mbar_init(&s_empty[i], 4);
    }
    mbar_init(p_full, 4);
    mbar_init(pv_done, 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t t_s[2] = {tmem, tmem + 128};
  const uint32_t t_o = tmem + 256;

  if (warp == 0) {
    if (lane == 0) {
      tma_prefetch_desc(&map_q);
      tma_prefetch_desc(&map_k);
      tma_prefetch_desc(&map_vt);
      mbar_arrive_expect_tx(q_full, FA_TILE);
      for (int c = 0; c < 2; ++c)
        tma_load_3d_nohint(smem + FaSmem::Q + c * FA_KB, &map_q, q_full, c * 64, head, start + q0);
      for (int j = 0; j < nblk; ++j) {
        const int st = j & 1;
        const uint32_t ph = ((j >> 1) & 1) ^ 1;
        const int key0 = start + j * FA_BN;
        mbar_wait(&k_empty[st], ph);
        mbar_arrive_expect_tx(&k_full[st], FA_TILE);
        for (int c = 0; c < 2; ++c)
          tma_load_3d_nohint(smem + FaSmem::K0 + st * FA_TILE + c * FA_KB, &map_k, &k_full[st], c * 64, kvh, key0);
        mbar_wait(&v_empty[st], ph);
        mbar_arrive_expect_tx(&v_full[st], FA_TILE);
        for (int c = 0; c < 2; ++c)
          tma_load_3d_nohint(smem + FaSmem::V0 + st * FA_TILE + c * FA_KB, &map_vt, &v_full[st],
                             vstart + j * FA_BN + c * 64, 0, kvh);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    constexpr uint32_t idesc = make_idesc(FA_BM, FA_BN, true);  // M = 128, N = 128 (keys or d)
    const uint64_t dq = make_smem_desc_sw128(smem_u32(smem + FaSmem::Q));
    const uint64_t dk = make_smem_desc_sw128(smem_u32(smem + FaSmem::K0));
    const uint64_t dv = make_smem_desc_sw128(smem_u32(smem + FaSmem::V0));
    const uint64_t dp = make_smem_desc_sw128(smem_u32(smem + FaSmem::P));
    constexpr uint64_t kKb = FA_KB >> 4, kTile = FA_TILE >> 4;
    mbar_wait(q_full, 0);
    auto issue_s = [&](int j) {  // S_j = Q K_j^T into S[j & 1]
      const int st = j & 1;
      mbar_wait(&k_full[st], (j >> 1) & 1);
      mbar_wait(&s_empty[st], ((j >> 1) & 1) ^ 1);
      tc_fence_after();
      if (elect_one()) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {  // d = 128 = 2 k-blocks x 4 steps of 16
          const uint64_t off = (uint64_t)(k >> 2) * kKb + (uint64_t)(k & 3) * 2;
          mma_bf16(t_s[st], dq + off, dk + st * kTile + off, idesc, k > 0 ? 1u : 0u);
        }
        tc_commit(&s_full[st]);
        tc_commit(&k_empty[st]);
      }
      __syncwarp();
    };
    issue_s(0);
    for (int j = 0; j < nblk; ++j) {
      if (j + 1 < nblk) issue_s(j + 1);
      const int st = j & 1;
      mbar_wait(p_full, j & 1);
      mbar_wait(&v_full[st], (j >> 1) & 1);
      tc_fence_after();
      if (elect_one()) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {  // keys = 128 = 2 k-blocks x 4 steps of 16
          const uint64_t off = (uint64_t)(k >> 2) * kKb + (uint64_t)(k & 3) * 2;
          mma_bf16(t_o, dp + off, dv + st * kTile + off, idesc, (j > 0 || k > 0) ? 1u : 0u);
        }
        tc_commit(pv_done);
        tc_commit(&v_empty[st]);
      }
      __syncwarp();
    }
  } else if (warp >= 4) {
    const int ew = warp - 4;
    const int r = ew * 32 + lane;           // query row in the tile
    const int qpos = q0 + r;                // position in the prompt
    const uint32_t lane_off = (uint32_t)(ew * 32) << 16;
    float m_used = -1e30f, l = 0.f;
    const uint32_t p_base = smem_u32(smem + FaSmem::P) + (uint32_t)r * 128;
    for (int j = 0; j < nblk; ++j) {
      const int st = j & 1;
      mbar_wait(&s_full[st], (j >> 1) & 1);
      tc_fence_after();
      uint32_t s[128];
#pragma unroll
      for (int c = 0; c < 4; ++c) tmem_ld32(t_s[st] + lane_off + c * 32, *reinterpret_cast<uint32_t(*)[32]>(s + 32 * c));
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&s_empty[st]);
      // scale to log2 units, mask, row max
      const bool diag = (j == nblk - 1);
      const int kpos0 = j * FA_BN;
      float mx = -1e30f;
#pragma unroll
      for (int c = 0; c < 128; ++c) {
        float v = __uint_as_float(s[c]) * p.scale_log2;
        if (diag && (kpos0 + c > qpos || kpos0 + c >= len)) v = -INFINITY;
        s[c] = __float_as_uint(v);
        mx = fmaxf(mx, v);
      }
      float alpha = 1.f;
      const bool resc = mx > m_used + kRescaleThresh;
      if (resc) {
        alpha = fast_exp2(m_used - mx);
        m_used = mx;
        l *= alpha;
      }
      // p = exp2(s - m), row sum, bf16 pack (64 words)
      uint32_t pk[64];
      float sum = 0.f;
#pragma unroll
      for (int c = 0; c < 64; ++c) {
        const float a = fast_exp2(__uint_as_float(s[2 * c]) - m_used);
        const float b = fast_exp2(__uint_as_float(s[2 * c + 1]) - m_used);
        sum += a + b;
        pk[c] = pack_bf16x2(a, b);
      }
      l += sum;
      // PV_{j-1} done: the P buffer is free and O is final for blocks < j
      if (j > 0) mbar_wait(pv_done, (j - 1) & 1);
      tc_fence_after();
      if (j > 0 && __any_sync(0xffffffffu, resc)) {  // rare: rescale this warp's O rows in TMEM
#pragma unroll 1
        for (int c = 0; c < 4; ++c) {
          uint32_t o[32];
          tmem_ld32(t_o + lane_off + c * 32, o);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
          tmem_st32(t_o + lane_off + c * 32, o);
        }
        tmem_st_wait();
      }
      // P row -> smem: 2 k-blocks of 64 keys, 16-B chunk q of row r at (q ^ (r & 7))
#pragma unroll
      for (int kb = 0; kb < 2; ++kb)
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int w0 = kb * 32 + q * 4;
          st_shared_v4(p_base + kb * FA_KB + ((q ^ (r & 7)) << 4), pk[w0], pk[w0 + 1], pk[w0 + 2], pk[w0 + 3]);
        }
      fence_proxy_async_smem();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(p_full);
    }
    // epilogue: O / l -> bf16 -> o[start + qpos, head, :]
    mbar_wait(pv_done, (nblk - 1) & 1);
    tc_fence_after();
    const float inv = 1.f / l;
    const bool valid = qpos < len;
    __nv_bfloat16* dst = p.o + ((int64_t)(start + qpos) * p.Hq + head) * FA_D;
#pragma unroll 1
    for (int c = 0; c < 4; ++c) {
      uint32_t o[32];
      tmem_ld32(t_o + lane_off + c * 32, o);
      tmem_ld_wait();
      if (valid) {
#pragma unroll
        for (int i = 0; i < 32; i += 8) {
          uint4 v;
          v.x = pack_bf16x2(__uint_as_float(o[i]) * inv, __uint_as_float(o[i + 1]) * inv);
          v.y = pack_bf16x2(__uint_as_float(o[i + 2]) * inv, __uint_as_float(o[i + 3]) * inv);
          v.z = pack_bf16x2(__uint_as_float(o[i + 4]) * inv, __uint_as_float(o[i + 5]) * inv);
          v.w = pack_bf16x2(__uint_as_float(o[i + 6]) * inv, __uint_as_float(o[i + 7]) * inv);
          *reinterpret_cast<uint4*>(dst + c * 32 + i) = v;
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// ------------------------------------------------------------------ elementwise kernels
// RMSNorm of rows of n (multiple of 8) bf16 values: warp per row, fp32 math.
__global__ void __launch_bounds__(256) rmsnorm_kernel(const __nv_bfloat16* __restrict__ x,
                                                      const __nv_bfloat16* __restrict__ w, int64_t rows, int n,
                                                      float eps, __nv_bfloat16* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t r = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (r >= rows) return;
  const uint4* src = reinterpret_cast<const uint4*>(x + r * n);
  const int nv = n / 8;
  float ss = 0.f;
  for (int v = lane; v < nv; v += 32) {
    const uint4 u = src[v];
    const uint32_t a[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) ss += bf16_lo(a[q]) * bf16_lo(a[q]) + bf16_hi(a[q]) * bf16_hi(a[q]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  const float rs = rsqrtf(ss / n + eps);
  const uint4* wv = reinterpret_cast<const uint4*>(w);
  uint4* dst = reinterpret_cast<uint4*>(out + r * n);
  for (int v = lane; v < nv; v += 32) {
    const uint4 u = src[v], g = wv[v];
    const uint32_t a[4] = {u.x, u.y, u.z, u.w}, b[4] = {g.x, g.y, g.z, g.w};
    uint32_t o[4];
#pragma unroll
    for (int q = 0; q < 4; ++q)
      o[q] = pack_bf16x2(bf16_lo(a[q]) * rs * bf16_lo(b[q]), bf16_hi(a[q]) * rs * bf16_hi(b[q]));
    dst[v] = make_uint4(o[0], o[1], o[2], o[3]);
  }
}

// x' = bf16(x + a); xn2 = RMSNorm(x'; w) (the norm reads the rounded x', as the next layer does)
__global__ void __launch_bounds__(256) residual_rmsnorm_kernel(const __nv_bfloat16* __restrict__ x,
                                                               const __nv_bfloat16* __restrict__ a,
                                                               const __nv_bfloat16* __restrict__ w, int64_t rows,
                                                               int n, float eps, __nv_bfloat16* __restrict__ xo,
                                                               __nv_bfloat16* __restrict__ xn) {
  const int lane = threadIdx.x & 31;
  const int64_t r = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (r >= rows) return;
  const uint4* xs = reinterpret_cast<const uint4*>(x + r * n);
  const uint4* as = reinterpret_cast<const uint4*>(a + r * n);
  uint4* xd = reinterpret_cast<uint4*>(xo + r * n);
  const int nv = n / 8;
  float ss = 0.f;
  for (int v = lane; v < nv; v += 32) {
    const uint4 u = xs[v], b = as[v];
    const uint32_t p[4] = {u.x, u.y, u.z, u.w}, q[4] = {b.x, b.y, b.z, b.w};
    uint32_t o[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      o[i] = pack_bf16x2(bf16_lo(p[i]) + bf16_lo(q[i]), bf16_hi(p[i]) + bf16_hi(q[i]));
      ss += bf16_lo(o[i]) * bf16_lo(o[i]) + bf16_hi(o[i]) * bf16_hi(o[i]);
    }
    xd[v] = make_uint4(o[0], o[1], o[2], o[3]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  const float rs = rsqrtf(ss / n + eps);
  __syncwarp();
  const uint4* wv = reinterpret_cast<const uint4*>(w);
  uint4* nd = reinterpret_cast<uint4*>(xn + r * n);
  for (int v = lane; v < nv; v += 32) {
    const uint4 u = xd[v], g = wv[v];  // this lane wrote xd[v] itself
    const uint32_t p[4] = {u.x, u.y, u.z, u.w}, b[4] = {g.x, g.y, g.z, g.w};
    uint32_t o[4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
      o[i] = pack_bf16x2(bf16_lo(p[i]) * rs * bf16_lo(b[i]), bf16_hi(p[i]) * rs * bf16_hi(b[i]));
    nd[v] = make_uint4(o[0], o[1], o[2], o[3]);
  }
}

// q / k heads of the fused QKV rows: per-head RMSNorm (d = 128) then rotate-half RoPE at the
// token's position in its prompt.  One warp per (token, head); lane holds elements
// lane, lane+32, lane+64, lane+96 (pairs (i, i+64)).
__global__ void __launch_bounds__(256) qk_rope_kernel(const __nv_bfloat16* __restrict__ qkv, int64_t T, int Hq,
                                                      int Hkv, const int32_t* __restrict__ cu, int B,
                                                      const __nv_bfloat16* __restrict__ w_qn,
                                                      const __nv_bfloat16* __restrict__ w_kn, float eps,
                                                      float log2_theta, __nv_bfloat16* __restrict__ q_out,
                                                      __nv_bfloat16* __restrict__ k_out) {
  const int lane = threadIdx.x & 31;
  const int nh = Hq + Hkv;
  const int64_t gw = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (gw >= T * nh) return;
  const int64_t t = gw / nh;
  const int hh = (int)(gw - t * nh);
  // position of t in its prompt (binary search over cu)
  int lo = 0, hi = B;  // cu[lo] <= t < cu[hi]
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (cu[mid] <= t) lo = mid;
    else hi = mid;
  }
  const float pos = (float)(t - cu[lo]);
  const __nv_bfloat16* src = qkv + t * (int64_t)(Hq + 2 * Hkv) * FA_D + (int64_t)hh * FA_D;
  const __nv_bfloat16* w = hh < Hq ? w_qn : w_kn;
  float v[4], g[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    v[i] = __bfloat162float(src[lane + 32 * i]);
    g[i] = __bfloat162float(w[lane + 32 * i]);
  }
  float ss = v[0] * v[0] + v[1] * v[1] + v[2] * v[2] + v[3] * v[3];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  const float rs = rsqrtf(ss / FA_D + eps);
  // the normalised head is rounded to bf16 (as a separate norm kernel would store it)
#pragma unroll
  for (int i = 0; i < 4; ++i) v[i] = __bfloat162float(__float2bfloat16_rn(v[i] * rs * g[i]));
  __nv_bfloat16* dst = hh < Hq ? q_out + (t * Hq + hh) * FA_D : k_out + (t * Hkv + (hh - Hq)) * FA_D;
#pragma unroll
  for (int i = 0; i < 2; ++i) {  // pair (e, e + 64), e = lane + 32 i
    const int e = lane + 32 * i;
    const float inv_freq = exp2f(-(2.0f * e / FA_D) * log2_theta);
    float sn, cs;
    sincosf(pos * inv_freq, &sn, &cs);
    const float a = v[i], b = v[i + 2];
    dst[e] = __float2bfloat16_rn(a * cs - b * sn);
    dst[e + 64] = __float2bfloat16_rn(b * cs + a * sn);
  }
}

// V of the fused QKV rows -> V^T [Hkv][d][ldv] (tokens contiguous; prompt b's keys at columns
// vcu[b] + position): 32 x 32 smem transpose.  Pad columns are zeroed by the caller.
__global__ void __launch_bounds__(256) v_transpose_kernel(const __nv_bfloat16* __restrict__ qkv, int64_t T, int Hq,
                                                          int Hkv, const int32_t* __restrict__ cu,
                                                          const int32_t* __restrict__ vcu, int B, int64_t ldv,
                                                          __nv_bfloat16* __restrict__ vt) {
  __shared__ __nv_bfloat16 tile[32][33];
  __shared__ int64_t col[32];
  const int64_t t0 = (int64_t)blockIdx.x * 32;
  const int c0 = blockIdx.y * 32;  // column in [0, Hkv d)
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int64_t ld = (int64_t)(Hq + 2 * Hkv) * FA_D;
  const __nv_bfloat16* v = qkv + (int64_t)(Hq + Hkv) * FA_D;
  if (ty == 0) {
    const int64_t t = t0 + tx;
    int64_t c = -1;
    if (t < T) {
      int lo = 0, hi = B;  // cu[lo] <= t < cu[hi]
      while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (cu[mid] <= t) lo = mid;
        else hi = mid;
      }
      c = vcu[lo] + (t - cu[lo]);
    }
    col[tx] = c;
  }
  for (int i = ty; i < 32; i += 8) {
    const int64_t t = t0 + i;
    tile[i][tx] = t < T ? v[t * ld + c0 + tx] : __float2bfloat16_rn(0.f);
  }
  __syncthreads();
  const int64_t c = col[tx];
  if (c < 0) return;
  for (int i = ty; i < 32; i += 8) vt[(int64_t)(c0 + i) * ldv + c] = tile[tx][i];
}

// vcu[b] = sum_{i<b} roundup8(cu[i+1] - cu[i]): one block, chunked scan.
__global__ void __launch_bounds__(1024) vt_offsets_kernel(const int32_t* __restrict__ cu, int B,
                                                          int32_t* __restrict__ vcu) {
  __shared__ int32_t part[1024];
  __shared__ int32_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int base = 0; base < B; base += 1024) {
    const int b = base + threadIdx.x;
    const int32_t n = b < B ? (cu[b + 1] - cu[b] + 7) / 8 * 8 : 0;
    part[threadIdx.x] = n;
    __syncthreads();
    for (int off = 1; off < 1024; off <<= 1) {  // inclusive Hillis-Steele scan
      const int32_t v = threadIdx.x >= off ? part[threadIdx.x - off] : 0;
      __syncthreads();
      part[threadIdx.x] += v;
      __syncthreads();
    }
    if (b < B) vcu[b + 1] = carry + part[threadIdx.x];
    __syncthreads();
    if (threadIdx.x == 1023) carry += part[1023];
    __syncthreads();
  }
  if (threadIdx.x == 0) vcu[0] = 0;
}

}  // namespace

// ------------------------------------------------------------------ launchers
void launch_rmsnorm(const bf16* x, const bf16* w, int64_t rows, int n, float eps, bf16* out, cudaStream_t s) {
  if (rows <= 0) return;
  rmsnorm_kernel<<<(unsigned)((rows + 7) / 8), 256, 0, s>>>(x, w, rows, n, eps, out);
}

void launch_residual_rmsnorm(const bf16* x, const bf16* a, const bf16* w, int64_t rows, int n, float eps, bf16* xo,
                             bf16* xn, cudaStream_t s) {
  if (rows <= 0) return;
  residual_rmsnorm_kernel<<<(unsigned)((rows + 7) / 8), 256, 0, s>>>(x, a, w, rows, n, eps, xo, xn);
}

void launch_qk_rope(const bf16* qkv, int64_t T, int Hq, int Hkv, const int32_t* cu, int B, const bf16* w_qn,
                    const bf16* w_kn, float eps, float theta, bf16* q, bf16* k, cudaStream_t s) {
  if (T <= 0) return;
  const int64_t warps = T * (Hq + Hkv);
  qk_rope_kernel<<<(unsigned)((warps + 7) / 8), 256, 0, s>>>(qkv, T, Hq, Hkv, cu, B, w_qn, w_kn, eps, log2f(theta),
                                                             q, k);
}

void launch_v_transpose(const bf16* qkv, int64_t T, int Hq, int Hkv, const int32_t* cu, int B, int32_t* vcu,
                        int64_t ldv, bf16* vt, cudaStream_t s) {
  if (T <= 0) return;
  vt_offsets_kernel<<<1, 1024, 0, s>>>(cu, B, vcu);
  cudaMemsetAsync(vt, 0, (size_t)Hkv * FA_D * ldv * 2, s);  // pad columns must be finite (P = 0 there)
  dim3 grid((unsigned)((T + 31) / 32), (unsigned)(Hkv * FA_D / 32));
  v_transpose_kernel<<<grid, 256, 0, s>>>(qkv, T, Hq, Hkv, cu, vcu, B, ldv, vt);
}

bool launch_flash_attn(const bf16* q, const bf16* k, const bf16* vt, int64_t ldv, const int32_t* cu,
                       const int32_t* vcu, int B, int64_t T, int Hq, int Hkv, bf16* o, cudaStream_t s) {
  if (T <= 0 || B <= 0) return true;
  CUtensorMap mq, mk, mv;
  {
    const uint64_t dims[3] = {(uint64_t)FA_D, (uint64_t)Hq, (uint64_t)T};
    const uint64_t strides[2] = {(uint64_t)FA_D * 2, (uint64_t)Hq * FA_D * 2};
    const uint32_t box[3] = {64, 1, FA_BM};
    if (!encode_tmap(&mq, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, q, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B))
      return false;
  }
  {
    const uint64_t dims[3] = {(uint64_t)FA_D, (uint64_t)Hkv, (uint64_t)T};
    const uint64_t strides[2] = {(uint64_t)FA_D * 2, (uint64_t)Hkv * FA_D * 2};
    const uint32_t box[3] = {64, 1, FA_BN};
    if (!encode_tmap(&mk, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, k, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B))
      return false;
  }
  {
    const uint64_t dims[3] = {(uint64_t)ldv, (uint64_t)FA_D, (uint64_t)Hkv};
    const uint64_t strides[2] = {(uint64_t)ldv * 2, (uint64_t)FA_D * ldv * 2};
    const uint32_t box[3] = {64, FA_D, 1};
    if (!encode_tmap(&mv, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, vt, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B))
      return false;
  }
  static std::once_flag once;
  std::call_once(once, [] {
    cudaFuncSetAttribute(flash_attn_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, FaSmem::ALLOC);
  });
  FaArgs a{};
  a.cu = cu;
  a.vcu = vcu;
  a.B = B;
  a.Hq = Hq;
  a.Hkv = Hkv;
  a.scale_log2 = (float)(1.4426950408889634 / sqrt((double)FA_D));
  a.o = o;
  const int64_t tiles_upper = (T + FA_BM - 1) / FA_BM + B;  // sum_b ceil(L_b / 128) <= this
  dim3 grid((unsigned)Hq, (unsigned)tiles_upper);
  flash_attn_kernel<<<grid, FA_NTHREADS, FaSmem::ALLOC, s>>>(mq, mk, mv, a);
  return true;
}

}  // namespace aep
