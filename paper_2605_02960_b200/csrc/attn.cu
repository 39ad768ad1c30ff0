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
// flash_attn4 (the kernel below) is a persistent CTA per SM holding two 128-query tiles of one
// (prompt, head) item, P kept in TMEM.  Earlier generations -- a single-tile kernel (P through
// smem), the non-persistent two-tile kernel ("v2") and a 64-key variant ("v3") -- were measured
// slower and removed (S6, profiles/r01/ab_attn_*.log).
// The rows of a tile past the end of its prompt are computed but never stored.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdlib>
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
constexpr float kRescaleThresh = 8.0f;  // log2 units

struct FaArgs {
  const int32_t* cu;   // [B+1] prompt offsets (tokens)
  const int32_t* vcu;  // [B+1] prompt offsets in the V^T columns (multiples of 8: TMA needs a
                       // 16-B aligned start along the contiguous dimension)
  int B;
  int Hq, Hkv;
  float scale_log2;  // softmax scale * log2(e)
  __nv_bfloat16* o;  // [T, Hq, d]
};

// 2^x on the FMA / ALU pipes (FA-style SFU offload): x = n + f with n = rint(x) by the 1.5 * 2^23
// magic add, 2^f on [-1/2, 1/2] by a cubic (rel. err 7.7e-5, far below the bf16 rounding of P),
// and 2^n added to the exponent bits.  x is clamped at -125 (masked -inf -> 2^-125 ~ 0; the
// exponent field then stays >= 1).
__device__ __forceinline__ float poly_exp2(float x) {
  x = fmaxf(x, -125.f);
  const float t = x + 12582912.f;
  const float f = x - (t - 12582912.f);
  float p = fmaf(0.05508877f, f, 0.24260466f);
  p = fmaf(p, f, 0.69327628f);
  p = fmaf(p, f, 0.9999289f);
  return __int_as_float(__float_as_int(p) + (__float_as_int(t) << 23));
}

#ifndef FA_POLY_EVERY
#define FA_POLY_EVERY 4  // one exp2 in FA_POLY_EVERY pairs on the FMA pipe (0: all on the SFU)
#endif

// ------------------------------------------------------------------ flash attention, two query tiles
// v2: one CTA per (query head, pair of 128-query tiles of a prompt) = 256 queries sharing every
// K / V^T block (half the operand traffic per FLOP of v1).  320 threads:
//   warps 0-3  softmax of tile A (rows 0-127), warps 4-7 softmax of tile B (rows 128-255):
//              two softmax warps per SMSP, so one's exp / pack / max latency hides the other's
//   warp 8     TMA producer (Q_A, Q_B once; K and V^T blocks in a 2-stage ring)
//   warp 9     TMEM allocator + MMA issuer
// TMEM (512 columns): per tile t, S_t at [256t, 256t + 128) and O_t at [256t + 128, 256t + 256).
// P_t is written by the softmax threads (tcgen05.st, bf16 pairs) over the first 64 columns of
// S_t and read from TMEM by PV_t (A operand in TMEM, "ts" MMA) -- no smem round trip, no proxy
// fence.  Issue order per key block j: PV_A(j), S_A(j+1), PV_B(j), S_B(j+1); the tensor pipe
// executes one thread's MMAs in order, so S_t(j+1) overwrites S/P_t only after PV_t(j) read it,
// and each softmax group has the other tile's PV + S time to produce its next P.
constexpr int FA2_NTHREADS = 320;
struct Fa2Smem {
  static constexpr int QA = 0;
  static constexpr int QB = QA + FA_TILE;
  static constexpr int K0 = QB + FA_TILE;
  static constexpr int V0 = K0 + 2 * FA_TILE;
  static constexpr int BAR = V0 + 2 * FA_TILE;
  static constexpr int BYTES = BAR + 256;
  static constexpr int ALLOC = BYTES + 1024;
};

// (prompt, tile pair) of linear index u: prompts in order, each prompt's pairs heaviest first
__device__ bool fa2_pair(const int32_t* cu, int B, int u, int& b, int& pair, int& start, int& len) {
  int acc = 0;
  for (int i = 0; i < B; ++i) {
    const int s = cu[i], L = cu[i + 1] - s;
    const int np = (L + 2 * FA_BM - 1) / (2 * FA_BM);
    if (u < acc + np) {
      b = i;
      start = s;
      len = L;
      pair = np - 1 - (u - acc);
      return true;
    }
    acc += np;
  }
  return false;
}

// ------------------------------------------------------------------ flash attention v4 (persistent v2)
// v2's CTA (two query tiles, P in TMEM, two softmax warpgroups), made persistent: one CTA per SM
// walks the (pair, head) work items heaviest-first (item w: head = w % Hq, pair list index
// w / Hq), and the per-item fixed costs overlap the neighbouring items: the producer loads the
// next item's Q as soon as the current item's last S has read Q (q_empty), the MMA starts the
// next item's S while the softmax warps finish the current item, and the next PV waits only
// for the softmax warps to have read O out of TMEM (o_empty).  All barrier phases run on
// counters that continue across items.
__device__ __forceinline__ bool fa4_item(const FaArgs& p, int w, int& head, int& start, int& len, int& vstart,
                                         int& pair) {
  head = w % p.Hq;
  int b = 0;
  if (!fa2_pair(p.cu, p.B, w / p.Hq, b, pair, start, len)) return false;  // past the last pair
  vstart = p.vcu[b];
  return true;
}

constexpr int FA4_RING = 4;
// consumer side of the work-item ring: lane 0 waits for item number seq and releases its slot
__device__ __forceinline__ int fa4_next(uint64_t* r_full, uint64_t* r_empty, const int32_t* ring, int seq, int lane) {
  int w = 0;
  if (lane == 0) {
    const int slot = seq % FA4_RING;
    mbar_wait(&r_full[slot], (uint32_t)(seq / FA4_RING) & 1u);
    w = ring[slot];
    mbar_arrive(&r_empty[slot]);
  }
  return __shfl_sync(0xffffffffu, w, 0);
}

__global__ void __launch_bounds__(FA2_NTHREADS, 1)
    flash_attn4_kernel(const __grid_constant__ CUtensorMap map_q, const __grid_constant__ CUtensorMap map_k,
                       const __grid_constant__ CUtensorMap map_vt, const FaArgs p, int n_items, int* sched) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Fa2Smem::BAR);
  uint64_t* q_full = bars + 0;
  uint64_t* q_empty = bars + 1;
  uint64_t* k_full = bars + 2;    // [2]
  uint64_t* k_empty = bars + 4;   // [2]
  uint64_t* v_full = bars + 6;    // [2]
  uint64_t* v_empty = bars + 8;   // [2]
  uint64_t* s_full = bars + 10;   // [tile]
  uint64_t* p_full = bars + 12;   // [tile]
  uint64_t* pv_done = bars + 14;  // [tile]
  uint64_t* o_empty = bars + 16;  // [tile]
  uint64_t* r_full = bars + 18;   // [FA4_RING] work-item ring: published
  uint64_t* r_empty = bars + 22;  // [FA4_RING]                 consumed (MMA + 8 softmax warps)
  int32_t* ring = reinterpret_cast<int32_t*>(bars + 26);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(ring + FA4_RING);

  const int warp = warp_id(), lane = lane_id();
  if (threadIdx.x == 0) {
    for (int i = 0; i < FA4_RING; ++i) {
      mbar_init(&r_full[i], 1);
      mbar_init(&r_empty[i], 9);
    }
    mbar_init(q_full, 1);
    mbar_init(q_empty, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&k_full[i], 1);
      mbar_init(&k_empty[i], 1);
      mbar_init(&v_full[i], 1);
      mbar_init(&v_empty[i], 1);
      mbar_init(&s_full[i], 1);
      mbar_init(&p_full[i], 4);
      mbar_init(&pv_done[i], 1);
      mbar_init(&o_empty[i], 4);
    }
    fence_barrier_init();
  }
  if (warp == 9) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 8) {
    if (lane == 0) {
      tma_prefetch_desc(&map_q);
      tma_prefetch_desc(&map_k);
      tma_prefetch_desc(&map_vt);
      int g = 0;  // K/V blocks loaded so far (ring position)
      for (int it = 0;; ++it) {
        // scheduler: take the next work item from the global counter and publish it to the
        // MMA and softmax warps through the ring (heavier items come first in the item order)
        const int slot = it % FA4_RING;
        mbar_wait(&r_empty[slot], ((uint32_t)(it / FA4_RING) & 1u) ^ 1u);
        const int w = atomicAdd(sched, 1);
        ring[slot] = w;
        mbar_arrive(&r_full[slot]);
        int head, start, len, vstart, pair;
        if (w >= n_items || !fa4_item(p, w, head, start, len, vstart, pair)) break;
        const int q0 = pair * 2 * FA_BM, nB = 2 * pair + 2, kvh = head / (p.Hq / p.Hkv);
        mbar_wait(q_empty, (it & 1) ^ 1);  // the previous item's S MMAs are done with Q
        mbar_arrive_expect_tx(q_full, 2 * FA_TILE);
        for (int c = 0; c < 2; ++c) {
          tma_load_3d_nohint(smem + Fa2Smem::QA + c * FA_KB, &map_q, q_full, c * 64, head, start + q0);
          tma_load_3d_nohint(smem + Fa2Smem::QB + c * FA_KB, &map_q, q_full, c * 64, head, start + q0 + FA_BM);
        }
        for (int j = 0; j < nB; ++j, ++g) {
          const int st = g & 1;
          const uint32_t ph = ((g >> 1) & 1) ^ 1;
          mbar_wait(&k_empty[st], ph);
          mbar_arrive_expect_tx(&k_full[st], FA_TILE);
          for (int c = 0; c < 2; ++c)
            tma_load_3d_nohint(smem + Fa2Smem::K0 + st * FA_TILE + c * FA_KB, &map_k, &k_full[st], c * 64, kvh,
                               start + j * FA_BN);
          mbar_wait(&v_empty[st], ph);
          mbar_arrive_expect_tx(&v_full[st], FA_TILE);
          for (int c = 0; c < 2; ++c)
            tma_load_3d_nohint(smem + Fa2Smem::V0 + st * FA_TILE + c * FA_KB, &map_vt, &v_full[st],
                               vstart + j * FA_BN + c * 64, 0, kvh);
        }
      }
    }
    __syncwarp();
  } else if (warp == 9) {
    constexpr uint32_t idesc = make_idesc(FA_BM, FA_BN, true);
    const uint64_t dq[2] = {make_smem_desc_sw128(smem_u32(smem + Fa2Smem::QA)),
                            make_smem_desc_sw128(smem_u32(smem + Fa2Smem::QB))};
    const uint64_t dk = make_smem_desc_sw128(smem_u32(smem + Fa2Smem::K0));
    const uint64_t dv = make_smem_desc_sw128(smem_u32(smem + Fa2Smem::V0));
    constexpr uint64_t kKb = FA_KB >> 4, kTile = FA_TILE >> 4;
    int g = 0;                   // K/V ring position
    int ns[2] = {0, 0}, np[2] = {0, 0};  // S issued / PV issued per tile (barrier phases)
    for (int it = 0;; ++it) {
      const int w = fa4_next(r_full, r_empty, ring, it, lane);
      int head, start, len, vstart, pair;
      if (w >= n_items || !fa4_item(p, w, head, start, len, vstart, pair)) break;
      const int nA = 2 * pair + 1, nB = 2 * pair + 2;
      mbar_wait(q_full, it & 1);
      auto issue_s = [&](int t, int j, bool last) {
        const int gg = g + j, st = gg & 1;
        if (t == 0 || j >= nA) mbar_wait(&k_full[st], (gg >> 1) & 1);
        tc_fence_after();
        if (elect_one()) {
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const uint64_t off = (uint64_t)(k >> 2) * kKb + (uint64_t)(k & 3) * 2;
            mma_bf16(tmem + 256 * t, dq[t] + off, dk + st * kTile + off, idesc, k > 0 ? 1u : 0u);
          }
          tc_commit(&s_full[t]);
          if (t == 1) tc_commit(&k_empty[st]);
          if (last) tc_commit(q_empty);  // the item's last read of Q
        }
        __syncwarp();
        ++ns[t];
      };
      auto issue_pv = [&](int t, int j) {
        const int gg = g + j, st = gg & 1;
        mbar_wait(&p_full[t], np[t] & 1);
        if (t == 0 || j >= nA) mbar_wait(&v_full[st], (gg >> 1) & 1);
        if (j == 0 && it > 0) mbar_wait(&o_empty[t], (it - 1) & 1);  // previous item's O has been read out
        tc_fence_after();
        if (elect_one()) {
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const uint64_t off = (uint64_t)(k >> 2) * kKb + (uint64_t)(k & 3) * 2;
            mma_bf16_ts(tmem + 256 * t + 128, tmem + 256 * t + 8 * k, dv + st * kTile + off, idesc,
                        (j > 0 || k > 0) ? 1u : 0u);
          }
          tc_commit(&pv_done[t]);
          if (t == 1) tc_commit(&v_empty[st]);
        }
        __syncwarp();
        ++np[t];
      };
      issue_s(0, 0, false);
      issue_s(1, 0, nB == 1);
      for (int j = 0; j < nB; ++j) {
        if (j < nA) {
          issue_pv(0, j);
          if (j + 1 < nA) issue_s(0, j + 1, false);
        }
        issue_pv(1, j);
        if (j + 1 < nB) issue_s(1, j + 1, j + 2 == nB);
      }
      g += nB;
    }
  } else {
    const int t = warp >> 2;
    const int r = (warp & 3) * 32 + lane;
    const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
    const uint32_t t_s = tmem + 256 * t + lane_off, t_o = t_s + 128;
    const float scl = p.scale_log2;
    int nb = 0;  // blocks processed by this tile's softmax across items (barrier phases)
    for (int it = 0;; ++it) {
      const int w = fa4_next(r_full, r_empty, ring, it, lane);
      int head, start, len, vstart, pair;
      if (w >= n_items || !fa4_item(p, w, head, start, len, vstart, pair)) break;
      const int q0 = pair * 2 * FA_BM;
      const int qpos = q0 + t * FA_BM + r;
      const int nblk = t == 0 ? 2 * pair + 1 : 2 * pair + 2;
      float m_used = -1e30f, l0 = 0.f, l1 = 0.f;
      for (int j = 0; j < nblk; ++j, ++nb) {
        mbar_wait(&s_full[t], nb & 1);
        tc_fence_after();
        uint32_t s[128];
#pragma unroll
        for (int c = 0; c < 4; ++c) tmem_ld32(t_s + c * 32, *reinterpret_cast<uint32_t(*)[32]>(s + 32 * c));
        tmem_ld_wait();
        if (j == nblk - 1 || (t == 1 && j == nblk - 2)) {
          const int lim = min(qpos, len - 1) - j * FA_BN;
#pragma unroll
          for (int c = 0; c < 128; ++c)
            if (c > lim) s[c] = __float_as_uint(-INFINITY);
        }
        float mx = -1e30f;
#pragma unroll
        for (int c = 0; c < 128; c += 2) mx = fmaxf(mx, fmaxf(__uint_as_float(s[c]), __uint_as_float(s[c + 1])));
        mx *= scl;
        float alpha = 1.f;
        const bool resc = mx > m_used + kRescaleThresh;
        if (resc) {
          alpha = fast_exp2(m_used - mx);
          m_used = mx;
          l0 *= alpha;
          l1 *= alpha;
        }
        const float nm = -m_used;
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          uint32_t pk[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const float xa = fmaf(__uint_as_float(s[64 * c + 2 * i]), scl, nm);
            const float xb = fmaf(__uint_as_float(s[64 * c + 2 * i + 1]), scl, nm);
            const bool poly = FA_POLY_EVERY > 0 && (i % (FA_POLY_EVERY > 0 ? FA_POLY_EVERY : 1)) == 0;
            const float a = poly ? poly_exp2(xa) : fast_exp2(xa);
            const float b = poly ? poly_exp2(xb) : fast_exp2(xb);
            add2(l0, l1, l0, l1, a, b);
            pk[i] = pack_bf16x2(a, b);
          }
          tmem_st32(t_s + 32 * c, pk);
        }
        if (j > 0) mbar_wait(&pv_done[t], (nb - 1) & 1);
        tc_fence_after();
        if (j > 0 && __any_sync(0xffffffffu, resc)) {
#pragma unroll 1
          for (int c = 0; c < 4; ++c) {
            uint32_t o[32];
            tmem_ld32(t_o + c * 32, o);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
            tmem_st32(t_o + c * 32, o);
          }
        }
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[t]);
      }
      // epilogue: read O out of TMEM (then release it to the next item), normalise, store
      mbar_wait(&pv_done[t], (nb - 1) & 1);
      tc_fence_after();
      uint32_t o[128];
#pragma unroll
      for (int c = 0; c < 4; ++c) tmem_ld32(t_o + c * 32, *reinterpret_cast<uint32_t(*)[32]>(o + 32 * c));
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&o_empty[t]);
      if (qpos < len) {
        const float inv = 1.f / (l0 + l1);
        __nv_bfloat16* dst = p.o + ((int64_t)(start + qpos) * p.Hq + head) * FA_D;
#pragma unroll
        for (int i = 0; i < 128; i += 8) {
          uint4 v;
          v.x = pack_bf16x2(__uint_as_float(o[i]) * inv, __uint_as_float(o[i + 1]) * inv);
          v.y = pack_bf16x2(__uint_as_float(o[i + 2]) * inv, __uint_as_float(o[i + 3]) * inv);
          v.z = pack_bf16x2(__uint_as_float(o[i + 4]) * inv, __uint_as_float(o[i + 5]) * inv);
          v.w = pack_bf16x2(__uint_as_float(o[i + 6]) * inv, __uint_as_float(o[i + 7]) * inv);
          *reinterpret_cast<uint4*>(dst + i) = v;
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 9) {
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
// token's position in its prompt.  One warp per token: lane l owns the rotation pairs
// (e, e + 64) for e = 2l, 2l + 1, computes their cos / sin once, and walks the token's
// Hq + Hkv heads with 4-byte (bf16x2) loads and stores.
__global__ void __launch_bounds__(256) qk_rope_kernel(const __nv_bfloat16* __restrict__ qkv, int64_t T, int Hq,
                                                      int Hkv, const int32_t* __restrict__ cu, int B,
                                                      const __nv_bfloat16* __restrict__ w_qn,
                                                      const __nv_bfloat16* __restrict__ w_kn, float eps,
                                                      float log2_theta, __nv_bfloat16* __restrict__ q_out,
                                                      __nv_bfloat16* __restrict__ k_out) {
  const int lane = threadIdx.x & 31;
  const int64_t t = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (t >= T) return;
  int lo = 0, hi = B;  // cu[lo] <= t < cu[hi]
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (cu[mid] <= t) lo = mid;
    else hi = mid;
  }
  const float pos = (float)(t - cu[lo]);
  float cs[2], sn[2];
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int e = 2 * lane + i;
    sincosf(pos * exp2f(-(2.0f * e / FA_D) * log2_theta), &sn[i], &cs[i]);
  }
  const uint32_t* wq = reinterpret_cast<const uint32_t*>(w_qn);
  const uint32_t* wk = reinterpret_cast<const uint32_t*>(w_kn);
  const uint32_t gq0 = wq[lane], gq1 = wq[32 + lane], gk0 = wk[lane], gk1 = wk[32 + lane];
  const uint32_t* row = reinterpret_cast<const uint32_t*>(qkv + t * (int64_t)(Hq + 2 * Hkv) * FA_D);
  for (int hh = 0; hh < Hq + Hkv; ++hh) {
    const uint32_t a2 = row[hh * 64 + lane], b2 = row[hh * 64 + 32 + lane];  // (2l, 2l+1), (64+2l, 64+2l+1)
    float v[4] = {bf16_lo(a2), bf16_hi(a2), bf16_lo(b2), bf16_hi(b2)};
    float ss = v[0] * v[0] + v[1] * v[1] + v[2] * v[2] + v[3] * v[3];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    const float rs = rsqrtf(ss / FA_D + eps);
    const bool isq = hh < Hq;
    const uint32_t g0 = isq ? gq0 : gk0, g1 = isq ? gq1 : gk1;
    // the normalised head is rounded to bf16 (as a separate norm kernel would store it)
    const uint32_t n0 = pack_bf16x2(v[0] * rs * bf16_lo(g0), v[1] * rs * bf16_hi(g0));
    const uint32_t n1 = pack_bf16x2(v[2] * rs * bf16_lo(g1), v[3] * rs * bf16_hi(g1));
    const float x0 = bf16_lo(n0), x1 = bf16_hi(n0), y0 = bf16_lo(n1), y1 = bf16_hi(n1);
    uint32_t* dst = reinterpret_cast<uint32_t*>(isq ? q_out + (t * Hq + hh) * FA_D
                                                    : k_out + (t * Hkv + (hh - Hq)) * FA_D);
    dst[lane] = pack_bf16x2(x0 * cs[0] - y0 * sn[0], x1 * cs[1] - y1 * sn[1]);
    dst[32 + lane] = pack_bf16x2(y0 * cs[0] + x0 * sn[0], y1 * cs[1] + x1 * sn[1]);
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
  qk_rope_kernel<<<(unsigned)((T + 7) / 8), 256, 0, s>>>(qkv, T, Hq, Hkv, cu, B, w_qn, w_kn, eps, log2f(theta),
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
                       const int32_t* vcu, int B, int64_t T, int Hq, int Hkv, bf16* o, int* sched,
                       cudaStream_t s) {
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
    cudaFuncSetAttribute(flash_attn4_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, Fa2Smem::ALLOC);
  });
  FaArgs a{};
  a.cu = cu;
  a.vcu = vcu;
  a.B = B;
  a.Hq = Hq;
  a.Hkv = Hkv;
  a.scale_log2 = (float)(1.4426950408889634 / sqrt((double)FA_D));
  a.o = o;
  // exact item count needs the prompt lengths on the host; the upper bound is enough: items past
  // the end map to no pair (fa2_pair fails) -- guarded by counting the real pairs on the device
  const int64_t pairs_upper = (T + 2 * FA_BM - 1) / (2 * FA_BM) + B;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // the dynamic scheduler's counter lives in caller-owned memory (one per call, zeroed on the
  // launching stream), so concurrent calls on different streams / devices never share it
  if (cudaMemsetAsync(sched, 0, sizeof(int), s) != cudaSuccess) return false;
  flash_attn4_kernel<<<sms, FA2_NTHREADS, Fa2Smem::ALLOC, s>>>(mq, mk, mv, a, (int)(pairs_upper * Hq), sched);
  return true;
}

}  // namespace aep
