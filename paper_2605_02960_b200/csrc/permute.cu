// permute.cu -- step (2): local permute / dispatch ("all top-k dispatch
// is local"; "auxiliary kernels (reshaping, token permutation/alignment)").
//
//   hist    : per-CTA (64-token chunk) expert histogram          -> blk_counts[nblk][E]
//   scan    : per-expert exclusive scan over chunks + over experts -> row base of every
//             (chunk, expert), offsets[E+1] (padded to the GEMM M tile), m-tile prefix
//             tile_start[E+1], counts[E]
//   scatter : stable rank of every (t, j) inside its expert in (t, j) order (warp
//             __match_any_sync + popc), then one warp per token copies x_t (16-B vectors)
//             to its k destination rows of X_perm.
// Pure integer work + data movement: the result is bit-exact and deterministic.
#include <cstdlib>

#include "common.cuh"
#include "kernels.cuh"

namespace aep {

namespace {

__global__ void perm_hist_kernel(const int32_t* __restrict__ ids, int64_t T, int k, int E, int nblk,
                                 int32_t* __restrict__ blk_counts) {
  extern __shared__ int32_t hist[];
  for (int e = threadIdx.x; e < E; e += blockDim.x) hist[e] = 0;
  __syncthreads();
  const int64_t t0 = (int64_t)blockIdx.x * kPermTokensPerBlock;
  const int64_t tn = min((int64_t)kPermTokensPerBlock, T - t0);
  const int n = (int)tn * k;
  const int32_t* p = ids + t0 * k;
  for (int i = threadIdx.x; i < n; i += blockDim.x) atomicAdd(&hist[p[i]], 1);
  __syncthreads();
  for (int e = threadIdx.x; e < E; e += blockDim.x) blk_counts[(int64_t)e * nblk + blockIdx.x] = hist[e];
}

// One CTA per expert: exclusive scan of that expert's per-chunk counts (row e of the
// [E][nblk] matrix) -> chunk base inside the expert; the last CTA to finish scans the
// expert totals -> offsets[E+1], tile_start[E+1], counts[E].
constexpr int SCAN_THREADS = 256;
__global__ void __launch_bounds__(SCAN_THREADS) perm_scan_kernel(int32_t* __restrict__ bc, int nblk, int E,
                                                                 int32_t* __restrict__ offsets,
                                                                 int32_t* __restrict__ tile_start,
                                                                 int32_t* __restrict__ counts,
                                                                 unsigned int* __restrict__ done,
                                                                 int32_t* __restrict__ src_tok) {
  __shared__ int32_t warp_tot[SCAN_THREADS / 32];
  __shared__ int32_t tot[kMaxExperts];
  __shared__ int32_t s_off[kMaxExperts + 1];  // padded row offsets (the last CTA's copy)
  __shared__ bool last;
  const int e = blockIdx.x, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  int32_t* row = bc + (int64_t)e * nblk;
  const int per = (nblk + SCAN_THREADS - 1) / SCAN_THREADS;  // consecutive chunks per thread
  const int b0 = tid * per;
  int32_t local = 0;
  for (int i = 0; i < per; ++i)
    if (b0 + i < nblk) local += row[b0 + i];
  // block exclusive scan of `local`
  int32_t incl = local;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int32_t v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) warp_tot[wid] = incl;
  __syncthreads();
  int32_t wbase = 0;
  for (int w = 0; w < wid; ++w) wbase += warp_tot[w];
  int32_t run = wbase + incl - local;
  for (int i = 0; i < per; ++i)
    if (b0 + i < nblk) {
      const int32_t c = row[b0 + i];
      row[b0 + i] = run;
      run += c;
    }
  if (tid == SCAN_THREADS - 1) {
    counts[e] = run;  // expert total (thread holding the last chunk ends at the total)
    __threadfence();
    last = (atomicAdd(done, 1u) == (unsigned)(gridDim.x - 1));
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  for (int i = tid; i < E; i += SCAN_THREADS) tot[i] = ((volatile int32_t*)counts)[i];
  __syncthreads();
  // exclusive scan of the padded tile counts over experts (E <= kMaxExperts <= SCAN_THREADS):
  // offsets[e] = kRowAlign * tile_start[e], expert row ranges padded to kRowAlign
  static_assert(kMaxExperts <= SCAN_THREADS, "one thread per expert");
  const int32_t tiles = tid < E ? (tot[tid] + kRowAlign - 1) / kRowAlign : 0;
  int32_t inc = tiles;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int32_t v = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += v;
  }
  __syncthreads();  // warp_tot is reused
  if (lane == 31) warp_tot[wid] = inc;
  __syncthreads();
  int32_t base = 0;
  for (int w = 0; w < wid; ++w) base += warp_tot[w];
  const int32_t ts = base + inc - tiles;
  if (tid < E) {
    s_off[tid] = ts * kRowAlign;
    offsets[tid] = ts * kRowAlign;
    tile_start[tid] = ts;
  }
  if (tid == E - 1) {
    s_off[E] = (ts + tiles) * kRowAlign;
    offsets[E] = (ts + tiles) * kRowAlign;
    tile_start[E] = ts + tiles;
  }
  if (tid == 0) *done = 0;  // re-arm for the next forward (stream-ordered)
  __syncthreads();
  // padding rows of every expert gather token 0 (their GEMM rows are never read): one warp per
  // expert, offsets from shared memory
  for (int i = wid; i < E; i += SCAN_THREADS / 32) {
    const int32_t b = s_off[i] + tot[i], end = s_off[i + 1];
    for (int r = b + lane; r < end; r += 32) src_tok[r] = 0;
  }
}

// The row copy of the dispatch: the warp's whole token row in registers (VPL 16-B vectors per lane,
// all loads in flight at once), then its k destination rows written with 16-B stores.
template <int VPL>
__device__ __forceinline__ void copy_row_regs(const uint4* __restrict__ src, bf16* __restrict__ xperm,
                                              const int32_t (&d)[kMaxTopK], int k, int H, int lane) {
  uint4 val[VPL];
#pragma unroll
  for (int i = 0; i < VPL; ++i)
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(val[i].x), "=r"(val[i].y), "=r"(val[i].z), "=r"(val[i].w)
                 : "l"(src + lane + 32 * i));
#pragma unroll
  for (int j = 0; j < kMaxTopK; ++j)
    if (j < k) {
      uint4* dst = reinterpret_cast<uint4*>(xperm + (int64_t)d[j] * H) + lane;
#pragma unroll
      for (int i = 0; i < VPL; ++i) dst[32 * i] = val[i];
    }
}

__global__ void __launch_bounds__(256) perm_scatter_kernel(const bf16* __restrict__ x,
                                                           const int32_t* __restrict__ ids,
                                                           const int32_t* __restrict__ blk_base,
                                                           const int32_t* __restrict__ offsets, int nblk,
                                                           int64_t T, int H, int k, int E,
                                                           int32_t* __restrict__ dest,
                                                           int32_t* __restrict__ src_tok,
                                                           bf16* __restrict__ xperm) {
  constexpr int NW = 8;                                        // warps per CTA (blockDim 256)
  constexpr int MAXR = kPermTokensPerBlock * kMaxTopK / (NW * 32);  // rounds of 32 entries per warp
  __shared__ int32_t wcnt[NW][kMaxExperts];  // per (warp, expert): entries, then the warp's base row
  __shared__ int32_t dst[kPermTokensPerBlock * kMaxTopK];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t t0 = (int64_t)blockIdx.x * kPermTokensPerBlock;
  const int tn = (int)min((int64_t)kPermTokensPerBlock, T - t0);
  const int n = tn * k;
  // the chunk's entries in (t, j) order, split into NW contiguous ranges of whole 32-entry rounds
  const int per = ((n + NW * 32 - 1) / (NW * 32)) * 32;
  const int i0 = warp * per;
  for (int e = threadIdx.x; e < NW * E; e += blockDim.x) wcnt[e / E][e % E] = 0;
  __syncthreads();
  const unsigned lt = (1u << lane) - 1u;
  int ev[MAXR];
  // pass 1: this warp's per-expert entry counts
#pragma unroll
  for (int r = 0; r < MAXR; ++r) {
    const int i = i0 + 32 * r + lane;
    const bool valid = 32 * r < per && i < n;
    ev[r] = valid ? ids[t0 * k + i] : -1;
    const unsigned peers = __match_any_sync(0xffffffffu, ev[r]);
    if (valid && (peers & lt) == 0) wcnt[warp][ev[r]] += __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  // per expert: chunk base (offsets + the scan's chunk base), then exclusive prefix over the warps
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    int32_t run = offsets[e] + blk_base[(int64_t)e * nblk + blockIdx.x];  // first row of this chunk in e
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      const int32_t c = wcnt[w][e];
      wcnt[w][e] = run;
      run += c;
    }
  }
  __syncthreads();
  // pass 2: stable rank inside each expert = warp base + rank among this warp's earlier entries
#pragma unroll
  for (int r = 0; r < MAXR; ++r) {
    const int i = i0 + 32 * r + lane;
    const bool valid = 32 * r < per && i < n;
    const int e = ev[r];
    const unsigned peers = __match_any_sync(0xffffffffu, e);
    int d = 0;
    if (valid) d = wcnt[warp][e] + __popc(peers & lt);
    __syncwarp();
    if (valid && (peers & lt) == 0) wcnt[warp][e] += __popc(peers);
    __syncwarp();
    if (valid) {
      dst[i] = d;
      dest[t0 * k + i] = d;
      src_tok[d] = (int32_t)(t0 + i / k);
    }
  }
  if (xperm == nullptr) return;
  __syncthreads();
  // copy: one warp per token, 16-B vectors, each x row read once and written k times
  for (int tl = warp; tl < tn; tl += blockDim.x / 32) {
    const uint4* src = reinterpret_cast<const uint4*>(x + (t0 + tl) * (int64_t)H);
    const int nv = H / 8;
    int32_t d[kMaxTopK];
#pragma unroll
    for (int j = 0; j < kMaxTopK; ++j) d[j] = (j < k) ? dst[tl * k + j] : 0;
    if (H == 4096) { copy_row_regs<16>(src, xperm, d, k, H, lane); continue; }
    if (H == 2048) { copy_row_regs<8>(src, xperm, d, k, H, lane); continue; }
#pragma unroll 4
    for (int v = lane; v < nv; v += 32) {
      uint4 val;
      asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                   : "=r"(val.x), "=r"(val.y), "=r"(val.z), "=r"(val.w)
                   : "l"(src + v));
#pragma unroll
      for (int j = 0; j < kMaxTopK; ++j)
        if (j < k) reinterpret_cast<uint4*>(xperm + (int64_t)d[j] * H)[v] = val;
    }
  }
}
// FP8 dispatch (reading R6): x_t is quantised once per token to OCP E4M3 with a per-token
// scale and written to its k permuted rows:
//   amax = max_i |x_t[i]|;  inv = 448 / amax (fp32);  q_i = e4m3_rn_satfinite(x_t[i] * inv);
//   scale = amax / 448 (fp32), dequantised value = q_i * scale   (amax == 0 -> q = 0, scale = 0)
__global__ void __launch_bounds__(256) perm_quant_kernel(const bf16* __restrict__ x, const int32_t* __restrict__ dest,
                                                         int64_t T, int H, int k, uint8_t* __restrict__ xq,
                                                         float* __restrict__ xscale) {
  const int lane = threadIdx.x & 31;
  const int64_t t = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (t >= T) return;
  const uint4* src = reinterpret_cast<const uint4*>(x + t * H);
  const int nv = H / 8;
  float amax = 0.f;
  for (int v = lane; v < nv; v += 32) {
    const uint4 u = src[v];
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) amax = fmaxf(amax, fmaxf(fabsf(bf16_lo(w[q])), fabsf(bf16_hi(w[q]))));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
  const float inv = amax > 0.f ? 448.0f / amax : 0.f;
  const float sc = amax / 448.0f;
  int32_t d[kMaxTopK];
  if (!dest) k = 1;  // token-major output: row t
#pragma unroll
  for (int j = 0; j < kMaxTopK; ++j) d[j] = (j < k) ? (dest ? dest[t * k + j] : (int32_t)t) : 0;
  for (int v = lane; v < nv; v += 32) {
    const uint4 u = src[v];
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
    uint2 o;
    o.x = (uint32_t)e4m3x2(bf16_lo(w[0]) * inv, bf16_hi(w[0]) * inv) |
          ((uint32_t)e4m3x2(bf16_lo(w[1]) * inv, bf16_hi(w[1]) * inv) << 16);
    o.y = (uint32_t)e4m3x2(bf16_lo(w[2]) * inv, bf16_hi(w[2]) * inv) |
          ((uint32_t)e4m3x2(bf16_lo(w[3]) * inv, bf16_hi(w[3]) * inv) << 16);
#pragma unroll
    for (int j = 0; j < kMaxTopK; ++j)
      if (j < k) reinterpret_cast<uint2*>(xq + (int64_t)d[j] * H)[v] = o;
  }
  if (lane < k) xscale[d[lane]] = sc;
}

// perm_quant_kernel with the row in registers (H = 256 * VPL): one read of x, all VPL 16-B loads
// of a lane in flight at once, 8-B e4m3 stores per destination row (256 contiguous bytes per warp).
template <int VPL>
__global__ void __launch_bounds__(256) perm_quant_reg_kernel(const bf16* __restrict__ x,
                                                             const int32_t* __restrict__ dest, int64_t T, int k,
                                                             uint8_t* __restrict__ xq, float* __restrict__ xscale) {
  constexpr int H = 256 * VPL;
  const int lane = threadIdx.x & 31;
  const int64_t t = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (t >= T) return;
  const uint4* src = reinterpret_cast<const uint4*>(x + t * H);
  uint4 u[VPL];
#pragma unroll
  for (int i = 0; i < VPL; ++i)
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(u[i].x), "=r"(u[i].y), "=r"(u[i].z), "=r"(u[i].w)
                 : "l"(src + lane + 32 * i));
  const int32_t dl = lane < k ? dest[t * k + lane] : 0;
  uint32_t m = 0;  // max |x| over packed bf16 magnitudes (unsigned order = magnitude order)
#pragma unroll
  for (int i = 0; i < VPL; ++i) {
    m = __vmaxu2(m, u[i].x & 0x7fff7fffu);
    m = __vmaxu2(m, u[i].y & 0x7fff7fffu);
    m = __vmaxu2(m, u[i].z & 0x7fff7fffu);
    m = __vmaxu2(m, u[i].w & 0x7fff7fffu);
  }
  float amax = fmaxf(bf16_lo(m), bf16_hi(m));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
  const float inv = amax > 0.f ? 448.0f / amax : 0.f;
  uint2 o[VPL];
#pragma unroll
  for (int i = 0; i < VPL; ++i) {
    const uint32_t w[4] = {u[i].x, u[i].y, u[i].z, u[i].w};
    o[i].x = (uint32_t)e4m3x2(bf16_lo(w[0]) * inv, bf16_hi(w[0]) * inv) |
             ((uint32_t)e4m3x2(bf16_lo(w[1]) * inv, bf16_hi(w[1]) * inv) << 16);
    o[i].y = (uint32_t)e4m3x2(bf16_lo(w[2]) * inv, bf16_hi(w[2]) * inv) |
             ((uint32_t)e4m3x2(bf16_lo(w[3]) * inv, bf16_hi(w[3]) * inv) << 16);
  }
  for (int j = 0; j < k; ++j) {
    const int32_t d = __shfl_sync(0xffffffffu, dl, j);
    uint2* dst = reinterpret_cast<uint2*>(xq + (int64_t)d * H) + lane;
#pragma unroll
    for (int i = 0; i < VPL; ++i) dst[32 * i] = o[i];
  }
  if (lane < k) xscale[dl] = amax / 448.0f;
}

// Token-major form of perm_quant_kernel for the fused dispatch (x_q row t = token t): the same
// rule, with no destination list, so a warp needs few registers and 64 warps fit on an SM.
__global__ void __launch_bounds__(256, 8) quant_tokens_kernel(const bf16* __restrict__ x, int64_t T, int H,
                                                               uint8_t* __restrict__ xq, float* __restrict__ xscale) {
  const int lane = threadIdx.x & 31;
  const int64_t t = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (t >= T) return;
  const uint4* src = reinterpret_cast<const uint4*>(x + t * H);
  const int nv = H / 8;
  float amax = 0.f;
  for (int v = lane; v < nv; v += 32) {
    const uint4 u = src[v];
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) amax = fmaxf(amax, fmaxf(fabsf(bf16_lo(w[q])), fabsf(bf16_hi(w[q]))));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
  const float inv = amax > 0.f ? 448.0f / amax : 0.f;
  uint2* dst = reinterpret_cast<uint2*>(xq + t * H);
  for (int v = lane; v < nv; v += 32) {
    const uint4 u = src[v];
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
    uint2 o;
    o.x = (uint32_t)e4m3x2(bf16_lo(w[0]) * inv, bf16_hi(w[0]) * inv) |
          ((uint32_t)e4m3x2(bf16_lo(w[1]) * inv, bf16_hi(w[1]) * inv) << 16);
    o.y = (uint32_t)e4m3x2(bf16_lo(w[2]) * inv, bf16_hi(w[2]) * inv) |
          ((uint32_t)e4m3x2(bf16_lo(w[3]) * inv, bf16_hi(w[3]) * inv) << 16);
    dst[v] = o;
  }
  if (lane == 0) xscale[t] = amax / 448.0f;
}

// FP8 intermediate: act (bf16, written by the GEMM1 epilogue together with the row amax of
// |act| in act_amax, as fp32 bits) -> e4m3 codes + per-row scale, same rule as above.
__global__ void __launch_bounds__(256) act_quant_kernel(const bf16* __restrict__ act, uint32_t* __restrict__ act_amax,
                                                        const int32_t* __restrict__ offsets, int E, int64_t R, int h,
                                                        uint8_t* __restrict__ aq, float* __restrict__ ascale) {
  const int lane = threadIdx.x & 31;
  const int64_t r = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (r >= R || r >= offsets[E]) return;  // rows past the last expert tile were never written
  const float amax = __uint_as_float(act_amax[r]);
  const float inv = amax > 0.f ? 448.0f / amax : 0.f;
  const uint4* src = reinterpret_cast<const uint4*>(act + r * h);
  for (int v = lane; v < h / 8; v += 32) {
    const uint4 u = src[v];
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
    uint2 o;
    o.x = (uint32_t)e4m3x2(bf16_lo(w[0]) * inv, bf16_hi(w[0]) * inv) |
          ((uint32_t)e4m3x2(bf16_lo(w[1]) * inv, bf16_hi(w[1]) * inv) << 16);
    o.y = (uint32_t)e4m3x2(bf16_lo(w[2]) * inv, bf16_hi(w[2]) * inv) |
          ((uint32_t)e4m3x2(bf16_lo(w[3]) * inv, bf16_hi(w[3]) * inv) << 16);
    reinterpret_cast<uint2*>(aq + r * h)[v] = o;
  }
  __syncwarp();
  if (lane == 0) {
    ascale[r] = amax / 448.0f;
    act_amax[r] = 0u;  // re-armed for the next forward
  }
}
}  // namespace

void launch_perm_quant(const bf16* x, const int32_t* dest, int64_t T, int H, int k, uint8_t* xq, float* xscale,
                       cudaStream_t s) {
  if (T <= 0) return;
  static const bool tok_kernel = getenv("ASYNCEP_QUANT_TOKENS") == nullptr || atoi(getenv("ASYNCEP_QUANT_TOKENS")) != 0;
  const unsigned grid = (unsigned)((T + 7) / 8);
  if (!dest && tok_kernel) quant_tokens_kernel<<<grid, 256, 0, s>>>(x, T, H, xq, xscale);
  else if (dest && H == 4096) perm_quant_reg_kernel<16><<<grid, 256, 0, s>>>(x, dest, T, k, xq, xscale);
  else if (dest && H == 2048) perm_quant_reg_kernel<8><<<grid, 256, 0, s>>>(x, dest, T, k, xq, xscale);
  else perm_quant_kernel<<<grid, 256, 0, s>>>(x, dest, T, H, k, xq, xscale);
}

void launch_act_quant(const bf16* act, uint32_t* act_amax, const int32_t* offsets, int E, int64_t R, int h,
                      uint8_t* aq, float* ascale, cudaStream_t s) {
  if (R <= 0) return;
  act_quant_kernel<<<(unsigned)((R + 7) / 8), 256, 0, s>>>(act, act_amax, offsets, E, R, h, aq, ascale);
}

void launch_perm_hist(const int32_t* ids, int64_t T, int k, int E, int32_t* blk_counts, cudaStream_t s) {
  const int nblk = (int)((T + kPermTokensPerBlock - 1) / kPermTokensPerBlock);
  perm_hist_kernel<<<nblk, 256, sizeof(int32_t) * E, s>>>(ids, T, k, E, nblk, blk_counts);
}

void launch_perm_scan(int32_t* blk_counts, int nblk, int E, int32_t* offsets, int32_t* tile_start,
                      int32_t* counts, unsigned int* done, int32_t* src_tok, cudaStream_t s) {
  perm_scan_kernel<<<E, SCAN_THREADS, 0, s>>>(blk_counts, nblk, E, offsets, tile_start, counts, done, src_tok);
}

void launch_perm_scatter(const bf16* x, const int32_t* ids, const int32_t* blk_base, const int32_t* offsets,
                         int64_t T, int H, int k, int E, int32_t* dest, int32_t* src_tok, bf16* xperm,
                         cudaStream_t s) {
  const int nblk = (int)((T + kPermTokensPerBlock - 1) / kPermTokensPerBlock);
  perm_scatter_kernel<<<nblk, 256, 0, s>>>(x, ids, blk_base, offsets, nblk, T, H, k, E, dest, src_tok, xperm);
}

}  // namespace aep
