// gemm_simt.cu -- CUDA-core grouped expert GEMM (reference / sanitizer path, selected by
// ASYNCEP_FLAG_SIMT_GEMM).  Same math and tile decomposition as the tcgen05 path
// (gemm_tc.cu): m-tiles of kTileM rows of one expert, fixed K order, fp32 accumulate,
//   GEMM1: act = bf16( silu(X_perm W_gate^T) * (X_perm W_up^T) )        (R4, R5)
//   GEMM2: Y_perm = bf16( act W_down^T )
#include "common.cuh"
#include "kernels.cuh"

namespace aep {

namespace {
constexpr int SN = 64;   // output columns per CTA
constexpr int SK = 16;   // K chunk

__device__ __forceinline__ void decode_mtile(int mt, const int32_t* ts, const int32_t* off, const int32_t* cnt,
                                             int E, int& e, int& row0, int& row_end) {
  constexpr int per = kRowAlign / kTileM;  // 128-row tiles per padded row tile
  const int pt = mt / per;
  int lo = 0, hi = E - 1;  // largest e with ts[e] <= pt
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (ts[mid] <= pt) lo = mid; else hi = mid - 1;
  }
  e = lo;
  row0 = mt * kTileM;
  row_end = off[e] + cnt[e];
}

template <bool SWIGLU>
__global__ void __launch_bounds__(256) gemm_simt_kernel(GroupedArgs g, const bf16* __restrict__ A,
                                                        const uint8_t* __restrict__ layer, size_t expert_bytes,
                                                        size_t b_off, int K, int b_row_stride_elems,
                                                        int Nout, bf16* __restrict__ out) {
  __shared__ float As[SK][kTileM];
  __shared__ float Bg[SK][SN];
  __shared__ float Bu[SWIGLU ? SK : 1][SWIGLU ? SN : 1];
  const int tid = threadIdx.x;
  const int tx = tid % 16, ty = tid / 16;
  const int n0 = blockIdx.x * SN;
  const int total = g.tile_start[g.E] * (kRowAlign / kTileM);
  for (int mt = blockIdx.y; mt < total; mt += gridDim.y) {
    int e, row0, row_end;
    decode_mtile(mt, g.tile_start, g.offsets, g.counts, g.E, e, row0, row_end);
    const bf16* W = reinterpret_cast<const bf16*>(layer + (size_t)e * expert_bytes + b_off);
    // B rows for this CTA's output columns
    // packed W_gu row of act column j: 256-row block j/128, 32-row group (j%128)/16, gate at
    // offset j%16 and the matching up row 16 rows later (asyncep.h layout)
    auto gate_row = [](int j) { return (j / 128) * 256 + ((j % 128) / 16) * 32 + (j % 16); };
    float acc[8][4], accu[SWIGLU ? 8 : 1][SWIGLU ? 4 : 1];
#pragma unroll
    for (int a = 0; a < 8; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        acc[a][b] = 0.f;
        if (SWIGLU) accu[a][b] = 0.f;
      }
    for (int k0 = 0; k0 < K; k0 += SK) {
      {
        const int r = tid / 2, kp = (tid % 2) * 8;
        const int row = row0 + r;
        uint4 v = make_uint4(0, 0, 0, 0);
        if (row < row_end) v = *reinterpret_cast<const uint4*>(A + (int64_t)row * K + k0 + kp);
        const uint32_t u[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          As[kp + 2 * q][r] = bf16_lo(u[q]);
          As[kp + 2 * q + 1][r] = bf16_hi(u[q]);
        }
      }
      {
        const int r = tid / 4, kp = (tid % 4) * 4;
        const bool ok = (n0 + r) < Nout;
        uint2 v = make_uint2(0, 0);
        const int64_t rg = SWIGLU ? gate_row(n0 + r) : n0 + r;
        if (ok) v = *reinterpret_cast<const uint2*>(W + rg * b_row_stride_elems + k0 + kp);
        Bg[kp][r] = bf16_lo(v.x);
        Bg[kp + 1][r] = bf16_hi(v.x);
        Bg[kp + 2][r] = bf16_lo(v.y);
        Bg[kp + 3][r] = bf16_hi(v.y);
        if (SWIGLU) {
          uint2 w = make_uint2(0, 0);
          if (ok) w = *reinterpret_cast<const uint2*>(W + (rg + 16) * b_row_stride_elems + k0 + kp);
          Bu[kp][r] = bf16_lo(w.x);
          Bu[kp + 1][r] = bf16_hi(w.x);
          Bu[kp + 2][r] = bf16_lo(w.y);
          Bu[kp + 3][r] = bf16_hi(w.y);
        }
      }
      __syncthreads();
#pragma unroll
      for (int kk = 0; kk < SK; ++kk) {
        float av[8], bv[4];
#pragma unroll
        for (int a = 0; a < 8; ++a) av[a] = As[kk][ty * 8 + a];
#pragma unroll
        for (int b = 0; b < 4; ++b) bv[b] = Bg[kk][tx * 4 + b];
#pragma unroll
        for (int a = 0; a < 8; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b) acc[a][b] = fmaf(av[a], bv[b], acc[a][b]);
        if (SWIGLU) {
#pragma unroll
          for (int b = 0; b < 4; ++b) bv[b] = Bu[kk][tx * 4 + b];
#pragma unroll
          for (int a = 0; a < 8; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b) accu[a][b] = fmaf(av[a], bv[b], accu[a][b]);
        }
      }
      __syncthreads();
    }
#pragma unroll
    for (int a = 0; a < 8; ++a) {
      const int row = row0 + ty * 8 + a;
      if (row >= row_end) continue;
      const int col = n0 + tx * 4;
      if (col >= Nout) continue;
      float o[4];
#pragma unroll
      for (int b = 0; b < 4; ++b) o[b] = SWIGLU ? silu_f(acc[a][b]) * accu[a][b] : acc[a][b];
      uint2 pk;
      pk.x = pack_bf16x2(o[0], o[1]);
      pk.y = pack_bf16x2(o[2], o[3]);
      *reinterpret_cast<uint2*>(out + (int64_t)row * Nout + col) = pk;
    }
  }
}
}  // namespace

void launch_gemm1_simt(const GroupedArgs& g, const bf16* xperm, const uint8_t* layer, size_t expert_bytes,
                       int H, int h, bf16* act, cudaStream_t s) {
  dim3 grid(h / SN, (unsigned)min(g.max_m_tiles * (kRowAlign / kTileM), 4096));
  gemm_simt_kernel<true><<<grid, 256, 0, s>>>(g, xperm, layer, expert_bytes, 0, H, H, h, act);
}

void launch_gemm2_simt(const GroupedArgs& g, const bf16* act, const uint8_t* layer, size_t expert_bytes,
                       int H, int h, bf16* yperm, cudaStream_t s) {
  dim3 grid((H + SN - 1) / SN, (unsigned)min(g.max_m_tiles * (kRowAlign / kTileM), 4096));
  gemm_simt_kernel<false><<<grid, 256, 0, s>>>(g, act, layer, expert_bytes, (size_t)2 * h * H * 2, h, h, H,
                                               yperm);
}

}  // namespace aep
