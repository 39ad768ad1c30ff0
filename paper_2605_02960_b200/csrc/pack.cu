// pack.cu -- natural-layout expert weights -> packed expert blobs (layout in asyncep.h):
//   W_gu [2h, H]: 256-row blocks b of 8 groups g of 32 rows: rows [256b + 32g, 256b + 32g + 16)
//                 = gate rows j = 128b + 16g + [0, 16), the next 16 rows = the matching up rows;
//   W_down [H, h] as given.   One CTA per (expert, packed row); 16-B vector copies.
#include "common.cuh"
#include "kernels.cuh"

namespace aep {

namespace {
// Packed W_gu row r -> (gate?, natural row): b = r / 256, q = r % 256, g = q / 32, w = q % 32.
__device__ __forceinline__ int gu_src_row(int r, bool& is_gate) {
  const int b = r / 256, q = r % 256, g = q / 32, w = q % 32;
  is_gate = w < 16;
  return b * 128 + g * 16 + (w & 15);
}
__global__ void pack_bf16_kernel(const bf16* __restrict__ gate, const bf16* __restrict__ up,
                                 const bf16* __restrict__ down, int H, int h, size_t expert_bytes,
                                 uint8_t* __restrict__ out) {
  const int e = blockIdx.y;
  const int r = blockIdx.x;  // 0 .. 2h + H - 1
  uint8_t* blob = out + (size_t)e * expert_bytes;
  const uint4* src;
  uint4* dst;
  int nv;
  if (r < 2 * h) {
    bool is_gate;
    const int srow = gu_src_row(r, is_gate);
    const bf16* m = is_gate ? gate : up;
    src = reinterpret_cast<const uint4*>(m + ((size_t)e * h + srow) * H);
    dst = reinterpret_cast<uint4*>(blob + (size_t)r * H * 2);
    nv = H / 8;
  } else {
    const int rr = r - 2 * h;
    src = reinterpret_cast<const uint4*>(down + ((size_t)e * H + rr) * h);
    dst = reinterpret_cast<uint4*>(blob + (size_t)2 * h * H * 2 + (size_t)rr * h * 2);
    nv = h / 8;
  }
  for (int v = threadIdx.x; v < nv; v += blockDim.x) dst[v] = src[v];
}
// FP8 blob: [W_gu codes 2h x H | W_down codes H x h | s_gu 2h fp32 | s_down H fp32], W_gu rows
// (and their scales) interleaved exactly like the BF16 layout.
__global__ void pack_fp8_kernel(const uint8_t* __restrict__ gate, const uint8_t* __restrict__ up,
                                const uint8_t* __restrict__ down, const float* __restrict__ gs,
                                const float* __restrict__ us, const float* __restrict__ ds, int H, int h,
                                size_t expert_bytes, uint8_t* __restrict__ out) {
  const int e = blockIdx.y;
  const int r = blockIdx.x;  // 0 .. 2h + H - 1
  uint8_t* blob = out + (size_t)e * expert_bytes;
  float* sgu = reinterpret_cast<float*>(blob + (size_t)3 * H * h);
  float* sd = sgu + 2 * h;
  const uint4* src;
  uint4* dst;
  int nv;
  if (r < 2 * h) {
    bool is_gate;
    const int srow = gu_src_row(r, is_gate);
    src = reinterpret_cast<const uint4*>((is_gate ? gate : up) + ((size_t)e * h + srow) * H);
    dst = reinterpret_cast<uint4*>(blob + (size_t)r * H);
    nv = H / 16;
    if (threadIdx.x == 0) sgu[r] = (is_gate ? gs : us)[(size_t)e * h + srow];
  } else {
    const int rr = r - 2 * h;
    src = reinterpret_cast<const uint4*>(down + ((size_t)e * H + rr) * h);
    dst = reinterpret_cast<uint4*>(blob + (size_t)2 * h * H + (size_t)rr * h);
    nv = h / 16;
    if (threadIdx.x == 0) sd[rr] = ds[(size_t)e * H + rr];
  }
  for (int v = threadIdx.x; v < nv; v += blockDim.x) dst[v] = src[v];
}
}  // namespace

void launch_pack_fp8(const uint8_t* gate, const uint8_t* up, const uint8_t* down, const float* gs, const float* us,
                     const float* ds, int count, int H, int h, size_t expert_bytes, uint8_t* out, cudaStream_t s) {
  if (count <= 0) return;
  dim3 grid(2 * h + H, count);
  pack_fp8_kernel<<<grid, 128, 0, s>>>(gate, up, down, gs, us, ds, H, h, expert_bytes, out);
}

void launch_pack_bf16(const bf16* gate, const bf16* up, const bf16* down, int count, int H, int h,
                      size_t expert_bytes, uint8_t* out, cudaStream_t s) {
  if (count <= 0) return;
  dim3 grid(2 * h + H, count);
  pack_bf16_kernel<<<grid, 128, 0, s>>>(gate, up, down, H, h, expert_bytes, out);
}

}  // namespace aep
