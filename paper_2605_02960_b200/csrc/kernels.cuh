// kernels.cuh -- internal launcher interface between the C ABI (asyncep.cu) and the
// kernels.  Not part of the public ABI.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace aep {

typedef __nv_bfloat16 bf16;

constexpr int kPermTokensPerBlock = 64;  // permute/dispatch granularity (tokens per CTA)
constexpr int kTileM = 128;              // grouped-GEMM M rows per CTA (UMMA M slice)
constexpr int kRowAlign = 256;           // expert row ranges are padded to this (one CTA-pair tile)
constexpr int kMaxExperts = 256;
constexpr int kMaxTopK = 16;

// Step (1): router GEMM (fp32 logits) + softmax + top-k, CUDA cores.
// x [T,H] bf16, wr [E,H] bf16 -> ids [T,k] int32, w [T,k] fp32.
void launch_router_simt(const bf16* x, const bf16* wr, int64_t T, int H, int E, int k, int norm_topk,
                        int32_t* ids, float* w, cudaStream_t s);

// Step (1) on tensor cores: tcgen05 logits tile (128 tokens x E) + top-k epilogue.
struct RouterTc {
  CUtensorMap map_wr;  // [E, H] bf16 (3-D {H, E, 1}), box {64, E_pad, 1}, SW128 -- per layer
  CUtensorMap map_wr2; // same, box {64, E_pad / 2, 1}: the half each CTA of a pair loads
  int E_pad;           // E rounded up to a multiple of 16 (MMA N)
  bool pair;           // E_pad >= 64 (and a multiple of 32): CTA-pair router, 256 tokens per tile
};
bool make_router_wmap(RouterTc& rt, const bf16* wr, int H, int E);
// x map is built per call (x is the caller's buffer): [T, H] bf16, box {64, 128}
bool launch_router_tc(const RouterTc& rt, const bf16* x, int64_t T, int H, int E, int k, int norm_topk,
                      int32_t* ids, float* w, int num_sms, cudaStream_t s, int* sched = nullptr);

// Step (2): permute / dispatch.
void launch_perm_hist(const int32_t* ids, int64_t T, int k, int E, int32_t* blk_counts, cudaStream_t s);
// blk_counts is [E][nblk]; `done` is a zero-initialised device counter (re-armed by the kernel).
void launch_perm_scan(int32_t* blk_counts, int nblk, int E, int32_t* offsets, int32_t* tile_start,
                      int32_t* counts, unsigned int* done, int32_t* src_tok, cudaStream_t s);
// xperm == nullptr: ranks / dest / src_tok only (the GEMM gathers the rows itself)
void launch_perm_scatter(const bf16* x, const int32_t* ids, const int32_t* blk_base, const int32_t* offsets,
                         int64_t T, int H, int k, int E, int32_t* dest, int32_t* src_tok, bf16* xperm,
                         cudaStream_t s);

// FP8 (R6): per-token e4m3 quantisation of x into its k permuted rows (after the scatter
// computed dest; dest == nullptr: into token row t of a token-major x_q, for the fused
// dispatch), and per-row quantisation of the GEMM1 intermediate.
void launch_perm_quant(const bf16* x, const int32_t* dest, int64_t T, int H, int k, uint8_t* xq, float* xscale,
                       cudaStream_t s);
void launch_act_quant(const bf16* act, uint32_t* act_amax, const int32_t* offsets, int E, int64_t R, int h,
                      uint8_t* aq, float* ascale, cudaStream_t s);

// Step (3): grouped expert GEMM.  Weights come from a packed layer (see asyncep.h):
// per expert blob of expert_bytes; W_gu at blob offset 0 ([2h, H]), W_down at 2h*H*2.
// Expert e's rows of X_perm / act / Y_perm are [offsets[e], offsets[e] + counts[e]);
// offsets are padded to kRowAlign multiples (offsets[e] = kRowAlign * tile_start[e]) so
// every GEMM row tile belongs to exactly one expert.
struct GroupedArgs {
  const int32_t* offsets;    // [E+1] padded row offsets
  const int32_t* tile_start; // [E+1] prefix of ceil(n_e / kRowAlign)
  const int32_t* counts;     // [E] rows per expert
  int E;
  int max_m_tiles;           // host upper bound on tile_start[E] (row tiles of kRowAlign)
  int* sched = nullptr;      // [4] dynamic tile counters, zeroed before each forward:
                             // [0] router, [1] GEMM1, [2] GEMM2, [3] MX GEMM2's 224-wide tiles
                             // (nullptr: static schedule)
  int group_mod = 0;         // > 0: group g uses expert g % group_mod of the weight blob
  int swap_max = 0;          // > 0: an expert's last row tile with <= swap_max rows runs swap-AB
                             // (weights as M = 256, its tokens as N = rows rounded up to 16): GEMM1
  int swap_max2 = 0;         // the same for GEMM2
};
// rows of the permuted buffers for T tokens: T*k + E*(kRowAlign-1), rounded up to kRowAlign
inline int64_t perm_rows(int64_t T, int k, int E) {
  return ((T * k + (int64_t)E * (kRowAlign - 1)) + kRowAlign - 1) / kRowAlign * kRowAlign;
}
// CUDA-core reference path (debug / sanitizer): SwiGLU GEMM1 and plain GEMM2.
void launch_gemm1_simt(const GroupedArgs& g, const bf16* xperm, const uint8_t* layer, size_t expert_bytes,
                       int H, int h, bf16* act, cudaStream_t s);
void launch_gemm2_simt(const GroupedArgs& g, const bf16* act, const uint8_t* layer, size_t expert_bytes,
                       int H, int h, bf16* yperm, cudaStream_t s);

// tcgen05 path.  One set of TMA maps per weight source (resident layer or slot).
struct GemmMaps {
  CUtensorMap wgu;   // 3D {H, 2h, E}, box {128 B, 256/NCTA rows, 1}
  CUtensorMap wd;    // 3D {h, H, E},  box {128 B, BN2/NCTA rows, 1}
  bool fp8 = false;
};
// Gathered layers: experts [lo, hi) (this rank's own shard) are read by the GEMMs straight from
// the rank's resident shard (maps over its hi - lo experts), so the copy transports never copy
// the own shard into the slot.
struct OwnShard {
  const GemmMaps* maps = nullptr;
  const uint8_t* base = nullptr;  // own shard base (FP8 scales)
  int lo = 0, hi = 0;
};
// FP8 experts (R6): where the GEMMs find their scales.
struct F8Args {
  const float* x_scale;    // [R] per permuted row (per token), from the permute quantisation
  const float* act_scale;  // [R] per row of the intermediate, from launch_act_quant
  uint32_t* act_amax;      // [R] per-row max |act| accumulated by the GEMM1 epilogue
  const uint8_t* layer;    // packed FP8 layer (E blobs)
  size_t expert_bytes;
  size_t sgu_off, sd_off;  // byte offsets of s_gu [2h] / s_down [H] inside a blob
  bool mx = false;         // MX intermediate (R6b): GEMM1 writes e4m3 act + E8M0 scales (act_sf),
  uint32_t* act_sf = nullptr;  // GEMM2 runs block-scaled; act_scale / act_amax unused
};
struct ActMaps {
  CUtensorMap xq;        // FP8: 2D {H, R_max} e4m3, box {128, 128}  (GEMM1 A)
  CUtensorMap aq;        // FP8: 2D {h, R_max} e4m3, box {128, 128}  (GEMM2 A)
  CUtensorMap xperm;     // 2D {H, R_max}, box {64, 128}  (GEMM1 A)
  CUtensorMap act;       // 2D {h, R_max}, box {64, 128}  (GEMM2 A)
  CUtensorMap act_out;   // 2D {h, R_max}, box {64, 32}   (GEMM1 epilogue TMA store)
  CUtensorMap yperm_out; // 2D {H, R_max}, box {64, 32}   (GEMM2 epilogue TMA store)
  CUtensorMap aq_out;    // MX: 2D {h, R_max} e4m3, box {128, 32} (GEMM1 epilogue TMA store)
  CUtensorMap sfa;       // MX: the intermediate's scale chunks, 2D u32 {128, R_max/128 * h/128}, box {128, 1}
  int bn2;               // GEMM2 N tile
  bool mx = false;       // aq_out / sfa are valid
};
bool make_weight_maps(GemmMaps& m, const void* layer, size_t expert_bytes, int E, int H, int h, int bn2, bool fp8);
// xq / aq: FP8 operand buffers (nullable when the experts are BF16)
// asf (nullable): the MX scale chunks ((R_max / 128) * (h / 128) chunks of 512 B): MX maps too
bool make_act_maps(ActMaps& m, const bf16* xperm, const bf16* act, int64_t R_max, int H, int h, const uint8_t* xq,
                   const uint8_t* aq, const uint32_t* asf = nullptr);
int gemm2_bn(int H);
// x_gather != nullptr: A rows are gathered from the token-major x [T, H] (bf16, or the e4m3
// x_q with f8) through src_tok by cp.async warps inside the GEMM, i.e. the dispatch is fused
// into the GEMM and X_perm is never written.
bool launch_gemm1_tc(const GroupedArgs& g, const ActMaps& am, const GemmMaps& wm, int H, int h, bf16* act,
                     const void* x_gather, int64_t T, const int32_t* src_tok, int num_sms, cudaStream_t s,
                     const F8Args* f8 = nullptr, const OwnShard* own = nullptr);
void launch_gemm2_tc(const GroupedArgs& g, const ActMaps& am, const GemmMaps& wm, int H, int h, bf16* yperm,
                     int num_sms, cudaStream_t s, const F8Args* f8 = nullptr, const OwnShard* own = nullptr);

// Step (4): weighted combine (+ residual).
void launch_combine(const bf16* yperm, const int32_t* dest, const float* w, const bf16* residual, bf16* y,
                    int64_t T, int H, int k, cudaStream_t s);

// Weight packing (natural layout -> packed expert blobs), BF16 and FP8 (codes + scales).
void launch_pack_bf16(const bf16* gate, const bf16* up, const bf16* down, int count, int H, int h,
                      size_t expert_bytes, uint8_t* out, cudaStream_t s);
void launch_pack_fp8(const uint8_t* gate, const uint8_t* up, const uint8_t* down, const float* gs, const float* us,
                     const float* ds, int count, int H, int h, size_t expert_bytes, uint8_t* out, cudaStream_t s);

// One thread spinning on %globaltimer for `ns` nanoseconds (link-bandwidth emulation).
// co-resident SM copy (gather transport); bytes % 16 == 0, 16-B aligned pointers
// min_ns > 0: the copy takes at least min_ns (1-GPU link emulation, overlapping copy and link time)
void launch_gather_copy(void* dst, const void* src, size_t bytes, int ctas, cudaStream_t s, uint64_t min_ns = 0);
void launch_spin_ns(uint64_t ns, cudaStream_t s);

// ---- NEXT-3 attention layer (attn.cu) ----
void launch_rmsnorm(const bf16* x, const bf16* w, int64_t rows, int n, float eps, bf16* out, cudaStream_t s);
void launch_residual_rmsnorm(const bf16* x, const bf16* a, const bf16* w, int64_t rows, int n, float eps, bf16* xo,
                             bf16* xn, cudaStream_t s);
void launch_qk_rope(const bf16* qkv, int64_t T, int Hq, int Hkv, const int32_t* cu, int B, const bf16* w_qn,
                    const bf16* w_kn, float eps, float theta, bf16* q, bf16* k, cudaStream_t s);
// vcu [B+1] (output): per-prompt V^T column offsets, each prompt padded to 8 columns
void launch_v_transpose(const bf16* qkv, int64_t T, int Hq, int Hkv, const int32_t* cu, int B, int32_t* vcu,
                        int64_t ldv, bf16* vt, cudaStream_t s);
// sched: one int of caller-owned device memory (zeroed here, on s) for the dynamic item scheduler
bool launch_flash_attn(const bf16* q, const bf16* k, const bf16* vt, int64_t ldv, const int32_t* cu,
                       const int32_t* vcu, int B, int64_t T, int Hq, int Hkv, bf16* o, int* sched,
                       cudaStream_t s);
// dense out[M, N] = A[M, K] . W[N, K]^T on the tcgen05 GEMM (CTA pairs, N % 256 == 0,
// K % 64 == 0); sched: a zeroed int for the dynamic tile scheduler (nullable)
bool launch_dense_gemm_tc(const bf16* A, int64_t M, int K, const bf16* W, int N, bf16* out, int* sched, int num_sms,
                          cudaStream_t s);

// Driver entry point for cuTensorMapEncodeTiled (resolved once through the runtime).
bool encode_tmap(CUtensorMap* map, CUtensorMapDataType dtype, int rank, const void* base, const uint64_t* dims,
                 const uint64_t* strides_bytes /* rank-1 entries */, const uint32_t* box, CUtensorMapSwizzle sw);

}  // namespace aep
