// gemm_tc.cu -- step (3): the grouped expert GEMM on 5th-gen tensor cores (sm_100a),
// and the router logits GEMM of step (1) with its top-k fused into the epilogue.
//
//   GEMM1 (per expert e, rows R_e of X_perm):  G = X_perm[R_e] . W_gu[e]^T  -> SwiGLU epilogue
//          act = bf16( silu(G_gate) * G_up )                     (R4, R5)
//   GEMM2:  Y_perm[R_e] = bf16( act[R_e] . W_down[e]^T )
//   router: logits = x . W_r^T (fp32, R3) -> top-k -> weights    (R1, R2)
//
// Persistent, warp-specialised kernel, 256 threads per CTA, one CTA per SM:
//   warp 0      TMA producer: A tile {64 x 128 rows} (2-D map over X_perm / act / x) and
//               B tile {64 x BN/NCTA rows x 1 expert} (3-D map over the packed layer) into
//               an S-stage shared-memory ring (128-B swizzle); mbarrier full/empty pairs.
//   warp 1      MMA issuer (leader CTA only): one thread issues tcgen05.mma kind::f16
//               (M = 128*NCTA, N = BN, K = 16) x 4 per stage into a TMEM accumulator;
//               tcgen05.commit frees the smem stage / publishes the accumulator.
//   warp 2      TMEM allocator (512 columns = 2 accumulators x 256).
//   warps 4-7   epilogue: tcgen05.ld 32x32b (thread = accumulator row) -> SwiGLU / plain
//               bf16 pack -> swizzled smem staging -> TMA bulk tensor store; or top-k.
// NCTA = 2 (the grouped GEMMs): a CTA pair (cluster of 2) runs cta_group::2 MMAs with
// M = 256: each CTA loads its own 128 rows of A and HALF of the BN rows of B, so every
// SM reads 8 KB of operands per 256x256x16 MMA instead of 12 KB per 128x256x16 (the
// 1-CTA kernel was shared-memory-read bound, ncu: 90 % sm__mem_tensor).  For GEMM1 the
// CTA0 half of a 256-row W_gu tile is exactly the gate rows and the CTA1 half the
// matching up rows, so each CTA's accumulator holds [gate | up] and SwiGLU stays local.
// Tiles: t -> (row tile, n-tile); row tile -> expert via the device-side prefix
// tile_start (permute scan; expert rows padded to 256), no host sync.  Every output tile
// is produced by one CTA (pair) in a fixed K order: bitwise deterministic results that do
// not depend on the grid size.
#include <cstdio>
#include <cstdlib>
#include <mutex>

#include "common.cuh"
#include "kernels.cuh"

namespace aep {

namespace {
int env_int(const char* name, int dflt) {
  const char* v = getenv(name);
  return (v && *v) ? atoi(v) : dflt;
}
constexpr int BM = kTileM;          // 128 rows per CTA (per-CTA UMMA M slice)
constexpr int BK = 64;              // 64 bf16 = 128 B = one swizzle row
constexpr int A_BYTES = BM * BK * 2;           // 16 KB
constexpr int STG_BYTES = 32 * 128;            // per epilogue warp: 32 rows x 64 bf16 (SW128)
constexpr int SCL_BYTES = 256 * 4;             // per epilogue warp: the tile's 256 FP8 weight scales
constexpr int TMEM_COLS = 512;
constexpr int RING = 8;
  // tile ids in flight between the scheduler and the consumers

enum { EPI_PLAIN = 0, EPI_SWIGLU = 1, EPI_ROUTER = 2, EPI_ROUTER16 = 3 };  // router: top-k <= 8 / <= 16

#ifndef GEMM_WAITPROF
#define GEMM_WAITPROF 0  // 1: the MMA / gather / producer threads printf their barrier-wait cycles (A/B only)
#endif
#if GEMM_WAITPROF
#define WP_DECL(n) long long n = 0;
#define WP_WAIT(acc, stmt) { const long long c_ = clock64(); stmt; acc += clock64() - c_; }
#else
#define WP_DECL(n)
#define WP_WAIT(acc, stmt) stmt;
#endif
// Without the fused gather, warp 3 issues the B (weight) loads and warp 0 the A loads (and runs the
// scheduler): GEMM2's single producer spent ~40 % of its time issuing TMA loads.
#define PROD2 1
// Shared memory plan per (CTA group, epilogue mode): S-stage operand ring, one 32-row staging
// buffer and one 256-scale buffer per epilogue warp, barriers, the tile_start prefix.
// (Measured and dropped, S6: double-buffered staging, 8 epilogue warps.)
// MX block-scaled GEMM2 (MXIN): per stage one 512-B chunk of A scale factors (E8M0, the
// tcgen05.cp 32x128b.warpx4 layout), plus one constant 512-B chunk of B scale factors (1.0).
template <int NCTA, int MODE, bool MXIN = false>
struct Cfg {
  static constexpr int B_BYTES_MAX = (256 / NCTA) * BK * 2;  // B rows per CTA <= 256 / NCTA
  static constexpr int STAGES = NCTA == 2 ? 6 : 4;
  static constexpr int EW = 4;                // epilogue warps (one per TMEM lane quadrant)
  static constexpr int NTHR = 128 + 32 * EW;  // warps 0-3 roles, then EW epilogue warps
  static constexpr int NSTG = 1;
  static constexpr int NSCL = SCL_BYTES;
  static constexpr int SF_BYTES = MXIN ? (STAGES * 512 + 512 + 1023) / 1024 * 1024 : 0;
  static constexpr size_t SMEM = 1024 + (size_t)STAGES * (A_BYTES + B_BYTES_MAX) + SF_BYTES + EW * NSTG * STG_BYTES +
                                 EW * NSCL + 512 + (2 * kMaxExperts + 1) * sizeof(int32_t);
  static_assert(SMEM <= 232448, "shared memory budget");
};
// MX GEMM2 TMEM columns: accumulator 0 [0, 256) for 256-wide N tiles, accumulator 1 [256, 480) for
// 224-wide ones, the B scale factors [480, 488), four A scale-factor slots [488, 504).
constexpr int kMxSfbCol = 480;
constexpr int kMxSfaCol = 488;
constexpr int kMxWide = 256, kMxNarrow = 224, kMxPeriod = kMxWide + kMxNarrow;

struct TcArgs {
  const int32_t* tile_start;  // grouped mode: [E+1] prefix of row tiles (rows padded to 128*NCTA)
  int E;                      // groups (experts); router mode: number of experts (columns)
  int dense_rows;             // > 0: dense mode, one group of dense_rows rows (router)
  int K;        // contraction length (multiple of 64)
  int BN;       // N tile (multiple of 16*NCTA, <= 256); each CTA loads BN/NCTA rows of B
  int n_tiles;  // N tiles per row tile
  int n_out;    // output columns
  int ts_scale; // row tiles (of 128*NCTA rows) per tile_start unit (kRowAlign rows)
  int raster;   // 0: row-tile-major order; G > 0: groups of G row tiles walked row-first
  int pol_a, pol_b;  // L2 policy of the A / B loads: 0 normal, 1 evict_last, 2 evict_first, 3 none (A)
  int pol_gather;    // L2 policy of the fused dispatch's cp.async row gathers: 0 normal, 1 evict_last, 2 evict_first
  // FP8 (kind::f8f6f4) scales: dequantised D[r][c] = acc * a_scale[r] * b_scale(e)[B row of c]
  const float* a_scale;
  const uint8_t* b_scale_base;  // layer base + offset of the scale block inside an expert blob
  size_t expert_bytes;
  uint32_t* amax_out;           // GEMM1 FP8: per-row max |act| (fp32 bits, atomicMax)
  int* sched;                   // dynamic tile counter (zeroed before the launch)
  int n_tiles2;                 // MX GEMM2: 224-wide N tiles per row tile (n_tiles: 256-wide ones)
  uint32_t* mx_sf_out;          // MX GEMM1: E8M0 scale chunks of the e4m3 intermediate
  int mx_nkb;                   // MX: 128-column k-blocks of the intermediate (h / 128)
  int mx_sf_warp;               // MXIN: the warp issuing the scale-chunk loads (0: with A, 2: its own)
  int group_mod;                // > 0: B expert = group % group_mod (EP contrast: groups are
                                // (source rank, local expert) pairs over a shard of group_mod experts)
  // fused dispatch: non-null gather_rows = A rows are gathered by warps 2-3 (cp.async) from the
  // token-major matrix gather_src (gather_ld bytes per token) at token gather_rows[permuted row];
  // the FP8 a_scale is then indexed by token
  const int32_t* gather_rows;
  const uint8_t* gather_src;
  int64_t gather_ld;
  // experts [own_lo, own_hi) are read through map_b2 (this rank's own shard, local index e - own_lo)
  int own_lo, own_hi;
  const uint8_t* b_scale_base_own;
  // router epilogue
  int top_k, norm_topk;
  int32_t* ids;
  float* w;
  // swap-AB tail tiles (grouped CTA-pair GEMMs): an expert's last row tile holding r <= swap_max
  // rows runs with the weights as the M = 256 operand and its r tokens (rounded up to 16) as N, so
  // the MMA does r/256 of a full tile's work instead of computing padding rows.  The epilogue
  // writes out_ptr (row stride n_out) directly, transposing through the staging buffer.
  const int32_t* counts;
  int swap_max;
  bf16* out_ptr;
};

// linear tile index -> (row tile, n tile)
__device__ __forceinline__ void decode_tile(int t, int n_tiles, int total_rt, int raster, int& mt, int& nt) {
  if (raster <= 0) {
    mt = t / n_tiles;
    nt = t - mt * n_tiles;
  } else {
    const int gsz = raster * n_tiles;
    const int g = t / gsz, r = t - g * gsz;
    const int rows = min(raster, total_rt - g * raster);
    mt = g * raster + r % rows;
    nt = r / rows;
  }
}

__device__ __forceinline__ int find_expert(const int32_t* ts, int E, int mt) {
  int lo = 0, hi = E - 1;  // largest e with ts[e] <= mt (skips empty experts)
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (ts[mid] <= mt) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// Swap-AB classification of row tile mt of expert e (s_ts: row-tile prefix, s_cnt: rows per
// expert, TM rows per tile): the expert's last tile with r <= swap_max rows -> ntok = r rounded up
// to 16 (the MMA's N), else 0 (a normal tile).
__device__ __forceinline__ int swap_ntok(const int32_t* s_ts, const int32_t* s_cnt, int e, int mt, int TM,
                                         int swap_max) {
  if (swap_max <= 0 || mt != s_ts[e + 1] - 1) return 0;
  const int r = s_cnt[e] - (mt - s_ts[e]) * TM;
  return (r > 0 && r <= swap_max) ? (r + 15) & ~15 : 0;
}

// MX GEMM2 tile geometry.  The output columns are covered by alternating 256- and 224-wide N
// tiles (period 480; the last ones clipped to n_out), so the two accumulators (256 + 224 TMEM
// columns) leave room for the scale factors.  Tile ids [0, totalW) are the 256-wide tiles
// (n_wide per row tile), [totalW, total) the 224-wide ones (n_narrow per row tile); each width
// class always uses its own accumulator (buf).
struct TileGeo {
  int mt, col0, width, buf;
};
__device__ __forceinline__ TileGeo tile_geo_mx(int t, int totalW, int n_wide, int n_narrow, int n_out) {
  TileGeo g;
  if (t < totalW) {
    g.mt = t / n_wide;
    g.col0 = (t - g.mt * n_wide) * kMxPeriod;
    g.width = min(kMxWide, n_out - g.col0);
    g.buf = 0;
  } else {
    const int u = t - totalW;
    g.mt = u / n_narrow;
    g.col0 = (u - g.mt * n_narrow) * kMxPeriod + kMxWide;
    g.width = min(kMxNarrow, n_out - g.col0);
    g.buf = 1;
  }
  return g;
}

// Router epilogue, one thread = one token row of the logits tile (E <= 256 fp32 columns
// in TMEM): a running top-KMAX list in registers (KMAX >= k), fed 8 columns at a time.
// Logits arrive in increasing expert id, so a strict '>' keeps equal logits in id order
// (ties -> lower expert id, R2); most columns fail the one-compare rejection test against
// the current KMAX-th value and never touch the insertion network (compact code: the
// fully unrolled version thrashed the instruction cache).  Weights: softmax over the k
// selected logits (norm_topk, R1) or the full-E softmax entry (second TMEM pass).
template <int KMAX>
__device__ __forceinline__ void router_epilogue(uint32_t tb, int E, int k, int norm_topk, bool valid,
                                                int32_t* ids, float* w) {
  float tv[KMAX];
  int ti[KMAX];
#pragma unroll
  for (int j = 0; j < KMAX; ++j) { tv[j] = -INFINITY; ti[j] = 0; }
#pragma unroll 1
  for (int c0 = 0; c0 < E; c0 += 8) {
    uint32_t r[8];
    tmem_ld8(tb + c0, r);
    tmem_ld_wait();
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      float v = __uint_as_float(r[i]);
      if (c0 + i < E && v > tv[KMAX - 1]) {
        int e = c0 + i;
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
#pragma unroll 1
    for (int c0 = 0; c0 < E; c0 += 8) {
      uint32_t r[8];
      tmem_ld8(tb + c0, r);
      tmem_ld_wait();
#pragma unroll
      for (int i = 0; i < 8; ++i)
        if (c0 + i < E) denom += expf(__uint_as_float(r[i]) - ref);
    }
  }
  if (valid) {
#pragma unroll
    for (int j = 0; j < KMAX; ++j)
      if (j < k) {
        ids[j] = ti[j];
        w[j] = expf(tv[j] - ref) / denom;
      }
  }
}

// Epilogue store of 64 bf16 columns (32 packed words) of this thread's row through the
// warp's 32 x 128 B staging buffer (128-B swizzle: 16-B chunk j of row r at chunk
// j ^ (r & 7), conflict-free) and one TMA bulk tensor store of the {64 x 32} box.
// With NSTG = 2 buffers (chunk parity picks one) only the store before last must have been read.
#if GEMM_WAITPROF
#define g_wp_store wp_store_acc
#else
#define g_wp_store 0
#endif
template <int NSTG>
__device__ __forceinline__ void stage_and_store(const uint32_t (&o)[32], uint8_t* stg, int lane,
                                                const CUtensorMap* map_out, int col0, int row0
#if GEMM_WAITPROF
                                                , long long& wp_store_acc
#endif
                                                ) {
  if (lane == 0) {  // the store that last used this buffer has finished reading it
#if GEMM_WAITPROF
    const long long c_ = clock64();
#endif
    if (NSTG == 2) bulk_wait_read1();
    else bulk_wait_read0();
#if GEMM_WAITPROF
    wp_store_acc += clock64() - c_;
#endif
  }
  __syncwarp();
  const uint32_t base = smem_u32(stg) + lane * 128;
#pragma unroll
  for (int j = 0; j < 8; ++j)
    st_shared_v4(base + ((j ^ (lane & 7)) << 4), o[4 * j], o[4 * j + 1], o[4 * j + 2], o[4 * j + 3]);
  fence_proxy_async_smem();
  __syncwarp();
  if (lane == 0) {
    tma_store_2d(map_out, stg, col0, row0);
    bulk_commit();
  }
}

// MX quantisation of one block of 32 intermediate values (reading R6b), 16 packed bf16 words in
// column order -> 8 words of e4m3 codes (q), returns the E8M0 scale byte.  e is the smallest
// integer with amax <= 448 * 2^e: amax = 1.m * 2^E gives e = E - 8, plus 1 when 1.m > 1.75
// (448 = 1.75 * 2^8); the clamp at -127 is the E8M0 range (finite bf16 values give e <= 120).
// The codes are RNE(v * 2^-e) (an exact power-of-two product), never saturated.
__device__ __forceinline__ uint32_t mx_block(const uint32_t* o, uint32_t* q) {
  uint32_t m = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) m = __vmaxu2(m, o[i] & 0x7fff7fffu);
  const uint32_t a = max(m & 0xffffu, m >> 16) << 16;  // fp32 bits of the block's max |v|
  const int e = max((int)(a >> 23) - 135 + ((a & 0x7fffffu) > 0x600000u ? 1 : 0), -127);
  const float inv = __uint_as_float((uint32_t)(127 - e) << 23);  // 2^-e
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    float x0, x1, x2, x3;
    mul2(x0, x1, bf16_lo(o[2 * i]), bf16_hi(o[2 * i]), inv, inv);
    mul2(x2, x3, bf16_lo(o[2 * i + 1]), bf16_hi(o[2 * i + 1]), inv, inv);
    q[i] = (uint32_t)e4m3x2(x0, x1) | ((uint32_t)e4m3x2(x2, x3) << 16);
  }
  return (uint32_t)(e + 127);
}

// Dynamic tile scheduler.  The leader CTA's producer thread takes the next tile id from a
// global atomic counter (so the tiles in flight on the whole GPU always form one contiguous
// window: no drift between persistent CTAs, which kept L2 reuse of the A row-tiles and the
// expert weights poor with a static round-robin assignment) and publishes it through a
// RING-deep smem ring: locally with an mbarrier arrive, to the peer CTA with st.async
// (complete_tx on the peer's ring barrier).  Consumers release a ring slot on the leader's
// sempty barrier.  p.sched == nullptr falls back to the static assignment unit + seq*nunits.
struct TileRing {
  uint64_t* sfull;
  uint64_t* sempty;
  int32_t* ring;
};

// scheduler side (leader producer thread): fetch + publish the id of tile number seq
// MX GEMM2 (MxSched::nw > 0): the counter hands out units (row tile, j) in row-tile-major
// order; a unit is the 256-wide tile j followed by its 224-wide sibling (when j < nn), published
// back to back, so a pair's consecutive tiles alternate accumulators (except after a unit without
// a sibling) and the wide and narrow tiles of a row tile are read at the same time (L2).
struct MxSched {
  int nw = 0, nn = 0, totalW = 0, total = 0;
  int pending = -1;  // the narrow sibling still to publish
  int units = 0;     // units taken (static schedule)
};
template <int NCTA>
__device__ __forceinline__ int sched_publish(const TileRing& r, int* sched, int seq, int unit, int nunits,
                                             MxSched* mx = nullptr) {
  const int slot = seq % RING;
  const uint32_t ph = (uint32_t)(seq / RING) & 1u;
  mbar_wait(&r.sempty[slot], ph ^ 1u);
  int t;
  if (mx && mx->pending >= 0) {
    t = mx->pending;
    mx->pending = -1;
  } else {
    if (mx) {  // unit u = the wide tile of the same id (ids run row-tile-major in both classes)
      t = sched ? atomicAdd(sched, 1) : unit + (mx->units++) * nunits;
      const int mt = t / mx->nw, j = t - mt * mx->nw;
      if (t >= mx->totalW) t = mx->total;
      else if (j < mx->nn) mx->pending = mx->totalW + mt * mx->nn + j;
    } else {
      t = sched ? atomicAdd(sched, 1) : unit + seq * nunits;
    }
  }
  r.ring[slot] = t;
  mbar_arrive(&r.sfull[slot]);
  if (NCTA == 2) st_async_u32(&r.ring[slot], &r.sfull[slot], 1, (uint32_t)t);
  return t;
}

// consumer side (one thread): read tile id seq and release the slot to the leader.
// arm = true for the single peer thread that arms the peer ring barrier for the st.async.
template <int NCTA>
__device__ __forceinline__ int sched_consume(const TileRing& r, int seq, bool leader, bool arm) {
  const int slot = seq % RING;
  const uint32_t ph = (uint32_t)(seq / RING) & 1u;
  if (arm) mbar_arrive_expect_tx(&r.sfull[slot], 4);
  mbar_wait(&r.sfull[slot], ph);
  const int t = r.ring[slot];
  if (NCTA == 2 && !leader) mbar_arrive_cluster_relaxed(&r.sempty[slot], 0);
  else mbar_arrive(&r.sempty[slot]);
  return t;
}

// FP8 epilogue: the 256 per-channel weight scales of this tile (contiguous in the blob) are
// copied once per tile into the warp's smem buffer and then read as broadcasts (a per-element
// global load for every thread made the FP8 epilogue, not the MMA, the limiter).
__device__ __forceinline__ const float* stage_scales(float* dst, const float* src, int n, int lane) {
  __syncwarp();
  for (int i = lane * 4; i < n; i += 128) *reinterpret_cast<float4*>(dst + i) = __ldg(reinterpret_cast<const float4*>(src + i));
  __syncwarp();
  return dst;
}

// Register cap: every GEMM CTA leaves >= 4K registers free on its SM, so the gather transport's
// copy CTAs (128 threads x 32 registers) co-reside with it and the next layer's gather makes
// progress during the GEMM (without the cap the FP8 SwiGLU kernel took 250 registers/thread,
// the whole register file, and the gather stalled for its entire duration).
// MX (FP8 experts, MX intermediate, reading R6b): with MODE == EPI_SWIGLU (MXOUT) the GEMM1
// epilogue writes the intermediate as e4m3 with one E8M0 scale per 32 columns (map_out = the
// e4m3 act map, p.mx_sf_out the scale chunks); with MODE == EPI_PLAIN (MXIN) GEMM2 runs
// kind::mxf8f6f4.block_scale MMAs on it (map_sf: the A scale chunks) over 256/224-wide N tiles.
template <int MODE, int NCTA, bool F8, bool MX = false>
__global__ void __launch_bounds__(Cfg<NCTA, MODE>::NTHR, 1) __maxnreg__((Cfg<NCTA, MODE>::NTHR == 256 ? 224 : 168))
    gemm_tc_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                   const __grid_constant__ CUtensorMap map_out, const __grid_constant__ CUtensorMap map_b2,
                   const __grid_constant__ CUtensorMap map_sf, const TcArgs p) {
  constexpr bool MXIN = MX && MODE == EPI_PLAIN && F8 && NCTA == 2;
  constexpr bool MXOUT = MX && MODE == EPI_SWIGLU && F8 && NCTA == 2;
  using C = Cfg<NCTA, MODE, MXIN>;
  constexpr int STAGES = C::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = sA + STAGES * A_BYTES;
  uint8_t* sSF = sB + STAGES * C::B_BYTES_MAX;  // MXIN: STAGES A scale chunks, then the B chunk
  uint8_t* sStg = sSF + C::SF_BYTES;
  float* sScl = reinterpret_cast<float*>(sStg + C::EW * C::NSTG * STG_BYTES);
  uint64_t* full = reinterpret_cast<uint64_t*>(sStg + C::EW * C::NSTG * STG_BYTES + C::EW * C::NSCL);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* sfull = tempty + 2;          // tile-id ring (dynamic scheduler): filled
  uint64_t* sempty = sfull + RING;       //                                    released
  uint64_t* afull = sempty + RING;       // fused dispatch: this CTA's gathered A stage landed
  int32_t* sring = reinterpret_cast<int32_t*>(afull + STAGES);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sring + RING);
  int32_t* s_ts = reinterpret_cast<int32_t*>(reinterpret_cast<uint8_t*>(full) + 512);
  int32_t* s_cnt = s_ts + kMaxExperts + 1;

  const int warp = warp_id(), lane = lane_id();
  const uint32_t rank = NCTA == 2 ? cluster_ctarank() : 0;
  const bool leader = rank == 0;
  const int unit = NCTA == 2 ? (int)cluster_id_x() : (int)blockIdx.x;  // CTA pair (or CTA) index
  const int nunits = NCTA == 2 ? (int)nclusters_x() : (int)gridDim.x;
  constexpr int TM = BM * NCTA;  // rows per tile (per CTA pair)
  const int G = p.dense_rows > 0 ? 1 : p.E;  // number of groups
  if (p.dense_rows > 0) {
    if (threadIdx.x == 0) {
      s_ts[0] = 0;
      s_ts[1] = (p.dense_rows + TM - 1) / TM;
    }
  } else {
    for (int i = threadIdx.x; i <= p.E; i += C::NTHR) s_ts[i] = p.tile_start[i] * p.ts_scale;
    if (p.swap_max > 0)
      for (int i = threadIdx.x; i < p.E; i += C::NTHR) s_cnt[i] = p.counts[i];
  }
  // swap-AB tail tiles: CTA-pair grouped GEMMs with full 256-row weight tiles only
  const int swap_max = (NCTA == 2 && (MODE == EPI_SWIGLU || MODE == EPI_PLAIN) && p.dense_rows <= 0 &&
                        p.BN == 256 && p.group_mod == 0) ? p.swap_max : 0;
  const bool gather = p.gather_rows != nullptr;
  const bool sf_w2 = MXIN && !gather && p.mx_sf_warp == 2;  // warp 2 is a third producer (scales)
  if (warp == 0 && lane == 0) {
    if (!gather) tma_prefetch_desc(&map_a);
    tma_prefetch_desc(&map_b);
    if (p.own_hi > p.own_lo) tma_prefetch_desc(&map_b2);
    if (MODE == EPI_PLAIN || MODE == EPI_SWIGLU) tma_prefetch_desc(&map_out);
    for (int s = 0; s < STAGES; ++s) {
      // leader: own expect_tx arrive + peer producer's arrive (+ peer's gathered-A forward)
      mbar_init(&full[s], (PROD2 && !gather ? 2 : 1) * NCTA + (gather && NCTA == 2 ? 1 : 0) + (sf_w2 ? NCTA : 0));
      mbar_init(&empty[s], 1);
      mbar_init(&afull[s], 64);  // one .noinc cp.async arrival per gather thread
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], C::EW * NCTA);  // one arrive per epilogue warp of each CTA
    }
    for (int r = 0; r < RING; ++r) {
      mbar_init(&sfull[r], 1);
      // consumers of a tile id: leader {MMA thread, 4 epilogue warps} + peer {producer, 4 epilogue
      // warps}; fused dispatch adds the 2 gather warps of each CTA and the peer's forwarder
      mbar_init(&sempty[r], (1 + C::EW) * NCTA + (gather ? 2 * NCTA + (NCTA == 2 ? 1 : 0) : 0) +
                                (PROD2 && !gather ? NCTA : 0) + (sf_w2 ? NCTA : 0));
    }
    fence_barrier_init();
  }
  if (warp == 2) {
    if (NCTA == 2) tmem_alloc2(tmem_slot, TMEM_COLS);
    else tmem_alloc(tmem_slot, TMEM_COLS);
  }
  if (MXIN) {  // B scale factors: E8M0 1.0 (0x7F) for every row and k (the weights keep their
               // per-row fp32 scale, applied in the epilogue)
    for (int i = threadIdx.x; i < 128; i += C::NTHR)
      reinterpret_cast<uint32_t*>(sSF + STAGES * 512)[i] = 0x7F7F7F7Fu;
    fence_proxy_async_smem();
  }
  tc_fence_before();
  if (NCTA == 2) cluster_sync_all(); else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int total_rt = s_ts[G];
  const int totalW = total_rt * p.n_tiles;  // MXIN: the 256-wide tiles come first
  const int total = MXIN ? totalW + total_rt * p.n_tiles2 : totalW;
  constexpr int KB_ELEMS = F8 ? 128 : BK;  // elements per 128-B k-block row
  const int nkb = p.K / KB_ELEMS;
  const int bn_cta = p.BN / NCTA;  // B rows loaded by this CTA
  const TileRing ring{sfull, sempty, sring};

  if (warp == 0 || (PROD2 && !gather && warp == 3) || (sf_w2 && warp == 2)) {
    // Producer warp, lane 0: arms the stage barrier and loads B (and A unless it is gathered).
    // PROD2 without the gather: warp 0 loads A (and runs the scheduler), warp 3 loads B; MXIN:
    // the A scale chunks with A, or from warp 2 (ASYNCEP_MX_SF_WARP=2).
    const bool do_a = !gather && (!PROD2 || warp == 0);
    const bool do_b = !PROD2 || gather || warp == 3;
    const bool do_sf = MXIN && (sf_w2 ? warp == 2 : warp == 0);
    const bool sched_lead = warp == 0;
    if (lane == 0) {
      const uint32_t tx = (uint32_t)NCTA * ((do_a ? (uint32_t)A_BYTES : 0u) + (do_sf ? 512u : 0u) +
                                            (do_b ? (uint32_t)bn_cta * BK * 2 : 0u));
      const uint64_t pol_a = make_policy(p.pol_a), pol_b = make_policy(p.pol_b);
      int stage = 0;
      uint32_t phase = 0;
      WP_DECL(wp_e) WP_DECL(wp_s) WP_DECL(wp_i)
#if GEMM_WAITPROF
      const long long wp_t0 = clock64();
#endif
      // The scheduler publishes one tile ahead: the global atomic that fetches tile seq+1 is in
      // flight while tile seq's loads are issued (on short-K tiles its latency otherwise sat
      // between two tiles' loads), and with the fused gather the gather warps fetch the next
      // tile's row indices while they copy the current tile (in the peer CTA a gather warp is
      // then the consumer that arms the ring slot for the st.async; without the gather the peer
      // producer arms it -- a complete_tx that lands before the arm leaves the phase pending).
      MxSched mxs;
      mxs.nw = p.n_tiles;
      mxs.nn = p.n_tiles2;
      mxs.totalW = totalW;
      mxs.total = total;
      MxSched* const mxp = MXIN ? &mxs : nullptr;
      int t_next = (leader && sched_lead) ? sched_publish<NCTA>(ring, p.sched, 0, unit, nunits, mxp) : 0;
      for (int seq = 0;; ++seq) {
        int t;
        if (!sched_lead) {
          WP_WAIT(wp_s, t = sched_consume<NCTA>(ring, seq, leader, false))
        } else if (leader) {
          t = t_next;
          if (t < total) WP_WAIT(wp_s, t_next = sched_publish<NCTA>(ring, p.sched, seq + 1, unit, nunits, mxp))
        } else {
          WP_WAIT(wp_s, t = sched_consume<NCTA>(ring, seq, false, !gather))
        }
        if (t >= total) break;
        int mt, nt = 0, brow;
        if (MXIN) {
          const TileGeo g = tile_geo_mx(t, totalW, p.n_tiles, p.n_tiles2, p.n_out);
          mt = g.mt;
          brow = g.col0 + (int)rank * (g.width >> 1);  // B box: bn_cta rows (over-fetch on narrow tiles)
        } else {
          decode_tile(t, p.n_tiles, total_rt, p.raster, mt, nt);
          brow = nt * p.BN + (int)rank * bn_cta;
        }
        int e = find_expert(s_ts, G, mt);
        const int ntok = swap_ntok(s_ts, s_cnt, e, mt, TM, swap_max);
        if (p.group_mod > 0) e %= p.group_mod;  // group (source rank, local expert) -> expert
        const bool own_e = e >= p.own_lo && e < p.own_hi;
        const CUtensorMap* mb = own_e ? &map_b2 : &map_b;
        if (own_e) e -= p.own_lo;
        // swap: this CTA's ntok/2 token rows go to the B stage, its 128 weight rows to the A stage
        const int row0 = ntok ? mt * TM + (int)rank * (ntok >> 1) : mt * TM + (int)rank * BM;
        uint8_t* const dA = ntok ? sB : sA;  // token operand
        uint8_t* const dB = ntok ? sA : sB;  // weight operand
        for (int kb = 0; kb < nkb; ++kb) {
          WP_WAIT(wp_e, mbar_wait(&empty[stage], phase ^ 1))
#if GEMM_WAITPROF
          const long long wp_c = clock64();
#endif
          if (NCTA == 2) {
            if (leader) mbar_arrive_expect_tx(&full[stage], tx);
            else mbar_arrive_cluster_relaxed(&full[stage], 0);
            static_assert(A_BYTES == C::B_BYTES_MAX || NCTA == 1, "swap-AB exchanges the A and B stages");
            if (do_a) {
              if (p.pol_a == 3) tma_load_2d_pair(dA + stage * A_BYTES, &map_a, &full[stage], kb * KB_ELEMS, row0);
              else tma_load_2d_pair_hint(dA + stage * A_BYTES, &map_a, &full[stage], kb * KB_ELEMS, row0, pol_a);
            }
            // the k-block's 512-B chunk of this CTA's 128 A rows' scale factors
            if (do_sf) tma_load_2d_pair(sSF + stage * 512, &map_sf, &full[stage], 0, (mt * 2 + (int)rank) * p.mx_nkb + kb);
            if (do_b) tma_load_3d_pair(dB + stage * C::B_BYTES_MAX, mb, &full[stage], kb * KB_ELEMS, brow, e, pol_b);
          } else {
            mbar_arrive_expect_tx(&full[stage], tx);
            if (do_a) {
              if (p.pol_a == 3) tma_load_2d_nohint(sA + stage * A_BYTES, &map_a, &full[stage], kb * KB_ELEMS, row0);
              else tma_load_2d(sA + stage * A_BYTES, &map_a, &full[stage], kb * KB_ELEMS, row0, pol_a);
            }
            if (do_b) tma_load_3d(sB + stage * C::B_BYTES_MAX, mb, &full[stage], kb * KB_ELEMS, brow, e, pol_b);
          }
#if GEMM_WAITPROF
          wp_i += clock64() - wp_c;
#endif
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
#if GEMM_WAITPROF
      printf("WPP %d %d %lld %lld %lld %lld\n", (int)blockIdx.x, (int)rank, clock64() - wp_t0, wp_e, wp_s, wp_i);
#endif
    }
    __syncwarp();
  } else if (gather && (warp == 2 || warp == 3)) {
    // Fused dispatch (step 2 folded into the A load): 64 threads gather the CTA's 128 A rows of
    // each k-block straight from the token-major input.  Thread g copies 16-B chunk (g & 7) of
    // rows (g >> 3) + 8i, i < 16: 8 consecutive threads read one row's contiguous 128 B, and
    // the chunk lands at its 128-B-swizzle position j ^ (row & 7) (row & 7 is fixed per thread).
    const int gt = (int)threadIdx.x - 64;
    const int rr = gt >> 3, ch = gt & 7;
    const uint32_t off0 = (uint32_t)(rr * 128 + ((ch ^ (rr & 7)) << 4));
    // swap-AB tail tiles: this CTA's ntok/2 token rows go to the B stage (the MMA's N operand)
    int stage = 0;
    uint32_t phase = 0;
    const bool arm = NCTA == 2 && !leader && warp == 2;  // peer: this warp arms the ring slots
    auto next_tile = [&](int seq) {
      int t = 0;
      if (lane == 0) t = sched_consume<NCTA>(ring, seq, leader, arm);
      return __shfl_sync(0xffffffffu, t, 0);
    };
    // the tile's row indices of this thread (16, or ntok/16 for a swap tile) and its stage base
    auto load_rows = [&](int t, int32_t (&tok)[16], int& nrow, uint32_t& base) {
      if (t >= total) return;
      int mt, nt;
      decode_tile(t, p.n_tiles, total_rt, p.raster, mt, nt);
      const int ntok = swap_ntok(s_ts, s_cnt, find_expert(s_ts, G, mt), mt, TM, swap_max);
      const int row0 = ntok ? mt * TM + (int)rank * (ntok >> 1) : mt * TM + (int)rank * BM;
      nrow = ntok ? ntok >> 4 : 16;
      base = smem_u32(ntok ? sB : sA) + off0;
#pragma unroll
      for (int i = 0; i < 16; ++i) tok[i] = i < nrow ? __ldg(p.gather_rows + row0 + rr + 8 * i) : 0;
    };
    WP_DECL(wp_e)
#if GEMM_WAITPROF
    const long long wp_t0 = clock64();
#endif
    const int gpol = p.pol_gather == 1 || p.pol_gather == 2 ? p.pol_gather : 0;
    int t = next_tile(0);
    int32_t tok[16];
    int nrow = 16;
    uint32_t base = smem_u32(sA) + off0;
    load_rows(t, tok, nrow, base);
    for (int seq = 0;; ++seq) {
      if (t >= total) break;
      const int tn = next_tile(seq + 1);  // published one tile ahead: prefetch its row indices
      int32_t tok_n[16];
      int nrow_n = 16;
      uint32_t base_n = base;
      load_rows(tn, tok_n, nrow_n, base_n);
      const uint8_t* src[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) src[i] = p.gather_src + (int64_t)tok[i] * p.gather_ld + ch * 16;
      for (int kb = 0; kb < nkb; ++kb) {
        WP_WAIT(wp_e, mbar_wait(&empty[stage], phase ^ 1))
        const uint32_t dst = base + (uint32_t)(stage * A_BYTES);
        // L2 policy of the gathered token rows (ASYNCEP_POL_GATHER; evict_last by default: ncu of the
        // BF16 GEMM1 at 32K tokens, profiles/r02/l2policy/: 4.79 vs 4.89 ms at the same clock)
        const uint64_t gpolicy = make_policy(gpol);
        if (nrow == 16) {
#pragma unroll
          for (int i = 0; i < 16; ++i) cp_async16_hint(dst + i * 8 * 128, src[i] + kb * 128, gpolicy);
        } else {
#pragma unroll
          for (int i = 0; i < 16; ++i)
            if (i < nrow) cp_async16_hint(dst + i * 8 * 128, src[i] + kb * 128, gpolicy);
        }
        cp_async_mbar_arrive_noinc(&afull[stage]);
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
      t = tn;
      nrow = nrow_n;
      base = base_n;
#pragma unroll
      for (int i = 0; i < 16; ++i) tok[i] = tok_n[i];
    }
#if GEMM_WAITPROF
    if (lane == 0 && warp == 2) printf("WPG %d %d %lld %lld\n", (int)blockIdx.x, (int)rank, clock64() - wp_t0, wp_e);
#endif
    __syncwarp();
  } else if (warp == 1) {
    if (gather && NCTA == 2 && !leader) {
      // peer forwarder: this CTA's gathered A stage has landed -> one arrival on the leader's
      // stage barrier (the MMA reads both CTAs' A halves).  Relaxed and without a proxy fence
      // (as CUTLASS's cp.async -> UMMA pipelines): completion of the copies is observed through
      // the mbarrier; a release.cluster arrive + fence.proxy.async here cost 1.8x on GEMM1.
      if (lane == 0) {
        int stage = 0;
        uint32_t phase = 0;
        for (int seq = 0;; ++seq) {
          if (sched_consume<NCTA>(ring, seq, false, false) >= total) break;
          for (int kb = 0; kb < nkb; ++kb) {
            mbar_wait(&afull[stage], phase);
            mbar_arrive_cluster_relaxed(&full[stage], 0);
            if (++stage == STAGES) { stage = 0; phase ^= 1; }
          }
        }
      }
    } else if (leader) {
      // MMA issuer: the whole warp runs the loop (warp-uniform state in uniform registers);
      // one elected lane issues the MMAs and the commits that track them.
      const uint32_t idesc = make_idesc(TM, p.BN, !F8);
      const uint64_t a_desc0 = make_smem_desc_sw128(smem_u32(sA));
      const uint64_t b_desc0 = make_smem_desc_sw128(smem_u32(sB));
      int stage = 0;
      uint32_t phase = 0;
      uint32_t uses0 = 0, uses1 = 0;  // tiles issued into accumulator 0 / 1 (barrier parity)
      WP_DECL(wp_f) WP_DECL(wp_a) WP_DECL(wp_t) WP_DECL(wp_s)
#if GEMM_WAITPROF
      const long long wp_t0 = clock64();
#endif
      if (MXIN) {  // the constant B scale factors of both 128-row halves of an N tile
        if (elect_one()) {
          tc_cp_sf_2(tmem_base + kMxSfbCol, smem_u32(sSF + STAGES * 512));
          tc_cp_sf_2(tmem_base + kMxSfbCol + 4, smem_u32(sSF + STAGES * 512));
        }
        __syncwarp();
      }
      for (int seq = 0;; ++seq) {
        int t = 0;
        WP_WAIT(wp_s, if (lane == 0) t = sched_consume<NCTA>(ring, seq, true, false))
        t = __shfl_sync(0xffffffffu, t, 0);
        if (t >= total) break;
        uint32_t id = idesc;
        int acc = seq & 1;
        if (MXIN) {
          const TileGeo g = tile_geo_mx(t, totalW, p.n_tiles, p.n_tiles2, p.n_out);
          acc = g.buf;
          id = make_idesc_mx(TM, g.width, 0);
        }
        if (swap_max > 0) {  // swap-AB tail: M = 256 weight rows, N = the tile's tokens
          int mt, nt;
          decode_tile(t, p.n_tiles, total_rt, p.raster, mt, nt);
          const int ntok = swap_ntok(s_ts, s_cnt, find_expert(s_ts, G, mt), mt, TM, swap_max);
          if (ntok) id = make_idesc(TM, ntok, !F8);
        }
        const uint32_t acc_phase = (acc ? uses1 : uses0) & 1u;
        WP_WAIT(wp_t, mbar_wait(&tempty[acc], acc_phase ^ 1))
        tc_fence_after();
        const uint32_t d = tmem_base + (uint32_t)(acc * 256);
        for (int kb = 0; kb < nkb; ++kb) {
          WP_WAIT(wp_f, mbar_wait(&full[stage], phase))
          WP_WAIT(wp_a, if (gather) mbar_wait(&afull[stage], phase))  // own gathered A half
          tc_fence_after();
          // descriptor start address field is addr >> 4: a stage / a 32-B K step are plain adds
          const uint64_t ad = a_desc0 + (uint64_t)((stage * A_BYTES) >> 4);
          const uint64_t bd = b_desc0 + (uint64_t)((stage * C::B_BYTES_MAX) >> 4);
          if (elect_one()) {
            // MX: the k-block's A scale factors into one of 4 TMEM slots (tcgen05.cp and
            // tcgen05.mma execute in issue order, so the slot's previous MMAs have read it)
            const uint32_t sfa = tmem_base + kMxSfaCol + 4u * (uint32_t)(kb & 3);
            if (MXIN) tc_cp_sf_2(sfa, smem_u32(sSF + stage * 512));
#pragma unroll
            for (int k = 0; k < 4; ++k) {  // 4 MMAs of 32 B of K (16 bf16 / 32 e4m3) per 128-B k-block
              const uint32_t acc_on = (kb | k) != 0 ? 1u : 0u;
              if (MXIN) {
                mma_mx_2(d, ad + 2 * k, bd + 2 * k, id | ((uint32_t)k << 4) | ((uint32_t)k << 29), sfa,
                         tmem_base + kMxSfbCol, acc_on);
              } else if (F8) {
                if (NCTA == 2) mma_f8_2(d, ad + 2 * k, bd + 2 * k, id, acc_on);
                else mma_f8(d, ad + 2 * k, bd + 2 * k, id, acc_on);
              } else {
                if (NCTA == 2) mma_bf16_2(d, ad + 2 * k, bd + 2 * k, id, acc_on);
                else mma_bf16(d, ad + 2 * k, bd + 2 * k, id, acc_on);
              }
            }
            if (NCTA == 2) tc_commit2_mc(&empty[stage], 0x3);
            else tc_commit(&empty[stage]);
          }
          __syncwarp();
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        if (elect_one()) {
          if (NCTA == 2) tc_commit2_mc(&tfull[acc], 0x3);
          else tc_commit(&tfull[acc]);
        }
        __syncwarp();
        if (acc) ++uses1; else ++uses0;
      }
#if GEMM_WAITPROF
      if (lane == 0) printf("WPM %d %lld %lld %lld %lld %lld\n", (int)blockIdx.x, clock64() - wp_t0, wp_f, wp_a, wp_t, wp_s);
#endif
    }
    __syncwarp();
  } else if (warp >= 4) {
    const int ew = warp - 4;           // epilogue warp index (staging / scale buffers)
    const int quad = warp & 3;         // TMEM lanes [32*quad, 32*quad+32): this warp's rows
    uint8_t* stg = sStg + ew * C::NSTG * STG_BYTES;
    uint32_t chunk = 0;  // stores issued by this warp (staging buffer parity)
    uint32_t uses0 = 0, uses1 = 0;  // tiles read out of accumulator 0 / 1 (barrier parity)
    WP_DECL(wp_f) WP_DECL(wp_s) WP_DECL(wp_store_acc)
#if GEMM_WAITPROF
    const long long wp_t0 = clock64();
#endif
    for (int seq = 0;; ++seq) {
      int t = 0;
      WP_WAIT(wp_s, if (lane == 0) t = sched_consume<NCTA>(ring, seq, leader, false))
      t = __shfl_sync(0xffffffffu, t, 0);
      if (t >= total) break;
      int mt, nt = 0, acc = seq & 1, col0 = 0, width = 0;  // col0 / width: MXIN tile columns
      if (MXIN) {
        const TileGeo g = tile_geo_mx(t, totalW, p.n_tiles, p.n_tiles2, p.n_out);
        mt = g.mt;
        acc = g.buf;
        col0 = g.col0;
        width = g.width;
      } else {
        decode_tile(t, p.n_tiles, total_rt, p.raster, mt, nt);
      }
      const uint32_t acc_phase = (acc ? uses1 : uses0) & 1u;
      if (acc) ++uses1; else ++uses0;
      const int wrow0 = mt * TM + (int)rank * BM + quad * 32;  // first row of this warp's slice
      WP_WAIT(wp_f, mbar_wait(&tfull[acc], acc_phase))
      tc_fence_after();
      const uint32_t tb = tmem_base + ((uint32_t)(quad * 32) << 16) + (uint32_t)(acc * 256);
      // hand the accumulator back to the MMA as soon as the warp's last tcgen05.ld has landed
      // (before the final chunk's math and store), not after the stores
      bool released = false;
      auto release = [&]() {
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if (NCTA == 2) mbar_arrive_remote(&tempty[acc], 0);
          else mbar_arrive(&tempty[acc]);
        }
        released = true;
      };
      const int ntok = swap_max > 0 ? swap_ntok(s_ts, s_cnt, find_expert(s_ts, G, mt), mt, TM, swap_max) : 0;
      if ((MODE == EPI_SWIGLU || MODE == EPI_PLAIN) && ntok) {
        // Swap-AB tail tile: TMEM lane = weight row of this CTA, column c = token row mt*TM + c.
        // GEMM1: lanes [0,16) of the quadrant hold gate rows j = jq, lanes [16,32) the up rows of
        // the same j (the packed W_gu's 32-row groups, asyncep.h); GEMM2: lane = output column.  The values are
        // transposed through the warp's staging buffer and written to out_ptr row by row.
        const int trow0 = mt * TM;  // the tile's first (token) row
        const bool upper = lane >= 16;
        int ge = find_expert(s_ts, G, mt);
        const bool own_g = ge >= p.own_lo && ge < p.own_hi;
        float* tsc = sScl + ew * 256;  // FP8: the tile's token (row) scales
        const float* wsc = nullptr;    // FP8: this expert's weight scales of the N tile
        if (F8) {
          wsc = reinterpret_cast<const float*>(own_g ? p.b_scale_base_own + (size_t)(ge - p.own_lo) * p.expert_bytes
                                                     : p.b_scale_base + (size_t)ge * p.expert_bytes) + nt * 256;
          __syncwarp();
          for (int i = lane; i < ntok; i += 32)
            tsc[i] = p.a_scale[(MODE == EPI_SWIGLU && gather) ? __ldg(p.gather_rows + trow0 + i) : trow0 + i];
          __syncwarp();
        }
        if (lane == 0) bulk_wait_read0();  // earlier TMA stores have finished reading the staging buffer
        __syncwarp();
        if (MODE == EPI_SWIGLU) {
          // FP8: each lane scales its own weight row (packed row rank*128 + quad*32 + lane of the
          // N tile: the gate row for lane < 16, the up row for lane >= 16) before the exchange
          const float swr = F8 ? __ldg(wsc + (int)rank * 128 + quad * 32 + lane) : 1.f;
          bf16* outc = p.out_ptr + nt * 128 + (int)rank * 64 + quad * 16;
#pragma unroll 1
          for (int c0 = 0; c0 < ntok; c0 += 32) {
            uint32_t v[32];
            tmem_ld32(tb + c0, v);
            tmem_ld_wait();
            if (c0 + 32 >= ntok) release();
            const int cb = upper ? 16 : 0;  // this lane's 16 token columns of the chunk
#pragma unroll
            for (int i = 0; i < 16; i += 2) {
              float g[2], u[2];
#pragma unroll
              for (int q2 = 0; q2 < 2; ++q2) {
                // keep this lane's token column cb + i + q2, send the partner's (16 - cb) + i + q2
                // (selects between two static indices: a runtime index would put v[] in local memory)
                float keep = __uint_as_float(upper ? v[16 + i + q2] : v[i + q2]);
                float send = __uint_as_float(upper ? v[i + q2] : v[16 + i + q2]);
                if (F8) {
                  keep *= swr * tsc[c0 + cb + i + q2];
                  send *= swr * tsc[c0 + 16 - cb + i + q2];
                }
                const float recv = __shfl_xor_sync(0xffffffffu, send, 16);
                g[q2] = upper ? recv : keep;
                u[q2] = upper ? keep : recv;
              }
              float a0, a1;
              mul2(a0, a1, silu_f(g[0]), silu_f(g[1]), u[0], u[1]);
              const uint32_t pk = pack_bf16x2(a0, a1);
              // staging [32 tokens][16 act columns] bf16
              *reinterpret_cast<uint16_t*>(stg + (cb + i) * 32 + (lane & 15) * 2) = (uint16_t)(pk & 0xffffu);
              *reinterpret_cast<uint16_t*>(stg + (cb + i + 1) * 32 + (lane & 15) * 2) = (uint16_t)(pk >> 16);
            }
            __syncwarp();
            {  // lane = token row c0 + lane: 16 act columns = 32 B
              const uint4* src = reinterpret_cast<const uint4*>(stg + lane * 32);
              uint4* dst = reinterpret_cast<uint4*>(outc + (int64_t)(trow0 + c0 + lane) * p.n_out);
              dst[0] = src[0];
              dst[1] = src[1];
              if (F8) {  // per-token max |act| of this warp's 16 columns (bf16 magnitudes)
                const uint16_t* r16 = reinterpret_cast<const uint16_t*>(stg + lane * 32);
                uint32_t m = 0;
#pragma unroll
                for (int j = 0; j < 16; ++j) m = max(m, (uint32_t)(r16[j] & 0x7fffu));
                if (c0 + lane < ntok) atomicMax(p.amax_out + trow0 + c0 + lane, m << 16);
              }
            }
            __syncwarp();
          }
        } else {
          const int ncol = (int)rank * 128 + quad * 32 + lane;  // output column within the N tile
          const float sw = F8 ? __ldg(wsc + ncol) : 1.f;
          bf16* outc = p.out_ptr + nt * p.BN + (int)rank * 128 + quad * 32;
#pragma unroll 1
          for (int c0 = 0; c0 < ntok; c0 += 32) {
            uint32_t v[32];
            tmem_ld32(tb + c0, v);
            tmem_ld_wait();
            if (c0 + 32 >= ntok) release();
#pragma unroll
            for (int i = 0; i < 32; i += 2) {
              float x0 = __uint_as_float(v[i]), x1 = __uint_as_float(v[i + 1]);
              if (F8) {
                x0 *= sw * tsc[c0 + i];
                x1 *= sw * tsc[c0 + i + 1];
              }
              const uint32_t pk = pack_bf16x2(x0, x1);
              // staging [32 tokens][32 output columns] bf16
              *reinterpret_cast<uint16_t*>(stg + i * 64 + lane * 2) = (uint16_t)(pk & 0xffffu);
              *reinterpret_cast<uint16_t*>(stg + (i + 1) * 64 + lane * 2) = (uint16_t)(pk >> 16);
            }
            __syncwarp();
            const uint4* src = reinterpret_cast<const uint4*>(stg + lane * 64);
            uint4* dst = reinterpret_cast<uint4*>(outc + (int64_t)(trow0 + c0 + lane) * p.n_out);
#pragma unroll
            for (int j = 0; j < 4; ++j) dst[j] = src[j];
            __syncwarp();
          }
        }
        (void)ge;
      } else if (MODE == EPI_ROUTER || MODE == EPI_ROUTER16) {
        const int row = wrow0 + lane;
        router_epilogue<MODE == EPI_ROUTER ? 8 : 16>(tb, p.E, p.top_k, p.norm_topk, row < p.dense_rows,
                                                     p.ids + (int64_t)row * p.top_k, p.w + (int64_t)row * p.top_k);
      } else if (MODE == EPI_SWIGLU) {
        // accumulator column 32g + i (g < 8, i < 16) = gate of act column nt*128 + 16g + i, column
        // 32g + 16 + i = its up (the packed W_gu layout, asyncep.h)
        float sa = 1.f, amax = 0.f;
        const float* sb = nullptr;
        if (F8) {
          sa = p.a_scale[gather ? __ldg(p.gather_rows + wrow0 + lane) : wrow0 + lane];
          int ge = find_expert(s_ts, G, mt);
          if (p.group_mod > 0) ge %= p.group_mod;
          sb = reinterpret_cast<const float*>(
                   (ge >= p.own_lo && ge < p.own_hi ? p.b_scale_base_own + (size_t)(ge - p.own_lo) * p.expert_bytes
                                                    : p.b_scale_base + (size_t)ge * p.expert_bytes)) +
               nt * 256;
          sb = stage_scales(sScl + ew * 256, sb, 256, lane);
        }
        uint32_t sfw = 0;  // MXOUT: the row's 4 E8M0 scale bytes of this 128-column k-block
        if (MXOUT) {
          if (lane == 0) bulk_wait_read0();  // the warp's previous store has read the staging buffer
          __syncwarp();
        }
#pragma unroll 1
        for (int c0 = 0; c0 < 128; c0 += 64) {  // act columns c0 .. c0+63 = packed groups c0/16 .. +3
          uint32_t o[32];
          uint32_t amax2 = 0;  // |bf16| bit patterns of both halves: unsigned order = magnitude order
          uint32_t vv[4][32];  // the chunk's 4 groups of [16 gate | 16 up] columns, one wait
#pragma unroll
          for (int grp = 0; grp < 4; ++grp) tmem_ld32(tb + 2 * c0 + 32 * grp, vv[grp]);
          tmem_ld_wait();
          if (c0 + 64 >= 128) release();  // last TMEM read of the tile
#pragma unroll
          for (int grp = 0; grp < 4; ++grp) {
            const uint32_t(&v)[32] = vv[grp];
#pragma unroll
            for (int q = 0; q < 4; ++q) {  // 4 act columns per step
              float gv[4], uv[4];
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                gv[j] = __uint_as_float(v[4 * q + j]);
                uv[j] = __uint_as_float(v[16 + 4 * q + j]);
              }
              if (F8) {  // dequantise: acc * (a row scale) * (w channel scale)
                const int cc = 2 * c0 + 32 * grp + 4 * q;  // packed column of the gate values
                const float4 sg = ld_shared_f4(smem_u32(sb) + 4 * cc);
                const float4 su = ld_shared_f4(smem_u32(sb) + 4 * (cc + 16));
                float s0, s1, s2, s3, t0, t1, t2, t3;
                mul2(s0, s1, sa, sa, sg.x, sg.y);
                mul2(s2, s3, sa, sa, sg.z, sg.w);
                mul2(t0, t1, sa, sa, su.x, su.y);
                mul2(t2, t3, sa, sa, su.z, su.w);
                mul2(gv[0], gv[1], gv[0], gv[1], s0, s1);
                mul2(gv[2], gv[3], gv[2], gv[3], s2, s3);
                mul2(uv[0], uv[1], uv[0], uv[1], t0, t1);
                mul2(uv[2], uv[3], uv[2], uv[3], t2, t3);
              }
#pragma unroll
              for (int j = 0; j < 2; ++j) {
                float a0, a1;
                mul2(a0, a1, silu_f(gv[2 * j]), silu_f(gv[2 * j + 1]), uv[2 * j], uv[2 * j + 1]);
                const uint32_t pk = pack_bf16x2(a0, a1);
                o[8 * grp + 2 * q + j] = pk;
                if (F8 && !MXOUT) amax2 = __vmaxu2(amax2, pk & 0x7fff7fffu);
              }
            }
          }
          if (MXOUT) {
            // two MX blocks (act columns c0 .. c0+31, c0+32 .. c0+63) -> 64 e4m3 bytes = 16-B chunks
            // 4h .. 4h+3 (h = c0 / 64) of the row's 128-B line in the 128-B-swizzled staging buffer
            uint32_t qa[8], qb[8];
            const uint32_t ea = mx_block(o, qa), eb = mx_block(o + 16, qb);
            const int hf = c0 >> 6;
            sfw |= (ea | (eb << 8)) << (16 * hf);
            const uint32_t base = smem_u32(stg) + lane * 128;
            st_shared_v4(base + (((4 * hf + 0) ^ (lane & 7)) << 4), qa[0], qa[1], qa[2], qa[3]);
            st_shared_v4(base + (((4 * hf + 1) ^ (lane & 7)) << 4), qa[4], qa[5], qa[6], qa[7]);
            st_shared_v4(base + (((4 * hf + 2) ^ (lane & 7)) << 4), qb[0], qb[1], qb[2], qb[3]);
            st_shared_v4(base + (((4 * hf + 3) ^ (lane & 7)) << 4), qb[4], qb[5], qb[6], qb[7]);
          } else {
            stage_and_store<C::NSTG>(o, stg + (chunk++ % C::NSTG) * STG_BYTES, lane, &map_out, nt * 128 + c0, wrow0
#if GEMM_WAITPROF
                                    , wp_store_acc
#endif
                                    );
          }
          if (F8 && !MXOUT) amax = fmaxf(amax, fmaxf(bf16_lo(amax2), bf16_hi(amax2)));
        }
        if (MXOUT) {
          // the tile's 128 e4m3 columns x 32 rows in one TMA store; the scale word of row m of the
          // CTA's 128-row block at word (m % 32) * 4 + m / 32 of the block's chunk for k-block nt
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            tma_store_2d(&map_out, stg, nt * 128, wrow0);
            bulk_commit();
          }
          p.mx_sf_out[((size_t)(mt * 2 + (int)rank) * p.mx_nkb + nt) * 128 + lane * 4 + quad] = sfw;
        } else if (F8) {
          atomicMax(p.amax_out + wrow0 + lane, __float_as_uint(amax));
        }
      } else {
        float sa = 1.f;  // MXIN: the A scales were applied by the block-scaled MMA
        const float* sb = nullptr;
        const int ocol = MXIN ? col0 : nt * p.BN;  // the tile's first output column
        if (F8) {
          if (!MXIN) sa = p.a_scale[wrow0 + lane];
          int ge = find_expert(s_ts, G, mt);
          if (p.group_mod > 0) ge %= p.group_mod;
          sb = reinterpret_cast<const float*>(
                   (ge >= p.own_lo && ge < p.own_hi ? p.b_scale_base_own + (size_t)(ge - p.own_lo) * p.expert_bytes
                                                    : p.b_scale_base + (size_t)ge * p.expert_bytes)) +
               ocol;
          sb = stage_scales(sScl + ew * 256, sb, MXIN ? width : p.BN, lane);
        }
        const int cbeg = 0;
        const int cend = MXIN ? width : min(p.BN, max(p.n_out - nt * p.BN, 0));
#pragma unroll 1
        for (int c0 = cbeg; c0 < cend; c0 += 64) {
          if (MXIN && c0 + 32 == cend) {
            // a 32-column remainder (224-wide tiles): 64 B of this thread's row, stored directly
            uint32_t r[32];
            tmem_ld32(tb + c0, r);
            tmem_ld_wait();
            release();
            uint32_t o[16];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              const float4 sv = ld_shared_f4(smem_u32(sb) + 4 * (c0 + 4 * q));
              float v0, v1, v2, v3;
              mul2(v0, v1, __uint_as_float(r[4 * q]), __uint_as_float(r[4 * q + 1]), sv.x, sv.y);
              mul2(v2, v3, __uint_as_float(r[4 * q + 2]), __uint_as_float(r[4 * q + 3]), sv.z, sv.w);
              o[2 * q] = pack_bf16x2(v0, v1);
              o[2 * q + 1] = pack_bf16x2(v2, v3);
            }
            uint4* dst = reinterpret_cast<uint4*>(p.out_ptr + (int64_t)(wrow0 + lane) * p.n_out + ocol + c0);
#pragma unroll
            for (int j = 0; j < 4; ++j) dst[j] = make_uint4(o[4 * j], o[4 * j + 1], o[4 * j + 2], o[4 * j + 3]);
            break;
          }
          uint32_t o[32];
          uint32_t rr[2][32];  // the chunk's 64 columns, one wait
          tmem_ld32(tb + c0, rr[0]);
          tmem_ld32(tb + c0 + 32, rr[1]);
          tmem_ld_wait();
          if (c0 + 64 >= cend) release();  // last TMEM read of the tile: the MMA may reuse it
#pragma unroll
          for (int half = 0; half < 2; ++half) {
            const uint32_t(&r)[32] = rr[half];
#pragma unroll
            for (int q = 0; q < 8; ++q) {  // 4 columns per step
              float v[4];
#pragma unroll
              for (int j = 0; j < 4; ++j) v[j] = __uint_as_float(r[4 * q + j]);
              if (F8) {  // dequantise: acc * (a row scale) * (w channel scale)
                const int cc = c0 + 32 * half + 4 * q;
                const float4 sv = ld_shared_f4(smem_u32(sb) + 4 * cc);
                float s0, s1, s2, s3;
                mul2(s0, s1, sa, sa, sv.x, sv.y);
                mul2(s2, s3, sa, sa, sv.z, sv.w);
                mul2(v[0], v[1], v[0], v[1], s0, s1);
                mul2(v[2], v[3], v[2], v[3], s2, s3);
              }
              o[16 * half + 2 * q] = pack_bf16x2(v[0], v[1]);
              o[16 * half + 2 * q + 1] = pack_bf16x2(v[2], v[3]);
            }
          }
          stage_and_store<C::NSTG>(o, stg + (chunk++ % C::NSTG) * STG_BYTES, lane, &map_out, ocol + c0, wrow0
#if GEMM_WAITPROF
                                  , wp_store_acc
#endif
                                  );
        }
      }
      if (!released) release();  // router epilogue, or no stored columns
    }
#if GEMM_WAITPROF
    if (lane == 0 && warp == 4) printf("WPE %d %d %lld %lld %lld %lld\n", (int)blockIdx.x, (int)rank, clock64() - wp_t0, wp_f, wp_s, g_wp_store);
#endif
    if ((MODE == EPI_PLAIN || MODE == EPI_SWIGLU) && lane == 0) bulk_wait0();  // this warp's stores done
    __syncwarp();
  }
  tc_fence_before();
  if (NCTA == 2) cluster_sync_all(); else __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    if (NCTA == 2) tmem_dealloc2(tmem_base, TMEM_COLS);
    else tmem_dealloc(tmem_base, TMEM_COLS);
  }
}

template <int MODE, int NCTA, bool F8 = false, bool MX = false>
void launch_mode(const TcArgs& a, const CUtensorMap& ma, const CUtensorMap& mb, const CUtensorMap& mo, int grid,
                 cudaStream_t s, const CUtensorMap* mb2 = nullptr, const CUtensorMap* msf = nullptr) {
  using C = Cfg<NCTA, MODE, MX && MODE == EPI_PLAIN>;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaFuncSetAttribute(gemm_tc_kernel<MODE, NCTA, F8, MX>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)C::SMEM);
  });
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(C::NTHR);
  cfg.dynamicSmemBytes = C::SMEM;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = NCTA;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, gemm_tc_kernel<MODE, NCTA, F8, MX>, ma, mb, mo, mb2 ? *mb2 : mb, msf ? *msf : mb, a);
}

// Grouped GEMMs run as CTA pairs by default.  ASYNCEP_GEMM_NCTA=1 selects the 1-CTA
// kernel and ASYNCEP_GEMM_RASTER=G a grouped rasterisation (A/B experiments only).
int grouped_ncta() {
  static const int n = env_int("ASYNCEP_GEMM_NCTA", 2) == 1 ? 1 : 2;
  return n;
}
int grouped_raster() {
  static const int r = env_int("ASYNCEP_GEMM_RASTER", 0);
  return r;
}

void launch_grouped(const GroupedArgs& g, const CUtensorMap& ma, const CUtensorMap& mb, const CUtensorMap& mo,
                    int K, int BN, int n_tiles, int mode, int n_out, int num_sms, cudaStream_t s,
                    const int32_t* gather_rows = nullptr, const F8Args* f8 = nullptr, bool gemm2 = false,
                    const void* gather_src = nullptr, int64_t gather_ld = 0, const OwnShard* own = nullptr,
                    bf16* out = nullptr, const CUtensorMap* msf = nullptr) {
  static const bool dyn = env_int("ASYNCEP_STATIC_SCHED", 0) == 0;
  const int ncta = f8 ? 2 : grouped_ncta();
  const bool mx = f8 && f8->mx;
  TcArgs a{};
  a.tile_start = g.tile_start;
  a.E = g.E;
  a.K = K;
  a.BN = BN;
  a.n_tiles = n_tiles;
  a.n_out = n_out;
  a.ts_scale = kRowAlign / (kTileM * ncta);
  a.raster = grouped_raster();
  a.pol_a = env_int("ASYNCEP_POL_A", 0);
  a.pol_b = env_int("ASYNCEP_POL_B", 1);
  a.pol_gather = env_int("ASYNCEP_POL_GATHER", 1);
  a.gather_rows = gather_rows;
  a.gather_src = static_cast<const uint8_t*>(gather_src);
  a.gather_ld = gather_ld;
  const CUtensorMap* mb2 = nullptr;
  a.counts = g.counts;
  a.swap_max = (ncta == 2 && out && g.counts && !mx) ? (gemm2 ? g.swap_max2 : g.swap_max) : 0;
  a.out_ptr = out;
  if (own && own->maps && own->hi > own->lo) {
    a.own_lo = own->lo;
    a.own_hi = own->hi;
    mb2 = gemm2 ? &own->maps->wd : &own->maps->wgu;
    if (f8) a.b_scale_base_own = own->base + (gemm2 ? f8->sd_off : f8->sgu_off);
  }
  a.sched = (dyn && g.sched) ? g.sched + (gemm2 ? 2 : 1) : nullptr;
  a.group_mod = g.group_mod;
  int tiles_per_rt = n_tiles;
  if (mx && gemm2) {  // 256- and 224-wide N tiles, alternating (period 480) over the n_out columns
    a.n_tiles = (n_out + kMxPeriod - 1) / kMxPeriod;
    a.n_tiles2 = n_out > kMxWide ? (n_out - kMxWide + kMxPeriod - 1) / kMxPeriod : 0;
    a.mx_nkb = K / 128;
    static const int sfw = env_int("ASYNCEP_MX_SF_WARP", 2);
    a.mx_sf_warp = sfw;
    tiles_per_rt = a.n_tiles + a.n_tiles2;
  } else if (mx) {
    a.mx_sf_out = f8->act_sf;
    a.mx_nkb = n_tiles;  // GEMM1 N tile nt = GEMM2 k-block nt (128 act columns)
  }
  if (f8) {
    a.a_scale = gemm2 ? f8->act_scale : f8->x_scale;
    a.b_scale_base = f8->layer + (gemm2 ? f8->sd_off : f8->sgu_off);
    a.expert_bytes = f8->expert_bytes;
    a.amax_out = gemm2 ? nullptr : f8->act_amax;
  }
  const int units = num_sms / ncta;
  const int upper = g.max_m_tiles * a.ts_scale * tiles_per_rt;
  const int grid = ncta * (upper < units ? (upper > 0 ? upper : 1) : units);
  if (f8 && mx) {  // FP8 experts with the MX intermediate
    if (mode == EPI_SWIGLU) launch_mode<EPI_SWIGLU, 2, true, true>(a, ma, mb, mo, grid, s, mb2);
    else launch_mode<EPI_PLAIN, 2, true, true>(a, ma, mb, mo, grid, s, mb2, msf);
  } else if (f8) {  // FP8 experts: CTA pairs only
    if (mode == EPI_SWIGLU) launch_mode<EPI_SWIGLU, 2, true>(a, ma, mb, mo, grid, s, mb2);
    else launch_mode<EPI_PLAIN, 2, true>(a, ma, mb, mo, grid, s, mb2);
  } else if (ncta == 2) {
    if (mode == EPI_SWIGLU) launch_mode<EPI_SWIGLU, 2>(a, ma, mb, mo, grid, s, mb2);
    else launch_mode<EPI_PLAIN, 2>(a, ma, mb, mo, grid, s, mb2);
  } else {
    if (mode == EPI_SWIGLU) launch_mode<EPI_SWIGLU, 1>(a, ma, mb, mo, grid, s, mb2);
    else launch_mode<EPI_PLAIN, 1>(a, ma, mb, mo, grid, s, mb2);
  }
}
}  // namespace

int gemm2_bn(int H) { return H >= 256 ? 256 : H; }

bool make_act_maps(ActMaps& m, const bf16* xperm, const bf16* act, int64_t R_max, int H, int h, const uint8_t* xq,
                   const uint8_t* aq, const uint32_t* asf) {
  const uint32_t box[2] = {BK, BM};
  if (aq && asf) {  // MX intermediate: e4m3 store map {128 cols, 32 rows}; scale chunks as [chunks][128] u32
    const uint32_t sbox[2] = {128, 32};
    const uint64_t d1[2] = {(uint64_t)h, (uint64_t)R_max};
    const uint64_t s1[1] = {(uint64_t)h};
    if (!encode_tmap(&m.aq_out, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, aq, d1, s1, sbox, CU_TENSOR_MAP_SWIZZLE_128B))
      return false;
    const uint32_t fbox[2] = {128, 1};
    const uint64_t d2[2] = {128, (uint64_t)(R_max / 128) * (uint64_t)(h / 128)};
    const uint64_t s2[1] = {512};
    if (!encode_tmap(&m.sfa, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, asf, d2, s2, fbox, CU_TENSOR_MAP_SWIZZLE_NONE))
      return false;
    m.mx = true;
  }
  if (xq && aq) {  // FP8 operands: 128 e4m3 = 128 B per k-block row
    const uint32_t qbox[2] = {128, BM};
    const uint64_t d1[2] = {(uint64_t)H, (uint64_t)R_max};
    const uint64_t s1[1] = {(uint64_t)H};
    if (!encode_tmap(&m.xq, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, xq, d1, s1, qbox, CU_TENSOR_MAP_SWIZZLE_128B))
      return false;
    const uint64_t d2[2] = {(uint64_t)h, (uint64_t)R_max};
    const uint64_t s2[1] = {(uint64_t)h};
    if (!encode_tmap(&m.aq, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, aq, d2, s2, qbox, CU_TENSOR_MAP_SWIZZLE_128B))
      return false;
  }
  {
    const uint64_t dims[2] = {(uint64_t)H, (uint64_t)R_max};
    const uint64_t strides[1] = {(uint64_t)H * 2};
    if (!encode_tmap(&m.xperm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, xperm, dims, strides, box,
                     CU_TENSOR_MAP_SWIZZLE_128B))
      return false;
  }
  {
    const uint64_t dims[2] = {(uint64_t)h, (uint64_t)R_max};
    const uint64_t strides[1] = {(uint64_t)h * 2};
    if (!encode_tmap(&m.act, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, act, dims, strides, box,
                     CU_TENSOR_MAP_SWIZZLE_128B))
      return false;
  }
  {  // epilogue TMA-store maps: box {64 cols, 32 rows}
    const uint32_t sbox[2] = {64, 32};
    const uint64_t d1[2] = {(uint64_t)h, (uint64_t)R_max};
    const uint64_t s1[1] = {(uint64_t)h * 2};
    if (!encode_tmap(&m.act_out, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, act, d1, s1, sbox,
                     CU_TENSOR_MAP_SWIZZLE_128B))
      return false;
    const uint64_t d2[2] = {(uint64_t)H, (uint64_t)R_max};
    const uint64_t s2[1] = {(uint64_t)H * 2};
    if (!encode_tmap(&m.yperm_out, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, xperm, d2, s2, sbox,
                     CU_TENSOR_MAP_SWIZZLE_128B))
      return false;
  }
  m.bn2 = gemm2_bn(H);
  return true;
}

bool make_weight_maps(GemmMaps& m, const void* layer, size_t expert_bytes, int E, int H, int h, int bn2, bool fp8) {
  const int b = fp8 ? 1 : 2;  // bytes per weight
  const int ncta = fp8 ? 2 : grouped_ncta();
  const CUtensorMapDataType dt = fp8 ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
  const uint32_t kb = 128 / b;  // elements per 128-B row of a k-block
  {
    const uint64_t dims[3] = {(uint64_t)H, (uint64_t)(2 * h), (uint64_t)E};
    const uint64_t strides[2] = {(uint64_t)H * b, (uint64_t)expert_bytes};
    const uint32_t box[3] = {kb, (uint32_t)(256 / ncta), 1};
    if (!encode_tmap(&m.wgu, dt, 3, layer, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B)) return false;
  }
  {
    const uint8_t* wd = reinterpret_cast<const uint8_t*>(layer) + (size_t)2 * h * H * b;
    const uint64_t dims[3] = {(uint64_t)h, (uint64_t)H, (uint64_t)E};
    const uint64_t strides[2] = {(uint64_t)h * b, (uint64_t)expert_bytes};
    const uint32_t box[3] = {kb, (uint32_t)(bn2 / ncta), 1};
    if (!encode_tmap(&m.wd, dt, 3, wd, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B)) return false;
  }
  m.fp8 = fp8;
  return true;
}

bool launch_gemm1_tc(const GroupedArgs& g, const ActMaps& am, const GemmMaps& wm, int H, int h, bf16* act,
                     const void* x_gather, int64_t T, const int32_t* src_tok, int num_sms, cudaStream_t s,
                     const F8Args* f8, const OwnShard* own) {
  if (f8 && f8->mx && !am.mx) return false;
  // N tiles of 256 packed W_gu rows = 128 gate + 128 up columns -> 128 act columns.
  // x_gather != nullptr: dispatch fused into the A load (rows gathered from the token-major
  // x / x_q through src_tok); the A map is then unused.
  const int64_t ld = (int64_t)H * (f8 ? 1 : 2);
  const CUtensorMap& ma = f8 ? am.xq : am.xperm;
  launch_grouped(g, ma, wm.wgu, (f8 && f8->mx) ? am.aq_out : am.act_out, H, 256, (2 * h) / 256, EPI_SWIGLU, h,
                 num_sms, s, x_gather ? src_tok : nullptr, f8, false, x_gather, ld, own, act);
  (void)T;
  return true;
}

void launch_gemm2_tc(const GroupedArgs& g, const ActMaps& am, const GemmMaps& wm, int H, int h, bf16* yperm,
                     int num_sms, cudaStream_t s, const F8Args* f8, const OwnShard* own) {
  const int bn = am.bn2;
  launch_grouped(g, f8 ? am.aq : am.act, wm.wd, am.yperm_out, h, bn, (H + bn - 1) / bn, EPI_PLAIN, H, num_sms, s,
                 nullptr, f8, true, nullptr, 0, own, yperm, &am.sfa);
}

// ------------------------------------------------------------------ dense GEMM (NEXT-3 projections)
bool launch_dense_gemm_tc(const bf16* A, int64_t M, int K, const bf16* W, int N, bf16* out, int* sched, int num_sms,
                          cudaStream_t s) {
  if (M <= 0) return true;
  if (K % 64 || N % 256) return false;
  CUtensorMap ma, mb, mo;
  {
    const uint64_t dims[2] = {(uint64_t)K, (uint64_t)M};
    const uint64_t strides[1] = {(uint64_t)K * 2};
    const uint32_t box[2] = {BK, BM};
    if (!encode_tmap(&ma, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, A, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B))
      return false;
  }
  {
    const uint64_t dims[3] = {(uint64_t)K, (uint64_t)N, 1};
    const uint64_t strides[2] = {(uint64_t)K * 2, (uint64_t)K * 2 * N};
    const uint32_t box[3] = {BK, 128, 1};  // 256-row W tile, half per CTA of the pair
    if (!encode_tmap(&mb, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, W, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B))
      return false;
  }
  {
    const uint64_t dims[2] = {(uint64_t)N, (uint64_t)M};
    const uint64_t strides[1] = {(uint64_t)N * 2};
    const uint32_t box[2] = {64, 32};
    if (!encode_tmap(&mo, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, out, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B))
      return false;
  }
  TcArgs a{};
  a.E = 1;
  a.dense_rows = (int)M;
  a.K = K;
  a.BN = 256;
  a.n_tiles = N / 256;
  a.n_out = N;
  a.ts_scale = 1;
  a.raster = 0;
  a.pol_a = 0;
  a.pol_b = 1;  // the weight tile is reused by every row tile
  a.sched = sched;
  const int units = num_sms / 2;
  const int64_t total = (M + 255) / 256 * a.n_tiles;
  const int grid = 2 * (int)(total < units ? total : units);
  launch_mode<EPI_PLAIN, 2>(a, ma, mb, mo, grid, s);
  return true;
}

// ------------------------------------------------------------------ router on tcgen05
// Logits tile = 128 tokens x E_pad experts (M=128, N=E_pad, K=H, 1-CTA) in TMEM, fp32;
// the epilogue threads (one per token) do the top-k straight out of TMEM.
// With E_pad >= 64 the router runs on CTA pairs (M = 256 tokens, each CTA loading half of W_r):
// W_r is streamed through shared memory once per 256 tokens instead of once per 128, and each
// CTA's accumulator still holds its 128 tokens x all E logits (the top-k epilogue is unchanged).
bool make_router_wmap(RouterTc& rt, const bf16* wr, int H, int E) {
  static const bool pair_ok = env_int("ASYNCEP_ROUTER_PAIR", 1) != 0;
  rt.E_pad = (E + 15) / 16 * 16;
  rt.pair = pair_ok && rt.E_pad >= 64 && rt.E_pad % 32 == 0;
  const uint64_t dims[3] = {(uint64_t)H, (uint64_t)E, 1};
  const uint64_t strides[2] = {(uint64_t)H * 2, (uint64_t)H * 2 * E};
  const uint32_t box[3] = {BK, (uint32_t)rt.E_pad, 1};
  const uint32_t box2[3] = {BK, (uint32_t)rt.E_pad / 2, 1};
  return encode_tmap(&rt.map_wr, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, wr, dims, strides, box,
                     CU_TENSOR_MAP_SWIZZLE_128B) &&
         encode_tmap(&rt.map_wr2, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, wr, dims, strides, box2,
                     CU_TENSOR_MAP_SWIZZLE_128B);
}

bool launch_router_tc(const RouterTc& rt, const bf16* x, int64_t T, int H, int E, int k, int norm_topk,
                      int32_t* ids, float* w, int num_sms, cudaStream_t s, int* sched) {
  if (T <= 0) return true;
  CUtensorMap map_x;
  const uint64_t dims[2] = {(uint64_t)H, (uint64_t)T};
  const uint64_t strides[1] = {(uint64_t)H * 2};
  const uint32_t box[2] = {BK, BM};
  if (!encode_tmap(&map_x, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, x, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B))
    return false;
  TcArgs a{};
  a.E = E;
  a.dense_rows = (int)T;
  a.K = H;
  a.BN = rt.E_pad;
  a.n_tiles = 1;
  a.ts_scale = 1;
  a.sched = sched;
  a.top_k = k;
  a.norm_topk = norm_topk;
  a.ids = ids;
  a.w = w;
  if (rt.pair) {
    const int tiles = (int)((T + 2 * BM - 1) / (2 * BM)), units = num_sms / 2;
    const int grid = 2 * (tiles < units ? tiles : units);
    if (k <= 8) launch_mode<EPI_ROUTER, 2>(a, map_x, rt.map_wr2, map_x, grid, s);
    else launch_mode<EPI_ROUTER16, 2>(a, map_x, rt.map_wr2, map_x, grid, s);
    return true;
  }
  const int tiles = (int)((T + BM - 1) / BM);
  if (k <= 8) launch_mode<EPI_ROUTER, 1>(a, map_x, rt.map_wr, map_x, tiles < num_sms ? tiles : num_sms, s);
  else launch_mode<EPI_ROUTER16, 1>(a, map_x, rt.map_wr, map_x, tiles < num_sms ? tiles : num_sms, s);
  return true;
}

// ------------------------------------------------------------------ tensor-map encoding
bool encode_tmap(CUtensorMap* map, CUtensorMapDataType dtype, int rank, const void* base, const uint64_t* dims,
                 const uint64_t* strides_bytes, const uint32_t* box, CUtensorMapSwizzle sw) {
  typedef CUresult (*encode_fn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static encode_fn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<encode_fn>(p);
  });
  if (!fn) return false;
  cuuint64_t d[5];
  cuuint64_t st[4];
  cuuint32_t b[5], es[5];
  for (int i = 0; i < rank; ++i) {
    d[i] = dims[i];
    b[i] = box[i];
    es[i] = 1;
    if (i + 1 < rank) st[i] = strides_bytes[i];
  }
  static const int promo = env_int("ASYNCEP_L2_PROMO", 256);
  const CUtensorMapL2promotion pr = promo == 0     ? CU_TENSOR_MAP_L2_PROMOTION_NONE
                                    : promo == 64  ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
                                    : promo == 128 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B
                                                   : CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
  const CUresult r = fn(map, dtype, (cuuint32_t)rank, const_cast<void*>(base), d, st, b, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, sw, pr, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

}  // namespace aep
