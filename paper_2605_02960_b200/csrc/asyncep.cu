// asyncep.cu -- the C ABI (include/asyncep.h): context, workspace carving, the
// double-buffered expert slot with its CUDA-event ordering, the NCCL AllGather
// ("MoE gatherer") and the four-step forward.
#include <dlfcn.h>
#include <link.h>

#include <cstdarg>
#include <cstdio>
#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "asyncep.h"
#include "common.cuh"
#include "kernels.cuh"

using aep::bf16;

namespace {

thread_local std::string g_last_error;

asyncep_status fail(asyncep_status st, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return st;
}

// The gather's transport primitives (asyncep_set_gather_transport):
//  ASYNCEP_GATHER_COPY_KERNEL: aep::launch_gather_copy, a copy kernel whose small CTAs co-reside
//    with the persistent GEMM CTAs (measured: the driver's same-device D2D memcpy stalls for the
//    whole duration of a persistent GEMM, profiles/copy_timeline.py);
//  ASYNCEP_GATHER_COPY_ENGINE: one cudaMemcpyAsync per chunk -- for IPC-mapped peer pointers on
//    another GPU the driver moves the bytes with the copy engines, no SMs.
// The default copy mode comes from ASYNCEP_GATHER_COPY (memcpy / ce: copy engine).
int default_copy_mode() {
  const char* e = getenv("ASYNCEP_GATHER_COPY");
  return (e && (!strcmp(e, "ce") || !strcmp(e, "memcpy"))) ? ASYNCEP_GATHER_COPY_ENGINE : ASYNCEP_GATHER_COPY_KERNEL;
}
// copy-kernel CTAs: ASYNCEP_GATHER_CTAS, else one per SM (asyncep_set_gather_copy_ctas at run time).
// Interleaved same-box A/B of the 8-rank emulation at 32K tokens/GPU (profiles/r02/interf_*.jsonl):
// one CTA per SM exposes 1.5-4.7 % (BF16) / 3.8-6.7 % (FP8) of the layer, two per SM 4.5-6.0 % /
// 7.6-9.3 % (GEMM2 +8 % beside them), 96 CTAs no better, 37 too few to keep the link rate.
int default_copy_ctas() {
  int dev = 0, n = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  const char* e = getenv("ASYNCEP_GATHER_CTAS");
  return (e && *e && atoi(e) > 0) ? atoi(e) : n;
}
cudaError_t gather_copy(void* dst, const void* src, size_t n, cudaStream_t st, uint64_t min_ns = 0,
                        int mode = ASYNCEP_GATHER_COPY_KERNEL, int ctas = 0) {
  if (mode == ASYNCEP_GATHER_COPY_KERNEL && ((uintptr_t)dst % 16 == 0) && ((uintptr_t)src % 16 == 0) && n % 16 == 0) {
    static const int dflt = default_copy_ctas();
    aep::launch_gather_copy(dst, src, n, ctas > 0 ? ctas : dflt, st, min_ns);
    return cudaGetLastError();
  }
  if (min_ns) aep::launch_spin_ns(min_ns, st);  // copy engine: link time, then the copy
  return cudaMemcpyAsync(dst, src, n, cudaMemcpyDefault, st);
}

// Swap-AB tail tiles of the grouped GEMMs (gemm_tc.cu): an expert's last 256-row tile holding at
// most this many rows runs with the weights as M and its tokens as N.  Same-process interleaved A/B
// (profiles/ab_flags.py, profiles/r02/swap/ab_swap_*.jsonl): FP8 GEMM1 gains (stack +0.7 % at 32K,
// +8 % at 16K, +23-25 % at 8K tokens/GPU); the FP8 down GEMM (short K) loses 5-8 % (and 1-4 % per
// step with the TMA-fed A, profiles/r02/swap_xperm/).  BF16 lost 0.5-1.7 % with the fused gather but
// gains 1.3-1.6 % per step (GEMM1 -2 to -4 %) since the dispatch is materialised (swap_xperm/, both
// A/B orders).  Defaults: 240 rows for both BF16 GEMMs and the FP8 GEMM1, the FP8 GEMM2 off.
// ASYNCEP_SWAP_MAX_BF16 / ASYNCEP_SWAP_MAX_FP8 / ASYNCEP_SWAP_MAX_F8G2 override (0 = off).
int env_rows(const char* name, int dflt) {
  const char* e = getenv(name);
  return (e && *e) ? atoi(e) : dflt;
}
int swap_max_rows(bool fp8, bool gemm2) {
  static const int b = env_rows("ASYNCEP_SWAP_MAX_BF16", 240);
  static const int f1 = env_rows("ASYNCEP_SWAP_MAX_FP8", 240);
  static const int f2 = env_rows("ASYNCEP_SWAP_MAX_F8G2", 0);
  return fp8 ? (gemm2 ? f2 : f1) : b;
}

// NVTX ranges around the host-side enqueue of each call (the paper's gated per-layer hooks,
// PAPER.md:650-655); free when no tool is attached.
struct NvtxRange {
  explicit NvtxRange(const char* fmt, int layer) {
    char b[64];
    snprintf(b, sizeof(b), fmt, layer);
    nvtxRangePushA(b);
  }
  ~NvtxRange() { nvtxRangePop(); }
};

}  // namespace

namespace aep {
// error reporting for the other translation units of the library (admission.cpp)
asyncep_status set_error(asyncep_status st, const char* msg) {
  g_last_error = msg;
  return st;
}
}  // namespace aep

namespace {

#define CUDA_TRY(expr)                                                                              \
  do {                                                                                              \
    cudaError_t _e = (expr);                                                                        \
    if (_e != cudaSuccess)                                                                          \
      return fail(ASYNCEP_ERR_CUDA, "%s failed: %s (%s:%d)", #expr, cudaGetErrorString(_e), __FILE__, \
                  __LINE__);                                                                        \
  } while (0)

// NCCL entry points, resolved in the running process (the caller's torch already loaded
// libnccl.so.2; we never link a second copy).
typedef int (*nccl_allgather_fn)(const void*, void*, size_t, int, void*, cudaStream_t);
typedef const char* (*nccl_errstr_fn)(int);
typedef int (*nccl_async_err_fn)(void*, int*);
typedef int (*nccl_p2p_fn)(const void*, size_t, int, int, void*, cudaStream_t);  // send: buf,count,type,peer
typedef int (*nccl_recv_fn)(void*, size_t, int, int, void*, cudaStream_t);
typedef int (*nccl_group_fn)();
struct NcclApi {
  nccl_allgather_fn allgather = nullptr;
  nccl_errstr_fn errstr = nullptr;
  nccl_async_err_fn async_err = nullptr;
  nccl_p2p_fn send = nullptr;
  nccl_recv_fn recv = nullptr;
  nccl_group_fn group_start = nullptr, group_end = nullptr;
};
// the path of the libnccl the process already loaded (torch's wheel copy), so we bind to the
// very library that created the borrowed communicator and never load a second NCCL
int find_nccl_cb(struct dl_phdr_info* info, size_t, void* data) {
  if (info->dlpi_name && strstr(info->dlpi_name, "libnccl.so")) {
    *static_cast<std::string*>(data) = info->dlpi_name;
    return 1;
  }
  return 0;
}
bool resolve_nccl(NcclApi& api) {
  std::string path;
  dl_iterate_phdr(find_nccl_cb, &path);
  void* h = path.empty() ? nullptr : dlopen(path.c_str(), RTLD_NOW | RTLD_NOLOAD);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
  if (!h) h = RTLD_DEFAULT;
  api.allgather = (nccl_allgather_fn)dlsym(h, "ncclAllGather");
  api.errstr = (nccl_errstr_fn)dlsym(h, "ncclGetErrorString");
  api.async_err = (nccl_async_err_fn)dlsym(h, "ncclCommGetAsyncError");
  api.send = (nccl_p2p_fn)dlsym(h, "ncclSend");
  api.recv = (nccl_recv_fn)dlsym(h, "ncclRecv");
  api.group_start = (nccl_group_fn)dlsym(h, "ncclGroupStart");
  api.group_end = (nccl_group_fn)dlsym(h, "ncclGroupEnd");
  return api.allgather != nullptr;
}
constexpr int kNcclUint8 = 1;
constexpr int kNcclInt32 = 2;

size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

struct WsLayout {
  size_t ids, w, dest, src_tok, blk, offsets, tile_start, counts, done, sched, xperm, act, total;
  size_t xq, xscale, amax, aq, ascale, asf;  // FP8 experts only (asf: MX scale chunks)
};
WsLayout ws_layout(const asyncep_config& c) {
  WsLayout L{};
  const size_t Tm = (size_t)c.max_tokens, k = (size_t)c.top_k, E = (size_t)c.num_experts;
  const size_t R = Tm * k;
  const size_t Rp = (size_t)aep::perm_rows((int64_t)Tm, (int)k, (int)E);  // padded permuted rows
  const size_t nblk = (Tm + aep::kPermTokensPerBlock - 1) / aep::kPermTokensPerBlock;
  size_t o = 0;
  auto take = [&](size_t bytes) {
    const size_t at = o;
    o = align_up(o + bytes, 256);
    return at;
  };
  L.ids = take(R * 4);
  L.w = take(R * 4);
  L.dest = take(R * 4);
  L.src_tok = take(Rp * 4);  // indexed by padded permuted row
  L.blk = take(nblk * E * 4);
  L.offsets = take((E + 1) * 4);
  L.tile_start = take((E + 1) * 4);
  L.counts = take(E * 4);
  L.done = take(4);
  L.sched = take(16);  // dynamic tile counters of the router / GEMM1 / GEMM2 launches
  L.xperm = take(Rp * (size_t)c.hidden * 2);  // X_perm, reused as Y_perm after GEMM1
  L.act = take(Rp * (size_t)c.ffn * 2);
  if (c.expert_dtype == ASYNCEP_FP8_E4M3) {
    L.xq = take(Rp * (size_t)c.hidden);
    L.xscale = take(Rp * 4);
    L.amax = take(Rp * 4);
    L.aq = take(Rp * (size_t)c.ffn);
    L.ascale = take(Rp * 4);
    L.asf = take(Rp * (size_t)c.ffn / 32);  // one E8M0 byte per 32 intermediate values
  }
  L.total = o;
  return L;
}

asyncep_status check_config(const asyncep_config* c) {
  if (!c) return fail(ASYNCEP_ERR_INVALID_ARG, "config is NULL");
  if (c->num_layers <= 0) return fail(ASYNCEP_ERR_INVALID_ARG, "num_layers must be > 0");
  if (c->num_experts <= 0 || c->num_experts > aep::kMaxExperts)
    return fail(ASYNCEP_ERR_INVALID_ARG, "num_experts must be in [1, %d]", aep::kMaxExperts);
  if (c->top_k <= 0 || c->top_k > c->num_experts || c->top_k > aep::kMaxTopK)
    return fail(ASYNCEP_ERR_INVALID_ARG, "top_k must be in [1, min(E, %d)]", aep::kMaxTopK);
  if (c->hidden <= 0 || c->hidden % 64) return fail(ASYNCEP_ERR_INVALID_ARG, "hidden must be a multiple of 64");
  if (c->hidden >= 256 && c->hidden % 256)
    return fail(ASYNCEP_ERR_INVALID_ARG, "hidden >= 256 must be a multiple of 256");
  if (c->ffn <= 0 || c->ffn % 128) return fail(ASYNCEP_ERR_INVALID_ARG, "ffn must be a multiple of 128");
  if (c->expert_dtype != ASYNCEP_BF16 && c->expert_dtype != ASYNCEP_FP8_E4M3)
    return fail(ASYNCEP_ERR_UNSUPPORTED, "expert_dtype %d not supported by this build", c->expert_dtype);
  if ((c->flags & ASYNCEP_FLAG_MX_ACT) && c->expert_dtype != ASYNCEP_FP8_E4M3)
    return fail(ASYNCEP_ERR_INVALID_ARG, "ASYNCEP_FLAG_MX_ACT needs FP8 experts");
  if (c->expert_dtype == ASYNCEP_FP8_E4M3 && (c->flags & ASYNCEP_FLAG_SIMT_GEMM))
    return fail(ASYNCEP_ERR_UNSUPPORTED, "the SIMT reference GEMM is BF16 only");
  if (c->expert_dtype == ASYNCEP_FP8_E4M3 && c->hidden < 256)
    return fail(ASYNCEP_ERR_UNSUPPORTED, "FP8 experts need hidden >= 256");
  if (c->world_size <= 0 || c->rank < 0 || c->rank >= c->world_size)
    return fail(ASYNCEP_ERR_INVALID_ARG, "bad world_size/rank");
  if (c->num_experts % c->world_size)
    return fail(ASYNCEP_ERR_INVALID_ARG, "num_experts (%d) %% world_size (%d) != 0", c->num_experts,
                c->world_size);
  if (c->max_tokens <= 0 || (int64_t)c->max_tokens * c->top_k >= (int64_t)1 << 31)
    return fail(ASYNCEP_ERR_INVALID_ARG, "max_tokens out of range");
  if (!(c->gamma >= 1.0f)) return fail(ASYNCEP_ERR_INVALID_ARG, "gamma must be >= 1");
  return ASYNCEP_OK;
}

constexpr int kStages = 6;
constexpr int kEventsPerFwd = kStages + 1;
constexpr int kMaxPendingFwd = 512;

}  // namespace

struct asyncep_ctx {
  asyncep_config cfg;
  void* comm = nullptr;
  void* gather_comm = nullptr;  // communicator of the NCCL gather (default: comm)
  NcclApi nccl;
  cudaStream_t cs = nullptr, ms = nullptr;
  std::vector<const void*> router_w, shard;
  void* slot[2] = {nullptr, nullptr};
  uint8_t* ws = nullptr;
  WsLayout L;
  size_t expert_bytes = 0, slot_bytes = 0, shard_bytes = 0;
  int num_sms = 148;
  int dev_sms = 148;
  int transport = -1;  // ASYNCEP_GATHER_*; -1: copy (default mode) when peer shards are set, else NCCL
  int copy_mode = ASYNCEP_GATHER_COPY_KERNEL;
  int copy_ctas = 0;  // 0: default_copy_ctas()
  // slot bookkeeping (host side): layer held / being gathered, and whether its forward ran
  int slot_layer[2] = {-1, -1};
  bool slot_consumed[2] = {true, true};
  cudaEvent_t ag_done[2] = {nullptr, nullptr}, slot_free[2] = {nullptr, nullptr};
  // tcgen05 tensor maps
  aep::ActMaps act_maps;
  std::vector<aep::GemmMaps> layer_maps;  // per resident layer (index l), valid if resident[l]
  std::vector<aep::GemmMaps> own_maps;    // per gathered layer: maps over this rank's own shard
  std::vector<char> resident;
  aep::GemmMaps slot_maps[2];
  std::vector<aep::RouterTc> router_maps;  // per layer
  // stage timing
  std::vector<cudaEvent_t> ev_pool;  // ring of kMaxPendingFwd forwards x kEventsPerFwd events
  int ev_head = 0;  // ring slot of the oldest pending (recorded, not yet read) forward
  int ev_used = 0;  // pending forwards
  double stage_ms[kStages] = {0};
  int64_t fwd_count = 0;
  std::vector<int32_t> ev_layer;                 // layer of the forward in each ring slot
  std::vector<std::pair<int32_t, double>> recent;  // (layer, total ms) of flushed forwards
  // event timeline (asyncep_timeline_begin / _read): epoch on both streams, then per forward
  // (start, dispatch done, GEMM1 start = after the slot wait, end) and per gather (start, end),
  // ms since the epoch
  cudaEvent_t epoch = nullptr;
  bool timeline = false;
  std::vector<asyncep_timeline_rec> tl;                          // flushed records
  std::vector<std::pair<int32_t, std::pair<cudaEvent_t, cudaEvent_t>>> tl_gather;  // pending gathers
  int64_t launches = 0;
  double link_bps = 0.0;  // prefetch_layer_local pacing (0 = off)
  // asyncep_set_gather_gate: prefetches are held on the host (pending) and enqueued by the next
  // forward at its gate point -- after its dispatch -- with the comm stream waiting on gate_ev there
  struct PendingGather {
    int32_t layer;
    std::vector<const void*> shards;  // empty: peer shards / NCCL
  };
  std::vector<PendingGather> pending;
  cudaEvent_t gate_ev = nullptr;
  bool gate_on = false, probing = false, flushing = false;
  std::vector<const void*> peer;  // P2P gather: [layer * N + rank] peer-mapped shard pointers (empty: NCCL)
  std::vector<aep::GemmMaps> ep_maps;  // EP contrast: maps over this rank's shard of each layer
  std::vector<char> ep_maps_ok;
  // NEXT-2 offload: host backing store + w-deep device window
  bool offload = false;
  int w = 0;
  cudaStream_t hs = nullptr;
  std::vector<const void*> host_shard;
  std::vector<void*> window;
  std::vector<cudaEvent_t> h2d_done, win_free;
  std::vector<int> win_layer;
  std::vector<char> win_consumed;
  std::vector<aep::GemmMaps> win_maps;  // world_size == 1: the forward reads the window
};

namespace {

bool layer_resident(const asyncep_ctx* c, int l) {
  return c->cfg.world_size == 1 || (l == 0 && c->cfg.replicate_layer0);
}

// An asynchronous NCCL fault (a peer died, a network error) surfaces at the next call instead of
// as a hang (ncclCommGetAsyncError; ncclInProgress = 7 is not an error).
asyncep_status check_nccl_async(asyncep_ctx* c) {
  if (!c->nccl.async_err) return ASYNCEP_OK;
  for (void* comm : {c->comm, c->gather_comm}) {
    if (!comm) continue;
    int e = 0;
    const int r = c->nccl.async_err(comm, &e);
    if (r == 0 && (e == 0 || e == 7)) continue;
    const int code = r ? r : e;
    return fail(ASYNCEP_ERR_NCCL, "NCCL asynchronous error on a borrowed communicator: %s (%d)",
                c->nccl.errstr ? c->nccl.errstr(code) : "?", code);
  }
  return ASYNCEP_OK;
}

// the gather transport a prefetch uses
int gather_transport(const asyncep_ctx* c) {
  if (c->transport >= 0) return c->transport;
  return c->peer.empty() ? ASYNCEP_GATHER_NCCL : c->copy_mode;
}

// Reads the pending forwards' events oldest first.  blocking = false (the forward path when the
// ring is full): wait only for the OLDEST forward to finish, then read every forward that has
// already completed -- the host never drains the GPU queue, it just stays <= kMaxPendingFwd
// forwards ahead.  blocking = true (the query calls): wait for all of them.
asyncep_status flush_timing(asyncep_ctx* c, bool blocking = true) {
  bool first = true;
  while (c->ev_used > 0) {
    cudaEvent_t* e = &c->ev_pool[(size_t)c->ev_head * kEventsPerFwd];
    if (blocking || first) {
      CUDA_TRY(cudaEventSynchronize(e[kStages]));
    } else {
      const cudaError_t q = cudaEventQuery(e[kStages]);
      if (q == cudaErrorNotReady) break;
      CUDA_TRY(q);
    }
    first = false;
    for (int s = 0; s < kStages; ++s) {
      float ms = 0.f;
      CUDA_TRY(cudaEventElapsedTime(&ms, e[s], e[s + 1]));
      c->stage_ms[s] += ms;
    }
    float tot = 0.f;
    CUDA_TRY(cudaEventElapsedTime(&tot, e[0], e[kStages]));
    c->recent.emplace_back(c->ev_layer[(size_t)c->ev_head], (double)tot);
    if (c->timeline && c->epoch) {
      float t0 = 0.f, t2 = 0.f, t3 = 0.f, t6 = 0.f;
      CUDA_TRY(cudaEventElapsedTime(&t0, c->epoch, e[0]));
      CUDA_TRY(cudaEventElapsedTime(&t2, c->epoch, e[2]));
      CUDA_TRY(cudaEventElapsedTime(&t3, c->epoch, e[3]));
      CUDA_TRY(cudaEventElapsedTime(&t6, c->epoch, e[kStages]));
      c->tl.push_back(asyncep_timeline_rec{ASYNCEP_TL_FORWARD, c->ev_layer[(size_t)c->ev_head], t0, t2, t3, t6});
    }
    if (c->recent.size() > 4096) c->recent.erase(c->recent.begin(), c->recent.begin() + 2048);
    c->ev_head = (c->ev_head + 1) % kMaxPendingFwd;
    --c->ev_used;
    ++c->fwd_count;
  }
  return ASYNCEP_OK;
}

}  // namespace

extern "C" {

int32_t asyncep_abi_version(void) { return ASYNCEP_ABI_VERSION; }
const char* asyncep_last_error(void) { return g_last_error.c_str(); }

size_t asyncep_expert_bytes(const asyncep_config* c) {
  if (!c) return 0;
  if (c->expert_dtype == ASYNCEP_FP8_E4M3)  // codes + per-row fp32 scales of W_gu (2h) and W_down (H)
    return (size_t)3 * c->hidden * c->ffn + (size_t)(2 * c->ffn + c->hidden) * 4;
  return (size_t)3 * c->hidden * c->ffn * 2;
}
size_t asyncep_slot_bytes(const asyncep_config* c) {
  return c ? asyncep_expert_bytes(c) * (size_t)c->num_experts : 0;
}
size_t asyncep_shard_bytes(const asyncep_config* c) {
  return (c && c->world_size > 0) ? asyncep_expert_bytes(c) * (size_t)(c->num_experts / c->world_size) : 0;
}
size_t asyncep_workspace_size(const asyncep_config* c) {
  if (check_config(c) != ASYNCEP_OK) return 0;
  return ws_layout(*c).total;
}

asyncep_status asyncep_pack_experts(const asyncep_config* cfg, int32_t count, const void* gate, const void* up,
                                    const void* down, const float* gs, const float* us, const float* ds, void* out,
                                    void* stream) {
  asyncep_status st = check_config(cfg);
  if (st) return st;
  if (count < 0 || count > cfg->num_experts) return fail(ASYNCEP_ERR_INVALID_ARG, "bad expert count");
  if (count == 0) return ASYNCEP_OK;
  if (!gate || !up || !down || !out) return fail(ASYNCEP_ERR_INVALID_ARG, "null pointer");
  if (((uintptr_t)gate | (uintptr_t)up | (uintptr_t)down | (uintptr_t)out) & 15)
    return fail(ASYNCEP_ERR_INVALID_ARG, "pointers must be 16-B aligned");
  if (cfg->expert_dtype == ASYNCEP_FP8_E4M3) {
    if (!gs || !us || !ds) return fail(ASYNCEP_ERR_INVALID_ARG, "FP8 packing needs the three scale arrays");
    aep::launch_pack_fp8((const uint8_t*)gate, (const uint8_t*)up, (const uint8_t*)down, gs, us, ds, count,
                         cfg->hidden, cfg->ffn, asyncep_expert_bytes(cfg), (uint8_t*)out, (cudaStream_t)stream);
  } else {
    if (gs || us || ds) return fail(ASYNCEP_ERR_INVALID_ARG, "scales must be NULL for BF16");
    aep::launch_pack_bf16((const bf16*)gate, (const bf16*)up, (const bf16*)down, count, cfg->hidden, cfg->ffn,
                          asyncep_expert_bytes(cfg), (uint8_t*)out, (cudaStream_t)stream);
  }
  CUDA_TRY(cudaGetLastError());
  return ASYNCEP_OK;
}

asyncep_status asyncep_init(const asyncep_config* cfg, void* nccl_comm, void* compute_stream, void* comm_stream,
                            const void* const* router_w, const void* const* expert_shard, void* slot0,
                            void* slot1, void* workspace, asyncep_ctx** out) {
  asyncep_status st = check_config(cfg);
  if (st) return st;
  if (!out || !router_w || !expert_shard || !workspace) return fail(ASYNCEP_ERR_INVALID_ARG, "null pointer");
  *out = nullptr;
  if ((uintptr_t)workspace & 255) return fail(ASYNCEP_ERR_INVALID_ARG, "workspace must be 256-B aligned");
  const int L = cfg->num_layers;
  const bool offload = (cfg->flags & ASYNCEP_FLAG_OFFLOAD) != 0;
  for (int l = 0; l < L; ++l) {
    // offloaded layers (every layer >= 1 at N == 1, every gathered layer at N > 1) live on the host
    const bool host_only = offload && (cfg->world_size == 1 ? l > 0 : !(l == 0 && cfg->replicate_layer0));
    if (!router_w[l] || (!expert_shard[l] && !host_only))
      return fail(ASYNCEP_ERR_INVALID_ARG, "null weight pointer (layer %d)", l);
    if (((uintptr_t)router_w[l] | (uintptr_t)expert_shard[l]) & 15)
      return fail(ASYNCEP_ERR_INVALID_ARG, "weights must be 16-B aligned (layer %d)", l);
  }
  int dev = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  cudaDeviceProp prop;
  CUDA_TRY(cudaGetDeviceProperties(&prop, dev));
  if (prop.major != 10) return fail(ASYNCEP_ERR_UNSUPPORTED, "device is sm_%d%d; this library is sm_100a", prop.major, prop.minor);

  asyncep_ctx* c = new asyncep_ctx();
  c->cfg = *cfg;
  c->cs = (cudaStream_t)compute_stream;
  c->ms = (cudaStream_t)comm_stream;
  c->num_sms = prop.multiProcessorCount;
  c->dev_sms = prop.multiProcessorCount;
  c->copy_mode = default_copy_mode();
  if (cfg->world_size > 1) {  // leave SMs to NCCL's AllGather kernels (persistent GEMMs fill every SM)
    const char* rs = getenv("ASYNCEP_RESERVE_SMS");
    const int reserve = rs && *rs ? atoi(rs) : 0;
    if (reserve > 0 && reserve < c->num_sms - 2) c->num_sms -= reserve & ~1;
  }
  c->router_w.assign(router_w, router_w + L);
  c->shard.assign(expert_shard, expert_shard + L);
  c->ws = (uint8_t*)workspace;
  c->L = ws_layout(*cfg);
  c->expert_bytes = asyncep_expert_bytes(cfg);
  c->slot_bytes = asyncep_slot_bytes(cfg);
  c->shard_bytes = asyncep_shard_bytes(cfg);
  auto bail = [&](asyncep_status s) {
    asyncep_destroy(c);
    return s;
  };
  if (cfg->world_size > 1) {
    if (!slot0 || !slot1 || ((uintptr_t)slot0 | (uintptr_t)slot1) & 15)
      return bail(fail(ASYNCEP_ERR_INVALID_ARG, "world_size > 1 needs two 16-B aligned slots"));
    if (!c->ms) return bail(fail(ASYNCEP_ERR_INVALID_ARG, "world_size > 1 needs a comm stream"));
    c->slot[0] = slot0;
    c->slot[1] = slot1;
    c->comm = nccl_comm;
    if (nccl_comm && !resolve_nccl(c->nccl))
      return bail(fail(ASYNCEP_ERR_NCCL, "ncclAllGather not found in the process (load torch's NCCL first)"));
  } else if (nccl_comm) {
    c->comm = nccl_comm;
    if (!resolve_nccl(c->nccl)) return bail(fail(ASYNCEP_ERR_NCCL, "ncclAllGather not found in the process"));
  }
  for (int i = 0; i < 2; ++i) {
    if (cudaEventCreateWithFlags(&c->ag_done[i], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->slot_free[i], cudaEventDisableTiming) != cudaSuccess)
      return bail(fail(ASYNCEP_ERR_CUDA, "cudaEventCreate failed"));
  }
  const bool fp8 = cfg->expert_dtype == ASYNCEP_FP8_E4M3;
  const int64_t Rp = aep::perm_rows(cfg->max_tokens, cfg->top_k, cfg->num_experts);
  if (cudaMemsetAsync(c->ws + c->L.done, 0, 4, c->cs) != cudaSuccess ||
      (fp8 && cudaMemsetAsync(c->ws + c->L.amax, 0, (size_t)Rp * 4, c->cs) != cudaSuccess))
    return bail(fail(ASYNCEP_ERR_CUDA, "cudaMemsetAsync failed"));
  // TMA descriptors: activations (fixed workspace addresses), each resident layer, both slots.
  const int64_t R = aep::perm_rows(cfg->max_tokens, cfg->top_k, cfg->num_experts);
  if (!aep::make_act_maps(c->act_maps, (const bf16*)(c->ws + c->L.xperm), (const bf16*)(c->ws + c->L.act), R,
                          cfg->hidden, cfg->ffn, fp8 ? c->ws + c->L.xq : nullptr, fp8 ? c->ws + c->L.aq : nullptr,
                          fp8 ? (const uint32_t*)(c->ws + c->L.asf) : nullptr))
    return bail(fail(ASYNCEP_ERR_CUDA, "cuTensorMapEncodeTiled failed (activations)"));
  c->layer_maps.resize(L);
  c->resident.assign(L, 0);
  for (int l = 0; l < L; ++l) {
    if (!layer_resident(c, l) || !c->shard[l]) continue;
    c->resident[l] = 1;
    if (!aep::make_weight_maps(c->layer_maps[l], c->shard[l], c->expert_bytes, cfg->num_experts, cfg->hidden,
                               cfg->ffn, c->act_maps.bn2, fp8))
      return bail(fail(ASYNCEP_ERR_CUDA, "cuTensorMapEncodeTiled failed (layer %d)", l));
  }
  // gathered layers: the GEMMs read this rank's own experts straight from its shard
  c->own_maps.resize(L);
  for (int l = 0; l < L; ++l) {
    if (layer_resident(c, l) || !c->shard[l]) continue;
    if (!aep::make_weight_maps(c->own_maps[l], c->shard[l], c->expert_bytes, cfg->num_experts / cfg->world_size,
                               cfg->hidden, cfg->ffn, c->act_maps.bn2, fp8))
      return bail(fail(ASYNCEP_ERR_CUDA, "cuTensorMapEncodeTiled failed (own shard %d)", l));
  }
  c->router_maps.resize(L);
  for (int l = 0; l < L; ++l)
    if (!aep::make_router_wmap(c->router_maps[l], (const bf16*)c->router_w[l], cfg->hidden, cfg->num_experts))
      return bail(fail(ASYNCEP_ERR_CUDA, "cuTensorMapEncodeTiled failed (router %d)", l));
  for (int i = 0; i < 2; ++i)
    if (c->slot[i] && !aep::make_weight_maps(c->slot_maps[i], c->slot[i], c->expert_bytes, cfg->num_experts,
                                             cfg->hidden, cfg->ffn, c->act_maps.bn2, fp8))
      return bail(fail(ASYNCEP_ERR_CUDA, "cuTensorMapEncodeTiled failed (slot %d)", i));
  *out = c;
  return ASYNCEP_OK;
}

static asyncep_status prefetch_common(asyncep_ctx* c, int32_t layer, const void* const* shards) {
  if (!c) return fail(ASYNCEP_ERR_INVALID_ARG, "ctx is NULL");
  if (layer < 0 || layer >= c->cfg.num_layers) return fail(ASYNCEP_ERR_INVALID_ARG, "layer out of range");
  if (layer_resident(c, layer)) return ASYNCEP_OK;
  NvtxRange nv("asyncep_gather L%d", layer);
  if (asyncep_status e = check_nccl_async(c)) return e;
  const int tr = gather_transport(c);
  const int s = layer % 2;
  if (!c->slot_consumed[s] && c->slot_layer[s] != layer)
    return fail(ASYNCEP_ERR_INVALID_ARG,
                "slot %d still holds layer %d whose forward has not been issued (at most 2 layers in flight)", s,
                c->slot_layer[s]);
  // gated: held until the next forward's gate point, after its HBM-bound dispatch (the grouped GEMMs
  // then hide the gather, instead of the combine / router / dispatch); the slot is
  // claimed now, so the forward's checks see the layer as prefetched
  if (c->gate_on && !c->probing && !c->flushing) {
    asyncep_ctx::PendingGather p{layer, {}};
    if (shards) p.shards.assign(shards, shards + c->cfg.world_size);
    c->pending.push_back(std::move(p));
    c->slot_layer[s] = layer;
    c->slot_consumed[s] = false;
    return ASYNCEP_OK;
  }
  // WAR: the slot's previous occupant must have finished its GEMMs.
  CUDA_TRY(cudaStreamWaitEvent(c->ms, c->slot_free[s], 0));
  const void* own = c->shard[layer];
  int wi = -1;
  if (c->offload) {  // the own shard comes from the H2D window (staged by asyncep_stage_layer)
    wi = layer % c->w;
    if (c->win_layer[wi] != layer || c->win_consumed[wi])
      return fail(ASYNCEP_ERR_NOT_PREFETCHED, "layer %d was not staged (asyncep_stage_layer)", layer);
    CUDA_TRY(cudaStreamWaitEvent(c->ms, c->h2d_done[wi], 0));
    own = c->window[wi];
  }
  // timeline events of this gather, released on every early return (kept on success)
  struct TlEvents {
    cudaEvent_t a = nullptr, b = nullptr;
    ~TlEvents() {
      if (a) cudaEventDestroy(a);
      if (b) cudaEventDestroy(b);
    }
  } tg;
  if (c->timeline) {
    CUDA_TRY(cudaEventCreate(&tg.a));
    CUDA_TRY(cudaEventCreate(&tg.b));
    CUDA_TRY(cudaEventRecord(tg.a, c->ms));
  }
  if (!shards && tr != ASYNCEP_GATHER_NCCL) {  // P2P gather over the IPC-mapped peer shards
    if (c->peer.empty()) return fail(ASYNCEP_ERR_INVALID_ARG, "copy transport without peer shards (asyncep_set_peer_shards)");
    shards = c->peer.data() + (size_t)layer * c->cfg.world_size;
  }
  if (shards) {
    const int mode = tr == ASYNCEP_GATHER_NCCL ? c->copy_mode : tr;  // local shards (emulation): a copy
    // copy-engine gather: the N - 1 peer shards (then the own one), each rank starting at its
    // right-hand neighbour so that the N readers of a shard are spread over time
    constexpr size_t kChunk = (size_t)64 << 20;
    const int N = c->cfg.world_size;
    for (int i = 1; i <= N; ++i) {
      const int r = (c->cfg.rank + i) % N;
      if (!shards[r]) return fail(ASYNCEP_ERR_INVALID_ARG, "null shard %d", r);
      // the tcgen05 GEMMs read the own shard in place (the SIMT debug GEMM reads the whole slot)
      if (r == c->cfg.rank && !c->offload && !(c->cfg.flags & ASYNCEP_FLAG_SIMT_GEMM)) continue;
      uint8_t* dst = (uint8_t*)c->slot[s] + (size_t)r * c->shard_bytes;
      const uint8_t* src = (const uint8_t*)(r == c->cfg.rank && c->offload ? own : shards[r]);
      const bool paced = c->link_bps > 0 && r != c->cfg.rank;  // own shard is a local copy
      for (size_t o = 0; o < c->shard_bytes; o += kChunk) {
        const size_t n = std::min(kChunk, c->shard_bytes - o);
        CUDA_TRY(gather_copy(dst + o, src + o, n, c->ms, paced ? (uint64_t)((double)n / c->link_bps * 1e9) : 0,
                             mode, c->copy_ctas));
        c->launches += 1;
      }
    }
  } else {
    void* gcomm = c->gather_comm ? c->gather_comm : c->comm;
    if (!gcomm) return fail(ASYNCEP_ERR_NCCL, "no NCCL communicator (use asyncep_prefetch_layer_local)");
    const int r = c->nccl.allgather(own, c->slot[s], c->shard_bytes, kNcclUint8, gcomm, c->ms);
    if (r != 0)
      return fail(ASYNCEP_ERR_NCCL, "ncclAllGather: %s", c->nccl.errstr ? c->nccl.errstr(r) : "error");
  }
  CUDA_TRY(cudaEventRecord(c->ag_done[s], c->ms));
  if (tg.b) {
    CUDA_TRY(cudaEventRecord(tg.b, c->ms));
    c->tl_gather.push_back({layer, {tg.a, tg.b}});
    tg.a = tg.b = nullptr;  // owned by the context now
  }
  if (wi >= 0) {  // the gather has read the window buffer: it may be re-staged
    CUDA_TRY(cudaEventRecord(c->win_free[wi], c->ms));
    c->win_consumed[wi] = true;
  }
  c->slot_layer[s] = layer;
  c->slot_consumed[s] = false;
  return ASYNCEP_OK;
}

asyncep_status asyncep_enable_offload(asyncep_ctx* c, const void* const* host_shards, void* const* window, int32_t w,
                                      void* h2d_stream) {
  if (!c || !host_shards || !window || w < 1 || !h2d_stream) return fail(ASYNCEP_ERR_INVALID_ARG, "bad arguments");
  if (c->offload) return fail(ASYNCEP_ERR_INVALID_ARG, "offload already enabled");
  const asyncep_config& cf = c->cfg;
  const size_t bytes = cf.world_size == 1 ? c->slot_bytes : c->shard_bytes;
  c->host_shard.assign(cf.num_layers, nullptr);
  for (int l = 0; l < cf.num_layers; ++l) {
    const bool needs = cf.world_size == 1 ? l > 0 : !layer_resident(c, l);
    if (needs && !host_shards[l]) return fail(ASYNCEP_ERR_INVALID_ARG, "null host shard (layer %d)", l);
    c->host_shard[l] = host_shards[l];
  }
  c->window.assign(window, window + w);
  for (int i = 0; i < w; ++i)
    if (!window[i] || ((uintptr_t)window[i] & 15)) return fail(ASYNCEP_ERR_INVALID_ARG, "bad window buffer %d", i);
  c->h2d_done.assign(w, nullptr);
  c->win_free.assign(w, nullptr);
  for (int i = 0; i < w; ++i) {
    CUDA_TRY(cudaEventCreateWithFlags(&c->h2d_done[i], cudaEventDisableTiming));
    CUDA_TRY(cudaEventCreateWithFlags(&c->win_free[i], cudaEventDisableTiming));
  }
  c->win_layer.assign(w, -1);
  c->win_consumed.assign(w, 1);
  if (cf.world_size == 1) {
    c->win_maps.resize(w);
    for (int i = 0; i < w; ++i)
      if (!aep::make_weight_maps(c->win_maps[i], window[i], c->expert_bytes, cf.num_experts, cf.hidden, cf.ffn,
                                 c->act_maps.bn2, cf.expert_dtype == ASYNCEP_FP8_E4M3))
        return fail(ASYNCEP_ERR_CUDA, "cuTensorMapEncodeTiled failed (window %d)", i);
  }
  c->w = w;
  c->hs = (cudaStream_t)h2d_stream;
  c->offload = true;
  (void)bytes;
  return ASYNCEP_OK;
}

asyncep_status asyncep_stage_layer(asyncep_ctx* c, int32_t layer) {
  if (!c || !c->offload) return fail(ASYNCEP_ERR_INVALID_ARG, "offload not enabled");
  if (layer < 0 || layer >= c->cfg.num_layers) return fail(ASYNCEP_ERR_INVALID_ARG, "layer out of range");
  const bool n1 = c->cfg.world_size == 1;
  if (n1 ? layer == 0 : layer_resident(c, layer)) return ASYNCEP_OK;  // resident: nothing to stage
  const int i = layer % c->w;
  if (!c->win_consumed[i] && c->win_layer[i] != layer)
    return fail(ASYNCEP_ERR_INVALID_ARG, "window %d still holds layer %d, not yet consumed", i, c->win_layer[i]);
  CUDA_TRY(cudaStreamWaitEvent(c->hs, c->win_free[i], 0));  // WAR vs the previous occupant's reader
  CUDA_TRY(cudaMemcpyAsync(c->window[i], c->host_shard[layer], n1 ? c->slot_bytes : c->shard_bytes,
                           cudaMemcpyHostToDevice, c->hs));
  CUDA_TRY(cudaEventRecord(c->h2d_done[i], c->hs));
  c->win_layer[i] = layer;
  c->win_consumed[i] = false;
  return ASYNCEP_OK;
}

asyncep_status asyncep_prefetch_layer(asyncep_ctx* c, int32_t layer) { return prefetch_common(c, layer, nullptr); }

asyncep_status asyncep_prefetch_layer_local(asyncep_ctx* c, int32_t layer, const void* const* shards) {
  if (!c) return fail(ASYNCEP_ERR_INVALID_ARG, "ctx is NULL");
  if (c->cfg.world_size < 2) return fail(ASYNCEP_ERR_INVALID_ARG, "prefetch_layer_local needs world_size > 1");
  if (!shards) return fail(ASYNCEP_ERR_INVALID_ARG, "shards is NULL");
  return prefetch_common(c, layer, shards);
}

asyncep_status asyncep_set_peer_shards(asyncep_ctx* c, const void* const* shards) {
  if (!c) return fail(ASYNCEP_ERR_INVALID_ARG, "ctx is NULL");
  const int L = c->cfg.num_layers, N = c->cfg.world_size;
  if (!shards) {
    c->peer.clear();
    return ASYNCEP_OK;
  }
  if (N < 2) return fail(ASYNCEP_ERR_INVALID_ARG, "peer shards need world_size > 1");
  for (int l = 0; l < L; ++l)
    for (int r = 0; r < N; ++r)
      if (!layer_resident(c, l) && (!shards[(size_t)l * N + r] || ((uintptr_t)shards[(size_t)l * N + r] & 15)))
        return fail(ASYNCEP_ERR_INVALID_ARG, "peer shard (layer %d, rank %d) is null or misaligned", l, r);
  c->peer.assign(shards, shards + (size_t)L * N);
  return ASYNCEP_OK;
}

asyncep_status asyncep_set_gather_transport(asyncep_ctx* c, int32_t transport, int32_t reserve_sms) {
  if (!c) return fail(ASYNCEP_ERR_INVALID_ARG, "ctx is NULL");
  if (transport < -1 || transport > ASYNCEP_GATHER_NCCL)
    return fail(ASYNCEP_ERR_INVALID_ARG, "unknown gather transport %d", transport);
  if (transport == ASYNCEP_GATHER_NCCL && !c->comm && !c->gather_comm)
    return fail(ASYNCEP_ERR_NCCL, "NCCL transport without a communicator");
  if (reserve_sms < 0 || reserve_sms >= c->dev_sms - 2)
    return fail(ASYNCEP_ERR_INVALID_ARG, "reserve_sms %d out of range", reserve_sms);
  c->transport = transport;
  if (transport == ASYNCEP_GATHER_COPY_KERNEL || transport == ASYNCEP_GATHER_COPY_ENGINE) c->copy_mode = transport;
  c->num_sms = c->dev_sms - (reserve_sms & ~1);  // the grouped GEMMs' persistent grid (CTA pairs)
  return ASYNCEP_OK;
}

asyncep_status asyncep_set_gather_comm(asyncep_ctx* c, void* nccl_comm) {
  if (!c) return fail(ASYNCEP_ERR_INVALID_ARG, "ctx is NULL");
  if (nccl_comm && !c->nccl.allgather && !resolve_nccl(c->nccl))
    return fail(ASYNCEP_ERR_NCCL, "ncclAllGather not found in the process");
  c->gather_comm = nccl_comm;
  return ASYNCEP_OK;
}

asyncep_status asyncep_set_gather_copy_ctas(asyncep_ctx* c, int32_t ctas) {
  if (!c || ctas < 0) return fail(ASYNCEP_ERR_INVALID_ARG, "bad arguments");
  c->copy_ctas = ctas;
  return ASYNCEP_OK;
}

asyncep_status asyncep_probe_gather(asyncep_ctx* c, int32_t layer, const void* const* shards, double* ms_out,
                                    double* bytes_out) {
  if (!c) return fail(ASYNCEP_ERR_INVALID_ARG, "ctx is NULL");
  if (c->cfg.world_size < 2) return fail(ASYNCEP_ERR_INVALID_ARG, "probe_gather needs world_size > 1");
  if (layer < 0 || layer >= c->cfg.num_layers || layer_resident(c, layer))
    return fail(ASYNCEP_ERR_INVALID_ARG, "probe_gather: layer %d is not a gathered layer", layer);
  const int s = layer % 2;
  if (!c->slot_consumed[s]) return fail(ASYNCEP_ERR_INVALID_ARG, "probe_gather: slot %d is in use", s);
  cudaEvent_t e0, e1;
  CUDA_TRY(cudaEventCreate(&e0));
  CUDA_TRY(cudaEventCreate(&e1));
  CUDA_TRY(cudaStreamWaitEvent(c->ms, c->slot_free[s], 0));
  CUDA_TRY(cudaEventRecord(e0, c->ms));
  c->probing = true;  // the probe's gather runs alone: never gated
  asyncep_status st = prefetch_common(c, layer, shards);
  c->probing = false;
  if (st == ASYNCEP_OK) {
    CUDA_TRY(cudaEventRecord(e1, c->ms));
    CUDA_TRY(cudaEventSynchronize(e1));
    float ms = 0.f;
    CUDA_TRY(cudaEventElapsedTime(&ms, e0, e1));
    // the slot held the layer but no forward read it: hand it back (same stream orders the next fill)
    c->slot_consumed[s] = true;
    CUDA_TRY(cudaEventRecord(c->slot_free[s], c->ms));
    if (ms_out) *ms_out = ms;
    // bytes each rank receives: the N - 1 peer shards
    if (bytes_out) *bytes_out = (double)(c->cfg.world_size - 1) * (double)c->shard_bytes;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return st;
}

asyncep_status asyncep_gather_copy(void* dst, const void* src, size_t bytes, void* stream) {
  if ((!dst || !src) && bytes) return fail(ASYNCEP_ERR_INVALID_ARG, "null pointer");
  if (!bytes) return ASYNCEP_OK;
  CUDA_TRY(gather_copy(dst, src, bytes, (cudaStream_t)stream));
  return ASYNCEP_OK;
}

// Enqueue the held (gated) gathers; gated: the comm stream first waits for gate_stream (which may be
// the legacy default stream, handle 0) to reach this point.
static asyncep_status flush_pending(asyncep_ctx* c, bool gated, cudaStream_t gate_stream) {
  if (c->pending.empty()) return ASYNCEP_OK;
  if (gated) {
    if (!c->gate_ev) CUDA_TRY(cudaEventCreateWithFlags(&c->gate_ev, cudaEventDisableTiming));
    CUDA_TRY(cudaEventRecord(c->gate_ev, gate_stream));
    CUDA_TRY(cudaStreamWaitEvent(c->ms, c->gate_ev, 0));
  }
  std::vector<asyncep_ctx::PendingGather> todo;
  todo.swap(c->pending);
  c->flushing = true;
  asyncep_status st = ASYNCEP_OK;
  for (auto& p : todo) {
    st = prefetch_common(c, p.layer, p.shards.empty() ? nullptr : p.shards.data());
    if (st) break;
  }
  c->flushing = false;
  return st;
}

asyncep_status asyncep_set_gather_gate(asyncep_ctx* c, int32_t on) {
  if (!c) return fail(ASYNCEP_ERR_INVALID_ARG, "ctx is NULL");
  c->gate_on = on != 0;
  if (!c->gate_on) return flush_pending(c, false, nullptr);  // held gathers start now
  return ASYNCEP_OK;
}

asyncep_status asyncep_set_link_emulation(asyncep_ctx* c, double bytes_per_s) {
  if (!c || bytes_per_s < 0) return fail(ASYNCEP_ERR_INVALID_ARG, "bad arguments");
  c->link_bps = bytes_per_s;
  return ASYNCEP_OK;
}

asyncep_status asyncep_moe_forward(asyncep_ctx* c, int32_t layer, const void* x, int64_t T, const void* residual,
                                   void* y, int32_t* ids_out, float* w_out, int32_t* counts_out) {
  if (!c) return fail(ASYNCEP_ERR_INVALID_ARG, "ctx is NULL");
  const asyncep_config& cf = c->cfg;
  if (layer < 0 || layer >= cf.num_layers) return fail(ASYNCEP_ERR_INVALID_ARG, "layer out of range");
  if (T < 0) return fail(ASYNCEP_ERR_INVALID_ARG, "num_tokens < 0");
  if (T > cf.max_tokens) return fail(ASYNCEP_ERR_WORKSPACE, "num_tokens %lld > max_tokens %lld", (long long)T,
                                     (long long)cf.max_tokens);
  if (T > 0 && (!x || !y)) return fail(ASYNCEP_ERR_INVALID_ARG, "x / y is NULL");
  NvtxRange nv("asyncep_moe_forward L%d", layer);
  if (asyncep_status e = check_nccl_async(c)) return e;
  if (((uintptr_t)x | (uintptr_t)y | (uintptr_t)residual) & 15)
    return fail(ASYNCEP_ERR_INVALID_ARG, "x / y / residual must be 16-B aligned");
  if (T > 0 && x == y) return fail(ASYNCEP_ERR_INVALID_ARG, "y must not alias x");
  const bool from_window = c->offload && cf.world_size == 1 && layer > 0;  // NEXT-2, N == 1
  const bool res = !from_window && layer_resident(c, layer);
  const int s = layer % 2;
  const int wi = from_window ? layer % c->w : -1;
  if (from_window && (c->win_layer[wi] != layer || c->win_consumed[wi]))
    return fail(ASYNCEP_ERR_NOT_PREFETCHED, "layer %d was not staged (asyncep_stage_layer)", layer);
  if (!res && !from_window && (c->slot_layer[s] != layer || c->slot_consumed[s]))
    return fail(ASYNCEP_ERR_NOT_PREFETCHED, "layer %d was not prefetched", layer);
  if (T == 0) {
    // No tokens on this rank (a DP rank with an empty batch still takes part in every gather): no
    // compute, but the schedule's bookkeeping stays -- held gathers start, and the slot / window
    // buffer is released in stream order after its gather, so the next prefetch into it proceeds.
    cudaStream_t st0 = c->cs;
    if (!c->pending.empty()) {
      if (asyncep_status e = flush_pending(c, true, st0)) return e;
    }
    if (from_window) {
      CUDA_TRY(cudaStreamWaitEvent(st0, c->h2d_done[wi], 0));
      CUDA_TRY(cudaEventRecord(c->win_free[wi], st0));
      c->win_consumed[wi] = true;
    } else if (!res) {
      CUDA_TRY(cudaStreamWaitEvent(st0, c->ag_done[s], 0));
      CUDA_TRY(cudaEventRecord(c->slot_free[s], st0));
      c->slot_consumed[s] = true;
    }
    return ASYNCEP_OK;
  }

  const int E = cf.num_experts, k = cf.top_k, H = cf.hidden, h = cf.ffn;
  cudaStream_t st = c->cs;
  uint8_t* ws = c->ws;
  int32_t* ids = (int32_t*)(ws + c->L.ids);
  float* w = (float*)(ws + c->L.w);
  int32_t* dest = (int32_t*)(ws + c->L.dest);
  int32_t* src_tok = (int32_t*)(ws + c->L.src_tok);
  int32_t* blk = (int32_t*)(ws + c->L.blk);
  int32_t* offsets = (int32_t*)(ws + c->L.offsets);
  int32_t* tile_start = (int32_t*)(ws + c->L.tile_start);
  int32_t* counts = (int32_t*)(ws + c->L.counts);
  bf16* xperm = (bf16*)(ws + c->L.xperm);
  bf16* act = (bf16*)(ws + c->L.act);
  const int nblk = (int)((T + aep::kPermTokensPerBlock - 1) / aep::kPermTokensPerBlock);

  const bool timing = (cf.flags & ASYNCEP_FLAG_STAGE_TIMING) != 0;
  cudaEvent_t* ev = nullptr;
  int* sched = (int*)(ws + c->L.sched);
  CUDA_TRY(cudaMemsetAsync(sched, 0, 16, st));
  if (timing) {
    if (c->ev_used == kMaxPendingFwd) {
      asyncep_status fs = flush_timing(c, /*blocking=*/false);
      if (fs) return fs;
    }
    if (c->ev_pool.empty()) {
      c->ev_pool.resize((size_t)kMaxPendingFwd * kEventsPerFwd);
      for (auto& e : c->ev_pool) CUDA_TRY(cudaEventCreate(&e));
      c->ev_layer.assign(kMaxPendingFwd, -1);
    }
    const int slot = (c->ev_head + c->ev_used) % kMaxPendingFwd;
    ev = &c->ev_pool[(size_t)slot * kEventsPerFwd];
    ++c->ev_used;
    c->ev_layer[(size_t)slot] = layer;
    CUDA_TRY(cudaEventRecord(ev[0], st));
  }
  // (1) router GEMM + softmax + top-k
  if (cf.flags & ASYNCEP_FLAG_SIMT_ROUTER)
    aep::launch_router_simt((const bf16*)x, (const bf16*)c->router_w[layer], T, H, E, k, cf.norm_topk, ids, w, st);
  else if (!aep::launch_router_tc(c->router_maps[layer], (const bf16*)x, T, H, E, k, cf.norm_topk, ids, w,
                                  c->num_sms, st, sched))
    return fail(ASYNCEP_ERR_CUDA, "cuTensorMapEncodeTiled failed (router x map)");
  c->launches += 1;
  if (timing) CUDA_TRY(cudaEventRecord(ev[1], st));
  // (2) permute / dispatch
  aep::launch_perm_hist(ids, T, k, E, blk, st);
  // Fused dispatch (optional, ASYNCEP_FLAG_FUSED_DISPATCH): GEMM1's cp.async gather warps read the
  // token rows of x -- or of the token-major x_q -- through src_tok, so X_perm is never written.
  // Otherwise (the default, and the identity / SIMT debug paths) X_perm is materialised.
  const bool fp8 = cf.expert_dtype == ASYNCEP_FP8_E4M3;
  const bool identity = (cf.flags & ASYNCEP_FLAG_IDENTITY_EXPERTS) != 0;
  // The dispatch materialises X_perm by default (BF16 rows, or the e4m3 rows the quantisation pass
  // writes for each of a token's k experts) and GEMM1 TMA-loads A: per step 10-12 % (FP8) and
  // 0.3-3 % (BF16) faster than GEMM1 gathering the rows itself (FLAG_FUSED_DISPATCH; S6)
  const bool fused = (cf.flags & ASYNCEP_FLAG_FUSED_DISPATCH) != 0;
  const bool gather_a = fused &&
                        !(cf.flags & (ASYNCEP_FLAG_XPERM | ASYNCEP_FLAG_IDENTITY_EXPERTS | ASYNCEP_FLAG_SIMT_GEMM)) &&
                        ((uintptr_t)x % 16 == 0) && ((size_t)H * 2) % 16 == 0;
  const bool materialise = identity || (!gather_a && !fp8);
  aep::launch_perm_scan(blk, nblk, E, offsets, tile_start, counts, (unsigned int*)(ws + c->L.done), src_tok, st);
  aep::launch_perm_scatter((const bf16*)x, ids, blk, offsets, T, H, k, E, dest, src_tok,
                           materialise ? xperm : nullptr, st);
  c->launches += 3;
  aep::F8Args f8{};
  if (fp8 && !identity) {  // per-token e4m3 quantisation of x into its permuted rows (R6)
    f8.x_scale = (const float*)(ws + c->L.xscale);
    f8.act_scale = (const float*)(ws + c->L.ascale);
    f8.act_amax = (uint32_t*)(ws + c->L.amax);
    f8.expert_bytes = c->expert_bytes;
    f8.sgu_off = (size_t)3 * H * h;
    f8.sd_off = f8.sgu_off + (size_t)2 * h * 4;
    f8.mx = (cf.flags & ASYNCEP_FLAG_MX_ACT) != 0;
    f8.act_sf = (uint32_t*)(ws + c->L.asf);
    aep::launch_perm_quant((const bf16*)x, gather_a ? nullptr : dest, T, H, k, ws + c->L.xq,
                           (float*)(ws + c->L.xscale), st);
    c->launches += 1;
  }
  if (timing) CUDA_TRY(cudaEventRecord(ev[2], st));
  // gated gathers (asyncep_set_gather_gate) held since their prefetch are enqueued here: after the
  // dispatch, before the wait for this layer's slot (a held gather of this very layer included)
  if (!c->pending.empty()) {
    if (asyncep_status e = flush_pending(c, true, st)) return e;
  }
  // wait for this layer's gathered experts (placed just before GEMM1 so router and
  // permute also overlap the gather tail)
  if (from_window) CUDA_TRY(cudaStreamWaitEvent(st, c->h2d_done[wi], 0));
  else if (!res) CUDA_TRY(cudaStreamWaitEvent(st, c->ag_done[s], 0));
  if (timing) CUDA_TRY(cudaEventRecord(ev[3], st));
  // (3) grouped GEMM: gate/up + SwiGLU, then down.  Y_perm overwrites X_perm.
  const uint8_t* wl = (const uint8_t*)(from_window ? c->window[wi] : res ? c->shard[layer] : c->slot[s]);
  const aep::GemmMaps& wm = from_window ? c->win_maps[wi] : res ? c->layer_maps[layer] : c->slot_maps[s];
  // gathered layer: this rank's experts come from its own shard (the slot's copy of it is skipped)
  aep::OwnShard own_sh;
  const bool use_own = !from_window && !res && !c->offload && c->shard[layer];
  if (use_own) {
    const int per = E / cf.world_size;
    own_sh = aep::OwnShard{&c->own_maps[layer], (const uint8_t*)c->shard[layer], cf.rank * per, (cf.rank + 1) * per};
  }
  const aep::OwnShard* own = use_own ? &own_sh : nullptr;
  aep::GroupedArgs g{offsets, tile_start, counts, E, (int)(aep::perm_rows(T, k, E) / aep::kRowAlign), sched};
  const bool swap_on = !(cf.flags & ASYNCEP_FLAG_NO_SWAP_TAILS);
  const bool swap_all = (cf.flags & ASYNCEP_FLAG_SWAP_TAILS) != 0;
  const bool fp8e = cf.expert_dtype == ASYNCEP_FP8_E4M3;
  g.swap_max = !swap_on ? 0 : swap_all ? 240 : swap_max_rows(fp8e, false);
  g.swap_max2 = !swap_on ? 0 : swap_all ? 240 : swap_max_rows(fp8e, true);
  bf16* yperm = xperm;
  if (cf.flags & ASYNCEP_FLAG_IDENTITY_EXPERTS) {
    // Y_perm = X_perm (already in place)
  } else if (cf.flags & ASYNCEP_FLAG_SIMT_GEMM) {
    aep::launch_gemm1_simt(g, xperm, wl, c->expert_bytes, H, h, act, st);
    if (timing) CUDA_TRY(cudaEventRecord(ev[4], st));
    aep::launch_gemm2_simt(g, act, wl, c->expert_bytes, H, h, yperm, st);
    c->launches += 2;
  } else if (fp8) {
    f8.layer = wl;
    aep::launch_gemm1_tc(g, c->act_maps, wm, H, h, act, gather_a ? (const void*)(ws + c->L.xq) : nullptr, T, src_tok,
                         c->num_sms, st, &f8, own);
    // stage boundary before the intermediate's quantisation: the GEMM1 stage is the GEMM1 kernel
    // alone (the roofline's dominant kernel); act_quant is timed with GEMM2, whose A operand it makes
    if (timing) CUDA_TRY(cudaEventRecord(ev[4], st));
    if (!f8.mx) {  // MX: GEMM1 already wrote the e4m3 intermediate and its block scales
      aep::launch_act_quant(act, f8.act_amax, offsets, E, aep::perm_rows(T, k, E), h, ws + c->L.aq,
                            (float*)(ws + c->L.ascale), st);
      c->launches += 1;
    }
    aep::launch_gemm2_tc(g, c->act_maps, wm, H, h, yperm, c->num_sms, st, &f8, own);
    c->launches += 2;
  } else {
    aep::launch_gemm1_tc(g, c->act_maps, wm, H, h, act, gather_a ? x : nullptr, T, src_tok, c->num_sms, st, nullptr,
                         own);
    if (timing) CUDA_TRY(cudaEventRecord(ev[4], st));
    aep::launch_gemm2_tc(g, c->act_maps, wm, H, h, yperm, c->num_sms, st, nullptr, own);
    c->launches += 2;
  }
  if (timing && (cf.flags & ASYNCEP_FLAG_IDENTITY_EXPERTS)) CUDA_TRY(cudaEventRecord(ev[4], st));
  if (timing) CUDA_TRY(cudaEventRecord(ev[5], st));
  if (from_window) {
    CUDA_TRY(cudaEventRecord(c->win_free[wi], st));
    c->win_consumed[wi] = true;
  } else if (!res) {
    CUDA_TRY(cudaEventRecord(c->slot_free[s], st));
    c->slot_consumed[s] = true;
  }
  // (4) weighted combine (+ residual)
  aep::launch_combine(yperm, dest, w, (const bf16*)residual, (bf16*)y, T, H, k, st);
  c->launches += 1;
  if (timing) CUDA_TRY(cudaEventRecord(ev[6], st));
  if (ids_out) CUDA_TRY(cudaMemcpyAsync(ids_out, ids, (size_t)T * k * 4, cudaMemcpyDeviceToDevice, st));
  if (w_out) CUDA_TRY(cudaMemcpyAsync(w_out, w, (size_t)T * k * 4, cudaMemcpyDeviceToDevice, st));
  if (counts_out) CUDA_TRY(cudaMemcpyAsync(counts_out, counts, (size_t)E * 4, cudaMemcpyDeviceToDevice, st));
  CUDA_TRY(cudaGetLastError());
  return ASYNCEP_OK;
}


// ------------------------------------------------------------------ EP contrast layer
namespace {
int64_t pad_rows(int64_t n) { return (n + aep::kRowAlign - 1) / aep::kRowAlign * aep::kRowAlign; }

struct EpWs {
  size_t recv, act, offsets, tile_start, counts, rcounts, total;
};
EpWs ep_layout(const asyncep_config& c, int64_t max_recv_rows) {
  EpWs L{};
  size_t o = 0;
  auto take = [&](size_t bytes) {
    const size_t at = o;
    o = align_up(o + bytes, 256);
    return at;
  };
  const size_t R = (size_t)pad_rows(max_recv_rows);
  L.recv = take(R * (size_t)c.hidden * 2);  // received X rows, then the expert outputs (Y)
  L.act = take(R * (size_t)c.ffn * 2);
  L.offsets = take(((size_t)c.num_experts + 1) * 4);
  L.tile_start = take(((size_t)c.num_experts + 1) * 4);
  L.counts = take((size_t)c.num_experts * 4);
  L.rcounts = take((size_t)c.num_experts * 4);
  L.total = o;
  return L;
}
}  // namespace

asyncep_status asyncep_ep_plan(const asyncep_config* cfg, const int32_t* sc, const int32_t* rc, int64_t* send_off,
                               int64_t* send_rows, int64_t* recv_off, int64_t* recv_rows, int64_t* group_off,
                               int64_t* recv_total) {
  if (!cfg || !sc || !rc) return fail(ASYNCEP_ERR_INVALID_ARG, "null argument");
  const int E = cfg->num_experts, N = cfg->world_size;
  if (N <= 0 || E % N) return fail(ASYNCEP_ERR_INVALID_ARG, "E %% N != 0");
  const int per = E / N;
  // send side: this rank's X_perm lays experts out in order, each padded to kRowAlign, so
  // the rows for rank d are one contiguous range
  int64_t o = 0;
  for (int d = 0; d < N; ++d) {
    int64_t n = 0;
    for (int j = 0; j < per; ++j) n += pad_rows(sc[d * per + j]);
    if (send_off) send_off[d] = o;
    if (send_rows) send_rows[d] = n;
    o += n;
  }
  // receive side: source-major, each source's chunk expert-ordered and padded the same way
  int64_t r = 0;
  for (int s = 0; s < N; ++s) {
    int64_t n = 0;
    for (int j = 0; j < per; ++j) {
      if (group_off) group_off[s * per + j] = r + n;
      n += pad_rows(rc[s * per + j]);
    }
    if (recv_off) recv_off[s] = r;
    if (recv_rows) recv_rows[s] = n;
    r += n;
  }
  if (group_off) group_off[E] = r;
  if (recv_total) *recv_total = r;
  return ASYNCEP_OK;
}

size_t asyncep_ep_workspace_size(const asyncep_config* cfg, int64_t max_recv_rows) {
  if (check_config(cfg) != ASYNCEP_OK || max_recv_rows <= 0) return 0;
  return ep_layout(*cfg, max_recv_rows).total;
}

asyncep_status asyncep_ep_forward(asyncep_ctx* c, int32_t layer, const void* x, int64_t T, const void* residual,
                                  void* y, void* ep_ws, int64_t max_recv_rows) {
  if (!c) return fail(ASYNCEP_ERR_INVALID_ARG, "ctx is NULL");
  const asyncep_config& cf = c->cfg;
  if (layer < 0 || layer >= cf.num_layers) return fail(ASYNCEP_ERR_INVALID_ARG, "layer out of range");
  if (cf.expert_dtype != ASYNCEP_BF16) return fail(ASYNCEP_ERR_UNSUPPORTED, "EP contrast layer is BF16 only");
  if (T < 0 || T > cf.max_tokens) return fail(ASYNCEP_ERR_WORKSPACE, "num_tokens out of range");
  // T == 0 at N == 1: nothing to do; at N > 1 the rank still joins both AllToAlls (it sends no rows
  // but computes the rows other ranks send to its experts)
  if (T == 0 && cf.world_size == 1) return ASYNCEP_OK;
  if ((T > 0 && (!x || !y)) || !ep_ws || max_recv_rows <= 0) return fail(ASYNCEP_ERR_INVALID_ARG, "null argument");
  if (((uintptr_t)x | (uintptr_t)y | (uintptr_t)residual | (uintptr_t)ep_ws) & 15)
    return fail(ASYNCEP_ERR_INVALID_ARG, "pointers must be 16-B aligned");
  NvtxRange nv("asyncep_ep_forward L%d", layer);
  if (asyncep_status e = check_nccl_async(c)) return e;
  const int N = cf.world_size, E = cf.num_experts, per = E / N, k = cf.top_k, H = cf.hidden, h = cf.ffn;
  if (N > 1 && (!c->comm || !c->nccl.send || !c->nccl.recv))
    return fail(ASYNCEP_ERR_NCCL, "EP contrast with world_size > 1 needs an NCCL communicator");
  cudaStream_t st = c->cs;
  uint8_t* ws = c->ws;
  const EpWs EL = ep_layout(cf, max_recv_rows);
  uint8_t* ew = (uint8_t*)ep_ws;
  // this rank's shard of the layer: E/N expert blobs
  if (c->ep_maps.empty()) {
    c->ep_maps.resize(cf.num_layers);
    c->ep_maps_ok.assign(cf.num_layers, 0);
  }
  const bool full = layer_resident(c, layer) && N > 1;  // a full layer: take this rank's part
  const uint8_t* wl = (const uint8_t*)c->shard[layer] + (full ? (size_t)cf.rank * c->shard_bytes : 0);
  if (!c->ep_maps_ok[layer]) {
    if (!aep::make_weight_maps(c->ep_maps[layer], wl, c->expert_bytes, per, H, h, c->act_maps.bn2, false))
      return fail(ASYNCEP_ERR_CUDA, "cuTensorMapEncodeTiled failed (EP shard maps)");
    c->ep_maps_ok[layer] = 1;
  }
  int32_t* ids = (int32_t*)(ws + c->L.ids);
  float* w = (float*)(ws + c->L.w);
  int32_t* dest = (int32_t*)(ws + c->L.dest);
  int32_t* src_tok = (int32_t*)(ws + c->L.src_tok);
  int32_t* blk = (int32_t*)(ws + c->L.blk);
  int32_t* offsets = (int32_t*)(ws + c->L.offsets);
  int32_t* tile_start = (int32_t*)(ws + c->L.tile_start);
  int32_t* counts = (int32_t*)(ws + c->L.counts);
  bf16* xperm = (bf16*)(ws + c->L.xperm);
  int* sched = (int*)(ws + c->L.sched);
  const int nblk = (int)((T + aep::kPermTokensPerBlock - 1) / aep::kPermTokensPerBlock);
  CUDA_TRY(cudaMemsetAsync(sched, 0, 16, st));
  if (T > 0) {
    // (1) router + (2) local permute, as in the AsyncEP forward
    if (!aep::launch_router_tc(c->router_maps[layer], (const bf16*)x, T, H, E, k, cf.norm_topk, ids, w, c->num_sms,
                               st, sched))
      return fail(ASYNCEP_ERR_CUDA, "cuTensorMapEncodeTiled failed (router x map)");
    aep::launch_perm_hist(ids, T, k, E, blk, st);
    aep::launch_perm_scan(blk, nblk, E, offsets, tile_start, counts, (unsigned int*)(ws + c->L.done), src_tok, st);
    aep::launch_perm_scatter((const bf16*)x, ids, blk, offsets, T, H, k, E, dest, src_tok, xperm, st);
    c->launches += 4;
  } else {
    CUDA_TRY(cudaMemsetAsync(counts, 0, (size_t)E * 4, st));  // sends no rows
  }
  // (a) exchange the per-expert counts (E/N to every rank), read them back: host sync
  int32_t* d_rc = (int32_t*)(ew + EL.rcounts);
  if (N > 1) {
    c->nccl.group_start();
    for (int d = 0; d < N; ++d) {
      c->nccl.send(counts + d * per, (size_t)per, kNcclInt32, d, c->comm, st);
      c->nccl.recv(d_rc + d * per, (size_t)per, kNcclInt32, d, c->comm, st);
    }
    if (c->nccl.group_end() != 0) return fail(ASYNCEP_ERR_NCCL, "count exchange failed");
  } else {
    CUDA_TRY(cudaMemcpyAsync(d_rc, counts, (size_t)E * 4, cudaMemcpyDeviceToDevice, st));
  }
  std::vector<int32_t> hsc(E), hrc(E);
  CUDA_TRY(cudaMemcpyAsync(hsc.data(), counts, (size_t)E * 4, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaMemcpyAsync(hrc.data(), d_rc, (size_t)E * 4, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  std::vector<int64_t> so(N), sr(N), ro(N), rr(N), go(E + 1);
  int64_t rtot = 0;
  asyncep_status ps = asyncep_ep_plan(&cf, hsc.data(), hrc.data(), so.data(), sr.data(), ro.data(), rr.data(),
                                      go.data(), &rtot);
  if (ps) return ps;
  if (rtot > pad_rows(max_recv_rows))
    return fail(ASYNCEP_ERR_WORKSPACE, "EP receive rows %lld > capacity %lld", (long long)rtot,
                (long long)max_recv_rows);
  // receive-side group table (groups = (source rank, local expert))
  std::vector<int32_t> g_off(E + 1), g_ts(E + 1);
  for (int g = 0; g <= E; ++g) {
    g_off[g] = (int32_t)go[g];
    g_ts[g] = (int32_t)(go[g] / aep::kRowAlign);
  }
  int32_t* d_goff = (int32_t*)(ew + EL.offsets);
  int32_t* d_gts = (int32_t*)(ew + EL.tile_start);
  CUDA_TRY(cudaMemcpyAsync(d_goff, g_off.data(), (size_t)(E + 1) * 4, cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaMemcpyAsync(d_gts, g_ts.data(), (size_t)(E + 1) * 4, cudaMemcpyHostToDevice, st));
  // (b) dispatch AllToAll of the permuted rows (on the critical path)
  bf16* recv = (bf16*)(ew + EL.recv);
  const size_t row_b = (size_t)H * 2;
  auto exchange = [&](const bf16* sbuf, const std::vector<int64_t>& soff, const std::vector<int64_t>& srows,
                      bf16* rbuf, const std::vector<int64_t>& roff, const std::vector<int64_t>& rrows) -> asyncep_status {
    if (N > 1) {
      c->nccl.group_start();
      for (int d = 0; d < N; ++d) {
        if (srows[d]) c->nccl.send(sbuf + soff[d] * H, (size_t)srows[d] * row_b, kNcclUint8, d, c->comm, st);
        if (rrows[d]) c->nccl.recv(rbuf + roff[d] * H, (size_t)rrows[d] * row_b, kNcclUint8, d, c->comm, st);
      }
      if (c->nccl.group_end() != 0) return fail(ASYNCEP_ERR_NCCL, "AllToAll failed");
    } else if (srows[0]) {
      CUDA_TRY(cudaMemcpyAsync(rbuf + roff[0] * H, sbuf + soff[0] * H, (size_t)srows[0] * row_b,
                               cudaMemcpyDeviceToDevice, st));
    }
    return ASYNCEP_OK;
  };
  asyncep_status xs = exchange(xperm, so, sr, recv, ro, rr);
  if (xs) return xs;
  // (c) this rank's experts on the rows of all ranks: groups g -> expert g % (E/N)
  aep::ActMaps am{};
  bf16* act = (bf16*)(ew + EL.act);
  if (!aep::make_act_maps(am, recv, act, std::max<int64_t>(rtot, aep::kRowAlign), H, h, nullptr, nullptr))
    return fail(ASYNCEP_ERR_CUDA, "cuTensorMapEncodeTiled failed (EP activations)");
  aep::GroupedArgs g{d_goff, d_gts, nullptr, E, (int)(rtot / aep::kRowAlign), sched, per};
  aep::launch_gemm1_tc(g, am, c->ep_maps[layer], H, h, act, nullptr, rtot, nullptr, c->num_sms, st);
  aep::launch_gemm2_tc(g, am, c->ep_maps[layer], H, h, recv, c->num_sms, st);
  c->launches += 2;
  // (d) combine AllToAll: expert outputs back to their tokens' ranks, into X_perm's rows
  xs = exchange(recv, ro, rr, xperm, so, sr);
  if (xs) return xs;
  // (e) weighted combine (+ residual)
  if (T > 0) {
    aep::launch_combine(xperm, dest, w, (const bf16*)residual, (bf16*)y, T, H, k, st);
    c->launches += 1;
  }
  CUDA_TRY(cudaGetLastError());
  return ASYNCEP_OK;
}

asyncep_status asyncep_saturation_T(const asyncep_config* cfg, double flops_per_s, double ag_bytes_per_s,
                                    double* tokens_out, double* flops_out) {
  if (!cfg) return fail(ASYNCEP_ERR_INVALID_ARG, "config is NULL");
  if (cfg->num_experts <= 0 || cfg->top_k <= 0 || cfg->hidden <= 0 || cfg->ffn <= 0 || cfg->world_size <= 0)
    return fail(ASYNCEP_ERR_INVALID_ARG, "bad shape");
  if (!(flops_per_s > 0) || !(ag_bytes_per_s > 0)) return fail(ASYNCEP_ERR_INVALID_ARG, "rates must be > 0");
  if (!(cfg->gamma >= 1.0f)) return fail(ASYNCEP_ERR_INVALID_ARG, "gamma must be >= 1");
  const double b = cfg->expert_dtype == ASYNCEP_FP8_E4M3 ? 1.0 : 2.0;
  const double n = (double)cfg->world_size;
  const double per_tok_flops = 6.0 * cfg->top_k * (double)cfg->hidden * (double)cfg->ffn;
  // t_AG = (N-1)/N * E*3*H*h*b / BW ; T_FLOPs = gamma * t_AG * F ; T_tok = T_FLOPs / (6 k H h)
  const double t_ag = (n - 1.0) / n * (double)cfg->num_experts * 3.0 * cfg->hidden * (double)cfg->ffn * b /
                      ag_bytes_per_s;
  const double tf = (double)cfg->gamma * t_ag * flops_per_s;
  if (flops_out) *flops_out = tf;
  if (tokens_out) *tokens_out = tf / per_tok_flops;
  return ASYNCEP_OK;
}

asyncep_status asyncep_stage_times(asyncep_ctx* c, double* ms_out, int32_t n, int64_t* fwd_out) {
  if (!c) return fail(ASYNCEP_ERR_INVALID_ARG, "ctx is NULL");
  asyncep_status st = flush_timing(c);
  if (st) return st;
  for (int i = 0; i < n && i < kStages; ++i) ms_out[i] = c->stage_ms[i];
  if (fwd_out) *fwd_out = c->fwd_count;
  return ASYNCEP_OK;
}

asyncep_status asyncep_reset_stage_times(asyncep_ctx* c) {
  if (!c) return fail(ASYNCEP_ERR_INVALID_ARG, "ctx is NULL");
  asyncep_status st = flush_timing(c);
  if (st) return st;
  for (double& v : c->stage_ms) v = 0.0;
  c->fwd_count = 0;
  c->recent.clear();
  return ASYNCEP_OK;
}

asyncep_status asyncep_forward_times(asyncep_ctx* c, double* ms_out, int32_t* layer_out, int32_t n, int32_t* n_out) {
  if (!c || n < 0) return fail(ASYNCEP_ERR_INVALID_ARG, "bad arguments");
  asyncep_status st = flush_timing(c);
  if (st) return st;
  const int32_t m = (int32_t)std::min<size_t>((size_t)n, c->recent.size());
  const size_t base = c->recent.size() - (size_t)m;
  for (int32_t i = 0; i < m; ++i) {
    if (ms_out) ms_out[i] = c->recent[base + i].second;
    if (layer_out) layer_out[i] = c->recent[base + i].first;
  }
  if (n_out) *n_out = m;
  return ASYNCEP_OK;
}

asyncep_status asyncep_timeline_begin(asyncep_ctx* c) {
  if (!c) return fail(ASYNCEP_ERR_INVALID_ARG, "ctx is NULL");
  if (!(c->cfg.flags & ASYNCEP_FLAG_STAGE_TIMING))
    return fail(ASYNCEP_ERR_INVALID_ARG, "timeline needs a context created with ASYNCEP_FLAG_STAGE_TIMING");
  asyncep_status st = flush_timing(c);
  if (st) return st;
  for (auto& g : c->tl_gather) {
    cudaEventDestroy(g.second.first);
    cudaEventDestroy(g.second.second);
  }
  c->tl_gather.clear();
  c->tl.clear();
  if (!c->epoch) CUDA_TRY(cudaEventCreate(&c->epoch));
  CUDA_TRY(cudaEventRecord(c->epoch, c->cs));
  if (c->ms) CUDA_TRY(cudaStreamWaitEvent(c->ms, c->epoch, 0));  // no gather starts before the epoch
  c->timeline = true;
  return ASYNCEP_OK;
}

asyncep_status asyncep_timeline_read(asyncep_ctx* c, asyncep_timeline_rec* out, int32_t n, int32_t* n_out) {
  if (!c || n < 0 || (n > 0 && !out)) return fail(ASYNCEP_ERR_INVALID_ARG, "bad arguments");
  if (!c->timeline) return fail(ASYNCEP_ERR_INVALID_ARG, "asyncep_timeline_begin was not called");
  asyncep_status st = flush_timing(c);
  if (st) return st;
  for (auto& g : c->tl_gather) {
    CUDA_TRY(cudaEventSynchronize(g.second.second));
    float a = 0.f, b = 0.f;
    CUDA_TRY(cudaEventElapsedTime(&a, c->epoch, g.second.first));
    CUDA_TRY(cudaEventElapsedTime(&b, c->epoch, g.second.second));
    c->tl.push_back(asyncep_timeline_rec{ASYNCEP_TL_GATHER, g.first, a, b, b, b});
    cudaEventDestroy(g.second.first);
    cudaEventDestroy(g.second.second);
  }
  c->tl_gather.clear();
  const int32_t m = (int32_t)std::min<size_t>((size_t)n, c->tl.size());
  for (int32_t i = 0; i < m; ++i) out[i] = c->tl[(size_t)i];
  if (n_out) *n_out = (int32_t)c->tl.size();
  c->timeline = false;
  return ASYNCEP_OK;
}

asyncep_status asyncep_calibrated_T(double gamma, double t_e, double t_c, double c_dummy, double* flops_out) {
  if (!(gamma >= 1.0) || !(t_c > 0) || !(t_e >= 0) || !(c_dummy >= 0))
    return fail(ASYNCEP_ERR_INVALID_ARG, "calibrated_T: need gamma >= 1, t_c > 0, t_e >= 0, C_dummy >= 0");
  // T = gamma * (t_e / t_c) * C_dummy; collapses to gamma * C_dummy when transfers are hidden
  const double ratio = t_e <= t_c ? 1.0 : t_e / t_c;
  if (flops_out) *flops_out = gamma * ratio * c_dummy;
  return ASYNCEP_OK;
}

asyncep_status asyncep_calibrate_T(asyncep_ctx* c, double gamma, int64_t n_ref, double* flops_out,
                                   double* tokens_out, double* t_c_out, double* t_e_out) {
  if (!c || n_ref <= 0) return fail(ASYNCEP_ERR_INVALID_ARG, "calibrate_T: null ctx or n_ref <= 0");
  if (!(c->cfg.flags & ASYNCEP_FLAG_STAGE_TIMING))
    return fail(ASYNCEP_ERR_INVALID_ARG, "calibrate_T: the context was created without ASYNCEP_FLAG_STAGE_TIMING");
  asyncep_status st = flush_timing(c);
  if (st) return st;
  const int L = c->cfg.num_layers;
  if ((int)c->recent.size() < L)
    return fail(ASYNCEP_ERR_INVALID_ARG, "calibrate_T: %d forwards recorded, the profile pass needs %d",
                (int)c->recent.size(), L);
  // the profile pass = the last L forwards: t_c = the resident layer 0 (pure compute),
  // t_e = max over the gathered layers >= 1 (each the envelope max(compute, transfer))
  double t_c = -1.0, t_e = -1.0;
  for (size_t i = c->recent.size() - (size_t)L; i < c->recent.size(); ++i) {
    if (c->recent[i].first == 0) t_c = c->recent[i].second;
    else t_e = std::max(t_e, c->recent[i].second);
  }
  if (t_c <= 0) return fail(ASYNCEP_ERR_INVALID_ARG, "calibrate_T: layer 0 is not among the last %d forwards", L);
  if (t_e < 0) t_e = t_c;  // a one-layer stack: nothing gathered
  // C_dummy = f_tok * n_ref, f_tok = per-token FLOPs of one MoE layer (router 2HE + experts 6kHh)
  const double H = c->cfg.hidden, E = c->cfg.num_experts, k = c->cfg.top_k, h = c->cfg.ffn;
  const double f_tok = 2.0 * H * E + 6.0 * k * H * h;
  const double g = gamma > 0 ? gamma : (double)c->cfg.gamma;
  double T = 0.0;
  st = asyncep_calibrated_T(g, t_e, t_c, f_tok * (double)n_ref, &T);
  if (st) return st;
  if (flops_out) *flops_out = T;
  if (tokens_out) *tokens_out = T / f_tok;
  if (t_c_out) *t_c_out = t_c;
  if (t_e_out) *t_e_out = t_e;
  return ASYNCEP_OK;
}

// ------------------------------------------------------------------ NEXT-3 attention layer
namespace {
struct AttnWs {
  size_t xn, qkv, q, k, vt, vcu, o, ao, cnt, total;
  int64_t ldv;
};
AttnWs attn_layout(const asyncep_attn_config& c) {
  AttnWs L{};
  const int64_t T = c.max_tokens, H = c.hidden, d = c.head_dim;
  const int64_t nqkv = (int64_t)(c.q_heads + 2 * c.kv_heads) * d;
  const int64_t P = c.max_prompts > 0 ? c.max_prompts : T;
  L.ldv = (T + 7 * P + 7) / 8 * 8;  // every prompt's V^T columns start on a multiple of 8
  size_t o = 0;
  auto take = [&](size_t bytes) {
    const size_t at = o;
    o += (bytes + 255) / 256 * 256;
    return at;
  };
  L.xn = take((size_t)T * H * 2);
  L.qkv = take((size_t)T * nqkv * 2);
  L.q = take((size_t)T * c.q_heads * d * 2);
  L.k = take((size_t)T * c.kv_heads * d * 2);
  L.vt = take((size_t)c.kv_heads * d * L.ldv * 2);
  L.vcu = take((size_t)(P + 1) * 4);
  L.o = take((size_t)T * c.q_heads * d * 2);
  L.ao = take((size_t)T * H * 2);
  L.cnt = take(256);
  L.total = o;
  return L;
}
asyncep_status attn_check(const asyncep_attn_config* c) {
  if (!c) return fail(ASYNCEP_ERR_INVALID_ARG, "attn config is NULL");
  if (c->head_dim != 128) return fail(ASYNCEP_ERR_INVALID_ARG, "head_dim must be 128 (got %d)", c->head_dim);
  if (c->q_heads <= 0 || c->kv_heads <= 0 || c->q_heads % c->kv_heads)
    return fail(ASYNCEP_ERR_INVALID_ARG, "q_heads must be a positive multiple of kv_heads");
  if (c->hidden <= 0 || c->hidden % 256) return fail(ASYNCEP_ERR_INVALID_ARG, "hidden must be a multiple of 256");
  if (((int64_t)(c->q_heads + 2 * c->kv_heads) * c->head_dim) % 256)
    return fail(ASYNCEP_ERR_INVALID_ARG, "(q_heads + 2 kv_heads) * head_dim must be a multiple of 256");
  if (c->max_tokens < 0) return fail(ASYNCEP_ERR_INVALID_ARG, "max_tokens < 0");
  return ASYNCEP_OK;
}
int device_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
  }
  return n;
}
}  // namespace

size_t asyncep_attn_workspace_size(const asyncep_attn_config* c) {
  if (attn_check(c) != ASYNCEP_OK) return 0;
  return attn_layout(*c).total;
}

asyncep_status asyncep_attention(const asyncep_attn_config* c, const void* q, const void* k, const void* vt,
                                 int64_t ldv, const int32_t* vt_cu, const int32_t* cu, int32_t B, int64_t T, void* o,
                                 int32_t* sched, void* stream) {
  if (asyncep_status st = attn_check(c)) return st;
  if (T == 0) return ASYNCEP_OK;
  if (!q || !k || !vt || !vt_cu || !cu || !o || !sched || B <= 0 || T < 0 || ldv < T || ldv % 8)
    return fail(ASYNCEP_ERR_INVALID_ARG, "asyncep_attention: bad pointers / B / T / ldv");
  if (((uintptr_t)q | (uintptr_t)k | (uintptr_t)vt | (uintptr_t)o) % 16)
    return fail(ASYNCEP_ERR_INVALID_ARG, "asyncep_attention: tensors must be 16-B aligned");
  if (!aep::launch_flash_attn((const bf16*)q, (const bf16*)k, (const bf16*)vt, ldv, cu, vt_cu, B, T, c->q_heads,
                              c->kv_heads, (bf16*)o, sched, (cudaStream_t)stream))
    return fail(ASYNCEP_ERR_CUDA, "attention launch failed (tensor maps or scheduler counter)");
  CUDA_TRY(cudaGetLastError());
  return ASYNCEP_OK;
}

asyncep_status asyncep_attn_layer(const asyncep_attn_config* c, const void* x, int64_t T, const int32_t* cu,
                                  int32_t B, const void* w_ln1, const void* w_qkv, const void* w_qn,
                                  const void* w_kn, const void* w_o, const void* w_ln2, void* x_out, void* xn2_out,
                                  void* workspace, size_t ws_bytes, void* stream) {
  if (asyncep_status st = attn_check(c)) return st;
  if (T == 0) return ASYNCEP_OK;
  if (T < 0 || T > c->max_tokens) return fail(ASYNCEP_ERR_WORKSPACE, "T=%lld > max_tokens", (long long)T);
  if (c->max_prompts > 0 && B > c->max_prompts) return fail(ASYNCEP_ERR_WORKSPACE, "B=%d > max_prompts", B);
  if (!x || !cu || B <= 0 || !w_ln1 || !w_qkv || !w_qn || !w_kn || !w_o || !w_ln2 || !x_out || !xn2_out ||
      !workspace)
    return fail(ASYNCEP_ERR_INVALID_ARG, "asyncep_attn_layer: null argument");
  const AttnWs L = attn_layout(*c);
  if (ws_bytes < L.total || (uintptr_t)workspace % 256)
    return fail(ASYNCEP_ERR_INVALID_ARG, "asyncep_attn_layer: workspace too small or misaligned");
  if (x_out == x || xn2_out == x) return fail(ASYNCEP_ERR_INVALID_ARG, "outputs may not alias x");
  cudaStream_t st = (cudaStream_t)stream;
  uint8_t* ws = (uint8_t*)workspace;
  const int H = c->hidden, Hq = c->q_heads, Hkv = c->kv_heads, d = c->head_dim;
  const int nqkv = (Hq + 2 * Hkv) * d;
  const float eps = (float)c->eps;
  int* cnt = (int*)(ws + L.cnt);
  CUDA_TRY(cudaMemsetAsync(cnt, 0, 2 * sizeof(int), st));
  bf16* xn = (bf16*)(ws + L.xn);
  bf16* qkv = (bf16*)(ws + L.qkv);
  bf16* qb = (bf16*)(ws + L.q);
  bf16* kb = (bf16*)(ws + L.k);
  bf16* vt = (bf16*)(ws + L.vt);
  bf16* ob = (bf16*)(ws + L.o);
  bf16* ao = (bf16*)(ws + L.ao);
  aep::launch_rmsnorm((const bf16*)x, (const bf16*)w_ln1, T, H, eps, xn, st);
  if (!aep::launch_dense_gemm_tc(xn, T, H, (const bf16*)w_qkv, nqkv, qkv, cnt, device_sms(), st))
    return fail(ASYNCEP_ERR_CUDA, "QKV projection: tensor map encoding failed");
  aep::launch_qk_rope(qkv, T, Hq, Hkv, cu, B, (const bf16*)w_qn, (const bf16*)w_kn, eps, (float)c->rope_theta, qb, kb,
                      st);
  int32_t* vcu = (int32_t*)(ws + L.vcu);
  const int64_t ldv = (T + 7 * (int64_t)B + 7) / 8 * 8;
  aep::launch_v_transpose(qkv, T, Hq, Hkv, cu, B, vcu, ldv, vt, st);
  if (!aep::launch_flash_attn(qb, kb, vt, ldv, cu, vcu, B, T, Hq, Hkv, ob, cnt + 2, st))
    return fail(ASYNCEP_ERR_CUDA, "attention: launch failed (tensor maps or scheduler counter)");
  if (!aep::launch_dense_gemm_tc(ob, T, Hq * d, (const bf16*)w_o, H, ao, cnt + 1, device_sms(), st))
    return fail(ASYNCEP_ERR_CUDA, "O projection: tensor map encoding failed");
  aep::launch_residual_rmsnorm((const bf16*)x, ao, (const bf16*)w_ln2, T, H, eps, (bf16*)x_out, (bf16*)xn2_out, st);
  CUDA_TRY(cudaGetLastError());
  return ASYNCEP_OK;
}

int64_t asyncep_kernel_launches(const asyncep_ctx* c) { return c ? c->launches : 0; }

asyncep_status asyncep_destroy(asyncep_ctx* c) {
  if (!c) return ASYNCEP_OK;
  for (int i = 0; i < 2; ++i) {
    if (c->ag_done[i]) cudaEventDestroy(c->ag_done[i]);
    if (c->slot_free[i]) cudaEventDestroy(c->slot_free[i]);
  }
  for (auto& e : c->ev_pool)
    if (e) cudaEventDestroy(e);
  for (auto& g : c->tl_gather) {
    cudaEventDestroy(g.second.first);
    cudaEventDestroy(g.second.second);
  }
  if (c->epoch) cudaEventDestroy(c->epoch);
  if (c->gate_ev) cudaEventDestroy(c->gate_ev);
  for (auto& e : c->h2d_done)
    if (e) cudaEventDestroy(e);
  for (auto& e : c->win_free)
    if (e) cudaEventDestroy(e);
  delete c;
  return ASYNCEP_OK;
}

}  // extern "C"
