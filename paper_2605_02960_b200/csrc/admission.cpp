// admission.cpp -- NEXT-4: saturation-bounded admission (the consumer of T on the frontend).
//
// PAPER.md:401-406 (S7.4 "Overlap-Aware Balancing") and Algorithm 1 (App. A,
// PAPER.md:591-619): drain the request queue in arrival order; for each request evaluate the
// unsaturated GPUs (L_i < T), pick the longest block-level prefix match (ties: least loaded,
// then lowest index), charge the true FLOPs cost of Eq. 2
//     Delta_r = C_pfx(P_r - M_r) + C_sfx(S_r, P_r),
// and mark the GPU saturated once L_i >= T; each saturated GPU ends in [T, T + Delta_last].
// Functional forms (reading R18, the SPEC's standard transformer terms, since the paper gives
// only orders): C_pfx(n) = n f_tok + 2 n^2 HL; C_sfx(S,P) = S f_tok + 2 S^2 HL + 4 S P HL,
// with HL = hidden x attention layers.  Block tables: committed U pending hash sets per GPU
// (App. B.2); the uncached blocks of an assigned request become pending.
// Host-only code; no device work.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <unordered_set>
#include <vector>

#include "asyncep.h"

struct asyncep_router {
  asyncep_router_config cfg;
  std::vector<double> load;
  std::vector<std::unordered_set<uint64_t>> committed, pending;
};

namespace aep {
asyncep_status set_error(asyncep_status st, const char* msg);  // asyncep.cu: asyncep_last_error()
}

namespace {
asyncep_status bad(const char* msg) { return aep::set_error(ASYNCEP_ERR_INVALID_ARG, msg); }
double c_pfx(const asyncep_router_config& c, double n) { return n * c.f_tok + 2.0 * n * n * c.attn_hl; }
double c_sfx(const asyncep_router_config& c, double S, double P) {
  return S * c.f_tok + 2.0 * S * S * c.attn_hl + 4.0 * S * P * c.attn_hl;
}
bool has(const asyncep_router* r, int g, uint64_t h) {
  return r->committed[g].count(h) || r->pending[g].count(h);
}
}  // namespace

extern "C" {

double asyncep_cost_delta(const asyncep_router_config* c, int64_t P, int64_t M, int64_t S) {
  if (!c || P < 0 || M < 0 || M > P || S < 0) return NAN;
  return c_pfx(*c, (double)(P - M)) + c_sfx(*c, (double)S, (double)P);
}

asyncep_status asyncep_router_create(const asyncep_router_config* cfg, asyncep_router** out) {
  if (!cfg || !out || cfg->num_gpus <= 0 || cfg->block_size <= 0 || !(cfg->f_tok > 0) || cfg->attn_hl < 0 ||
      !(cfg->T_flops > 0))
    return bad("asyncep_router_create: need num_gpus > 0, block_size > 0, f_tok > 0, attn_hl >= 0, T_flops > 0");
  asyncep_router* r = new asyncep_router();
  r->cfg = *cfg;
  r->load.assign(cfg->num_gpus, 0.0);
  r->committed.resize(cfg->num_gpus);
  r->pending.resize(cfg->num_gpus);
  *out = r;
  return ASYNCEP_OK;
}

asyncep_status asyncep_router_destroy(asyncep_router* r) {
  delete r;
  return ASYNCEP_OK;
}

asyncep_status asyncep_router_set_T(asyncep_router* r, double T_flops) {
  if (!r || !(T_flops > 0)) return bad("asyncep_router_set_T: null router or T_flops <= 0");
  r->cfg.T_flops = T_flops;
  return ASYNCEP_OK;
}

asyncep_status asyncep_router_loads(const asyncep_router* r, double* loads_out) {
  if (!r || !loads_out) return bad("asyncep_router_loads: null argument");
  for (size_t i = 0; i < r->load.size(); ++i) loads_out[i] = r->load[i];
  return ASYNCEP_OK;
}

asyncep_status asyncep_router_schedule_round(asyncep_router* r, int32_t reset_loads, int64_t n_req,
                                             const int64_t* chain_off, const uint64_t* hashes,
                                             const int64_t* prefix_len, const int64_t* suffix_len, int32_t* gpu_out,
                                             double* delta_out, int64_t* admitted_out) {
  if (!r || n_req < 0 || (n_req > 0 && (!chain_off || !prefix_len || !suffix_len || !gpu_out)))
    return bad("asyncep_router_schedule_round: null argument or n_req < 0");
  // validate every request before any state changes, so a malformed round changes nothing
  for (int64_t q = 0; q < n_req; ++q) {
    if (chain_off[q + 1] < chain_off[q] || chain_off[q] < 0 || prefix_len[q] < 0 || suffix_len[q] < 0)
      return bad("asyncep_router_schedule_round: request with chain_off[q+1] < chain_off[q] or negative length");
  }
  if (n_req > 0 && chain_off[n_req] > chain_off[0] && !hashes)
    return bad("asyncep_router_schedule_round: hashes is NULL with a non-empty block chain");
  const int N = r->cfg.num_gpus;
  const double T = r->cfg.T_flops;
  if (reset_loads)
    for (double& v : r->load) v = 0.0;  // Algorithm 1 line 1: L_i <- 0
  std::vector<char> active(N);
  int n_active = 0;
  for (int i = 0; i < N; ++i) n_active += (active[i] = r->load[i] < T);
  int64_t admitted = 0;
  for (int64_t q = 0; q < n_req; ++q) {
    gpu_out[q] = -1;
    if (delta_out) delta_out[q] = 0.0;
    if (n_active == 0) continue;  // requests stay queued for the next round
    const int64_t b0 = chain_off[q], b1 = chain_off[q + 1];
    int best = -1;
    int64_t best_m = -1;
    for (int i = 0; i < N; ++i) {
      if (!active[i]) continue;
      int64_t m = 0;  // BlockMatch: longest run of leading blocks in committed U pending
      while (b0 + m < b1 && has(r, i, hashes[b0 + m])) ++m;
      if (m > best_m || (m == best_m && r->load[i] < r->load[best])) {
        best = i;
        best_m = m;
      }
    }
    const int64_t P = prefix_len[q];
    const int64_t M = std::min<int64_t>(best_m * r->cfg.block_size, P);
    const double d = asyncep_cost_delta(&r->cfg, P, M, suffix_len[q]);
    r->load[best] += d;
    for (int64_t j = b0; j < b1; ++j)  // uncached blocks become pending on i* (in-batch reuse)
      if (!r->committed[best].count(hashes[j])) r->pending[best].insert(hashes[j]);
    gpu_out[q] = best;
    if (delta_out) delta_out[q] = d;
    ++admitted;
    if (r->load[best] >= T) {
      active[best] = 0;
      --n_active;
    }
  }
  if (admitted_out) *admitted_out = admitted;
  return ASYNCEP_OK;
}

asyncep_status asyncep_router_blocks_stored(asyncep_router* r, int32_t gpu, const uint64_t* hashes, int64_t n) {
  if (!r || gpu < 0 || gpu >= r->cfg.num_gpus || n < 0 || (n > 0 && !hashes))
    return bad("asyncep_router_blocks_stored: bad router / gpu / hashes");
  for (int64_t i = 0; i < n; ++i) {  // pending -> committed (App. B.2 promotion)
    r->pending[gpu].erase(hashes[i]);
    r->committed[gpu].insert(hashes[i]);
  }
  return ASYNCEP_OK;
}

asyncep_status asyncep_router_progress(asyncep_router* r, int32_t gpu, int64_t tokens) {
  if (!r || gpu < 0 || gpu >= r->cfg.num_gpus || tokens < 0)
    return bad("asyncep_router_progress: bad router / gpu / tokens");
  // App. B.3: L_i <- max(0, L_i - tokens * f_tok)
  r->load[gpu] = std::max(0.0, r->load[gpu] - (double)tokens * r->cfg.f_tok);
  return ASYNCEP_OK;
}

}  // extern "C"
