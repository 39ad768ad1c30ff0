/*
 * oracle/moe_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct CPU oracle for the AsyncEP MoE-layer hot path of
 * arxiv/paper_2605_02960 ("MoE-Prefill").  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.  It shares
 * no code, header, table or constant generator with the CUDA path
 * (paper_2605_02960_b200/csrc); neither includes the other.
 *
 * All arithmetic is IEEE fp64 (inputs are fp32 arrays holding bf16- or e4m3-
 * representable values, i.e. exact).  Every function cites the passage it follows:
 *   PAPER.md:61  (S2.2 "Mixture-of-Experts"): "E parallel experts, each a two-layer
 *                MLP; a lightweight router dispatches each token to its top-k experts
 *                ... and sums their outputs."
 *   PAPER.md:311 (S6.2 "Weight layout and execution"): experts sharded 1/N by
 *                expert index; the AllGather re-assembles the full set.
 *   PAPER.md:315-319 (S6.2, Eq. 1): T = t_EP x F_GPU x gamma.
 *   PAPER.md:544 (S8.6 Tier 1): AsyncEP does not change the layer's math.
 * Readings of silent points (R1..R15) are listed in DESIGN.md S3 and in SURVEY.md S8(c2).
 *
 * Loop order: the per-token definition is evaluated expert-major with a block of
 * tokens per weight row (so a weight row is read once per block).  Each dot product
 * is still a plain sequential sum over the contraction index -- no reassociation.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORACLE_OK 0
#define ORACLE_EINVAL 1
#define ORACLE_ENOMEM 2

int oracle_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

void oracle_set_num_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

/* silu(z) = z * sigma(z) = z / (1 + e^{-z})  -- reading R4 (SwiGLU expert). */
static double silu(double z) { return z / (1.0 + exp(-z)); }

/*
 * Router of one token ("router dispatches each token to its top-k experts"),
 * readings R1-R3:
 *   logits[e] = sum_i Wr[e,i] * x[i]                              (fp64 here)
 *   p         = softmax(logits) over all E experts
 *   S         = top-k experts by logit, descending; ties -> lower expert id  (R2)
 *   w_j       = p[S_j] / sum_{j'} p[S_j'] if norm_topk else p[S_j]          (R1)
 *   gap       = logit of k-th minus logit of (k+1)-th choice (inf if k == E)
 * If ids_in != NULL the selection is taken from ids_in (reading R15: the GPU's
 * choice for near-tie tokens) and only the weights are computed here.
 */
static void route_one(const float *x, const float *wr, int H, int E, int k, int norm_topk,
                      const int32_t *ids_in, double *logits, int32_t *ids, double *w,
                      double *gap, char *taken) {
    for (int e = 0; e < E; ++e) {
        double s = 0.0;
        const float *row = wr + (size_t)e * H;
        for (int i = 0; i < H; ++i) s += (double)row[i] * (double)x[i];
        logits[e] = s;
    }
    /* softmax over all E (max-subtracted for range; mathematically identical) */
    double m = logits[0];
    for (int e = 1; e < E; ++e) if (logits[e] > m) m = logits[e];
    double z = 0.0;
    for (int e = 0; e < E; ++e) z += exp(logits[e] - m);

    memset(taken, 0, (size_t)E);
    if (ids_in) {
        for (int j = 0; j < k; ++j) { ids[j] = ids_in[j]; taken[ids_in[j]] = 1; }
    } else {
        for (int j = 0; j < k; ++j) {
            int best = -1;
            for (int e = 0; e < E; ++e) {
                if (taken[e]) continue;
                if (best < 0 || logits[e] > logits[best]) best = e;  /* strict: lower id wins ties */
            }
            ids[j] = best;
            taken[best] = 1;
        }
    }
    if (gap) {
        int nxt = -1;
        for (int e = 0; e < E; ++e) {
            if (taken[e]) continue;
            if (nxt < 0 || logits[e] > logits[nxt]) nxt = e;
        }
        double kth = logits[ids[0]];
        for (int j = 1; j < k; ++j) if (logits[ids[j]] < kth) kth = logits[ids[j]];
        *gap = (nxt < 0) ? INFINITY : (kth - logits[nxt]);
    }
    double psel = 0.0;
    for (int j = 0; j < k; ++j) {
        w[j] = exp(logits[ids[j]] - m) / z;   /* p_{S_j} */
        psel += w[j];
    }
    if (norm_topk)
        for (int j = 0; j < k; ++j) w[j] = w[j] / psel;
}

/*
 * oracle_router: the router for T tokens.  x [T,H], wr [E,H] (fp32 holding bf16 values).
 * Outputs (any may be NULL except ids, w): logits [T,E] fp64, ids [T,k] int32,
 * w [T,k] fp64, counts [E] int64 (= histogram of ids), gap [T] fp64.
 */
int oracle_router(const float *x, const float *wr, int64_t T, int H, int E, int k, int norm_topk,
                  const int32_t *ids_in, double *logits, int32_t *ids, double *w,
                  int64_t *counts, double *gap) {
    if (T < 0 || H <= 0 || E <= 0 || k <= 0 || k > E || !x || !wr || !ids || !w)
        return ORACLE_EINVAL;
    int err = 0;
#pragma omp parallel
    {
        double *lg = (double *)malloc(sizeof(double) * (size_t)E);
        char *taken = (char *)malloc((size_t)E);
        if (!lg || !taken) {
#pragma omp atomic write
            err = 1;
        } else {
#pragma omp for schedule(static)
            for (int64_t t = 0; t < T; ++t) {
                route_one(x + (size_t)t * H, wr, H, E, k, norm_topk,
                          ids_in ? ids_in + (size_t)t * k : NULL, lg,
                          ids + (size_t)t * k, w + (size_t)t * k, gap ? gap + t : NULL, taken);
                if (logits) memcpy(logits + (size_t)t * E, lg, sizeof(double) * (size_t)E);
            }
        }
        free(lg);
        free(taken);
    }
    if (err) return ORACLE_ENOMEM;
    if (counts) {
        for (int e = 0; e < E; ++e) counts[e] = 0;
        for (int64_t i = 0; i < T * (int64_t)k; ++i) counts[ids[i]] += 1;
    }
    return ORACLE_OK;
}

/*
 * One expert, "a two-layer MLP" in its gated SwiGLU form (reading R4,
 * SPEC.md:57 3*H*h weights per expert), for a block of nb tokens:
 *   g = Wg x ; u = Wu x ; a = silu(g) * u ; o = Wd a
 * wg, wu: [h,H]; wd: [H,h]; xt: [H][nb] (token block, transposed so that the
 * independent per-token sums sit side by side); out: [nb][H].
 * identity != 0 replaces the MLP with o = x (test hook for the plumbing pin).
 */
#define NB 32
static void quant_row_e4m3(const float *v, int n, double *out);
static void quant_row_mx(const float *v, int n, double *out);
static float to_bf16(double v);

static void expert_block(const float *wg, const float *wu, const float *wd, int H, int h, int nb,
                         const double *xt, double *at, double *out, int identity, int act_quant) {
    if (identity) {
        for (int b = 0; b < nb; ++b)
            for (int i = 0; i < H; ++i) out[(size_t)b * H + i] = xt[(size_t)i * NB + b];
        return;
    }
    double g[NB], u[NB];
    for (int r = 0; r < h; ++r) {
        const float *rg = wg + (size_t)r * H, *ru = wu + (size_t)r * H;
        for (int b = 0; b < NB; ++b) { g[b] = 0.0; u[b] = 0.0; }
        for (int i = 0; i < H; ++i) {
            const double cg = rg[i], cu = ru[i];
            const double *xi = xt + (size_t)i * NB;
            for (int b = 0; b < NB; ++b) { g[b] += cg * xi[b]; u[b] += cu * xi[b]; }
        }
        for (int b = 0; b < NB; ++b) at[(size_t)r * NB + b] = silu(g[b]) * u[b];
    }
    if (act_quant) {  /* emulate the GPU: intermediate -> bf16 -> per-row e4m3 (R5, R6), or
                         act_quant == 2: -> bf16 -> MX 1x32 blocks with E8M0 scales (R6b) */
        float *row = (float *)malloc(sizeof(float) * (size_t)h);
        double *dq = (double *)malloc(sizeof(double) * (size_t)h);
        for (int b = 0; b < nb; ++b) {
            for (int r = 0; r < h; ++r) row[r] = to_bf16(at[(size_t)r * NB + b]);
            if (act_quant == 2) quant_row_mx(row, h, dq);
            else quant_row_e4m3(row, h, dq);
            for (int r = 0; r < h; ++r) at[(size_t)r * NB + b] = dq[r];
        }
        free(row); free(dq);
    }
    double o[NB];
    for (int r = 0; r < H; ++r) {
        const float *rd = wd + (size_t)r * h;
        for (int b = 0; b < NB; ++b) o[b] = 0.0;
        for (int i = 0; i < h; ++i) {
            const double c = rd[i];
            const double *ai = at + (size_t)i * NB;
            for (int b = 0; b < NB; ++b) o[b] += c * ai[b];
        }
        for (int b = 0; b < nb; ++b) out[(size_t)b * H + r] = o[b];
    }
}

/*
 * oracle_moe_layer: the MoE FFN forward of one layer for T tokens, by definition
 * (SURVEY.md S8(c1)):
 *   (ids, w) = router(x)                                              [oracle_router]
 *   o_{t,j}  = expert_{ids[t,j]}(x_t)                                 [expert_block]
 *   y_t      = (add_residual ? x_t : 0) + sum_{j=0..k-1} w[t,j] * o_{t,j}   (j order; R9)
 * Weights in natural layout: wg, wu [E,h,H]; wd [E,H,h]; wr [E,H].
 * ids_in (nullable [T,k]) forces the routing (R15).  Outputs: y [T,H] fp64 (required);
 * ids [T,k], w [T,k], logits [T,E], gap [T] (nullable).
 */
int oracle_moe_layer(const float *x, const float *wr, const float *wg, const float *wu,
                     const float *wd, int64_t T, int H, int E, int k, int h, int norm_topk,
                     int add_residual, int identity_experts, int act_quant, const int32_t *ids_in,
                     double *y, int32_t *ids_out, double *w_out, double *logits, double *gap) {
    if (T < 0 || H <= 0 || E <= 0 || k <= 0 || k > E || h <= 0 || !x || !wr || !y) return ORACLE_EINVAL;
    if (!identity_experts && (!wg || !wu || !wd)) return ORACLE_EINVAL;
    if (T == 0) return ORACLE_OK;
    const size_t TK = (size_t)T * (size_t)k;
    int32_t *ids = ids_out ? ids_out : (int32_t *)malloc(sizeof(int32_t) * TK);
    double *w = w_out ? w_out : (double *)malloc(sizeof(double) * TK);
    double *o = (double *)malloc(sizeof(double) * TK * (size_t)H);  /* o_{t,j} */
    int64_t *cnt = (int64_t *)calloc((size_t)E + 1, sizeof(int64_t));
    int64_t *lst = (int64_t *)malloc(sizeof(int64_t) * TK);  /* (t*k+j) entries grouped by expert */
    int rc = ORACLE_OK;
    if (!ids || !w || !o || !cnt || !lst) { rc = ORACLE_ENOMEM; goto done; }
    rc = oracle_router(x, wr, T, H, E, k, norm_topk, ids_in, logits, ids, w, NULL, gap);
    if (rc) goto done;

    /* group (t,j) entries by expert, in (t,j) order */
    for (size_t i = 0; i < TK; ++i) cnt[ids[i] + 1] += 1;
    for (int e = 0; e < E; ++e) cnt[e + 1] += cnt[e];
    {
        int64_t *fill = (int64_t *)malloc(sizeof(int64_t) * (size_t)E);
        if (!fill) { rc = ORACLE_ENOMEM; goto done; }
        for (int e = 0; e < E; ++e) fill[e] = cnt[e];
        for (size_t i = 0; i < TK; ++i) lst[fill[ids[i]]++] = (int64_t)i;
        free(fill);
    }

    /* work items: (expert, block of NB entries) */
    {
        int64_t nitems = 0;
        for (int e = 0; e < E; ++e) nitems += (cnt[e + 1] - cnt[e] + NB - 1) / NB;
        int64_t *item_e = (int64_t *)malloc(sizeof(int64_t) * (size_t)(nitems + 1));
        int64_t *item_s = (int64_t *)malloc(sizeof(int64_t) * (size_t)(nitems + 1));
        if (!item_e || !item_s) { free(item_e); free(item_s); rc = ORACLE_ENOMEM; goto done; }
        int64_t it = 0;
        for (int e = 0; e < E; ++e)
            for (int64_t s = cnt[e]; s < cnt[e + 1]; s += NB) { item_e[it] = e; item_s[it] = s; ++it; }
        int err = 0;
#pragma omp parallel
        {
            double *xt = (double *)malloc(sizeof(double) * (size_t)H * NB);
            double *at = (double *)malloc(sizeof(double) * (size_t)h * NB);
            double *ob = (double *)malloc(sizeof(double) * (size_t)H * NB);
            double *xq = (double *)malloc(sizeof(double) * (size_t)H);
            if (!xt || !at || !ob || !xq) {
#pragma omp atomic write
                err = 1;
            } else {
#pragma omp for schedule(dynamic, 1)
                for (int64_t q = 0; q < nitems; ++q) {
                    const int e = (int)item_e[q];
                    const int64_t s0 = item_s[q];
                    const int nb = (int)((cnt[e + 1] - s0) < NB ? (cnt[e + 1] - s0) : NB);
                    for (int b = 0; b < NB; ++b) {
                        const int64_t t = (b < nb) ? lst[s0 + b] / k : -1;
                        if (t >= 0 && act_quant) {  /* the experts see the e4m3-quantised token (R6) */
                            quant_row_e4m3(x + (size_t)t * H, H, xq);
                            for (int i = 0; i < H; ++i) xt[(size_t)i * NB + b] = xq[i];
                        } else {
                            for (int i = 0; i < H; ++i)
                                xt[(size_t)i * NB + b] = (t >= 0) ? (double)x[(size_t)t * H + i] : 0.0;
                        }
                    }
                    expert_block(identity_experts ? NULL : wg + (size_t)e * h * H,
                                 identity_experts ? NULL : wu + (size_t)e * h * H,
                                 identity_experts ? NULL : wd + (size_t)e * H * h, H, h, nb, xt, at,
                                 ob, identity_experts, act_quant);
                    for (int b = 0; b < nb; ++b)
                        memcpy(o + (size_t)lst[s0 + b] * H, ob + (size_t)b * H, sizeof(double) * (size_t)H);
                }
            }
            free(xt); free(at); free(ob); free(xq);
        }
        free(item_e); free(item_s);
        if (err) { rc = ORACLE_ENOMEM; goto done; }
    }

    /* weighted combine, j order, plus optional residual ("sums their outputs"; R9) */
#pragma omp parallel for schedule(static)
    for (int64_t t = 0; t < T; ++t) {
        double *yt = y + (size_t)t * H;
        for (int i = 0; i < H; ++i) yt[i] = add_residual ? (double)x[(size_t)t * H + i] : 0.0;
        for (int j = 0; j < k; ++j) {
            const double wj = w[(size_t)t * k + j];
            const double *ot = o + ((size_t)t * k + j) * H;
            for (int i = 0; i < H; ++i) yt[i] += wj * ot[i];
        }
    }
done:
    if (!ids_out) free(ids);
    if (!w_out) free(w);
    free(o); free(cnt); free(lst);
    return rc;
}

/* ---------------- FP8 (reading R6) ---------------- */

/* OCP E4M3 (FN) decode: 1 sign, 4 exponent (bias 7), 3 mantissa; no inf; 0x7F/0xFF = NaN. */
double oracle_e4m3_decode(uint8_t b) {
    const int s = b >> 7, ex = (b >> 3) & 0xF, m = b & 7;
    double v;
    if (ex == 0xF && m == 7) return NAN;
    if (ex == 0) v = ldexp((double)m / 8.0, -6);
    else v = ldexp(1.0 + (double)m / 8.0, ex - 7);
    return s ? -v : v;
}

void oracle_e4m3_decode_array(const uint8_t *q, int64_t n, float *out) {
    for (int64_t i = 0; i < n; ++i) out[i] = (float)oracle_e4m3_decode(q[i]);
}

/*
 * Round-to-nearest-even, saturating (satfinite) encode of a double into E4M3 --
 * the brute-force definition: pick the representable finite value nearest to v,
 * ties to the even code; |v| beyond 448 saturates to +-448.  Used by the
 * activation-quantisation emulation mode (R6).
 */
uint8_t oracle_e4m3_encode(double v) {
    if (isnan(v)) return 0x7F;
    const int neg = signbit(v) ? 1 : 0;
    double a = fabs(v);
    int best = 0;
    double bestd = INFINITY;
    for (int c = 0; c <= 0x7E; ++c) {  /* all finite non-negative codes */
        const double d = fabs(oracle_e4m3_decode((uint8_t)c) - a);
        if (d < bestd || (d == bestd && (c & 1) == 0 && (best & 1) == 1)) { bestd = d; best = c; }
    }
    return (uint8_t)(best | (neg << 7));
}

/*
 * The same encoder computed arithmetically (pinned against oracle_e4m3_encode by an
 * exhaustive test): |v| = m * 2^e; normal codes carry 3 mantissa bits, subnormals are
 * multiples of 2^-9; round half to even; saturate at 448.
 */
uint8_t oracle_e4m3_encode_fast(double v) {
    if (isnan(v)) return 0x7F;
    const int neg = signbit(v) ? 1 : 0;
    double a = fabs(v);
    int code;
    if (a >= 448.0) {
        code = 0x7E;
    } else if (a < ldexp(1.0, -6)) {                 /* subnormal range: step 2^-9 */
        double q = a / ldexp(1.0, -9);
        double f = floor(q);
        double r = q - f;
        int m = (int)f;
        if (r > 0.5 || (r == 0.5 && (m & 1))) m += 1;  /* m == 8 is the smallest normal, code 0x08 */
        code = m;
    } else {
        int ex;
        double fr = frexp(a, &ex);                    /* a = fr * 2^ex, fr in [0.5, 1) */
        int e = ex - 1;                               /* a = (2 fr) * 2^e, 2fr in [1, 2) */
        double q = (2.0 * fr - 1.0) * 8.0;            /* mantissa in units of 1/8 */
        double f = floor(q);
        double r = q - f;
        int m = (int)f;
        if (r > 0.5 || (r == 0.5 && (m & 1))) m += 1;
        if (m == 8) { m = 0; e += 1; }
        code = ((e + 7) << 3) | m;
        if (code > 0x7E) code = 0x7E;
    }
    return (uint8_t)(code | (neg << 7));
}

/* bf16 round-to-nearest-even of a double (via float), as the GPU stores the intermediate (R5) */
static float to_bf16(double v) {
    float f = (float)v;
    uint32_t u;
    memcpy(&u, &f, 4);
    if ((u & 0x7F800000u) == 0x7F800000u) return f;  /* inf / nan */
    u = (u + 0x7FFFu + ((u >> 16) & 1u)) & 0xFFFF0000u;
    memcpy(&f, &u, 4);
    return f;
}

/* Exported for the pins (tests/test_oracle_pins.py): to_bf16 over an array. */
void oracle_to_bf16_array(const double *v, int64_t n, float *out) {
    for (int64_t i = 0; i < n; ++i) out[i] = to_bf16(v[i]);
}

/*
 * FP8 activation-quantisation emulation (reading R6, the rule the CUDA path applies):
 *   amax = max_i |v_i| (fp32); inv = 448 / amax (fp32); q_i = RNE_satfinite_e4m3(fp32(v_i * inv));
 *   result_i = decode(q_i) * (amax / 448) (fp32 scale, product in fp64)
 */
static void quant_row_e4m3(const float *v, int n, double *out) {
    float amax = 0.f;
    for (int i = 0; i < n; ++i) { const float a = fabsf(v[i]); if (a > amax) amax = a; }
    if (amax == 0.f) { for (int i = 0; i < n; ++i) out[i] = 0.0; return; }
    const float inv = 448.0f / amax;
    const float sc = amax / 448.0f;
    for (int i = 0; i < n; ++i) {
        const float p = v[i] * inv;
        out[i] = oracle_e4m3_decode(oracle_e4m3_encode_fast((double)p)) * (double)sc;
    }
}

/*
 * MX intermediate quantisation (reading R6b, S3; OCP MX layout: blocks of 32
 * consecutive elements along the contraction, one power-of-two E8M0 scale per block):
 *   per block of 32:  amax = max |v_i| (the bf16 values, exact);
 *                     e = the smallest integer with amax <= 448 * 2^e, clamped to [-127, 127];
 *                     result_i = decode(RNE_satfinite_e4m3(v_i / 2^e)) * 2^e.
 * (The smallest such e maps the block's amax into (224, 448]: no element saturates.)
 * n must be a multiple of 32 (the FFN width is a multiple of 128).
 */
static void quant_row_mx(const float *v, int n, double *out) {
    for (int b0 = 0; b0 < n; b0 += 32) {
        double amax = 0.0;
        for (int i = b0; i < b0 + 32 && i < n; ++i) { const double a = fabs((double)v[i]); if (a > amax) amax = a; }
        int e = -127;
        while (e < 127 && amax > ldexp(448.0, e)) ++e;
        for (int i = b0; i < b0 + 32 && i < n; ++i)
            out[i] = ldexp(oracle_e4m3_decode(oracle_e4m3_encode_fast(ldexp((double)v[i], -e))), e);
    }
}

/* Exported for the pins: the MX rule over one row of n values (n a multiple of 32). */
void oracle_quant_row_mx(const float *v, int n, double *out) { quant_row_mx(v, n, out); }

/* ---------------- Saturation threshold, Eq. 1 ---------------- */

/* Eq. 1 literal: T = t_EP * F_GPU * gamma [FLOPs]. */
double oracle_eq1_threshold(double t_ep, double f_gpu, double gamma) { return t_ep * f_gpu * gamma; }

/*
 * Per-layer, token-denominated reading (R11, R12):
 *   W_layer = E*3*H*h*b                        (SPEC.md:57,61 per-expert 3*H*h*b)
 *   t_AG    = (N-1)/N * W_layer / BW_AG        (receive bytes of the AllGather / bandwidth)
 *   T_FLOPs = gamma * t_AG * F                 (Eq. 1 with t_EP = t_AG)
 *   T_tok   = T_FLOPs / (6*k*H*h)              (grouped-GEMM FLOPs per token per layer)
 * N == 1 -> 0 (nothing to gather).
 */
int oracle_saturation_T(int E, int k, int H, int h, double bytes_per_elem, int N, double gamma,
                        double flops_per_s, double ag_bytes_per_s, double *t_tok, double *t_flops) {
    if (E <= 0 || k <= 0 || H <= 0 || h <= 0 || N <= 0 || bytes_per_elem <= 0 || gamma < 1.0 ||
        flops_per_s <= 0 || ag_bytes_per_s <= 0)
        return ORACLE_EINVAL;
    const double w_layer = (double)E * 3.0 * (double)H * (double)h * bytes_per_elem;
    const double t_ag = ((double)(N - 1) / (double)N) * w_layer / ag_bytes_per_s;
    const double tf = oracle_eq1_threshold(t_ag, flops_per_s, gamma);
    if (t_flops) *t_flops = tf;
    if (t_tok) *t_tok = tf / (6.0 * (double)k * (double)H * (double)h);
    return ORACLE_OK;
}

/* Calibrated form, App. B.4 Eq. 3: T = gamma * (t_e/t_c) * C_dummy,
 * collapsing to gamma * C_dummy when t_e <= t_c. */
double oracle_calibrated_T(double gamma, double t_e, double t_c, double c_dummy) {
    const double r = (t_e <= t_c) ? 1.0 : t_e / t_c;
    return gamma * r * c_dummy;
}
