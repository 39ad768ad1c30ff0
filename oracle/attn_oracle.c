/*
 * oracle/attn_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain fp64 CPU oracle for NEXT-3: the data-parallel attention layer
 * that precedes each MoE layer, in the paper's KV-cache-free prefill mode.
 *   PAPER.md:275 (S5 "System overview"): "the backend runs each batch as pure DP attention";
 *   PAPER.md:311 (S6.2): "each GPU holds a full replica of attention weights ... After
 *                computing attention locally, each GPU evaluates the current MoE layer";
 *   PAPER.md:351-353 (S6.3 "KV dimension: KV-cache-free execution"): "disables KV storage
 *                entirely and computes attention on the fly [flashattention]".
 * The paper fixes no attention architecture; reading R19 (S3) takes the
 * Qwen3-MoE decoder block the benchmark model uses: pre-RMSNorm, fused QKV projection,
 * per-head RMSNorm of q and k (QK-norm), rotary embedding (rotate-half, theta 1e6),
 * causal grouped-query attention per prompt, output projection + residual, and the
 * post-attention RMSNorm that feeds the MoE router.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
 * may load this library.  It shares nothing with paper_2605_02960_b200/csrc.  Every value is
 * fp64; inputs are fp32 arrays holding bf16-representable values.  Every dot product is a
 * plain sequential sum; softmax is the textbook exp(s - max) / sum.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORACLE_OK 0
#define ORACLE_EINVAL 1
#define ORACLE_ENOMEM 2

/* RMSNorm (Qwen3 convention): out[i] = x[i] / sqrt(mean_j x[j]^2 + eps) * w[i]. */
static void rmsnorm_row(const double *x, const float *w, int n, double eps, double *out) {
    double ss = 0.0;
    for (int i = 0; i < n; ++i) ss += x[i] * x[i];
    const double r = 1.0 / sqrt(ss / n + eps);
    for (int i = 0; i < n; ++i) out[i] = x[i] * r * (w ? (double)w[i] : 1.0);
}

int oracle_rmsnorm(const float *x, const float *w, int64_t rows, int n, double eps, double *out) {
    if (!x || !out || rows < 0 || n <= 0) return ORACLE_EINVAL;
    double *tmp = (double *)malloc(sizeof(double) * (size_t)n);
    if (!tmp) return ORACLE_ENOMEM;
    for (int64_t r = 0; r < rows; ++r) {
        for (int i = 0; i < n; ++i) tmp[i] = x[r * n + i];
        rmsnorm_row(tmp, w, n, eps, out + r * n);
    }
    free(tmp);
    return ORACLE_OK;
}

/* Rotary embedding, rotate-half form: for i < d/2, with inv_freq_i = theta^(-2i/d) and
 * angle = pos * inv_freq_i,
 *   out[i]       = x[i] cos(angle) - x[i + d/2] sin(angle)
 *   out[i + d/2] = x[i + d/2] cos(angle) + x[i] sin(angle).                            */
static void rope_vec(double *x, int d, int32_t pos, double theta) {
    const int half = d / 2;
    for (int i = 0; i < half; ++i) {
        const double ang = (double)pos * pow(theta, -2.0 * i / d);
        const double c = cos(ang), s = sin(ang);
        const double a = x[i], b = x[i + half];
        x[i] = a * c - b * s;
        x[i + half] = b * c + a * s;
    }
}

int oracle_rope(double *x, const int32_t *pos, int64_t T, int nh, int d, double theta) {
    if (!x || !pos || T < 0 || nh <= 0 || d <= 0 || d % 2) return ORACLE_EINVAL;
    for (int64_t t = 0; t < T; ++t)
        for (int h = 0; h < nh; ++h) rope_vec(x + (t * nh + h) * d, d, pos[t], theta);
    return ORACLE_OK;
}

/* Softmax attention of one query against keys/values [j0, j1) of one kv head:
 *   s_j = scale * <q, k_j>;  p_j = exp(s_j - max s) / sum exp(s - max s);  o = sum_j p_j v_j */
static void attend_one(const double *q, const double *k, const double *v, int64_t j0, int64_t j1,
                       int64_t kv_stride, int d, double scale, double *s, double *o) {
    double mx = -INFINITY;
    for (int64_t j = j0; j < j1; ++j) {
        double acc = 0.0;
        const double *kj = k + j * kv_stride;
        for (int c = 0; c < d; ++c) acc += q[c] * kj[c];
        s[j - j0] = scale * acc;
        if (s[j - j0] > mx) mx = s[j - j0];
    }
    double den = 0.0;
    for (int64_t j = j0; j < j1; ++j) {
        s[j - j0] = exp(s[j - j0] - mx);
        den += s[j - j0];
    }
    for (int c = 0; c < d; ++c) o[c] = 0.0;
    for (int64_t j = j0; j < j1; ++j) {
        const double p = s[j - j0] / den;
        const double *vj = v + j * kv_stride;
        for (int c = 0; c < d; ++c) o[c] += p * vj[c];
    }
}

/* Grouped-query attention over a packed batch of prompts (KV-cache-free prefill):
 * prompt b holds tokens [cu[b], cu[b+1]); query head h reads kv head h / (Hq / Hkv); with
 * causal != 0 the query at position t attends to keys at positions <= t of its own prompt.
 * k and v [T, Hkv, d]; rows (nullable) lists the query tokens to evaluate; q and out hold
 * one row per evaluated query: [nrows, Hq, d] (or [T, Hq, d] when rows is NULL). */
int oracle_attention(const double *q, const double *k, const double *v, const int32_t *cu, int B, int Hq, int Hkv,
                     int d, int causal, double scale, const int64_t *rows, int64_t nrows, double *out) {
    if (!q || !k || !v || !cu || !out || B < 0 || Hq <= 0 || Hkv <= 0 || Hq % Hkv || d <= 0) return ORACLE_EINVAL;
    const int64_t T = cu[B];
    const int64_t n = rows ? nrows : T;
    const int group = Hq / Hkv;
    int64_t maxlen = 1;
    for (int b = 0; b < B; ++b) {
        if (cu[b + 1] < cu[b]) return ORACLE_EINVAL;
        if (cu[b + 1] - cu[b] > maxlen) maxlen = cu[b + 1] - cu[b];
    }
    int err = ORACLE_OK;
#pragma omp parallel
    {
        double *s = (double *)malloc(sizeof(double) * (size_t)maxlen);
        if (!s) err = ORACLE_ENOMEM;
#pragma omp for schedule(dynamic, 1)
        for (int64_t i = 0; i < n; ++i) {
            if (!s) continue;
            const int64_t t = rows ? rows[i] : i;
            int b = 0;
            while (b < B && cu[b + 1] <= t) ++b;
            if (b >= B || t < 0) {
                err = ORACLE_EINVAL;
                continue;
            }
            const int64_t j1 = causal ? t + 1 : cu[b + 1];
            for (int h = 0; h < Hq; ++h)
                attend_one(q + (i * Hq + h) * d, k + (int64_t)(h / group) * d, v + (int64_t)(h / group) * d, cu[b],
                           j1, (int64_t)Hkv * d, d, scale, s, out + (i * Hq + h) * d);
        }
        free(s);
    }
    return err;
}

/* One DP attention layer (reading R19), for the query tokens in rows (nullable = all):
 *   xn   = RMSNorm(x; w_ln1)                                   [T, H]
 *   qkv  = xn . W_qkv^T,  W_qkv [(Hq + 2 Hkv) d, H]: rows [0, Hq d) = q, then k, then v
 *   q_h  = RoPE(RMSNorm(q_h; w_qn)),  k_g = RoPE(RMSNorm(k_g; w_kn))   (per head, d-long)
 *   o    = causal GQA attention per prompt, scale 1/sqrt(d)
 *   x'   = x + o . W_o^T,  W_o [H, Hq d]
 *   xn2  = RMSNorm(x'; w_ln2)                                  (the MoE router's input)
 * Positions restart at 0 in every prompt.  K and V are formed only for the tokens some
 * requested query can see. */
int oracle_attn_layer(const float *x, int64_t T, int H, const int32_t *cu, int B, int Hq, int Hkv, int d,
                      const float *w_ln1, const float *w_qkv, const float *w_qn, const float *w_kn, const float *w_o,
                      const float *w_ln2, double eps, double theta, const int64_t *rows, int64_t nrows, float *x_out,
                      float *xn2_out) {
    if (!x || !cu || !w_qkv || !w_o || !x_out || B <= 0 || cu[B] != T || Hq % Hkv || d % 2) return ORACLE_EINVAL;
    const int64_t n = rows ? nrows : T;
    const int nq = Hq * d, nkv = Hkv * d;
    char *need = (char *)calloc((size_t)T, 1);           /* tokens whose k/v some query reads */
    int32_t *pos = (int32_t *)malloc(sizeof(int32_t) * (size_t)T);
    double *K = (double *)malloc(sizeof(double) * (size_t)T * nkv);
    double *V = (double *)malloc(sizeof(double) * (size_t)T * nkv);
    double *Q = (double *)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1) * nq);
    double *O = (double *)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1) * nq);
    int64_t *qrows = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
    if (!need || !pos || !K || !V || !Q || !O || !qrows) {
        free(need); free(pos); free(K); free(V); free(Q); free(O); free(qrows);
        return ORACLE_ENOMEM;
    }
    for (int b = 0; b < B; ++b)
        for (int64_t t = cu[b]; t < cu[b + 1]; ++t) pos[t] = (int32_t)(t - cu[b]);
    for (int64_t i = 0; i < n; ++i) {
        const int64_t t = rows ? rows[i] : i;
        qrows[i] = t;
        int b = 0;
        while (b < B && cu[b + 1] <= t) ++b;
        for (int64_t u = cu[b]; u <= t; ++u) need[u] = 1;
    }
    /* token-wise projections (needed tokens only) */
#pragma omp parallel
    {
        double *xr = (double *)malloc(sizeof(double) * (size_t)H);
        double *xn = (double *)malloc(sizeof(double) * (size_t)H);
#pragma omp for schedule(dynamic, 4)
        for (int64_t t = 0; t < T; ++t) {
            if (!need[t]) continue;
            for (int i = 0; i < H; ++i) xr[i] = x[t * H + i];
            rmsnorm_row(xr, w_ln1, H, eps, xn);
            for (int c = 0; c < nkv; ++c) {
                double ak = 0.0, av = 0.0;
                const float *wk = w_qkv + (int64_t)(nq + c) * H, *wv = w_qkv + (int64_t)(nq + nkv + c) * H;
                for (int i = 0; i < H; ++i) ak += xn[i] * wk[i];
                for (int i = 0; i < H; ++i) av += xn[i] * wv[i];
                K[t * nkv + c] = ak;
                V[t * nkv + c] = av;
            }
            for (int g = 0; g < Hkv; ++g) {
                double tmp[1024];
                rmsnorm_row(K + t * nkv + g * d, w_kn, d, eps, tmp);
                rope_vec(tmp, d, pos[t], theta);
                memcpy(K + t * nkv + g * d, tmp, sizeof(double) * d);
            }
        }
#pragma omp for schedule(dynamic, 4)
        for (int64_t i = 0; i < n; ++i) {
            const int64_t t = qrows[i];
            for (int j = 0; j < H; ++j) xr[j] = x[t * H + j];
            rmsnorm_row(xr, w_ln1, H, eps, xn);
            for (int c = 0; c < nq; ++c) {
                double a = 0.0;
                const float *wq = w_qkv + (int64_t)c * H;
                for (int j = 0; j < H; ++j) a += xn[j] * wq[j];
                Q[i * nq + c] = a;
            }
            for (int h = 0; h < Hq; ++h) {
                double tmp[1024];
                rmsnorm_row(Q + i * nq + h * d, w_qn, d, eps, tmp);
                rope_vec(tmp, d, pos[t], theta);
                memcpy(Q + i * nq + h * d, tmp, sizeof(double) * d);
            }
        }
        free(xr);
        free(xn);
    }
    int err = oracle_attention(Q, K, V, cu, B, Hq, Hkv, d, 1, 1.0 / sqrt((double)d), qrows, n, O);
    if (err == ORACLE_OK) {
#pragma omp parallel
        {
            double *xo = (double *)malloc(sizeof(double) * (size_t)H);
            double *xn = (double *)malloc(sizeof(double) * (size_t)H);
#pragma omp for schedule(dynamic, 4)
            for (int64_t i = 0; i < n; ++i) {
                const int64_t t = qrows[i];
                for (int r = 0; r < H; ++r) {
                    double a = 0.0;
                    const float *wo = w_o + (int64_t)r * nq;
                    for (int c = 0; c < nq; ++c) a += O[i * nq + c] * wo[c];
                    xo[r] = (double)x[t * H + r] + a;
                }
                rmsnorm_row(xo, w_ln2, H, eps, xn);
                for (int r = 0; r < H; ++r) {
                    x_out[i * H + r] = (float)xo[r];
                    if (xn2_out) xn2_out[i * H + r] = (float)xn[r];
                }
            }
            free(xo);
            free(xn);
        }
    }
    free(need); free(pos); free(K); free(V); free(Q); free(O); free(qrows);
    return err;
}
