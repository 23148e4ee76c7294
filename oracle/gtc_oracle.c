/*
 * gtc_oracle.c -- plain, slow, obviously-correct CPU oracle for GTC.
 *
 * TEST INFRASTRUCTURE ONLY (see gtc_oracle.h).  Single-threaded, no blocking,
 * no vector tricks: one loop per step of PAPER.md:222, in the paper's order.
 * Build: gcc -O2 -fno-fast-math -ffp-contract=off -fPIC -shared -lm
 */
#include "gtc_oracle.h"

#include <math.h>
#include <stdlib.h>

static int oracle_check_args(int64_t n, float tau)
{
    /* R3: the index lives in 31 bits of the 32-bit word ("single 32-bit
     * integer field", one bit spent on the sign). */
    if (n < 0 || n >= ((int64_t)1 << 31)) return ORACLE_EDIM;
    /* tau is "a constant" threshold; S:128 requires tau > 0. */
    if (!(tau > 0.0f) || isinf(tau)) return ORACLE_EINVAL;
    return ORACLE_OK;
}

int oracle_encode(int64_t n, float tau, int cmp_mode,
                  const float* g, float* r,
                  uint32_t* words, int64_t* k_out, int* nonfinite_out)
{
    int st = oracle_check_args(n, tau);
    if (st != ORACLE_OK) return st;
    if (cmp_mode != ORACLE_CMP_GT && cmp_mode != ORACLE_CMP_GE) return ORACLE_EINVAL;

    int64_t k = 0;
    int nonfinite = 0;
    for (int64_t i = 0; i < n; ++i) {
        /* Step 1 ("residual gradients ... are aggregated locally"):
         * the new gradient is added to what was not sent before (R5: r starts
         * at 0 and is never reset; that is the caller's buffer). */
        float v = (g != NULL) ? (r[i] + g[i]) : r[i];
        if (!isfinite(v)) nonfinite = 1; /* R9 */

        /* Step 2 ("absolute magnitude is greater than a constant"). */
        int sel;
        if (cmp_mode == ORACLE_CMP_GT) sel = fabsf(v) > tau;
        else                           sel = fabsf(v) >= tau;

        if (sel) {
            /* Step 3 ("1-bit quantization ... deltas of +-tau"): one
             * quantum of size tau with the sign of v leaves the worker (R2);
             * the rest stays in the residual. */
            int neg = (v < 0.0f);
            float sent = neg ? -tau : tau;
            r[i] = v - sent;
            /* Step 4 ("packing quantized gradient and integer index into
             * single 32-bit integer field"), layout R3: index in bits 31..1,
             * bit 0 = 1 for -tau.  Ascending i gives the canonical order (R4). */
            words[k] = ((uint32_t)i << 1) | (uint32_t)neg;
            k = k + 1;
        } else {
            r[i] = v;
        }
    }
    *k_out = k;
    if (nonfinite_out) *nonfinite_out = nonfinite;
    return ORACLE_OK;
}

int oracle_decode_counts(int64_t n, int nmsg,
                         const uint32_t* const* msgs, const int64_t* ks,
                         int32_t* counts)
{
    if (n < 0 || n >= ((int64_t)1 << 31)) return ORACLE_EDIM;
    if (nmsg < 0) return ORACLE_EINVAL;
    for (int64_t i = 0; i < n; ++i) counts[i] = 0;

    /* P:222 "conversely receives all sparse updates from other workers. The
     * received sparse gradient updates are aggregated": R6 keeps the sum as a
     * signed count of quanta, c[i] in [-N, N]. */
    for (int m = 0; m < nmsg; ++m) {
        int64_t prev = -1;
        for (int64_t j = 0; j < ks[m]; ++j) {
            uint32_t w = msgs[m][j];
            int64_t idx = (int64_t)(w >> 1);
            int neg = (int)(w & 1u);
            if (idx >= n || idx <= prev) return ORACLE_ECORRUPT;
            prev = idx;
            if (neg) counts[idx] = counts[idx] - 1;
            else     counts[idx] = counts[idx] + 1;
        }
    }
    return ORACLE_OK;
}

int oracle_apply(int64_t n, float tau, const int32_t* counts,
                 float* target, float alpha, int accum_mode)
{
    int st = oracle_check_args(n, tau);
    if (st != ORACLE_OK) return st;
    if (accum_mode != ORACLE_ACCUM_WEIGHTS && accum_mode != ORACLE_ACCUM_UPDATE)
        return ORACLE_EINVAL;
    /* P:222 "weights are updated based on the aggregate"; R8 fixes the
     * operation order: the aggregate value of element i is c[i] quanta of tau,
     * rounded once to float, then applied with one rounding. */
    for (int64_t i = 0; i < n; ++i) {
        if (counts[i] == 0) continue;
        float u = (float)counts[i] * tau;
        if (accum_mode == ORACLE_ACCUM_WEIGHTS) target[i] = fmaf(alpha, u, target[i]);
        else                                    target[i] = target[i] + u;
    }
    return ORACLE_OK;
}

int oracle_apply_momentum(int64_t n, float tau, const int32_t* counts,
                          float* w, float* buf, float alpha, float mu)
{
    int st = oracle_check_args(n, tau);
    if (st != ORACLE_OK) return st;
    if (!isfinite(mu) || !isfinite(alpha)) return ORACLE_EINVAL;
    /* SPEC:85 "buf' = momentum*buf + grad; params' = params - lr*buf'" with
     * grad = the aggregate c[i] quanta of tau, alpha = -lr (M1). */
    for (int64_t i = 0; i < n; ++i) {
        float u = (float)counts[i] * tau;
        float b = mu * buf[i];
        b = b + u;
        buf[i] = b;
        w[i] = fmaf(alpha, b, w[i]);
    }
    return ORACLE_OK;
}

int oracle_step(int64_t n, float tau, int cmp_mode, int nworkers,
                const float* const* g, float* const* r,
                uint32_t* const* words, int64_t* ks,
                int32_t* counts, float* target, float alpha, int accum_mode,
                int* nonfinite_out)
{
    int st;
    int any_nonfinite = 0;
    if (nworkers < 1) return ORACLE_EINVAL;
    /* Every worker encodes independently (data parallelism). */
    for (int w = 0; w < nworkers; ++w) {
        int nf = 0;
        st = oracle_encode(n, tau, cmp_mode, g ? g[w] : NULL, r[w], words[w], &ks[w], &nf);
        if (st != ORACLE_OK) return st;
        any_nonfinite |= nf;
    }
    /* All-to-all broadcast: every worker holds all messages; the
     * replicas are identical, so aggregating once stands for every worker. */
    st = oracle_decode_counts(n, nworkers, (const uint32_t* const*)words, ks, counts);
    if (st != ORACLE_OK) return st;
    st = oracle_apply(n, tau, counts, target, alpha, accum_mode);
    if (nonfinite_out) *nonfinite_out = any_nonfinite;
    return st;
}

/* ---------------------------------------------------------------- BMUF */
int oracle_bmuf_step(int64_t n, int nworkers, const float* const* w, float* wg, float* delta,
                     float eta, float zeta, float* const* w_out)
{
    if (n < 0) return ORACLE_EDIM;
    if (nworkers < 1) return ORACLE_EINVAL;
    for (int64_t j = 0; j < n; ++j) {
        /* Eq. (1): model average, worker-rank order, double accumulator */
        double acc = 0.0;
        for (int i = 0; i < nworkers; ++i) acc = acc + (double)w[i][j];
        float wbar = (float)(acc / (double)nworkers);
        /* Eq. (2) */
        float g = wbar - wg[j];
        /* Eq. (3) */
        float d = eta * delta[j];
        float zg = zeta * g;
        d = d + zg;
        delta[j] = d;
        /* Eq. (4), Nesterov block momentum */
        float x = wg[j] + d;
        float look = eta * d;
        x = x + look;
        wg[j] = x;
    }
    /* every worker restarts from the new global model */
    for (int i = 0; i < nworkers; ++i)
        for (int64_t j = 0; j < n; ++j) w_out[i][j] = wg[j];
    return ORACLE_OK;
}

double oracle_bmuf_zeta(double C, int N, double eta)
{
    return C * (double)N * (1.0 - eta);
}
