/*
 * gtc_oracle.h -- CPU ORACLE for Gradient Threshold Compression (GTC).
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing on the product path may include, link,
 * load or call this file: only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs use it.  It shares no code, header,
 * table or constant with paper_1904_10584_b200/ (the CUDA path).
 *
 * What it computes is the GTC step of
 *   PAPER.md:221-222 (Sec. VI-A "Gradient Threshold Compression"),
 * written out element by element in the paper's order:
 *   1. residual accumulation  "The residual gradients which are not sent to
 *      other workers are aggregated locally for later iterations"
 *   2. threshold              "only gradient elements whose absolute magnitude
 *      is greater than a constant ... gradient-threshold (tau) are sent"
 *   3. 1-bit quantization     "each worker simply sends gradient deltas of +-tau"
 *   4. packing                "packing quantized gradient and integer index into
 *      single 32-bit integer field"
 *   5. all-to-all broadcast   "Each worker communicates the sparse update to all
 *      other workers and conversely receives all sparse updates"
 *   6. aggregation + update   "The received sparse gradient updates are
 *      aggregated and weights are updated based on the aggregate"
 * Readings where the paper is silent are listed in DESIGN.md (R1..R10) and cited
 * next to the code that takes them.
 *
 * Arithmetic: IEEE-754 binary32, round-to-nearest-even, denormals kept, no
 * contraction (built with -O2 -fno-fast-math -ffp-contract=off); the only fused
 * operation is the explicit fmaf() of reading R8.
 */
#ifndef GTC_ORACLE_H
#define GTC_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* R1: threshold comparison.  P:222 says "greater than" (strict); the task's
 * north_star says |r| >= tau.  Both are implemented. */
#define ORACLE_CMP_GT 0
#define ORACLE_CMP_GE 1
/* R8: what the aggregate updates. */
#define ORACLE_ACCUM_WEIGHTS 0 /* W[i] = fmaf(alpha, fl(c[i]*tau), W[i]) */
#define ORACLE_ACCUM_UPDATE  1 /* U[i] = fl(U[i] + fl(c[i]*tau))        */

#define ORACLE_OK        0
#define ORACLE_EDIM      1 /* n < 0 or n >= 2^31 (31-bit index field, R3)   */
#define ORACLE_EINVAL    2 /* tau not finite or not > 0, bad mode            */
#define ORACLE_ECORRUPT  3 /* message word index >= n or not strictly rising */

/* Steps 1-4 for ONE worker.  For i = 0..n-1 in ascending order:
 *   v = fl(r[i] + g[i])            (g == NULL: v = r[i], i.e. r already holds r+g)
 *   sel = |v| > tau  (CMP_GT)   or  |v| >= tau  (CMP_GE)
 *   if sel: neg = v < 0; r[i] = fl(v -+ tau); words[k++] = (i << 1) | neg
 *   else  : r[i] = v
 * words must have room for n entries.  *k_out = number of words.
 * *nonfinite_out = 1 if any v was NaN or +-Inf (R9), else 0.            */
int oracle_encode(int64_t n, float tau, int cmp_mode,
                  const float* g, float* r,
                  uint32_t* words, int64_t* k_out, int* nonfinite_out);

/* Step 6a: aggregate the N received messages into signed integer counts
 * (R6): c[i] = sum over messages m, words w in m with (w>>1) == i of
 *        (+1 if (w & 1) == 0 else -1).
 * counts[n] is overwritten.  Checks every message is strictly ascending in
 * index with index < n (S:153's corrupt-update rule). */
int oracle_decode_counts(int64_t n, int nmsg,
                         const uint32_t* const* msgs, const int64_t* ks,
                         int32_t* counts);

/* Step 6b: weights are updated based on the aggregate (R8).
 * For every i with c[i] != 0:  u = fl((float)c[i] * tau) and
 *   ACCUM_WEIGHTS: target[i] = fmaf(alpha, u, target[i])
 *   ACCUM_UPDATE : target[i] = fl(target[i] + u)
 * Entries with c[i] == 0 are not touched.                               */
int oracle_apply(int64_t n, float tau, const int32_t* counts,
                 float* target, float alpha, int accum_mode);

/* Step 6b with the SGD-momentum update (reading M1): the
 * aggregate is the gradient of an SGD step with momentum, "stochastic
 * gradient descent (SGD)", in SPEC:82-85's form buf' = mu*buf + grad,
 * params' = params - lr*buf' (alpha = -lr, as in ACCUM_WEIGHTS).  For EVERY i
 * (the decaying momentum moves untouched weights too):
 *   u = fl((float)c[i] * tau)          (+0 where c[i] == 0)
 *   buf[i] = fl(fl(mu * buf[i]) + u)
 *   w[i]   = fmaf(alpha, buf[i], w[i])                                   */
int oracle_apply_momentum(int64_t n, float tau, const int32_t* counts,
                          float* w, float* buf, float alpha, float mu);

/* One synchronous GTC step for nworkers simulated workers ("we select
 * the synchronous variant"):  every worker encodes its own g/r, all messages
 * are "received" by everyone (concatenation in rank order), counts are
 * aggregated and applied once to the replicated target.
 *   g[w]     : worker w's gradient (may be NULL entries -> r already holds r+g)
 *   r[w]     : worker w's residual, in/out
 *   words[w] : room for n words each; ks[w] receives k_w
 *   counts   : n int32 out (may be NULL -> internal scratch not available; must be given)
 */
int oracle_step(int64_t n, float tau, int cmp_mode, int nworkers,
                const float* const* g, float* const* r,
                uint32_t* const* words, int64_t* ks,
                int32_t* counts, float* target, float alpha, int accum_mode,
                int* nonfinite_out);

/* ---------------------------------------------------------------- BMUF
 * Blockwise Model Update Filtering with Nesterov block momentum, the paper's
 * other trainer: PAPER.md:224-244 (Sec. VI-B), Eqs. (1)-(5).  One BMUF step
 * ("the global model is updated using the following procedure"), element by
 * element:
 *   (1) Wbar = (1/N) sum_{i=1..N} W^i        (readings B3: sum in worker-rank
 *       order in double, one division by N, one rounding to float)
 *   (2) G     = fl(Wbar - Wg)
 *   (3) Delta = fl(fl(eta * Delta) + fl(zeta * G))
 *   (4) Wg    = fl(fl(Wg + Delta) + fl(eta * Delta))   (NBM, eta_{t+1} = eta: B1)
 * and every worker restarts the next block from Wg (B2, "the initial
 * global model (W_g) is broadcasted to all workers").  w_out may alias w. */
int oracle_bmuf_step(int64_t n, int nworkers, const float* const* w, float* wg, float* delta,
                     float eta, float zeta, float* const* w_out);

/* Eq. (5): zeta / (N (1 - eta)) = C  =>  zeta = C * N * (1 - eta), in double. */
double oracle_bmuf_zeta(double C, int N, double eta);

#ifdef __cplusplus
}
#endif
#endif
