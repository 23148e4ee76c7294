/*
 * bmuf.h -- C ABI (part of libgtc.so) of the paper's second data-parallel
 * trainer: Blockwise Model Update Filtering with Nesterov block momentum,
 * PAPER.md:224-244 (Sec. VI-B), Eqs. (1)-(5):
 *
 *   (1) Wbar(t)  = (1/N) sum_i W(t)^i                 model average
 *   (2) G(t)     = Wbar(t) - Wg(t-1)
 *   (3) Delta(t) = eta Delta(t-1) + zeta G(t)          block momentum
 *   (4) Wg(t)    = Wg(t-1) + Delta(t) + eta Delta(t)   Nesterov (NBM)
 *   (5) zeta / (N (1 - eta)) = C
 *
 * and every worker restarts its next block of local SGD from Wg(t) (P:227
 * "the initial global model (W_g) is broadcasted to all workers").
 * Readings (B1-B4): constant eta and zeta (eta_{t+1} = eta); the
 * model broadcast is Wg(t) of Eq. (4), look-ahead included; arithmetic in
 * fp32 with the operation order
 *     G = fl(Wbar - Wg);  D = fl(fl(eta*D) + fl(zeta*G));  Wg = fl(fl(Wg + D) + fl(eta*D)).
 *
 * B200 design (world > 1): ONE reduce-scatter of the local models (in place,
 * NCCL over NVLink), ONE fused elementwise kernel applying (1)-(4) to this
 * rank's shard only -- Wg and Delta are sharded across ranks, 1/N of the
 * state per rank -- writing the new Wg shard into the local model, then ONE
 * in-place all-gather of the Wg shards into every rank's local model.  Here
 * Wbar = fl(sum_fp32 / N) with NCCL's summation order (results are identical
 * on all ranks).  Single GPU, simulated workers (bmuf_sync_sim): the mean is
 * a rank-ordered double sum divided by N, rounded once (the oracle's).
 *
 * p2p mode (bmuf_bind_workspace; world <= 8, one node): the local models
 * live in caller-allocated workspaces that are CUDA-IPC mapped on every
 * rank, and bmuf_sync is ONE kernel with no NCCL call: rank r reads shard r of
 * every rank's model over NVLink, forms Wbar as the rank-ordered double sum
 * divided by N, rounded once (the simulated workers' and the oracle's
 * reading, so the result is bit-exact with oracle_bmuf_step), updates its Wg /
 * Delta shard and stores the new Wg shard into every rank's model.
 * Synchronisation is device-side (system-scope release/acquire flags in the
 * workspaces); a peer that does not arrive within 30 s raises GTC_EPEER,
 * reported by bmuf_check.
 *
 * Memory: all device pointers are caller-owned.  Local models are
 * float[padded_len] (padded_len = world * shard_len >= n, shard_len a
 * multiple of 4; the tail beyond n is ignored but moved).
 */
#ifndef GTC_BMUF_H
#define GTC_BMUF_H

#include <stdint.h>

#include <cuda_runtime_api.h>

#include "gtc.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct bmuf_ctx bmuf_ctx;

/* n: parameters; rank/world; nccl_unique_id: 128 bytes from gtc_get_unique_id
 * on rank 0 (NULL iff world == 1); cuda_device: this rank's device. */
gtc_status bmuf_init(bmuf_ctx** out, int64_t n, int rank, int world, const void* nccl_unique_id,
                     int cuda_device);

/* Elements of this rank's shard of Wg and Delta, and of a padded local model. */
int64_t bmuf_shard_len(const bmuf_ctx* ctx);
int64_t bmuf_padded_len(const bmuf_ctx* ctx);

/* One BMUF step on `stream` (Eqs. 1-4).
 *  w_local     : float[padded_len] device: this rank's model after its block
 *                (in); the new global model Wg(t) (out), identical on all ranks.
 *  wg_shard    : float[shard_len] device, in/out: this rank's shard of Wg
 *                (elements [rank*shard_len, (rank+1)*shard_len)).
 *  delta_shard : float[shard_len] device, in/out: same shard of Delta (zero at t=0).
 * 16-byte aligned pointers. */
gtc_status bmuf_sync(bmuf_ctx* ctx, float* w_local, float* wg_shard, float* delta_shard, float eta,
                     float zeta, cudaStream_t stream);

/* p2p workspace: *bytes = 4096 + 4 * padded_len.  Binding (collective: every
 * rank calls it) zeroes the flags, maps every rank's workspace and returns
 * GTC_EUNSUPPORTED on every rank if any mapping fails (then use NCCL mode:
 * do not bind).  The workspace (256-byte aligned, caller-owned, from
 * cudaMalloc or torch's allocator) must outlive the context.  After binding,
 * bmuf_sync's w_local must be bmuf_model(ctx). */
gtc_status bmuf_workspace_size(const bmuf_ctx* ctx, size_t* bytes);
gtc_status bmuf_bind_workspace(bmuf_ctx* ctx, void* workspace, size_t bytes);
/* The local model inside the bound workspace (float[padded_len]); NULL if unbound. */
float* bmuf_model(const bmuf_ctx* ctx);
/* Synchronises the device; GTC_EPEER if a p2p step timed out waiting for a peer. */
gtc_status bmuf_check(bmuf_ctx* ctx);

/* Simulated workers on one GPU (world == 1 context): nmodels local models
 * (host array of device pointers, float[n] each), full Wg and Delta (float[n]);
 * every model is overwritten with the new Wg. */
gtc_status bmuf_sync_sim(bmuf_ctx* ctx, float* const* w_locals, int nmodels, float* wg, float* delta,
                         float eta, float zeta, cudaStream_t stream);

/* Eq. (5): zeta = C * N * (1 - eta). */
double bmuf_zeta(double C, int N, double eta);

/* Collective (every rank calls it; world > 1): wait for the device, then an
 * NCCL barrier, so no peer still reads or pushes into this rank's workspace.
 * Call it before bmuf_destroy and before freeing the workspace. */
gtc_status bmuf_quiesce(bmuf_ctx* ctx);

/* Destroy the communicator and the peer mappings; never frees caller memory.
 * Local: no collective (run bmuf_quiesce on every rank first when peers may
 * still access this workspace). */
void bmuf_destroy(bmuf_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* GTC_BMUF_H */
