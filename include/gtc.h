/*
 * gtc.h -- C ABI of libgtc.so: the B200 hot path of Gradient Threshold
 * Compression (GTC), PAPER.md:221-222 (Sec. VI-A "Gradient Threshold
 * Compression", arXiv 1904.10584).
 *
 * One synchronous data-parallel step on every rank ("we select the
 * synchronous variant"):
 *
 *   gtc_encode        residual += grad; every element with |residual| > tau
 *                     (or >= tau, GTC_CMP_GE) sends ONE quantum +-tau and keeps
 *                     the rest; the survivors are packed into 32-bit words
 *                     (index << 1 | negative) in ascending index order.
 *                     P:222 "only gradient elements whose absolute magnitude is
 *                     greater than a constant ... (tau) are sent", "The residual
 *                     gradients which are not sent ... are aggregated locally",
 *                     "1-bit quantization ... deltas of +-tau", "packing quantized
 *                     gradient and integer index into single 32-bit integer field".
 *   gtc_exchange      all-gather of every rank's message over NCCL/NVLink.
 *                     P:222 "Each worker communicates the sparse update to all
 *                     other workers and conversely receives all sparse updates".
 *   gtc_decode_apply  signed integer count c[i] in [-N, N] of the quanta every
 *                     rank sent for element i, then target[i] is updated by
 *                     c[i]*tau.  P:222 "The received sparse gradient updates are
 *                     aggregated and weights are updated based on the aggregate".
 *
 * Readings the paper leaves open (R1..R10): strict vs. non-strict
 * threshold (flag), word layout, one quantum per element per step, integer
 * counts as the aggregate, the apply arithmetic
 *     u = fl((float)c * tau);   WEIGHTS: t = fmaf(alpha, u, t);   UPDATE: t = fl(t + u)
 * applied only where c != 0, IEEE fp32 RNE with denormals kept.
 *
 * Conventions
 *  - Memory: every device pointer is CUDA device memory OWNED BY THE CALLER.
 *    libgtc never calls cudaMalloc/cudaFree.  Its scratch ("workspace") is one
 *    caller allocation whose size gtc_workspace_size() reports and which
 *    gtc_bind_workspace() hands over for the life of the context.  The context
 *    owns its NCCL communicator and one small pinned host buffer.
 *  - Streams: every call that takes a stream enqueues device work on it and
 *    returns without waiting, EXCEPT gtc_exchange with world > 1 (one host wait
 *    for the per-rank word counts), gtc_decode_apply_msgs (validates the
 *    messages, waits) and gtc_check (waits).  Consecutive calls on one context
 *    must be ordered (same stream, or caller-ordered streams).
 *  - Order: gtc_init -> gtc_workspace_size -> gtc_bind_workspace ->
 *    (gtc_encode -> gtc_exchange -> gtc_decode_apply)*.  Out-of-order calls
 *    return GTC_ESTATE.  gtc_decode_apply_msgs may be called any time after bind.
 *  - Alignment: grad/residual/target must be 16-byte aligned (GTC_EALIGN);
 *    n need not be a multiple of 4.
 *  - Errors: no exception or abort crosses the ABI.  Device-side conditions
 *    (non-finite residual seen, message overflowing the capacity, corrupt
 *    message) set sticky flags, reported by gtc_exchange (world > 1) or
 *    gtc_check (any world), and cleared once reported.
 */
#ifndef GTC_H
#define GTC_H

#include <stddef.h>
#include <stdint.h>

#include <cuda_runtime_api.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct gtc_ctx gtc_ctx; /* opaque; one per rank */

typedef enum {
    GTC_OK = 0,
    GTC_EINVAL = 1,      /* bad argument (tau <= 0 or non-finite, bad mode, NULL) */
    GTC_EDIM = 2,        /* n_params < 0 or >= 2^31 (31-bit index field)         */
    GTC_EALIGN = 3,      /* a pointer is not 16-byte aligned                      */
    GTC_ECUDA = 4,       /* a CUDA runtime call failed (see gtc_last_error_detail) */
    GTC_ENCCL = 5,       /* an NCCL call failed                                   */
    GTC_ENONFINITE = 6,  /* a NaN/Inf residual was seen (step still completed:
                            NaN is never sent, +-Inf is sent every step)          */
    GTC_ECORRUPT = 7,    /* a message word is out of range or not ascending      */
    GTC_ESTATE = 8,      /* call out of order / workspace not bound              */
    GTC_ECAPACITY = 9,   /* a message exceeded max_words_per_rank                 */
    GTC_EUNSUPPORTED = 10,/* e.g. world > GTC_MAX_MSGS, p2p mapping impossible   */
    GTC_EPEER = 11       /* a peer did not publish its message within the timeout
                            (GTC_PEER_TIMEOUT_MS, default 30 s).  p2p: raised on
                            EVERY rank (the rank that timed out sets it in each
                            rank's flags over NVLink); the step is INCOMPLETE --
                            some tiles may have been applied on some ranks, so
                            weights/residuals are no longer consistent replicas:
                            restore them from a checkpoint.  NCCL mode: this
                            rank's communicator was aborted (ncclCommAbort) and
                            the context accepts no further steps.               */
} gtc_status;

/* Threshold comparison (R1). */
enum { GTC_CMP_GT = 0, /* paper, "greater than": |v| > tau (default) */
       GTC_CMP_GE = 1  /* BASELINE.json north_star: |v| >= tau             */ };

/* Exchange mode for world > 1 (OR-ed into gtc_init's flags). */
enum { GTC_EXCHANGE_P2P = 0,     /* default: peers' messages are read straight from
                                    their memory over NVLink (CUDA IPC mapping made at
                                    bind time); no host sync, no staging copy     */
       GTC_EXCHANGE_NCCL = 16    /* ncclAllGather of counts, one host wait, then
                                    ncclAllGather of the words and tile offsets  */ };

/* gtc_step at world > 1 with the p2p exchange (OR-ed into gtc_init's flags). */
enum { GTC_STEP_FUSED = 0,       /* default: the whole step is ONE kernel
                                    (gtc_step_ticket_kernel)  */
       GTC_STEP_SPLIT = 32       /* encode + decode_apply as two kernels (kept for
                                    comparison: slower at every measured density
                                    and world size)          */ };

/* gtc_init flag: one rank of a LOOPBACK group -- all `world` ranks are
 * contexts of ONE process (tests and single-process drivers; no NCCL
 * communicator, no CUDA IPC, nccl_unique_id must be NULL, p2p exchange,
 * world <= 8).  After every rank's gtc_bind_workspace, gtc_connect_loopback
 * links them.  A rank's gtc_encode then also launches a one-thread publish
 * kernel (its ready flag); the group steps either with the separate calls (every rank's
 * gtc_encode, then every rank's gtc_exchange, then every rank's
 * gtc_decode_apply, in that order, so no kernel waits on one not yet queued)
 * or with gtc_step_group (the fused step of all ranks as ONE launch).
 * gtc_step on a loopback context returns GTC_EUNSUPPORTED. */
enum { GTC_LOOPBACK = 64 };

/* gtc_init flag (world 2..8, p2p): OWNER-COMPUTES decode:
 * rank m owns tiles [ceil(m T / N), ceil((m+1) T / N)) of the T = ceil(n /
 * GTC_TILE) tiles.  gtc_exchange counts the owned tiles from every rank's
 * message (peer reads over NVLink) and publishes one sparse (index, count)
 * list per tile; gtc_decode_apply applies every tile's list, read from its
 * owner.  Per rank it reads (N-1)/N of each peer's message plus the other
 * owners' lists instead of every peer's whole message.  gtc_step runs the
 * three calls (no fused kernel).  Results are bit-identical to the default. */
enum { GTC_DECODE_SHARDED = 128 };

/* What decode_apply updates (R8, M1). */
enum { GTC_ACCUM_WEIGHTS = 0, /* target[i] = fmaf(alpha, fl(c[i]*tau), target[i]) */
       GTC_ACCUM_UPDATE = 1,  /* target[i] = fl(target[i] + fl(c[i]*tau))        */
       GTC_ACCUM_MOMENTUM = 2 /* SGD with momentum, EVERY i (M1):
                                 buf[i] = fl(fl(mu*buf[i]) + fl(c[i]*tau));
                                 target[i] = fmaf(alpha, buf[i], target[i]);
                                 buf / mu from gtc_bind_momentum, alpha = -lr  */ };

/* Most messages one decode_apply can aggregate (ranks or simulated workers). */
#define GTC_MAX_MSGS 64
/* Parameters per tile of the encode/decode kernels; tile offsets are per tile. */
#define GTC_TILE 4096

/* Fill 128 bytes with a fresh NCCL unique id (rank 0 calls it and broadcasts
 * the bytes to the other ranks, e.g. over a torch.distributed group). */
gtc_status gtc_get_unique_id(void* out_128_bytes);

/* Create a context for one rank.
 *  n_params   : length of the flat parameter vector ("for each trainable
 *               weight" -- one global index space, R7), 0 <= n < 2^31.
 *  tau        : the gradient threshold (P:249 uses 8), finite, > 0.
 *  rank/world : this process's rank, number of data-parallel workers.
 *  nccl_unique_id : 128 bytes from gtc_get_unique_id on rank 0; NULL iff world == 1.
 *  cuda_device: device ordinal this rank runs on (made current for the call).
 *  flags      : GTC_CMP_GT or GTC_CMP_GE, OR-ed with GTC_EXCHANGE_P2P (default) or
 *               GTC_EXCHANGE_NCCL, OR-ed with GTC_STEP_FUSED (default) or
 *               GTC_STEP_SPLIT, optionally OR-ed with GTC_LOOPBACK (then
 *               nccl_unique_id is NULL) and GTC_DECODE_SHARDED.  Other bits
 *               or combinations: GTC_EINVAL.
 * The environment variable GTC_PEER_TIMEOUT_MS (read here) sets how long a
 * p2p kernel, or the NCCL-mode host wait, waits for a peer (default 30000).
 * On success *out is a new context (free with gtc_destroy). Blocks on NCCL
 * communicator creation when world > 1. */
gtc_status gtc_init(gtc_ctx** out, int64_t n_params, float tau, int rank, int world,
                    const void* nccl_unique_id, int cuda_device, uint32_t flags);

/* Bytes of device workspace needed (include/gtc.h layout in gtc.cu):
 *  - the segmented message of the hot path (per-tile slots, 4*n bytes, x2 in
 *    p2p mode for step parity) -- it can never overflow;
 *  - one contiguous message of at most max_words_per_rank words (<= 0 means
 *    n_params): the wire format of the NCCL exchange (x world for the receive
 *    buffer) and of gtc_message; a larger message there is GTC_ECAPACITY;
 *  - tile offsets for gtc_decode_apply_msgs calls of up to max_sim_msgs
 *    messages (0 allowed). */
gtc_status gtc_workspace_size(const gtc_ctx* ctx, int64_t max_words_per_rank,
                              int max_sim_msgs, size_t* bytes);

/* Hand the workspace to the context (256-byte aligned, >= the size above for
 * the SAME max_words_per_rank / max_sim_msgs).  Initialises it with a
 * synchronous cudaMemset.  The caller keeps ownership and must keep it alive
 * until gtc_destroy.  world > 1, p2p mode: collective over all ranks (every
 * rank binds with the same sizes); exports this workspace with CUDA IPC and
 * maps every peer's (GTC_EUNSUPPORTED if that is impossible on any rank: use
 * GTC_EXCHANGE_NCCL).  The workspace must come from cudaMalloc (e.g. PyTorch's
 * default caching allocator), not from a virtual-memory-mapped pool. */
gtc_status gtc_bind_workspace(gtc_ctx* ctx, void* dev_ptr, size_t bytes,
                              int64_t max_words_per_rank, int max_sim_msgs);

/* Steps 1-4 of P:222 for this rank: ONE fused streaming kernel on `stream`
 * (residual accumulate, threshold, quantize, pack, per-tile compaction).
 *  grad     : float[n] device, read only; NULL means residual already holds
 *             residual + grad (the caller accumulated into it).
 *  residual : float[n] device, in/out; the caller zeroes it once at the start
 *             of training (R5) and checkpoints it with the weights.
 * The message stays in the workspace, segmented by tile: the packed words of
 * tile t (ascending index) in slot t plus an epoch-stamped per-tile count.
 * gtc_message / gtc_read_message pack it contiguously on demand. */
gtc_status gtc_encode(gtc_ctx* ctx, const float* grad, float* residual, cudaStream_t stream);

/* Make every rank's message available to every other rank (world > 1).
 *  p2p : no device work (decode_apply raises this rank's ready flag, release
 *        at system scope, and reads the peers' tiles in place); loopback
 *        group: a one-thread kernel raises the ready flag.  No host wait.
 *        Errors of any rank are reported by gtc_check after decode_apply.
 *  nccl: ncclAllGather of (k, flags), ONE host wait for the counts, then
 *        ncclAllGather of the words padded to the largest k and of the
 *        per-tile offsets.  Returns GTC_ENONFINITE if any rank flagged a
 *        non-finite residual (the exchange still completed; decode_apply may
 *        proceed), GTC_ECAPACITY if any rank's k exceeded the capacity.
 * world == 1: no device work. */
gtc_status gtc_exchange(gtc_ctx* ctx, cudaStream_t stream);

/* Steps 5-6 of P:222 on `stream` (p2p: the kernel first raises this rank's
 * ready flag, waits on the device for every peer's ready flag of this step,
 * then reads the peers' messages over NVLink; if a peer misses the timeout,
 * the CTAs that timed out apply nothing and every rank's gtc_check reports
 * GTC_EPEER; if this rank's message overflowed its capacity nothing is
 * applied): signed integer counts of all ranks' quanta
 * (deterministic, atomic-free, rank order irrelevant) and the apply of
 * count * tau to target (float[n] device, in/out) for every element with a
 * non-zero count (mode GTC_ACCUM_WEIGHTS with alpha, or GTC_ACCUM_UPDATE), or
 * the momentum update of every element (GTC_ACCUM_MOMENTUM; GTC_ESTATE if no
 * buffer is bound).
 * counts_out: int8[n] device or NULL; if given receives every count (debug /
 * parity; costs n extra bytes written). */
gtc_status gtc_decode_apply(gtc_ctx* ctx, float* target, float alpha, int mode,
                            int8_t* counts_out, cudaStream_t stream);

/* Optimizer state of mode GTC_ACCUM_MOMENTUM (the SGD step
 * after the path, in SPEC:82-85's form buf' = mu*buf + grad, params' =
 * params - lr*buf'): buf is float[n] device (caller-owned, 16-byte aligned,
 * zero at the start of training), mu finite.  The apply is dense (every
 * element's momentum decays), 16 B/param more than the sparse modes; at
 * world 1 gtc_step fuses it into the encode kernel.  buf = NULL unbinds.
 * Returns GTC_EINVAL / GTC_EALIGN on bad arguments. */
gtc_status gtc_bind_momentum(gtc_ctx* ctx, float* buf, float mu);

/* One whole step: gtc_encode, gtc_exchange, gtc_decode_apply in one call
 * (same arguments and results; returns the first failing status, or
 * GTC_ENONFINITE from the exchange after completing the step).  It is ONE
 * kernel launch at world 1 (the encode applies the rank's own quanta) and, by
 * default, at world > 1 with the p2p exchange (PAPER.md:222 encode ->
 * exchange -> aggregate -> apply fused); there device-side
 * faults (GTC_EPEER, GTC_ENONFINITE) are sticky and reported by gtc_check.
 * GTC_STEP_SPLIT, GTC_ACCUM_* all supported; GTC_EXCHANGE_NCCL runs the
 * three calls. */
gtc_status gtc_step(gtc_ctx* ctx, const float* grad, float* residual, float* target, float alpha,
                    int mode, cudaStream_t stream);

/* Same aggregate+apply over caller-supplied messages, no NCCL: used for
 * simulated workers on one GPU and for tests.
 *  msgs   : host array of nmsg DEVICE pointers to uint32 words (ascending)
 *  counts : host array of nmsg word counts
 * Validates every message (GTC_ECORRUPT on a word with index >= n or a
 * non-increasing index; nothing is applied then) and waits for the stream. */
gtc_status gtc_decode_apply_msgs(gtc_ctx* ctx, const uint32_t* const* msgs,
                                 const int64_t* counts, int nmsg, float* target,
                                 float alpha, int mode, int8_t* counts_out,
                                 cudaStream_t stream);

/* Per-rank word counts of the last gtc_exchange (world entries; for world == 1
 * this reads the local count back and waits on the last encode's stream). */
gtc_status gtc_last_counts(gtc_ctx* ctx, int64_t* k_per_rank);

/* Device pointer to the int64 word count of the last encode (for async reads). */
gtc_status gtc_local_count(const gtc_ctx* ctx, const int64_t** dev_k);

/* Device pointer + length of rank `rank`'s message after the last exchange
 * (world == 1: the local message; k is read back, waiting on the stream). */
gtc_status gtc_message(gtc_ctx* ctx, int rank, const uint32_t** dev_words, int64_t* k);

/* Copy rank `rank`'s message of the last step into host memory (tests,
 * debugging; waits for the device).  max_words is the room at host_words. */
gtc_status gtc_read_message(gtc_ctx* ctx, int rank, uint32_t* host_words, int64_t max_words, int64_t* k);

/* Wire format of a SparseUpdate (host-only, no device
 * work, callable without a GPU).  The hot path's words are (index << 1) | neg
 * (R3: sorting words sorts indices); SPEC's interchange layout is
 * bit 31 = sign (1 => -tau), bits 0..30 = index.  A serialized update is,
 * little-endian: magic "GTCU" (4 bytes), dim (u64), tau (f32), word count
 * (u32), then the SPEC-layout words (u32 each): 20 + 4 k bytes
 * ("bytes per update == 4 x word count + 16" counts the header
 * without the magic).
 *  gtc_wire_pack  : words = k canonical words (index << 1 | neg), ascending,
 *                   every index < dim < 2^31 (else GTC_ECORRUPT, GTC_EDIM);
 *                   writes 20 + 4k bytes to out (out_bytes too small:
 *                   GTC_EINVAL, *written = the size needed).
 *  gtc_wire_unpack: the inverse; validates magic, sizes, dim < 2^31, tau
 *                   finite > 0, indices < dim and strictly ascending
 *                   (GTC_ECORRUPT otherwise); writes the canonical words
 *                   (at most max_words, else GTC_EINVAL) and *k, *dim, *tau. */
gtc_status gtc_wire_pack(const uint32_t* words, int64_t k, uint64_t dim, float tau, void* out,
                         size_t out_bytes, size_t* written);
gtc_status gtc_wire_unpack(const void* in, size_t in_bytes, uint32_t* words, int64_t max_words,
                           int64_t* k, uint64_t* dim, float* tau);

/* Wait for `stream`, then report and clear this rank's sticky device flags:
 * GTC_EPEER, GTC_ECAPACITY, GTC_ECORRUPT, GTC_ENONFINITE or GTC_OK.  A peer
 * timeout anywhere in a p2p step is raised in EVERY rank's flags, so every
 * rank's gtc_check reports GTC_EPEER (see GTC_EPEER for what it means). */
gtc_status gtc_check(gtc_ctx* ctx, cudaStream_t stream);

/* Loopback group (GTC_LOOPBACK): ctxs[r] is rank r of `world`, every one
 * created with GTC_LOOPBACK and the same n, tau and flags, and bound with the
 * same sizes.  Gives every rank a view of every rank's workspace (same
 * process: plain device pointers; ranks on other devices: peer access is
 * enabled).  GTC_EINVAL / GTC_ESTATE on a mismatched or unbound rank. */
gtc_status gtc_connect_loopback(gtc_ctx* const* ctxs, int world);

/* Loopback group, every rank on ONE device: the fused one-kernel step
 * (PAPER.md:222 encode -> exchange -> aggregate -> apply; the kernel of
 * gtc_step at world > 1) of all `world` ranks as ONE launch on `stream`:
 * CTAs take tickets from one group counter, ticket g being CTA g / world of
 * rank g % world, so a CTA only waits on tiles of lower tickets, exactly as
 * in the per-rank kernel.
 *  grads[r] / residuals[r] / targets[r]: rank r's arguments of gtc_step
 *  (grads == NULL, or grads[r] == NULL on every rank: residuals hold r + g).
 *  debug_flags: bit r set = rank r's CTAs exit at once (a rank that never
 *  shows up: the others raise GTC_EPEER after the timeout); 0 in normal use.
 * Waits for `stream` first (the parameters are staged in pinned memory). */
gtc_status gtc_step_group(gtc_ctx* const* ctxs, int world, const float* const* grads, float* const* residuals,
                          float* const* targets, float alpha, int mode, uint32_t debug_flags, cudaStream_t stream);

/* Collective (every rank calls it; world > 1, p2p, not loopback): wait for
 * the device, then an NCCL barrier, so no peer is still reading this rank's
 * workspace.  Call it before gtc_destroy and before freeing the workspace. */
gtc_status gtc_quiesce(gtc_ctx* ctx);

/* GTC_EXCHANGE_P2P or GTC_EXCHANGE_NCCL (world > 1), 0 for world == 1. */
int gtc_exchange_mode(const gtc_ctx* ctx);

/* Number of kernels libgtc launched on this context so far (NCCL's excluded). */
int64_t gtc_kernel_launches(const gtc_ctx* ctx);

/* Debug: with GTC_DECODE_TRACE=1 in the environment, the counting decode
 * kernel stamps %globaltimer (ns) at 6 phase boundaries (start, peers ready,
 * tag counts, per-rank counts, non-zero list, end) for its first 4096 CTAs;
 * this copies up to max_entries stamps (CTA-major) of the last decode to
 * host memory.  Not for production use. */
gtc_status gtc_debug_decode_trace(uint64_t* host, int max_entries);

/* Debug: with GTC_DECODE_TRACE=1, the fused p2p step kernel (gtc_step at
 * world > 1) stamps %globaltimer (ns) at 5 phase boundaries (start, every
 * rank's tile tag seen, counts done, encode done, end) plus the SM id, 6
 * entries per CTA for its first 16384 CTAs; this copies up to max_entries of
 * the last fused step to host memory.  Not for production use. */
gtc_status gtc_debug_step_trace(uint64_t* host, int max_entries);

const char* gtc_strerror(gtc_status status);
const char* gtc_last_error_detail(const gtc_ctx* ctx);

/* Destroy the NCCL communicator, the peer mappings and host state; never
 * frees caller memory.  Local: no collective (run gtc_quiesce on every rank
 * first when peers may still read this workspace). */
void gtc_destroy(gtc_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* GTC_H */
