// gtc.cu -- the C ABI of libgtc.so (include/gtc.h): context, workspace layout,
// argument validation, call ordering and the exchange ("Each
// worker communicates the sparse update to all other workers and conversely
// receives all sparse updates from other workers").
//
// The hot-path message is segmented (gtc_internal.cuh): encode writes each
// tile's packed words into that tile's slot and publishes a per-tile tag.
// Exchange modes for world > 1:
//   p2p  (default): every rank's workspace is mapped into its peers with CUDA
//        IPC at bind time; decode_apply reads every rank's tags and words for
//        its tiles straight from the owner's memory over NVLink, waiting per
//        tile on the owner's tag (epoch-stamped, release/acquire at system
//        scope).  No host sync, no collective launch, no staging copy; the
//        segmented buffers are double-buffered by step parity.
//   nccl (GTC_EXCHANGE_NCCL): the message is packed contiguously, then
//        ncclAllGather of (k, flags), one host wait for the largest k,
//        ncclAllGather of the words and tile offsets.

#include <algorithm>
#include <chrono>
#include <cmath>
#include <thread>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "gtc_internal.cuh"
#include "tile_encode.cuh"  // kTileThreads, entry_stamp (host side of the fused step parameters)

#include <nvtx3/nvToolsExt.h>

using namespace gtc;

namespace {

enum class Stage { kBound, kEncoded, kExchanged };

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// Workspace layout (offsets from the bound base, each 256-byte aligned):
//   ctrl      Ctrl                               k, flags
//   group_sum u32[ceil(T / kGroupTiles)]         packing scratch
//   seg[p]    { u64 tags[T] | u32 words[T*kTile] } segmented message, p < nseg
//                                                (nseg = 2 in p2p mode: step parity)
//   msg       { MsgHeader | i32 tile_off[T+1] | u32 words[capacity] }
//                                                contiguous message (NCCL / on demand)
//   ipc       128 B x world                      bind-time IPC records (world > 1)
//   kx_all    i64[2 * world]                     nccl: all-gathered (k, flags)
//   recv      u32[world * capacity]              nccl: all-gathered messages
//   recv_off  i32[world * (T + 1)]               nccl: all-gathered tile offsets
//   sim_off   i32[max_sim_msgs * (T + 1)]        tile offsets for decode_apply_msgs
//   push[p][m] T records of kPushRec bytes        p2p: what rank m pushed (fused step), p < 2
//   group     FusedStepParams[world]             loopback: the group launch's parameters
//   ctags[p], clist[p]  { u64 tags[T] | u32 entries[T*kTile] }  sharded decode: count lists, p < 2
struct Layout {
    int nseg;
    size_t ctrl, group_sum, seg_tags[2], seg_words[2];
    size_t ctags[2], clist[2];
    size_t msg_hdr, msg_off, msg_words;
    size_t ipc, kx_all, recv, recv_off, sim_off;
    size_t push, push_slot;  // push[p][m] at push + (p * world + m) * push_slot
    size_t group;
    size_t total;
};

constexpr size_t kIpcRecord = kIpcRecordBytes;

Layout make_layout(long long n, int world, bool p2p, bool loopback, bool sharded, long long capacity,
                   int max_sim_msgs) {
    const long long tiles = (n + kTile - 1) / kTile;
    const size_t T = (size_t)std::max(tiles, 1LL);
    Layout L{};
    size_t o = 0;
    L.ctrl = o;      o = align_up(o + sizeof(Ctrl), 256);
    L.group_sum = o; o = align_up(o + sizeof(unsigned) * ((T + kGroupTiles - 1) / kGroupTiles), 256);
    L.nseg = (world > 1 && p2p) ? 2 : 1;
    for (int i = 0; i < 2; ++i) {
        L.seg_tags[i] = L.seg_words[i] = 0;
        if (i >= L.nseg) continue;
        L.seg_tags[i] = o;  o = align_up(o + sizeof(unsigned long long) * T, 256);
        L.seg_words[i] = o; o = align_up(o + sizeof(unsigned) * T * kTile, 256);
    }
    L.msg_hdr = o;   o = align_up(o + sizeof(MsgHeader), 256);
    L.msg_off = o;   o = align_up(o + sizeof(int) * (size_t)(tiles + 1), 256);
    L.msg_words = o; o = align_up(o + sizeof(unsigned) * (size_t)std::max(capacity, 1LL), 256);
    L.ipc = L.kx_all = L.recv = L.recv_off = 0;
    if (world > 1) {
        L.ipc = o; o = align_up(o + kIpcRecord * (size_t)world, 256);
    }
    if (world > 1 && !p2p) {
        L.kx_all = o;   o = align_up(o + sizeof(long long) * 2 * (size_t)world, 256);
        L.recv = o;     o = align_up(o + sizeof(unsigned) * (size_t)world * (size_t)std::max(capacity, 1LL), 256);
        L.recv_off = o; o = align_up(o + sizeof(int) * (size_t)world * (size_t)(tiles + 1), 256);
    }
    L.sim_off = o;   o = align_up(o + sizeof(int) * (size_t)std::max(max_sim_msgs, 0) * (size_t)(tiles + 1), 256);
    L.push = L.push_slot = 0;
    if (world > 1 && p2p) {
        L.push_slot = align_up((size_t)kPushRec * T, 256);
        L.push = o;  o = align_up(o + 2 * (size_t)world * L.push_slot, 256);
    }
    L.group = 0;
    if (loopback) {
        L.group = o; o = align_up(o + sizeof(FusedStepParams) * (size_t)world, 256);
    }
    for (int i = 0; i < 2; ++i) {
        L.ctags[i] = L.clist[i] = 0;
        if (!sharded) continue;
        L.ctags[i] = o; o = align_up(o + sizeof(unsigned long long) * T, 256);
        L.clist[i] = o; o = align_up(o + sizeof(unsigned) * T * kTile, 256);
    }
    L.total = o;
    return L;
}


}  // namespace

struct gtc_ctx {
    long long n = 0;
    float tau = 0.f;
    int rank = 0, world = 1, device = 0;
    int cmp_mode = GTC_CMP_GT;
    bool p2p = false;
    bool loopback = false;          // GTC_LOOPBACK: a rank of an in-process group (no NCCL, no IPC)
    bool sharded = false;           // GTC_DECODE_SHARDED: owner-computes decode (sharded.cu)
    bool connected = false;         // loopback: gtc_connect_loopback done
    bool dead = false;              // the NCCL communicator was aborted (timeout)
    unsigned long long timeout_ns = 30ull * 1000 * 1000 * 1000;  // p2p: longest wait for a peer
    bool split_step = false;        // GTC_STEP_SPLIT: gtc_step as encode + decode_apply kernels
    int num_tiles = 0;
    ncclComm_t comm = nullptr;

    unsigned char* ws = nullptr;
    size_t ws_bytes = 0;
    long long capacity = 0;
    int max_sim_msgs = 0;
    Layout L{};

    Ctrl* ctrl = nullptr;
    long long* kx_all = nullptr;
    unsigned* recv = nullptr;
    int* recv_off = nullptr;
    int* sim_off = nullptr;

    // every rank's workspace base as seen from this process (self = ws)
    std::vector<unsigned char*> peer_ws;
    std::vector<void*> peer_alloc;  // what cudaIpcOpenMemHandle returned (to close)
    unsigned epoch = 0;             // step counter: tag stamp; parity selects the p2p buffer
    unsigned long long encodes = 0; // encodes since bind (the step value of the p2p ready flags)
    float* mom_buf = nullptr;       // GTC_ACCUM_MOMENTUM state (gtc_bind_momentum)
    float mom_mu = 0.f;
    FusedStepParams* host_group = nullptr;  // loopback rank 0: pinned staging of the group parameters
    int packed_rank = -1;           // whose message the contiguous region holds (-1: stale)
    bool push_clean[2] = {true, true};  // p2p: the last step of this parity was fused (or none yet)

    long long* host_kx = nullptr;  // pinned, 2 * world
    std::vector<long long> last_k;
    long long max_k = 0;

    Stage stage = Stage::kBound;
    bool bound = false;
    long long launches = 0;
    std::string detail;
};

namespace {

// Phase tracing: every API call is an NVTX range (header-only NVTX v3, a no-op
// unless a profiler is attached), so a timeline shows encode / exchange /
// decode_apply / step per rank next to the kernels they enqueue.
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};

gtc_status fail(gtc_ctx* c, gtc_status s, const std::string& what) {
    if (c) c->detail = what;
    return s;
}

gtc_status cuda_fail(gtc_ctx* c, cudaError_t e, const char* where) {
    return fail(c, GTC_ECUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

gtc_status nccl_fail(gtc_ctx* c, ncclResult_t r, const char* where) {
    return fail(c, GTC_ENCCL, std::string(where) + ": " + ncclGetErrorString(r));
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        int cur = -1;
        if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
    }
};

gtc_status flags_to_status(unsigned long long f) {
    if (f & kFlagPeer) return GTC_EPEER;
    if (f & kFlagCapacity) return GTC_ECAPACITY;
    if (f & kFlagCorrupt) return GTC_ECORRUPT;
    if (f & kFlagNonFinite) return GTC_ENONFINITE;
    return GTC_OK;
}

int seg_parity(const gtc_ctx* c) { return c->L.nseg == 2 ? (int)(c->epoch & 1u) : 0; }

// workspace base of `rank` as seen from this process
unsigned char* rank_ws(const gtc_ctx* c, int rank) {
    return (c->world > 1 && c->p2p) ? c->peer_ws[rank] : c->ws;
}

// p2p: map every peer's workspace (ipc.cu); all ranks agree on the outcome.
// (Loopback contexts are connected by gtc_connect_loopback instead.)
gtc_status connect_peers(gtc_ctx* c) {
    const IpcResult r = ipc_map_peers(c->comm, c->rank, c->world, c->ws, c->L.total, c->ws + c->L.ipc, c->peer_ws,
                                      c->peer_alloc);
    switch (r) {
        case IpcResult::kOk: return GTC_OK;
        case IpcResult::kCudaError: return fail(c, GTC_ECUDA, "bind: CUDA IPC exchange");
        case IpcResult::kNcclError: return fail(c, GTC_ENCCL, "bind: NCCL IPC exchange");
        default:
            return fail(c, GTC_EUNSUPPORTED,
                        "p2p exchange: workspaces cannot be mapped across ranks (use GTC_EXCHANGE_NCCL)");
    }
}

// Pack rank `rank`'s segmented message of the current step into this rank's
// contiguous region (header, tile offsets, words).
gtc_status pack_contiguous(gtc_ctx* c, int rank, cudaStream_t stream) {
    unsigned char* src = rank_ws(c, rank);
    const int par = seg_parity(c);
    CompactParams q{};
    q.seg = reinterpret_cast<const unsigned*>(src + c->L.seg_words[par]);
    q.tags = reinterpret_cast<const unsigned long long*>(src + c->L.seg_tags[par]);
    q.group_sum = reinterpret_cast<unsigned*>(c->ws + c->L.group_sum);
    q.num_tiles = c->num_tiles;
    q.words = reinterpret_cast<unsigned*>(c->ws + c->L.msg_words);
    q.tile_off = reinterpret_cast<int*>(c->ws + c->L.msg_off);
    q.hdr = reinterpret_cast<MsgHeader*>(c->ws + c->L.msg_hdr);
    q.capacity = c->capacity;
    q.ctrl = c->ctrl;
    q.stamped = (c->world > 1 && c->p2p) ? 1 : 0;
    if (c->num_tiles == 0) {
        cudaError_t e = cudaMemsetAsync(c->ws + c->L.msg_hdr, 0, sizeof(MsgHeader), stream);
        if (e == cudaSuccess) e = cudaMemsetAsync(c->ws + c->L.msg_off, 0, sizeof(int), stream);
        if (e != cudaSuccess) return cuda_fail(c, e, "pack: n == 0");
    } else {
        cudaError_t e = launch_compact(q, stream);
        if (e != cudaSuccess) return cuda_fail(c, e, "pack: launch");
        c->launches += 2;
    }
    c->packed_rank = rank;
    return GTC_OK;
}

}  // namespace

extern "C" {

const char* gtc_strerror(gtc_status s) {
    switch (s) {
        case GTC_OK: return "ok";
        case GTC_EINVAL: return "invalid argument";
        case GTC_EDIM: return "n_params out of range [0, 2^31)";
        case GTC_EALIGN: return "pointer not 16-byte aligned";
        case GTC_ECUDA: return "CUDA error";
        case GTC_ENCCL: return "NCCL error";
        case GTC_ENONFINITE: return "non-finite residual seen";
        case GTC_ECORRUPT: return "corrupt message";
        case GTC_ESTATE: return "call out of order or workspace not bound";
        case GTC_ECAPACITY: return "message exceeded max_words_per_rank";
        case GTC_EUNSUPPORTED: return "unsupported configuration";
        case GTC_EPEER: return "a peer did not publish its message in time";
    }
    return "unknown status";
}

const char* gtc_last_error_detail(const gtc_ctx* c) { return c ? c->detail.c_str() : ""; }

gtc_status gtc_get_unique_id(void* out) {
    if (!out) return GTC_EINVAL;
    ncclUniqueId id;
    if (ncclGetUniqueId(&id) != ncclSuccess) return GTC_ENCCL;
    static_assert(sizeof(ncclUniqueId) == 128, "NCCL unique id is 128 bytes");
    std::memcpy(out, &id, sizeof(id));
    return GTC_OK;
}

gtc_status gtc_init(gtc_ctx** out, int64_t n_params, float tau, int rank, int world,
                    const void* nccl_unique_id, int cuda_device, uint32_t flags) {
    if (!out) return GTC_EINVAL;
    *out = nullptr;
    if (n_params < 0 || n_params >= (1LL << 31)) return GTC_EDIM;
    if (!(tau > 0.f) || std::isinf(tau)) return GTC_EINVAL;
    if (world < 1 || rank < 0 || rank >= world) return GTC_EINVAL;
    if (world > GTC_MAX_MSGS) return GTC_EUNSUPPORTED;
    if (flags & ~(uint32_t)(GTC_CMP_GE | GTC_EXCHANGE_NCCL | GTC_STEP_SPLIT | GTC_LOOPBACK | GTC_DECODE_SHARDED))
        return GTC_EINVAL;
    if ((flags & GTC_DECODE_SHARDED) && (world < 2 || (flags & GTC_EXCHANGE_NCCL) || world > kFusedMaxRanks))
        return GTC_EINVAL;  // the owner-computes decode is a p2p mode of 2..8 ranks
    const bool loopback = (flags & GTC_LOOPBACK) != 0;
    if (loopback) {
        // an in-process group: no NCCL id, p2p exchange only
        if (nccl_unique_id != nullptr || (flags & GTC_EXCHANGE_NCCL) || world < 2) return GTC_EINVAL;
        if (world > kFusedMaxRanks) return GTC_EUNSUPPORTED;
    } else if ((world > 1) != (nccl_unique_id != nullptr)) {
        return GTC_EINVAL;
    }

    gtc_ctx* c = new (std::nothrow) gtc_ctx();
    if (!c) return GTC_EINVAL;
    c->n = n_params;
    c->tau = tau;
    c->rank = rank;
    c->world = world;
    c->device = cuda_device;
    c->cmp_mode = (int)(flags & GTC_CMP_GE);
    c->p2p = world > 1 && !(flags & GTC_EXCHANGE_NCCL);
    c->loopback = loopback;
    c->sharded = (flags & GTC_DECODE_SHARDED) != 0;
    c->split_step = (flags & GTC_STEP_SPLIT) != 0;
    if (const char* e = std::getenv("GTC_PEER_TIMEOUT_MS")) {
        const long long ms = std::atoll(e);
        if (ms > 0) c->timeout_ns = (unsigned long long)ms * 1000000ull;
    }
    c->num_tiles = (int)((n_params + kTile - 1) / kTile);
    c->last_k.assign(world, 0);

    DeviceGuard g(cuda_device);
    cudaError_t e = cudaHostAlloc(reinterpret_cast<void**>(&c->host_kx),
                                  sizeof(long long) * 2 * (size_t)world, cudaHostAllocDefault);
    if (e != cudaSuccess) {
        delete c;
        return GTC_ECUDA;
    }
    if (loopback && rank == 0) {
        e = cudaHostAlloc(reinterpret_cast<void**>(&c->host_group), sizeof(FusedStepParams) * kFusedMaxRanks,
                          cudaHostAllocDefault);
        if (e != cudaSuccess) {
            cudaFreeHost(c->host_kx);
            delete c;
            return GTC_ECUDA;
        }
    }
    if (world > 1 && !loopback) {
        ncclUniqueId id;
        std::memcpy(&id, nccl_unique_id, sizeof(id));
        ncclResult_t r = ncclCommInitRank(&c->comm, world, id, rank);
        if (r != ncclSuccess) {
            cudaFreeHost(c->host_kx);
            delete c;
            return GTC_ENCCL;
        }
    }
    *out = c;
    return GTC_OK;
}

gtc_status gtc_workspace_size(const gtc_ctx* c, int64_t max_words_per_rank, int max_sim_msgs,
                              size_t* bytes) {
    if (!c || !bytes) return GTC_EINVAL;
    if (max_sim_msgs < 0 || max_sim_msgs > GTC_MAX_MSGS) return GTC_EINVAL;
    const long long cap = max_words_per_rank <= 0 ? c->n : std::min<long long>(max_words_per_rank, c->n);
    *bytes = make_layout(c->n, c->world, c->p2p, c->loopback, c->sharded, cap, max_sim_msgs).total;
    return GTC_OK;
}

gtc_status gtc_bind_workspace(gtc_ctx* c, void* dev_ptr, size_t bytes, int64_t max_words_per_rank,
                              int max_sim_msgs) {
    if (!c || !dev_ptr) return fail(c, GTC_EINVAL, "bind: null");
    if (c->bound) return fail(c, GTC_ESTATE, "bind: workspace already bound");
    if (reinterpret_cast<uintptr_t>(dev_ptr) & 255u) return fail(c, GTC_EALIGN, "workspace not 256-byte aligned");
    if (max_sim_msgs < 0 || max_sim_msgs > GTC_MAX_MSGS) return fail(c, GTC_EINVAL, "max_sim_msgs");
    const long long cap = max_words_per_rank <= 0 ? c->n : std::min<long long>(max_words_per_rank, c->n);
    const Layout L = make_layout(c->n, c->world, c->p2p, c->loopback, c->sharded, cap, max_sim_msgs);
    if (bytes < L.total) return fail(c, GTC_EINVAL, "workspace too small");
    DeviceGuard g(c->device);
    unsigned char* b = static_cast<unsigned char*>(dev_ptr);
    // control block, group sums, tags (epoch 0 = never published) and the
    // contiguous header/offsets start at 0
    cudaError_t e = cudaMemset(b, 0, L.seg_tags[0]);
    // (p2p: the words too -- entry 0 carries stamp 0, never valid; tile_encode.cuh)
    const size_t seg_words_bytes = sizeof(unsigned) * (size_t)std::max(c->num_tiles, 1) * kTile;
    for (int i = 0; i < L.nseg && e == cudaSuccess; ++i)
        e = cudaMemset(b + L.seg_tags[i], 0, L.seg_words[i] - L.seg_tags[i] + (L.nseg == 2 ? seg_words_bytes : 0));
    if (e == cudaSuccess) e = cudaMemset(b + L.msg_hdr, 0, L.msg_words - L.msg_hdr);
    if (e == cudaSuccess && L.push_slot) e = cudaMemset(b + L.push, 0, 2 * (size_t)c->world * L.push_slot);
    if (e != cudaSuccess) return cuda_fail(c, e, "bind: cudaMemset");
    e = cudaDeviceSynchronize();
    if (e != cudaSuccess) return cuda_fail(c, e, "bind: sync");
    c->ws = b;
    c->ws_bytes = bytes;
    c->capacity = cap;
    c->max_sim_msgs = max_sim_msgs;
    c->L = L;
    c->ctrl = reinterpret_cast<Ctrl*>(b + L.ctrl);
    if (c->world > 1 && !c->p2p) {
        c->kx_all = reinterpret_cast<long long*>(b + L.kx_all);
        c->recv = reinterpret_cast<unsigned*>(b + L.recv);
        c->recv_off = reinterpret_cast<int*>(b + L.recv_off);
    }
    c->sim_off = reinterpret_cast<int*>(b + L.sim_off);
    if (c->world > 1 && c->p2p && !c->loopback) {
        gtc_status s = connect_peers(c);
        if (s != GTC_OK) {
            c->ws = nullptr;
            return s;
        }
    }
    c->epoch = 0;
    c->encodes = 0;
    c->bound = true;
    c->stage = Stage::kBound;
    return GTC_OK;
}

static gtc_status check_encode_args(gtc_ctx* c, const float* grad, float* residual) {
    if (!c->bound) return fail(c, GTC_ESTATE, "encode: workspace not bound");
    if (c->dead) return fail(c, GTC_ESTATE, "the NCCL communicator was aborted after a timeout");
    if (c->loopback && !c->connected) return fail(c, GTC_ESTATE, "loopback: call gtc_connect_loopback first");
    if (c->n > 0 && !residual) return fail(c, GTC_EINVAL, "encode: residual is null");
    if (!aligned16(residual) || !aligned16(grad)) return fail(c, GTC_EALIGN, "encode: grad/residual alignment");
    return GTC_OK;
}

// A new step: epoch (tag stamp, parity), step count (p2p ready value).
static void begin_step(gtc_ctx* c) {
    c->epoch = c->epoch == 0xffffffffu ? 1u : c->epoch + 1u;  // 0 is never a published stamp
    c->encodes += 1;
    c->packed_rank = -1;
}

// Encode every tile of the current step on `stream`.
static gtc_status encode_launch(gtc_ctx* c, const float* grad, float* residual, cudaStream_t stream,
                                float* fused_target, float fused_alpha, int fused_mode) {
    const int par = seg_parity(c);
    EncodeParams p{};
    p.g = grad;
    p.r = residual;
    p.n = c->n;
    p.tau = c->tau;
    p.seg = reinterpret_cast<unsigned*>(c->ws + c->L.seg_words[par]);
    p.tags = reinterpret_cast<unsigned long long*>(c->ws + c->L.seg_tags[par]);
    p.ctrl = c->ctrl;
    p.k_acc = &c->ctrl->k_acc[c->epoch & 1u];
    p.k_next = &c->ctrl->k_acc[(c->epoch + 1u) & 1u];
    p.target = fused_target;
    p.alpha = fused_alpha;
    p.accum_mode = fused_mode;
    p.buf = c->mom_buf;
    p.mu = c->mom_mu;
    p.epoch = c->epoch;
    p.publish_sys = (c->world > 1 && c->p2p) ? 1 : 0;
    if (p.publish_sys) c->push_clean[par] = false;  // this parity's push records are not maintained
    p.num_tiles = c->num_tiles;
    p.step = c->encodes;
    cudaError_t e = launch_encode(p, c->cmp_mode, stream);
    if (e != cudaSuccess) return cuda_fail(c, e, "encode: launch");
    c->launches += 1;
    return GTC_OK;
}

static gtc_status encode_impl(gtc_ctx* c, const float* grad, float* residual, cudaStream_t stream,
                              float* fused_target, float fused_alpha, int fused_mode) {
    if (!c) return GTC_EINVAL;
    gtc_status s = check_encode_args(c, grad, residual);
    if (s != GTC_OK) return s;
    DeviceGuard g(c->device);
    begin_step(c);
    if (c->num_tiles == 0) {  // n == 0: empty message
        cudaError_t e = cudaMemsetAsync(&c->ctrl->k_acc[c->epoch & 1u], 0, sizeof(unsigned long long), stream);
        if (e != cudaSuccess) return cuda_fail(c, e, "encode: n == 0");
        c->stage = Stage::kEncoded;
        return GTC_OK;
    }
    // p2p: the decode kernel raises ready when it starts (no publish launch)
    s = encode_launch(c, grad, residual, stream, fused_target, fused_alpha, fused_mode);
    if (s != GTC_OK) return s;
    if (c->loopback) {
        // loopback group: every rank's encode is queued before any rank's
        // exchange/decode, so the flag goes up here (one one-thread kernel) --
        // no kernel ever waits on one not yet queued
        const cudaError_t e = launch_publish(&c->ctrl->ready, c->encodes, stream);
        if (e != cudaSuccess) return cuda_fail(c, e, "encode: publish");
        c->launches += 1;
    }
    c->stage = Stage::kEncoded;
    return GTC_OK;
}

gtc_status gtc_encode(gtc_ctx* c, const float* grad, float* residual, cudaStream_t stream) {
    NvtxRange nvtx("gtc_encode");
    return encode_impl(c, grad, residual, stream, nullptr, 0.f, GTC_ACCUM_WEIGHTS);
}

// Sharded decode (sharded.cu) parameters of the current step.
static ShardParams shard_params(gtc_ctx* c) {
    const int par = seg_parity(c);
    ShardParams q{};
    for (int i = 0; i < c->world; ++i) {
        unsigned char* b = rank_ws(c, i);
        Ctrl* ci = reinterpret_cast<Ctrl*>(b + c->L.ctrl);
        q.seg[i] = reinterpret_cast<const unsigned*>(b + c->L.seg_words[par]);
        q.tags[i] = reinterpret_cast<const unsigned long long*>(b + c->L.seg_tags[par]);
        q.ready[i] = &ci->ready;
        q.counted[i] = &ci->counted;
        q.peer_flags[i] = &ci->flags;
        q.clist_of[i] = reinterpret_cast<const unsigned*>(b + c->L.clist[par]);
        q.ctags_of[i] = reinterpret_cast<const unsigned long long*>(b + c->L.ctags[par]);
    }
    q.clist = reinterpret_cast<unsigned*>(c->ws + c->L.clist[par]);
    q.ctags = reinterpret_cast<unsigned long long*>(c->ws + c->L.ctags[par]);
    q.nranks = c->world;
    q.rank = c->rank;
    q.n = c->n;
    q.num_tiles = c->num_tiles;
    q.epoch = c->epoch;
    q.step = c->encodes;
    q.timeout_ns = c->timeout_ns;
    q.tau = c->tau;
    q.flags = &c->ctrl->flags;
    return q;
}

// gtc_exchange, sharded: the owner count of this rank's tiles (its block 0
// raises this rank's ready flag first), then `counted` goes up.
static gtc_status owner_count(gtc_ctx* c, cudaStream_t stream) {
    ShardParams q = shard_params(c);
    q.publish = &c->ctrl->ready;
    cudaError_t e = launch_owner_count(q, stream);
    if (e == cudaSuccess && c->num_tiles > 0) {
        c->launches += 1;
        e = launch_publish(&c->ctrl->counted, c->encodes, stream);
        c->launches += 1;
    }
    if (e != cudaSuccess) return cuda_fail(c, e, "exchange: owner count");
    return GTC_OK;
}

static gtc_status exchange_nccl(gtc_ctx* c, cudaStream_t stream) {
    // 0. the wire format: this rank's message, contiguous
    gtc_status s = pack_contiguous(c, c->rank, stream);
    if (s != GTC_OK) return s;
    // 1. (k, flags) of every rank: the packed message's header.
    ncclResult_t r = ncclAllGather(c->ws + c->L.msg_hdr, c->kx_all, 2, ncclInt64, c->comm, stream);
    if (r != ncclSuccess) return nccl_fail(c, r, "exchange: ncclAllGather(counts)");
    cudaError_t e = cudaMemcpyAsync(c->host_kx, c->kx_all, sizeof(long long) * 2 * c->world,
                                    cudaMemcpyDeviceToHost, stream);
    if (e != cudaSuccess) return cuda_fail(c, e, "exchange: count readback");
    // Flags are reported now; clear the local copy (stream-ordered after the gather).
    e = cudaMemsetAsync(&c->ctrl->flags, 0, sizeof(unsigned long long), stream);
    if (e != cudaSuccess) return cuda_fail(c, e, "exchange: flag clear");
    // 2. the one host wait of the step; poll NCCL for asynchronous errors
    //    meanwhile, and give up after the peer timeout: a rank that never
    //    joins the all-gather would otherwise hang this one forever.  The
    //    communicator is aborted (ncclCommAbort) and the context is dead.
    const auto t_wait = std::chrono::steady_clock::now();
    while (true) {
        e = cudaStreamQuery(stream);
        if (e == cudaSuccess) break;
        if (e != cudaErrorNotReady) return cuda_fail(c, e, "exchange: wait");
        ncclResult_t ar = ncclSuccess;
        if (ncclCommGetAsyncError(c->comm, &ar) == ncclSuccess && ar != ncclSuccess)
            return nccl_fail(c, ar, "exchange: async");
        const auto waited = std::chrono::steady_clock::now() - t_wait;
        if ((unsigned long long)std::chrono::duration_cast<std::chrono::nanoseconds>(waited).count() > c->timeout_ns) {
            ncclCommAbort(c->comm);
            c->comm = nullptr;
            c->dead = true;
            c->stage = Stage::kBound;
            return fail(c, GTC_EPEER, "exchange: a peer did not join the all-gather in time (communicator aborted)");
        }
        std::this_thread::yield();
    }
    unsigned long long any_flags = 0;
    long long max_k = 0;
    for (int i = 0; i < c->world; ++i) {
        c->last_k[i] = c->host_kx[2 * i];
        any_flags |= (unsigned long long)c->host_kx[2 * i + 1];
        max_k = std::max(max_k, c->last_k[i]);
    }
    if (any_flags & kFlagCapacity || max_k > c->capacity) {
        c->stage = Stage::kBound;
        return fail(c, GTC_ECAPACITY, "exchange: a rank's message exceeded the capacity");
    }
    c->max_k = max_k;
    // 3. words (padded to the largest k) and tile offsets, one NCCL group.
    r = ncclGroupStart();
    if (r == ncclSuccess && max_k > 0)
        r = ncclAllGather(c->ws + c->L.msg_words, c->recv, (size_t)max_k, ncclUint32, c->comm, stream);
    if (r == ncclSuccess)
        r = ncclAllGather(c->ws + c->L.msg_off, c->recv_off, (size_t)c->num_tiles + 1, ncclInt32, c->comm, stream);
    ncclResult_t r2 = ncclGroupEnd();
    if (r != ncclSuccess) return nccl_fail(c, r, "exchange: ncclAllGather(words)");
    if (r2 != ncclSuccess) return nccl_fail(c, r2, "exchange: ncclGroupEnd");
    c->stage = Stage::kExchanged;
    return (any_flags & kFlagNonFinite) ? fail(c, GTC_ENONFINITE, "exchange: a rank saw a non-finite residual")
                                        : GTC_OK;
}

gtc_status gtc_exchange(gtc_ctx* c, cudaStream_t stream) {
    NvtxRange nvtx("gtc_exchange");
    if (!c) return GTC_EINVAL;
    if (c->stage != Stage::kEncoded) return fail(c, GTC_ESTATE, "exchange: no encode since the last exchange");
    if (c->sharded) {
        DeviceGuard g(c->device);
        gtc_status s = owner_count(c, stream);
        if (s != GTC_OK) return s;
        c->stage = Stage::kExchanged;
        return GTC_OK;
    }
    if (c->world == 1 || c->p2p) {
        // world 1: nothing to send.  p2p: decode_apply raises this rank's
        // ready flag when it starts (loopback: gtc_encode did) and reads the
        // peers' tiles in place over NVLink once theirs are up.
        c->stage = Stage::kExchanged;
        return GTC_OK;
    }
    DeviceGuard g(c->device);
    return exchange_nccl(c, stream);
}

static gtc_status check_apply_args(gtc_ctx* c, float* target, int mode) {
    if (c->n > 0 && !target) return fail(c, GTC_EINVAL, "decode_apply: target is null");
    if (!aligned16(target)) return fail(c, GTC_EALIGN, "decode_apply: target alignment");
    if (mode != GTC_ACCUM_WEIGHTS && mode != GTC_ACCUM_UPDATE && mode != GTC_ACCUM_MOMENTUM)
        return fail(c, GTC_EINVAL, "decode_apply: mode");
    if (mode == GTC_ACCUM_MOMENTUM && c->n > 0 && !c->mom_buf)
        return fail(c, GTC_ESTATE, "decode_apply: GTC_ACCUM_MOMENTUM needs gtc_bind_momentum");
    return GTC_OK;
}

gtc_status gtc_bind_momentum(gtc_ctx* c, float* buf, float mu) {
    if (!c) return GTC_EINVAL;
    if (!std::isfinite(mu)) return fail(c, GTC_EINVAL, "bind_momentum: mu not finite");
    if (!aligned16(buf)) return fail(c, GTC_EALIGN, "bind_momentum: buffer alignment");
    c->mom_buf = buf;
    c->mom_mu = mu;
    return GTC_OK;
}

// Decode + apply every tile of the current step on `stream` (p2p: waiting on
// every rank's ready flag).
static gtc_status decode_launch(gtc_ctx* c, float* target, float alpha, int mode, int8_t* counts_out,
                                cudaStream_t stream) {
    if (c->sharded) {
        ShardParams q = shard_params(c);
        q.alpha = alpha;
        q.target = target;
        q.buf = c->mom_buf;
        q.mu = c->mom_mu;
        q.counts_out = reinterpret_cast<signed char*>(counts_out);
        const cudaError_t e = launch_apply_counts(q, mode, stream);
        if (e != cudaSuccess) return cuda_fail(c, e, "decode_apply: apply counts");
        if (c->num_tiles > 0) c->launches += 1;
        return GTC_OK;
    }
    DecodeParams p{};
    if (c->world == 1 || c->p2p) {
        const int par = seg_parity(c);
        p.segmented = 1;
        p.stamped = (c->world > 1 && c->p2p) ? 1 : 0;
        for (int i = 0; i < c->world; ++i) {
            unsigned char* b = rank_ws(c, i);
            p.seg[i] = reinterpret_cast<const unsigned*>(b + c->L.seg_words[par]);
            p.tags[i] = reinterpret_cast<const unsigned long long*>(b + c->L.seg_tags[par]);
        }
        p.epoch = c->epoch;
        p.step = c->encodes;
        p.wait = c->world > 1 ? 1 : 0;
        for (int i = 0; i < c->world && p.wait; ++i) {
            Ctrl* ci = reinterpret_cast<Ctrl*>(rank_ws(c, i) + c->L.ctrl);
            p.ready[i] = &ci->ready;
            p.peer_flags[i] = &ci->flags;
        }
        if (p.wait) p.publish = &c->ctrl->ready;
        p.timeout_ns = c->timeout_ns;
    } else {
        p.segmented = 0;
        for (int i = 0; i < c->world; ++i) {
            p.words[i] = c->recv + (size_t)i * (size_t)c->max_k;
            p.off[i] = c->recv_off + (size_t)i * (size_t)(c->num_tiles + 1);
        }
    }
    p.nmsg = c->world;
    p.n = c->n;
    p.num_tiles = c->num_tiles;
    p.tau = c->tau;
    p.alpha = alpha;
    p.target = target;
    p.buf = c->mom_buf;
    p.mu = c->mom_mu;
    p.counts_out = reinterpret_cast<signed char*>(counts_out);
    p.flags = &c->ctrl->flags;
    p.trace = decode_trace_enabled() ? 1 : 0;
    cudaError_t e = launch_decode_apply(p, mode, stream);
    if (e != cudaSuccess) return cuda_fail(c, e, "decode_apply: launch");
    if (c->num_tiles > 0) c->launches += 1;
    return GTC_OK;
}

gtc_status gtc_decode_apply(gtc_ctx* c, float* target, float alpha, int mode, int8_t* counts_out,
                            cudaStream_t stream) {
    NvtxRange nvtx("gtc_decode_apply");
    if (!c) return GTC_EINVAL;
    if (c->stage != Stage::kExchanged) return fail(c, GTC_ESTATE, "decode_apply: call gtc_exchange first");
    gtc_status s = check_apply_args(c, target, mode);
    if (s != GTC_OK) return s;
    DeviceGuard g(c->device);
    s = decode_launch(c, target, alpha, mode, counts_out, stream);
    if (s != GTC_OK) return s;
    c->stage = Stage::kBound;
    return GTC_OK;
}

// p2p, world > 1: the fused one-kernel step (step_p2p.cu) unless GTC_STEP_FUSED=0.
static bool fused_step_enabled() {
    static int v = -1;
    if (v < 0) {
        const char* e = std::getenv("GTC_STEP_FUSED");
        v = (e && e[0] == '0') ? 0 : 1;
    }
    return v == 1;
}

// The fused one-kernel step's parameters of rank c (begins the step: epoch,
// parity); clears this rank's push records on the peers first if the last
// step of this parity was not fused.
static gtc_status fill_fused(gtc_ctx* c, const float* grad, float* residual, float* target, float alpha,
                             cudaStream_t stream, int ranks_per_device, FusedStepParams& f) {
    begin_step(c);
    const int par = seg_parity(c);
    f = FusedStepParams{};
    EncodeParams& p = f.enc;
    p.g = grad;
    p.r = residual;
    p.n = c->n;
    p.tau = c->tau;
    p.seg = reinterpret_cast<unsigned*>(c->ws + c->L.seg_words[par]);
    p.tags = reinterpret_cast<unsigned long long*>(c->ws + c->L.seg_tags[par]);
    p.ctrl = c->ctrl;
    p.k_acc = &c->ctrl->k_acc[c->epoch & 1u];
    p.k_next = &c->ctrl->k_acc[(c->epoch + 1u) & 1u];
    p.epoch = c->epoch;
    p.buf = c->mom_buf;
    p.mu = c->mom_mu;
    p.publish_sys = 1;
    p.num_tiles = c->num_tiles;
    p.step = c->encodes;
    for (int i = 0; i < c->world; ++i) {
        unsigned char* b = rank_ws(c, i);
        f.seg[i] = reinterpret_cast<const unsigned*>(b + c->L.seg_words[par]);
        f.tags[i] = reinterpret_cast<const unsigned long long*>(b + c->L.seg_tags[par]);
        f.peer_flags[i] = &reinterpret_cast<Ctrl*>(b + c->L.ctrl)->flags;
        f.push_out[i] = nullptr;
        f.push_in[i] = nullptr;
        if (i == c->rank) continue;
        // this rank's records in rank i's push region, and rank i's in ours
        unsigned char* out = b + c->L.push + ((size_t)par * c->world + c->rank) * c->L.push_slot;
        if (!c->push_clean[par]) {
            // the last step of this parity was not fused: our records on the
            // peers may hold entries of older steps; clear them
            cudaError_t e = cudaMemsetAsync(out, 0, c->L.push_slot, stream);
            if (e != cudaSuccess) return cuda_fail(c, e, "step: push region reset");
        }
        f.push_out[i] = out;
        f.push_in[i] = c->ws + c->L.push + ((size_t)par * c->world + i) * c->L.push_slot;
    }
    c->push_clean[par] = true;
    f.rank = c->rank;
    f.nranks = c->world;
    f.spec_window = kTileThreads / c->world;
    f.spec_shift = -1;
    for (int sh = 0; sh < 9; ++sh)
        if ((1 << sh) == f.spec_window) f.spec_shift = sh;
    f.stamp = entry_stamp(c->epoch);
    f.lag_tiles = step_p2p_lag_tiles(c->num_tiles, ranks_per_device);
    f.ticket = &c->ctrl->ticket;
    f.target = target;
    f.alpha = alpha;
    f.flags = &c->ctrl->flags;
    f.timeout_ns = c->timeout_ns;
    f.trace = decode_trace_enabled() ? 1 : 0;
    return GTC_OK;
}

static gtc_status step_fused_p2p(gtc_ctx* c, const float* grad, float* residual, float* target, float alpha,
                                 int mode, cudaStream_t stream) {
    FusedStepParams f;
    gtc_status s = fill_fused(c, grad, residual, target, alpha, stream, 1, f);
    if (s != GTC_OK) return s;
    cudaError_t e = launch_step_p2p(f, c->cmp_mode, mode, stream);
    if (e != cudaSuccess) return cuda_fail(c, e, "step: fused p2p launch");
    c->launches += 1;
    c->stage = Stage::kBound;
    return GTC_OK;
}

gtc_status gtc_step(gtc_ctx* c, const float* grad, float* residual, float* target, float alpha, int mode,
                    cudaStream_t stream) {
    NvtxRange nvtx("gtc_step");
    if (c && c->world == 1) {
        // world 1: the aggregate is this rank's own quanta (c = +-1 on its
        // message), so the encode kernel applies them itself: one launch per step
        gtc_status s = check_apply_args(c, target, mode);
        if (s != GTC_OK) return s;
        if (c->n > 0 && c->num_tiles > 0) {
            s = encode_impl(c, grad, residual, stream, target, alpha, mode);
            if (s != GTC_OK) return s;
        } else {
            s = gtc_encode(c, grad, residual, stream);
            if (s != GTC_OK) return s;
        }
        c->stage = Stage::kBound;
        return GTC_OK;
    }
    if (c && c->loopback)
        // one rank's whole step would wait on ranks whose encode is not yet
        // queued: a loopback group steps with gtc_step_group, or with every
        // rank's encode, then exchange, then decode_apply
        return fail(c, GTC_EUNSUPPORTED, "step: loopback contexts step with gtc_step_group");
    if (c && c->world > 1 && c->p2p && c->bound && c->num_tiles > 1 && !c->split_step && !c->sharded &&
        fused_step_enabled() && c->world <= kFusedMaxRanks) {
        gtc_status s = check_encode_args(c, grad, residual);
        if (s == GTC_OK) s = check_apply_args(c, target, mode);
        if (s != GTC_OK) return s;
        DeviceGuard g(c->device);
        return step_fused_p2p(c, grad, residual, target, alpha, mode, stream);
    }
    gtc_status s = gtc_encode(c, grad, residual, stream);
    if (s != GTC_OK) return s;
    const gtc_status sx = gtc_exchange(c, stream);
    if (sx != GTC_OK && sx != GTC_ENONFINITE) return sx;
    s = gtc_decode_apply(c, target, alpha, mode, nullptr, stream);
    return s != GTC_OK ? s : sx;
}

gtc_status gtc_connect_loopback(gtc_ctx* const* ctxs, int world) {
    if (!ctxs || world < 2 || world > kFusedMaxRanks) return GTC_EINVAL;
    for (int r = 0; r < world; ++r) {
        gtc_ctx* c = ctxs[r];
        if (!c || !c->loopback || c->world != world || c->rank != r) return fail(c, GTC_EINVAL, "loopback: ranks");
        if (!c->bound) return fail(c, GTC_ESTATE, "loopback: bind every workspace first");
        if (c->n != ctxs[0]->n || c->tau != ctxs[0]->tau || c->cmp_mode != ctxs[0]->cmp_mode ||
            c->L.total != ctxs[0]->L.total)
            return fail(c, GTC_EINVAL, "loopback: every rank needs the same n, tau, flags and workspace sizes");
    }
    // peers on other devices of this process: their memory must be mapped
    for (int r = 0; r < world; ++r) {
        for (int m = 0; m < world; ++m) {
            if (ctxs[m]->device == ctxs[r]->device) continue;
            DeviceGuard g(ctxs[r]->device);
            cudaError_t e = cudaDeviceEnablePeerAccess(ctxs[m]->device, 0);
            if (e == cudaErrorPeerAccessAlreadyEnabled) {
                cudaGetLastError();
            } else if (e != cudaSuccess) {
                return cuda_fail(ctxs[r], e, "loopback: cudaDeviceEnablePeerAccess");
            }
        }
    }
    for (int r = 0; r < world; ++r) {
        gtc_ctx* c = ctxs[r];
        c->peer_ws.assign(world, nullptr);
        for (int m = 0; m < world; ++m) c->peer_ws[m] = ctxs[m]->ws;
        c->peer_alloc.assign(world, nullptr);
        c->connected = true;
    }
    return GTC_OK;
}

gtc_status gtc_step_group(gtc_ctx* const* ctxs, int world, const float* const* grads, float* const* residuals,
                          float* const* targets, float alpha, int mode, uint32_t debug_flags, cudaStream_t stream) {
    NvtxRange nvtx("gtc_step_group");
    if (!ctxs || world < 2 || world > kFusedMaxRanks || !residuals || !targets) return GTC_EINVAL;
    gtc_ctx* c0 = ctxs[0];
    if (!c0 || !c0->host_group) return fail(c0, GTC_EINVAL, "step_group: ctxs[0] is not rank 0 of a loopback group");
    if (debug_flags >> kFusedMaxRanks) return fail(c0, GTC_EINVAL, "step_group: debug_flags");
    for (int r = 0; r < world; ++r) {
        gtc_ctx* c = ctxs[r];
        if (!c || !c->loopback || c->rank != r || c->world != world) return fail(c0, GTC_EINVAL, "step_group: ranks");
        if (c->device != c0->device) return fail(c, GTC_EUNSUPPORTED, "step_group: every rank on one device");
        const float* g = grads ? grads[r] : nullptr;
        if ((g == nullptr) != (grads == nullptr || grads[0] == nullptr))
            return fail(c, GTC_EINVAL, "step_group: grads on every rank or on none");
        gtc_status s = check_encode_args(c, g, residuals[r]);
        if (s == GTC_OK) s = check_apply_args(c, targets[r], mode);
        if (s != GTC_OK) return s;
    }
    if (c0->num_tiles == 0) return GTC_OK;
    DeviceGuard guard(c0->device);
    // the previous launch must be done reading the staging buffer
    cudaError_t e = cudaStreamSynchronize(stream);
    if (e != cudaSuccess) return cuda_fail(c0, e, "step_group: sync");
    for (int r = 0; r < world; ++r) {
        gtc_ctx* c = ctxs[r];
        gtc_status s = fill_fused(c, grads ? grads[r] : nullptr, residuals[r], targets[r], alpha, stream, world,
                                  c0->host_group[r]);
        if (s != GTC_OK) return s;
        c0->host_group[r].skip = (int)((debug_flags >> r) & 1u);
    }
    FusedStepParams* dev = reinterpret_cast<FusedStepParams*>(c0->ws + c0->L.group);
    e = cudaMemcpyAsync(dev, c0->host_group, sizeof(FusedStepParams) * world, cudaMemcpyHostToDevice, stream);
    if (e != cudaSuccess) return cuda_fail(c0, e, "step_group: parameters");
    e = launch_step_p2p_group(dev, c0->host_group[0], world, c0->cmp_mode, mode, stream);
    if (e != cudaSuccess) return cuda_fail(c0, e, "step_group: launch");
    for (int r = 0; r < world; ++r) {
        ctxs[r]->launches += 1;
        ctxs[r]->stage = Stage::kBound;
    }
    return GTC_OK;
}

gtc_status gtc_decode_apply_msgs(gtc_ctx* c, const uint32_t* const* msgs, const int64_t* counts, int nmsg,
                                 float* target, float alpha, int mode, int8_t* counts_out,
                                 cudaStream_t stream) {
    if (!c) return GTC_EINVAL;
    if (!c->bound) return fail(c, GTC_ESTATE, "decode_apply_msgs: workspace not bound");
    if (nmsg < 0 || nmsg > c->max_sim_msgs) return fail(c, GTC_EINVAL, "decode_apply_msgs: nmsg > max_sim_msgs");
    if (nmsg > 0 && (!msgs || !counts)) return fail(c, GTC_EINVAL, "decode_apply_msgs: null arrays");
    gtc_status s = check_apply_args(c, target, mode);
    if (s != GTC_OK) return s;
    for (int m = 0; m < nmsg; ++m) {
        if (counts[m] < 0 || counts[m] > c->n) return fail(c, GTC_ECORRUPT, "decode_apply_msgs: count out of range");
        if (counts[m] > 0 && !msgs[m]) return fail(c, GTC_EINVAL, "decode_apply_msgs: null message");
    }
    DeviceGuard g(c->device);
    if (c->num_tiles == 0) return GTC_OK;
    // Clear a stale corrupt flag so this call's validation stands alone.
    cudaError_t e = cudaMemsetAsync(&c->ctrl->flags, 0, sizeof(unsigned long long), stream);
    if (e != cudaSuccess) return cuda_fail(c, e, "decode_apply_msgs: flag clear");
    BoundsParams b{};
    DecodeParams p{};
    static const unsigned kEmpty = 0u;
    for (int m = 0; m < nmsg; ++m) {
        b.words[m] = msgs[m] ? msgs[m] : &kEmpty;
        b.k[m] = counts[m];
        b.off[m] = c->sim_off + (size_t)m * (size_t)(c->num_tiles + 1);
        p.words[m] = b.words[m];
        p.off[m] = b.off[m];
    }
    b.nmsg = nmsg;
    b.n = c->n;
    b.num_tiles = c->num_tiles;
    b.flags = &c->ctrl->flags;
    e = launch_tile_bounds(b, stream);
    if (e != cudaSuccess) return cuda_fail(c, e, "decode_apply_msgs: bounds launch");
    if (nmsg > 0) c->launches += 1;
    p.segmented = 0;
    p.nmsg = nmsg;
    p.n = c->n;
    p.num_tiles = c->num_tiles;
    p.tau = c->tau;
    p.alpha = alpha;
    p.target = target;
    p.buf = c->mom_buf;
    p.mu = c->mom_mu;
    p.counts_out = reinterpret_cast<signed char*>(counts_out);
    p.flags = &c->ctrl->flags;
    e = launch_decode_apply(p, mode, stream);
    if (e != cudaSuccess) return cuda_fail(c, e, "decode_apply_msgs: launch");
    c->launches += 1;
    unsigned long long f = 0;
    e = cudaMemcpyAsync(c->host_kx, &c->ctrl->flags, sizeof(f), cudaMemcpyDeviceToHost, stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
    if (e != cudaSuccess) return cuda_fail(c, e, "decode_apply_msgs: wait");
    f = (unsigned long long)c->host_kx[0];
    if (f & kFlagCorrupt) {
        cudaMemsetAsync(&c->ctrl->flags, 0, sizeof(unsigned long long), stream);
        cudaStreamSynchronize(stream);
        return fail(c, GTC_ECORRUPT, "decode_apply_msgs: message not canonical");
    }
    return GTC_OK;
}

gtc_status gtc_local_count(const gtc_ctx* c, const int64_t** dev_k) {
    if (!c || !dev_k) return GTC_EINVAL;
    if (!c->bound) return GTC_ESTATE;
    *dev_k = reinterpret_cast<const int64_t*>(&c->ctrl->k_acc[c->epoch & 1u]);
    return GTC_OK;
}

// Contiguous copy of `rank`'s message of the current step in this rank's
// contiguous region (packs it if needed); waits for the device.
static gtc_status contiguous_message(gtc_ctx* c, int rank, const uint32_t** dev_words, int64_t* k) {
    DeviceGuard g(c->device);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) return cuda_fail(c, e, "message: sync");
    if (c->packed_rank != rank) {
        gtc_status s = pack_contiguous(c, rank, 0);
        if (s != GTC_OK) return s;
        e = cudaDeviceSynchronize();
        if (e != cudaSuccess) return cuda_fail(c, e, "message: pack");
    }
    MsgHeader h{};
    e = cudaMemcpy(&h, c->ws + c->L.msg_hdr, sizeof(h), cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return cuda_fail(c, e, "message: header");
    if (h.k > c->capacity) return fail(c, GTC_ECAPACITY, "message: larger than max_words_per_rank");
    *dev_words = reinterpret_cast<const uint32_t*>(c->ws + c->L.msg_words);
    *k = h.k;
    return GTC_OK;
}

gtc_status gtc_last_counts(gtc_ctx* c, int64_t* k_per_rank) {
    if (!c || !k_per_rank) return GTC_EINVAL;
    if (!c->bound) return fail(c, GTC_ESTATE, "last_counts: workspace not bound");
    if (c->world > 1 && !c->p2p) {
        for (int i = 0; i < c->world; ++i) k_per_rank[i] = c->last_k[i];
        return GTC_OK;
    }
    DeviceGuard g(c->device);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) return cuda_fail(c, e, "last_counts: sync");
    // sum of every rank's tile counts of the last encode
    const int par = seg_parity(c);
    std::vector<unsigned long long> tags(c->num_tiles);
    for (int i = 0; i < c->world; ++i) {
        if (c->num_tiles > 0) {
            e = cudaMemcpy(tags.data(), rank_ws(c, i) + c->L.seg_tags[par],
                           sizeof(unsigned long long) * c->num_tiles, cudaMemcpyDeviceToHost);
            if (e != cudaSuccess) return cuda_fail(c, e, "last_counts: readback");
        }
        long long k = 0;
        for (unsigned long long v : tags) k += (long long)(v & 0xffffffffull);
        k_per_rank[i] = k;
    }
    return GTC_OK;
}

gtc_status gtc_message(gtc_ctx* c, int rank, const uint32_t** dev_words, int64_t* k) {
    if (!c || !dev_words || !k) return GTC_EINVAL;
    if (!c->bound) return fail(c, GTC_ESTATE, "message: workspace not bound");
    if (rank < 0 || rank >= c->world) return fail(c, GTC_EINVAL, "message: rank");
    if (c->world > 1 && !c->p2p) {
        *dev_words = c->recv + (size_t)rank * (size_t)c->max_k;
        *k = c->last_k[rank];
        return GTC_OK;
    }
    return contiguous_message(c, rank, dev_words, k);
}

gtc_status gtc_read_message(gtc_ctx* c, int rank, uint32_t* host_words, int64_t max_words, int64_t* k) {
    if (!c || !k) return GTC_EINVAL;
    const uint32_t* dev = nullptr;
    gtc_status s = gtc_message(c, rank, &dev, k);
    if (s != GTC_OK) return s;
    if (*k > max_words || (*k > 0 && !host_words)) return fail(c, GTC_EINVAL, "read_message: buffer too small");
    DeviceGuard g(c->device);
    cudaError_t e = cudaDeviceSynchronize();
    if (e == cudaSuccess && *k > 0) e = cudaMemcpy(host_words, dev, sizeof(uint32_t) * (size_t)*k, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return cuda_fail(c, e, "read_message: copy");
    return GTC_OK;
}

gtc_status gtc_wire_pack(const uint32_t* words, int64_t k, uint64_t dim, float tau, void* out,
                         size_t out_bytes, size_t* written) {
    if (!written || k < 0 || (k > 0 && !words)) return GTC_EINVAL;
    if (dim >= (1ull << 31)) return GTC_EDIM;
    if (!(tau > 0.f) || !std::isfinite(tau)) return GTC_EINVAL;
    const size_t need = 20 + 4 * (size_t)k;
    *written = need;
    if (!out || out_bytes < need) return GTC_EINVAL;
    for (int64_t j = 0; j < k; ++j) {
        const uint32_t i = words[j] >> 1;
        if (i >= dim || (j > 0 && i <= (words[j - 1] >> 1))) return GTC_ECORRUPT;
    }
    unsigned char* o = static_cast<unsigned char*>(out);
    const uint32_t kk = (uint32_t)k;
    std::memcpy(o, "GTCU", 4);
    std::memcpy(o + 4, &dim, 8);  // the ABI's hosts are little-endian (x86-64, aarch64)
    std::memcpy(o + 12, &tau, 4);
    std::memcpy(o + 16, &kk, 4);
    for (int64_t j = 0; j < k; ++j) {
        const uint32_t w = ((words[j] & 1u) << 31) | (words[j] >> 1);  // SPEC: bit 31 = sign, bits 0..30 = index
        std::memcpy(o + 20 + 4 * j, &w, 4);
    }
    return GTC_OK;
}

gtc_status gtc_wire_unpack(const void* in, size_t in_bytes, uint32_t* words, int64_t max_words, int64_t* k,
                           uint64_t* dim, float* tau) {
    if (!in || !k || !dim || !tau) return GTC_EINVAL;
    const unsigned char* b = static_cast<const unsigned char*>(in);
    if (in_bytes < 20 || std::memcmp(b, "GTCU", 4) != 0) return GTC_ECORRUPT;
    uint64_t d;
    float t;
    uint32_t kk;
    std::memcpy(&d, b + 4, 8);
    std::memcpy(&t, b + 12, 4);
    std::memcpy(&kk, b + 16, 4);
    if (d >= (1ull << 31) || !(t > 0.f) || !std::isfinite(t) || in_bytes != 20 + 4 * (size_t)kk) return GTC_ECORRUPT;
    if ((int64_t)kk > max_words || (kk > 0 && !words)) return GTC_EINVAL;
    uint32_t prev = 0;
    for (uint32_t j = 0; j < kk; ++j) {
        uint32_t w;
        std::memcpy(&w, b + 20 + 4 * (size_t)j, 4);
        const uint32_t i = w & 0x7fffffffu;
        if (i >= d || (j > 0 && i <= prev)) return GTC_ECORRUPT;
        prev = i;
        words[j] = (i << 1) | (w >> 31);
    }
    *k = kk;
    *dim = d;
    *tau = t;
    return GTC_OK;
}

gtc_status gtc_check(gtc_ctx* c, cudaStream_t stream) {
    if (!c) return GTC_EINVAL;
    if (!c->bound) return fail(c, GTC_ESTATE, "check: workspace not bound");
    DeviceGuard g(c->device);
    cudaError_t e = cudaMemcpyAsync(c->host_kx, &c->ctrl->flags, sizeof(unsigned long long),
                                    cudaMemcpyDeviceToHost, stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
    if (e != cudaSuccess) return cuda_fail(c, e, "check: wait");
    const unsigned long long f = (unsigned long long)c->host_kx[0];
    if (f) {
        e = cudaMemsetAsync(&c->ctrl->flags, 0, sizeof(unsigned long long), stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
        if (e != cudaSuccess) return cuda_fail(c, e, "check: clear");
    }
    return flags_to_status(f);
}

int gtc_exchange_mode(const gtc_ctx* c) {
    if (!c) return -1;
    return c->world == 1 ? 0 : (c->p2p ? GTC_EXCHANGE_P2P : GTC_EXCHANGE_NCCL);
}

int64_t gtc_kernel_launches(const gtc_ctx* c) { return c ? c->launches : 0; }

gtc_status gtc_debug_decode_trace(uint64_t* host, int max_entries) {
    if (!host || max_entries < 0) return GTC_EINVAL;
    return read_decode_trace(reinterpret_cast<unsigned long long*>(host), max_entries) == cudaSuccess ? GTC_OK
                                                                                                    : GTC_ECUDA;
}

gtc_status gtc_debug_step_trace(uint64_t* host, int max_entries) {
    if (!host || max_entries < 0) return GTC_EINVAL;
    return read_step_trace(reinterpret_cast<unsigned long long*>(host), max_entries) == cudaSuccess ? GTC_OK
                                                                                                : GTC_ECUDA;
}

gtc_status gtc_quiesce(gtc_ctx* c) {
    if (!c) return GTC_EINVAL;
    DeviceGuard g(c->device);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) return cuda_fail(c, e, "quiesce: sync");
    if (c->bound && c->p2p && c->comm && !c->dead) {
        // barrier: no peer may still be reading this rank's workspace (and
        // this rank is done with theirs) when the mappings go away
        int* d = reinterpret_cast<int*>(c->ws + c->L.ipc);
        ncclResult_t r = ncclAllReduce(d, d, 1, ncclInt32, ncclSum, c->comm, 0);
        if (r != ncclSuccess) return nccl_fail(c, r, "quiesce: barrier");
        e = cudaStreamSynchronize(0);
        if (e != cudaSuccess) return cuda_fail(c, e, "quiesce: barrier wait");
    }
    return GTC_OK;
}

void gtc_destroy(gtc_ctx* c) {
    if (!c) return;
    DeviceGuard g(c->device);
    cudaDeviceSynchronize();
    ipc_unmap(c->peer_alloc);
    if (c->comm) ncclCommDestroy(c->comm);
    if (c->host_kx) cudaFreeHost(c->host_kx);
    if (c->host_group) cudaFreeHost(c->host_group);
    delete c;
}

}  // extern "C"
