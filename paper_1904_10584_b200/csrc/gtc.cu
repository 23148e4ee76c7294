// gtc.cu -- the C ABI of libgtc.so (include/gtc.h): context, workspace layout,
// argument validation, call ordering and the NCCL exchange (PAPER.md:222
// "Each worker communicates the sparse update to all other workers and
// conversely receives all sparse updates from other workers").
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "gtc_internal.cuh"

using namespace gtc;

namespace {

enum class Stage { kBound, kEncoded, kExchanged };

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// Workspace layout (offsets from the bound base, each 256-byte aligned):
//   ctrl      Ctrl                              k, flags
//   chunk_sum u32[kMaxChunks]                   words per encode-kernel-1 chunk
//   tile_cnt  i32[num_tiles]                    words per tile
//   tile_off  i32[num_tiles + 1]                this rank's tile offsets
//   scratch   u32[num_tiles * kTile]            tile-major words (encode kernel 1)
//   send      u32[capacity]                     this rank's message
//   kx_all    i64[2 * world]                    all-gathered (k, flags)   (world > 1)
//   recv      u32[world * capacity]             all-gathered messages     (world > 1)
//   recv_off  i32[world * (num_tiles + 1)]      all-gathered tile offsets (world > 1)
//   sim_off   i32[max_sim_msgs * (num_tiles+1)] tile offsets for decode_apply_msgs
struct Layout {
    size_t ctrl, chunk_sum, tile_cnt, tile_off, scratch, send, kx_all, recv, recv_off, sim_off, total;
};

Layout make_layout(long long n, int world, long long capacity, int max_sim_msgs) {
    const long long tiles = (n + kTile - 1) / kTile;
    Layout L{};
    size_t o = 0;
    L.ctrl = o;      o = align_up(o + sizeof(Ctrl), 256);
    L.chunk_sum = o; o = align_up(o + sizeof(unsigned) * (size_t)kMaxChunks, 256);
    L.tile_cnt = o;  o = align_up(o + sizeof(int) * (size_t)std::max(tiles, 1LL), 256);
    L.tile_off = o;  o = align_up(o + sizeof(int) * (size_t)(tiles + 1), 256);
    L.scratch = o;   o = align_up(o + sizeof(unsigned) * (size_t)std::max(tiles, 1LL) * kTile, 256);
    L.send = o;      o = align_up(o + sizeof(unsigned) * (size_t)std::max(capacity, 1LL), 256);
    if (world > 1) {
        L.kx_all = o;   o = align_up(o + sizeof(long long) * 2 * (size_t)world, 256);
        L.recv = o;     o = align_up(o + sizeof(unsigned) * (size_t)world * (size_t)std::max(capacity, 1LL), 256);
        L.recv_off = o; o = align_up(o + sizeof(int) * (size_t)world * (size_t)(tiles + 1), 256);
    } else {
        L.kx_all = L.recv = L.recv_off = 0;
    }
    L.sim_off = o;   o = align_up(o + sizeof(int) * (size_t)std::max(max_sim_msgs, 0) * (size_t)(tiles + 1), 256);
    L.total = o;
    return L;
}

}  // namespace

struct gtc_ctx {
    long long n = 0;
    float tau = 0.f;
    int rank = 0, world = 1, device = 0;
    int cmp_mode = GTC_CMP_GT;
    int num_tiles = 0;
    ncclComm_t comm = nullptr;

    unsigned char* ws = nullptr;
    size_t ws_bytes = 0;
    long long capacity = 0;
    int max_sim_msgs = 0;
    Layout L{};

    Ctrl* ctrl = nullptr;
    unsigned* chunk_sum = nullptr;
    int* tile_cnt = nullptr;
    int* tile_off = nullptr;
    unsigned* scratch = nullptr;
    unsigned* send = nullptr;
    long long* kx_all = nullptr;
    unsigned* recv = nullptr;
    int* recv_off = nullptr;
    int* sim_off = nullptr;

    long long* host_kx = nullptr;  // pinned, 2 * world
    std::vector<long long> last_k;
    long long max_k = 0;

    Stage stage = Stage::kBound;
    bool bound = false;
    long long launches = 0;
    std::string detail;
};

namespace {

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
    if (f & kFlagCapacity) return GTC_ECAPACITY;
    if (f & kFlagCorrupt) return GTC_ECORRUPT;
    if (f & kFlagNonFinite) return GTC_ENONFINITE;
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
    if (flags != GTC_CMP_GT && flags != GTC_CMP_GE) return GTC_EINVAL;
    if ((world > 1) != (nccl_unique_id != nullptr)) return GTC_EINVAL;

    gtc_ctx* c = new (std::nothrow) gtc_ctx();
    if (!c) return GTC_EINVAL;
    c->n = n_params;
    c->tau = tau;
    c->rank = rank;
    c->world = world;
    c->device = cuda_device;
    c->cmp_mode = (int)flags;
    c->num_tiles = (int)((n_params + kTile - 1) / kTile);
    c->last_k.assign(world, 0);

    DeviceGuard g(cuda_device);
    cudaError_t e = cudaHostAlloc(reinterpret_cast<void**>(&c->host_kx),
                                  sizeof(long long) * 2 * (size_t)world, cudaHostAllocDefault);
    if (e != cudaSuccess) {
        delete c;
        return GTC_ECUDA;
    }
    if (world > 1) {
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
    *bytes = make_layout(c->n, c->world, cap, max_sim_msgs).total;
    return GTC_OK;
}

gtc_status gtc_bind_workspace(gtc_ctx* c, void* dev_ptr, size_t bytes, int64_t max_words_per_rank,
                              int max_sim_msgs) {
    if (!c || !dev_ptr) return fail(c, GTC_EINVAL, "bind: null");
    if (reinterpret_cast<uintptr_t>(dev_ptr) & 255u) return fail(c, GTC_EALIGN, "workspace not 256-byte aligned");
    if (max_sim_msgs < 0 || max_sim_msgs > GTC_MAX_MSGS) return fail(c, GTC_EINVAL, "max_sim_msgs");
    const long long cap = max_words_per_rank <= 0 ? c->n : std::min<long long>(max_words_per_rank, c->n);
    const Layout L = make_layout(c->n, c->world, cap, max_sim_msgs);
    if (bytes < L.total) return fail(c, GTC_EINVAL, "workspace too small");
    DeviceGuard g(c->device);
    unsigned char* b = static_cast<unsigned char*>(dev_ptr);
    // Control block, chunk sums, counts and offsets start at 0.
    cudaError_t e = cudaMemset(b, 0, L.scratch);
    if (e != cudaSuccess) return cuda_fail(c, e, "bind: cudaMemset");
    e = cudaDeviceSynchronize();
    if (e != cudaSuccess) return cuda_fail(c, e, "bind: sync");
    c->ws = b;
    c->ws_bytes = bytes;
    c->capacity = cap;
    c->max_sim_msgs = max_sim_msgs;
    c->L = L;
    c->ctrl = reinterpret_cast<Ctrl*>(b + L.ctrl);
    c->chunk_sum = reinterpret_cast<unsigned*>(b + L.chunk_sum);
    c->tile_cnt = reinterpret_cast<int*>(b + L.tile_cnt);
    c->tile_off = reinterpret_cast<int*>(b + L.tile_off);
    c->scratch = reinterpret_cast<unsigned*>(b + L.scratch);
    c->send = reinterpret_cast<unsigned*>(b + L.send);
    if (c->world > 1) {
        c->kx_all = reinterpret_cast<long long*>(b + L.kx_all);
        c->recv = reinterpret_cast<unsigned*>(b + L.recv);
        c->recv_off = reinterpret_cast<int*>(b + L.recv_off);
    }
    c->sim_off = reinterpret_cast<int*>(b + L.sim_off);
    c->bound = true;
    c->stage = Stage::kBound;
    return GTC_OK;
}

gtc_status gtc_encode(gtc_ctx* c, const float* grad, float* residual, cudaStream_t stream) {
    if (!c) return GTC_EINVAL;
    if (!c->bound) return fail(c, GTC_ESTATE, "encode: workspace not bound");
    if (c->n > 0 && !residual) return fail(c, GTC_EINVAL, "encode: residual is null");
    if (!aligned16(residual) || !aligned16(grad)) return fail(c, GTC_EALIGN, "encode: grad/residual alignment");
    DeviceGuard g(c->device);

    if (c->num_tiles == 0) {  // n == 0: empty message
        cudaError_t e = cudaMemsetAsync(&c->ctrl->k, 0, sizeof(long long), stream);
        if (e == cudaSuccess) e = cudaMemsetAsync(c->tile_off, 0, sizeof(int), stream);
        if (e != cudaSuccess) return cuda_fail(c, e, "encode: n == 0");
        c->stage = Stage::kEncoded;
        return GTC_OK;
    }

    EncodeParams p{};
    p.g = grad;
    p.r = residual;
    p.n = c->n;
    p.tau = c->tau;
    p.words = c->send;
    p.capacity = c->capacity;
    p.scratch = c->scratch;
    p.tile_cnt = c->tile_cnt;
    p.chunk_sum = c->chunk_sum;
    p.tile_off = c->tile_off;
    p.ctrl = c->ctrl;
    p.num_tiles = c->num_tiles;
    cudaError_t e = launch_encode(p, c->cmp_mode, stream);
    if (e != cudaSuccess) return cuda_fail(c, e, "encode: launch");
    c->launches += 2;
    c->stage = Stage::kEncoded;
    return GTC_OK;
}

gtc_status gtc_exchange(gtc_ctx* c, cudaStream_t stream) {
    if (!c) return GTC_EINVAL;
    if (c->stage != Stage::kEncoded) return fail(c, GTC_ESTATE, "exchange: no encode since the last exchange");
    if (c->world == 1) {
        c->stage = Stage::kExchanged;
        return GTC_OK;
    }
    DeviceGuard g(c->device);
    // 1. (k, flags) of every rank.  Ctrl::k and Ctrl::flags are adjacent.
    ncclResult_t r = ncclAllGather(&c->ctrl->k, c->kx_all, 2, ncclInt64, c->comm, stream);
    if (r != ncclSuccess) return nccl_fail(c, r, "exchange: ncclAllGather(counts)");
    cudaError_t e = cudaMemcpyAsync(c->host_kx, c->kx_all, sizeof(long long) * 2 * c->world,
                                    cudaMemcpyDeviceToHost, stream);
    if (e != cudaSuccess) return cuda_fail(c, e, "exchange: count readback");
    // Flags are reported now; clear the local copy (stream-ordered after the gather).
    e = cudaMemsetAsync(&c->ctrl->flags, 0, sizeof(unsigned long long), stream);
    if (e != cudaSuccess) return cuda_fail(c, e, "exchange: flag clear");
    // 2. the one host wait of the step; poll NCCL for asynchronous errors meanwhile.
    while (true) {
        e = cudaStreamQuery(stream);
        if (e == cudaSuccess) break;
        if (e != cudaErrorNotReady) return cuda_fail(c, e, "exchange: wait");
        ncclResult_t ar = ncclSuccess;
        if (ncclCommGetAsyncError(c->comm, &ar) == ncclSuccess && ar != ncclSuccess)
            return nccl_fail(c, ar, "exchange: async");
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
        r = ncclAllGather(c->send, c->recv, (size_t)max_k, ncclUint32, c->comm, stream);
    if (r == ncclSuccess)
        r = ncclAllGather(c->tile_off, c->recv_off, (size_t)c->num_tiles + 1, ncclInt32, c->comm, stream);
    ncclResult_t r2 = ncclGroupEnd();
    if (r != ncclSuccess) return nccl_fail(c, r, "exchange: ncclAllGather(words)");
    if (r2 != ncclSuccess) return nccl_fail(c, r2, "exchange: ncclGroupEnd");
    c->stage = Stage::kExchanged;
    return (any_flags & kFlagNonFinite) ? fail(c, GTC_ENONFINITE, "exchange: a rank saw a non-finite residual")
                                        : GTC_OK;
}

static gtc_status check_apply_args(gtc_ctx* c, float* target, int mode) {
    if (c->n > 0 && !target) return fail(c, GTC_EINVAL, "decode_apply: target is null");
    if (!aligned16(target)) return fail(c, GTC_EALIGN, "decode_apply: target alignment");
    if (mode != GTC_ACCUM_WEIGHTS && mode != GTC_ACCUM_UPDATE) return fail(c, GTC_EINVAL, "decode_apply: mode");
    return GTC_OK;
}

gtc_status gtc_decode_apply(gtc_ctx* c, float* target, float alpha, int mode, int8_t* counts_out,
                            cudaStream_t stream) {
    if (!c) return GTC_EINVAL;
    if (c->stage != Stage::kExchanged) return fail(c, GTC_ESTATE, "decode_apply: call gtc_exchange first");
    gtc_status s = check_apply_args(c, target, mode);
    if (s != GTC_OK) return s;
    DeviceGuard g(c->device);
    DecodeParams p{};
    if (c->world == 1) {
        p.m.words[0] = c->send;
        p.m.off[0] = c->tile_off;
    } else {
        for (int i = 0; i < c->world; ++i) {
            p.m.words[i] = c->recv + (size_t)i * (size_t)c->max_k;
            p.m.off[i] = c->recv_off + (size_t)i * (size_t)(c->num_tiles + 1);
        }
    }
    p.nmsg = c->world;
    p.n = c->n;
    p.num_tiles = c->num_tiles;
    p.tau = c->tau;
    p.alpha = alpha;
    p.target = target;
    p.counts_out = reinterpret_cast<signed char*>(counts_out);
    p.flags = &c->ctrl->flags;
    cudaError_t e = launch_decode_apply(p, mode, stream);
    if (e != cudaSuccess) return cuda_fail(c, e, "decode_apply: launch");
    if (c->num_tiles > 0) c->launches += 1;
    c->stage = Stage::kBound;
    return GTC_OK;
}

gtc_status gtc_step(gtc_ctx* c, const float* grad, float* residual, float* target, float alpha, int mode,
                    cudaStream_t stream) {
    gtc_status s = gtc_encode(c, grad, residual, stream);
    if (s != GTC_OK) return s;
    const gtc_status sx = gtc_exchange(c, stream);
    if (sx != GTC_OK && sx != GTC_ENONFINITE) return sx;
    s = gtc_decode_apply(c, target, alpha, mode, nullptr, stream);
    return s != GTC_OK ? s : sx;
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
        p.m.words[m] = b.words[m];
        p.m.off[m] = b.off[m];
    }
    b.nmsg = nmsg;
    b.n = c->n;
    b.num_tiles = c->num_tiles;
    b.flags = &c->ctrl->flags;
    e = launch_tile_bounds(b, stream);
    if (e != cudaSuccess) return cuda_fail(c, e, "decode_apply_msgs: bounds launch");
    if (nmsg > 0) c->launches += 1;
    p.nmsg = nmsg;
    p.n = c->n;
    p.num_tiles = c->num_tiles;
    p.tau = c->tau;
    p.alpha = alpha;
    p.target = target;
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
    *dev_k = reinterpret_cast<const int64_t*>(&c->ctrl->k);
    return GTC_OK;
}

gtc_status gtc_last_counts(gtc_ctx* c, int64_t* k_per_rank) {
    if (!c || !k_per_rank) return GTC_EINVAL;
    if (!c->bound) return fail(c, GTC_ESTATE, "last_counts: workspace not bound");
    if (c->world == 1) {
        DeviceGuard g(c->device);
        long long k = 0;
        cudaError_t e = cudaMemcpy(&k, &c->ctrl->k, sizeof(k), cudaMemcpyDeviceToHost);
        if (e != cudaSuccess) return cuda_fail(c, e, "last_counts: readback");
        k_per_rank[0] = k;
        return GTC_OK;
    }
    for (int i = 0; i < c->world; ++i) k_per_rank[i] = c->last_k[i];
    return GTC_OK;
}

gtc_status gtc_message(gtc_ctx* c, int rank, const uint32_t** dev_words, int64_t* k) {
    if (!c || !dev_words || !k) return GTC_EINVAL;
    if (!c->bound) return fail(c, GTC_ESTATE, "message: workspace not bound");
    if (rank < 0 || rank >= c->world) return fail(c, GTC_EINVAL, "message: rank");
    if (c->world == 1) {
        int64_t kk = 0;
        gtc_status s = gtc_last_counts(c, &kk);
        if (s != GTC_OK) return s;
        *dev_words = c->send;
        *k = kk;
        return GTC_OK;
    }
    *dev_words = c->recv + (size_t)rank * (size_t)c->max_k;
    *k = c->last_k[rank];
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

int64_t gtc_kernel_launches(const gtc_ctx* c) { return c ? c->launches : 0; }

void gtc_destroy(gtc_ctx* c) {
    if (!c) return;
    DeviceGuard g(c->device);
    if (c->comm) ncclCommDestroy(c->comm);
    if (c->host_kx) cudaFreeHost(c->host_kx);
    delete c;
}

}  // extern "C"
