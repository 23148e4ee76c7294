// bmuf.cu -- BMUF-NBM step for sm_100a (Sec. VI-B, Eqs. 1-5;
// C ABI in include/bmuf.h).
//
// world > 1:  ncclReduceScatter (in place, sum) of the local models -> one
// fused elementwise kernel over this rank's shard: Eqs. (1)-(4) and the
// write of the new Wg shard into the local model -> ncclAllGather (in place)
// of the shards.  HBM-bound; per element of the shard the kernel reads the
// summed model, Wg and Delta (12 B) and writes Wg, Delta and the local model
// (12 B).  The collectives move 2 (N-1)/N x 4 B per parameter over NVLink.
// Simulated workers (one GPU): one kernel reads every model in rank order
// (double accumulator, the oracle's reading B3), updates Wg and Delta and
// writes Wg back into every model.
//
// world > 1 with a bound workspace (p2p, the default of the Python binding):
// the local models live in CUDA-IPC-mapped workspaces and ONE kernel per step
// does the whole exchange over NVLink -- rank r reads its shard of every
// rank's model in rank order (the simulated workers' double mean, bit-exact
// with the oracle), updates its Wg / Delta shard and stores the new Wg shard
// straight into every rank's model.  Handshake (system-scope release /
// acquire on flags in the workspaces): block 0 raises this rank's ready(t)
// (its model is final); every CTA waits for all ready(t) before reading; the
// last CTA to finish (device-scope arrival counter) raises pushed[rank](t) in
// every peer's flags and waits until every peer has pushed into this rank's
// model.  NVLink bytes per rank are those of RS + AG; there is no NCCL call
// and no second pass over HBM.
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <new>
#include <vector>

#include "bmuf.h"
#include "gtc_internal.cuh"

#include <nvtx3/nvToolsExt.h>

namespace {

constexpr int kThreads = 256;
constexpr int kMaxSim = 64;

struct SimModels {
    float* w[kMaxSim];
};

// Eqs. (2)-(4) for one element, fixed fp32 operation order (bmuf.h)
__device__ __forceinline__ void bmuf_elem(float wbar, float& wg, float& d, float eta, float zeta) {
    const float g = __fsub_rn(wbar, wg);
    d = __fadd_rn(__fmul_rn(eta, d), __fmul_rn(zeta, g));
    wg = __fadd_rn(__fadd_rn(wg, d), __fmul_rn(eta, d));
}

// world > 1: sum (already reduced into the shard of w_local) -> new Wg shard
__global__ void __launch_bounds__(kThreads) bmuf_shard_kernel(float* __restrict__ wl_shard,
                                                              float* __restrict__ wg, float* __restrict__ delta,
                                                              long long len4, float n_f,
                                                              float eta, float zeta) {
    const long long stride = (long long)gridDim.x * kThreads;
    for (long long q = (long long)blockIdx.x * kThreads + threadIdx.x; q < len4; q += stride) {
        float4 s = reinterpret_cast<const float4*>(wl_shard)[q];
        float4 g = reinterpret_cast<const float4*>(wg)[q];
        float4 d = reinterpret_cast<const float4*>(delta)[q];
        // Eq. (1): Wbar = sum / N (IEEE division, correctly rounded)
        bmuf_elem(__fdiv_rn(s.x, n_f), g.x, d.x, eta, zeta);
        bmuf_elem(__fdiv_rn(s.y, n_f), g.y, d.y, eta, zeta);
        bmuf_elem(__fdiv_rn(s.z, n_f), g.z, d.z, eta, zeta);
        bmuf_elem(__fdiv_rn(s.w, n_f), g.w, d.w, eta, zeta);
        reinterpret_cast<float4*>(wg)[q] = g;
        reinterpret_cast<float4*>(delta)[q] = d;
        reinterpret_cast<float4*>(wl_shard)[q] = g;  // this rank's part of the broadcast model
    }
}

// simulated workers: rank-ordered double mean, full Wg / Delta, write back
__global__ void __launch_bounds__(kThreads) bmuf_sim_kernel(SimModels m, int nm, float* __restrict__ wg,
                                                            float* __restrict__ delta, long long n, float eta,
                                                            float zeta) {
    const long long stride = (long long)gridDim.x * kThreads;
    for (long long j = (long long)blockIdx.x * kThreads + threadIdx.x; j < n; j += stride) {
        double acc = 0.0;
        for (int i = 0; i < nm; ++i) acc = __dadd_rn(acc, (double)m.w[i][j]);
        const float wbar = __double2float_rn(__ddiv_rn(acc, (double)nm));
        float g = wg[j], d = delta[j];
        bmuf_elem(wbar, g, d, eta, zeta);
        wg[j] = g;
        delta[j] = d;
        for (int i = 0; i < nm; ++i) m.w[i][j] = g;
    }
}

// ---------------------------------------------------------------- p2p step
constexpr int kMaxRanks = 8;
constexpr unsigned long long kTimeoutNs = 30ull * 1000 * 1000 * 1000;

// Workspace: [flags 0..1023 | IPC records 1024..2047 | pad | model float[padded]]
struct Flags {
    unsigned long long ready;               // this rank's model is final for step t
    unsigned long long pad0[7];
    unsigned long long pushed[kMaxRanks];   // pushed[i]: rank i has stored its Wg shard here
    unsigned int done;                      // CTAs of this rank's kernel that finished
    int error;                              // 1: a peer timed out
};
constexpr size_t kIpcOff = 1024;
constexpr size_t kModelOff = 4096;
static_assert(sizeof(Flags) <= kIpcOff, "flags fit");
static_assert(kIpcOff + gtc::kIpcRecordBytes * kMaxRanks <= kModelOff, "IPC records fit");

struct P2PParams {
    float* model[kMaxRanks];              // every rank's model (own included), shard offset applied
    Flags* flags[kMaxRanks];              // every rank's flags
    float* wg;
    float* delta;
    long long len4;
    int rank, world;
    float eta, zeta;
    unsigned long long step;
};

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* a) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(a) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long* a, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(a), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ bool wait_at_least(const unsigned long long* a, unsigned long long step) {
    unsigned long long v = ld_acquire_sys(a);
    if (v >= step) return true;
    const unsigned long long t0 = globaltimer_ns();
    while (v < step) {
        if (globaltimer_ns() - t0 > kTimeoutNs) return false;
        __nanosleep(128);
        v = ld_acquire_sys(a);
    }
    return true;
}

// fl(sum / W): division by a power of two is the exact product with 1/W
template <int W>
__device__ __forceinline__ float mean_of(double sum) {
    if constexpr ((W & (W - 1)) == 0) return __double2float_rn(__dmul_rn(sum, 1.0 / W));
    else return __double2float_rn(__ddiv_rn(sum, (double)W));
}

template <int W>
__global__ void __launch_bounds__(kThreads, 3) bmuf_p2p_kernel(const P2PParams p) {
    __shared__ int s_abort;
    Flags* own = p.flags[p.rank];
    if (threadIdx.x == 0) {
        s_abort = 0;
        if (blockIdx.x == 0) {  // this rank's model (written by earlier kernels on the stream) is final
            __threadfence_system();
            st_release_sys(&own->ready, p.step);
        }
    }
    __syncthreads();
    // ready(t) of every rank; a peer is at most one step ahead (its next step
    // waits for this rank's pushes), hence >=
    if (threadIdx.x < p.world && !wait_at_least(&p.flags[threadIdx.x]->ready, p.step)) {
        s_abort = 1;
        atomicExch(&own->error, 1);
    }
    __syncthreads();
    if (!s_abort) {
        // U float4 per thread per iteration, all W * U loads issued up front
        // (the remote ones cross NVLink: latency-bound without enough in flight)
        constexpr int U = W <= 4 ? 2 : 1;
        const long long stride = (long long)gridDim.x * kThreads;
        for (long long q0 = (long long)blockIdx.x * kThreads + threadIdx.x; q0 < p.len4; q0 += stride * U) {
            float4 v[U][W];
#pragma unroll
            for (int u = 0; u < U; ++u)
#pragma unroll
                for (int i = 0; i < W; ++i)
                    if (q0 + u * stride < p.len4)
                        v[u][i] = __ldcg(reinterpret_cast<const float4*>(p.model[i]) + q0 + u * stride);
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const long long q = q0 + u * stride;
                if (q >= p.len4) break;
                // Eq. (1): rank-ordered double sum, divided by N, rounded once (B3)
                double ax = 0.0, ay = 0.0, az = 0.0, aw = 0.0;
#pragma unroll
                for (int i = 0; i < W; ++i) {
                    ax = __dadd_rn(ax, (double)v[u][i].x);
                    ay = __dadd_rn(ay, (double)v[u][i].y);
                    az = __dadd_rn(az, (double)v[u][i].z);
                    aw = __dadd_rn(aw, (double)v[u][i].w);
                }
                float4 g = reinterpret_cast<const float4*>(p.wg)[q];
                float4 d = reinterpret_cast<const float4*>(p.delta)[q];
                bmuf_elem(mean_of<W>(ax), g.x, d.x, p.eta, p.zeta);
                bmuf_elem(mean_of<W>(ay), g.y, d.y, p.eta, p.zeta);
                bmuf_elem(mean_of<W>(az), g.z, d.z, p.eta, p.zeta);
                bmuf_elem(mean_of<W>(aw), g.w, d.w, p.eta, p.zeta);
                reinterpret_cast<float4*>(p.wg)[q] = g;
                reinterpret_cast<float4*>(p.delta)[q] = d;
#pragma unroll
                for (int i = 0; i < W; ++i) __stcg(reinterpret_cast<float4*>(p.model[i]) + q, g);
            }
        }
    }
    // last CTA of this rank: publish the pushes, then wait for every peer's
    __syncthreads();
    __shared__ bool s_last;
    if (threadIdx.x == 0) {
        __threadfence_system();
        const unsigned prev = atomicAdd(&own->done, 1u);
        s_last = (prev == gridDim.x - 1);
        if (s_last) {
            own->done = 0;
            __threadfence_system();
        }
    }
    __syncthreads();
    if (!s_last) return;
    if (threadIdx.x < p.world) st_release_sys(&p.flags[threadIdx.x]->pushed[p.rank], p.step);
    __syncthreads();
    if (threadIdx.x < p.world && !wait_at_least(&own->pushed[threadIdx.x], p.step)) atomicExch(&own->error, 1);
}

int sm_count() {
    static int sms = 0;
    if (sms == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) sms = 148;
    }
    return sms;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

}  // namespace

struct bmuf_ctx {
    long long n = 0, shard = 0;
    int rank = 0, world = 1, device = 0;
    ncclComm_t comm = nullptr;
    // p2p (bmuf_bind_workspace)
    unsigned char* ws = nullptr;
    std::vector<unsigned char*> peer_ws;
    std::vector<void*> peer_alloc;
    unsigned long long steps = 0;
    int grid = 0;
    void (*kernel)(P2PParams) = nullptr;
};

namespace {
Flags* flags_of(unsigned char* ws) { return reinterpret_cast<Flags*>(ws); }
float* model_of(unsigned char* ws) { return reinterpret_cast<float*>(ws + kModelOff); }
size_t workspace_bytes(const bmuf_ctx* c) { return kModelOff + sizeof(float) * (size_t)c->shard * c->world; }

using P2PKernel = void (*)(P2PParams);
P2PKernel p2p_kernel(int world) {
    switch (world) {
        case 1: return bmuf_p2p_kernel<1>;
        case 2: return bmuf_p2p_kernel<2>;
        case 3: return bmuf_p2p_kernel<3>;
        case 4: return bmuf_p2p_kernel<4>;
        case 5: return bmuf_p2p_kernel<5>;
        case 6: return bmuf_p2p_kernel<6>;
        case 7: return bmuf_p2p_kernel<7>;
        default: return bmuf_p2p_kernel<8>;
    }
}

// one resident wave: every CTA spins on the ready flags at once
int p2p_grid(P2PKernel k) {
    int per = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k, kThreads, 0) != cudaSuccess || per < 1) per = 1;
    return per * sm_count();
}
}  // namespace

extern "C" {

gtc_status bmuf_init(bmuf_ctx** out, int64_t n, int rank, int world, const void* nccl_unique_id,
                     int cuda_device) {
    if (!out) return GTC_EINVAL;
    *out = nullptr;
    if (n < 0 || n >= (1LL << 40)) return GTC_EDIM;
    if (world < 1 || rank < 0 || rank >= world) return GTC_EINVAL;
    if ((world > 1) != (nccl_unique_id != nullptr)) return GTC_EINVAL;
    bmuf_ctx* c = new (std::nothrow) bmuf_ctx();
    if (!c) return GTC_EINVAL;
    c->n = n;
    c->rank = rank;
    c->world = world;
    c->device = cuda_device;
    const long long per = (n + world - 1) / world;
    c->shard = (per + 3) / 4 * 4;  // 16-byte aligned shards
    if (world > 1) {
        int prev = 0;
        cudaGetDevice(&prev);
        cudaSetDevice(cuda_device);
        ncclUniqueId id;
        std::memcpy(&id, nccl_unique_id, sizeof(id));
        const ncclResult_t r = ncclCommInitRank(&c->comm, world, id, rank);
        cudaSetDevice(prev);
        if (r != ncclSuccess) {
            delete c;
            return GTC_ENCCL;
        }
    }
    *out = c;
    return GTC_OK;
}

int64_t bmuf_shard_len(const bmuf_ctx* c) { return c ? c->shard : 0; }
int64_t bmuf_padded_len(const bmuf_ctx* c) { return c ? c->shard * c->world : 0; }

gtc_status bmuf_workspace_size(const bmuf_ctx* c, size_t* bytes) {
    if (!c || !bytes) return GTC_EINVAL;
    if (c->world > kMaxRanks) return GTC_EUNSUPPORTED;
    *bytes = workspace_bytes(c);
    return GTC_OK;
}

gtc_status bmuf_bind_workspace(bmuf_ctx* c, void* workspace, size_t bytes) {
    if (!c || !workspace) return GTC_EINVAL;
    if (c->ws) return GTC_ESTATE;
    if (c->world > kMaxRanks) return GTC_EUNSUPPORTED;
    if (bytes < workspace_bytes(c)) return GTC_ECAPACITY;
    if ((reinterpret_cast<uintptr_t>(workspace) & 255u) != 0) return GTC_EALIGN;
    int prev = 0;
    cudaGetDevice(&prev);
    if (prev != c->device) cudaSetDevice(c->device);
    unsigned char* ws = static_cast<unsigned char*>(workspace);
    gtc_status st = GTC_OK;
    if (cudaMemset(ws, 0, kModelOff) != cudaSuccess) st = GTC_ECUDA;
    if (st == GTC_OK && c->world > 1) {
        switch (gtc::ipc_map_peers(c->comm, c->rank, c->world, ws, workspace_bytes(c), ws + kIpcOff, c->peer_ws,
                                   c->peer_alloc)) {
            case gtc::IpcResult::kOk: break;
            case gtc::IpcResult::kCudaError: st = GTC_ECUDA; break;
            case gtc::IpcResult::kNcclError: st = GTC_ENCCL; break;
            default: st = GTC_EUNSUPPORTED;
        }
        // the IPC records overlapped nothing live; clear the flags again
        if (st == GTC_OK && cudaMemset(ws, 0, kModelOff) != cudaSuccess) st = GTC_ECUDA;
        // no rank may start a step before every rank has cleared its flags
        if (st == GTC_OK) {
            int* one = reinterpret_cast<int*>(ws + kIpcOff);
            if (ncclAllReduce(one, one, 1, ncclInt32, ncclSum, c->comm, 0) != ncclSuccess ||
                cudaStreamSynchronize(0) != cudaSuccess)
                st = GTC_ENCCL;
        }
    } else if (st == GTC_OK) {
        c->peer_ws.assign(1, ws);
        c->peer_alloc.assign(1, nullptr);
    }
    if (st == GTC_OK) {
        c->ws = ws;
        c->steps = 0;
        c->kernel = p2p_kernel(c->world);
        c->grid = p2p_grid(c->kernel);
    }
    if (prev != c->device) cudaSetDevice(prev);
    return st;
}

float* bmuf_model(const bmuf_ctx* c) { return (c && c->ws) ? model_of(c->ws) : nullptr; }

gtc_status bmuf_check(bmuf_ctx* c) {
    if (!c) return GTC_EINVAL;
    if (!c->ws) return GTC_OK;
    int err = 0;
    if (cudaMemcpy(&err, &flags_of(c->ws)->error, sizeof(int), cudaMemcpyDeviceToHost) != cudaSuccess)
        return GTC_ECUDA;
    return err ? GTC_EPEER : GTC_OK;
}

static gtc_status bmuf_sync_impl(bmuf_ctx* c, float* w_local, float* wg_shard, float* delta_shard, float eta,
                                 float zeta, cudaStream_t stream) {
    if (!c) return GTC_EINVAL;
    if (c->shard > 0 && (!w_local || !wg_shard || !delta_shard)) return GTC_EINVAL;
    if (!aligned16(w_local) || !aligned16(wg_shard) || !aligned16(delta_shard)) return GTC_EALIGN;
    if (!std::isfinite(eta) || !std::isfinite(zeta)) return GTC_EINVAL;
    if (c->ws && w_local != model_of(c->ws)) return GTC_EINVAL;  // p2p: the model lives in the workspace
    if (c->shard == 0) return GTC_OK;
    int prev = 0;
    cudaGetDevice(&prev);
    if (prev != c->device) cudaSetDevice(c->device);
    if (c->ws) {
        P2PParams p{};
        const size_t off = (size_t)c->rank * (size_t)c->shard;
        for (int i = 0; i < c->world; ++i) {
            p.model[i] = model_of(c->peer_ws[i]) + off;
            p.flags[i] = flags_of(c->peer_ws[i]);
        }
        p.wg = wg_shard;
        p.delta = delta_shard;
        p.len4 = c->shard / 4;
        p.rank = c->rank;
        p.world = c->world;
        p.eta = eta;
        p.zeta = zeta;
        p.step = ++c->steps;
        c->kernel<<<c->grid, kThreads, 0, stream>>>(p);
        const cudaError_t e = cudaGetLastError();
        if (prev != c->device) cudaSetDevice(prev);
        return e == cudaSuccess ? GTC_OK : GTC_ECUDA;
    }
    float* mine = w_local + (size_t)c->rank * (size_t)c->shard;
    gtc_status st = GTC_OK;
    if (c->world > 1 &&
        ncclReduceScatter(w_local, mine, (size_t)c->shard, ncclFloat32, ncclSum, c->comm, stream) != ncclSuccess)
        st = GTC_ENCCL;
    if (st == GTC_OK) {
        const long long len4 = c->shard / 4;
        const int grid = (int)std::min<long long>((len4 + kThreads - 1) / kThreads, (long long)sm_count() * 8);
        bmuf_shard_kernel<<<grid, kThreads, 0, stream>>>(mine, wg_shard, delta_shard, len4, (float)c->world,
                                                         eta, zeta);
        if (cudaGetLastError() != cudaSuccess) st = GTC_ECUDA;
    }
    if (st == GTC_OK && c->world > 1 &&
        ncclAllGather(mine, w_local, (size_t)c->shard, ncclFloat32, c->comm, stream) != ncclSuccess)
        st = GTC_ENCCL;
    if (prev != c->device) cudaSetDevice(prev);
    return st;
}

gtc_status bmuf_sync(bmuf_ctx* c, float* w_local, float* wg_shard, float* delta_shard, float eta, float zeta,
                     cudaStream_t stream) {
    nvtxRangePushA("bmuf_sync");  // phase tracing (gtc.cu)
    const gtc_status st = bmuf_sync_impl(c, w_local, wg_shard, delta_shard, eta, zeta, stream);
    nvtxRangePop();
    return st;
}

gtc_status bmuf_sync_sim(bmuf_ctx* c, float* const* w_locals, int nmodels, float* wg, float* delta, float eta,
                         float zeta, cudaStream_t stream) {
    if (!c || !w_locals || nmodels < 1 || nmodels > kMaxSim) return GTC_EINVAL;
    if (c->world != 1) return GTC_ESTATE;
    if (c->n > 0 && (!wg || !delta)) return GTC_EINVAL;
    if (c->n == 0) return GTC_OK;
    SimModels m{};
    for (int i = 0; i < nmodels; ++i) {
        if (!w_locals[i]) return GTC_EINVAL;
        m.w[i] = w_locals[i];
    }
    int prev = 0;
    cudaGetDevice(&prev);
    if (prev != c->device) cudaSetDevice(c->device);
    const int grid = (int)std::min<long long>((c->n + kThreads - 1) / kThreads, (long long)sm_count() * 8);
    bmuf_sim_kernel<<<grid, kThreads, 0, stream>>>(m, nmodels, wg, delta, c->n, eta, zeta);
    const cudaError_t e = cudaGetLastError();
    if (prev != c->device) cudaSetDevice(prev);
    return e == cudaSuccess ? GTC_OK : GTC_ECUDA;
}

double bmuf_zeta(double C, int N, double eta) { return C * (double)N * (1.0 - eta); }

gtc_status bmuf_quiesce(bmuf_ctx* c) {
    if (!c) return GTC_EINVAL;
    if (!(c->comm && c->ws && c->world > 1)) return GTC_OK;
    int prev = 0;
    cudaGetDevice(&prev);
    if (prev != c->device) cudaSetDevice(c->device);
    gtc_status s = GTC_OK;
    if (cudaDeviceSynchronize() != cudaSuccess) s = GTC_ECUDA;
    int* one = reinterpret_cast<int*>(c->ws + kIpcOff);
    if (s == GTC_OK && ncclAllReduce(one, one, 1, ncclInt32, ncclSum, c->comm, 0) != ncclSuccess) s = GTC_ENCCL;
    if (s == GTC_OK && cudaStreamSynchronize(0) != cudaSuccess) s = GTC_ECUDA;
    if (prev != c->device) cudaSetDevice(prev);
    return s;
}

void bmuf_destroy(bmuf_ctx* c) {
    if (!c) return;
    if (c->ws && c->world > 1) gtc::ipc_unmap(c->peer_alloc);
    if (c->comm) ncclCommDestroy(c->comm);
    delete c;
}

}  // extern "C"
