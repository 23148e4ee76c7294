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
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <new>

#include "bmuf.h"

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
};

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

gtc_status bmuf_sync(bmuf_ctx* c, float* w_local, float* wg_shard, float* delta_shard, float eta, float zeta,
                     cudaStream_t stream) {
    if (!c) return GTC_EINVAL;
    if (c->shard > 0 && (!w_local || !wg_shard || !delta_shard)) return GTC_EINVAL;
    if (!aligned16(w_local) || !aligned16(wg_shard) || !aligned16(delta_shard)) return GTC_EALIGN;
    if (!std::isfinite(eta) || !std::isfinite(zeta)) return GTC_EINVAL;
    if (c->shard == 0) return GTC_OK;
    int prev = 0;
    cudaGetDevice(&prev);
    if (prev != c->device) cudaSetDevice(c->device);
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

void bmuf_destroy(bmuf_ctx* c) {
    if (!c) return;
    if (c->comm) ncclCommDestroy(c->comm);
    delete c;
}

}  // extern "C"
