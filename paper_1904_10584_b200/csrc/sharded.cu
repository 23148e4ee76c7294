// sharded.cu -- owner-computes decode for world > 1, p2p (GTC_DECODE_SHARDED;
// SURVEY.md 8(e) "Alternative", 8(f) #4): the aggregate of PAPER.md:222 ("The
// received sparse gradient updates are aggregated and weights are updated
// based on the aggregate") computed ONCE per parameter range by its owner
// instead of by every rank.
//
// Rank m owns tiles [tile_begin(m), tile_begin(m + 1)), tile_begin(m) =
// ceil(m T / N) (gtc_internal.cuh).
//   gtc_owner_count_kernel (gtc_exchange): every rank's stamped entries of the
//     owner's tiles are read in place (peer memory over NVLink: (N-1)/N of a
//     message per peer instead of all of it), counted into int8 shared-memory
//     counts in ordered per-rank passes (indices unique within one rank's tile:
//     no atomics, deterministic), and written as one COUNT LIST per tile:
//     entries (local << 8) | (count & 0xff) in ascending local index, tag
//     (epoch << 32) | length.  A one-thread publish kernel then raises the
//     rank's `counted` flag (system-scope release).
//   gtc_apply_counts_kernel (gtc_decode_apply): waits for every owner's
//     `counted` flag, reads each tile's count list from its owner and applies
//     u = fl(c * tau); WEIGHTS t = fmaf(alpha, u, t) / UPDATE t = fl(t + u)
//     (R8) to the touched elements, or the dense SGD-momentum update (M1).
// Bytes per rank per step: peer reads (N-1) rho n / N words + the list
// entries of the other owners' tiles, (N-1)/N rho_U n entries, against
// (N-1) rho n words for the replicated decode: fewer when many ranks' updates
// overlap (rho_U << N rho, high density / many ranks), more otherwise.
#include "gtc_internal.cuh"
#include "tile_encode.cuh"

#include <algorithm>

namespace gtc {
namespace {

constexpr int kThreads = 256;
constexpr int kBatch = 4;  // independent loads per thread before their use
static_assert(kTile == kThreads * 16, "16 counts per thread");

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* a) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(a) : "memory");
    return v;
}

__device__ __forceinline__ unsigned long long now_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Every CTA: wait until every rank's flag (ready or counted) reaches this
// step; on timeout raise kFlagPeer on every rank and return false.
__device__ bool wait_all(const ShardParams& p, const unsigned long long* const* flag, int* s_abort) {
    if (threadIdx.x == 0) *s_abort = 0;
    __syncthreads();
    if (threadIdx.x < (unsigned)p.nranks) {
        const unsigned long long* f = flag[threadIdx.x];
        unsigned long long v = ld_acquire_sys(f);
        const unsigned long long t0 = now_ns();
        while (v < p.step) {
            if (now_ns() - t0 > p.timeout_ns) {
                *s_abort = 1;
                break;
            }
            __nanosleep(64);
            v = ld_acquire_sys(f);
        }
    }
    __syncthreads();
    if (*s_abort) {
        if (threadIdx.x < (unsigned)p.nranks) atomicOr_system(p.peer_flags[threadIdx.x], kFlagPeer);
        return false;
    }
    return true;
}

__device__ __forceinline__ void publish_at_start(const ShardParams& p) {
    if (p.publish && blockIdx.x == 0 && threadIdx.x == 0) {
        // stream order puts every store of the previous kernel before this one
        __threadfence_system();
        asm volatile("st.release.sys.global.u64 [%0], %1;" :: "l"(p.publish), "l"(p.step) : "memory");
    }
}

// Block-wide exclusive scan of one value per thread; returns the total.
__device__ __forceinline__ unsigned block_scan(unsigned v, unsigned& excl, unsigned* s_warp) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    unsigned base = 0, total = 0;
#pragma unroll
    for (int w = 0; w < kThreads / 32; ++w) {
        const unsigned x = s_warp[w];
        base += (w < warp) ? x : 0u;
        total += x;
    }
    excl = base + incl - v;
    __syncthreads();  // s_warp is reused by the next scan
    return total;
}

__global__ void __launch_bounds__(kThreads) gtc_owner_count_kernel(const ShardParams p) {
    __shared__ int4 s_cnt4[kTile / 16];
    __shared__ int s_k[kFusedMaxRanks];
    __shared__ unsigned s_warp[kThreads / 32];
    __shared__ int s_abort;
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;");
    publish_at_start(p);
    if (!wait_all(p, p.ready, &s_abort)) return;
    signed char* s_cnt = reinterpret_cast<signed char*>(s_cnt4);
    const int tid = threadIdx.x;
    const long long tb = shard_tile_begin(p.rank, p.nranks, p.num_tiles);
    const long long te = shard_tile_begin(p.rank + 1, p.nranks, p.num_tiles);
    for (long long t = tb + blockIdx.x; t < te; t += gridDim.x) {
        s_cnt4[tid] = make_int4(0, 0, 0, 0);
        if (tid < p.nranks) s_k[tid] = (int)(__ldcg(p.tags[tid] + t) & 0xffffffffull);
        __syncthreads();
        // ordered per-rank passes (no two threads of a pass touch one count)
        for (int m = 0; m < p.nranks; ++m) {
            const unsigned* src = p.seg[m] + t * kTile;
            const int k = s_k[m];
            for (int j0 = tid; j0 < k; j0 += kBatch * kThreads) {
                unsigned e[kBatch];
#pragma unroll
                for (int u = 0; u < kBatch; ++u) {
                    const int j = j0 + u * kThreads;
                    e[u] = j < k ? __ldcg(src + j) : 0u;
                }
#pragma unroll
                for (int u = 0; u < kBatch; ++u) {
                    if (j0 + u * kThreads < k) {
                        signed char& c = s_cnt[(e[u] >> 1) & (kTile - 1)];
                        c = (signed char)(c + ((e[u] & 1u) ? -1 : 1));
                    }
                }
            }
            __syncthreads();
        }
        // the tile's count list: thread tid holds counts [16 tid, 16 tid + 16)
        const int4 q = s_cnt4[tid];
        const unsigned x[4] = {(unsigned)q.x, (unsigned)q.y, (unsigned)q.z, (unsigned)q.w};
        unsigned msk = 0;
#pragma unroll
        for (int h = 0; h < 4; ++h)
#pragma unroll
            for (int b = 0; b < 4; ++b) msk |= (((x[h] >> (8 * b)) & 0xffu) != 0u ? 1u : 0u) << (4 * h + b);
        unsigned pos;
        const unsigned total = block_scan(__popc(msk), pos, s_warp);
        unsigned* dst = p.clist + t * kTile;
        while (msk) {
            const int b = __ffs(msk) - 1;
            msk &= msk - 1u;
            const unsigned c = (x[b >> 2] >> (8 * (b & 3))) & 0xffu;
            dst[pos++] = ((unsigned)(16 * tid + b) << 8) | c;
        }
        if (tid == 0) p.ctags[t] = make_tag(p.epoch, total);
        __syncthreads();  // s_cnt4 / s_k reused by the next tile
    }
}

template <int MODE>
__device__ __forceinline__ float apply_count(float t, int c, float tau, float alpha) {
    const float u = __fmul_rn((float)c, tau);
    return (MODE == GTC_ACCUM_WEIGHTS) ? __fmaf_rn(alpha, u, t) : __fadd_rn(t, u);
}

template <int MODE>
__global__ void __launch_bounds__(kThreads) gtc_apply_counts_kernel(const ShardParams p) {
    __shared__ int4 s_cnt4[kTile / 16];
    __shared__ int s_abort;
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;");
    publish_at_start(p);
    if (!wait_all(p, p.counted, &s_abort)) return;
    signed char* s_cnt = reinterpret_cast<signed char*>(s_cnt4);
    const int tid = threadIdx.x;
    const bool dense = MODE == GTC_ACCUM_MOMENTUM || p.counts_out != nullptr;
    for (long long t = blockIdx.x; t < p.num_tiles; t += gridDim.x) {
        const int o = shard_owner(t, p.nranks, p.num_tiles);
        const int len = (int)(__ldcg(p.ctags_of[o] + t) & 0xffffffffull);
        const unsigned* src = p.clist_of[o] + t * kTile;
        const long long base = t * kTile;
        if (!dense) {
            // sparse read-modify-write of the listed elements (distinct)
            for (int j0 = tid; j0 < len; j0 += kBatch * kThreads) {
                unsigned e[kBatch];
                float v[kBatch];
#pragma unroll
                for (int u = 0; u < kBatch; ++u) {
                    const int j = j0 + u * kThreads;
                    e[u] = j < len ? __ldcg(src + j) : 0u;
                }
#pragma unroll
                for (int u = 0; u < kBatch; ++u)
                    if (j0 + u * kThreads < len) v[u] = p.target[base + (e[u] >> 8)];
#pragma unroll
                for (int u = 0; u < kBatch; ++u)
                    if (j0 + u * kThreads < len)
                        p.target[base + (e[u] >> 8)] =
                            apply_count<MODE>(v[u], (int)(signed char)(e[u] & 0xffu), p.tau, p.alpha);
            }
            continue;
        }
        // dense: scatter the list into int8 counts, then sweep the tile
        s_cnt4[tid] = make_int4(0, 0, 0, 0);
        __syncthreads();
        for (int j = tid; j < len; j += kThreads) {
            const unsigned e = __ldcg(src + j);
            s_cnt[e >> 8] = (signed char)(e & 0xffu);
        }
        __syncthreads();
        const int4 q = s_cnt4[tid];
        if (p.counts_out) {
            if (base + 16 * (tid + 1) <= p.n) {
                reinterpret_cast<int4*>(p.counts_out + base)[tid] = q;
            } else {
                for (int e = 0; e < 16 && base + 16 * tid + e < p.n; ++e) p.counts_out[base + 16 * tid + e] = s_cnt[16 * tid + e];
            }
        }
        const long long e0 = base + 16ll * tid;
        if constexpr (MODE == GTC_ACCUM_MOMENTUM) {
            // M1 over every element: buf = fl(fl(mu * buf) + fl(c * tau)), w = fmaf(alpha, buf, w)
            for (int e = 0; e < 16 && e0 + e < p.n; ++e) {
                const float u = __fmul_rn((float)(int)s_cnt[16 * tid + e], p.tau);
                const float b = __fadd_rn(__fmul_rn(p.mu, p.buf[e0 + e]), u);
                p.buf[e0 + e] = b;
                p.target[e0 + e] = __fmaf_rn(p.alpha, b, p.target[e0 + e]);
            }
        } else {
            for (int e = 0; e < 16 && e0 + e < p.n; ++e) {
                const int c = s_cnt[16 * tid + e];
                if (c) p.target[e0 + e] = apply_count<MODE>(p.target[e0 + e], c, p.tau, p.alpha);
            }
        }
        __syncthreads();  // s_cnt4 reused by the next tile
    }
}

int sms() {
    static int v = 0;
    if (v == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) v = 148;
    }
    return v;
}

template <typename K>
cudaError_t launch_pdl(K kern, int grid, const ShardParams& p, cudaStream_t s) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)std::max(grid, 1));
    cfg.blockDim = dim3(kThreads);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, p);
}

}  // namespace

// One wave at most: every CTA spins on the flags at its start, so all of them
// must be resident (8 CTAs of 256 threads per SM fit).
cudaError_t launch_owner_count(const ShardParams& p, cudaStream_t s) {
    if (p.num_tiles == 0) return cudaSuccess;
    const long long range = shard_tile_begin(p.rank + 1, p.nranks, p.num_tiles) -
                            shard_tile_begin(p.rank, p.nranks, p.num_tiles);
    const int grid = (int)std::min<long long>(std::max(range, 1LL), (long long)sms() * 8);
    return launch_pdl(gtc_owner_count_kernel, grid, p, s);
}

cudaError_t launch_apply_counts(const ShardParams& p, int accum_mode, cudaStream_t s) {
    if (p.num_tiles == 0) return cudaSuccess;
    const int grid = (int)std::min<long long>(p.num_tiles, (long long)sms() * 8);
    if (accum_mode == GTC_ACCUM_MOMENTUM) return launch_pdl(gtc_apply_counts_kernel<GTC_ACCUM_MOMENTUM>, grid, p, s);
    if (accum_mode == GTC_ACCUM_UPDATE) return launch_pdl(gtc_apply_counts_kernel<GTC_ACCUM_UPDATE>, grid, p, s);
    return launch_pdl(gtc_apply_counts_kernel<GTC_ACCUM_WEIGHTS>, grid, p, s);
}

}  // namespace gtc
