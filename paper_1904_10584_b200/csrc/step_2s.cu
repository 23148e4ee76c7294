// step_2s.cu -- EXPERIMENT (GTC_STEP_2S=1): the world > 1 step as two
// concurrent kernels.  On the caller's stream a pure encode (rows a1-a5,
// stamped entries and tags as relaxed system-scope stores, no push, no
// apply); on the context's second stream, started with it, a small persistent
// decode kernel (one CTA of 4 warps per SM, in the registers the encode
// leaves free) whose warps follow the encode front and pull every rank's tags
// and entries of their tiles over NVLink with cp.async, count them and apply
// (rows a6-a8).  The caller's stream then waits for the decode.
#include "gtc_internal.cuh"
#include "tile_encode.cuh"

#include <algorithm>
#include <mutex>

namespace gtc {
namespace {

__device__ __forceinline__ unsigned long long ld_sys(const unsigned long long* a) {
    unsigned long long v;
    asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(a) : "memory");
    return v;
}
__device__ __forceinline__ unsigned ld_sys(const unsigned* a) {
    unsigned v;
    asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(a) : "memory");
    return v;
}
__device__ __forceinline__ unsigned long long now() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ unsigned smem_addr(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

// ---------------------------------------------------------------- encode
template <int CMP, bool HAS_G>
__global__ void __maxnreg__(56) gtc_step2s_encode_kernel(const EncodeParams p) {
    __shared__ unsigned s_scan[kTileVec * kTileWarps];
    __shared__ unsigned s_total, s_prev;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const long long tile = blockIdx.x, base = tile * kTile;
    const bool full_tile = base + kTile <= p.n;
    unsigned prev = 0u;
    if (tid == kTileThreads - 1) prev = ld_tag_count(p.tags + tile);
    float4 rv[kTileVec], gv[kTileVec];
    load_tile<HAS_G>(p, base, full_tile, tid, rv, gv);
    unsigned sel, neg;
    bool nonfinite;
    quantize<CMP, HAS_G>(rv, gv, p.tau, sel, neg, nonfinite);
    store_residual(p, base, full_tile, tid, rv);
    if (__any_sync(0xffffffffu, nonfinite) && lane == 0) atomicOr(&p.ctrl->flags, kFlagNonFinite);
    unsigned my_off[kTileVec];
    tile_scan_ballots(sel, lane, warp, my_off, s_scan);
    __syncthreads();
    if (warp == kTileWarps - 1) {
        const unsigned incl = tile_scan_finish(lane, s_scan);
        if (lane == 31) {
            s_total = incl;
            s_prev = prev;
            if (incl) atomicAdd(p.k_acc, (unsigned long long)incl);
            if (tile == 0) *p.k_next = 0ull;
        }
    }
    __syncthreads();
    store_words<true, true>(p.seg + base, base, tid, sel, neg, my_off, s_scan, warp, s_total, s_prev,
                            entry_stamp(p.epoch));
    if (tid == 0) st_relaxed_sys(p.tags + tile, make_tag(p.epoch, s_total));
}

// ---------------------------------------------------------------- decode
constexpr int kDw = 4;                 // decode warps per CTA
constexpr int kSpec = 8;               // entry slots per lane per tile
constexpr int kSlots = 32 * kSpec;
constexpr int kBatch = 4;
constexpr int kDecSmemPerWarp = 4 * (kTile / 4 + 2 * kSlots + 32);

template <int MODE>
__device__ __forceinline__ float apply_c(float t, int c, float tau, float alpha) {
    const float u = __fmul_rn((float)c, tau);
    return (MODE == GTC_ACCUM_WEIGHTS) ? __fmaf_rn(alpha, u, t) : __fadd_rn(t, u);
}

__device__ __forceinline__ void count_b(unsigned* cw, unsigned e) {
    const unsigned idx = (e >> 1) & (kTile - 1);
    const unsigned sh = 8u * (idx & 3u);
    atomicAdd(cw + (idx >> 2), (e & 1u) ? (0u - (1u << sh)) : (1u << sh));
}

// every rank's tag (lane m < N) and the first S = kSlots / NR entries of
// every rank, by 16-byte cp.async (peers: over NVLink)
template <int NR>
__device__ __forceinline__ unsigned long long load_msgs(const FusedStepParams& f, long long d, int lane, unsigned* buf) {
    constexpr int S = kSlots / NR;
    const int N = f.nranks;
    unsigned long long tag = 0ull;
    if (lane < N) tag = ld_sys(f.tags[lane] + d);
#pragma unroll
    for (int h = 0; h < kSlots / 4 / 32; ++h) {
        const int c = lane + 32 * h, m = (4 * c) / S;
        if (m < N)
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;"
                         :: "r"(smem_addr(buf + 4 * c)), "l"(f.seg[m] + d * kTile + (4 * c - m * S)) : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    return tag;
}

__device__ __forceinline__ bool front_passed(const FusedStepParams& f, long long q, long long T, int lane) {
    int ok = 1;
    if (lane == 0 && q < T) ok = (unsigned)(ld_sys(f.enc.tags + q) >> 32) == f.enc.epoch;
    return __shfl_sync(0xffffffffu, ok, 0) != 0;
}

template <int MODE, int NR>
__device__ __forceinline__ bool decode_tile(const FusedStepParams& f, long long d, int lane, unsigned long long tag,
                                            unsigned* buf, unsigned* cw, unsigned* bm, long long nxt, long long T,
                                            long long W, unsigned* nbuf, unsigned long long& ntag, bool& nloaded) {
    const EncodeParams& p = f.enc;
    constexpr int S = kSlots / NR;
    const int N = f.nranks;
    const unsigned stamp = entry_stamp(p.epoch);
    const bool nxt_live = nxt < T;
    const long long q = nxt + W;
    unsigned long long probe = 0ull;
    if (lane == 0 && nxt_live && q < T) probe = ld_sys(p.tags + q);
    bool ok = true;
    unsigned long long t0 = 0ull;
    for (;;) {
        const bool ready = lane >= N || (unsigned)(tag >> 32) == p.epoch;
        if (__all_sync(0xffffffffu, ready)) break;
        int give_up = 0;
        if (lane == 0) {
            const unsigned long long t = now();
            if (t0 == 0ull) t0 = t;
            give_up = (t - t0 > f.timeout_ns || (ld_sys(f.flags) & kFlagPeer)) ? 1 : 0;
        }
        if (__shfl_sync(0xffffffffu, give_up, 0)) {
            ok = false;
            break;
        }
        __nanosleep(256);
        if (!ready) tag = ld_sys(f.tags[lane] + d);
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncwarp();
    const int kl = lane < N ? (int)(unsigned)tag : 0;
    int kk[NR];
#pragma unroll
    for (int m = 0; m < NR; ++m) kk[m] = __shfl_sync(0xffffffffu, kl, m);
    unsigned claimed = 0u;
    bool dense = false;
    if (ok) {
        unsigned ev[kSpec], valid = 0u;
#pragma unroll
        for (int u = 0; u < kSpec; ++u) ev[u] = buf[lane + 32 * u];
#pragma unroll
        for (int u = 0; u < kSpec; ++u) {
            const int m = (32 * u) / S, j = 32 * u - m * S + lane;
            if (j < kk[m]) valid |= 1u << u;
        }
#pragma unroll
        for (int u = 0; u < kSpec; ++u) {
            if (((valid >> u) & 1u) && (ev[u] >> kStampShift) != stamp) {
                const int m = (32 * u) / S, j = 32 * u - m * S + lane;
                const unsigned long long ts = now();
                const unsigned* a = f.seg[m] + d * kTile + j;
                unsigned e;
                do {
                    __nanosleep(128);
                    e = ld_sys(a);
                    if (now() - ts > f.timeout_ns) {
                        ok = false;
                        break;
                    }
                } while ((e >> kStampShift) != stamp);
                ev[u] = e;
                buf[lane + 32 * u] = e;
                if ((e >> kStampShift) != stamp) valid &= ~(1u << u);
            }
        }
#pragma unroll
        for (int u = 0; u < kSpec; ++u)
            if ((valid >> u) & 1u) count_b(cw, ev[u]);
        unsigned old[kSpec];
#pragma unroll
        for (int u = 0; u < kSpec; ++u) {
            const unsigned wd = (ev[u] >> 3) & (kTile / 4 - 1);
            old[u] = ((valid >> u) & 1u) ? atomicOr(bm + (wd >> 5), 1u << (wd & 31u)) : ~0u;
        }
#pragma unroll
        for (int u = 0; u < kSpec; ++u)
            if (!((old[u] >> ((ev[u] >> 3) & 31u)) & 1u)) claimed |= 1u << u;
        const int ovl = lane < N ? max(0, kl - S) : 0;
        int ovx = ovl;
#pragma unroll
        for (int o = 1; o < kFusedMaxRanks; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, ovx, o);
            if (lane >= o) ovx += y;
        }
        const int OV = __shfl_sync(0xffffffffu, ovx, kFusedMaxRanks - 1);
        ovx -= ovl;
        dense = OV > 0;
        const unsigned long long t_ov = OV ? now() : 0ull;
        for (int c0 = 0; c0 < OV && __all_sync(0xffffffffu, ok); c0 += 32 * kBatch) {
            unsigned ov[kBatch];
            const unsigned* a[kBatch];
            unsigned have = 0u, pnd = 0u;
#pragma unroll
            for (int u = 0; u < kBatch; ++u) {
                const int fo = c0 + lane + 32 * u;
                a[u] = nullptr;
                int m = 0;
#pragma unroll
                for (int qq = 1; qq < kFusedMaxRanks; ++qq)
                    if (qq < N && __shfl_sync(0xffffffffu, ovx, qq) <= fo) m = qq;
                const int rem = fo - __shfl_sync(0xffffffffu, ovx, m);
                if (fo < OV) {
                    a[u] = f.seg[m] + d * kTile + S + rem;
                    ov[u] = ld_sys(a[u]);
                    have |= 1u << u;
                }
            }
#pragma unroll
            for (int u = 0; u < kBatch; ++u)
                if (((have >> u) & 1u) && (ov[u] >> kStampShift) != stamp) pnd |= 1u << u;
            while (pnd) {
                if (now() - t_ov > f.timeout_ns) {
                    pnd = 0u;
                    have = 0u;
                    ok = false;
                    break;
                }
                __nanosleep(128);
#pragma unroll
                for (int u = 0; u < kBatch; ++u) {
                    if (!((pnd >> u) & 1u)) continue;
                    ov[u] = ld_sys(a[u]);
                    if ((ov[u] >> kStampShift) == stamp) pnd &= ~(1u << u);
                }
            }
#pragma unroll
            for (int u = 0; u < kBatch; ++u)
                if ((have >> u) & 1u) count_b(cw, ov[u]);
        }
    }
    ok = __all_sync(0xffffffffu, ok);
    __syncwarp();
    auto load_next = [&]() {
        nloaded = false;
        if (!nxt_live) return;
        const int passed = q >= T || (unsigned)(probe >> 32) == p.epoch;
        if (__shfl_sync(0xffffffffu, passed, 0)) {
            ntag = load_msgs<NR>(f, nxt, lane, nbuf);
            nloaded = true;
        }
    };
    const long long db = d * kTile;
    auto apply_word = [&](int v, const float4& tv) {
        const unsigned c = cw[v];
        cw[v] = 0x80808080u;
        const long long e0 = db + 4ll * v;
        const int cc[4] = {(int)(c & 0xffu) - 128, (int)((c >> 8) & 0xffu) - 128, (int)((c >> 16) & 0xffu) - 128,
                           (int)(c >> 24) - 128};
        if (e0 + 4 <= p.n) {
            float4 t = tv;
            if (cc[0]) t.x = apply_c<MODE>(t.x, cc[0], p.tau, f.alpha);
            if (cc[1]) t.y = apply_c<MODE>(t.y, cc[1], p.tau, f.alpha);
            if (cc[2]) t.z = apply_c<MODE>(t.z, cc[2], p.tau, f.alpha);
            if (cc[3]) t.w = apply_c<MODE>(t.w, cc[3], p.tau, f.alpha);
            *reinterpret_cast<float4*>(f.target + e0) = t;
        } else {
            for (int e = 0; e < 4 && e0 + e < p.n; ++e)
                if (cc[e]) f.target[e0 + e] = apply_c<MODE>(f.target[e0 + e], cc[e], p.tau, f.alpha);
        }
    };
    bool first = true;
    if (__any_sync(0xffffffffu, dense || !ok)) {
        unsigned touched = 0u;
#pragma unroll 8
        for (int i = 0; i < kTile / 4 / 32; ++i)
            if (cw[lane + 32 * i] != 0x80808080u) touched |= 1u << i;
        if (!ok) {
            for (unsigned m = touched; m; m &= m - 1u) cw[lane + 32 * (__ffs(m) - 1)] = 0x80808080u;
            touched = 0u;
        }
        while (__any_sync(0xffffffffu, touched != 0u)) {
            int iv[kBatch];
            float4 tv[kBatch];
#pragma unroll
            for (int u = 0; u < kBatch; ++u) {
                iv[u] = -1;
                if (touched) {
                    iv[u] = lane + 32 * (__ffs(touched) - 1);
                    touched &= touched - 1u;
                    const long long e0 = db + 4ll * iv[u];
                    if (e0 + 4 <= p.n) tv[u] = *reinterpret_cast<const float4*>(f.target + e0);
                }
            }
            if (first) {
                load_next();
                first = false;
            }
#pragma unroll
            for (int u = 0; u < kBatch; ++u)
                if (iv[u] >= 0) apply_word(iv[u], tv[u]);
        }
    } else {
        while (__any_sync(0xffffffffu, claimed != 0u)) {
            int iv[kBatch];
            float4 tv[kBatch];
#pragma unroll
            for (int u = 0; u < kBatch; ++u) {
                iv[u] = -1;
                if (claimed) {
                    const int su = __ffs(claimed) - 1;
                    claimed &= claimed - 1u;
                    iv[u] = (int)((buf[lane + 32 * su] >> 3) & (kTile / 4 - 1));
                    const long long e0 = db + 4ll * iv[u];
                    if (e0 + 4 <= p.n) tv[u] = *reinterpret_cast<const float4*>(f.target + e0);
                }
            }
            if (first) {
                load_next();
                first = false;
            }
#pragma unroll
            for (int u = 0; u < kBatch; ++u)
                if (iv[u] >= 0) apply_word(iv[u], tv[u]);
        }
    }
    if (first) load_next();
    __syncwarp();
    bm[lane] = 0u;
    __syncwarp();
    return ok;
}

template <int MODE, int NR>
__global__ void __maxnreg__(64) gtc_step2s_decode_kernel(const FusedStepParams f) {
    extern __shared__ __align__(16) unsigned s_dyn[];
    const int lane = threadIdx.x & 31, dw = threadIdx.x >> 5;
    unsigned* cw = s_dyn + dw * (kDecSmemPerWarp / 4);
    unsigned* msg0 = cw + kTile / 4;
    unsigned* bm = msg0 + 2 * kSlots;
    bm[lane] = 0u;
#pragma unroll
    for (int i = 0; i < kTile / 4 / 4 / 32; ++i)
        reinterpret_cast<uint4*>(cw)[lane + 32 * i] = make_uint4(0x80808080u, 0x80808080u, 0x80808080u, 0x80808080u);
    __syncwarp();
    const long long T = f.enc.num_tiles, W = (long long)gridDim.x * kDw;
    long long cur = (long long)blockIdx.x * kDw + dw;
    unsigned long long tag = 0ull, ntag = 0ull;
    bool loaded = false;
    unsigned b = 0u;
    while (cur < T) {
        const long long nxt = cur + W;
        if (!loaded) {
            while (!front_passed(f, cur + W, T, lane)) __nanosleep(512);
            tag = load_msgs<NR>(f, cur, lane, msg0 + b * kSlots);
        }
        if (!decode_tile<MODE, NR>(f, cur, lane, tag, msg0 + b * kSlots, cw, bm, nxt, T, W, msg0 + (b ^ 1u) * kSlots,
                                   ntag, loaded) &&
            lane < f.nranks)
            atomicOr_system(f.peer_flags[lane], kFlagPeer);
        cur = nxt;
        if (loaded) {
            tag = ntag;
            b ^= 1u;
        }
    }
}

int sm_count() {
    static std::once_flag once;
    static int sms = 148;
    std::call_once(once, [] {
        int dev = 0, v = 0;
        if (cudaGetDevice(&dev) == cudaSuccess &&
            cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && v > 0)
            sms = v;
    });
    return sms;
}

template <typename K>
cudaError_t launch_dec(K kernel, const FusedStepParams& f, cudaStream_t s) {
    static std::mutex mu;
    static std::vector<const void*> done;
    {
        std::lock_guard<std::mutex> lock(mu);
        const void* k = reinterpret_cast<const void*>(kernel);
        if (std::find(done.begin(), done.end(), k) == done.end()) {
            cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kDw * kDecSmemPerWarp);
            done.push_back(k);
        }
    }
    kernel<<<sm_count(), 32 * kDw, kDw * kDecSmemPerWarp, s>>>(f);
    return cudaGetLastError();
}

template <int MODE>
cudaError_t launch_dec_nr(const FusedStepParams& f, cudaStream_t s) {
    const int N = f.nranks;
    if (N <= 2) return launch_dec(gtc_step2s_decode_kernel<MODE, 2>, f, s);
    if (N <= 4) return launch_dec(gtc_step2s_decode_kernel<MODE, 4>, f, s);
    return launch_dec(gtc_step2s_decode_kernel<MODE, 8>, f, s);
}

}  // namespace

cudaError_t launch_step_2s(const FusedStepParams& f, int cmp_mode, int accum_mode, cudaStream_t enc_stream,
                           cudaStream_t dec_stream, cudaEvent_t start, cudaEvent_t done) {
    const EncodeParams& p = f.enc;
    if (p.num_tiles == 0) return cudaSuccess;
    cudaError_t e = cudaEventRecord(start, enc_stream);
    if (e != cudaSuccess) return e;
    const unsigned grid = (unsigned)p.num_tiles;
    if (cmp_mode == GTC_CMP_GE) {
        if (p.g) gtc_step2s_encode_kernel<GTC_CMP_GE, true><<<grid, kTileThreads, 0, enc_stream>>>(p);
        else gtc_step2s_encode_kernel<GTC_CMP_GE, false><<<grid, kTileThreads, 0, enc_stream>>>(p);
    } else {
        if (p.g) gtc_step2s_encode_kernel<GTC_CMP_GT, true><<<grid, kTileThreads, 0, enc_stream>>>(p);
        else gtc_step2s_encode_kernel<GTC_CMP_GT, false><<<grid, kTileThreads, 0, enc_stream>>>(p);
    }
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    if ((e = cudaStreamWaitEvent(dec_stream, start, 0)) != cudaSuccess) return e;
    e = accum_mode == GTC_ACCUM_UPDATE ? launch_dec_nr<GTC_ACCUM_UPDATE>(f, dec_stream)
                                       : launch_dec_nr<GTC_ACCUM_WEIGHTS>(f, dec_stream);
    if (e != cudaSuccess) return e;
    if ((e = cudaEventRecord(done, dec_stream)) != cudaSuccess) return e;
    return cudaStreamWaitEvent(enc_stream, done, 0);
}

}  // namespace gtc
