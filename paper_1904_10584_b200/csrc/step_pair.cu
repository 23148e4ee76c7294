// step_pair.cu -- EXPERIMENT (GTC_STEP_PAIR=1): the world > 1 step as two
// kernels chained by programmatic dependent launch on the caller's stream:
//   A: one CTA per tile encodes it (rows a1-a5) and pushes its record to
//      every peer by bulk copy (round 1's encode CTA: no ticket, no decode);
//   B: groups of kDecGroup tiles per CTA decode and apply every rank's
//      records (round 1's decode CTA), launched when A's last CTAs started,
//      so it overlaps A's tail; it waits for A's grid only at its end, so the
//      next step's A (which waits for B) starts after both.
// B only waits on tiles A encodes, and A never waits: no deadlock in any
// dispatch order.
#include "gtc_internal.cuh"
#include "tile_encode.cuh"

#include <algorithm>

namespace gtc {
namespace {

constexpr int kDecGroup = 8;
constexpr int kSpecPerThread = 4;
constexpr int kApplyBatch = 4;

__device__ __forceinline__ unsigned long long ld_relaxed_sys(const unsigned long long* a) {
    unsigned long long v;
    asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(a) : "memory");
    return v;
}
__device__ __forceinline__ unsigned ld_relaxed_sys(const unsigned* a) {
    unsigned v;
    asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(a) : "memory");
    return v;
}
__device__ __forceinline__ unsigned long long now_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
template <int MODE>
__device__ __forceinline__ float apply_count(float t, int c, float tau, float alpha) {
    const float u = __fmul_rn((float)c, tau);
    return (MODE == GTC_ACCUM_WEIGHTS) ? __fmaf_rn(alpha, u, t) : __fadd_rn(t, u);
}
__device__ __forceinline__ void count_entry(signed char* cnt, unsigned e) {
    signed char& c = cnt[(e >> 1) & (kTile - 1)];
    c = (signed char)(c + ((e & 1u) ? -1 : 1));
}
__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

template <int CMP, bool HAS_G>
__device__ __forceinline__ void encode_cta(const FusedStepParams& f, long long t, unsigned* s_scan, unsigned* s_misc,
                                           unsigned long long* s_rec) {
    const EncodeParams& p = f.enc;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const long long base = t * kTile;
    const bool full_tile = base + kTile <= p.n;
    // this slot's previous same-parity count (its entries beyond the new count
    // are cleared), loaded first so its latency hides under the tile loads
    unsigned prev_ld = 0u;
    if (tid == kTileThreads - 1) prev_ld = ld_tag_count(p.tags + t);
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
            s_misc[0] = incl;
            s_misc[1] = prev_ld;
            if (incl) atomicAdd(p.k_acc, (unsigned long long)incl);
            if (t == 0) *p.k_next = 0ull;
        }
    }
    __syncthreads();
    const unsigned total = s_misc[0], prev = s_misc[1];
    const unsigned stamp = entry_stamp(p.epoch);
    unsigned* dst = p.seg + base;
    unsigned* s_ent = reinterpret_cast<unsigned*>(s_rec + 2);
    if (total != 0) {
#pragma unroll
        for (int j = 0; j < kTileVec; ++j) {
            unsigned o = s_scan[j * kTileWarps + warp] + my_off[j];
            const unsigned l0 = (unsigned)(j * kTileThreads + tid) * 4u;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                if ((sel >> (4 * j + e)) & 1u) {
                    const unsigned w = make_entry(stamp, l0 + e, (neg >> (4 * j + e)) & 1u);
                    st_relaxed_sys(dst + o, w);
                    if (o < (unsigned)kPushCap) s_ent[o] = w;
                    ++o;
                }
            }
        }
    }
    for (unsigned o = total + tid; o < prev; o += kTileThreads) st_relaxed_sys(dst + o, 0u);
    const unsigned clr = min(max(total, prev), (unsigned)kPushCap);
    const unsigned clr4 = (clr + 3u) & ~3u;  // bulk copies move multiples of 16 bytes
    for (unsigned o = total + tid; o < clr4; o += kTileThreads) s_ent[o] = 0u;
    const unsigned long long tag = make_tag(p.epoch, total);
    if (tid == 0) {
        st_relaxed_sys(p.tags + t, tag);
        s_rec[0] = tag;
        s_rec[1] = 0ull;
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // smem writes -> the bulk copies
    __syncthreads();
    if (tid == 0) {
        const unsigned bytes = 16u + 4u * clr4;
#pragma unroll
        for (int m = 0; m < kFusedMaxRanks; ++m) {
            if (m >= f.nranks || !f.push_out[m]) continue;
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                         :: "l"(f.push_out[m] + t * kPushRec), "r"(smem_u32(s_rec)), "r"(bytes) : "memory");
        }
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    }
}

// ------------------------------------------------------------ decode CTA
// A peer missed the timeout: GTC_EPEER on EVERY rank (system-scope atomics on
// each rank's flags), so no replica carries on unaware; this CTA applies nothing.

__device__ __forceinline__ void raise_peer_error(const FusedStepParams& f) {
    if (threadIdx.x < (unsigned)f.nranks) atomicOr_system(f.peer_flags[threadIdx.x], kFlagPeer);
}

// Tiles [t0, t0 + ng) of every rank.  A peer timeout sets kFlagPeer.
template <int MODE, typename Stamp>
__device__ __forceinline__ void decode_cta(const FusedStepParams& f, long long t0, int ng, signed char* s_cnt,
                                           int* s_k, int* s_abort, const Stamp& stamp_ph) {
    const EncodeParams& p = f.enc;
    const int tid = threadIdx.x;
    const int N = f.nranks;
    const int SP = kSpecPerThread * kTileThreads / (kDecGroup * N);  // speculative entries per (tile, rank)

    // all loads in flight at once: tags, then the speculative entries
    // (flat index (i, m, j), j fastest: coalesced per (tile, rank) slot)
    // rank m's tag and entry j of tile t: peers from this rank's push region
    // (entries beyond kPushCap from the owner's buffer, over NVLink), this
    // rank from its own segmented buffer
    auto tag_ptr = [&](int m, long long t) -> const unsigned long long* {
        return f.push_in[m] ? reinterpret_cast<const unsigned long long*>(f.push_in[m] + t * kPushRec) : f.tags[m] + t;
    };
    auto entry_ptr = [&](int m, long long t, int j) -> const unsigned* {
        if (f.push_in[m] && j < kPushCap) return reinterpret_cast<const unsigned*>(f.push_in[m] + t * kPushRec + 16) + j;
        return f.seg[m] + t * kTile + j;
    };
    unsigned long long tagv = 0;
    const int ti = tid / N, tm = tid - ti * N;
    if (ti < ng) tagv = ld_relaxed_sys(tag_ptr(tm, t0 + ti));
    // speculative entry u of this thread: (tile i, rank m, entry j) of flat
    // index tid + u * kTileThreads, j fastest
    auto spec_at = [&](int u, int& i, int& m, int& j) {
        const int fl = tid + u * kTileThreads;
        i = fl / (N * SP);
        m = (fl / SP) % N;
        j = fl % SP;
    };
    unsigned spec[kSpecPerThread];
#pragma unroll
    for (int u = 0; u < kSpecPerThread; ++u) {
        int i, m, j;
        spec_at(u, i, m, j);
        spec[u] = 0u;
        if (i < ng) spec[u] = ld_relaxed_sys(entry_ptr(m, t0 + i, j));
    }
    int4* c4 = reinterpret_cast<int4*>(s_cnt);
    for (int q = tid; q < kDecGroup * kTile / 16; q += kTileThreads) c4[q] = make_int4(0, 0, 0, 0);
    if (tid == 0) *s_abort = 0;
    __syncthreads();
    if (ti < ng) {
        if ((unsigned)(tagv >> 32) != p.epoch) {
            const unsigned long long t0ns = now_ns();
            do {
                if (now_ns() - t0ns > f.timeout_ns) {
                    *s_abort = 1;
                    break;
                }
                __nanosleep(32);
                tagv = ld_relaxed_sys(tag_ptr(tm, t0 + ti));
            } while ((unsigned)(tagv >> 32) != p.epoch);
        }
        s_k[ti * kFusedMaxRanks + tm] = (int)(tagv & 0xffffffffull);
    }
    __syncthreads();
    stamp_ph(1);
    if (*s_abort) {
        raise_peer_error(f);
        return;
    }

    // Entries beyond the speculative blocks ("overflow", dense tiles):
    // exclusive prefix of their counts over the (tile, rank) pairs
    __shared__ int s_ovo[kDecGroup * kFusedMaxRanks + 1];
    if (tid < 32) {
        int v[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int pr = 2 * tid + h;
            v[h] = pr < ng * N ? max(0, s_k[(pr / N) * kFusedMaxRanks + pr % N] - SP) : 0;
        }
        int incl = v[0] + v[1];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, o);
            if (tid >= o) incl += y;
        }
        s_ovo[2 * tid] = incl - v[0] - v[1];
        s_ovo[2 * tid + 1] = incl - v[1];
        if (tid == 31) s_ovo[2 * 32] = incl;
    }
    __syncthreads();
    const int OV = s_ovo[kDecGroup * kFusedMaxRanks];
    const unsigned stamp = entry_stamp(p.epoch);
    const unsigned long long t_start = now_ns();
    bool ok = true;
    // re-poll the stale entries of a batch together until all carry this
    // step's stamp (the tag can land before the entries of its record)
    auto settle = [&](unsigned* e, const unsigned** a, unsigned pend) {
        while (pend && ok) {
            __nanosleep(64);
#pragma unroll
            for (int u = 0; u < kSpecPerThread; ++u)
                if ((pend >> u) & 1u) e[u] = ld_relaxed_sys(a[u]);
#pragma unroll
            for (int u = 0; u < kSpecPerThread; ++u)
                if (((pend >> u) & 1u) && (e[u] >> kStampShift) == stamp) pend &= ~(1u << u);
            if (pend && now_ns() - t_start > f.timeout_ns) ok = false;
        }
    };
    {
        const unsigned* a[kSpecPerThread];
        unsigned pend = 0u;
#pragma unroll
        for (int u = 0; u < kSpecPerThread; ++u) {
            int i, m, j;
            spec_at(u, i, m, j);
            a[u] = entry_ptr(m, t0 + i, j);
            if (i < ng && j < s_k[i * kFusedMaxRanks + m] && (spec[u] >> kStampShift) != stamp) pend |= 1u << u;
        }
        settle(spec, a, pend);
    }
    constexpr int kOvChunk = kSpecPerThread * kTileThreads;
    for (int c0 = 0;; c0 += kOvChunk) {
        unsigned ov[kSpecPerThread];
        int opr[kSpecPerThread];
        const unsigned* a[kSpecPerThread];
        unsigned pend = 0u;
#pragma unroll
        for (int u = 0; u < kSpecPerThread; ++u) {
            const int fo = c0 + tid + u * kTileThreads;
            opr[u] = -1;
            a[u] = nullptr;
            if (fo < OV) {
                int lo = 0, hi = kDecGroup * kFusedMaxRanks;  // s_ovo[lo] <= fo < s_ovo[hi]
                while (hi - lo > 1) {
                    const int mid = (lo + hi) >> 1;
                    if (s_ovo[mid] <= fo) lo = mid; else hi = mid;
                }
                opr[u] = lo;
                a[u] = entry_ptr(lo % N, t0 + lo / N, SP + fo - s_ovo[lo]);
                ov[u] = ld_relaxed_sys(a[u]);
            }
        }
#pragma unroll
        for (int u = 0; u < kSpecPerThread; ++u)
            if (opr[u] >= 0 && (ov[u] >> kStampShift) != stamp) pend |= 1u << u;
        settle(ov, a, pend);
        if (!ok) *s_abort = 1;
        // ordered per-rank passes over the batch (plus, first, the speculative entries)
        for (int m = 0; m < N; ++m) {
            if (c0 == 0) {
#pragma unroll
                for (int u = 0; u < kSpecPerThread; ++u) {
                    int i, mm, j;
                    spec_at(u, i, mm, j);
                    if (ok && mm == m && i < ng && j < s_k[i * kFusedMaxRanks + m]) count_entry(s_cnt + i * kTile, spec[u]);
                }
            }
#pragma unroll
            for (int u = 0; u < kSpecPerThread; ++u)
                if (ok && opr[u] >= 0 && opr[u] % N == m) count_entry(s_cnt + (opr[u] / N) * kTile, ov[u]);
            __syncthreads();  // the next rank's pass may touch the same counts
        }
        if (c0 + kOvChunk >= OV) break;
    }
    stamp_ph(2);
    if (*s_abort) {
        raise_peer_error(f);
        return;
    }

    if constexpr (MODE == GTC_ACCUM_MOMENTUM) {
        // SGD-momentum (M1) over EVERY element of the tiles (an untouched
        // weight still moves by its decaying momentum): u = fl(c * tau),
        // buf = fl(fl(mu * buf) + u), w = fmaf(alpha, buf, w); float4 v of a
        // tile is element 4v, thread tid takes v = tid + 256 h (coalesced),
        // the tile's 4 float4 of w and of buf in flight together
        for (int i = 0; i < ng; ++i) {
            const long long tb = (t0 + i) * kTile;
            float4 wv[kTileVec], bv[kTileVec];
#pragma unroll
            for (int h = 0; h < kTileVec; ++h) {
                const long long e0 = tb + 4ll * (tid + h * kTileThreads);
                if (e0 + 4 <= p.n) {
                    wv[h] = ld_v4(reinterpret_cast<const float4*>(f.target + e0));
                    bv[h] = ld_v4(reinterpret_cast<const float4*>(p.buf + e0));
                }
            }
#pragma unroll
            for (int h = 0; h < kTileVec; ++h) {
                const int v = tid + h * kTileThreads;
                const long long e0 = tb + 4ll * v;
                const int packed = reinterpret_cast<const int*>(s_cnt + i * kTile)[v];
                auto mom = [&](float& w, float& bf, int e) {
                    const float u = __fmul_rn((float)(int)(signed char)((unsigned)packed >> (8 * e)), p.tau);
                    bf = __fadd_rn(__fmul_rn(p.mu, bf), u);
                    w = __fmaf_rn(f.alpha, bf, w);
                };
                if (e0 + 4 <= p.n) {
                    mom(wv[h].x, bv[h].x, 0);
                    mom(wv[h].y, bv[h].y, 1);
                    mom(wv[h].z, bv[h].z, 2);
                    mom(wv[h].w, bv[h].w, 3);
                    st_stream(reinterpret_cast<float4*>(f.target + e0), wv[h]);
                    st_stream(reinterpret_cast<float4*>(p.buf + e0), bv[h]);
                } else {
                    for (int e = 0; e < 4 && e0 + e < p.n; ++e) mom(f.target[e0 + e], p.buf[e0 + e], e);
                }
            }
        }
        return;
    }

    // apply: thread tid owns elements [16 tid, 16 tid + 16) of each tile, as
    // four float4 (bit i * 4 + h of `todo`: float4 h of tile i is touched)
    unsigned todo = 0u;
    for (int i = 0; i < ng; ++i) {
        const int4 c = c4[i * (kTile / 16) + tid];
        const unsigned x[4] = {(unsigned)c.x, (unsigned)c.y, (unsigned)c.z, (unsigned)c.w};
#pragma unroll
        for (int h = 0; h < 4; ++h) todo |= (x[h] != 0u ? 1u : 0u) << (i * 4 + h);
    }
    while (todo) {
        int bit[kApplyBatch];
        float4 tv[kApplyBatch];
#pragma unroll
        for (int u = 0; u < kApplyBatch; ++u) {
            bit[u] = -1;
            if (todo) {
                bit[u] = __ffs(todo) - 1;
                todo &= todo - 1u;
                const long long i0 = (t0 + (bit[u] >> 2)) * kTile + 16 * tid + 4 * (bit[u] & 3);
                if (i0 + 4 <= p.n) tv[u] = *reinterpret_cast<const float4*>(f.target + i0);
            }
        }
#pragma unroll
        for (int u = 0; u < kApplyBatch; ++u) {
            if (bit[u] < 0) continue;
            const int i = bit[u] >> 2, h = bit[u] & 3;
            const long long i0 = (t0 + i) * kTile + 16 * tid + 4 * h;
            const int packed = reinterpret_cast<const int*>(s_cnt + i * kTile)[4 * tid + h];
            const int cc[4] = {(int)(signed char)(packed & 0xff), (int)(signed char)((packed >> 8) & 0xff),
                               (int)(signed char)((packed >> 16) & 0xff), (int)(signed char)((unsigned)packed >> 24)};
            if (i0 + 4 <= p.n) {
                float4 t = tv[u];
                if (cc[0]) t.x = apply_count<MODE>(t.x, cc[0], p.tau, f.alpha);
                if (cc[1]) t.y = apply_count<MODE>(t.y, cc[1], p.tau, f.alpha);
                if (cc[2]) t.z = apply_count<MODE>(t.z, cc[2], p.tau, f.alpha);
                if (cc[3]) t.w = apply_count<MODE>(t.w, cc[3], p.tau, f.alpha);
                *reinterpret_cast<float4*>(f.target + i0) = t;
            } else {
                for (int e = 0; e < 4 && i0 + e < p.n; ++e)
                    if (cc[e]) f.target[i0 + e] = apply_count<MODE>(f.target[i0 + e], cc[e], p.tau, f.alpha);
            }
        }
    }
}

template <int CMP, bool HAS_G>
__global__ void __launch_bounds__(kTileThreads, 4) gtc_pair_encode_kernel(const FusedStepParams f) {
    __shared__ unsigned s_scan[kTileVec * kTileWarps];
    __shared__ unsigned s_misc[2];
    __shared__ __align__(128) unsigned long long s_rec[kPushRec / 8];
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;");
    encode_cta<CMP, HAS_G>(f, blockIdx.x, s_scan, s_misc, s_rec);
}

template <int MODE>
__global__ void __launch_bounds__(kTileThreads, 4) gtc_pair_decode_kernel(const FusedStepParams f) {
    __shared__ int4 s_cnt4[kDecGroup * kTile / 16];
    __shared__ int s_k[kDecGroup * kFusedMaxRanks];
    __shared__ int s_abort;
    asm volatile("griddepcontrol.launch_dependents;");
    const long long t0 = (long long)blockIdx.x * kDecGroup;
    const int ng = (int)min((long long)kDecGroup, (long long)f.enc.num_tiles - t0);
    auto no_stamp = [](int) {};
    decode_cta<MODE>(f, t0, ng, reinterpret_cast<signed char*>(s_cnt4), s_k, &s_abort, no_stamp);
    // complete only after the encode grid (the next step's encode waits on this one)
    asm volatile("griddepcontrol.wait;" ::: "memory");
}

}  // namespace

cudaError_t launch_step_pair(const FusedStepParams& f, int cmp_mode, int accum_mode, cudaStream_t s) {
    const long long T = f.enc.num_tiles;
    if (T == 0) return cudaSuccess;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cudaLaunchConfig_t cfg = {};
    cfg.blockDim = dim3(kTileThreads);
    cfg.stream = s;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cfg.gridDim = dim3((unsigned)T);
    cudaError_t e;
    if (cmp_mode == GTC_CMP_GE)
        e = f.enc.g ? cudaLaunchKernelEx(&cfg, gtc_pair_encode_kernel<GTC_CMP_GE, true>, f)
                    : cudaLaunchKernelEx(&cfg, gtc_pair_encode_kernel<GTC_CMP_GE, false>, f);
    else
        e = f.enc.g ? cudaLaunchKernelEx(&cfg, gtc_pair_encode_kernel<GTC_CMP_GT, true>, f)
                    : cudaLaunchKernelEx(&cfg, gtc_pair_encode_kernel<GTC_CMP_GT, false>, f);
    if (e != cudaSuccess) return e;
    cfg.gridDim = dim3((unsigned)((T + kDecGroup - 1) / kDecGroup));
    if (accum_mode == GTC_ACCUM_MOMENTUM) return cudaLaunchKernelEx(&cfg, gtc_pair_decode_kernel<GTC_ACCUM_MOMENTUM>, f);
    if (accum_mode == GTC_ACCUM_UPDATE) return cudaLaunchKernelEx(&cfg, gtc_pair_decode_kernel<GTC_ACCUM_UPDATE>, f);
    return cudaLaunchKernelEx(&cfg, gtc_pair_decode_kernel<GTC_ACCUM_WEIGHTS>, f);
}

}  // namespace gtc
