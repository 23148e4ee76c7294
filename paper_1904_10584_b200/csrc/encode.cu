// encode.cu -- fused GTC encode for sm_100a (Sec. VI-A, steps 1-4).
//
// One pass over the parameter vector, HBM-bound (no contraction, no tensor
// cores).  Per element i (fp32, RNE, no FTZ):
//     v = r[i] + g[i]                               residual accumulation
//     sel = |v| > tau   (GT)   /   |v| >= tau  (GE)  threshold
//     r[i] = sel ? v -+ tau : v                      one +-tau quantum leaves
//     word = (i << 1) | (v < 0)                      32-bit packing
// and the selected words are compacted, in ascending index order, into the
// message with a single-pass decoupled look-back scan:
//   - a CTA takes a dynamic ticket (= tile id, so every predecessor tile is
//     already resident: look-back cannot deadlock),
//   - 128-bit streaming loads of g and r (8 outstanding per thread),
//   - per-(round, warp) word counts from three __ballot_sync/__popc (a thread
//     holds <= 4 words per round), one 32-entry warp scan for the tile,
//   - warp 0 publishes the tile aggregate, sums predecessors' descriptors 32 at
//     a time until it meets an inclusive prefix, publishes its own prefix,
//   - the words are staged in shared memory and written out coalesced.
// Descriptors carry a per-call epoch, so no memset is needed between calls;
// the ticket counter of the next call is reset by tile 0 of this one.
//
// HBM bytes per parameter (algorithmic): 4 (read g) + 4 (read r) + 4 (write r)
// + 4*rho (write words) + 4/kTile (tile offset).
#include "gtc_internal.cuh"

namespace gtc {
namespace {

constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ float4 ld_stream_nc(const float4* p) {
    float4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
    return v;
}

__device__ __forceinline__ float4 ld_stream(const float4* p) {
    float4 v;
    asm volatile("ld.global.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
    return v;
}

__device__ __forceinline__ void st_stream(float4* p, const float4& v) {
    asm volatile("st.global.L1::no_allocate.v4.f32 [%0], {%1,%2,%3,%4};"
                 :: "l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
}

__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_relaxed_u64(unsigned long long* p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" :: "l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

__device__ __forceinline__ unsigned long long make_desc(unsigned epoch, unsigned status, unsigned value) {
    return ((unsigned long long)((epoch << 2) | status) << 32) | value;
}

__device__ __forceinline__ float comp(const float4& v, int e) {
    return e == 0 ? v.x : e == 1 ? v.y : e == 2 ? v.z : v.w;
}
__device__ __forceinline__ void set_comp(float4& v, int e, float x) {
    if (e == 0) v.x = x; else if (e == 1) v.y = x; else if (e == 2) v.z = x; else v.w = x;
}

__device__ __forceinline__ unsigned warp_sum(unsigned x) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(kFull, x, o);
    return x;
}

// Warp 0: publish this tile's aggregate, look back for the exclusive prefix,
// publish the inclusive prefix.  Returns the exclusive prefix (all lanes).
__device__ __forceinline__ unsigned look_back(const EncodeParams& p, unsigned ep, unsigned tile,
                                              unsigned total, int lane) {
    if (tile == 0) {
        if (lane == 0) st_relaxed_u64(&p.desc[0], make_desc(ep, kDescPrefix, total));
        return 0u;
    }
    if (lane == 0) st_relaxed_u64(&p.desc[tile], make_desc(ep, kDescAggregate, total));
    const unsigned tag_agg = (ep << 2) | kDescAggregate;
    const unsigned tag_pre = (ep << 2) | kDescPrefix;
    unsigned excl = 0;
    long long pred = (long long)tile - 1;
    while (true) {
        const long long t = pred - lane;  // lane 0 = nearest predecessor
        unsigned long long d = 0;
        bool ok = false;
        while (true) {
            if (!ok) {
                d = (t >= 0) ? ld_relaxed_u64(&p.desc[t]) : make_desc(ep, kDescPrefix, 0u);
                const unsigned tag = (unsigned)(d >> 32);
                ok = (tag == tag_agg) || (tag == tag_pre);
            }
            if (__all_sync(kFull, ok)) break;
        }
        const bool is_pre = ((unsigned)(d >> 32)) == tag_pre;
        const unsigned pm = __ballot_sync(kFull, is_pre);
        unsigned val = (unsigned)d;
        if (pm) {
            const int first = __ffs(pm) - 1;
            excl += warp_sum(lane <= first ? val : 0u);
            break;
        }
        excl += warp_sum(val);
        pred -= 32;
    }
    if (lane == 0) st_relaxed_u64(&p.desc[tile], make_desc(ep, kDescPrefix, excl + total));
    return excl;
}

template <int CMP, bool HAS_G>
__global__ void __launch_bounds__(kEncThreads, 4) gtc_encode_kernel(const EncodeParams p) {
    __shared__ unsigned s_words[kTile];          // staged message words of this tile
    __shared__ unsigned s_scan[kEncVec * kEncWarps];
    __shared__ unsigned s_tile, s_epoch, s_excl, s_total;

    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int warp = tid >> 5;

    if (tid == 0) {
        // The ticket address depends on the epoch just read, so the ticket is
        // taken after the read; the last tile advances the epoch only after
        // every other tile has published (hence read it): one launch sees one epoch.
        const unsigned ep = *reinterpret_cast<volatile unsigned*>(&p.ctrl->epoch);
        const unsigned t = atomicAdd(&p.ctrl->ticket[ep & 1u], 1u);
        if (t == 0) p.ctrl->ticket[(ep + 1u) & 1u] = 0u;
        s_tile = t;
        s_epoch = ep;
    }
    __syncthreads();
    const unsigned tile = s_tile;
    const long long base = (long long)tile * kTile;
    const bool full = base + kTile <= p.n;

    // ---- load: r (and g) for kEncVec rounds, all loads issued before use
    float4 rv[kEncVec];
    float4 gv[kEncVec];
    if (full) {
        const float4* r4 = reinterpret_cast<const float4*>(p.r + base);
#pragma unroll
        for (int j = 0; j < kEncVec; ++j) rv[j] = ld_stream(r4 + j * kEncThreads + tid);
        if (HAS_G) {
            const float4* g4 = reinterpret_cast<const float4*>(p.g + base);
#pragma unroll
            for (int j = 0; j < kEncVec; ++j) gv[j] = ld_stream_nc(g4 + j * kEncThreads + tid);
        }
    } else {
#pragma unroll
        for (int j = 0; j < kEncVec; ++j) {
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const long long i = base + (long long)(j * kEncThreads + tid) * 4 + e;
                set_comp(rv[j], e, i < p.n ? p.r[i] : 0.0f);
                if (HAS_G) set_comp(gv[j], e, i < p.n ? p.g[i] : 0.0f);
            }
        }
    }

    // ---- residual accumulate, threshold, quantize (R1, R2)
    const float tau = p.tau;
    unsigned sel = 0u, neg = 0u;
    bool nonfinite = false;
#pragma unroll
    for (int j = 0; j < kEncVec; ++j) {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const float v = HAS_G ? __fadd_rn(comp(rv[j], e), comp(gv[j], e)) : comp(rv[j], e);
            const float a = fabsf(v);
            nonfinite |= !(a <= 3.402823466e38f);  // NaN or Inf
            const bool s = (CMP == GTC_CMP_GT) ? (a > tau) : (a >= tau);
            const bool ng = v < 0.0f;
            const float rn = s ? (ng ? __fadd_rn(v, tau) : __fsub_rn(v, tau)) : v;
            set_comp(rv[j], e, rn);
            sel |= (unsigned)s << (j * 4 + e);
            neg |= (unsigned)(s && ng) << (j * 4 + e);
        }
    }

    // ---- write the residual back
    if (full) {
        float4* r4 = reinterpret_cast<float4*>(p.r + base);
#pragma unroll
        for (int j = 0; j < kEncVec; ++j) st_stream(r4 + j * kEncThreads + tid, rv[j]);
    } else {
#pragma unroll
        for (int j = 0; j < kEncVec; ++j) {
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const long long i = base + (long long)(j * kEncThreads + tid) * 4 + e;
                if (i < p.n) p.r[i] = comp(rv[j], e);
            }
        }
    }
    if (__any_sync(kFull, nonfinite) && lane == 0) atomicOr(&p.ctrl->flags, kFlagNonFinite);

    // ---- intra-tile ranks: element order is (round j, warp, lane, e)
    const unsigned lt = lanemask_lt();
    unsigned my_off[kEncVec];
#pragma unroll
    for (int j = 0; j < kEncVec; ++j) {
        const unsigned c = __popc((sel >> (4 * j)) & 0xfu);  // 0..4
        const unsigned b0 = __ballot_sync(kFull, c & 1u);
        const unsigned b1 = __ballot_sync(kFull, c & 2u);
        const unsigned b2 = __ballot_sync(kFull, c & 4u);
        my_off[j] = __popc(b0 & lt) + 2u * __popc(b1 & lt) + 4u * __popc(b2 & lt);
        if (lane == 0) s_scan[j * kEncWarps + warp] = __popc(b0) + 2u * __popc(b1) + 4u * __popc(b2);
    }
    __syncthreads();

    if (warp == 0) {
        const unsigned x = s_scan[lane];
        unsigned incl = x;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned y = __shfl_up_sync(kFull, incl, o);
            if (lane >= o) incl += y;
        }
        s_scan[lane] = incl - x;
        const unsigned total = __shfl_sync(kFull, incl, 31);
        const unsigned excl = look_back(p, s_epoch, tile, total, lane);
        if (lane == 0) {
            s_excl = excl;
            s_total = total;
            p.tile_off[tile] = (int)excl;
            if ((int)tile == p.num_tiles - 1) {
                p.ctrl->epoch = s_epoch >= kEpochMax ? 1u : s_epoch + 1u;
                const unsigned k = excl + total;
                p.tile_off[p.num_tiles] = (int)k;
                p.ctrl->k = (long long)k;
                if ((long long)k > p.capacity) atomicOr(&p.ctrl->flags, kFlagCapacity);
            }
        }
    }
    __syncthreads();

    // ---- pack (R3) into shared memory at each word's rank within the tile
#pragma unroll
    for (int j = 0; j < kEncVec; ++j) {
        unsigned o = s_scan[j * kEncWarps + warp] + my_off[j];
        const unsigned i0 = (unsigned)(base + (long long)(j * kEncThreads + tid) * 4);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            if ((sel >> (4 * j + e)) & 1u) {
                s_words[o] = ((i0 + e) << 1) | ((neg >> (4 * j + e)) & 1u);
                ++o;
            }
        }
    }
    __syncthreads();

    // ---- coalesced copy of the tile's words to its slice of the message
    const unsigned total = s_total;
    const long long excl = s_excl;
    for (unsigned i = tid; i < total; i += kEncThreads) {
        const long long pos = excl + i;
        if (pos < p.capacity) p.words[pos] = s_words[i];
    }
}

template <int CMP>
cudaError_t launch_cmp(const EncodeParams& p, cudaStream_t s) {
    if (p.num_tiles == 0) return cudaSuccess;
    if (p.g)
        gtc_encode_kernel<CMP, true><<<p.num_tiles, kEncThreads, 0, s>>>(p);
    else
        gtc_encode_kernel<CMP, false><<<p.num_tiles, kEncThreads, 0, s>>>(p);
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_encode(const EncodeParams& p, int cmp_mode, cudaStream_t s) {
    return cmp_mode == GTC_CMP_GE ? launch_cmp<GTC_CMP_GE>(p, s) : launch_cmp<GTC_CMP_GT>(p, s);
}

}  // namespace gtc
