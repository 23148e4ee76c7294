// encode.cu -- fused GTC encode for sm_100a (Sec. VI-A, steps 1-4).
//
// Per element i (fp32, RNE, no FTZ):
//     v = r[i] + g[i]                               residual accumulation
//     sel = |v| > tau   (GT)   /   |v| >= tau  (GE)  threshold (DESIGN R1)
//     r[i] = sel ? v -+ tau : v                      one +-tau quantum leaves (R2)
//     word = (i << 1) | (v < 0)                      32-bit packing (R3)
// and the selected words are compacted, in ascending index order (R4), into
// one contiguous message.  HBM-bound: no contraction, no tensor cores.
//
// gtc_encode_tile_kernel (default; the hot-path encode, and at world 1 with
//   gtc_step the whole step):
//   - one CTA per tile of kTile = 4096 params, 256 threads, 4 CTAs per SM;
//     every thread issues its four 128-bit loads of r and four of g before any
//     use (g: ld.global.nc.L1::no_allocate) and writes r back with 128-bit
//     stores; no state shared between CTAs;
//   - element order inside a tile is (round j, warp, lane, component) =
//     ascending index; intra-tile ranks come from three __ballot_sync/__popc
//     per round (a thread holds <= 4 words per round) and one 32-entry warp
//     scan over the (round, warp) totals;
//   - the tile's words go, compacted, to slot t of the segmented message; its
//     tag (epoch << 32 | count) to tags[t]; its count (integer atomicAdd) to
//     the step's word counter;
//   - world 1 (gtc_step): the rank's own quanta are the aggregate (c = +-1),
//     so the kernel also applies them to the target (loads issued right after
//     the threshold test to hide their latency);
//   - p2p: the slot holds stamped entries (tile_encode.cuh) that peers read
//     over NVLink once the rank's ready flag is up.
// (A persistent variant fed by 1-D TMA bulk copies and a one-tile variant
// loading through shared memory by TMA measured slower -- 59.7 and 58.4 us
// against 51.6 / 55.3 us, DESIGN.md Sec. 6 -- and were removed.)
// Packing (on demand: NCCL exchange, gtc_message): gtc_group_sums_kernel +
//   gtc_compact_kernel turn a segmented message (this rank's, or a peer's over
//   NVLink) into the contiguous wire format.
// Atomics: one integer atomicAdd per tile into the step's word counter (order-
// free), and atomicOr of the sticky non-finite flag.  No state is carried
// between calls except the epoch and the previous counts in the tags.
//
// HBM bytes per parameter (algorithmic): 4 (read g) + 4 (read r) + 4 (write r)
// + 4*rho (write words); + 8 B per tile (tag).
#include "gtc_internal.cuh"
#include "tile_encode.cuh"

#include <cstdlib>
#include <cstring>
#include <mutex>

namespace gtc {
namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kCompactThreads = 256;

// fused SGD-momentum apply (world 1, GTC_ACCUM_MOMENTUM; reading M1): for
// every element, u = fl(c * tau) with c in {-1, 0, +1}, buf = fl(fl(mu * buf) + u),
// w = fmaf(alpha, buf, w)
__device__ __forceinline__ void momentum_elem(float& w, float& b, int c, float tau, float alpha, float mu) {
    const float u = __fmul_rn((float)c, tau);
    b = __fadd_rn(__fmul_rn(mu, b), u);
    w = __fmaf_rn(alpha, b, w);
}

template <int CMP, bool HAS_G, bool MOM>
__global__ void __launch_bounds__(kTileThreads, 4) gtc_encode_tile_kernel(const EncodeParams p) {
    __shared__ unsigned s_scan[kTileVec * kTileWarps];
    __shared__ unsigned s_total, s_prev;

    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int warp = tid >> 5;
    const long long tile = blockIdx.x;
    const long long base = tile * kTile;
    const bool full_tile = base + kTile <= p.n;

    // Programmatic dependent launch: this grid may have been launched while
    // the previous kernel on the stream (e.g. the previous step) was still
    // draining; wait for it (and its memory) before touching any data, and let
    // the next launch begin as early as possible.
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;");

    // p2p: the count of this slot's previous (same-parity) step, whose entries
    // beyond the new count are cleared (tile_encode.cuh); loaded first so its
    // latency hides under the tile loads
    unsigned prev = 0u;
    if (p.publish_sys && tid == kTileThreads - 1) prev = ld_tag_count(p.tags + tile);
    float4 rv[kTileVec];
    float4 gv[kTileVec];
    load_tile<HAS_G>(p, base, full_tile, tid, rv, gv);

    const float tau = p.tau;
    unsigned sel, neg;
    bool nonfinite;
    quantize<CMP, HAS_G>(rv, gv, tau, sel, neg, nonfinite);

    // world 1 fused apply (gtc_step): this rank's own quanta are the whole
    // aggregate; load the selected targets now so the latency overlaps the
    // residual store, the scan and the word stores below.
    // (the first kEarly selected elements of the thread; at rho ~ 1 % a thread
    // holds ~0.16 of its 16, the rest, if any, are loaded late)
    constexpr int kEarly = 4;
    int eb[kEarly];
    float tv[kEarly];
    unsigned late = 0u;
    if (!MOM && p.target) {
        unsigned rem = sel;
#pragma unroll
        for (int q = 0; q < kEarly; ++q) {
            eb[q] = -1;
            if (rem) {
                const int b = __ffs(rem) - 1;
                rem &= rem - 1u;
                eb[q] = b;
                tv[q] = p.target[base + (long long)((b >> 2) * kTileThreads + tid) * 4 + (b & 3)];
            }
        }
        late = rem;
    }

    store_residual(p, base, full_tile, tid, rv);
    if (__any_sync(kFull, nonfinite) && lane == 0) atomicOr(&p.ctrl->flags, kFlagNonFinite);

    unsigned my_off[kTileVec];
    tile_scan_ballots(sel, lane, warp, my_off, s_scan);
    __syncthreads();
    if (warp == kTileWarps - 1) {
        const unsigned incl = tile_scan_finish(lane, s_scan);
        if (lane == 31) {
            s_total = incl;
            s_prev = prev;
            if (!p.publish_sys) p.tags[tile] = make_tag(p.epoch, incl);
            if (incl) atomicAdd(p.k_acc, (unsigned long long)incl);    // integer: order-free
            if (tile == 0) *p.k_next = 0ull;
        }
    }
    __syncthreads();
    const unsigned total = s_total;
    if (p.publish_sys)
        store_words<true>(p.seg + base, base, tid, sel, neg, my_off, s_scan, warp, total, s_prev,
                          entry_stamp(p.epoch));
    else
        store_words<false>(p.seg + base, base, tid, sel, neg, my_off, s_scan, warp, total, 0u, 0u);
    if (MOM) {
        // dense momentum apply over the whole tile: 16 B/param more
        if (full_tile) {
            float4* w4 = reinterpret_cast<float4*>(p.target + base);
            float4* b4 = reinterpret_cast<float4*>(p.buf + base);
            float4 wv[kTileVec], bv[kTileVec];
#pragma unroll
            for (int j = 0; j < kTileVec; ++j) {
                wv[j] = ld_v4(w4 + j * kTileThreads + tid);
                bv[j] = ld_v4(b4 + j * kTileThreads + tid);
            }
#pragma unroll
            for (int j = 0; j < kTileVec; ++j) {
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int b = j * 4 + e;
                    const int c = ((sel >> b) & 1u) ? (((neg >> b) & 1u) ? -1 : 1) : 0;
                    float wf = comp(wv[j], e), bf = comp(bv[j], e);
                    momentum_elem(wf, bf, c, tau, p.alpha, p.mu);
                    set_comp(wv[j], e, wf);
                    set_comp(bv[j], e, bf);
                }
                w4[j * kTileThreads + tid] = wv[j];
                b4[j * kTileThreads + tid] = bv[j];
            }
        } else {
#pragma unroll
            for (int j = 0; j < kTileVec; ++j) {
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const long long i = base + (long long)(j * kTileThreads + tid) * 4 + e;
                    if (i < p.n) {
                        const int b = j * 4 + e;
                        const int c = ((sel >> b) & 1u) ? (((neg >> b) & 1u) ? -1 : 1) : 0;
                        momentum_elem(p.target[i], p.buf[i], c, tau, p.alpha, p.mu);
                    }
                }
            }
        }
    } else if (p.target && sel) {
        // world 1 fused apply (loads issued early, see above): c = +-1 on the
        // selected elements, fl(+-1 * tau) = +-tau, target = fmaf(alpha, +-tau,
        // target) (R8) -- identical to decode_apply.
        auto apply = [&](int b, float t) {
            const float q = ((neg >> b) & 1u) ? -tau : tau;
            p.target[base + (long long)((b >> 2) * kTileThreads + tid) * 4 + (b & 3)] =
                (p.accum_mode == GTC_ACCUM_WEIGHTS) ? __fmaf_rn(p.alpha, q, t) : __fadd_rn(t, q);
        };
#pragma unroll
        for (int q = 0; q < kEarly; ++q)
            if (eb[q] >= 0) apply(eb[q], tv[q]);
        while (late) {
            const int b = __ffs(late) - 1;
            late &= late - 1u;
            apply(b, p.target[base + (long long)((b >> 2) * kTileThreads + tid) * 4 + (b & 3)]);
        }
    }
    if (p.publish_sys && tid == 0) p.tags[tile] = make_tag(p.epoch, total);  // p2p: after the scan's reads of the old tag
}

// Kernel 2 (packing, on demand): group sums of kGroupTiles tile counts, one
// warp per group.
constexpr int kCompactWarps = kCompactThreads / 32;
static_assert(kGroupTiles % kCompactWarps == 0, "a compact CTA never straddles a group");

__device__ __forceinline__ unsigned tag_count(const unsigned long long* tags, long long t) {
    return (unsigned)(__ldcg(tags + t) & 0xffffffffull);
}

__global__ void __launch_bounds__(kCompactThreads) gtc_group_sums_kernel(const CompactParams p) {
    const int lane = threadIdx.x & 31;
    const int g = blockIdx.x * kCompactWarps + (threadIdx.x >> 5);
    const int ng = (p.num_tiles + kGroupTiles - 1) / kGroupTiles;
    if (g >= ng) return;
    unsigned s = 0;
    for (int t = g * kGroupTiles + lane; t < min((g + 1) * kGroupTiles, p.num_tiles); t += 32)
        s += tag_count(p.tags, t);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(kFull, s, o);
    if (lane == 0) p.group_sum[g] = s;
}

// Kernel 3 (packing, on demand): one warp per tile, kCompactWarps tiles per
// CTA.  A CTA's global prefix = group sums of all earlier groups + counts of
// the earlier tiles of its group (all loads independent); each warp copies its
// tile's words (loads batched before stores).
__global__ void __launch_bounds__(kCompactThreads) gtc_compact_kernel(const CompactParams p) {
    __shared__ unsigned s_red[kCompactWarps];
    __shared__ unsigned s_cnt[kCompactWarps];

    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int warp = tid >> 5;
    const int t_cta = blockIdx.x * kCompactWarps;      // first tile of this CTA
    const int g = t_cta / kGroupTiles;                 // its group
    const int t_grp = g * kGroupTiles;                 // first tile of that group
    const int tile = t_cta + warp;
    const bool has_tile = tile < p.num_tiles;

    unsigned part = 0;
    for (int i = tid; i < g; i += kCompactThreads) part += __ldcg(p.group_sum + i);
    for (int i = t_grp + tid; i < t_cta; i += kCompactThreads) part += tag_count(p.tags, i);
    const unsigned my_cnt = has_tile ? tag_count(p.tags, tile) : 0u;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(kFull, part, o);
    if (lane == 0) {
        s_red[warp] = part;
        s_cnt[warp] = my_cnt;
    }
    __syncthreads();
    if (!has_tile) return;
    unsigned prefix = 0, before = 0;
#pragma unroll
    for (int w = 0; w < kCompactWarps; ++w) {
        prefix += s_red[w];
        before += (w < warp) ? s_cnt[w] : 0u;
    }
    const long long dst0 = (long long)prefix + before;

    if (lane == 0) {
        p.tile_off[tile] = (int)dst0;
        if (tile == p.num_tiles - 1) {
            const long long k = dst0 + my_cnt;
            p.tile_off[p.num_tiles] = (int)k;
            unsigned long long f = *reinterpret_cast<volatile unsigned long long*>(&p.ctrl->flags);
            if (k > p.capacity) {
                atomicOr(&p.ctrl->flags, kFlagCapacity);
                f |= kFlagCapacity;
            }
            p.hdr->k = k;
            p.hdr->flags = f;
        }
    }
    const unsigned* src = p.seg + (long long)tile * kTile;
    for (unsigned j0 = 0; j0 < my_cnt; j0 += 4 * 32) {
        unsigned w[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const unsigned j = j0 + u * 32 + lane;
            if (j < my_cnt) w[u] = __ldcg(src + j);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const unsigned j = j0 + u * 32 + lane;
            if (j < my_cnt && dst0 + j < p.capacity) p.words[dst0 + j] = p.stamped ? entry_word(w[u], tile) : w[u];
        }
    }
}

template <int CMP, bool HAS_G>
cudaError_t launch_tile(EncodeParams& p, cudaStream_t s) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)p.num_tiles);
    cfg.blockDim = dim3(kTileThreads);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (p.target && p.accum_mode == GTC_ACCUM_MOMENTUM)
        return cudaLaunchKernelEx(&cfg, gtc_encode_tile_kernel<CMP, HAS_G, true>, p);
    return cudaLaunchKernelEx(&cfg, gtc_encode_tile_kernel<CMP, HAS_G, false>, p);
}

template <int CMP>
cudaError_t launch_cmp(EncodeParams& p, cudaStream_t s) {
    return p.g ? launch_tile<CMP, true>(p, s) : launch_tile<CMP, false>(p, s);
}

}  // namespace

// Programmatic dependent launch of every hot-path kernel (GTC_PDL=0 disables).
bool pdl_enabled() {
    static int v = -1;
    if (v < 0) {
        const char* e = std::getenv("GTC_PDL");
        v = (e && e[0] == '0') ? 0 : 1;
    }
    return v == 1;
}

cudaError_t launch_encode(EncodeParams& p, int cmp_mode, cudaStream_t s) {
    if (p.num_tiles == 0) return cudaSuccess;
    return cmp_mode == GTC_CMP_GE ? launch_cmp<GTC_CMP_GE>(p, s) : launch_cmp<GTC_CMP_GT>(p, s);
}

// p2p loopback group (after gtc_encode) and the sharded decode (after the
// owner count): launched after the producing kernel on the same stream.  The
// kernel boundary orders every store of that kernel before this one; one
// system-scope fence then makes them visible to the peers and the release
// store raises the flag, which peers acquire before reading.  (Across
// processes the decode kernel's block 0 raises the ready flag at its start,
// saving this launch.)
__global__ void gtc_publish_kernel(unsigned long long* flag, unsigned long long step) {
    __threadfence_system();
    asm volatile("st.release.sys.global.u64 [%0], %1;" :: "l"(flag), "l"(step) : "memory");
}

cudaError_t launch_publish(unsigned long long* flag, unsigned long long step, cudaStream_t s) {
    gtc_publish_kernel<<<1, 1, 0, s>>>(flag, step);
    return cudaGetLastError();
}

cudaError_t launch_compact(const CompactParams& p, cudaStream_t s) {
    if (p.num_tiles == 0) return cudaSuccess;
    const int ng = (p.num_tiles + kGroupTiles - 1) / kGroupTiles;
    gtc_group_sums_kernel<<<(ng + kCompactWarps - 1) / kCompactWarps, kCompactThreads, 0, s>>>(p);
    gtc_compact_kernel<<<(p.num_tiles + kCompactWarps - 1) / kCompactWarps, kCompactThreads, 0, s>>>(p);
    return cudaGetLastError();
}

}  // namespace gtc
