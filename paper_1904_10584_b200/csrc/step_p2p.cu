// step_p2p.cu -- the whole GTC step for world > 1 (p2p exchange) as ONE kernel:
// encode (PAPER.md:222 steps 1-4), exchange ("Each worker communicates the
// sparse update to all other workers and conversely receives all sparse
// updates"), aggregate and apply ("The received sparse gradient updates are
// aggregated and weights are updated based on the aggregate").
//
// Grid: groups of kDecGroup ENCODE CTAs followed by one DECODE CTA, plus a
// tail of decode CTAs; kTileThreads threads, 4 CTAs per SM.
//   encode CTA (tile t): rows a1-a5 exactly as gtc_encode_tile_kernel, writing
//     stamped tile-local entries (tile_encode.cuh) and the tile's tag
//     (epoch << 32 | count) as relaxed system-scope stores -- no fence, no
//     flag -- and PUSHING the tile's record (tag + first kPushCap entries) to
//     every peer with one bulk (TMA) copy each, fire-and-forget;
//   decode CTA (group q - lag_groups): rows a6-a8 for kDecGroup tiles of EVERY
//     rank (itself included).  All its loads go out at once, all local: every
//     (tile, rank) tag and a speculative first block of every (tile, rank)
//     record's entries (peers: the records they pushed here; entries beyond
//     kPushCap are pulled over NVLink).  An entry counts only once its stamp
//     is this step's (a stale one is re-polled), so no writer-side fence is
//     needed.  Counts are int8 in
//     shared memory, accumulated in ordered per-rank passes (indices are unique
//     within one rank's tile: no two threads of a pass touch one count, no
//     atomics, deterministic).  Then u = fl(c * tau), WEIGHTS
//     t = fmaf(alpha, u, t) / UPDATE t = fl(t + u) on the touched elements
//     (R8), 128-bit read-modify-write of the float4s holding a non-zero count;
//     GTC_ACCUM_MOMENTUM: the dense SGD-momentum update (M1) of the tiles.
// Why this shape: a CTA slot is held for its whole lifetime, and the encode is
// bound by the HBM bytes its resident CTAs keep in flight.  Any NVLink round
// trip a CTA waits for (~3-9 us while the peer's HBM is saturated by its own
// encode) stretches its lifetime.  Measured alternatives: the
// decode of tile t - lag inside the CTA encoding tile t, pulling (-35 %) or
// pushing with plain remote stores (-45 %); decode CTAs pulling from the
// peers (-40 %).  Bulk copies return the slot as soon as shared memory is
// read, and the decode CTAs then only wait on local memory.
//
// Progress: a decode CTA waits only for tiles encoded by lower-numbered CTAs
// of each rank, whose encodes never wait.  HARDWARE ASSUMPTION: the CTAs of a
// grid are dispatched in increasing blockIdx order (so every CTA waited on has
// been dispatched; no MPS/green-context partitioning that could starve one).
// A wait longer than the context's timeout (30 s default) raises kFlagPeer
// (GTC_EPEER) on EVERY rank and the CTA gives up -- an error, never a hang;
// the replicas are then inconsistent (the other decode CTAs applied their
// tiles) and the caller must restore a checkpoint (gtc.h, gtc_check).
//
// Buffer reuse: the segmented buffers alternate with the step parity.  A rank
// overwrites parity p at step e + 2 only after its step e + 1 kernel read
// every rank's step e + 1 tiles, which each rank writes after its own step e
// kernel (the one reading parity p) completed (griddepcontrol.wait).
//
// Algorithmic bytes per launch (local HBM): the encode's 12 n + 4 k + 8 T,
// this rank's entries and tags read back (4 k + 8 T), 8 per touched element
// (target RMW); over NVLink: the peers' entries and tags, 4 (K - k) + 8 (N-1) T.
#include "gtc_internal.cuh"
#include "tile_encode.cuh"

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

namespace gtc {
namespace {

constexpr int kSpecPerThread = 4;   // speculative entry loads per thread (decode CTA)
constexpr int kApplyBatch = 4;      // target float4 loads per thread before their stores
static_assert(kDecGroup * kFusedMaxRanks <= kTileThreads, "one tag poller per (tile, rank)");

// Opt-in phase trace (GTC_DECODE_TRACE=1): thread 0 of each of the first
// kStepTraceCtas CTAs stamps %globaltimer at: start, tags seen (decode),
// counts done (decode), -, end; and (SM id | decode << 16).
constexpr int kStepTraceCtas = 16384;
constexpr int kStepTracePhases = 6;
__device__ unsigned long long g_step_trace[kStepTraceCtas * kStepTracePhases];

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

// ------------------------------------------------------------ encode CTA
__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

// The encode of tile t (rows a1-a5) as gtc_encode_tile_kernel, plus the push:
// the tile's record {tag, 0, entries [0, min(count, kPushCap))} is staged in
// shared memory and sent to every peer with one bulk copy each.  The CTA waits
// only until the copies have READ shared memory; the NVLink writes complete
// after it has exited, so no encode slot is held for an NVLink round trip.
// The copied range also covers the previous same-parity count, zero-filled,
// which keeps the records' stale-entry invariant (tile_encode.cuh).
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

// ------------------------------------------------------------ ticketed kernel
// The default fused step.  CTA with ticket b encodes tile b (b < T) and
// decodes tile d = b - L (0 <= d < T) of every rank; tickets [T, T + L) only
// decode, tickets [0, L) only encode.  Ticket = the order in which CTAs start
// (one atomicInc per CTA on the launch's counter, which wraps back to 0 when
// the launch's last CTA takes its ticket), so a CTA only ever waits on tiles
// encoded by CTAs that started before it, on every rank -- progress does not
// depend on the order in which the hardware dispatches CTAs.
//
// Both halves' loads go out together: r and g of tile b, every rank's tag of
// tile d and a speculative first block of each rank's entries (peers: their
// pushed records, local memory).  The decode counts tile d in biased bytes
// (0x80 + c, |c| <= 8: an integer add per entry never carries across bytes;
// shared-memory atomics, order-free, so the counts are deterministic), issues
// the target loads of the touched float4s, and the target stores go out after
// the encode's entry stores and pushes, so the target round trip overlaps
// them.  A CTA holds its slot for about one encode plus part of one round
// trip; nothing waits on NVLink unless a rank is more than L tiles behind.
constexpr int kOvPerThread = 4;     // overflow entry loads per thread per round

__device__ __forceinline__ void count_biased(unsigned* cw, unsigned e) {
    const unsigned idx = (e >> 1) & (kTile - 1);
    const unsigned sh = 8u * (idx & 3u);
    atomicAdd(cw + (idx >> 2), (e & 1u) ? (0u - (1u << sh)) : (1u << sh));
}

template <int CMP, bool HAS_G, int MODE>
__device__ __forceinline__ void ticket_cta(const FusedStepParams& f, long long b, long long trace_slot) {
    __shared__ unsigned s_scan[kTileVec * kTileWarps];
    __shared__ unsigned s_misc[2];
    __shared__ __align__(16) unsigned s_cw[kTile / 4];  // biased byte counts of tile d (word v: elements 4v..4v+3)
    __shared__ int s_k[kFusedMaxRanks];
    __shared__ int s_flag;
    __shared__ __align__(128) unsigned long long s_rec[kPushRec / 8];  // the encode's push record

    const EncodeParams& p = f.enc;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int N = f.nranks;
    const long long T = p.num_tiles;
    const long long te = b < T ? b : -1;       // tile encoded here
    const long long td = b - f.lag_tiles;      // tile decoded here
    const bool dec = td >= 0 && td < T && !(f.diag & 4);
    const bool trace = f.trace && tid == 0 && trace_slot < kStepTraceCtas;
    auto stamp_ph = [&](int ph) {
        if (trace) g_step_trace[trace_slot * kStepTracePhases + ph] = now_ns();
    };
    stamp_ph(0);
    if (trace) {
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        g_step_trace[trace_slot * kStepTracePhases + 5] = smid | (dec ? 1u << 16 : 0u) | (te < 0 ? 1u << 17 : 0u);
    }
    if (f.skip) return;  // loopback test hook: a rank that never shows up

    auto tag_ptr = [&](int m, long long t) -> const unsigned long long* {
        return f.push_in[m] ? reinterpret_cast<const unsigned long long*>(f.push_in[m] + t * kPushRec) : f.tags[m] + t;
    };
    auto entry_ptr = [&](int m, long long t, int j) -> const unsigned* {
        if (f.push_in[m] && j < kPushCap) return reinterpret_cast<const unsigned*>(f.push_in[m] + t * kPushRec + 16) + j;
        return f.seg[m] + t * kTile + j;
    };

    // ---- every load in flight at once
    const long long base = te * kTile;
    const bool full_tile = te >= 0 && base + kTile <= p.n;
    unsigned prev_ld = 0u;
    float4 rv[kTileVec], gv[kTileVec];
    if (te >= 0) {
        if (tid == kTileThreads - 1) prev_ld = ld_tag_count(p.tags + te);
        load_tile<HAS_G>(p, base, full_tile, tid, rv, gv);
    }
    const int S = kTileThreads / N;  // speculative entries per rank: thread tid reads entry sj of rank sm
    const int sm = tid / S, sj = tid - sm * S;
    unsigned long long tagv = 0ull;
    unsigned spec = 0u;
    // prefetch stage (tile tp = b - lag_pf, lag_pf < lag_tiles): the targets
    // this CTA's successors will read-modify-write are pulled into L2 now, so
    // the apply of tile tp (lag_tiles - lag_pf tickets later) waits on an L2
    // round trip, not an HBM one.  An entry carrying this step's stamp is
    // always one of its tile's (tile_encode.cuh), so no tag is needed; a record
    // not yet landed is simply not prefetched (a hint, never a wait).
    const long long tp = b - f.lag_pf;
    const bool pf = MODE != GTC_ACCUM_MOMENTUM && f.lag_pf > 0 && tp >= 0 && tp < T && sm < N;
    unsigned pfe = 0u;
    if (pf) pfe = ld_relaxed_sys(entry_ptr(sm, tp, sj));
    if (dec) {
        if (tid < N) tagv = ld_relaxed_sys(tag_ptr(tid, td));
        if (sm < N) spec = ld_relaxed_sys(entry_ptr(sm, td, sj));
        reinterpret_cast<uint4*>(s_cw)[tid] = make_uint4(0x80808080u, 0x80808080u, 0x80808080u, 0x80808080u);
    }

    // ---- encode, rows a1-a3 and the tile scan's ballots
    unsigned sel = 0u, neg = 0u, my_off[kTileVec];
    if (te >= 0) {
        bool nonfinite;
        quantize<CMP, HAS_G>(rv, gv, p.tau, sel, neg, nonfinite);
        store_residual(p, base, full_tile, tid, rv);
        if (__any_sync(0xffffffffu, nonfinite) && lane == 0) atomicOr(&p.ctrl->flags, kFlagNonFinite);
        tile_scan_ballots(sel, lane, warp, my_off, s_scan);
    }
    if (dec && tid < N) s_k[tid] = ((unsigned)(tagv >> 32) == p.epoch) ? (int)(unsigned)tagv : -1;
    const unsigned stamp = entry_stamp(p.epoch);
    if (pf && (pfe >> kStampShift) == stamp)
        asm volatile("prefetch.global.L2 [%0];" :: "l"(f.target + tp * kTile + ((pfe >> 1) & (kTile - 1))));
    __syncthreads();
    if (te >= 0 && warp == kTileWarps - 1) {
        const unsigned incl = tile_scan_finish(lane, s_scan);
        if (lane == 31) {
            s_misc[0] = incl;
            s_misc[1] = prev_ld;
            if (incl) atomicAdd(p.k_acc, (unsigned long long)incl);
            if (te == 0) *p.k_next = 0ull;
        }
    }

    // ---- decode tile d, rows a6-a7: wait until every rank's tag is this
    // step's and every speculative entry below its count carries this step's
    // stamp (a record's tag can land before its entries); rare at lag L
    bool failed = false;
    if (dec) {
        unsigned long long t0ns = 0ull;
        for (;;) {
            const bool notready = tid < N && s_k[tid] < 0;
            const bool unknown = sm < N && s_k[sm] < 0;
            const bool stale = sm < N && sj < s_k[sm] && (spec >> kStampShift) != stamp;
            if (!__syncthreads_or(notready || unknown || stale)) break;
            if (tid == 0) {
                // give up at the timeout, or at once if a peer timeout was
                // already raised on this rank (no cascade of waves of timeouts)
                const unsigned long long now = now_ns();
                if (t0ns == 0ull) t0ns = now;
                s_flag = (now - t0ns > f.timeout_ns || (ld_relaxed_sys(f.flags) & kFlagPeer)) ? 1 : 0;
            }
            __syncthreads();
            if (s_flag) {
                failed = true;
                break;
            }
            __nanosleep(64);
            if (notready) {
                tagv = ld_relaxed_sys(tag_ptr(tid, td));
                if ((unsigned)(tagv >> 32) == p.epoch) s_k[tid] = (int)(unsigned)tagv;
            }
            if (unknown || stale) spec = ld_relaxed_sys(entry_ptr(sm, td, sj));
            __syncthreads();
        }
        stamp_ph(1);
        if (!failed) {
            if (sm < N && sj < s_k[sm]) count_biased(s_cw, spec);
            // entries [S, k_m) of every rank (dense tiles); beyond kPushCap
            // they come from the owner's buffer over NVLink
            int OV = 0;
            for (int m = 0; m < N; ++m) OV += max(0, s_k[m] - S);
            const unsigned long long t_ov = OV ? now_ns() : 0ull;
            for (int c0 = 0; c0 < OV && !failed; c0 += kOvPerThread * kTileThreads) {
                unsigned ov[kOvPerThread];
                const unsigned* a[kOvPerThread];
                unsigned pend = 0u, have = 0u;
#pragma unroll
                for (int u = 0; u < kOvPerThread; ++u) {
                    const int fo = c0 + tid + u * kTileThreads;
                    a[u] = nullptr;
                    if (fo < OV) {
                        int m = 0, rem = fo;
                        while (rem >= max(0, s_k[m] - S)) {
                            rem -= max(0, s_k[m] - S);
                            ++m;
                        }
                        a[u] = entry_ptr(m, td, S + rem);
                        ov[u] = ld_relaxed_sys(a[u]);
                        have |= 1u << u;
                    }
                }
#pragma unroll
                for (int u = 0; u < kOvPerThread; ++u)
                    if (((have >> u) & 1u) && (ov[u] >> kStampShift) != stamp) pend |= 1u << u;
                while (pend && !failed) {
                    __nanosleep(64);
#pragma unroll
                    for (int u = 0; u < kOvPerThread; ++u)
                        if ((pend >> u) & 1u) ov[u] = ld_relaxed_sys(a[u]);
#pragma unroll
                    for (int u = 0; u < kOvPerThread; ++u)
                        if (((pend >> u) & 1u) && (ov[u] >> kStampShift) == stamp) pend &= ~(1u << u);
                    if (pend && now_ns() - t_ov > f.timeout_ns) failed = true;
                }
#pragma unroll
                for (int u = 0; u < kOvPerThread; ++u)
                    if (((have >> u) & 1u) && !failed) count_biased(s_cw, ov[u]);
            }
        }
    }
    // every count (and s_misc) visible; a timed-out wait anywhere aborts the decode
    failed = __syncthreads_or(failed) != 0;
    const bool apply = dec && !failed && !(f.diag & 2);
    if (dec && failed) raise_peer_error(f);
    stamp_ph(2);

    // ---- apply loads (row a8): float4 v = tid + 256 h of tile d is elements
    // 4v..4v+3, counts in word v of s_cw
    const long long db = td * kTile;
    float4 tv[kTileVec], bv[kTileVec];
    unsigned cw[kTileVec];
    unsigned todo = 0u;
    if (apply) {
#pragma unroll
        for (int h = 0; h < kTileVec; ++h) {
            const int v = tid + h * kTileThreads;
            cw[h] = s_cw[v];
            const long long e0 = db + 4ll * v;
            const bool full = e0 + 4 <= p.n;
            if (MODE == GTC_ACCUM_MOMENTUM) {
                if (full) {
                    tv[h] = ld_v4(reinterpret_cast<const float4*>(f.target + e0));
                    bv[h] = ld_v4(reinterpret_cast<const float4*>(p.buf + e0));
                }
                if (e0 < p.n) todo |= 1u << h;
            } else if (cw[h] != 0x80808080u) {
                todo |= 1u << h;
                if (full) tv[h] = *reinterpret_cast<const float4*>(f.target + e0);
            }
        }
    }

    // ---- encode, rows a4-a5: entries (stamped) to this rank's slot and the
    // push record, tag, then one bulk copy per peer
    if (te >= 0) {
        const unsigned total = s_misc[0], prev = s_misc[1];
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
        if (tid == 0) {
            const unsigned long long tag = make_tag(p.epoch, total);
            st_relaxed_sys(p.tags + te, tag);
            s_rec[0] = tag;
            s_rec[1] = 0ull;
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // smem writes -> the bulk copies
    }
    __syncthreads();
    if (te >= 0 && tid == 0 && !(f.diag & 16)) {
        const unsigned clr = min(max(s_misc[0], s_misc[1]), (unsigned)kPushCap);
        const unsigned bytes = 16u + 4u * ((clr + 3u) & ~3u);
#pragma unroll
        for (int m = 0; m < kFusedMaxRanks; ++m) {
            if (m >= N || !f.push_out[m]) continue;
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                         :: "l"(f.push_out[m] + te * kPushRec), "r"(smem_u32(s_rec)), "r"(bytes) : "memory");
        }
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }

    stamp_ph(3);
    // ---- apply stores: u = fl(c * tau); WEIGHTS fmaf(alpha, u, t), UPDATE
    // fl(t + u) (R8) on the touched elements; MOMENTUM (M1) on every element
    if (apply) {
#pragma unroll
        for (int h = 0; h < kTileVec; ++h) {
            if (!((todo >> h) & 1u)) continue;
            const long long e0 = db + 4ll * (tid + h * kTileThreads);
            const int cc[4] = {(int)(cw[h] & 0xffu) - 128, (int)((cw[h] >> 8) & 0xffu) - 128,
                               (int)((cw[h] >> 16) & 0xffu) - 128, (int)(cw[h] >> 24) - 128};
            if (MODE == GTC_ACCUM_MOMENTUM) {
                auto mom = [&](float& w, float& bf, int c) {
                    const float u = __fmul_rn((float)c, p.tau);
                    bf = __fadd_rn(__fmul_rn(p.mu, bf), u);
                    w = __fmaf_rn(f.alpha, bf, w);
                };
                if (e0 + 4 <= p.n) {
                    mom(tv[h].x, bv[h].x, cc[0]);
                    mom(tv[h].y, bv[h].y, cc[1]);
                    mom(tv[h].z, bv[h].z, cc[2]);
                    mom(tv[h].w, bv[h].w, cc[3]);
                    st_stream(reinterpret_cast<float4*>(f.target + e0), tv[h]);
                    st_stream(reinterpret_cast<float4*>(p.buf + e0), bv[h]);
                } else {
                    for (int e = 0; e < 4 && e0 + e < p.n; ++e) mom(f.target[e0 + e], p.buf[e0 + e], cc[e]);
                }
            } else if (e0 + 4 <= p.n) {
                float4 t = tv[h];
                if (cc[0]) t.x = apply_count<MODE>(t.x, cc[0], p.tau, f.alpha);
                if (cc[1]) t.y = apply_count<MODE>(t.y, cc[1], p.tau, f.alpha);
                if (cc[2]) t.z = apply_count<MODE>(t.z, cc[2], p.tau, f.alpha);
                if (cc[3]) t.w = apply_count<MODE>(t.w, cc[3], p.tau, f.alpha);
                *reinterpret_cast<float4*>(f.target + e0) = t;
            } else {
                for (int e = 0; e < 4 && e0 + e < p.n; ++e)
                    if (cc[e]) f.target[e0 + e] = apply_count<MODE>(f.target[e0 + e], cc[e], p.tau, f.alpha);
            }
        }
    }
    if (te >= 0 && tid == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    stamp_ph(4);
}

// The ticket of this CTA (one atomicInc; the counter wraps to 0 with the
// launch's last ticket).  The atomic is performed before griddepcontrol's
// launch_dependents, so a dependent launch on the stream (the next step) only
// takes tickets after every ticket of this launch is taken.
__device__ __forceinline__ unsigned take_ticket(unsigned* counter, unsigned last) {
    __shared__ unsigned s_ticket;
    if (threadIdx.x == 0) s_ticket = atomicInc(counter, last);
    __syncthreads();
    return s_ticket;
}

template <int CMP, bool HAS_G, int MODE>
#ifndef GTC_TICKET_CTAS
#define GTC_TICKET_CTAS 4
#endif
__global__ void __launch_bounds__(kTileThreads, GTC_TICKET_CTAS) gtc_step_ticket_kernel(const FusedStepParams f) {
    const unsigned b = (f.diag & 1) ? blockIdx.x : take_ticket(f.ticket, gridDim.x - 1u);
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;");
    ticket_cta<CMP, HAS_G, MODE>(f, b, b);
}

// Loopback group: one ticket sequence for the whole group (rank 0's
// counter); ticket g is CTA g / world of rank g % world, so every tile a CTA
// waits on (a lower CTA index of any rank) belongs to a lower ticket.
template <int CMP, bool HAS_G, int MODE>
__global__ void __launch_bounds__(kTileThreads, GTC_TICKET_CTAS)
gtc_step_ticket_group_kernel(const FusedStepParams* __restrict__ group, int world) {
    __shared__ FusedStepParams s_f;
    const unsigned g = take_ticket(group[0].ticket, gridDim.x - 1u);
    const int rank = (int)(g % (unsigned)world);
    const int* src = reinterpret_cast<const int*>(group + rank);
    int* dst = reinterpret_cast<int*>(&s_f);
    for (int i = threadIdx.x; i < (int)(sizeof(FusedStepParams) / sizeof(int)); i += blockDim.x) dst[i] = src[i];
    __syncthreads();
    ticket_cta<CMP, HAS_G, MODE>(s_f, g / (unsigned)world, g);
}

// CTA b of one rank's step.
template <int CMP, bool HAS_G, int MODE>
__device__ __forceinline__ void step_cta(const FusedStepParams& f, long long b, long long trace_slot) {
    __shared__ unsigned s_scan[kTileVec * kTileWarps];
    __shared__ unsigned s_misc[2];
    __shared__ int4 s_cnt4[kDecGroup * kTile / 16];  // int8 counts of the decode CTA's tiles
    __shared__ int s_k[kDecGroup * kFusedMaxRanks];
    __shared__ int s_abort;
    __shared__ __align__(128) unsigned long long s_rec[kPushRec / 8];  // the encode's push record

    const EncodeParams& p = f.enc;
    const bool trace = f.trace && threadIdx.x == 0 && trace_slot < kStepTraceCtas;
    auto stamp_ph = [&](int ph) {
        if (trace) g_step_trace[trace_slot * kStepTracePhases + ph] = now_ns();
    };
    stamp_ph(0);
    if (f.skip) return;  // loopback test hook: a rank that never shows up

    // CTA role: b < Q * (G + 1): group q = b / (G + 1), slot r = b % (G + 1);
    // r < G encodes tile q * G + r, r == G decodes group q - lag_groups; the
    // tail decodes the last min(lag_groups, Q) groups.
    const long long Q = f.num_groups;
    long long enc_tile = -1, dec_group = -1;
    if (b < Q * (kDecGroup + 1)) {
        const long long q = b / (kDecGroup + 1), r = b - q * (kDecGroup + 1);
        if (r < kDecGroup) enc_tile = q * kDecGroup + r;
        else dec_group = q - f.lag_groups;
    } else {
        dec_group = (Q - min((long long)f.lag_groups, Q)) + (b - Q * (kDecGroup + 1));
    }
    if (trace) {
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        g_step_trace[trace_slot * kStepTracePhases + 5] = smid | (enc_tile < 0 ? 1u << 16 : 0u);
    }
    if (enc_tile >= 0) {
        if (enc_tile < p.num_tiles) encode_cta<CMP, HAS_G>(f, enc_tile, s_scan, s_misc, s_rec);
    } else if (dec_group >= 0) {
        const long long t0 = dec_group * kDecGroup;
        const int ng = (int)min((long long)kDecGroup, (long long)p.num_tiles - t0);
        decode_cta<MODE>(f, t0, ng, reinterpret_cast<signed char*>(s_cnt4), s_k, &s_abort, stamp_ph);
    }
    stamp_ph(4);
}

template <int CMP, bool HAS_G, int MODE>
__global__ void __launch_bounds__(kTileThreads, 4) gtc_step_p2p_kernel(const FusedStepParams f) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;");
    step_cta<CMP, HAS_G, MODE>(f, blockIdx.x, blockIdx.x);
}

// Loopback group (tests): the steps of `world` ranks of one process as ONE
// launch.  Linear block b is CTA b / world of rank b % world, so every CTA a
// decode CTA waits on (a lower CTA index of any rank) has a lower linear index
// -- the same dispatch-order argument as the per-rank kernel.  Kernels that
// wait on each other are never launched separately on one GPU.
template <int CMP, bool HAS_G, int MODE>
__global__ void __launch_bounds__(kTileThreads, 4)
gtc_step_p2p_group_kernel(const FusedStepParams* __restrict__ group, int world) {
    __shared__ FusedStepParams s_f;
    const int rank = (int)(blockIdx.x % (unsigned)world);
    const int* src = reinterpret_cast<const int*>(group + rank);
    int* dst = reinterpret_cast<int*>(&s_f);
    for (int i = threadIdx.x; i < (int)(sizeof(FusedStepParams) / sizeof(int)); i += blockDim.x) dst[i] = src[i];
    __syncthreads();
    step_cta<CMP, HAS_G, MODE>(s_f, blockIdx.x / (unsigned)world, blockIdx.x);
}

// ------------------------------------------------------------ warp-specialized kernel
// The default fused step (WEIGHTS / UPDATE).  A persistent grid of two CTAs
// per SM, each with kWsGroups ENCODE GROUPS of 256 threads and kWsDecWarps
// DECODE WARPS.  Why: in every one-CTA-per-tile design the decode's latency-bound
// round trips sit inside the CTAs that also carry the encode's HBM stream, so
// they take slot time the stream needs (encode alone 55 us,
// + pushes 61, + counting 69, + apply 76 us at N=2).  Here the encode groups
// only stream (the register-load tile encode, 4 tiles in flight per SM, as in
// the world-1 kernel) and the decode warps, outside that budget, follow the
// encode by about one wave with two tiles in flight each.
//   encode group: takes tickets (atomicInc, the next one taken while the
//     current tile is processed) over (rank, tile) pairs and encodes the tile
//     exactly as ticket_cta: stamped entries + tag (relaxed system-scope
//     stores) and the record pushed to every peer by one bulk copy each.
//   decode warp: decodes (rank, tile) tickets gw, gw + W, ... (W decode warps
//     in the grid), which the encode front reaches in that order; for tile d of rank r
//     it polls every rank's tag (peers: the pushed records, local memory),
//     validates the speculative entries by their stamps, counts them in a
//     warp-private biased-byte array (shared-memory atomics: order-free,
//     deterministic), and read-modify-writes the touched float4s of the
//     target (R8).  The next tile's tags and entries are loaded before the
//     current tile's target round trip.
// Progress: an encode never waits, and every tile is encoded by whichever
// groups are running (tickets), so a waiting decode warp always waits on
// work that is in progress on some rank -- no assumption on which CTAs are
// resident.  A loopback group (R ranks of one process) runs every rank's
// tickets in every CTA (ticket g = rank g % R, tile g / R).
#ifndef GTC_WS_GROUPS
#define GTC_WS_GROUPS 2
#endif
#ifndef GTC_WS_DECW
#define GTC_WS_DECW 2
#endif
#ifndef GTC_WS_CTAS
#define GTC_WS_CTAS 2
#endif
constexpr int kWsGroups = GTC_WS_GROUPS;   // encode groups per CTA
constexpr int kWsDecWarps = GTC_WS_DECW;   // decode warps per CTA
constexpr int kWsCtasPerSm = GTC_WS_CTAS;  // resident CTAs per SM (launch bounds)
constexpr int kWsThreads = kWsGroups * kTileThreads + kWsDecWarps * 32;
constexpr int kWsSpec = 8;  // speculative entry loads per decode lane per tile
constexpr int kWsDecSmem = 4 * (kTile / 4 + 2 * 32 * kWsSpec + 32);  // dynamic smem per decode warp
constexpr int kWsBatch = 4; // target float4 loads in flight per decode lane
constexpr int kWsTraceTiles = 24;                       // debug trace: tiles per decode warp 0
constexpr long long kWsTraceBase = 2048ll * kStepTracePhases;  // ... after the CTA slots

struct alignas(128) WsGroupSmem {
    unsigned long long rec[kPushRec / 8];  // the encode's push record (bulk copy source)
    unsigned scan[kTileVec * kTileWarps];
    unsigned misc[2];
    unsigned ticket;
};

__device__ __forceinline__ void group_bar(int g) {
    asm volatile("bar.sync %0, %1;" :: "r"(g + 1), "n"(kTileThreads) : "memory");
}

// One tile of an encode group (rows a1-a5 + the push), as ticket_cta's encode.
// `nxt` (leader only) is the group's next ticket, published to the group here.
template <int CMP, bool HAS_G>
__device__ __forceinline__ unsigned ws_encode_tile(const FusedStepParams& f, long long t, int g, int gt,
                                                   WsGroupSmem& G, unsigned nxt) {
    const EncodeParams& p = f.enc;
    const int lane = gt & 31, lw = gt >> 5;
    const long long base = t * kTile;
    const bool full_tile = base + kTile <= p.n;
    unsigned prev_ld = 0u;
    if (gt == kTileThreads - 1) prev_ld = ld_tag_count(p.tags + t);
    float4 rv[kTileVec], gv[kTileVec];
    load_tile<HAS_G>(p, base, full_tile, gt, rv, gv);
    unsigned sel, neg;
    bool nonfinite;
    quantize<CMP, HAS_G>(rv, gv, p.tau, sel, neg, nonfinite);
    store_residual(p, base, full_tile, gt, rv);
    if (__any_sync(0xffffffffu, nonfinite) && lane == 0) atomicOr(&p.ctrl->flags, kFlagNonFinite);
    unsigned my_off[kTileVec];
    tile_scan_ballots(sel, lane, lw, my_off, G.scan);
    group_bar(g);
    if (lw == kTileWarps - 1) {
        const unsigned incl = tile_scan_finish(lane, G.scan);
        if (lane == 31) {
            G.misc[0] = incl;
            G.misc[1] = prev_ld;
            if (incl) atomicAdd(p.k_acc, (unsigned long long)incl);
            if (t == 0) *p.k_next = 0ull;
        }
    }
    group_bar(g);
    const unsigned total = G.misc[0], prev = G.misc[1];
    const unsigned stamp = entry_stamp(p.epoch);
    unsigned* dst = p.seg + base;
    unsigned* s_ent = reinterpret_cast<unsigned*>(G.rec + 2);
    if (total != 0) {
#pragma unroll
        for (int j = 0; j < kTileVec; ++j) {
            unsigned o = G.scan[j * kTileWarps + lw] + my_off[j];
            const unsigned l0 = (unsigned)(j * kTileThreads + gt) * 4u;
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
    for (unsigned o = total + gt; o < prev; o += kTileThreads) st_relaxed_sys(dst + o, 0u);
    const unsigned clr = min(max(total, prev), (unsigned)kPushCap);
    const unsigned clr4 = (clr + 3u) & ~3u;  // bulk copies move multiples of 16 bytes
    for (unsigned o = total + gt; o < clr4; o += kTileThreads) s_ent[o] = 0u;
    if (gt == 0) {
        const unsigned long long tag = make_tag(p.epoch, total);
        st_relaxed_sys(p.tags + t, tag);
        G.rec[0] = tag;
        G.rec[1] = 0ull;
        G.ticket = nxt;
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // smem writes -> the bulk copies
    group_bar(g);
    const unsigned next = G.ticket;
    if (gt == 0) {
        const unsigned bytes = 16u + 4u * clr4;
        for (int m = 0; m < f.nranks; ++m) {
            if (!f.push_out[m]) continue;
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                         :: "l"(f.push_out[m] + t * kPushRec), "r"(smem_u32(G.rec)), "r"(bytes) : "memory");
        }
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        // the record buffer is rewritten by the group's next tile
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    }
    return next;
}

// The decode warp's messages of one tile: every rank's tag in lane m < N's
// register, and the first S = (32 kWsSpec / N) & ~3 entries of every rank
// (flat index m S + j) copied by cp.async into the warp's shared buffer --
// no register holds an in-flight entry, so nothing spills and no copy waits
// for another (a register spill of a loaded value serialises the loads).
constexpr int kWsSlots = 32 * kWsSpec;  // entry slots per buffer
// NR: the rank count rounded up to 2, 4 or 8 (a template parameter: the
// window S = kWsSlots / NR and every slot's rank are compile-time constants)
__host__ __device__ constexpr int ws_nr(int N) { return N <= 2 ? 2 : N <= 4 ? 4 : 8; }

__device__ __forceinline__ const unsigned long long* ws_tag_ptr(const FusedStepParams& f, int m, long long t) {
    return f.push_in[m] ? reinterpret_cast<const unsigned long long*>(f.push_in[m] + t * kPushRec) : f.tags[m] + t;
}
__device__ __forceinline__ const unsigned* ws_entry_ptr(const FusedStepParams& f, int m, long long t, int j) {
    if (f.push_in[m] && j < kPushCap) return reinterpret_cast<const unsigned*>(f.push_in[m] + t * kPushRec + 16) + j;
    return f.seg[m] + t * kTile + j;
}

template <int NR>
__device__ __forceinline__ unsigned long long ws_load_msgs(const FusedStepParams& f, long long d, int lane,
                                                           unsigned* buf) {
    constexpr int S = kWsSlots / NR;
    const int N = f.nranks;
    unsigned long long tag = 0ull;
    if (lane < N) tag = ld_relaxed_sys(ws_tag_ptr(f, lane, d));
#pragma unroll
    for (int h = 0; h < kWsSlots / 4 / 32; ++h) {  // 16-byte chunks
        const int c = lane + 32 * h, m = (4 * c) / S;
        if (m < N) {
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;"
                         :: "r"(smem_u32(buf + 4 * c)), "l"(ws_entry_ptr(f, m, d, 4 * c - m * S)) : "memory");
        }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    return tag;
}

// The encode front has passed ticket q: its own-rank tile carries this step's
// tag (q >= TR, or a skipped rank: trivially).  A decode warp starts ticket c
// only once the front has passed c + W, one decode round (about one wave of
// the grid) later, so the tile's records have landed everywhere and one round
// trip fetches valid tags and entries.
__device__ __forceinline__ bool ws_front_passed(const FusedStepParams* par, int R, unsigned TR, unsigned q, int lane) {
    int ok = 1;
    if (lane == 0 && q < TR && !par[q % R].skip) {
        const EncodeParams& p = par[q % R].enc;
        ok = (unsigned)(ld_relaxed_sys(p.tags + q / R) >> 32) == p.epoch;
    }
    return __shfl_sync(0xffffffffu, ok, 0) != 0;
}

// Decode + apply tile d of rank f (rows a6-a8).  Returns false if a peer timed
// out (nothing of this tile applied).  tag / buf: this tile's messages
// (ws_load_msgs, its cp.async group the only one outstanding).  cw: the
// warp's biased counts, all 0x80808080 on entry and on return.  nxt: the
// warp's next (rank, tile) ticket; if the encode front has passed its round
// (a probe loaded at the start), its messages go into nbuf / ntag right after
// this tile's first target loads, so both round trips overlap.
template <int MODE, int NR>
__device__ __forceinline__ bool ws_decode_tile(const FusedStepParams& f, long long d, int lane,
                                               unsigned long long tag, unsigned* buf, unsigned* cw, unsigned* bm,
                                               unsigned nxt, const FusedStepParams* par, int R, unsigned TR,
                                               unsigned W, unsigned* nbuf, unsigned long long& ntag,
                                               bool& nloaded, unsigned long long* dts) {
    const EncodeParams& p = f.enc;
    constexpr int S = kWsSlots / NR;
    const int N = f.nranks;
    const unsigned stamp = entry_stamp(p.epoch);
    // 0. probe: has the encode front passed the next ticket's own round?
    const bool nxt_live = nxt < TR && !par[nxt % R].skip;
    const unsigned q = nxt + W;
    const bool q_trivial = q >= TR || par[q % R].skip;
    unsigned long long probe = 0ull;
    if (lane == 0 && nxt_live && !q_trivial) probe = ld_relaxed_sys(par[q % R].enc.tags + q / R);
    // 1. every rank's tag of this step (poll with a back-off; a peer timeout
    //    raised anywhere makes the wait give up at once)
    bool ok = true;
    unsigned long long t0 = 0ull;
    for (;;) {
        const bool ready = lane >= N || (unsigned)(tag >> 32) == p.epoch;
        if (__all_sync(0xffffffffu, ready)) break;
        int give_up = 0;
        if (lane == 0) {
            const unsigned long long now = now_ns();
            if (t0 == 0ull) t0 = now;
            give_up = (now - t0 > f.timeout_ns || (ld_relaxed_sys(f.flags) & kFlagPeer)) ? 1 : 0;
        }
        if (__shfl_sync(0xffffffffu, give_up, 0)) {
            ok = false;
            break;
        }
        __nanosleep(256);
        if (!ready) tag = ld_relaxed_sys(ws_tag_ptr(f, lane, d));
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncwarp();
    if (dts) dts[4] = now_ns();
    // 2. count the entries: lane m < N holds rank m's count, read by shuffle;
    //    an entry of this step still stale in the copy (a record's tag can
    //    land before its entries) is re-polled.  The first entry to touch a
    //    float4 (claim bitmap bm) makes its lane the one that applies it.
    const int kl = lane < N ? (int)(unsigned)tag : 0;
    int kk[NR];  // every rank's count, in every lane
#pragma unroll
    for (int m = 0; m < NR; ++m) kk[m] = __shfl_sync(0xffffffffu, kl, m);
    unsigned claimed = 0u;  // bit u: this lane applies the float4 of slot u's entry
    bool dense = false;     // entries beyond the window: apply by a full scan
    if (ok) {
        // slot u of this lane is entry j = 32 u - m S + lane of rank m = 32 u / S
        // (compile-time); all slots' loads first, then the atomics
        unsigned ev[kWsSpec], valid = 0u;
#pragma unroll
        for (int u = 0; u < kWsSpec; ++u) ev[u] = buf[lane + 32 * u];
#pragma unroll
        for (int u = 0; u < kWsSpec; ++u) {
            const int m = (32 * u) / S, j = 32 * u - m * S + lane;
            if (j < kk[m]) valid |= 1u << u;
        }
#pragma unroll
        for (int u = 0; u < kWsSpec; ++u) {
            if (((valid >> u) & 1u) && (ev[u] >> kStampShift) != stamp) {
                // rare: re-poll until this step's entry has landed
                const int fl = lane + 32 * u, m = (32 * u) / S, j = fl - m * S;
                const unsigned long long ts = now_ns();
                const unsigned* a = ws_entry_ptr(f, m, d, j);
                unsigned e;
                do {
                    __nanosleep(128);
                    e = ld_relaxed_sys(a);
                    if (now_ns() - ts > f.timeout_ns) {
                        ok = false;
                        break;
                    }
                } while ((e >> kStampShift) != stamp);
                ev[u] = e;
                buf[fl] = e;
                if ((e >> kStampShift) != stamp) valid &= ~(1u << u);
            }
        }
#pragma unroll
        for (int u = 0; u < kWsSpec; ++u) {
            if ((valid >> u) & 1u) count_biased(cw, ev[u]);
        }
        unsigned old[kWsSpec];
#pragma unroll
        for (int u = 0; u < kWsSpec; ++u) {
            const unsigned wd = (ev[u] >> 3) & (kTile / 4 - 1);
            old[u] = ((valid >> u) & 1u) ? atomicOr(bm + (wd >> 5), 1u << (wd & 31u)) : ~0u;
        }
#pragma unroll
        for (int u = 0; u < kWsSpec; ++u)
            if (!((old[u] >> ((ev[u] >> 3) & 31u)) & 1u)) claimed |= 1u << u;
        // entries beyond the window (tiles denser than S / 4096): rank m's are
        // overflow indices [ovx_m, ovx_m + ov_m)
        const int ovl = lane < N ? max(0, kl - S) : 0;
        int ovx = ovl;  // inclusive prefix over the lanes (ranks)
#pragma unroll
        for (int o = 1; o < kFusedMaxRanks; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, ovx, o);
            if (lane >= o) ovx += y;
        }
        const int OV = __shfl_sync(0xffffffffu, ovx, kFusedMaxRanks - 1);
        ovx -= ovl;  // exclusive
        dense = OV > 0;
        const unsigned long long t_ov = OV ? now_ns() : 0ull;
        for (int c0 = 0; c0 < OV && __all_sync(0xffffffffu, ok); c0 += 32 * kWsBatch) {
            unsigned ov[kWsBatch];
            const unsigned* a[kWsBatch];
            unsigned have = 0u, pnd = 0u;
#pragma unroll
            for (int u = 0; u < kWsBatch; ++u) {
                const int fo = c0 + lane + 32 * u;
                a[u] = nullptr;
                int m = 0;
#pragma unroll
                for (int qq = 1; qq < kFusedMaxRanks; ++qq)
                    if (qq < N && __shfl_sync(0xffffffffu, ovx, qq) <= fo) m = qq;
                const int rem = fo - __shfl_sync(0xffffffffu, ovx, m);
                if (fo < OV) {
                    a[u] = ws_entry_ptr(f, m, d, S + rem);
                    ov[u] = ld_relaxed_sys(a[u]);
                    have |= 1u << u;
                }
            }
#pragma unroll
            for (int u = 0; u < kWsBatch; ++u)
                if (((have >> u) & 1u) && (ov[u] >> kStampShift) != stamp) pnd |= 1u << u;
            while (pnd) {
                if (now_ns() - t_ov > f.timeout_ns) {
                    pnd = 0u;
                    have = 0u;
                    ok = false;
                    break;
                }
                __nanosleep(128);
#pragma unroll
                for (int u = 0; u < kWsBatch; ++u) {
                    if (!((pnd >> u) & 1u)) continue;
                    ov[u] = ld_relaxed_sys(a[u]);
                    if ((ov[u] >> kStampShift) == stamp) pnd &= ~(1u << u);
                }
            }
#pragma unroll
            for (int u = 0; u < kWsBatch; ++u)
                if ((have >> u) & 1u) count_biased(cw, ov[u]);
        }
    }
    ok = __all_sync(0xffffffffu, ok);
    __syncwarp();
    if (dts) dts[5] = now_ns();
    // 3. apply (R8): word v = lane + 32 i holds the counts of elements 4v..4v+3;
    //    every word is reset to 0x80808080 for the warp's next tile
    auto load_next = [&]() {
        nloaded = false;
        if (!nxt_live) return;
        const int passed = q_trivial || (unsigned)(probe >> 32) == par[q % R].enc.epoch;
        if (__shfl_sync(0xffffffffu, passed, 0)) {
            ntag = ws_load_msgs<NR>(par[nxt % R], nxt / R, lane, nbuf);
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
            if (cc[0]) t.x = apply_count<MODE>(t.x, cc[0], p.tau, f.alpha);
            if (cc[1]) t.y = apply_count<MODE>(t.y, cc[1], p.tau, f.alpha);
            if (cc[2]) t.z = apply_count<MODE>(t.z, cc[2], p.tau, f.alpha);
            if (cc[3]) t.w = apply_count<MODE>(t.w, cc[3], p.tau, f.alpha);
            *reinterpret_cast<float4*>(f.target + e0) = t;
        } else {
            for (int e = 0; e < 4 && e0 + e < p.n; ++e)
                if (cc[e]) f.target[e0 + e] = apply_count<MODE>(f.target[e0 + e], cc[e], p.tau, f.alpha);
        }
    };
    bool first = true;
    if (__any_sync(0xffffffffu, dense || !ok)) {
        // dense tile (or an abort): every word is scanned
        unsigned touched = 0u;
#pragma unroll 8
        for (int i = 0; i < kTile / 4 / 32; ++i)
            if (cw[lane + 32 * i] != 0x80808080u) touched |= 1u << i;
        if (!ok) {
            for (unsigned m = touched; m; m &= m - 1u) cw[lane + 32 * (__ffs(m) - 1)] = 0x80808080u;
            touched = 0u;
        }
        while (__any_sync(0xffffffffu, touched != 0u)) {
            int iv[kWsBatch];
            float4 tv[kWsBatch];
#pragma unroll
            for (int u = 0; u < kWsBatch; ++u) {
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
            for (int u = 0; u < kWsBatch; ++u)
                if (iv[u] >= 0) apply_word(iv[u], tv[u]);
        }
    } else {
        // the float4s this lane claimed, from its own entries
        while (__any_sync(0xffffffffu, claimed != 0u)) {
            int iv[kWsBatch];
            float4 tv[kWsBatch];
#pragma unroll
            for (int u = 0; u < kWsBatch; ++u) {
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
                if (dts) dts[6] = now_ns();
            }
#pragma unroll
            for (int u = 0; u < kWsBatch; ++u)
                if (iv[u] >= 0) apply_word(iv[u], tv[u]);
        }
    }
    if (first) load_next();
    __syncwarp();
    bm[lane] = 0u;  // the claim bitmap, cleared for the warp's next tile
    __syncwarp();
    if (dts) dts[7] = now_ns();
    return ok;
}

// An encode group passing over a ticket of a skipped rank (loopback test hook).
__device__ __forceinline__ unsigned ws_pass_ticket(WsGroupSmem& G, int g, int gt, unsigned nxt) {
    if (gt == 0) G.ticket = nxt;
    group_bar(g);
    const unsigned next = G.ticket;
    group_bar(g);
    return next;
}

// The CTA body; par[0..R) are the ranks whose work this grid does (one rank,
// or a loopback group), in shared memory.
template <int CMP, bool HAS_G, int MODE, int NR, bool GROUP>
__device__ __forceinline__ void ws_cta(const FusedStepParams* par, int R_) {
    const int R = GROUP ? R_ : 1;
    __shared__ WsGroupSmem s_grp[kWsGroups];
    // decode warps' arrays in dynamic shared memory (kWsDecSmem bytes per warp):
    // biased counts (4 KB), two message buffers (2 x 1 KB), claim bitmap
    extern __shared__ __align__(16) unsigned s_dyn[];
    __shared__ unsigned s_tiles;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const FusedStepParams& f0 = par[0];
    const unsigned TR = (unsigned)f0.enc.num_tiles * (unsigned)R;
    const long long slot = blockIdx.x;
    const bool trace = f0.trace && slot < kStepTraceCtas;
    if (trace && tid == 0) {
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        g_step_trace[slot * kStepTracePhases + 0] = now_ns();
        g_step_trace[slot * kStepTracePhases + 5] = smid | (1u << 18);
        s_tiles = 0u;
    }
    __syncthreads();
    if (warp < kWsGroups * kTileWarps) {
        // ---- encode group g
        const int g = warp / kTileWarps, gt = tid - g * kTileThreads;
        WsGroupSmem& G = s_grp[g];
        const unsigned last = TR + gridDim.x * kWsGroups - 1u;
        if (gt == 0) G.ticket = atomicInc(f0.ticket, last);
        group_bar(g);
        unsigned cur = G.ticket, done = 0u;
        while (cur < TR) {
            unsigned nxt = 0u;
            if (gt == 0) nxt = atomicInc(f0.ticket, last);  // in flight during this tile
            const FusedStepParams& f = par[cur % R];
            if (f.skip) {
                cur = ws_pass_ticket(G, g, gt, nxt);
                continue;
            }
            cur = ws_encode_tile<CMP, HAS_G>(f, cur / R, g, gt, G, nxt);
            ++done;
        }
        if (trace && gt == 0) {
            atomicAdd(&s_tiles, done);
            if (g == 0) g_step_trace[slot * kStepTracePhases + 1] = now_ns();
        }
    } else {
        // ---- decode warp
        const int dw = warp - kWsGroups * kTileWarps;
        unsigned* cw = s_dyn + dw * (kWsDecSmem / 4);
        unsigned* msg0 = cw + kTile / 4;
        unsigned* bm = msg0 + 2 * kWsSlots;
        bm[lane] = 0u;
#pragma unroll
        for (int i = 0; i < kTile / 4 / 4 / 32; ++i)
            reinterpret_cast<uint4*>(cw)[lane + 32 * i] = make_uint4(0x80808080u, 0x80808080u, 0x80808080u, 0x80808080u);
        __syncwarp();
        // tiles gw, gw + W, gw + 2 W, ... (static: a decode warp waits only on
        // encodes, which never wait, so any assignment makes progress; the
        // warps follow the encode front about one wave behind)
        const unsigned W = gridDim.x * kWsDecWarps;
        unsigned cur = blockIdx.x * kWsDecWarps + dw;
        unsigned long long tag = 0ull, ntag = 0ull;
        bool loaded = false;
        unsigned tiles_done = 0u, b = 0u;
        while (cur < TR) {
            const unsigned nxt = cur + W;
            const FusedStepParams& f = par[cur % R];
            if (f.skip) {
                cur = nxt;
                loaded = false;
                continue;
            }
            // debug trace (GTC_DECODE_TRACE=1): decode warp 0 of each CTA stamps
            // (arrival, messages issued, done, loaded-ahead, tags, counted,
            // first target loads, applied) per tile
            const bool dtr = trace && dw == 0 && lane == 0 && tiles_done < kWsTraceTiles;
            unsigned long long* dts = g_step_trace + kWsTraceBase + (slot * kWsTraceTiles + tiles_done) * 8;
            if (dtr) dts[0] = now_ns(), dts[3] = loaded ? 1ull : 0ull;
            if (!loaded) {
                while (!ws_front_passed(par, R, TR, cur + W, lane)) __nanosleep(512);
                tag = ws_load_msgs<NR>(f, cur / R, lane, msg0 + b * kWsSlots);
            }
            if (dtr) dts[1] = now_ns();
            if (!ws_decode_tile<MODE, NR>(f, cur / R, lane, tag, msg0 + b * kWsSlots, cw, bm, nxt, par, R, TR, W,
                                      msg0 + (b ^ 1u) * kWsSlots,
                                      ntag, loaded, dtr ? dts : nullptr) &&
                lane < f.nranks)
                atomicOr_system(f.peer_flags[lane], kFlagPeer);  // GTC_EPEER on every rank
            if (dtr) dts[2] = now_ns();
            ++tiles_done;
            cur = nxt;
            if (loaded) {
                tag = ntag;
                b ^= 1u;
            }
        }
        if (trace && dw == 0 && lane == 0) g_step_trace[slot * kStepTracePhases + 2] = now_ns();
    }
    if (trace) {
        __syncthreads();
        if (tid == 0) {
            g_step_trace[slot * kStepTracePhases + 3] = s_tiles;
            g_step_trace[slot * kStepTracePhases + 4] = now_ns();
        }
    }
}

template <int CMP, bool HAS_G, int MODE, int NR>
__global__ void __launch_bounds__(kWsThreads, kWsCtasPerSm) gtc_step_ws_kernel(const FusedStepParams f) {
    __shared__ FusedStepParams s_par[1];
    {
        const int* src = reinterpret_cast<const int*>(&f);
        int* dst = reinterpret_cast<int*>(s_par);
        for (int i = threadIdx.x; i < (int)(sizeof(FusedStepParams) / sizeof(int)); i += blockDim.x) dst[i] = src[i];
    }
    // the previous step's kernel is complete (its memory visible) before any
    // ticket is taken: every ticket of that launch is taken by then
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;");
    __syncthreads();
    ws_cta<CMP, HAS_G, MODE, NR, false>(s_par, 1);
}

// Loopback group: every CTA does the work of every rank (tickets interleave
// the ranks), so no CTA waits on a rank whose CTAs are not resident.
template <int CMP, bool HAS_G, int MODE, int NR>
__global__ void __launch_bounds__(kWsThreads, kWsCtasPerSm)
gtc_step_ws_group_kernel(const FusedStepParams* __restrict__ group, int world) {
    __shared__ FusedStepParams s_par[kFusedMaxRanks];
    const int* src = reinterpret_cast<const int*>(group);
    int* dst = reinterpret_cast<int*>(s_par);
    for (int i = threadIdx.x; i < (int)(sizeof(FusedStepParams) / sizeof(int)) * world; i += blockDim.x) dst[i] = src[i];
    __syncthreads();
    ws_cta<CMP, HAS_G, MODE, NR, true>(s_par, world);
}

// The decode warps' dynamic shared memory may exceed the 48 KB default.
template <typename K>
void ws_smem_attr(K kernel) {
    static std::mutex mu;
    static std::vector<const void*> done;  // kernels whose attribute is set
    std::lock_guard<std::mutex> lock(mu);
    const void* k = reinterpret_cast<const void*>(kernel);
    if (std::find(done.begin(), done.end(), k) == done.end()) {
        cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kWsDecWarps * kWsDecSmem);
        done.push_back(k);
    }
}

// Persistent grid: every CTA slot of the device.
int ws_grid() {
    static std::once_flag once;
    static int grid = 296;
    std::call_once(once, [] {
        int dev = 0, sms = 0, per_sm = 0;
        if (cudaGetDevice(&dev) == cudaSuccess &&
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess &&
            (ws_smem_attr(gtc_step_ws_kernel<GTC_CMP_GT, true, GTC_ACCUM_WEIGHTS, 2>), true) &&
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, gtc_step_ws_kernel<GTC_CMP_GT, true, GTC_ACCUM_WEIGHTS, 2>,
                                                          kWsThreads, kWsDecWarps * kWsDecSmem) == cudaSuccess &&
            sms > 0 && per_sm > 0)
            grid = sms * per_sm;
    });
    return grid;
}

// GTC_STEP_KERNEL=grouped: the previous design (groups of encode CTAs and a
// decode CTA, roles by blockIdx), kept for comparison
bool grouped_kernel() {
    static int v = -1;
    if (v < 0) {
        const char* e = std::getenv("GTC_STEP_KERNEL");
        v = (e && std::strcmp(e, "grouped") == 0) ? 1 : 0;
    }
    return v == 1;
}

// GTC_STEP_KERNEL=ticket: the ticketed one-CTA-per-tile kernel for every mode
// (default: the warp-specialized kernel for WEIGHTS / UPDATE, the ticketed
// one for MOMENTUM, whose dense apply is a second full stream)
bool ticket_kernel_forced() {
    static int v = -1;
    if (v < 0) {
        const char* e = std::getenv("GTC_STEP_KERNEL");
        v = (e && std::strcmp(e, "ticket") == 0) ? 1 : 0;
    }
    return v == 1;
}

bool use_ws(int mode) { return mode != GTC_ACCUM_MOMENTUM && !grouped_kernel() && !ticket_kernel_forced(); }

template <int CMP, bool HAS_G, int MODE>
cudaError_t launch_t(FusedStepParams& f, cudaStream_t s) {
    cudaLaunchConfig_t cfg = {};
    const long long Q = f.num_groups;
    const bool grouped = grouped_kernel();
    cfg.gridDim = grouped ? dim3((unsigned)(Q * (kDecGroup + 1) + std::min<long long>(f.lag_groups, Q)))
                          : dim3((unsigned)(f.enc.num_tiles + f.lag_tiles));
    cfg.blockDim = dim3(kTileThreads);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (grouped) return cudaLaunchKernelEx(&cfg, gtc_step_p2p_kernel<CMP, HAS_G, MODE>, f);
    if (use_ws(MODE)) {
        cfg.gridDim = dim3((unsigned)ws_grid());
        cfg.blockDim = dim3(kWsThreads);
        cfg.dynamicSmemBytes = kWsDecWarps * kWsDecSmem;
        switch (ws_nr(f.nranks)) {
            case 2: ws_smem_attr(gtc_step_ws_kernel<CMP, HAS_G, MODE, 2>);
                    return cudaLaunchKernelEx(&cfg, gtc_step_ws_kernel<CMP, HAS_G, MODE, 2>, f);
            case 4: ws_smem_attr(gtc_step_ws_kernel<CMP, HAS_G, MODE, 4>);
                    return cudaLaunchKernelEx(&cfg, gtc_step_ws_kernel<CMP, HAS_G, MODE, 4>, f);
            default: ws_smem_attr(gtc_step_ws_kernel<CMP, HAS_G, MODE, 8>);
                     return cudaLaunchKernelEx(&cfg, gtc_step_ws_kernel<CMP, HAS_G, MODE, 8>, f);
        }
    }
    return cudaLaunchKernelEx(&cfg, gtc_step_ticket_kernel<CMP, HAS_G, MODE>, f);
}

template <int CMP, bool HAS_G>
cudaError_t launch_g(FusedStepParams& f, int mode, cudaStream_t s) {
    if (mode == GTC_ACCUM_MOMENTUM) return launch_t<CMP, HAS_G, GTC_ACCUM_MOMENTUM>(f, s);
    return mode == GTC_ACCUM_UPDATE ? launch_t<CMP, HAS_G, GTC_ACCUM_UPDATE>(f, s)
                                    : launch_t<CMP, HAS_G, GTC_ACCUM_WEIGHTS>(f, s);
}

template <int CMP, bool HAS_G, int MODE>
cudaError_t launch_group_t(const FusedStepParams* group, const FusedStepParams& h, int world, cudaStream_t s) {
    const long long Q = h.num_groups;
    if (grouped_kernel()) {
        const long long per_rank = Q * (kDecGroup + 1) + std::min<long long>(h.lag_groups, Q);
        gtc_step_p2p_group_kernel<CMP, HAS_G, MODE><<<(unsigned)(per_rank * world), kTileThreads, 0, s>>>(group, world);
    } else if (use_ws(MODE)) {
        const unsigned g = (unsigned)ws_grid(), b = kWsThreads, sm = kWsDecWarps * kWsDecSmem;
        switch (ws_nr(world)) {
            case 2: ws_smem_attr(gtc_step_ws_group_kernel<CMP, HAS_G, MODE, 2>);
                    gtc_step_ws_group_kernel<CMP, HAS_G, MODE, 2><<<g, b, sm, s>>>(group, world);
                    break;
            case 4: ws_smem_attr(gtc_step_ws_group_kernel<CMP, HAS_G, MODE, 4>);
                    gtc_step_ws_group_kernel<CMP, HAS_G, MODE, 4><<<g, b, sm, s>>>(group, world);
                    break;
            default: ws_smem_attr(gtc_step_ws_group_kernel<CMP, HAS_G, MODE, 8>);
                     gtc_step_ws_group_kernel<CMP, HAS_G, MODE, 8><<<g, b, sm, s>>>(group, world);
        }
    } else {
        const long long per_rank = h.enc.num_tiles + h.lag_tiles;
        gtc_step_ticket_group_kernel<CMP, HAS_G, MODE><<<(unsigned)(per_rank * world), kTileThreads, 0, s>>>(group,
                                                                                                          world);
    }
    return cudaGetLastError();
}

template <int CMP, bool HAS_G>
cudaError_t launch_group_g(const FusedStepParams* group, const FusedStepParams& h, int world, int mode,
                           cudaStream_t s) {
    if (mode == GTC_ACCUM_MOMENTUM) return launch_group_t<CMP, HAS_G, GTC_ACCUM_MOMENTUM>(group, h, world, s);
    return mode == GTC_ACCUM_UPDATE ? launch_group_t<CMP, HAS_G, GTC_ACCUM_UPDATE>(group, h, world, s)
                                    : launch_group_t<CMP, HAS_G, GTC_ACCUM_WEIGHTS>(group, h, world, s);
}

}  // namespace

// Decode lag in groups: about one wave of resident CTAs of one rank
// (GTC_FUSED_LAG, in tiles, overrides).
int step_p2p_lag_groups(int num_tiles, int ranks_per_device) {
    static std::once_flag once;
    static int wave = 592;
    std::call_once(once, [] {
        int dev = 0, sms = 0, per_sm = 0;
        if (cudaGetDevice(&dev) == cudaSuccess &&
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess &&
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(
                &per_sm, gtc_step_p2p_kernel<GTC_CMP_GT, true, GTC_ACCUM_WEIGHTS>, kTileThreads, 0) == cudaSuccess &&
            sms > 0 && per_sm > 0)
            wave = sms * per_sm;
    });
    int w = wave / std::max(1, ranks_per_device);
    if (const char* e = std::getenv("GTC_FUSED_LAG")) {  // read per step: tests vary it
        if (std::atoi(e) > 0) w = std::atoi(e);
    }
    const int groups = (num_tiles + kDecGroup - 1) / kDecGroup;
    const int lag = (w + kDecGroup) / (kDecGroup + 1);  // groups of G + 1 CTAs per wave
    return std::max(1, std::min(lag, groups));
}

// Ticketed kernel: decode lag in tiles, one wave of resident CTAs of one rank
// (GTC_FUSED_LAG, in tiles, overrides).
static int ticket_wave() {
    static std::once_flag once;
    static int wave = 592;
    std::call_once(once, [] {
        int dev = 0, sms = 0, per_sm = 0;
        if (cudaGetDevice(&dev) == cudaSuccess &&
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess &&
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(
                &per_sm, gtc_step_ticket_kernel<GTC_CMP_GT, true, GTC_ACCUM_WEIGHTS>, kTileThreads, 0) == cudaSuccess &&
            sms > 0 && per_sm > 0)
            wave = sms * per_sm;
    });
    return wave;
}

static int env_tiles(const char* name, int dflt) {  // read per step: tests vary them
    const char* e = std::getenv(name);
    return (e && e[0]) ? std::atoi(e) : dflt;
}

// Ticketed kernel lags (tiles).  Decode lag: the prefetch lag plus half a
// wave (about one HBM round trip of the step's progress), GTC_FUSED_LAG
// overrides.  Prefetch lag: one wave of resident CTAs of one rank,
// GTC_PREFETCH_LAG overrides (0 = no prefetch stage), always below the decode
// lag.
void step_p2p_lags(int num_tiles, int ranks_per_device, int* lag_tiles, int* lag_pf) {
    const int w = std::max(1, ticket_wave() / std::max(1, ranks_per_device));
    int lp = env_tiles("GTC_PREFETCH_LAG", w);
    const int la = std::max(1, env_tiles("GTC_FUSED_LAG", lp > 0 ? lp + w / 2 : w));
    lp = std::max(0, std::min(lp, la - 1));
    *lag_tiles = std::min(la, num_tiles + lp);
    *lag_pf = std::min(lp, num_tiles);
}

cudaError_t read_step_trace(unsigned long long* host, int max_entries) {
    const int n = max_entries < kStepTraceCtas * kStepTracePhases ? max_entries : kStepTraceCtas * kStepTracePhases;
    return cudaMemcpyFromSymbol(host, g_step_trace, sizeof(unsigned long long) * n);
}

cudaError_t launch_step_p2p(FusedStepParams& f, int cmp_mode, int accum_mode, cudaStream_t s) {
    if (f.enc.num_tiles == 0) return cudaSuccess;
    f.num_groups = (f.enc.num_tiles + kDecGroup - 1) / kDecGroup;
    if (f.lag_groups < 1) f.lag_groups = 1;
    if (cmp_mode == GTC_CMP_GE)
        return f.enc.g ? launch_g<GTC_CMP_GE, true>(f, accum_mode, s) : launch_g<GTC_CMP_GE, false>(f, accum_mode, s);
    return f.enc.g ? launch_g<GTC_CMP_GT, true>(f, accum_mode, s) : launch_g<GTC_CMP_GT, false>(f, accum_mode, s);
}

// `host` is rank 0's parameters (num_groups, lag_groups set by the caller,
// identical on every rank); HAS_G from rank 0 (all ranks pass grad or none).
cudaError_t launch_step_p2p_group(const FusedStepParams* group, const FusedStepParams& h, int world, int cmp_mode,
                                  int accum_mode, cudaStream_t s) {
    if (h.enc.num_tiles == 0) return cudaSuccess;
    const bool g = h.enc.g != nullptr;
    if (cmp_mode == GTC_CMP_GE)
        return g ? launch_group_g<GTC_CMP_GE, true>(group, h, world, accum_mode, s)
                 : launch_group_g<GTC_CMP_GE, false>(group, h, world, accum_mode, s);
    return g ? launch_group_g<GTC_CMP_GT, true>(group, h, world, accum_mode, s)
             : launch_group_g<GTC_CMP_GT, false>(group, h, world, accum_mode, s);
}

}  // namespace gtc
