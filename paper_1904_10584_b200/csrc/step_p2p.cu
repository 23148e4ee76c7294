// step_p2p.cu -- the whole GTC step for world > 1 (p2p exchange) as ONE kernel:
// encode (PAPER.md:222 steps 1-4), exchange ("Each worker communicates the
// sparse update to all other workers and conversely receives all sparse
// updates"), aggregate and apply ("The received sparse gradient updates are
// aggregated and weights are updated based on the aggregate").
//
// gtc_step_ticket_kernel: T + L CTAs of 256 threads, 5 per SM.  The CTA with
// ticket b (the order in which CTAs start, one atomicInc each) encodes tile b
// (rows a1-a5, b < T), pushes the tile's record (tag + first kPushCap stamped
// entries) to every peer with one bulk (TMA) copy each, and decodes tile
// b - L of every rank (rows a6-a8, L <= b < T + L) from the records pushed here.
// Its two halves' loads go out together, so the decode's local round trips
// overlap the encode's HBM stream.  Details and the measured alternatives
// (round 1's grouped encode/decode CTAs, pulls over NVLink, an L2 prefetch
// stage of the targets, a warp-specialized persistent kernel, 5-6 CTAs per
// SM): DESIGN.md §6, profiles/r02/ticket, profiles/r02/ws.
//
// Progress: a CTA only waits on tiles encoded by CTAs with lower tickets, on
// every rank, and an encode never waits, so the kernel completes whatever
// order the hardware dispatches CTAs in.  A wait longer than the context's
// timeout (30 s default) raises kFlagPeer (GTC_EPEER) on EVERY rank; once it
// is raised every later wait gives up at once.  The step is then incomplete:
// some tiles were applied on some ranks, so the replicas must be restored from
// a checkpoint (gtc.h, gtc_check).
//
// Buffer reuse: the segmented buffers and push regions alternate with the
// step parity.  A rank overwrites parity p at step e + 2 only after its step
// e + 1 kernel read every rank's step e + 1 tiles, which each rank writes
// after its own step e kernel (the one reading parity p) completed
// (griddepcontrol.wait).
//
// Algorithmic bytes per launch (local HBM): the encode's 12 n + 4 k + 8 T,
// this rank's entries and tags read back (4 k + 8 T), the peers' records
// landing here (16 (N-1) T + 4 (K - k)), 8 per touched element (target RMW);
// over NVLink: the records, 16 (N-1) T + 4 (K - k) per rank.
#include "gtc_internal.cuh"
#include "tile_encode.cuh"

#include <algorithm>
#include <cstdlib>
#include <mutex>

namespace gtc {
namespace {


// Opt-in phase trace (GTC_DECODE_TRACE=1): thread 0 of each of the first
// kStepTraceCtas tickets stamps %globaltimer at: start, every rank's tag of
// the decode tile seen, counts done, apply stores issued, end; and
// (SM id | decodes << 16 | decode-only << 17).
#ifdef GTC_STEP_TRACE
constexpr bool kTraceBuild = true;
#else
constexpr bool kTraceBuild = false;  // production builds carry no trace code (tools/step_trace.py)
#endif
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

__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

// A peer missed the timeout: GTC_EPEER on EVERY rank (system-scope atomics on
// each rank's flags), so no replica carries on unaware.
__device__ __forceinline__ void raise_peer_error(const FusedStepParams& f) {
    if (threadIdx.x < (unsigned)f.nranks) atomicOr_system(f.peer_flags[threadIdx.x], kFlagPeer);
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
    const bool dec = td >= 0 && td < T;
    const bool trace = kTraceBuild && f.trace && tid == 0 && trace_slot < kStepTraceCtas;
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
    // speculative entries per rank (S = 256 / N, host-computed): thread tid
    // reads entry sj of rank sm (a shift when S is a power of two)
    const int S = f.spec_window;
    const int sm = f.spec_shift >= 0 ? tid >> f.spec_shift : tid / S, sj = tid - sm * S;
    unsigned long long tagv = 0ull;
    unsigned spec = 0u;
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
    const unsigned stamp = f.stamp;  // entry_stamp(p.epoch), host-computed
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
            const int OV = __reduce_add_sync(0xffffffffu, lane < N ? max(0, s_k[lane] - S) : 0);
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
    const bool apply = dec && !failed;
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
        // only the thread's selected elements (a few per thread at 1 %): its
        // word's slot is its (round, warp) base + the words before it in the
        // thread's round (my_off packed one byte per round: <= 124 each)
        const unsigned offs = my_off[0] | (my_off[1] << 8) | (my_off[2] << 16) | (my_off[3] << 24);
        for (unsigned m = sel; m; m &= m - 1u) {
            const int bi = __ffs(m) - 1, j = bi >> 2;
            const unsigned o = s_scan[j * kTileWarps + warp] + ((offs >> (8 * j)) & 0xffu) +
                               __popc(sel & ((1u << bi) - 1u) & (0xfu << (4 * j)));
            const unsigned w = make_entry(stamp, (unsigned)(j * kTileThreads + tid) * 4u + (bi & 3), (neg >> bi) & 1u);
            st_relaxed_sys(dst + o, w);
            if (o < (unsigned)kPushCap) s_ent[o] = w;
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
    if (te >= 0 && tid == 0) {
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
    // fl(t + u) (R8) on the touched elements; MOMENTUM (M1) on every element.
    // Sparse warps (no lane with more than 2 touched float4s: most warps at 1 %)
    // visit only the touched float4s; denser ones the unrolled 4.
    auto store_one = [&](long long e0, float4 t, unsigned c) {
        const int cc[4] = {(int)(c & 0xffu) - 128, (int)((c >> 8) & 0xffu) - 128, (int)((c >> 16) & 0xffu) - 128,
                           (int)(c >> 24) - 128};
        if (e0 + 4 <= p.n) {
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
    const bool sparse_warp = MODE != GTC_ACCUM_MOMENTUM && !__any_sync(0xffffffffu, __popc(todo) > 2);
    if (apply && sparse_warp) {
        for (unsigned m = todo; m; m &= m - 1u) {
            const int h = __ffs(m) - 1;
            const float4 t = h == 0 ? tv[0] : h == 1 ? tv[1] : h == 2 ? tv[2] : tv[3];
            const unsigned c = h == 0 ? cw[0] : h == 1 ? cw[1] : h == 2 ? cw[2] : cw[3];
            store_one(db + 4ll * (tid + h * kTileThreads), t, c);
        }
    } else if (apply && todo) {
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

#ifndef GTC_TICKET_CTAS
#define GTC_TICKET_CTAS 5  // resident CTAs per SM: 48 registers (measured 4 / 5 / 6: DESIGN.md §6)
#endif
template <int CMP, bool HAS_G, int MODE>
__global__ void __launch_bounds__(kTileThreads, GTC_TICKET_CTAS) gtc_step_ticket_kernel(const FusedStepParams f) {
    const unsigned b = take_ticket(f.ticket, gridDim.x - 1u);
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

// CTAs per launch: T + L; the loopback group runs every rank's CTAs in one grid.
template <int CMP, bool HAS_G, int MODE>
cudaError_t launch_t(FusedStepParams& f, cudaStream_t s) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(f.enc.num_tiles + f.lag_tiles));
    cfg.blockDim = dim3(kTileThreads);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
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
    const long long per_rank = h.enc.num_tiles + h.lag_tiles;
    gtc_step_ticket_group_kernel<CMP, HAS_G, MODE><<<(unsigned)(per_rank * world), kTileThreads, 0, s>>>(group, world);
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

// Decode lag in tiles: 1.5 waves of resident CTAs of one rank (a wave is the
// tiles the other ranks encode concurrently; the extra half wave covers ranks
// that run behind: measured 0.5-3 waves, DESIGN.md §6, 1.5 is fastest at
// N = 2 and 4, rho = 1 % and 10 %).  GTC_FUSED_LAG (tiles) overrides; tests
// use short lags so that CTAs wait on tiles still being encoded.
int step_p2p_lag_tiles(int num_tiles, int ranks_per_device) {
    static std::once_flag once;
    static int wave = 740;  // 148 SMs x 5 CTAs, if the occupancy query fails
    std::call_once(once, [] {
        int dev = 0, sms = 0, per_sm = 0;
        if (cudaGetDevice(&dev) == cudaSuccess &&
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess &&
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(
                &per_sm, gtc_step_ticket_kernel<GTC_CMP_GT, true, GTC_ACCUM_WEIGHTS>, kTileThreads, 0) == cudaSuccess &&
            sms > 0 && per_sm > 0)
            wave = sms * per_sm;
    });
    int w = wave * 3 / 2 / std::max(1, ranks_per_device);
    if (const char* e = std::getenv("GTC_FUSED_LAG")) {  // read per step: tests vary it
        if (std::atoi(e) > 0) w = std::atoi(e);
    }
    return std::max(1, std::min(w, num_tiles));
}

cudaError_t read_step_trace(unsigned long long* host, int max_entries) {
    const int n = max_entries < kStepTraceCtas * kStepTracePhases ? max_entries : kStepTraceCtas * kStepTracePhases;
    return cudaMemcpyFromSymbol(host, g_step_trace, sizeof(unsigned long long) * n);
}

cudaError_t launch_step_p2p(FusedStepParams& f, int cmp_mode, int accum_mode, cudaStream_t s) {
    if (f.enc.num_tiles == 0) return cudaSuccess;
    if (f.lag_tiles < 1) f.lag_tiles = 1;
    if (cmp_mode == GTC_CMP_GE)
        return f.enc.g ? launch_g<GTC_CMP_GE, true>(f, accum_mode, s) : launch_g<GTC_CMP_GE, false>(f, accum_mode, s);
    return f.enc.g ? launch_g<GTC_CMP_GT, true>(f, accum_mode, s) : launch_g<GTC_CMP_GT, false>(f, accum_mode, s);
}

// `host` is rank 0's parameters (lag_tiles set by the caller, identical on
// every rank); HAS_G from rank 0 (all ranks pass grad or none).
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
