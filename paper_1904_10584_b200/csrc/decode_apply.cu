// decode_apply.cu -- GTC aggregate + apply for sm_100a (Sec. VI-A:
// "The received sparse gradient updates are aggregated and weights are updated
// based on the aggregate").
//
// Messages come in two layouts (gtc_internal.cuh): SEGMENTED (the hot path:
// words of tile t in slot t of a tile-major buffer, tag[t] = epoch<<32 |
// count; in p2p mode the peers' buffers are read straight over NVLink, and
// their stamped entries are turned back into words, entry_word) or
// CONTIGUOUS (NCCL all-gather, caller messages: words + per-tile offsets).
//
// gtc_decode_apply_kernel (any number of messages):
//   One CTA per tiles_per_cta consecutive tiles of kTile params; the grid is
//   one wave of resident CTAs.  Per CTA:
//   0. p2p: one thread per rank acquires (system scope) that rank's ready flag
//      for this step, raised by its last encode CTA -- the exchange is this
//      wait plus the NVLink reads below; no collective, no host sync;
//   1. counts c[0..span) in shared memory, int8 (|c| <= nmsg <= 64);
//   2. ordered per-message passes over the CTA's words of each message:
//      indices are unique within a message, so in one pass no two threads
//      touch the same count; a barrier separates passes.  Integer sums: the
//      result is independent of message order and needs no atomics
//      (deterministic by construction, R6).  The first words of the
//      first 8 messages are loaded into registers before the passes (one
//      memory round trip);
//   3. sparse apply (R8): only elements with c != 0 are read-modify-written,
//        u = fl((float)c * tau);  WEIGHTS: t = fmaf(alpha, u, t);  UPDATE: t = fl(t + u)
//      via a shared-memory list of the non-zero counts (per-thread 16-count
//      masks from 128-bit shared loads, one block scan), applied by all
//      threads: the target loads are independent, one memory round trip;
//   4. optional dense int8 counts dump (tests / parity only).
// gtc_apply_single_*_kernel (one message, no counts dump): indices are
//   unique, c = +-1 exactly on the message -- word-parallel, two round trips,
//   no shared memory, no barriers.
//
// Algorithmic HBM bytes per launch: 4 * (sum of message words) (read) +
// 8 * nmsg * num_tiles (tags) + 8 * |{i : c_i != 0}| (target RMW).
#include "gtc_internal.cuh"
#include "tile_encode.cuh"

#include <algorithm>
#include <cstdlib>

namespace gtc {
namespace {

constexpr unsigned kFullMask = 0xffffffffu;
constexpr int kPre = 2;                 // words per thread per message preloaded
constexpr int kPreMsgs = 8;             // messages whose first words are preloaded
constexpr int kBatch = 8;               // words loaded per thread before their count updates
constexpr int kMaxTouched = 2048;       // non-zero counts applied through the list (else dense fallback)
constexpr int kChunksPerThread = kDecMaxTilesPerCta * (kTile / 16) / kDecThreads;

// Opt-in phase trace of the counting decode (GTC_DECODE_TRACE=1): thread 0 of
// each of the first kTraceCtas CTAs stamps %globaltimer at kTracePhases
// phase boundaries (start, peers ready, tags, counts, list, end).
constexpr int kTraceCtas = 4096;
constexpr int kTracePhases = 6;
__device__ unsigned long long g_trace[kTraceCtas * kTracePhases];

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* a) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(a) : "memory");
    return v;
}

__device__ __forceinline__ unsigned long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// p2p: wait (acquire, system scope) until rank m has published this step's
// message (ready = step).  A peer can be at most one step ahead (its next
// decode waits for this rank), hence >=.  False on timeout.
__device__ __forceinline__ bool wait_ready(const DecodeParams& p, int m) {
    unsigned long long v = ld_acquire_sys(p.ready[m]);
    if (v >= p.step) return true;
    const unsigned long long t0 = globaltimer_ns();
    while (v < p.step) {
        if (globaltimer_ns() - t0 > p.timeout_ns) return false;
        __nanosleep(64);
        v = ld_acquire_sys(p.ready[m]);
    }
    return true;
}

// Count of tile t of a segmented message (after wait_ready in p2p mode).
__device__ __forceinline__ int seg_count(const DecodeParams& p, int m, long long t) {
    return (int)(__ldcg(p.tags[m] + t) & 0xffffffffull);
}

template <int MODE>
__device__ __forceinline__ void apply_one(const DecodeParams& p, long long gi, int c, float t) {
    const float u = __fmul_rn((float)c, p.tau);
    p.target[gi] = (MODE == GTC_ACCUM_WEIGHTS) ? __fmaf_rn(p.alpha, u, t) : __fadd_rn(t, u);
}

// The listed non-zero counts, kApplyBatch independent target loads per
// thread before their stores (the listed indices are distinct).
constexpr int kApplyBatch = 4;
template <int MODE, typename GlobalOf>
__device__ __forceinline__ void apply_list(const DecodeParams& p, const unsigned short* list, const signed char* cnt,
                                           unsigned total, const GlobalOf& global_of) {
    for (unsigned i0 = threadIdx.x; i0 < total; i0 += kApplyBatch * kDecThreads) {
        long long gi[kApplyBatch];
        int c[kApplyBatch];
        float t[kApplyBatch];
#pragma unroll
        for (int u = 0; u < kApplyBatch; ++u) {
            const unsigned i = i0 + u * kDecThreads;
            gi[u] = -1;
            if (i < total) {
                const int local = list[i];
                const long long g = global_of(local);
                if (g < p.n) {
                    gi[u] = g;
                    c[u] = cnt[local];
                    t[u] = p.target[g];
                }
            }
        }
#pragma unroll
        for (int u = 0; u < kApplyBatch; ++u)
            if (gi[u] >= 0) apply_one<MODE>(p, gi[u], c[u], t[u]);
    }
}

// buf = fl(fl(mu * buf) + fl(c * tau)); w = fmaf(alpha, buf, w)  (M1)
__device__ __forceinline__ void momentum_one(float& w, float& b, int c, const DecodeParams& p) {
    const float u = __fmul_rn((float)c, p.tau);
    b = __fadd_rn(__fmul_rn(p.mu, b), u);
    w = __fmaf_rn(p.alpha, b, w);
}

__device__ __forceinline__ int count_byte(int packed, int e) {
    return (int)(signed char)((unsigned)packed >> (8 * e));
}

// every element of the CTA's tiles (slot i = tile t0 + i * G) of target / buf,
// counts in shared memory (4 int8 per int), kU float4 of each in flight per thread
__device__ __forceinline__ void dense_momentum(const DecodeParams& p, const int* s_cnt_q, int t0, int G, int nt) {
    constexpr int kU = 4;
    constexpr int kV = kTile / 4;  // float4 per tile
    const int nv = nt * kV;
    float4* w4 = reinterpret_cast<float4*>(p.target);
    float4* b4 = reinterpret_cast<float4*>(p.buf);
    for (int v0 = threadIdx.x; v0 < nv; v0 += kU * kDecThreads) {
        float4 w[kU], b[kU];
        long long e0[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const int v = v0 + u * kDecThreads;
            e0[u] = v < nv ? ((long long)t0 + (long long)(v / kV) * G) * kTile + 4ll * (v % kV) : p.n;
            if (e0[u] + 4 <= p.n) {
                w[u] = __ldcs(w4 + e0[u] / 4);
                b[u] = __ldcs(b4 + e0[u] / 4);
            }
        }
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            if (e0[u] >= p.n) continue;
            const int packed = s_cnt_q[v0 + u * kDecThreads];
            if (e0[u] + 4 <= p.n) {
                momentum_one(w[u].x, b[u].x, count_byte(packed, 0), p);
                momentum_one(w[u].y, b[u].y, count_byte(packed, 1), p);
                momentum_one(w[u].z, b[u].z, count_byte(packed, 2), p);
                momentum_one(w[u].w, b[u].w, count_byte(packed, 3), p);
                __stcs(w4 + e0[u] / 4, w[u]);
                __stcs(b4 + e0[u] / 4, b[u]);
            } else {
                for (int e = 0; e0[u] + e < p.n; ++e)
                    momentum_one(p.target[e0[u] + e], p.buf[e0[u] + e], count_byte(packed, e), p);
            }
        }
    }
}

template <int MODE, bool SEG>
__global__ void __launch_bounds__(kDecThreads) gtc_decode_apply_kernel(const DecodeParams p) {
    // dynamic shared memory: int8 counts [tiles_per_cta * kTile] | per message
    // the words before each of its tiles [nmsg][tiles_per_cta + 1] | contiguous
    // messages: the first word of each tile [nmsg][tiles_per_cta]
    extern __shared__ int4 s_cnt4[];
    const int npre = p.tiles_per_cta + 1;
    int* s_pre_flat = reinterpret_cast<int*>(reinterpret_cast<signed char*>(s_cnt4) + p.tiles_per_cta * kTile);
    int* s_tb_flat = s_pre_flat + p.nmsg * npre;
    auto s_pre = [&](int m, int i) -> int& { return s_pre_flat[m * npre + i]; };
    auto s_tb = [&](int m, int i) -> int& { return s_tb_flat[m * p.tiles_per_cta + i]; };
    __shared__ unsigned s_warp[kDecThreads / 32];
    __shared__ unsigned short s_list[kMaxTouched];  // local indices with c != 0 (< 32768)
    __shared__ int s_abort;

    const bool trace = p.trace && threadIdx.x == 0 && blockIdx.x < kTraceCtas;
    auto stamp = [&](int ph) {
        if (trace) g_trace[blockIdx.x * kTracePhases + ph] = globaltimer_ns();
    };
    stamp(0);
    // programmatic dependent launch: wait for the previous kernel (the encode)
    // and its memory before touching anything
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;");
    if (p.publish && blockIdx.x == 0 && threadIdx.x == 0) {
        // p2p: every store of this rank's encode precedes this kernel (stream
        // order); make them visible at system scope, then tell the peers
        __threadfence_system();
        asm volatile("st.release.sys.global.u64 [%0], %1;" :: "l"(p.publish), "l"(p.step) : "memory");
    }
    if (*p.flags & (kFlagCapacity | kFlagCorrupt)) return;  // nothing is applied

    signed char* s_cnt = reinterpret_cast<signed char*>(s_cnt4);
    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int warp = tid >> 5;
    // the CTA's tiles are strided by the grid (slot i holds tile t0 + i * G):
    // message density varies by parameter segment, and striding spreads the
    // dense segments' words evenly over the CTAs
    const int G = (int)gridDim.x;
    const int t0 = (int)blockIdx.x;
    const int nt = min(p.tiles_per_cta, (p.num_tiles - t0 + G - 1) / G);
    const float inv_g = 1.0f / (float)G;
    auto tile_of = [&](int i) -> long long { return (long long)t0 + (long long)i * G; };
    // local count index (slot * kTile + offset) <-> parameter index
    auto local_of = [&](unsigned idx) -> int {
        const int slot = __float2int_rn((float)((int)(idx / kTile) - t0) * inv_g);  // exact: a multiple of G
        return slot * kTile + (int)(idx & (kTile - 1));
    };
    auto global_of = [&](int local) -> long long {
        return tile_of(local / kTile) * kTile + (local & (kTile - 1));
    };
    const int nq = nt * (kTile / 16);  // int4 chunks of 16 counts

    if (tid == 0) s_abort = 0;
    for (int q = tid; q < nq; q += kDecThreads) s_cnt4[q] = make_int4(0, 0, 0, 0);
    __syncthreads();
    if (SEG) {
        // p2p: this is where the exchange waits -- one thread per peer acquires
        // its ready flag; the barrier extends the acquire to the whole CTA
        if (p.wait) {
            for (int m = tid; m < p.nmsg; m += kDecThreads)
                if (!wait_ready(p, m)) s_abort = 1;
            __syncthreads();
            stamp(1);
            if (s_abort) {
                // every rank learns of the timeout (gtc_check on any rank
                // reports GTC_EPEER); this CTA applies nothing
                for (int m = tid; m < p.nmsg; m += kDecThreads) atomicOr_system(p.peer_flags[m], kFlagPeer);
                return;
            }
        }
        // per (message, tile) counts
        for (int idx = tid; idx < p.nmsg * nt; idx += kDecThreads) {
            const int m = idx / nt, i = idx - m * nt;
            s_pre(m, i + 1) = seg_count(p, m, tile_of(i));
        }
        __syncthreads();
        for (int m = tid; m < p.nmsg; m += kDecThreads) {  // exclusive prefix over the CTA's tiles
            s_pre(m, 0) = 0;
            for (int i = 1; i <= nt; ++i) s_pre(m, i) += s_pre(m, i - 1);
        }
        stamp(2);
    } else {
        // contiguous messages: each tile's words start at off[m][tile]
        for (int idx = tid; idx < p.nmsg * nt; idx += kDecThreads) {
            const int m = idx / nt, i = idx - m * nt;
            const int b = __ldg(p.off[m] + tile_of(i));
            s_tb(m, i) = b;
            s_pre(m, i + 1) = __ldg(p.off[m] + tile_of(i) + 1) - b;
        }
        __syncthreads();
        for (int m = tid; m < p.nmsg; m += kDecThreads) {
            s_pre(m, 0) = 0;
            for (int i = 1; i <= nt; ++i) s_pre(m, i) += s_pre(m, i - 1);
        }
    }
    __syncthreads();

    // the f-th word of message m among this CTA's words
    auto word_at = [&](int m, int f) -> unsigned {
        int i = 0;
        while (i + 1 < nt && f >= s_pre(m, i + 1)) ++i;
        if (SEG) {
            const unsigned e = __ldcg(p.seg[m] + tile_of(i) * kTile + (f - s_pre(m, i)));
            return p.stamped ? entry_word(e, tile_of(i)) : e;
        }
        return __ldg(p.words[m] + s_tb(m, i) + (f - s_pre(m, i)));
    };

    // words [from, len) of message m into the counts, kBatch independent loads
    // per thread before their shared-memory updates (dense messages would
    // otherwise pay one memory round trip per word per thread)
    auto count_words = [&](int m, int from, int len) {
        for (int f0 = from + tid; f0 < len; f0 += kBatch * kDecThreads) {
            unsigned w[kBatch];
#pragma unroll
            for (int u = 0; u < kBatch; ++u) {
                const int f = f0 + u * kDecThreads;
                w[u] = f < len ? word_at(m, f) : 0u;
            }
#pragma unroll
            for (int u = 0; u < kBatch; ++u) {
                if (f0 + u * kDecThreads < len) {
                    const int local = local_of(w[u] >> 1);
                    s_cnt[local] = (signed char)(s_cnt[local] + ((w[u] & 1u) ? -1 : 1));
                }
            }
        }
    };

    // preload the first words of the first messages (one memory round trip)
    unsigned pre[kPreMsgs][kPre];
#pragma unroll
    for (int m = 0; m < kPreMsgs; ++m) {
#pragma unroll
        for (int u = 0; u < kPre; ++u) {
            pre[m][u] = 0u;
            if (m < p.nmsg) {
                const int f = u * kDecThreads + tid;
                if (f < s_pre(m, nt)) pre[m][u] = word_at(m, f);
            }
        }
    }

    // ordered per-message passes
#pragma unroll
    for (int m = 0; m < kPreMsgs; ++m) {
        if (m >= p.nmsg) break;
        const int len = s_pre(m, nt);
#pragma unroll
        for (int u = 0; u < kPre; ++u) {
            if (u * kDecThreads + tid < len) {
                const unsigned word = pre[m][u];
                const int local = local_of(word >> 1);
                s_cnt[local] = (signed char)(s_cnt[local] + ((word & 1u) ? -1 : 1));
            }
        }
        count_words(m, kPre * kDecThreads, len);
        __syncthreads();
    }
    for (int m = kPreMsgs; m < p.nmsg; ++m) {
        count_words(m, 0, s_pre(m, nt));
        __syncthreads();
    }

    stamp(3);
    // optional dense counts dump (tests / parity)
    if (p.counts_out) {
        for (int q = tid; q < nq; q += kDecThreads) {
            const int4 packed = s_cnt4[q];
            const long long i0 = global_of(q * 16);
            if (i0 + 16 <= p.n) {
                reinterpret_cast<int4*>(p.counts_out + i0)[0] = packed;
            } else {
                const signed char* c = reinterpret_cast<const signed char*>(&packed);
                for (int e = 0; e < 16; ++e)
                    if (i0 + e < p.n) p.counts_out[i0 + e] = c[e];
            }
        }
    }

    if constexpr (MODE == GTC_ACCUM_MOMENTUM) {
        // SGD-momentum (M1): dense over the CTA's elements -- every momentum
        // decays -- with 4 float4 of target and of buf in flight per thread
        dense_momentum(p, reinterpret_cast<const int*>(s_cnt), t0, G, nt);
        stamp(5);
        return;
    }

    // sparse apply through a list of the non-zero counts
    unsigned nz[kChunksPerThread];
    unsigned my = 0;
#pragma unroll
    for (int u = 0; u < kChunksPerThread; ++u) {
        const int q = u * kDecThreads + tid;
        unsigned msk = 0;
        if (q < nq) {
            const int4 packed = s_cnt4[q];
            const unsigned x[4] = {(unsigned)packed.x, (unsigned)packed.y, (unsigned)packed.z, (unsigned)packed.w};
#pragma unroll
            for (int h = 0; h < 4; ++h) {
#pragma unroll
                for (int b = 0; b < 4; ++b)
                    msk |= (((x[h] >> (8 * b)) & 0xffu) != 0u ? 1u : 0u) << (4 * h + b);
            }
        }
        nz[u] = msk;
        my += __popc(msk);
    }
    unsigned incl = my;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned y = __shfl_up_sync(kFullMask, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    unsigned wbase = 0, total = 0;
#pragma unroll
    for (int w = 0; w < kDecThreads / 32; ++w) {
        const unsigned v = s_warp[w];
        wbase += (w < warp) ? v : 0u;
        total += v;
    }
    stamp(4);
    if (total <= (unsigned)kMaxTouched) {
        unsigned pos = wbase + incl - my;
#pragma unroll
        for (int u = 0; u < kChunksPerThread; ++u) {
            unsigned msk = nz[u];
            const int q = u * kDecThreads + tid;
            while (msk) {
                const int b = __ffs(msk) - 1;
                msk &= msk - 1;
                s_list[pos++] = (unsigned short)(q * 16 + b);
            }
        }
        __syncthreads();
        apply_list<MODE>(p, s_list, s_cnt, total, global_of);
    } else {
        // dense CTA: one list per round u of 256 chunks (4096 counts), each
        // built by a block scan and applied with independent loads; a round
        // that alone overflows the list is applied per thread
        __syncthreads();  // everyone has read s_warp
#pragma unroll
        for (int u = 0; u < kChunksPerThread; ++u) {
            const unsigned msk_u = nz[u];
            const unsigned my_u = __popc(msk_u);
            unsigned inc = my_u;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned y = __shfl_up_sync(kFullMask, inc, o);
                if (lane >= o) inc += y;
            }
            if (lane == 31) s_warp[warp] = inc;
            __syncthreads();
            unsigned wb = 0, tot = 0;
#pragma unroll
            for (int w = 0; w < kDecThreads / 32; ++w) {
                const unsigned v = s_warp[w];
                wb += (w < warp) ? v : 0u;
                tot += v;
            }
            const int q = u * kDecThreads + tid;
            if (tot <= (unsigned)kMaxTouched) {
                unsigned pos = wb + inc - my_u;
                unsigned msk = msk_u;
                while (msk) {
                    const int b = __ffs(msk) - 1;
                    msk &= msk - 1;
                    s_list[pos++] = (unsigned short)(q * 16 + b);
                }
                __syncthreads();
                apply_list<MODE>(p, s_list, s_cnt, tot, global_of);
            } else {
                unsigned msk = msk_u;
                while (msk) {
                    const int b = __ffs(msk) - 1;
                    msk &= msk - 1;
                    const int local = q * 16 + b;
                    const long long gi = global_of(local);
                    if (gi < p.n) apply_one<MODE>(p, gi, s_cnt[local], p.target[gi]);
                }
            }
            __syncthreads();  // s_warp / s_list are reused by the next round
        }
    }
    stamp(5);
}

// One message (world == 1, or one simulated worker): indices are unique, so
// c[i] = +-1 exactly on the message's indices and 0 elsewhere; the aggregate
// needs no counts.  fl(+-1 * tau) = +-tau exactly, so the arithmetic is the
// general kernel's (R8).  Loads are batched (4 per thread) before the stores.
constexpr int kSingleThreads = 256;
constexpr int kSingleBatch = 4;

template <int MODE>
__device__ __forceinline__ void apply_words(const DecodeParams& p, const unsigned* w, int cnt, int lane,
                                            int stride) {
    for (int j0 = 0; j0 < cnt; j0 += stride * kSingleBatch) {
        unsigned wd[kSingleBatch];
        float t[kSingleBatch];
#pragma unroll
        for (int u = 0; u < kSingleBatch; ++u) {
            const int j = j0 + u * stride + lane;
            wd[u] = j < cnt ? __ldcg(w + j) : 0u;
        }
#pragma unroll
        for (int u = 0; u < kSingleBatch; ++u)
            if (j0 + u * stride + lane < cnt) t[u] = p.target[wd[u] >> 1];
#pragma unroll
        for (int u = 0; u < kSingleBatch; ++u) {
            if (j0 + u * stride + lane < cnt) {
                const float q = (wd[u] & 1u) ? -p.tau : p.tau;  // fl(c * tau) for c = -1 / +1
                p.target[wd[u] >> 1] = (MODE == GTC_ACCUM_WEIGHTS) ? __fmaf_rn(p.alpha, q, t[u])
                                                                   : __fadd_rn(t[u], q);
            }
        }
    }
}

// segmented: one warp per tile
template <int MODE>
__global__ void __launch_bounds__(kSingleThreads) gtc_apply_single_seg_kernel(const DecodeParams p) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;");
    if (*p.flags & (kFlagCapacity | kFlagCorrupt)) return;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long long stride = (long long)gridDim.x * (kSingleThreads / 32);
    for (long long t = (long long)blockIdx.x * (kSingleThreads / 32) + warp; t < p.num_tiles; t += stride) {
        const int cnt = (int)(__ldcg(p.tags[0] + t) & 0xffffffffull);
        if (cnt) apply_words<MODE>(p, p.seg[0] + t * kTile, cnt, lane, 32);
    }
}

// contiguous: word-parallel over the whole message (length from off[num_tiles])
template <int MODE>
__global__ void __launch_bounds__(kSingleThreads) gtc_apply_single_kernel(const DecodeParams p) {
    if (*p.flags & (kFlagCapacity | kFlagCorrupt)) return;
    const long long k = __ldg(p.off[0] + p.num_tiles);
    const long long per = (long long)kSingleThreads * kSingleBatch;
    for (long long j0 = (long long)blockIdx.x * per; j0 < k; j0 += (long long)gridDim.x * per)
        apply_words<MODE>(p, p.words[0] + j0, (int)min(per, k - j0), threadIdx.x, kSingleThreads);
}

// Tile offsets of caller-supplied messages (gtc_decode_apply_msgs): for every
// message m and tile t, off[m][t] = number of words with index < t*kTile
// (lower bound by binary search), off[m][num_tiles] = k; and validation of
// every word (index < n, strictly ascending) into kFlagCorrupt.
__global__ void gtc_tile_bounds_kernel(const BoundsParams p) {
    const int m = blockIdx.y;
    const unsigned* w = p.words[m];
    const long long k = p.k[m];
    const long long stride = (long long)gridDim.x * blockDim.x;
    const long long start = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    for (long long t = start; t <= p.num_tiles; t += stride) {
        long long v;
        if (t == p.num_tiles) {
            v = k;
        } else {
            const unsigned long long key = (unsigned long long)t * kTile;
            long long lo = 0, hi = k;
            while (lo < hi) {
                const long long mid = (lo + hi) >> 1;
                if ((unsigned long long)(__ldg(w + mid) >> 1) < key) lo = mid + 1; else hi = mid;
            }
            v = lo;
        }
        p.off[m][t] = (int)v;
    }
    bool bad = false;
    for (long long j = start; j < k; j += stride) {
        const unsigned long long idx = __ldg(w + j) >> 1;
        if ((long long)idx >= p.n) bad = true;
        if (j > 0 && (unsigned long long)(__ldg(w + j - 1) >> 1) >= idx) bad = true;
    }
    if (bad) atomicOr(p.flags, kFlagCorrupt);
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

template <int MODE, bool SEG>
cudaError_t launch_general(const DecodeParams& p_in, cudaStream_t s) {
    auto kern = gtc_decode_apply_kernel<MODE, SEG>;
    static int resident[GTC_MAX_MSGS + 1][kDecMaxTilesPerCta + 1] = {{0}};
    auto dyn_smem = [&](int tpc) {
        return (size_t)tpc * kTile + sizeof(int) * (size_t)p_in.nmsg * (2 * tpc + 1);
    };
    static cudaError_t attr = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                   kDecMaxTilesPerCta * kTile + sizeof(int) * GTC_MAX_MSGS *
                                                   (2 * kDecMaxTilesPerCta + 1));
    if (attr != cudaSuccess) return attr;
    DecodeParams p = p_in;
    const int sms = sm_count();
    const int range = p.num_tiles;
    if (range <= 0) return cudaSuccess;
    // smallest tiles_per_cta whose grid fits in one wave of resident CTAs
    // (GTC_DECODE_TPC overrides, for measurement)
    static int forced = -1;
    if (forced < 0) {
        const char* e = std::getenv("GTC_DECODE_TPC");
        forced = e ? std::atoi(e) : 0;
    }
    int tpc = 1;
    for (; tpc <= kDecMaxTilesPerCta; ++tpc) {
        int& res = resident[p.nmsg][tpc];
        if (res == 0) {
            int r = 0;
            if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&r, kern, kDecThreads, dyn_smem(tpc)) != cudaSuccess)
                r = 1;
            res = r < 1 ? 1 : r;
        }
        if ((long long)(range + tpc - 1) / tpc <= (long long)res * sms) break;
    }
    if (tpc > kDecMaxTilesPerCta) tpc = kDecMaxTilesPerCta;
    if (forced > 0) tpc = forced < kDecMaxTilesPerCta ? forced : kDecMaxTilesPerCta;
    p.tiles_per_cta = tpc;
    const int grid = (range + tpc - 1) / tpc;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(kDecThreads);
    cfg.dynamicSmemBytes = dyn_smem(tpc);
    cfg.stream = s;
    cudaLaunchAttribute la[1];
    la[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    la[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = la;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, p);
}

// GTC_DECODE_GENERAL=1 routes one-message decodes through the counting
// kernel too (for measurement).
bool force_general() {
    static int v = -1;
    if (v < 0) {
        const char* e = std::getenv("GTC_DECODE_GENERAL");
        v = (e && e[0] == '1') ? 1 : 0;
    }
    return v == 1;
}

template <int MODE>
cudaError_t launch_mode(const DecodeParams& p, cudaStream_t s) {
    if (MODE != GTC_ACCUM_MOMENTUM && p.nmsg == 1 && p.counts_out == nullptr && !p.wait && !force_general()) {
        if (p.segmented) {
            const int grid = (int)std::min<long long>((p.num_tiles + 7) / 8, (long long)sm_count() * 8);
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3((unsigned)grid);
            cfg.blockDim = dim3(kSingleThreads);
            cfg.stream = s;
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
            cfg.attrs = attr;
            cfg.numAttrs = 1;
            return cudaLaunchKernelEx(&cfg, gtc_apply_single_seg_kernel<MODE>, p);
        } else {
            gtc_apply_single_kernel<MODE><<<sm_count() * 8, kSingleThreads, 0, s>>>(p);
        }
        return cudaGetLastError();
    }
    return p.segmented ? launch_general<MODE, true>(p, s) : launch_general<MODE, false>(p, s);
}

}  // namespace

cudaError_t launch_decode_apply(const DecodeParams& p, int accum_mode, cudaStream_t s) {
    if (p.num_tiles == 0) return cudaSuccess;
    if (accum_mode == GTC_ACCUM_MOMENTUM) return launch_mode<GTC_ACCUM_MOMENTUM>(p, s);
    return accum_mode == GTC_ACCUM_UPDATE ? launch_mode<GTC_ACCUM_UPDATE>(p, s) : launch_mode<GTC_ACCUM_WEIGHTS>(p, s);
}

cudaError_t read_decode_trace(unsigned long long* host, int max_entries) {
    const int n = max_entries < kTraceCtas * kTracePhases ? max_entries : kTraceCtas * kTracePhases;
    return cudaMemcpyFromSymbol(host, g_trace, sizeof(unsigned long long) * n);
}

bool decode_trace_enabled() {
    static int v = -1;
    if (v < 0) {
        const char* e = std::getenv("GTC_DECODE_TRACE");
        v = (e && e[0] == '1') ? 1 : 0;
    }
    return v == 1;
}

cudaError_t launch_tile_bounds(const BoundsParams& p, cudaStream_t s) {
    if (p.nmsg == 0) return cudaSuccess;
    long long work = p.num_tiles + 1;
    for (int m = 0; m < p.nmsg; ++m) work = work > p.k[m] ? work : p.k[m];
    long long blocks = (work + 255) / 256;
    if (blocks > 1184) blocks = 1184;  // 8 per SM on 148 SMs, grid-stride beyond
    dim3 grid((unsigned)blocks, (unsigned)p.nmsg);
    gtc_tile_bounds_kernel<<<grid, 256, 0, s>>>(p);
    return cudaGetLastError();
}

}  // namespace gtc
