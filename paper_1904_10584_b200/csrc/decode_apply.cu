// decode_apply.cu -- GTC aggregate + apply for sm_100a (Sec. VI-A:
// "The received sparse gradient updates are aggregated and weights are updated
// based on the aggregate").
//
// One CTA per tiles_per_cta consecutive tiles of kTile params (the encode
// tiling, so every message's slice for the CTA is [off[t0], off[t0+nt]) and its
// reads are coalesced); tiles_per_cta is chosen so the grid is about one wave
// of 8 CTAs per SM.
//   1. counts c[0..kTile) in shared memory, int8 (|c| <= nmsg <= 64),
//   2. ordered per-message passes: indices are unique within a message, so in
//      one pass no two threads touch the same count; a barrier separates
//      passes.  Integer sums: the result is independent of message order and
//      needs no atomics (deterministic by construction, R6),
//   3. sparse apply (R8): only elements with c != 0 are read-modify-written:
//        u = fl((float)c * tau);  WEIGHTS: t = fmaf(alpha, u, t);  UPDATE: t = fl(t + u)
//      the non-zero counts of the CTA are compacted into a shared-memory list
//      (per-thread 16-count masks from 128-bit shared loads, one block scan),
//      then the list is applied by all threads: the target loads are all
//      independent, one memory round trip per CTA.
//   The first words of the first 8 messages are loaded into registers before
//   the ordered passes, so the word reads also cost one round trip.
//   4. optional dense int8 counts dump (tests / parity only).
//
// Algorithmic HBM bytes per launch: 4 * (sum of message words) (read) +
// 4 * nmsg * (num_tiles + 1) (tile offsets) + 8 * |{i : c_i != 0}| (target RMW).
#include "gtc_internal.cuh"

namespace gtc {
namespace {

constexpr unsigned kFullMask = 0xffffffffu;
constexpr int kPre = 2;                 // words per thread per message preloaded
constexpr int kPreMsgs = 8;             // messages whose first words are preloaded
constexpr int kMaxTouched = 4096;       // non-zero counts applied through the list
constexpr int kChunksPerThread = kDecMaxTilesPerCta * (kTile / 16) / kDecThreads;

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* a) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(a) : "memory");
    return v;
}

__device__ __forceinline__ unsigned long long ld_relaxed_sys(const unsigned long long* a) {
    unsigned long long v;
    asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(a) : "memory");
    return v;
}

__device__ __forceinline__ unsigned long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

constexpr unsigned long long kPeerTimeoutNs = 30ull * 1000 * 1000 * 1000;

// p2p exchange gate (thread 0 of every CTA): wait until every peer has
// published this step's message (ready[r] >= epoch: a peer can be at most one
// step ahead, because its next decode waits for this rank's next signal),
// then fold every rank's header flags.  Returns the flags; a capacity
// overflow anywhere or a timed-out peer means nothing is applied anywhere.
__device__ unsigned long long p2p_gate(const DecodeParams& p) {
    unsigned long long f = 0;
    const unsigned long long t0 = globaltimer_ns();
    for (int r = 0; r < p.nmsg; ++r) {
        if (r == p.self) continue;
        while (ld_acquire_sys(&p.ready[r]) < p.epoch) {
            if (globaltimer_ns() - t0 > kPeerTimeoutNs) {
                f |= kFlagPeer;
                break;
            }
            __nanosleep(64);
        }
        if (f & kFlagPeer) break;
    }
    if (!(f & kFlagPeer))
        for (int r = 0; r < p.nmsg; ++r) f |= ld_relaxed_sys(&p.hdr[r]->flags);
    return f;
}

template <int MODE>
__global__ void __launch_bounds__(kDecThreads) gtc_decode_apply_kernel(const DecodeParams p) {
    extern __shared__ int4 s_cnt4[];  // tiles_per_cta * kTile int8 counts
    __shared__ int s_rng[GTC_MAX_MSGS][2];
    __shared__ unsigned s_warp[kDecThreads / 32];
    __shared__ unsigned short s_list[kMaxTouched];  // local indices with c != 0 (< 32768)
    __shared__ unsigned long long s_gate;

    if (*p.flags & (kFlagCapacity | kFlagCorrupt)) return;  // nothing is applied
    if (p.ready) {
        if (threadIdx.x == 0) {
            const unsigned long long f = p2p_gate(p);
            s_gate = f;
            if (blockIdx.x == 0 && (f & (kFlagNonFinite | kFlagCapacity | kFlagPeer)))
                atomicOr(p.local_flags, f & (kFlagNonFinite | kFlagCapacity | kFlagPeer));
        }
        __syncthreads();
        if (s_gate & (kFlagCapacity | kFlagPeer)) return;
    }

    signed char* s_cnt = reinterpret_cast<signed char*>(s_cnt4);
    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int warp = tid >> 5;
    const int t0 = blockIdx.x * p.tiles_per_cta;
    const int nt = min(p.tiles_per_cta, p.num_tiles - t0);
    const long long base = (long long)t0 * kTile;
    const int span = nt * kTile;
    const int nq = span / 16;  // int4 chunks of 16 counts

    for (int q = tid; q < nq; q += kDecThreads) s_cnt4[q] = make_int4(0, 0, 0, 0);
    for (int m = tid; m < p.nmsg; m += kDecThreads) {
        s_rng[m][0] = __ldg(p.m.off[m] + t0);
        s_rng[m][1] = __ldg(p.m.off[m] + t0 + nt);
    }
    __syncthreads();

    // preload the first words of the first messages (one memory round trip)
    unsigned pre[kPreMsgs][kPre];
#pragma unroll
    for (int m = 0; m < kPreMsgs; ++m) {
#pragma unroll
        for (int u = 0; u < kPre; ++u) {
            if (m < p.nmsg) {
                const int j = s_rng[m][0] + u * kDecThreads + tid;
                pre[m][u] = j < s_rng[m][1] ? __ldg(p.m.words[m] + j) : 0u;
            }
        }
    }

    // ordered per-message passes; indices are unique within a message, so no
    // two threads of one pass touch the same count (no atomics)
#pragma unroll
    for (int m = 0; m < kPreMsgs; ++m) {
        if (m >= p.nmsg) break;
        const int b = s_rng[m][0], e = s_rng[m][1];
#pragma unroll
        for (int u = 0; u < kPre; ++u) {
            if (b + u * kDecThreads + tid < e) {
                const unsigned word = pre[m][u];
                const int local = (int)((word >> 1) - (unsigned)base);
                s_cnt[local] = (signed char)(s_cnt[local] + ((word & 1u) ? -1 : 1));
            }
        }
        const unsigned* w = p.m.words[m];
        for (int j = b + kPre * kDecThreads + tid; j < e; j += kDecThreads) {
            const unsigned word = __ldg(w + j);
            const int local = (int)((word >> 1) - (unsigned)base);
            s_cnt[local] = (signed char)(s_cnt[local] + ((word & 1u) ? -1 : 1));
        }
        __syncthreads();
    }
    for (int m = kPreMsgs; m < p.nmsg; ++m) {
        const unsigned* w = p.m.words[m];
        const int e = s_rng[m][1];
        for (int j = s_rng[m][0] + tid; j < e; j += kDecThreads) {
            const unsigned word = __ldg(w + j);
            const int local = (int)((word >> 1) - (unsigned)base);
            s_cnt[local] = (signed char)(s_cnt[local] + ((word & 1u) ? -1 : 1));
        }
        __syncthreads();
    }

    // optional dense counts dump (tests / parity)
    if (p.counts_out) {
        for (int q = tid; q < nq; q += kDecThreads) {
            const int4 packed = s_cnt4[q];
            const long long i0 = base + (long long)q * 16;
            if (i0 + 16 <= p.n) {
                reinterpret_cast<int4*>(p.counts_out + i0)[0] = packed;
            } else {
                const signed char* c = reinterpret_cast<const signed char*>(&packed);
                for (int e = 0; e < 16; ++e)
                    if (i0 + e < p.n) p.counts_out[i0 + e] = c[e];
            }
        }
    }

    // sparse apply: compact the non-zero counts of the whole CTA into one list
    // (block scan, no atomics), then every thread applies list entries -- all
    // target loads are independent: one memory round trip per CTA
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
        for (unsigned i = tid; i < total; i += kDecThreads) {
            const int local = s_list[i];
            const long long gi = base + local;
            if (gi < p.n) {
                const float t = p.target[gi];
                const float u = __fmul_rn((float)s_cnt[local], p.tau);
                p.target[gi] = (MODE == GTC_ACCUM_WEIGHTS) ? __fmaf_rn(p.alpha, u, t) : __fadd_rn(t, u);
            }
        }
    } else {
        // dense batch: each thread applies its own chunks
#pragma unroll
        for (int u = 0; u < kChunksPerThread; ++u) {
            unsigned msk = nz[u];
            const int q = u * kDecThreads + tid;
            while (msk) {
                const int b = __ffs(msk) - 1;
                msk &= msk - 1;
                const int local = q * 16 + b;
                const long long gi = base + local;
                if (gi < p.n) {
                    const float t = p.target[gi];
                    const float uu = __fmul_rn((float)s_cnt[local], p.tau);
                    p.target[gi] = (MODE == GTC_ACCUM_WEIGHTS) ? __fmaf_rn(p.alpha, uu, t) : __fadd_rn(t, uu);
                }
            }
        }
    }
}

// One message (world == 1, or one simulated worker): indices are unique, so
// c[i] = +-1 exactly on the message's indices and 0 elsewhere; the aggregate
// needs no counts at all.  Word-parallel: each thread loads 4 words, then the
// 4 targets, then stores -- two memory round trips, no shared memory, no
// barriers.  fl(+-1 * tau) = +-tau exactly, so the arithmetic is the general
// kernel's (R8).  The message length is read on the device (tile_off[num_tiles]).
constexpr int kSingleThreads = 256;
constexpr int kSingleBatch = 4;

template <int MODE>
__global__ void __launch_bounds__(kSingleThreads) gtc_apply_single_kernel(const DecodeParams p) {
    if (*p.flags & (kFlagCapacity | kFlagCorrupt)) return;
    const long long k = __ldg(p.m.off[0] + p.num_tiles);
    const unsigned* words = p.m.words[0];
    const long long stride = (long long)gridDim.x * kSingleThreads * kSingleBatch;
    for (long long j0 = (long long)blockIdx.x * kSingleThreads * kSingleBatch + threadIdx.x; j0 < k; j0 += stride) {
        unsigned w[kSingleBatch];
        float t[kSingleBatch];
#pragma unroll
        for (int u = 0; u < kSingleBatch; ++u) {
            const long long j = j0 + u * kSingleThreads;
            w[u] = j < k ? __ldg(words + j) : 0u;
        }
#pragma unroll
        for (int u = 0; u < kSingleBatch; ++u)
            if (j0 + u * kSingleThreads < k) t[u] = p.target[w[u] >> 1];
#pragma unroll
        for (int u = 0; u < kSingleBatch; ++u) {
            if (j0 + u * kSingleThreads < k) {
                const float q = (w[u] & 1u) ? -p.tau : p.tau;  // fl(c * tau) for c = -1 / +1
                p.target[w[u] >> 1] = (MODE == GTC_ACCUM_WEIGHTS) ? __fmaf_rn(p.alpha, q, t[u])
                                                                  : __fadd_rn(t[u], q);
            }
        }
    }
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

}  // namespace

cudaError_t launch_decode_apply(const DecodeParams& p_in, int accum_mode, cudaStream_t s) {
    if (p_in.num_tiles == 0) return cudaSuccess;
    static int sms = 0;
    if (sms == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaError_t e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (e != cudaSuccess) return e;
    }
    if (p_in.nmsg == 1 && p_in.counts_out == nullptr) {
        const int grid = sms * 8;
        if (accum_mode == GTC_ACCUM_UPDATE)
            gtc_apply_single_kernel<GTC_ACCUM_UPDATE><<<grid, kSingleThreads, 0, s>>>(p_in);
        else
            gtc_apply_single_kernel<GTC_ACCUM_WEIGHTS><<<grid, kSingleThreads, 0, s>>>(p_in);
        return cudaGetLastError();
    }
    // about one wave of 8 CTAs per SM, at most kDecMaxTilesPerCta tiles per CTA
    DecodeParams p = p_in;
    int tpc = (p.num_tiles + sms * 8 - 1) / (sms * 8);
    tpc = tpc < 1 ? 1 : (tpc > kDecMaxTilesPerCta ? kDecMaxTilesPerCta : tpc);
    p.tiles_per_cta = tpc;
    const int grid = (p.num_tiles + tpc - 1) / tpc;
    const size_t smem = (size_t)tpc * kTile;
    if (accum_mode == GTC_ACCUM_UPDATE)
        gtc_decode_apply_kernel<GTC_ACCUM_UPDATE><<<grid, kDecThreads, smem, s>>>(p);
    else
        gtc_decode_apply_kernel<GTC_ACCUM_WEIGHTS><<<grid, kDecThreads, smem, s>>>(p);
    return cudaGetLastError();
}

// p2p exchange: publish "this rank's message of step `epoch` is ready" into
// every peer's ready[self] (remote store over NVLink, release at system scope
// after a system fence; the message itself was written by the preceding
// encode kernels on the same stream).
__global__ void gtc_signal_kernel(const SignalParams p) {
    const int r = threadIdx.x;
    if (r < p.world && r != p.self) {
        __threadfence_system();
        unsigned long long* a = p.peer_ready[r] + p.self;
        asm volatile("st.release.sys.global.u64 [%0], %1;" :: "l"(a), "l"(p.epoch) : "memory");
    }
}

cudaError_t launch_signal(const SignalParams& p, cudaStream_t s) {
    gtc_signal_kernel<<<1, 64, 0, s>>>(p);
    return cudaGetLastError();
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
