// decode_apply.cu -- GTC aggregate + apply for sm_100a (Sec. VI-A:
// "The received sparse gradient updates are aggregated and weights are updated
// based on the aggregate").
//
// One CTA per parameter tile of kTile elements (the encode tiling, so every
// message's slice for the tile is [off[t], off[t+1]) and reads are coalesced).
//   1. counts c[0..kTile) in shared memory, int8 (|c| <= nmsg <= 64),
//   2. ordered per-message passes: indices are unique within a message, so in
//      one pass no two threads touch the same count; a barrier separates
//      passes.  Integer sums: the result is independent of message order and
//      needs no atomics (deterministic by construction, R6),
//   3. sparse apply (R8): only elements with c != 0 are read-modify-written:
//        u = fl((float)c * tau);  WEIGHTS: t = fmaf(alpha, u, t);  UPDATE: t = fl(t + u)
//      each thread owns 16 consecutive counts (one 128-bit shared load) and
//      issues its predicated loads before any store.
//   4. optional dense int8 counts dump (tests / parity only).
//
// Algorithmic HBM bytes per launch: 4 * (sum of message words) (read) +
// 4 * nmsg * (num_tiles + 1) (tile offsets) + 8 * |{i : c_i != 0}| (target RMW).
#include "gtc_internal.cuh"

namespace gtc {
namespace {

template <int MODE>
__global__ void __launch_bounds__(kDecThreads) gtc_decode_apply_kernel(const DecodeParams p) {
    __shared__ __align__(16) signed char s_cnt[kTile];

    if (*p.flags & (kFlagCapacity | kFlagCorrupt)) return;  // nothing is applied

    const int tid = threadIdx.x;
    const int tile = blockIdx.x;
    const long long base = (long long)tile * kTile;

    reinterpret_cast<int4*>(s_cnt)[tid] = make_int4(0, 0, 0, 0);
    __syncthreads();

    for (int m = 0; m < p.nmsg; ++m) {
        const int b = __ldg(p.m.off[m] + tile);
        const int e = __ldg(p.m.off[m] + tile + 1);
        const unsigned* w = p.m.words[m];
        for (int j = b + tid; j < e; j += kDecThreads) {
            const unsigned word = __ldg(w + j);
            const int local = (int)((word >> 1) - (unsigned)base);
            s_cnt[local] = (signed char)(s_cnt[local] + ((word & 1u) ? -1 : 1));
        }
        __syncthreads();
    }

    // sparse apply over this thread's 16 consecutive counts
    const int4 packed = reinterpret_cast<const int4*>(s_cnt)[tid];
    const signed char* c = reinterpret_cast<const signed char*>(&packed);
    const long long i0 = base + (long long)tid * 16;
    float t[16];
#pragma unroll
    for (int e = 0; e < 16; ++e)
        if (c[e] != 0 && i0 + e < p.n) t[e] = p.target[i0 + e];
#pragma unroll
    for (int e = 0; e < 16; ++e) {
        if (c[e] != 0 && i0 + e < p.n) {
            const float u = __fmul_rn((float)c[e], p.tau);
            p.target[i0 + e] = (MODE == GTC_ACCUM_WEIGHTS) ? __fmaf_rn(p.alpha, u, t[e])
                                                           : __fadd_rn(t[e], u);
        }
    }

    if (p.counts_out) {
        if (i0 + 16 <= p.n) {
            reinterpret_cast<int4*>(p.counts_out + i0)[0] = packed;
        } else {
#pragma unroll
            for (int e = 0; e < 16; ++e)
                if (i0 + e < p.n) p.counts_out[i0 + e] = c[e];
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

cudaError_t launch_decode_apply(const DecodeParams& p, int accum_mode, cudaStream_t s) {
    if (p.num_tiles == 0) return cudaSuccess;
    if (accum_mode == GTC_ACCUM_UPDATE)
        gtc_decode_apply_kernel<GTC_ACCUM_UPDATE><<<p.num_tiles, kDecThreads, 0, s>>>(p);
    else
        gtc_decode_apply_kernel<GTC_ACCUM_WEIGHTS><<<p.num_tiles, kDecThreads, 0, s>>>(p);
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
