// tile_encode.cuh -- device helpers for encoding one tile of kTile params with
// one CTA of kTileThreads threads (Sec. VI-A; R1-R4).
// Used by gtc_encode_tile_kernel (encode.cu) and by the fused p2p step kernel
// (step_p2p.cu).  Not installed.
//
// Element order inside a tile: thread `tid` holds float4 j (j < kTileVec) at
// element offset (j * kTileThreads + tid) * 4, so (round j, warp, lane,
// component) is ascending index; bit j*4+e of the thread's `sel`/`neg` masks
// is component e of its float4 j.
#pragma once

#include "gtc_internal.cuh"

namespace gtc {

constexpr int kTileThreads = 256;
constexpr int kTileWarps = kTileThreads / 32;
constexpr int kTileVec = kTile / (kTileThreads * 4);  // 4
static_assert(kTileVec * kTileWarps == 32, "one (round, warp) scan entry per lane");

// ---------------------------------------------------------------- p2p entries
// In p2p mode a rank's segmented message is read by its peers while it may
// still be being written (the fused step reads tile t of every rank a lag
// after it was encoded, with no fence on the writer's side).  Every 32-bit
// entry of a tile slot therefore carries the step that wrote it:
//     entry = stamp(epoch) << 13 | local << 1 | neg,   local = index - tile * kTile (< 4096)
// A reader accepts an entry only if its stamp is this step's.  The encoder
// also clears (entry 0, stamp 0 = never valid) the slots its previous count of
// the same parity used beyond its new count, so every slot holds either the
// previous same-parity step's entry or 0, and stamp(e) != stamp(e - 2).
constexpr int kStampShift = 13;
static_assert(kTile == 1 << (kStampShift - 1), "local index + sign fill the low 13 bits");
__host__ __device__ __forceinline__ unsigned entry_stamp(unsigned epoch) { return epoch % 524287u + 1u; }
__host__ __device__ __forceinline__ unsigned make_entry(unsigned stamp, unsigned local, unsigned neg) {
    return (stamp << kStampShift) | (local << 1) | neg;
}
// the canonical word (index << 1 | neg) of entry `e` of tile `tile`
__host__ __device__ __forceinline__ unsigned entry_word(unsigned e, long long tile) {
    return ((unsigned)(tile * kTile) + ((e >> 1) & (kTile - 1))) << 1 | (e & 1u);
}

__device__ __forceinline__ float4 ld_nc_v4(const float4* p) {
    float4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
    return v;
}

__device__ __forceinline__ float4 ld_v4(const float4* p) {
    float4 v;
    asm volatile("ld.global.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
    return v;
}

__device__ __forceinline__ void st_stream(float4* p, const float4& v) {
    asm volatile("st.global.L1::no_allocate.v4.f32 [%0], {%1,%2,%3,%4};"
                 :: "l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
}

// The count half of a tile tag (tags are little-endian u64: count in the low
// word); asm volatile so it is issued where it is written, before the tile loads.
__device__ __forceinline__ unsigned ld_tag_count(const unsigned long long* tag) {
    unsigned v;
    asm volatile("ld.global.cg.u32 %0, [%1];" : "=r"(v) : "l"(tag));
    return v;
}

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

__device__ __forceinline__ float comp(const float4& v, int e) {
    return e == 0 ? v.x : e == 1 ? v.y : e == 2 ? v.z : v.w;
}
__device__ __forceinline__ void set_comp(float4& v, int e, float x) {
    if (e == 0) v.x = x; else if (e == 1) v.y = x; else if (e == 2) v.z = x; else v.w = x;
}

// r (and g) of the tile into registers: 128-bit loads issued before any use
// (the ragged last tile element by element, zero-padded).
template <bool HAS_G>
__device__ __forceinline__ void load_tile(const EncodeParams& p, long long base, bool full_tile, int tid,
                                          float4 (&rv)[kTileVec], float4 (&gv)[kTileVec]) {
    if (full_tile) {
        const float4* r4 = reinterpret_cast<const float4*>(p.r + base);
#pragma unroll
        for (int j = 0; j < kTileVec; ++j) rv[j] = ld_v4(r4 + j * kTileThreads + tid);
        if (HAS_G) {
            const float4* g4 = reinterpret_cast<const float4*>(p.g + base);
#pragma unroll
            for (int j = 0; j < kTileVec; ++j) gv[j] = ld_nc_v4(g4 + j * kTileThreads + tid);
        }
    } else {
#pragma unroll
        for (int j = 0; j < kTileVec; ++j) {
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const long long i = base + (long long)(j * kTileThreads + tid) * 4 + e;
                set_comp(rv[j], e, i < p.n ? p.r[i] : 0.0f);
                if (HAS_G) set_comp(gv[j], e, i < p.n ? p.g[i] : 0.0f);
            }
        }
    }
}

// Packed fp32 pairs (sm_100: FADD2): two IEEE round-to-nearest adds /
// subtracts in one instruction, each lane exactly the scalar __fadd_rn /
// __fsub_rn (R12).
__device__ __forceinline__ float2 fadd2_rn(float2 a, float2 b) {
    float2 c;
    asm("{\n\t.reg .b64 ra, rb, rc;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
        "add.rn.f32x2 rc, ra, rb;\n\tmov.b64 {%0, %1}, rc;\n\t}"
        : "=f"(c.x), "=f"(c.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
    return c;
}
__device__ __forceinline__ float2 fsub2_rn(float2 a, float2 b) {
    float2 c;
    asm("{\n\t.reg .b64 ra, rb, rc;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
        "sub.rn.f32x2 rc, ra, rb;\n\tmov.b64 {%0, %1}, rc;\n\t}"
        : "=f"(c.x), "=f"(c.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
    return c;
}

// Rows a1-a3 on the thread's 16 elements: v = fl(r + g); sel = |v| > tau (GT)
// or >= tau (GE); r = sel ? fl(v -+ tau) : v.  rv holds the new residual.
// Elements go in pairs through the packed adds; v - copysign(tau, v) is
// v - tau or v + tau exactly as the scalar forms.
template <int CMP, bool HAS_G>
__device__ __forceinline__ void quantize(float4 (&rv)[kTileVec], const float4 (&gv)[kTileVec], float tau,
                                         unsigned& sel, unsigned& neg, bool& nonfinite) {
    sel = 0u;
    neg = 0u;
    nonfinite = false;
#pragma unroll
    for (int j = 0; j < kTileVec; ++j) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            float2 v = h == 0 ? make_float2(rv[j].x, rv[j].y) : make_float2(rv[j].z, rv[j].w);
            if (HAS_G) v = fadd2_rn(v, h == 0 ? make_float2(gv[j].x, gv[j].y) : make_float2(gv[j].z, gv[j].w));
            const float2 q = fsub2_rn(v, make_float2(copysignf(tau, v.x), copysignf(tau, v.y)));
            const float ax = fabsf(v.x), ay = fabsf(v.y);
            nonfinite |= !(ax <= 3.402823466e38f) || !(ay <= 3.402823466e38f);  // NaN or Inf
            const bool sx = (CMP == GTC_CMP_GT) ? (ax > tau) : (ax >= tau);
            const bool sy = (CMP == GTC_CMP_GT) ? (ay > tau) : (ay >= tau);
            const float2 rn = make_float2(sx ? q.x : v.x, sy ? q.y : v.y);
            if (h == 0) {
                rv[j].x = rn.x;
                rv[j].y = rn.y;
            } else {
                rv[j].z = rn.x;
                rv[j].w = rn.y;
            }
            const int b = j * 4 + 2 * h;
            sel |= ((unsigned)sx << b) | ((unsigned)sy << (b + 1));
            neg |= ((__float_as_uint(v.x) >> 31) << b) | ((__float_as_uint(v.y) >> 31) << (b + 1));
        }
    }
    neg &= sel;  // the sign bit is v < 0 for a selected v
}

__device__ __forceinline__ void store_residual(const EncodeParams& p, long long base, bool full_tile, int tid,
                                               const float4 (&rv)[kTileVec]) {
    if (full_tile) {
        float4* r4 = reinterpret_cast<float4*>(p.r + base);
#pragma unroll
        for (int j = 0; j < kTileVec; ++j) st_stream(r4 + j * kTileThreads + tid, rv[j]);
    } else {
#pragma unroll
        for (int j = 0; j < kTileVec; ++j) {
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const long long i = base + (long long)(j * kTileThreads + tid) * 4 + e;
                if (i < p.n) p.r[i] = comp(rv[j], e);
            }
        }
    }
}

// Row a5, first half: the thread's offsets of its selected elements among
// the tile's (my_off[j] = words before its float4 j within round j, warp),
// per (round, warp) totals into s_scan (then exclusive-scanned by warp 0 in
// tile_scan_finish).
__device__ __forceinline__ void tile_scan_ballots(unsigned sel, int lane, int warp, unsigned (&my_off)[kTileVec],
                                                  unsigned* s_scan) {
    const unsigned lt = lanemask_lt();
#pragma unroll
    for (int j = 0; j < kTileVec; ++j) {
        const unsigned c = __popc((sel >> (4 * j)) & 0xfu);  // 0..4
        const unsigned b0 = __ballot_sync(0xffffffffu, c & 1u);
        const unsigned b1 = __ballot_sync(0xffffffffu, c & 2u);
        const unsigned b2 = __ballot_sync(0xffffffffu, c & 4u);
        my_off[j] = __popc(b0 & lt) + 2u * __popc(b1 & lt) + 4u * __popc(b2 & lt);
        if (lane == 0) s_scan[j * kTileWarps + warp] = __popc(b0) + 2u * __popc(b1) + 4u * __popc(b2);
    }
}

// Warp 0: exclusive scan of the 32 (round, warp) totals; returns the tile's
// word count on every lane.
__device__ __forceinline__ unsigned tile_scan_finish(int lane, unsigned* s_scan) {
    const unsigned x = s_scan[lane];
    unsigned incl = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    s_scan[lane] = incl - x;
    return __shfl_sync(0xffffffffu, incl, 31);
}

__device__ __forceinline__ void st_relaxed_sys(unsigned* a, unsigned v) {
    asm volatile("st.relaxed.sys.global.u32 [%0], %1;" :: "l"(a), "r"(v) : "memory");
}

__device__ __forceinline__ void st_relaxed_sys(unsigned long long* a, unsigned long long v) {
    asm volatile("st.relaxed.sys.global.u64 [%0], %1;" :: "l"(a), "l"(v) : "memory");
}

// Rows a4-a5, second half: the thread's words, compacted in ascending index
// order, into the tile's slot.  STAMPED (p2p): stamped tile-local entries,
// and the slots [total, prev_total) of the previous same-parity step cleared;
// RELAXED: as relaxed system-scope stores (peers read them while this kernel
// runs, the fused step).
template <bool STAMPED, bool RELAXED = false>
__device__ __forceinline__ void store_words(unsigned* dst, long long base, int tid, unsigned sel, unsigned neg,
                                            const unsigned (&my_off)[kTileVec], const unsigned* s_scan, int warp,
                                            unsigned total, unsigned prev_total, unsigned stamp) {
    // only the thread's selected elements: its word's slot is its (round,
    // warp) base + the words before it in the thread's round
    const unsigned offs = my_off[0] | (my_off[1] << 8) | (my_off[2] << 16) | (my_off[3] << 24);
    for (unsigned m = sel; m; m &= m - 1u) {
        const int bi = __ffs(m) - 1, j = bi >> 2;
        const unsigned o = s_scan[j * kTileWarps + warp] + ((offs >> (8 * j)) & 0xffu) +
                           __popc(sel & ((1u << bi) - 1u) & (0xfu << (4 * j)));
        const unsigned l = (unsigned)(j * kTileThreads + tid) * 4u + (bi & 3), ng = (neg >> bi) & 1u;
        const unsigned w = STAMPED ? make_entry(stamp, l, ng) : (((unsigned)base + l) << 1) | ng;
        if (RELAXED) st_relaxed_sys(dst + o, w);
        else dst[o] = w;
    }
    if (STAMPED) {
        for (unsigned o = total + tid; o < prev_total; o += kTileThreads) {
            if (RELAXED) st_relaxed_sys(dst + o, 0u);
            else dst[o] = 0u;
        }
    }
}

}  // namespace gtc
