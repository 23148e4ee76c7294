// gtc_internal.cuh -- kernel-side declarations shared by the three translation
// units of libgtc.so (encode.cu, decode_apply.cu, gtc.cu).  Not installed;
// the public surface is include/gtc.h.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "gtc.h"

namespace gtc {

constexpr int kTile = GTC_TILE;                        // parameters per tile
constexpr int kEncThreads = 256;                       // encode CTA size
constexpr int kEncWarps = kEncThreads / 32;
constexpr int kEncVec = kTile / (kEncThreads * 4);     // float4 per thread per tensor
constexpr int kDecThreads = 256;                       // decode_apply CTA size
static_assert(kEncVec * kEncWarps == 32, "block scan assumes one (round, warp) entry per lane");
static_assert(kTile == kDecThreads * 16, "decode sweep assumes 16 counts per thread");

// Sticky device flags (Ctrl::flags).
enum : unsigned long long {
    kFlagNonFinite = 1ull,  // a residual element was NaN/Inf
    kFlagCapacity = 2ull,   // the message did not fit max_words_per_rank
    kFlagCorrupt = 4ull,    // a caller-supplied message was not canonical
};

// Control block at the start of the workspace.  k and flags are adjacent so
// one 16-byte all-gather carries both.
struct alignas(256) Ctrl {
    long long k;                  // words of the last encode
    unsigned long long flags;     // sticky flags
    unsigned int ticket[2];       // dynamic tile tickets, indexed by epoch parity
    unsigned int epoch;           // look-back epoch of the NEXT encode, 1..kEpochMax
};

// Look-back tile descriptor: [epoch:30 | status:2 | value:32].  The epoch
// lives on the device (Ctrl::epoch) and is advanced by the last tile, so an
// encode needs no host state and can be captured in a CUDA graph.  Every call
// rewrites every tile's descriptor, so a descriptor is never older than one
// call and the epoch may wrap (kEpochMax -> 1) without a reset.
enum : unsigned { kDescAggregate = 1u, kDescPrefix = 2u };
constexpr unsigned kEpochMax = (1u << 30) - 1u;

struct EncodeParams {
    const float* g;          // may be null (residual already holds r + g)
    float* r;
    long long n;
    float tau;
    unsigned int* words;     // message out
    long long capacity;      // words available
    unsigned long long* desc;  // [num_tiles] look-back descriptors
    int* tile_off;           // [num_tiles + 1] exclusive word offsets per tile
    Ctrl* ctrl;
    int num_tiles;
};

struct MsgSet {
    const unsigned int* words[GTC_MAX_MSGS];
    const int* off[GTC_MAX_MSGS];  // per message: [num_tiles + 1] tile offsets
};

struct DecodeParams {
    MsgSet m;
    int nmsg;
    long long n;
    int num_tiles;
    float tau;
    float alpha;
    float* target;
    signed char* counts_out;   // may be null
    const unsigned long long* flags;  // skip everything if capacity/corrupt set
};

struct BoundsParams {
    const unsigned int* words[GTC_MAX_MSGS];
    long long k[GTC_MAX_MSGS];
    int* off[GTC_MAX_MSGS];
    int nmsg;
    long long n;
    int num_tiles;
    unsigned long long* flags;
};

cudaError_t launch_encode(const EncodeParams& p, int cmp_mode, cudaStream_t s);
cudaError_t launch_decode_apply(const DecodeParams& p, int accum_mode, cudaStream_t s);
cudaError_t launch_tile_bounds(const BoundsParams& p, cudaStream_t s);

}  // namespace gtc
