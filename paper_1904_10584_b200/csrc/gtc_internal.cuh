// gtc_internal.cuh -- kernel-side declarations shared by the three translation
// units of libgtc.so (encode.cu, decode_apply.cu, gtc.cu).  Not installed;
// the public surface is include/gtc.h.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "gtc.h"

namespace gtc {

constexpr int kTile = GTC_TILE;                        // parameters per tile
constexpr int kEncThreads = 512;                       // encode CTA size
constexpr int kEncWarps = kEncThreads / 32;
constexpr int kEncVec = kTile / (kEncThreads * 4);     // float4 per thread per tensor
constexpr int kDecThreads = 256;                       // decode_apply CTA size
constexpr int kDecMaxTilesPerCta = 8;                  // <= 32 KB of int8 counts per CTA
static_assert(kEncVec * kEncWarps == 32, "block scan assumes one (round, warp) entry per lane");
static_assert(kTile == kDecThreads * 16, "decode sweep assumes 16 counts per thread");

// Sticky device flags (Ctrl::flags).
enum : unsigned long long {
    kFlagNonFinite = 1ull,  // a residual element was NaN/Inf
    kFlagCapacity = 2ull,   // the message did not fit max_words_per_rank
    kFlagCorrupt = 4ull,    // a caller-supplied message was not canonical
    kFlagPeer = 8ull,       // a peer did not signal its message in time (p2p exchange)
};

// Header at the start of every message region (what peers read first).
struct MsgHeader {
    long long k;                  // words in the message
    unsigned long long flags;     // the sender's sticky flags when it was packed
};

// Control block at the start of the workspace.  k and flags are adjacent so
// one 16-byte all-gather carries both.
struct alignas(256) Ctrl {
    long long k;                  // words of the last encode
    unsigned long long flags;     // sticky flags
};

// Encode runs as two kernels (encode.cu):
//   1. gtc_encode_tiles_kernel: CTA b streams a contiguous chunk of
//      chunk_tiles tiles of g and r, writes r, compacts each tile's words into
//      its slot of a tile-major scratch, writes the tile's word count and, at
//      the end, its chunk's word count (every entry rewritten every call: no
//      atomics, no zeroing, no state carried between calls);
//   2. gtc_compact_kernel: one warp per tile turns the counts into global tile
//      offsets (sum of earlier chunks + earlier tiles of its chunk) and copies
//      the words into the contiguous message.
struct EncodeParams {
    const float* g;          // may be null (residual already holds r + g)
    float* r;
    long long n;
    float tau;
    unsigned int* words;     // message out (contiguous)
    long long capacity;      // words available
    unsigned int* scratch;   // [num_tiles * kTile] tile-major words
    int* tile_cnt;           // [num_tiles] words per tile
    unsigned int* chunk_sum; // [num_chunks] words per chunk of kernel 1
    int* tile_off;           // [num_tiles + 1] exclusive word offsets per tile
    MsgHeader* hdr;          // header of the message region (k, flags)
    Ctrl* ctrl;
    int num_tiles;
    int chunk_tiles;         // tiles per kernel-1 CTA (set by launch_encode)
    int num_chunks;          // kernel-1 grid (set by launch_encode)
};

// Most kernel-1 CTAs (chunks) a launch may use: 148 SMs x 2, with headroom.
constexpr int kMaxChunks = 1024;

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
    int tiles_per_cta;         // set by launch_decode_apply
    // p2p exchange (world > 1, peers' messages read over NVLink); ready == null otherwise
    const MsgHeader* hdr[GTC_MAX_MSGS];  // every rank's header (peer pointers)
    const unsigned long long* ready;     // [world] local flags, peer r writes ready[r] = epoch
    unsigned long long epoch;            // this step's epoch
    int self;                            // this rank (does not wait on itself)
    unsigned long long* local_flags;     // remote flags are folded in here (Ctrl::flags)
};

struct SignalParams {
    unsigned long long* peer_ready[GTC_MAX_MSGS];  // peer r's ready array (IPC-mapped)
    int world;
    int self;
    unsigned long long epoch;
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
cudaError_t launch_signal(const SignalParams& p, cudaStream_t s);

}  // namespace gtc
