// gtc_internal.cuh -- kernel-side declarations shared by the three translation
// units of libgtc.so (encode.cu, decode_apply.cu, gtc.cu).  Not installed;
// the public surface is include/gtc.h.
#pragma once

#include <cstdint>
#include <vector>

#include <cuda_runtime.h>
#include <nccl.h>

#include "gtc.h"

namespace gtc {

constexpr int kTile = GTC_TILE;                        // parameters per tile
constexpr int kDecThreads = 256;                       // decode_apply CTA size
constexpr int kDecMaxTilesPerCta = 8;                  // <= 32 KB of int8 counts per CTA
static_assert(kTile == kDecThreads * 16, "decode sweep assumes 16 counts per thread");

// Sticky device flags (Ctrl::flags).
enum : unsigned long long {
    kFlagNonFinite = 1ull,  // a residual element was NaN/Inf
    kFlagCapacity = 2ull,   // a contiguous message did not fit max_words_per_rank
    kFlagCorrupt = 4ull,    // a caller-supplied message was not canonical
    kFlagPeer = 8ull,       // a peer did not publish in time (p2p exchange); raised on
                            // EVERY rank's flags by the rank that timed out
};

// Control block at the start of the workspace.  k and flags are adjacent so
// one 16-byte all-gather carries both (NCCL mode).
struct alignas(256) Ctrl {
    unsigned long long k_acc[2];  // words of the encode of step parity p (accumulated per tile)
    unsigned long long flags;     // sticky flags
    unsigned long long ready;     // p2p: the step (encodes since bind) whose message the
                                  // rank has published (separate calls)
    unsigned long long counted;   // p2p sharded decode: the step whose owner count lists
                                  // the rank has published (sharded.cu)
    unsigned ticket;              // fused step: next CTA ticket of the running launch (wraps to
                                  // 0 when the launch's last CTA takes its ticket; step_p2p.cu)
};

// Header of a contiguous message region.
struct MsgHeader {
    long long k;
    unsigned long long flags;
};

// ---------------------------------------------------------------- messages
// The hot path's message is SEGMENTED: the encode compacts the words of tile
// t (ascending index) into slot t of a tile-major buffer,
//     words of tile t = seg[t * kTile .. t * kTile + count_t),
// and tag[t] = (epoch << 32) | count_t.  In p2p mode a slot holds STAMPED
// tile-local entries instead (tile_encode.cuh: stamp(epoch) << 13 | local << 1
// | neg), so a reader can tell this step's entries from older ones without a
// writer-side fence.  The separate calls publish the whole message by raising
// Ctrl::ready = step after a system-scope fence -- done by block 0 of the
// decode kernel (stream order puts every encode store before it), or, in a
// loopback group, by the one-thread publish kernel gtc_exchange launches --
// and peers acquire that flag before reading over NVLink; the fused step
// (step_p2p.cu) instead pushes per-tile records and checks stamps.  Decode
// reads exactly the words of the tiles it owns, from every rank, without a
// global prefix scan.
// The CONTIGUOUS message (words in one array + per-tile offsets + header) is
// the wire format of the NCCL exchange and of gtc_message; gtc_compact_kernel
// builds it from a segmented one on demand.
inline __host__ __device__ unsigned long long make_tag(unsigned epoch, unsigned count) {
    return ((unsigned long long)epoch << 32) | count;
}

struct EncodeParams {
    const float* g;                // may be null (residual already holds r + g)
    float* r;
    long long n;
    float tau;
    unsigned int* seg;             // [num_tiles * kTile] tile-major words
    unsigned long long* tags;      // [num_tiles] (epoch << 32) | count
    Ctrl* ctrl;
    unsigned long long* k_acc;     // this step's word counter (tiles add their counts)
    unsigned long long* k_next;    // the other parity's counter, zeroed for the next step
    float* target;                 // world 1 fused apply (gtc_step): null = no apply
    float alpha;
    int accum_mode;
    float* buf;                    // GTC_ACCUM_MOMENTUM: momentum buffer [n]
    float mu;
    unsigned epoch;
    int publish_sys;               // p2p: peers read this message over NVLink
    unsigned long long step;       // p2p: encodes since bind (the value raised in Ctrl::ready)
    int num_tiles;
};
// Packing a segmented message first sums the counts of groups of kGroupTiles tiles.
constexpr int kGroupTiles = 64;

struct CompactParams {             // segmented (any rank) -> contiguous (local)
    const unsigned int* seg;
    const unsigned long long* tags;
    unsigned int* group_sum;       // [ceil(num_tiles / kGroupTiles)] local scratch
    int num_tiles;
    unsigned int* words;
    int* tile_off;                 // [num_tiles + 1]
    MsgHeader* hdr;
    long long capacity;
    Ctrl* ctrl;                    // local: sticky flags (capacity)
    int stamped;                   // p2p: seg holds stamped tile-local entries (tile_encode.cuh)
};

struct DecodeParams {
    int segmented;                 // 1: seg/tags (hot path), 0: words/off (contiguous)
    int stamped;                   // segmented p2p: stamped tile-local entries (tile_encode.cuh)
    const unsigned int* words[GTC_MAX_MSGS];       // contiguous
    const int* off[GTC_MAX_MSGS];                  // contiguous: [num_tiles + 1] tile offsets
    const unsigned int* seg[GTC_MAX_MSGS];         // segmented (peer pointers in p2p)
    const unsigned long long* tags[GTC_MAX_MSGS];  // segmented
    unsigned epoch;                // segmented: this step's epoch
    unsigned long long step;       // p2p: wait until every rank's Ctrl::ready >= step
    int wait;                      // segmented p2p: acquire every rank's ready flag first
    const unsigned long long* ready[GTC_MAX_MSGS];  // p2p: each rank's Ctrl::ready
    unsigned long long* peer_flags[GTC_MAX_MSGS];   // p2p: every rank's Ctrl::flags (timeout broadcast)
    unsigned long long* publish;   // p2p: raise this rank's ready flag (= step) first, or null
    unsigned long long timeout_ns; // p2p: longest wait for a peer
    int nmsg;
    long long n;
    int num_tiles;
    float tau;
    float alpha;
    float* target;
    float* buf;                    // GTC_ACCUM_MOMENTUM: momentum buffer [n] (dense apply)
    float mu;
    signed char* counts_out;       // may be null
    unsigned long long* flags;     // this rank's Ctrl::flags
    int tiles_per_cta;             // set by launch_decode_apply
    int trace;                     // GTC_DECODE_TRACE=1: stamp phase times (debug)
};

// The fused p2p step (step_p2p.cu): the CTA with ticket b encodes tile b and
// pushes its record -- tag and the first kPushCap entries -- into every peer's
// push region with one bulk (TMA) copy per peer, and decodes tile b -
// lag_tiles of every rank from the records pushed here (entries beyond
// kPushCap, tiles denser than 1/8, are read from the owner over NVLink).
constexpr int kFusedMaxRanks = 8;
constexpr int kPushCap = kTile / 8;
constexpr int kPushRec = 16 + 4 * kPushCap;          // bytes per tile record: {u64 tag, u64 0, u32 entries[kPushCap]}
struct FusedStepParams {
    EncodeParams enc;                                  // this rank's encode (stamped entries, no apply)
    const unsigned* seg[kFusedMaxRanks];               // every rank's words of this step's parity (peers: NVLink)
    const unsigned long long* tags[kFusedMaxRanks];    // every rank's tags of this step's parity
    unsigned char* push_out[kFusedMaxRanks];           // this rank's records in peer m's push region (null: self)
    const unsigned char* push_in[kFusedMaxRanks];      // rank m's records in this rank's push region (null: self)
    int rank;
    int nranks;
    int lag_tiles;                                     // CTA b encodes tile b, decodes tile b - lag_tiles
    int spec_window;                                   // speculative entries per rank, kTileThreads / nranks
    int spec_shift;                                    // log2(spec_window) if a power of two, else -1
    unsigned stamp;                                    // entry_stamp(enc.epoch)
    unsigned* ticket;                                  // the launch's CTA ticket counter (Ctrl::ticket;
                                                       // loopback group: rank 0's, shared by the group)
    float* target;
    float alpha;
    unsigned long long* flags;                         // this rank's Ctrl::flags
    unsigned long long* peer_flags[kFusedMaxRanks];    // every rank's Ctrl::flags (timeout broadcast)
    unsigned long long timeout_ns;                     // longest wait for a peer's tile
    int skip;                                          // loopback test hook: this rank does nothing
    int trace;                                         // GTC_DECODE_TRACE=1: phase stamps (debug)
};

// Owner-computes (sharded) decode, GTC_DECODE_SHARDED (sharded.cu; SURVEY
// 8(f) #4): rank m owns tiles [tile_begin(m), tile_begin(m + 1)) with
// tile_begin(m) = ceil(m T / N).  gtc_exchange: the owner counts its tiles
// from every rank's stamped entries (peer reads) and writes one COUNT LIST
// per tile -- entries (local << 8) | (count & 0xff), ascending local index,
// tag (epoch << 32) | length; gtc_decode_apply: every rank applies every
// tile from its owner's list.
__host__ __device__ __forceinline__ long long shard_tile_begin(int m, int nranks, long long tiles) {
    return (m * tiles + nranks - 1) / nranks;
}
__host__ __device__ __forceinline__ int shard_owner(long long t, int nranks, long long tiles) {
    return (int)((t * nranks) / tiles);
}

struct ShardParams {
    const unsigned* seg[kFusedMaxRanks];               // every rank's stamped entries (this step's parity)
    const unsigned long long* tags[kFusedMaxRanks];    // every rank's tile tags
    const unsigned long long* ready[kFusedMaxRanks];   // every rank's Ctrl::ready
    const unsigned long long* counted[kFusedMaxRanks]; // every rank's Ctrl::counted
    unsigned long long* peer_flags[kFusedMaxRanks];    // every rank's Ctrl::flags (timeout broadcast)
    unsigned long long* publish;                       // count: this rank's Ctrl::ready; apply: Ctrl::counted
    unsigned* clist;                                   // this rank's count lists (this parity), [T * kTile]
    unsigned long long* ctags;                         // this rank's count-list tags, [T]
    const unsigned* clist_of[kFusedMaxRanks];          // every owner's count lists
    const unsigned long long* ctags_of[kFusedMaxRanks];
    int nranks, rank;
    long long n;
    int num_tiles;
    unsigned epoch;
    unsigned long long step;
    unsigned long long timeout_ns;
    float tau, alpha;
    float* target;
    float* buf;                                        // GTC_ACCUM_MOMENTUM
    float mu;
    signed char* counts_out;                           // may be null
    unsigned long long* flags;                         // this rank's Ctrl::flags
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

// CUDA-IPC mapping of one buffer per rank (ipc.cu).  `slots` is device
// scratch of kIpcRecordBytes * world bytes; `tag` must agree on all ranks.
constexpr int kIpcRecordBytes = 128;
enum class IpcResult { kOk, kCudaError, kNcclError, kUnsupported };
IpcResult ipc_map_peers(ncclComm_t comm, int rank, int world, unsigned char* local, unsigned long long tag,
                        unsigned char* slots, std::vector<unsigned char*>& peers, std::vector<void*>& allocs);
void ipc_unmap(std::vector<void*>& allocs);

bool pdl_enabled();  // programmatic dependent launch (GTC_PDL=0 disables)
cudaError_t launch_encode(EncodeParams& p, int cmp_mode, cudaStream_t s);
cudaError_t launch_compact(const CompactParams& p, cudaStream_t s);
cudaError_t launch_publish(unsigned long long* flag, unsigned long long step, cudaStream_t s);
cudaError_t launch_owner_count(const ShardParams& p, cudaStream_t s);
cudaError_t launch_apply_counts(const ShardParams& p, int accum_mode, cudaStream_t s);
cudaError_t launch_decode_apply(const DecodeParams& p, int accum_mode, cudaStream_t s);
cudaError_t launch_tile_bounds(const BoundsParams& p, cudaStream_t s);
cudaError_t launch_step_p2p(FusedStepParams& p, int cmp_mode, int accum_mode, cudaStream_t s);
// Loopback group (tests): the fused step of `world` ranks as ONE launch; the
// per-rank parameters live in device memory (`group`, copied there by the
// caller); `host` holds the same parameters for the launch configuration.
cudaError_t launch_step_p2p_group(const FusedStepParams* group, const FusedStepParams& host, int world,
                                  int cmp_mode, int accum_mode, cudaStream_t s);
int step_p2p_lag_tiles(int num_tiles, int ranks_per_device);
cudaError_t read_step_trace(unsigned long long* host, int max_entries);
cudaError_t read_decode_trace(unsigned long long* host, int max_entries);
bool decode_trace_enabled();

}  // namespace gtc
