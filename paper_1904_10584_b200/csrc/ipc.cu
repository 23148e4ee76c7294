// ipc.cu -- CUDA-IPC mapping of a device buffer across the ranks of one node
// (used by the p2p GTC exchange and the p2p BMUF step): every rank exports the
// cudaMalloc allocation holding its buffer, the 128-byte records are
// all-gathered over NCCL, every rank maps every peer's buffer, and all ranks
// agree on the outcome (a second all-gather) so that either all or none of
// them run peer-to-peer.
#include <cstring>
#include <vector>

#include "gtc_internal.cuh"

namespace gtc {
namespace {

struct IpcRecord {
    cudaIpcMemHandle_t handle;   // 64 B, of the allocation holding the buffer
    unsigned long long offset;   // buffer - allocation base
    unsigned long long tag;      // must agree on every rank (e.g. the layout size)
    int ok;                      // this rank could export its buffer
    int device;
};
static_assert(sizeof(IpcRecord) <= kIpcRecordBytes, "IPC record fits its slot");

// Base address of the allocation holding p (driver API, resolved at run time
// so that libgtc.so does not link libcuda).
typedef int (*MemGetAddressRangeFn)(unsigned long long*, size_t*, unsigned long long);

bool allocation_base(const void* p, unsigned long long* base) {
    static MemGetAddressRangeFn fn = nullptr;
    if (!fn) {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess || !f)
            return false;
        fn = reinterpret_cast<MemGetAddressRangeFn>(f);
    }
    size_t size = 0;
    return fn(base, &size, reinterpret_cast<unsigned long long>(p)) == 0;
}

}  // namespace

IpcResult ipc_map_peers(ncclComm_t comm, int rank, int world, unsigned char* local, unsigned long long tag,
                        unsigned char* slots, std::vector<unsigned char*>& peers, std::vector<void*>& allocs) {
    IpcRecord rec{};
    unsigned long long base = 0;
    rec.ok = allocation_base(local, &base) &&
             cudaIpcGetMemHandle(&rec.handle, reinterpret_cast<void*>(base)) == cudaSuccess;
    cudaGetLastError();
    rec.offset = rec.ok ? reinterpret_cast<unsigned long long>(local) - base : 0ull;
    rec.tag = tag;
    cudaGetDevice(&rec.device);
    if (cudaMemcpy(slots + kIpcRecordBytes * rank, &rec, sizeof(rec), cudaMemcpyHostToDevice) != cudaSuccess)
        return IpcResult::kCudaError;
    if (ncclAllGather(slots + kIpcRecordBytes * rank, slots, kIpcRecordBytes, ncclUint8, comm, 0) != ncclSuccess)
        return IpcResult::kNcclError;
    if (cudaStreamSynchronize(0) != cudaSuccess) return IpcResult::kCudaError;
    std::vector<unsigned char> all(kIpcRecordBytes * world);
    if (cudaMemcpy(all.data(), slots, all.size(), cudaMemcpyDeviceToHost) != cudaSuccess) return IpcResult::kCudaError;
    peers.assign(world, nullptr);
    allocs.assign(world, nullptr);
    int ok = 1;
    for (int i = 0; i < world; ++i) {
        IpcRecord ri;
        std::memcpy(&ri, all.data() + kIpcRecordBytes * i, sizeof(ri));
        if (!ri.ok || ri.tag != tag) ok = 0;
    }
    for (int i = 0; i < world && ok; ++i) {
        if (i == rank) {
            peers[i] = local;
            continue;
        }
        IpcRecord ri;
        std::memcpy(&ri, all.data() + kIpcRecordBytes * i, sizeof(ri));
        void* p = nullptr;
        if (cudaIpcOpenMemHandle(&p, ri.handle, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
            cudaGetLastError();
            ok = 0;
            break;
        }
        allocs[i] = p;
        peers[i] = static_cast<unsigned char*>(p) + ri.offset;
    }
    // agree: every rank must have mapped every peer
    int* okd = reinterpret_cast<int*>(slots);
    if (cudaMemcpy(okd + rank, &ok, sizeof(int), cudaMemcpyHostToDevice) != cudaSuccess) return IpcResult::kCudaError;
    if (ncclAllGather(okd + rank, okd, 1, ncclInt32, comm, 0) != ncclSuccess) return IpcResult::kNcclError;
    std::vector<int> oks(world, 0);
    if (cudaMemcpy(oks.data(), okd, sizeof(int) * world, cudaMemcpyDeviceToHost) != cudaSuccess)
        return IpcResult::kCudaError;
    for (int v : oks) ok &= v;
    if (!ok) {
        ipc_unmap(allocs);
        return IpcResult::kUnsupported;
    }
    return IpcResult::kOk;
}

void ipc_unmap(std::vector<void*>& allocs) {
    for (void* p : allocs)
        if (p) cudaIpcCloseMemHandle(p);
    allocs.assign(allocs.size(), nullptr);
}

}  // namespace gtc
