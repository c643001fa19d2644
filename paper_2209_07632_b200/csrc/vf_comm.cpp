// vf_comm.cpp -- NCCL plumbing of the block-row (ROWS) mode: one communicator
// per handle, one ncclAllGather of the new Jacobi iterate's own rows per
// iteration.  NVLink 5 / NVSwitch carry it; on the
// single-node B200 box NCCL picks NVLS / P2P itself.
//
// libnccl is opened with dlopen("libnccl.so.2") so a process that already
// loaded torch's NCCL shares that copy (one NCCL per process); a standalone
// process gets the system library.  Types come from <nccl.h>.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <string>

#include "vf_internal.h"

namespace vf {
namespace {

struct Nccl {
    void* so = nullptr;
    ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*allGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    const char* (*errStr)(ncclResult_t) = nullptr;
    std::string err;
};

Nccl& nccl() {
    static Nccl n;
    static std::once_flag once;
    std::call_once(once, [] {
        const char* names[] = {"libnccl.so.2", "libnccl.so"};
        for (const char* nm : names) {
            n.so = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
            if (n.so) break;
        }
        if (!n.so) { n.err = std::string("dlopen libnccl.so.2 failed: ") + dlerror(); return; }
        n.getUniqueId = (decltype(n.getUniqueId))dlsym(n.so, "ncclGetUniqueId");
        n.commInitRank = (decltype(n.commInitRank))dlsym(n.so, "ncclCommInitRank");
        n.commDestroy = (decltype(n.commDestroy))dlsym(n.so, "ncclCommDestroy");
        n.allGather = (decltype(n.allGather))dlsym(n.so, "ncclAllGather");
        n.errStr = (decltype(n.errStr))dlsym(n.so, "ncclGetErrorString");
        if (!n.getUniqueId || !n.commInitRank || !n.commDestroy || !n.allGather || !n.errStr)
            n.err = "libnccl is missing a required symbol";
    });
    return n;
}

int nccl_ready() {
    Nccl& n = nccl();
    if (!n.err.empty()) return set_error(VF_ENCCL, n.err);
    return VF_OK;
}

int nccl_check(ncclResult_t r, const char* what) {
    if (r == ncclSuccess) return VF_OK;
    return set_error(VF_ENCCL, std::string(what) + ": " + nccl().errStr(r));
}

}  // namespace

int comm_get_id(void* id128) {
    int rc = nccl_ready();
    if (rc) return rc;
    ncclUniqueId id;
    if ((rc = nccl_check(nccl().getUniqueId(&id), "ncclGetUniqueId"))) return rc;
    std::memcpy(id128, &id, sizeof(id));
    return VF_OK;
}

int comm_init(Handle* h, int rank, int world, const void* id128) {
    int rc = nccl_ready();
    if (rc) return rc;
    if (h->comm) comm_destroy(h);
    ncclUniqueId id;
    std::memcpy(&id, id128, sizeof(id));
    if (h->device >= 0) cudaSetDevice(h->device);
    ncclComm_t c = nullptr;
    if ((rc = nccl_check(nccl().commInitRank(&c, world, id, rank), "ncclCommInitRank"))) return rc;
    h->comm = c;
    return VF_OK;
}

void comm_destroy(Handle* h) {
    if (!h->comm) return;
    if (nccl_ready() == VF_OK) nccl().commDestroy((ncclComm_t)h->comm);
    h->comm = nullptr;
}

int comm_allgather(Handle* h, const void* send, void* recv, size_t bytes_per_rank, void* stream) {
    return nccl_check(nccl().allGather(send, recv, bytes_per_rank, ncclUint8, (ncclComm_t)h->comm,
                                       (cudaStream_t)stream),
                      "ncclAllGather");
}

}  // namespace vf
