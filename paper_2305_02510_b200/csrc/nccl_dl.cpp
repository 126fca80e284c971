// NCCL resolved at run time (dlopen), so single-GPU use of the engine has no
// NCCL dependency and the process shares whichever libnccl.so.2 torch already
// loaded.  One in-place ncclAllGather of the spike bitmask per step is the
// only collective of the engine.
#include "nccl_dl.hpp"

#include <dlfcn.h>
#include <cstdlib>

#include <cstring>
#include <mutex>
#include <string>

namespace snb {

namespace {

struct NcclApi {
    bool loaded = false;
    std::string error;
    ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
    ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                               cudaStream_t) = nullptr;
    const char* (*get_error_string)(ncclResult_t) = nullptr;
};

NcclApi& api() {
    static NcclApi a;
    static std::once_flag once;
    std::call_once(once, [] {
        // SNB_NCCL_LIB first: a process that also uses torch must load torch's
        // own libnccl.so.2 -- whichever copy is loaded first owns the soname,
        // and torch's libtorch_cuda cannot bind to an older one loaded here
        // (the Python layer points this at the nvidia-nccl wheel, engine.py)
        void* h = nullptr;
        if (const char* p = std::getenv("SNB_NCCL_LIB"); p && *p) h = dlopen(p, RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            a.error = std::string("cannot load libnccl.so.2: ") + dlerror();
            return;
        }
        a.get_unique_id = reinterpret_cast<decltype(a.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
        a.comm_init_rank = reinterpret_cast<decltype(a.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
        a.comm_destroy = reinterpret_cast<decltype(a.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
        a.all_gather = reinterpret_cast<decltype(a.all_gather)>(dlsym(h, "ncclAllGather"));
        a.get_error_string = reinterpret_cast<decltype(a.get_error_string)>(dlsym(h, "ncclGetErrorString"));
        if (!a.get_unique_id || !a.comm_init_rank || !a.comm_destroy || !a.all_gather || !a.get_error_string) {
            a.error = "libnccl.so.2 lacks required symbols";
            return;
        }
        a.loaded = true;
    });
    if (!a.loaded) throw NcclError(a.error);
    return a;
}

void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess)
        throw NcclError(std::string("NCCL error in ") + what + ": " + api().get_error_string(r));
}

}  // namespace

void nccl_unique_id(uint8_t* out) {
    ncclUniqueId id;
    nccl_check(api().get_unique_id(&id), "ncclGetUniqueId");
    std::memcpy(out, id.internal, NCCL_UNIQUE_ID_BYTES);
}

NcclComm::NcclComm(const uint8_t* id, int rank, int world) : rank_(rank), world_(world) {
    ncclUniqueId uid;
    std::memcpy(uid.internal, id, NCCL_UNIQUE_ID_BYTES);
    nccl_check(api().comm_init_rank(&comm_, world, uid, rank), "ncclCommInitRank");
}

NcclComm::~NcclComm() {
    if (comm_) api().comm_destroy(comm_);
}

void NcclComm::all_gather_inplace(uint32_t* buf, size_t words_per_rank, cudaStream_t s) {
    nccl_check(api().all_gather(buf + static_cast<size_t>(rank_) * words_per_rank, buf, words_per_rank,
                                ncclUint32, comm_, s),
               "ncclAllGather");
}

}  // namespace snb
