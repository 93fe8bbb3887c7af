// NCCL for the in-engine shard exchange (include/synq/detail/exchange.hpp).
// Kept out of the header-only engine so user translation units that include
// synq/engine.hpp need not link NCCL themselves.
//
// libsynq does NOT link libnccl: NCCL is opened on first use (dlopen), and a
// libnccl.so.2 already in the process (e.g. torch's bundled one) is reused
// (RTLD_NOLOAD first).  Linking the system libnccl would otherwise shadow
// torch's newer one and break `import torch` after `import` of this package.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <stdexcept>
#include <string>

#include "synq/detail/exchange.hpp"

namespace synq::detail {

namespace {
struct nccl_api {
    ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
    ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;
};

const nccl_api& api() {
    static nccl_api a;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) throw std::runtime_error(std::string("NCCL not found: ") + dlerror());
        auto sym = [&](const char* name) {
            void* p = dlsym(h, name);
            if (!p) throw std::runtime_error(std::string("NCCL symbol missing: ") + name);
            return p;
        };
        a.get_unique_id = reinterpret_cast<decltype(a.get_unique_id)>(sym("ncclGetUniqueId"));
        a.comm_init_rank = reinterpret_cast<decltype(a.comm_init_rank)>(sym("ncclCommInitRank"));
        a.all_gather = reinterpret_cast<decltype(a.all_gather)>(sym("ncclAllGather"));
        a.comm_destroy = reinterpret_cast<decltype(a.comm_destroy)>(sym("ncclCommDestroy"));
        a.error_string = reinterpret_cast<decltype(a.error_string)>(sym("ncclGetErrorString"));
    });
    return a;
}

void check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) throw std::runtime_error(std::string(what) + ": " + api().error_string(r));
}
}  // namespace

void nccl_unique_id(char out[kNcclIdBytes]) {
    static_assert(sizeof(ncclUniqueId) == kNcclIdBytes, "ncclUniqueId size");
    ncclUniqueId id;
    check(api().get_unique_id(&id), "ncclGetUniqueId");
    std::memcpy(out, &id, sizeof id);
}

void* nccl_comm_init(uint32_t rank, uint32_t world, const char id[kNcclIdBytes]) {
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof uid);
    ncclComm_t comm = nullptr;
    check(api().comm_init_rank(&comm, static_cast<int>(world), uid, static_cast<int>(rank)), "ncclCommInitRank");
    return comm;
}

void nccl_allgather_u32(void* comm, const uint32_t* send, uint32_t* recv, size_t count, cudaStream_t stream) {
    check(api().all_gather(send, recv, count, ncclUint32, static_cast<ncclComm_t>(comm), stream), "ncclAllGather");
}

void nccl_comm_destroy(void* comm) {
    if (comm) api().comm_destroy(static_cast<ncclComm_t>(comm));
}

}  // namespace synq::detail
