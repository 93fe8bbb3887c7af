// NCCL for the in-engine shard exchange (include/synq/detail/exchange.hpp).
// Kept out of the header-only engine so user translation units that include
// synq/engine.hpp need not link NCCL themselves.
#include <nccl.h>

#include <cstring>
#include <stdexcept>
#include <string>

#include "synq/detail/exchange.hpp"

namespace synq::detail {

static void check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) throw std::runtime_error(std::string(what) + ": " + ncclGetErrorString(r));
}

void nccl_unique_id(char out[kNcclIdBytes]) {
    static_assert(sizeof(ncclUniqueId) == kNcclIdBytes, "ncclUniqueId size");
    ncclUniqueId id;
    check(ncclGetUniqueId(&id), "ncclGetUniqueId");
    std::memcpy(out, &id, sizeof id);
}

void* nccl_comm_init(uint32_t rank, uint32_t world, const char id[kNcclIdBytes]) {
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof uid);
    ncclComm_t comm = nullptr;
    check(ncclCommInitRank(&comm, static_cast<int>(world), uid, static_cast<int>(rank)), "ncclCommInitRank");
    return comm;
}

void nccl_allgather_u32(void* comm, const uint32_t* send, uint32_t* recv, size_t count, cudaStream_t stream) {
    check(ncclAllGather(send, recv, count, ncclUint32, static_cast<ncclComm_t>(comm), stream), "ncclAllGather");
}

void nccl_comm_destroy(void* comm) {
    if (comm) ncclCommDestroy(static_cast<ncclComm_t>(comm));
}

}  // namespace synq::detail
