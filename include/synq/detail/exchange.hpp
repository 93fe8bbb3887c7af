#pragma once
// In-engine shard exchange over NCCL (implemented in libsynq,
// paper_1912_07423_b200/csrc/nccl_glue.cu).  A sharded network created with
// an NCCL id runs export -> ncclAllGather -> import on its own stream after
// every batch of at most delay-1 steps, with no host synchronisation.
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

namespace synq::detail {

constexpr int kNcclIdBytes = 128;

void nccl_unique_id(char out[kNcclIdBytes]);
void* nccl_comm_init(uint32_t rank, uint32_t world, const char id[kNcclIdBytes]);
void nccl_allgather_u32(void* comm, const uint32_t* send, uint32_t* recv, size_t count, cudaStream_t stream);
void nccl_comm_destroy(void* comm);

}  // namespace synq::detail
