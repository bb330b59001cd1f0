// qlm_comm.h -- internal interface of the NCCL communicator (qlm_comm.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

namespace qlm {

constexpr int kCommIdBytes = 128;

struct Comm;

bool comm_unique_id(uint8_t id[kCommIdBytes], std::string &err);
Comm *comm_init(const uint8_t id[kCommIdBytes], int rank, int world, std::string &err);   // collective
void comm_destroy(Comm *c);
int comm_rank(const Comm *c);
int comm_world(const Comm *c);
// stream-ordered collectives on the caller's stream (no host synchronisation)
bool comm_allgather_bytes(Comm *c, const void *send, void *recv, size_t bytes, cudaStream_t st,
                          std::string &err);
bool comm_allreduce_sum_u32(Comm *c, uint32_t *buf, size_t n, cudaStream_t st, std::string &err);
bool comm_allreduce_max_i32(Comm *c, int32_t *buf, size_t n, cudaStream_t st, std::string &err);
int comm_nccl_version();

}  // namespace qlm
