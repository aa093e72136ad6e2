// comm.cuh — internal interface of the peer-memory communicator (comm.cu).
#pragma once
#include <cuda_runtime.h>

#include "../../include/if_b200.h"

namespace ifb {
// dst (+)= sum over the TP group of src (in group-rank order, bit-identical on all ranks)
if_status comm_allreduce_into(if_comm c, const float* src, float* dst, int64_t n, int accumulate, cudaStream_t st);
if_status comm_send(if_comm c, const float* src, int64_t n, cudaStream_t st);
if_status comm_recv(if_comm c, float* dst, int64_t n, cudaStream_t st);
int comm_group_size(if_comm c);
bool comm_engine(if_comm c, float** boxes, int* ngroup, int* me, int* hidden, int* grid);
}  // namespace ifb
