// gd_comm.cuh -- NCCL communicator for the multi-GPU paths (one process per
// GPU).  libnccl.so.2 is loaded lazily (dlopen) the first time a
// communicator is created, so single-GPU use never pays for it.
//
// Sharding: every rank holds a replica of the diff-CSR store
// and applies every batch.  PageRank splits the pull by destination range and
// all-gathers the rank vector after every sweep (plus an all-reduce of the
// residual).  TC splits the batch records into contiguous slices and
// all-reduces the count delta.  Both exchange over NVLink / NVSwitch.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "gd_common.cuh"

namespace gdb {

struct Comm {
    void* nccl = nullptr;  // ncclComm_t
    int rank = 0, world = 1, device = 0;
    // accounting: calls, all-gather / all-reduce payload bytes, ring bytes sent
    mutable int64_t n_calls = 0, ag_bytes = 0, ar_bytes = 0, sent_bytes = 0;

    // vertex range owned by this rank: [lo, hi), chunk = ceil(n / world)
    int64_t chunk(int64_t n) const { return (n + world - 1) / world; }
    int64_t lo(int64_t n) const { return std::min<int64_t>(n, (int64_t)rank * chunk(n)); }
    int64_t hi(int64_t n) const { return std::min<int64_t>(n, lo(n) + chunk(n)); }

    // In-place all-gather of `chunk` doubles per rank into buf (n_pad = chunk * world).
    void allgather_f64(double* buf, int64_t chunk, cudaStream_t s) const;
    void allreduce_max_f64(double* x, int64_t count, cudaStream_t s) const;
    void allreduce_sum_i64(int64_t* x, int64_t count, cudaStream_t s) const;
};

void comm_unique_id(uint8_t out[128]);
Comm* comm_create(int world, int rank, const uint8_t id[128], int device);
void comm_destroy(Comm* c);

}  // namespace gdb
