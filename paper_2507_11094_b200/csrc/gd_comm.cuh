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

// 1D block ownership of the vertex ids (the reference's partition.py:69-78
// block_ranges): rank r owns [lo(r), hi(r)); the first n % world ranks get
// one vertex more.
struct Blocks {
    int64_t n = 0, base = 0, rem = 0;
    int world = 1;
    __host__ __device__ Blocks() {}
    __host__ __device__ Blocks(int64_t n_, int world_) : n(n_), base(n_ / world_), rem(n_ % world_), world(world_) {}
    __host__ __device__ int64_t lo(int r) const { return (int64_t)r * base + (r < rem ? r : rem); }
    __host__ __device__ int64_t hi(int r) const { return lo(r + 1); }
    __host__ __device__ int owner(int64_t v) const {
        const int64_t big = rem * (base + 1);
        return v < big ? (int)(v / (base + 1)) : (int)(rem + (v - big) / base);
    }
    __host__ __device__ int64_t chunk() const { return base + (rem ? 1 : 0); }  // largest block
};

struct LocalGroup;  // gd_comm.cu

struct Comm {
    void* nccl = nullptr;  // ncclComm_t
    // In-process group (tests): `world` ranks driven by host threads of one
    // process, each with its own store and stream; collectives synchronise
    // the callers' streams, meet at a host barrier and move the data with
    // device copies -- the same call sequence as NCCL, no kernel waits on
    // another rank's kernel.
    LocalGroup* local = nullptr;
    int rank = 0, world = 1, device = 0;
    // accounting: calls, all-gather / all-reduce payload bytes, ring bytes sent
    // (p2p: the bytes this rank sends to other ranks)
    mutable int64_t n_calls = 0, ag_bytes = 0, ar_bytes = 0, sent_bytes = 0, p2p_bytes = 0;

    // In-place all-gather of `chunk` doubles per rank into buf (n_pad = chunk * world).
    void allgather_f64(double* buf, int64_t chunk, cudaStream_t s) const;
    void allreduce_max_f64(double* x, int64_t count, cudaStream_t s) const;
    void allreduce_sum_i64(int64_t* x, int64_t count, cudaStream_t s) const;
    void allreduce_sum_f64(double* x, int64_t count, cudaStream_t s) const;
    void allreduce_max_u8(uint8_t* x, int64_t count, cudaStream_t s) const;
    void allreduce_min_i32(int32_t* x, int64_t count, cudaStream_t s) const;
    // in-place all-gather of the block layout: rank r contributes
    // buf[lo(r), hi(r)) (grouped broadcasts, unequal blocks)
    void allgatherv(void* buf, const Blocks& b, int elem_bytes, cudaStream_t s) const;
    // send (world, padded to b.chunk() per rank) -> recv (b.chunk()) with max
    void reducescatter_max_u8(const uint8_t* send, uint8_t* recv, int64_t chunk, cudaStream_t s) const;
    // all-to-all of int32 records: d_send_counts[p] (device) records of
    // `width` int32 each go to peer p from `send` (peer-major); one read-back
    // of the send and receive counts sizes the exchange; recv grows to hold
    // what arrives (peer-major).  Returns the received record count.
    int64_t alltoallv_i32(const int32_t* send, const int64_t* d_send_counts, int width, DBuf<int32_t>& recv,
                          cudaStream_t s) const;
};

void comm_unique_id(uint8_t out[128]);
Comm* comm_create(int world, int rank, const uint8_t id[128], int device);
// a member of the in-process group `group` (any id shared by the `world`
// members; the group is created by its first member and freed by its last)
Comm* comm_create_local(int world, int rank, int64_t group, int device);
void comm_destroy(Comm* c);

}  // namespace gdb
