// gd_comm.cu -- lazily loaded NCCL (see gd_comm.cuh).
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>

#include "gd_comm.cuh"

namespace gdb {

namespace {

// entry points resolved at run time; types from the header torch ships with
using fn_get_id = decltype(&ncclGetUniqueId);
using fn_init = decltype(&ncclCommInitRank);
using fn_destroy = decltype(&ncclCommDestroy);
using fn_allgather = decltype(&ncclAllGather);
using fn_allreduce = decltype(&ncclAllReduce);
using fn_errstr = decltype(&ncclGetErrorString);

struct Api {
    void* h = nullptr;
    fn_get_id get_id = nullptr;
    fn_init init = nullptr;
    fn_destroy destroy = nullptr;
    fn_allgather allgather = nullptr;
    fn_allreduce allreduce = nullptr;
    fn_errstr errstr = nullptr;
};

Api& api() {
    static Api a;
    static std::once_flag once;
    std::call_once(once, [] {
        const char* names[] = {"libnccl.so.2", "libnccl.so",
                               "/opt/prime-rl/.venv/lib/python3.12/site-packages/nvidia/nccl/lib/libnccl.so.2"};
        for (const char* nm : names) {
            a.h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
            if (a.h) break;
        }
        if (!a.h) return;
        a.get_id = (fn_get_id)dlsym(a.h, "ncclGetUniqueId");
        a.init = (fn_init)dlsym(a.h, "ncclCommInitRank");
        a.destroy = (fn_destroy)dlsym(a.h, "ncclCommDestroy");
        a.allgather = (fn_allgather)dlsym(a.h, "ncclAllGather");
        a.allreduce = (fn_allreduce)dlsym(a.h, "ncclAllReduce");
        a.errstr = (fn_errstr)dlsym(a.h, "ncclGetErrorString");
    });
    if (!a.h || !a.get_id || !a.init || !a.allgather || !a.allreduce)
        throw GdError(GD_ERR_CUDA, "libnccl.so.2 could not be loaded");
    return a;
}

void check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) {
        Api& a = api();
        throw GdError(GD_ERR_CUDA, std::string(what) + ": " + (a.errstr ? a.errstr(r) : "nccl error"));
    }
}

}  // namespace

void comm_unique_id(uint8_t out[128]) {
    ncclUniqueId id;
    check(api().get_id(&id), "ncclGetUniqueId");
    std::memcpy(out, id.internal, 128);
}

Comm* comm_create(int world, int rank, const uint8_t idb[128], int device) {
    if (world < 1 || rank < 0 || rank >= world) throw GdError(GD_ERR_CONTRACT, "bad rank / world size");
    GD_CUDA(cudaSetDevice(device));
    ncclUniqueId id;
    std::memcpy(id.internal, idb, 128);
    auto* c = new Comm;
    c->rank = rank;
    c->world = world;
    c->device = device;
    try {
        ncclComm_t comm = nullptr;
        check(api().init(&comm, world, id, rank), "ncclCommInitRank");
        c->nccl = comm;
    } catch (...) {
        delete c;
        throw;
    }
    return c;
}

void comm_destroy(Comm* c) {
    if (!c) return;
    if (c->nccl && api().destroy) api().destroy((ncclComm_t)c->nccl);
    delete c;
}

void Comm::allgather_f64(double* buf, int64_t ch, cudaStream_t s) const {
    ++n_calls;
    ag_bytes += ch * 8 * world;
    sent_bytes += ch * 8 * (world - 1);
    check(api().allgather(buf + (int64_t)rank * ch, buf, (size_t)ch, ncclFloat64, (ncclComm_t)nccl, s),
          "ncclAllGather");
}

void Comm::allreduce_max_f64(double* x, int64_t count, cudaStream_t s) const {
    ++n_calls;
    ar_bytes += count * 8;
    sent_bytes += world > 1 ? count * 8 * 2 * (world - 1) / world : 0;
    check(api().allreduce(x, x, (size_t)count, ncclFloat64, ncclMax, (ncclComm_t)nccl, s), "ncclAllReduce(max)");
}

void Comm::allreduce_sum_i64(int64_t* x, int64_t count, cudaStream_t s) const {
    ++n_calls;
    ar_bytes += count * 8;
    sent_bytes += world > 1 ? count * 8 * 2 * (world - 1) / world : 0;
    check(api().allreduce(x, x, (size_t)count, ncclInt64, ncclSum, (ncclComm_t)nccl, s), "ncclAllReduce(sum)");
}

}  // namespace gdb
