// gd_comm.cu -- lazily loaded NCCL (see gd_comm.cuh).
#include <dlfcn.h>
#include <nccl.h>

#include <condition_variable>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <vector>

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
using fn_send = decltype(&ncclSend);
using fn_recv = decltype(&ncclRecv);
using fn_gstart = decltype(&ncclGroupStart);
using fn_gend = decltype(&ncclGroupEnd);
using fn_bcast = decltype(&ncclBroadcast);
using fn_rscatter = decltype(&ncclReduceScatter);

struct Api {
    void* h = nullptr;
    fn_get_id get_id = nullptr;
    fn_init init = nullptr;
    fn_destroy destroy = nullptr;
    fn_allgather allgather = nullptr;
    fn_allreduce allreduce = nullptr;
    fn_errstr errstr = nullptr;
    fn_send send = nullptr;
    fn_recv recv = nullptr;
    fn_gstart gstart = nullptr;
    fn_gend gend = nullptr;
    fn_bcast bcast = nullptr;
    fn_rscatter rscatter = nullptr;
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
        a.send = (fn_send)dlsym(a.h, "ncclSend");
        a.recv = (fn_recv)dlsym(a.h, "ncclRecv");
        a.gstart = (fn_gstart)dlsym(a.h, "ncclGroupStart");
        a.gend = (fn_gend)dlsym(a.h, "ncclGroupEnd");
        a.bcast = (fn_bcast)dlsym(a.h, "ncclBroadcast");
        a.rscatter = (fn_rscatter)dlsym(a.h, "ncclReduceScatter");
    });
    if (!a.h || !a.get_id || !a.init || !a.allgather || !a.allreduce || !a.send || !a.recv || !a.gstart ||
        !a.gend || !a.bcast || !a.rscatter)
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

// ---------------------------------------------------------------- in-process group
struct LocalGroup {
    int world = 1;
    int64_t id = 0;
    int members = 0;  // live Comm objects
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    int64_t gen = 0;
    std::vector<const void*> ptr;  // published per rank
    std::vector<std::vector<int64_t>> vals;
    void barrier() {
        std::unique_lock<std::mutex> lk(mu);
        const int64_t g = gen;
        if (++arrived == world) {
            arrived = 0;
            ++gen;
            cv.notify_all();
        } else {
            cv.wait(lk, [&] { return gen != g; });
        }
    }
};

namespace {
std::mutex g_groups_mu;
std::map<int64_t, LocalGroup*> g_groups;

__global__ void k_max_u8(uint8_t* a, const uint8_t* b, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        a[i] = a[i] > b[i] ? a[i] : b[i];
}

// all ranks' `count` elements of x -> host, reduced in rank order
template <typename T, typename Op>
void local_allreduce(const Comm& c, T* x, int64_t count, cudaStream_t s, Op op) {
    LocalGroup& g = *c.local;
    GD_CUDA(cudaStreamSynchronize(s));
    g.ptr[c.rank] = x;
    g.barrier();
    std::vector<T> acc((size_t)count), tmp((size_t)count);
    for (int r = 0; r < c.world; ++r) {
        GD_CUDA(cudaMemcpy(r ? tmp.data() : acc.data(), g.ptr[r], count * sizeof(T), cudaMemcpyDeviceToHost));
        if (r)
            for (int64_t i = 0; i < count; ++i) acc[i] = op(acc[i], tmp[i]);
    }
    g.barrier();  // every rank has read every x before any is overwritten
    GD_CUDA(cudaMemcpy(x, acc.data(), count * sizeof(T), cudaMemcpyHostToDevice));
}
}  // namespace

Comm* comm_create_local(int world, int rank, int64_t group, int device) {
    if (world < 1 || rank < 0 || rank >= world) throw GdError(GD_ERR_CONTRACT, "bad rank / world size");
    GD_CUDA(cudaSetDevice(device));
    std::lock_guard<std::mutex> lk(g_groups_mu);
    LocalGroup*& g = g_groups[group];
    if (!g) {
        g = new LocalGroup;
        g->world = world;
        g->id = group;
        g->ptr.assign(world, nullptr);
        g->vals.assign(world, {});
    } else if (g->world != world) {
        throw GdError(GD_ERR_CONTRACT, "in-process group size mismatch");
    }
    ++g->members;
    auto* c = new Comm;
    c->local = g;
    c->rank = rank;
    c->world = world;
    c->device = device;
    return c;
}

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
    if (c->local) {
        std::lock_guard<std::mutex> lk(g_groups_mu);
        if (--c->local->members == 0) {
            g_groups.erase(c->local->id);
            delete c->local;
        }
    }
    delete c;
}

void Comm::allgather_f64(double* buf, int64_t ch, cudaStream_t s) const {
    ++n_calls;
    ag_bytes += ch * 8 * world;
    sent_bytes += ch * 8 * (world - 1);
    if (local) {
        GD_CUDA(cudaStreamSynchronize(s));
        local->ptr[rank] = buf;
        local->barrier();
        for (int r = 0; r < world; ++r)
            if (r != rank)
                GD_CUDA(cudaMemcpyAsync(buf + (int64_t)r * ch, static_cast<const double*>(local->ptr[r]) + (int64_t)r * ch,
                                        ch * 8, cudaMemcpyDeviceToDevice, s));
        GD_CUDA(cudaStreamSynchronize(s));
        local->barrier();
        return;
    }
    check(api().allgather(buf + (int64_t)rank * ch, buf, (size_t)ch, ncclFloat64, (ncclComm_t)nccl, s),
          "ncclAllGather");
}

void Comm::allreduce_max_f64(double* x, int64_t count, cudaStream_t s) const {
    ++n_calls;
    ar_bytes += count * 8;
    sent_bytes += world > 1 ? count * 8 * 2 * (world - 1) / world : 0;
    if (local) return local_allreduce<double>(*this, x, count, s, [](double a, double b) { return a > b ? a : b; });
    check(api().allreduce(x, x, (size_t)count, ncclFloat64, ncclMax, (ncclComm_t)nccl, s), "ncclAllReduce(max)");
}

void Comm::allreduce_sum_i64(int64_t* x, int64_t count, cudaStream_t s) const {
    ++n_calls;
    ar_bytes += count * 8;
    sent_bytes += world > 1 ? count * 8 * 2 * (world - 1) / world : 0;
    if (local) return local_allreduce<int64_t>(*this, x, count, s, [](int64_t a, int64_t b) { return a + b; });
    check(api().allreduce(x, x, (size_t)count, ncclInt64, ncclSum, (ncclComm_t)nccl, s), "ncclAllReduce(sum)");
}

void Comm::allreduce_sum_f64(double* x, int64_t count, cudaStream_t s) const {
    ++n_calls;
    ar_bytes += count * 8;
    sent_bytes += world > 1 ? count * 8 * 2 * (world - 1) / world : 0;
    if (local) return local_allreduce<double>(*this, x, count, s, [](double a, double b) { return a + b; });
    check(api().allreduce(x, x, (size_t)count, ncclFloat64, ncclSum, (ncclComm_t)nccl, s), "ncclAllReduce(sum)");
}

void Comm::allreduce_max_u8(uint8_t* x, int64_t count, cudaStream_t s) const {
    ++n_calls;
    ar_bytes += count;
    sent_bytes += world > 1 ? count * 2 * (world - 1) / world : 0;
    if (local) return local_allreduce<uint8_t>(*this, x, count, s, [](uint8_t a, uint8_t b) { return a > b ? a : b; });
    check(api().allreduce(x, x, (size_t)count, ncclUint8, ncclMax, (ncclComm_t)nccl, s), "ncclAllReduce(max u8)");
}

void Comm::allreduce_min_i32(int32_t* x, int64_t count, cudaStream_t s) const {
    ++n_calls;
    ar_bytes += count * 4;
    sent_bytes += world > 1 ? count * 4 * 2 * (world - 1) / world : 0;
    if (world == 1) return;
    if (local) return local_allreduce<int32_t>(*this, x, count, s, [](int32_t a, int32_t b) { return a < b ? a : b; });
    check(api().allreduce(x, x, (size_t)count, ncclInt32, ncclMin, (ncclComm_t)nccl, s), "ncclAllReduce(min)");
}

void Comm::allgatherv(void* buf, const Blocks& b, int elem_bytes, cudaStream_t s) const {
    ++n_calls;
    ag_bytes += b.n * elem_bytes;
    sent_bytes += (b.hi(rank) - b.lo(rank)) * elem_bytes * (world - 1);
    if (world == 1) return;
    if (local) {
        GD_CUDA(cudaStreamSynchronize(s));
        local->ptr[rank] = buf;
        local->barrier();
        for (int r = 0; r < world; ++r)
            if (r != rank)
                GD_CUDA(cudaMemcpyAsync(static_cast<char*>(buf) + b.lo(r) * elem_bytes,
                                        static_cast<const char*>(local->ptr[r]) + b.lo(r) * elem_bytes,
                                        (b.hi(r) - b.lo(r)) * elem_bytes, cudaMemcpyDeviceToDevice, s));
        GD_CUDA(cudaStreamSynchronize(s));
        local->barrier();
        return;
    }
    Api& a = api();
    check(a.gstart(), "ncclGroupStart");
    for (int r = 0; r < world; ++r) {
        char* p = static_cast<char*>(buf) + b.lo(r) * elem_bytes;
        const size_t cnt = (size_t)(b.hi(r) - b.lo(r)) * elem_bytes;
        check(a.bcast(p, p, cnt, ncclUint8, r, (ncclComm_t)nccl, s), "ncclBroadcast");
    }
    check(a.gend(), "ncclGroupEnd");
}

void Comm::reducescatter_max_u8(const uint8_t* send, uint8_t* recv, int64_t chunk, cudaStream_t s) const {
    ++n_calls;
    ar_bytes += chunk * world;
    sent_bytes += chunk * (world - 1);
    if (world == 1) {
        GD_CUDA(cudaMemcpyAsync(recv, send, chunk, cudaMemcpyDeviceToDevice, s));
        return;
    }
    if (local) {
        GD_CUDA(cudaStreamSynchronize(s));
        local->ptr[rank] = send;
        local->barrier();
        DBuf<uint8_t> tmp(std::max<int64_t>(chunk, 1), s);
        for (int r = 0; r < world; ++r) {
            const uint8_t* src = static_cast<const uint8_t*>(local->ptr[r]) + (int64_t)rank * chunk;
            if (r == 0) {
                GD_CUDA(cudaMemcpyAsync(recv, src, chunk, cudaMemcpyDeviceToDevice, s));
            } else {
                GD_CUDA(cudaMemcpyAsync(tmp.get(), src, chunk, cudaMemcpyDeviceToDevice, s));
                k_max_u8<<<grid_for(chunk, 256), 256, 0, s>>>(recv, tmp.get(), chunk);
            }
        }
        GD_CUDA(cudaStreamSynchronize(s));
        local->barrier();
        return;
    }
    check(api().rscatter(send, recv, (size_t)chunk, ncclUint8, ncclMax, (ncclComm_t)nccl, s), "ncclReduceScatter");
}

int64_t Comm::alltoallv_i32(const int32_t* send, const int64_t* d_send_counts, int width, DBuf<int32_t>& recv,
                            cudaStream_t s) const {
    ++n_calls;
    if (local) {
        std::vector<int64_t> hsc(world);
        read_small(s, hsc.data(), d_send_counts, world * sizeof(int64_t));
        local->ptr[rank] = send;
        local->vals[rank] = hsc;
        local->barrier();
        int64_t tot = 0;
        for (int p = 0; p < world; ++p) tot += local->vals[p][rank];
        recv.ensure(std::max<int64_t>(tot, 1) * width, s);
        int64_t ro = 0;
        for (int p = 0; p < world; ++p) {
            int64_t off = 0;  // my records' position in peer p's send buffer
            for (int q = 0; q < rank; ++q) off += local->vals[p][q];
            const int64_t c = local->vals[p][rank];
            if (c)
                GD_CUDA(cudaMemcpyAsync(recv.get() + ro * width, static_cast<const int32_t*>(local->ptr[p]) + off * width,
                                        c * width * 4, cudaMemcpyDeviceToDevice, s));
            if (p != rank) {
                p2p_bytes += hsc[p] * width * 4;
                sent_bytes += hsc[p] * width * 4;
            }
            ro += c;
        }
        GD_CUDA(cudaStreamSynchronize(s));
        local->barrier();
        return tot;
    }
    Api& a = api();
    // the counts first (one int64 per peer), then one read-back of both
    // directions sizes the payload exchange
    DBuf<int64_t> cnt(2 * world, s);  // [send | recv]
    GD_CUDA(cudaMemcpyAsync(cnt.get(), d_send_counts, world * sizeof(int64_t), cudaMemcpyDeviceToDevice, s));
    if (world == 1) {
        GD_CUDA(cudaMemcpyAsync(cnt.get() + 1, cnt.get(), sizeof(int64_t), cudaMemcpyDeviceToDevice, s));
    } else {
        check(a.gstart(), "ncclGroupStart");
        for (int p = 0; p < world; ++p) {
            check(a.send(cnt.get() + p, 1, ncclInt64, p, (ncclComm_t)nccl, s), "ncclSend");
            check(a.recv(cnt.get() + world + p, 1, ncclInt64, p, (ncclComm_t)nccl, s), "ncclRecv");
        }
        check(a.gend(), "ncclGroupEnd");
    }
    std::vector<int64_t> h(2 * world);
    read_small(s, h.data(), cnt.get(), 2 * world * sizeof(int64_t));
    const int64_t* hsc = h.data();
    const int64_t* hrc = h.data() + world;
    int64_t tot = 0;
    for (int p = 0; p < world; ++p) tot += hrc[p];
    recv.ensure(std::max<int64_t>(tot, 1) * width, s);
    int64_t so = 0, ro = 0;
    if (world > 1) check(a.gstart(), "ncclGroupStart");
    for (int p = 0; p < world; ++p) {
        if (p == rank) {
            if (hsc[p])
                GD_CUDA(cudaMemcpyAsync(recv.get() + ro * width, send + so * width, hsc[p] * width * 4,
                                        cudaMemcpyDeviceToDevice, s));
        } else {
            if (hsc[p])
                check(a.send(send + so * width, (size_t)(hsc[p] * width), ncclInt32, p, (ncclComm_t)nccl, s),
                      "ncclSend");
            if (hrc[p])
                check(a.recv(recv.get() + ro * width, (size_t)(hrc[p] * width), ncclInt32, p, (ncclComm_t)nccl, s),
                      "ncclRecv");
            p2p_bytes += hsc[p] * width * 4;
            sent_bytes += hsc[p] * width * 4;
        }
        so += hsc[p];
        ro += hrc[p];
    }
    if (world > 1) check(a.gend(), "ncclGroupEnd");
    return tot;
}

}  // namespace gdb
