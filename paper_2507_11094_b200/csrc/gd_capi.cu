// gd_capi.cu -- the extern "C" boundary (include/gd_capi.h).  Maps
// exceptions to status codes + a thread-local message; no torch types, plain
// pointers and sizes.
#include <atomic>
#include <cstring>
#include <memory>
#include <string>

#include "gd_launch.cuh"
#include "gd_pr.cuh"
#include "gd_sssp.cuh"
#include "gd_tc.cuh"

struct gd_graph {
    std::unique_ptr<gdb::Store> st;
};
struct gd_sssp {
    gdb::SSSP* a;
};
struct gd_pr {
    gdb::PR* a;
};
struct gd_tc {
    gdb::TC* a;
};
struct gd_comm {
    gdb::Comm* c;
};

namespace gdb {

static std::atomic<int64_t> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
void count_library_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
int64_t launches_total() { return g_launches.load(); }

thread_local KernelProf* tl_prof = nullptr;

int prof_begin(const char* name, int64_t bytes, cudaStream_t s) {
    KernelProf* p = tl_prof;
    if (!p || !p->on) return -1;
    KernelProf::Rec r{name, p->event(), p->event(), bytes, -1, p->seq, false};  // pooled events
    GD_CUDA(cudaEventRecord(r.a, s));
    p->pending.push_back(r);
    return (int)p->pending.size() - 1;
}

void prof_tag(int idx, int64_t tag) {
    if (idx >= 0 && tl_prof) tl_prof->pending[(size_t)idx].tag = tag;
}

void prof_set_bytes(int idx, int64_t bytes) {
    if (idx >= 0 && tl_prof) tl_prof->pending[(size_t)idx].bytes = bytes;
}

void prof_end(int idx, cudaStream_t s) {
    KernelProf* p = tl_prof;
    if (idx < 0 || !p) return;
    GD_CUDA(cudaEventRecord(p->pending[(size_t)idx].b, s));
}

void KernelProf::reset_last() {
    if (pending.size() > 4096) flush();
    ++seq;
    last.clear();
}

void KernelProf::drop_sweeps_from(int64_t limit) {
    for (auto& r : pending)
        if (r.seq == seq && r.tag >= limit) r.drop = true;
}

void KernelProf::flush() {
    for (auto& r : pending) {
        if (!r.drop) {
            GD_CUDA(cudaEventSynchronize(r.b));
            float ms = 0;
            GD_CUDA(cudaEventElapsedTime(&ms, r.a, r.b));
            for (KernelStat* k : {&total[r.name], r.seq == seq ? &last[r.name] : nullptr}) {
                if (!k) continue;
                k->ms += ms;
                k->launches += 1;
                k->bytes += r.bytes;
            }
        }
        pool.push_back(r.a);
        pool.push_back(r.b);
    }
    pending.clear();
}

cudaEvent_t KernelProf::event() {
    if (!pool.empty()) {
        cudaEvent_t e = pool.back();
        pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    GD_CUDA(cudaEventCreate(&e));
    return e;
}

KernelProf::~KernelProf() {
    for (auto& r : pending) {
        cudaEventDestroy(r.a);
        cudaEventDestroy(r.b);
    }
    for (auto e : pool) cudaEventDestroy(e);
}

}  // namespace gdb

namespace {

thread_local std::string tl_err;

int ok() {
    tl_err.clear();
    return GD_OK;
}

template <typename F>
int guard(F&& f) {
    try {
        f();
        return ok();
    } catch (const gdb::GdError& e) {
        tl_err = e.what();
        return e.code;
    } catch (const std::bad_alloc&) {
        tl_err = "host out of memory";
        return GD_ERR_CUDA;
    } catch (const std::exception& e) {
        tl_err = e.what();
        return GD_ERR_CUDA;
    }
}

int null_handle() {
    tl_err = "null handle";
    return GD_ERR_CONTRACT;
}

void check_ids(const int64_t* a, const int64_t* b, int64_t k, int64_t n) {
    for (int64_t i = 0; i < k; ++i) {
        int64_t bad = -1;
        if (a[i] < 0 || a[i] >= n) bad = a[i];
        else if (b[i] < 0 || b[i] >= n) bad = b[i];
        if (bad != -1 || (a[i] < 0 || b[i] < 0))
            throw gdb::GdError(GD_ERR_CONTRACT,
                               "node id " + std::to_string(bad) + " out of range [0, " + std::to_string(n) + ")");
    }
}

gdb::AlgoBase* algo_of(const void* h) {
    // every algorithm handle struct holds its AlgoBase-derived pointer first
    return *reinterpret_cast<gdb::AlgoBase* const*>(h);
}

// stage int64 host arrays of the store API as device int32
struct HostIds {
    gdb::DBuf<int32_t> s, d, w;
};
HostIds upload_ids(cudaStream_t st, const int64_t* a, const int64_t* b, const int64_t* w, int64_t k) {
    HostIds h;
    std::vector<int32_t> ha(k), hb(k), hw(w ? k : 0);
    for (int64_t i = 0; i < k; ++i) {
        ha[i] = (int32_t)a[i];
        hb[i] = (int32_t)b[i];
        if (w) {
            if (w[i] < INT32_MIN || w[i] > INT32_MAX)
                throw gdb::GdError(GD_ERR_CONTRACT, "weight outside the int32 range of the B200 layout");
            hw[i] = (int32_t)w[i];
        }
    }
    h.s.alloc(k, st);
    h.d.alloc(k, st);
    if (k) {
        GD_CUDA(cudaMemcpyAsync(h.s.get(), ha.data(), k * 4, cudaMemcpyHostToDevice, st));
        GD_CUDA(cudaMemcpyAsync(h.d.get(), hb.data(), k * 4, cudaMemcpyHostToDevice, st));
    }
    if (w) {
        h.w.alloc(k, st);
        if (k) GD_CUDA(cudaMemcpyAsync(h.w.get(), hw.data(), k * 4, cudaMemcpyHostToDevice, st));
    }
    GD_CUDA(cudaStreamSynchronize(st));  // host vectors die here
    return h;
}

}  // namespace

template <typename H>
static int algo_batch_host(H* h, const uint8_t* kind, const int64_t* src, const int64_t* dst, const int64_t* w,
                           int64_t k, int64_t bi) {
    if (!h) return null_handle();
    return guard([&] {
        GD_CUDA(cudaSetDevice(h->a->g->device));
        gdb::DevBatch b;
        h->a->stage_host(b, kind, src, dst, w, k);
        h->a->batch(b, bi);
        GD_CUDA(cudaStreamSynchronize(h->a->stream()));
    });
}

template <typename H>
static int algo_batch_dev(H* h, const uint8_t* kind, const int32_t* src, const int32_t* dst, const int32_t* w,
                          int64_t k, int64_t bi) {
    if (!h) return null_handle();
    return guard([&] {
        GD_CUDA(cudaSetDevice(h->a->g->device));
        gdb::DevBatch b;
        h->a->stage_device(b, kind, src, dst, w, k);
        h->a->batch(b, bi);
        GD_CUDA(cudaStreamSynchronize(h->a->stream()));
    });
}

// run_batches over a host stream, pipelined (gd_capi.h: gd_*_run_stream).
// The copy stream carries, in order, up(0), up(1), then per batch j:
// D2H(j) after batch j, then up(j+2) -- so each copy runs alone on the link,
// and both hide behind the next batch's compute.
template <typename H, typename T, typename R>
static int algo_run_stream(H* h, const uint8_t* kind, const T* src, const T* dst, const T* w,
                           int64_t k, int64_t bs, int64_t first, R&& result) {
    if (!h) return null_handle();
    return guard([&] {
        if (k < 0 || bs <= 0) throw gdb::GdError(GD_ERR_CONTRACT, "run_stream needs k >= 0 and batch_size > 0");
        if (k && (!kind || !src || !dst)) throw gdb::GdError(GD_ERR_CONTRACT, "null record array");
        GD_CUDA(cudaSetDevice(h->a->g->device));
        auto* a = h->a;
        const int64_t nb = (k + bs - 1) / bs;
        if (nb == 0) return;
        a->reserve_uploads(std::min(bs, k));
        auto up = [&](int64_t j) {
            const int64_t o = j * bs, m = std::min(bs, k - o);
            a->upload_async((int)(j & 1), kind + o, src + o, dst + o, w ? w + o : nullptr, (int)sizeof(T), m);
        };
        // GD_UPLOAD_EARLY=1: queue batch j+1's upload before batch j starts (A/B)
        static const bool early = getenv("GD_UPLOAD_EARLY") != nullptr;
        try {
            up(0);
            for (int64_t j = 0; j < nb; ++j) {
                if (j + 1 < nb) {
                    if (early) up(j + 1);
                    else a->pending_upload = [&up, j] { up(j + 1); };  // at batch j's struct_done
                }
                const int64_t o = j * bs, m = std::min(bs, k - o);
                gdb::DevBatch b;
                a->stage_uploaded(b, (int)(j & 1), kind + o, src + o, dst + o, m);
                a->batch(b, first + j);
                if (a->pending_upload) {  // a batch that queued no structural update
                    auto f = std::move(a->pending_upload);
                    a->pending_upload = nullptr;
                    f();
                }
                result(j);
            }
        } catch (...) {  // no copy may touch the caller's buffers after return
            a->pending_upload = nullptr;
            a->stream_flush();
            cudaStreamSynchronize(a->stream());
            cudaStreamSynchronize(a->io_stream());
            throw;
        }
        a->stream_flush();
        GD_CUDA(cudaStreamSynchronize(a->stream()));
        a->wait_copies();
    });
}

extern "C" {

const char* gd_last_error(void) { return tl_err.c_str(); }
int gd_abi_version(void) { return 100; }
int64_t gd_kernel_launches(void) { return gdb::launches_total(); }

static int graph_create(int64_t n, const int64_t* src, const int64_t* dst, const int64_t* w, int64_t m, int directed,
                        int weighted, int with_reverse, int64_t merge_interval, int device, const gdb::Comm* part,
                        gd_graph** out) {
    return guard([&] {
        if (!out) throw gdb::GdError(GD_ERR_CONTRACT, "null output handle");
        if (n < 0 || n >= INT32_MAX)
            throw gdb::GdError(GD_ERR_CONTRACT, "node_count must lie in [0, 2^31-1) for the B200 layout");
        if (merge_interval < 1) throw gdb::GdError(GD_ERR_CONTRACT, "merge_interval must be >= 1");
        bool as_arcs = (directed & GD_ARCS) != 0;
        directed &= 1;
        int64_t arcs = (directed || as_arcs) ? m : 2 * m;
        // arcs are indexed by int32 positions while a store is built and its
        // index rebuilt (slot ids are int64): at most 2^31
        if (arcs > (int64_t)INT32_MAX + 1) throw gdb::GdError(GD_ERR_CONTRACT, "more than 2^31 arcs per store");
        for (int64_t i = 0; i < m; ++i) {  // dynamic.py:106-112
            if (src[i] < 0 || src[i] >= n || dst[i] < 0 || dst[i] >= n)
                throw gdb::GdError(GD_ERR_MALFORMED, "edge " + std::to_string(i) + ": node id out of range (src=" +
                                                         std::to_string(src[i]) + ", dst=" + std::to_string(dst[i]) +
                                                         ", node_count=" + std::to_string(n) + ")");
            if (w && weighted && w[i] < 0)
                throw gdb::GdError(GD_ERR_MALFORMED,
                                   "edge " + std::to_string(i) + ": negative weight " + std::to_string(w[i]));
            if (w && (w[i] > INT32_MAX || w[i] < INT32_MIN))
                throw gdb::GdError(GD_ERR_CONTRACT, "weight outside the int32 range of the B200 layout");
        }
        int ndev = 0;
        if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
            throw gdb::GdError(GD_ERR_CUDA, "no CUDA device: the B200 path has no CPU fallback");
        if (device < 0 || device >= ndev) throw gdb::GdError(GD_ERR_CUDA, "bad CUDA device index");
        auto* g = new gd_graph;
        g->st.reset(new gdb::Store(device, n, src, dst, weighted ? w : nullptr, m, directed != 0, weighted != 0,
                                   with_reverse != 0, merge_interval, as_arcs, part));
        *out = g;
    });
}

int gd_graph_create(int64_t n, const int64_t* src, const int64_t* dst, const int64_t* w, int64_t m, int directed,
                    int weighted, int with_reverse, int64_t merge_interval, int device, gd_graph** out) {
    return graph_create(n, src, dst, w, m, directed, weighted, with_reverse, merge_interval, device, nullptr, out);
}

int gd_graph_create_dist(int64_t n, const int64_t* src, const int64_t* dst, const int64_t* w, int64_t m,
                         int directed, int weighted, int with_reverse, int64_t merge_interval, int device,
                         gd_comm* comm, gd_graph** out) {
    if (!comm) return null_handle();
    return graph_create(n, src, dst, w, m, directed, weighted, with_reverse, merge_interval, device, comm->c, out);
}

int gd_graph_owned_range(gd_graph* g, int64_t* lo, int64_t* hi) {
    if (!g) return null_handle();
    if (lo) *lo = g->st->own_lo;
    if (hi) *hi = g->st->own_hi;
    return ok();
}

int gd_graph_destroy(gd_graph* g) {
    if (!g) return ok();
    return guard([&] {
        cudaSetDevice(g->st->device);
        delete g;
    });
}

int gd_graph_apply_deletes(gd_graph* g, const int64_t* src, const int64_t* dst, int64_t k, int64_t* applied,
                           int64_t* misses, uint8_t* miss_flags) {
    if (!g) return null_handle();
    return guard([&] {
        gdb::Store& st = *g->st;
        GD_CUDA(cudaSetDevice(st.device));
        check_ids(src, dst, k, st.n);
        HostIds h = upload_ids(st.stream, src, dst, nullptr, k);
        gdb::DBuf<uint8_t> found(k, st.stream);
        int64_t a = st.apply_deletes(h.s.get(), h.d.get(), k, found.get(), true);
        if (st.part && k) st.part->allreduce_max_u8(found.get(), k, st.stream);  // owners' flags to every rank
        if (miss_flags && k) {
            GD_CUDA(cudaMemcpyAsync(miss_flags, found.get(), k, cudaMemcpyDeviceToHost, st.stream));
            GD_CUDA(cudaStreamSynchronize(st.stream));
            for (int64_t i = 0; i < k; ++i) miss_flags[i] = miss_flags[i] ? 0 : 1;
        }
        GD_CUDA(cudaStreamSynchronize(st.stream));
        if (applied) *applied = a;
        if (misses) *misses = k - a;
    });
}

int gd_graph_apply_adds(gd_graph* g, const int64_t* src, const int64_t* dst, const int64_t* w, int64_t k) {
    if (!g) return null_handle();
    return guard([&] {
        gdb::Store& st = *g->st;
        GD_CUDA(cudaSetDevice(st.device));
        check_ids(src, dst, k, st.n);
        HostIds h = upload_ids(st.stream, src, dst, w, k);
        st.apply_adds(h.s.get(), h.d.get(), w ? h.w.get() : nullptr, k);
        GD_CUDA(cudaStreamSynchronize(st.stream));
    });
}

int gd_graph_merge(gd_graph* g) {
    if (!g) return null_handle();
    return guard([&] {
        GD_CUDA(cudaSetDevice(g->st->device));
        g->st->merge();
        GD_CUDA(cudaStreamSynchronize(g->st->stream));
    });
}

int gd_graph_stats(gd_graph* g, int64_t* live, int64_t* nseg, int64_t* slots) {
    if (!g) return null_handle();
    return guard([&] {
        if (live) {
            *live = g->st->live_count();
            if (g->st->part) {  // live_edge_count of the whole graph
                gdb::DBuf<int64_t> t(1, g->st->stream);
                GD_CUDA(cudaMemcpyAsync(t.get(), live, 8, cudaMemcpyHostToDevice, g->st->stream));
                g->st->part->allreduce_sum_i64(t.get(), 1, g->st->stream);
                *live = gdb::read_scalar(g->st->stream, t.get());
            }
        }
        if (nseg) *nseg = (int64_t)g->st->segs.size();
        if (slots) *slots = g->st->total_slots();
    });
}

int gd_graph_info(gd_graph* g, int64_t* n, int* directed, int* weighted, int* with_reverse, int64_t* mi) {
    if (!g) return null_handle();
    return guard([&] {
        if (n) *n = g->st->n;
        if (directed) *directed = g->st->directed;
        if (weighted) *weighted = g->st->weighted;
        if (with_reverse) *with_reverse = g->st->with_reverse;
        if (mi) *mi = g->st->merge_interval;
    });
}

int gd_graph_segment_slots(gd_graph* g, int64_t seg, int64_t* nslots) {
    if (!g) return null_handle();
    return guard([&] {
        if (seg < 0 || seg >= (int64_t)g->st->segs.size()) throw gdb::GdError(GD_ERR_CONTRACT, "segment index");
        *nslots = g->st->segs[(size_t)seg].nslots;
    });
}

int gd_graph_export_segment(gd_graph* g, int64_t seg, int64_t* off, int64_t* col, int64_t* w) {
    if (!g) return null_handle();
    return guard([&] {
        GD_CUDA(cudaSetDevice(g->st->device));
        if (seg < 0 || seg >= (int64_t)g->st->segs.size()) throw gdb::GdError(GD_ERR_CONTRACT, "segment index");
        g->st->export_segment(seg, off, col, w);
    });
}

int gd_graph_reverse_nnz(gd_graph* g, int64_t* nnz) {
    if (!g) return null_handle();
    return guard([&] {
        GD_CUDA(cudaSetDevice(g->st->device));
        if (!g->st->with_reverse)
            throw gdb::GdError(GD_ERR_CONFIG, "graph was loaded without reverse-adjacency maintenance");
        *nnz = g->st->rev_nnz_live();
    });
}

int gd_graph_export_reverse(gd_graph* g, int64_t* off, int64_t* src, int64_t* w) {
    if (!g) return null_handle();
    return guard([&] {
        GD_CUDA(cudaSetDevice(g->st->device));
        if (!g->st->with_reverse)
            throw gdb::GdError(GD_ERR_CONFIG, "graph was loaded without reverse-adjacency maintenance");
        g->st->export_rev(off, src, w);
    });
}

int gd_graph_export_reverse_slots(gd_graph* g, int64_t* off, int64_t* src, int64_t* seg, int64_t* idx,
                                  int64_t* w) {
    if (!g) return null_handle();
    return guard([&] {
        GD_CUDA(cudaSetDevice(g->st->device));
        if (!g->st->with_reverse)
            throw gdb::GdError(GD_ERR_CONFIG, "graph was loaded without reverse-adjacency maintenance");
        g->st->export_rev_slots(off, src, seg, idx, w);
    });
}

int gd_graph_propagate_flags(gd_graph* g, uint8_t* flags, int64_t* rounds) {
    if (!g) return null_handle();
    return guard([&] {
        gdb::Store& st = *g->st;
        GD_CUDA(cudaSetDevice(st.device));
        if (st.directed && !st.with_reverse)  // interp.py:82-85
            throw gdb::GdError(GD_ERR_CONFIG, "propagateNodeFlags on a directed graph needs reverse adjacency");
        gdb::DBuf<uint8_t> f(std::max<int64_t>(st.n, 1), st.stream);
        if (st.n) GD_CUDA(cudaMemcpyAsync(f.get(), flags, st.n, cudaMemcpyHostToDevice, st.stream));
        int64_t r = st.part ? gdb::flood_weak_components_dist(st, f.get(), nullptr)
                            : gdb::flood_weak_components(st, f.get(), nullptr);
        if (st.part) st.part->allgatherv(f.get(), st.blocks, 1, st.stream);
        if (st.n) GD_CUDA(cudaMemcpyAsync(flags, f.get(), st.n, cudaMemcpyDeviceToHost, st.stream));
        GD_CUDA(cudaStreamSynchronize(st.stream));
        if (rounds) *rounds = r;
    });
}

int gd_graph_stream(gd_graph* g, void** stream) {
    if (!g) return null_handle();
    *stream = (void*)g->st->stream;
    return ok();
}

int gd_graph_device_bytes(gd_graph* g, int64_t* bytes) {
    if (!g) return null_handle();
    *bytes = g->st->device_bytes();
    return ok();
}

// ---- algorithms -------------------------------------------------------------

#define ALGO_CREATE(T, handle_t, expr)   \
    return guard([&] {                   \
        if (!g || !out) throw gdb::GdError(GD_ERR_CONTRACT, "null handle"); \
        GD_CUDA(cudaSetDevice(g->st->device)); \
        auto* h = new handle_t;          \
        try {                            \
            h->a = expr;                 \
        } catch (...) {                  \
            delete h;                    \
            throw;                       \
        }                                \
        *out = h;                        \
    })

int gd_sssp_create(gd_graph* g, int64_t src, gd_sssp** out) { return gd_sssp_create_ex(g, src, 10, out); }
int gd_sssp_create_ex(gd_graph* g, int64_t src, int64_t iteration_cap_factor, gd_sssp** out) {
    ALGO_CREATE(gdb::SSSP, gd_sssp, new gdb::SSSP(g->st.get(), src, iteration_cap_factor));
}
int gd_sssp_batch(gd_sssp* s, const uint8_t* kind, const int64_t* src, const int64_t* dst, const int64_t* w,
                  int64_t k, int64_t bi) {
    return algo_batch_host(s, kind, src, dst, w, k, bi);
}
int gd_sssp_batch_device(gd_sssp* s, const uint8_t* kind, const int32_t* src, const int32_t* dst, const int32_t* w,
                         int64_t k, int64_t bi) {
    return algo_batch_dev(s, kind, src, dst, w, k, bi);
}
int gd_sssp_read(gd_sssp* s, int64_t* dist, int64_t* parent) {
    if (!s) return null_handle();
    return guard([&] {
        GD_CUDA(cudaSetDevice(s->a->g->device));
        s->a->read(dist, parent);
    });
}
int gd_sssp_read_async(gd_sssp* s, int64_t* dist, int64_t* parent) {
    if (!s) return null_handle();
    return guard([&] {
        GD_CUDA(cudaSetDevice(s->a->g->device));
        s->a->read_async(dist, parent);
    });
}
int gd_wait(const void* h) {
    if (!h) return null_handle();
    return guard([&] { algo_of(h)->wait_copies(); });
}
}  // extern "C"
template <typename T>
static int sssp_run_stream(gd_sssp* s, const uint8_t* kind, const T* src, const T* dst, const T* w, int64_t k,
                           int64_t batch_size, int64_t first_batch_index, int64_t* dist, int64_t* parent) {
    return algo_run_stream(s, kind, src, dst, w, k, batch_size, first_batch_index, [&](int64_t j) {
        if (!dist && !parent) return;
        const void* dev[2];
        void* host[2];
        size_t bytes[2];
        int na = 0;
        const size_t n = (size_t)s->a->g->n;
        if (dist) {
            dev[na] = s->a->dist.get();
            host[na] = dist;
            bytes[na++] = n * 8;
        }
        if (parent) {
            dev[na] = s->a->parent_i64();
            host[na] = parent;
            bytes[na++] = n * 8;
        }
        s->a->stream_result((int)(j & 1), na, dev, host, bytes);
    });
}
extern "C" {
int gd_sssp_run_stream(gd_sssp* s, const uint8_t* kind, const int64_t* src, const int64_t* dst, const int64_t* w,
                       int64_t k, int64_t batch_size, int64_t first_batch_index, int64_t* dist, int64_t* parent) {
    return sssp_run_stream(s, kind, src, dst, w, k, batch_size, first_batch_index, dist, parent);
}
int gd_sssp_run_stream32(gd_sssp* s, const uint8_t* kind, const int32_t* src, const int32_t* dst, const int32_t* w,
                         int64_t k, int64_t batch_size, int64_t first_batch_index, int64_t* dist, int64_t* parent) {
    return sssp_run_stream(s, kind, src, dst, w, k, batch_size, first_batch_index, dist, parent);
}
int gd_sssp_destroy(gd_sssp* s) {
    if (!s) return ok();
    return guard([&] {
        cudaSetDevice(s->a->g->device);
        cudaStreamSynchronize(s->a->stream());
        delete s->a;
        delete s;
    });
}

int gd_pr_create(gd_graph* g, double damping, double beta, int64_t maxiter, gd_pr** out) {
    ALGO_CREATE(gdb::PR, gd_pr, new gdb::PR(g->st.get(), damping, beta, maxiter));
}
int gd_pr_batch(gd_pr* p, const uint8_t* kind, const int64_t* src, const int64_t* dst, const int64_t* w, int64_t k,
                int64_t bi) {
    return algo_batch_host(p, kind, src, dst, w, k, bi);
}
int gd_pr_batch_device(gd_pr* p, const uint8_t* kind, const int32_t* src, const int32_t* dst, const int32_t* w,
                       int64_t k, int64_t bi) {
    return algo_batch_dev(p, kind, src, dst, w, k, bi);
}
int gd_pr_read(gd_pr* p, double* rank, int64_t* outdeg) {
    if (!p) return null_handle();
    return guard([&] {
        GD_CUDA(cudaSetDevice(p->a->g->device));
        p->a->gather();
        p->a->read(rank, outdeg);
    });
}
int gd_pr_read_affected(gd_pr* p, uint8_t* affected) {
    if (!p) return null_handle();
    return guard([&] {
        GD_CUDA(cudaSetDevice(p->a->g->device));
        p->a->gather();
        p->a->read_affected(affected);
    });
}
int gd_pr_read_async(gd_pr* p, double* rank) {
    if (!p) return null_handle();
    return guard([&] {
        GD_CUDA(cudaSetDevice(p->a->g->device));
        p->a->gather();
        p->a->copy_out_async(rank, p->a->rank.get(), (size_t)p->a->g->n * 8, 0);
    });
}
int gd_pr_rank_device(gd_pr* p, const double** rank) {
    if (!p) return null_handle();
    return guard([&] {
        GD_CUDA(cudaSetDevice(p->a->g->device));
        p->a->gather();
        *rank = p->a->rank.get();
    });
}
}  // extern "C"
template <typename T>
static int pr_run_stream(gd_pr* p, const uint8_t* kind, const T* src, const T* dst, const T* w, int64_t k,
                         int64_t batch_size, int64_t first_batch_index, double* rank) {
    return algo_run_stream(p, kind, src, dst, w, k, batch_size, first_batch_index, [&](int64_t j) {
        if (!rank) return;
        p->a->gather();
        const void* dev[1] = {p->a->rank.get()};
        void* host[1] = {rank};
        const size_t bytes[1] = {(size_t)p->a->g->n * 8};
        p->a->stream_result((int)(j & 1), 1, dev, host, bytes);
    });
}
extern "C" {
int gd_pr_run_stream(gd_pr* p, const uint8_t* kind, const int64_t* src, const int64_t* dst, const int64_t* w,
                     int64_t k, int64_t batch_size, int64_t first_batch_index, double* rank) {
    return pr_run_stream(p, kind, src, dst, w, k, batch_size, first_batch_index, rank);
}
int gd_pr_run_stream32(gd_pr* p, const uint8_t* kind, const int32_t* src, const int32_t* dst, const int32_t* w,
                       int64_t k, int64_t batch_size, int64_t first_batch_index, double* rank) {
    return pr_run_stream(p, kind, src, dst, w, k, batch_size, first_batch_index, rank);
}
int gd_pr_destroy(gd_pr* p) {
    if (!p) return ok();
    return guard([&] {
        cudaSetDevice(p->a->g->device);
        cudaStreamSynchronize(p->a->stream());
        delete p->a;
        delete p;
    });
}

int gd_tc_create(gd_graph* g, gd_tc** out) { ALGO_CREATE(gdb::TC, gd_tc, new gdb::TC(g->st.get())); }
int gd_tc_batch(gd_tc* t, const uint8_t* kind, const int64_t* src, const int64_t* dst, const int64_t* w, int64_t k,
                int64_t bi) {
    return algo_batch_host(t, kind, src, dst, w, k, bi);
}
int gd_tc_batch_device(gd_tc* t, const uint8_t* kind, const int32_t* src, const int32_t* dst, const int32_t* w,
                       int64_t k, int64_t bi) {
    return algo_batch_dev(t, kind, src, dst, w, k, bi);
}
int gd_tc_read(gd_tc* t, int64_t* count) {
    if (!t) return null_handle();
    *count = t->a->count;
    return ok();
}
int gd_tc_run_stream(gd_tc* t, const uint8_t* kind, const int64_t* src, const int64_t* dst, const int64_t* w,
                     int64_t k, int64_t batch_size, int64_t first_batch_index, int64_t* counts) {
    return algo_run_stream(t, kind, src, dst, w, k, batch_size, first_batch_index, [&](int64_t j) {
        if (counts) counts[j] = t->a->count;
    });
}
int gd_tc_run_stream32(gd_tc* t, const uint8_t* kind, const int32_t* src, const int32_t* dst, const int32_t* w,
                       int64_t k, int64_t batch_size, int64_t first_batch_index, int64_t* counts) {
    return algo_run_stream(t, kind, src, dst, w, k, batch_size, first_batch_index, [&](int64_t j) {
        if (counts) counts[j] = t->a->count;
    });
}
int gd_tc_destroy(gd_tc* t) {
    if (!t) return ok();
    return guard([&] {
        cudaSetDevice(t->a->g->device);
        cudaStreamSynchronize(t->a->stream());
        delete t->a;
        delete t;
    });
}

int gd_comm_unique_id(uint8_t id[128]) {
    return guard([&] { gdb::comm_unique_id(id); });
}
int gd_comm_create(int world, int rank, const uint8_t id[128], int device, gd_comm** out) {
    return guard([&] {
        if (!out) throw gdb::GdError(GD_ERR_CONTRACT, "null output handle");
        auto* h = new gd_comm{nullptr};
        try {
            h->c = gdb::comm_create(world, rank, id, device);
        } catch (...) {
            delete h;
            throw;
        }
        *out = h;
    });
}
// ---- the store's device primitives on host arrays (tests) ----
int gd_prim_sort(int key_bytes, void* keys, int32_t* vals, int64_t n, int end_bit, int device) {
    return guard([&] {
        GD_CUDA(cudaSetDevice(device));
        cudaStream_t s = nullptr;
        GD_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
        {
            gdb::DBuf<uint64_t> k((n * key_bytes + 7) / 8 + 1, s);
            gdb::DBuf<int32_t> v(vals ? n + 1 : 0, s);
            GD_CUDA(cudaMemcpyAsync(k.get(), keys, n * key_bytes, cudaMemcpyHostToDevice, s));
            if (vals) GD_CUDA(cudaMemcpyAsync(v.get(), vals, n * 4, cudaMemcpyHostToDevice, s));
            if (key_bytes == 8 && vals) gdb::sort_pairs_u64(s, k.get(), v.get(), n, end_bit);
            else if (key_bytes == 8) gdb::sort_keys_u64(s, k.get(), n, end_bit);
            else if (key_bytes == 4 && vals)
                gdb::sort_pairs_u32(s, reinterpret_cast<uint32_t*>(k.get()), v.get(), n, end_bit);
            else throw gdb::GdError(GD_ERR_CONTRACT, "key_bytes 8 (values optional) or 4 (with values)");
            GD_CUDA(cudaMemcpyAsync(keys, k.get(), n * key_bytes, cudaMemcpyDeviceToHost, s));
            if (vals) GD_CUDA(cudaMemcpyAsync(vals, v.get(), n * 4, cudaMemcpyDeviceToHost, s));
            GD_CUDA(cudaStreamSynchronize(s));
        }
        gdb::dev_cache_release(s);
        GD_CUDA(cudaStreamSynchronize(s));
        cudaStreamDestroy(s);
    });
}

int gd_prim_scan_select(const int64_t* in, int64_t* out, const uint8_t* flags, int32_t* idx, int64_t n,
                        int64_t* count, int device) {
    return guard([&] {
        GD_CUDA(cudaSetDevice(device));
        cudaStream_t s = nullptr;
        GD_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
        {
            gdb::DBuf<int64_t> a(n + 1, s), b(n + 1, s), c(1, s);
            gdb::DBuf<uint8_t> f(n + 1, s);
            gdb::DBuf<int32_t> o(n + 1, s);
            GD_CUDA(cudaMemcpyAsync(a.get(), in, n * 8, cudaMemcpyHostToDevice, s));
            GD_CUDA(cudaMemcpyAsync(f.get(), flags, n, cudaMemcpyHostToDevice, s));
            gdb::exclusive_scan_i64(s, a.get(), b.get(), n);
            gdb::select_flagged_index_async(s, f.get(), n, o.get(), c.get());
            GD_CUDA(cudaMemcpyAsync(out, b.get(), n * 8, cudaMemcpyDeviceToHost, s));
            GD_CUDA(cudaMemcpyAsync(count, c.get(), 8, cudaMemcpyDeviceToHost, s));
            GD_CUDA(cudaMemcpyAsync(idx, o.get(), n * 4, cudaMemcpyDeviceToHost, s));
            GD_CUDA(cudaStreamSynchronize(s));
        }
        gdb::dev_cache_release(s);
        GD_CUDA(cudaStreamSynchronize(s));
        cudaStreamDestroy(s);
    });
}

int gd_comm_create_local(int world, int rank, int64_t group, int device, gd_comm** out) {
    return guard([&] {
        if (!out) throw gdb::GdError(GD_ERR_CONTRACT, "null output handle");
        auto* h = new gd_comm{nullptr};
        try {
            h->c = gdb::comm_create_local(world, rank, group, device);
        } catch (...) {
            delete h;
            throw;
        }
        *out = h;
    });
}
int gd_comm_destroy(gd_comm* c) {
    if (!c) return ok();
    return guard([&] {
        gdb::comm_destroy(c->c);
        delete c;
    });
}
int gd_comm_stats(const gd_comm* c, int64_t out[4]) {
    if (!c || !c->c) return null_handle();
    out[0] = c->c->n_calls;
    out[1] = c->c->ag_bytes;
    out[2] = c->c->ar_bytes;
    out[3] = c->c->sent_bytes;
    return ok();
}

int gd_comm_stats_ex(const gd_comm* c, int64_t out[5]) {
    if (!c || !c->c) return null_handle();
    gd_comm_stats(c, out);
    out[4] = c->c->p2p_bytes;
    return ok();
}

int gd_comm_reset_stats(gd_comm* c) {
    if (!c || !c->c) return null_handle();
    c->c->n_calls = c->c->ag_bytes = c->c->ar_bytes = c->c->sent_bytes = c->c->p2p_bytes = 0;
    return ok();
}

int gd_pr_set_comm(gd_pr* p, gd_comm* c) {
    if (!p) return null_handle();
    return guard([&] {
        GD_CUDA(cudaSetDevice(p->a->g->device));
        p->a->set_comm(c ? c->c : nullptr);
    });
}
int gd_tc_set_comm(gd_tc* t, gd_comm* c) {
    if (!t) return null_handle();
    return guard([&] { t->a->comm = c ? c->c : nullptr; });
}

int gd_phase_times(const void* h, double ms[5]) {
    if (!h) return null_handle();
    gdb::AlgoBase* a = algo_of(h);
    for (int i = 0; i < 5; ++i) ms[i] = a->timer.total_ms[i];
    return ok();
}

int gd_iterations(const void* h, int64_t* it) {
    if (!h) return null_handle();
    *it = algo_of(h)->iterations;
    return ok();
}

int gd_kernel_time(const void* h, const char* name, double* ms, int64_t* launches, int64_t* bytes) {
    if (!h) return null_handle();
    gdb::AlgoBase* a = algo_of(h);
    a->prof.flush();
    auto it = a->prof.last.find(name);
    if (it == a->prof.last.end()) {
        *ms = 0;
        *launches = 0;
        if (bytes) *bytes = 0;
    } else {
        *ms = it->second.ms;
        *launches = it->second.launches;
        if (bytes) *bytes = it->second.bytes;
    }
    return ok();
}

int gd_kernel_time_total(const void* h, const char* name, double* ms, int64_t* launches, int64_t* bytes) {
    if (!h) return null_handle();
    gdb::AlgoBase* a = algo_of(h);
    a->prof.flush();
    auto it = a->prof.total.find(name);
    bool hit = it != a->prof.total.end();
    *ms = hit ? it->second.ms : 0;
    *launches = hit ? it->second.launches : 0;
    if (bytes) *bytes = hit ? it->second.bytes : 0;
    return ok();
}

int gd_set_profiling(const void* h, int on) {
    if (!h) return null_handle();
    gdb::KernelProf& p = algo_of(h)->prof;
    if (on && !p.on) {
        p.flush();
        p.total.clear();
    }
    p.on = on != 0;
    return ok();
}

}  // extern "C"
