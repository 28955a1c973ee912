// gd_algo.cu -- batch staging, validation, out-degrees and the weak-component flood.
#include <algorithm>

#include "gd_algo.cuh"

namespace gdb {

namespace {

// validation bits
constexpr int kBadKind = 1, kBadNode = 2, kBadWeight = 4;

template <typename T>  // host record ids: int64 (the C ABI) or int32 (the *_run_stream32 entry points)
__global__ void k_stage_host(const uint8_t* kind, const T* s64, const T* d64, const T* w64,
                             int64_t k, int64_t n, int32_t* s, int32_t* d, int32_t* w, uint8_t* isdel,
                             uint8_t* isadd, int* err, unsigned long long* bad_index) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < k; i += (int64_t)gridDim.x * blockDim.x) {
        uint8_t kd = kind[i];
        int64_t a = s64[i], b = d64[i];
        int64_t wt = w64 ? w64[i] : 1;
        int e = 0;
        if (kd != 'a' && kd != 'd') e |= kBadKind;
        if (a < 0 || a >= n || b < 0 || b >= n) e |= kBadNode;
        if (kd == 'a' && (wt < INT32_MIN || wt > INT32_MAX)) e |= kBadWeight;
        if (e) {
            atomicOr(err, e);
            atomicMax(bad_index, ~(unsigned long long)i);  // the first bad record, zero-initialised
        }
        s[i] = (int32_t)a;
        d[i] = (int32_t)b;
        w[i] = (int32_t)(kd == 'a' ? wt : 1);
        isdel[i] = kd == 'd';
        isadd[i] = kd == 'a';
    }
}

__global__ void k_stage_dev(const uint8_t* kind, const int32_t* s, const int32_t* d, int64_t k, int64_t n,
                            uint8_t* isdel, uint8_t* isadd, int* err, unsigned long long* bad_index) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < k; i += (int64_t)gridDim.x * blockDim.x) {
        uint8_t kd = kind[i];
        int e = 0;
        if (kd != 'a' && kd != 'd') e |= kBadKind;
        if (s[i] < 0 || s[i] >= n || d[i] < 0 || d[i] >= n) e |= kBadNode;
        if (e) {
            atomicOr(err, e);
            atomicMax(bad_index, ~(unsigned long long)i);  // the first bad record, zero-initialised
        }
        isdel[i] = kd == 'd';
        isadd[i] = kd == 'a';
    }
}

__global__ void k_gather_i32(const int32_t* in, const int32_t* sel, int64_t m, int32_t* out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = in[sel[i]];
}

}  // namespace

// Split validated records by kind in stream order.  `hdr` already holds
// [err, bad index, kdel, kadd] on the host (one sync for all of them).
void AlgoBase::split(DevBatch& b, const int32_t* sel_del, const int32_t* sel_add, const int32_t* s, const int32_t* d,
                     const int32_t* w, int64_t kdel, int64_t kadd) {
    cudaStream_t st = stream();
    b.kdel = kdel;
    b.kadd = kadd;
    b.ds.alloc(b.kdel, st);
    b.dd.alloc(b.kdel, st);
    if (b.kdel) {
        GD_KERNEL(k_gather_i32, grid_for(b.kdel, 256), 256, 0, st, s, sel_del, b.kdel, b.ds.get());
        GD_KERNEL(k_gather_i32, grid_for(b.kdel, 256), 256, 0, st, d, sel_del, b.kdel, b.dd.get());
    }
    b.as.alloc(b.kadd, st);
    b.ad.alloc(b.kadd, st);
    b.aw.alloc(b.kadd, st);
    if (b.kadd) {
        GD_KERNEL(k_gather_i32, grid_for(b.kadd, 256), 256, 0, st, s, sel_add, b.kadd, b.as.get());
        GD_KERNEL(k_gather_i32, grid_for(b.kadd, 256), 256, 0, st, d, sel_add, b.kadd, b.ad.get());
        if (w) GD_KERNEL(k_gather_i32, grid_for(b.kadd, 256), 256, 0, st, w, sel_add, b.kadd, b.aw.get());
        else fill_i32(st, b.aw.get(), b.kadd, 1);
    }
}

// message format of _validate_batch (engine/interp.py:563-570)
static void raise_validation(int err, unsigned long long idx, int64_t n, char kind, int64_t s, int64_t d) {
    if (err & kBadKind)
        throw GdError(GD_ERR_MALFORMED, "unknown update kind at record " + std::to_string(idx));
    if (err & kBadNode)
        throw GdError(GD_ERR_EXEC, std::string("update record ") + kind + " " + std::to_string(s) + " " +
                                       std::to_string(d) + " references a node outside [0, " + std::to_string(n) +
                                       ")");
    if (err & kBadWeight)
        throw GdError(GD_ERR_CONTRACT, "update record " + std::to_string(idx) +
                                           ": weight outside the int32 range of the B200 layout");
}

void AlgoBase::copy_out_async(void* host, const void* dev, size_t bytes, int slot) {
    cudaStream_t st = stream();
    if (!copy_stream) {
        GD_CUDA(cudaStreamCreateWithFlags(&copy_stream, cudaStreamNonBlocking));
        for (int k = 0; k < 2; ++k) {
            GD_CUDA(cudaEventCreateWithFlags(&ev_ready[k], cudaEventDisableTiming));
            GD_CUDA(cudaEventCreateWithFlags(&ev_copied[k], cudaEventDisableTiming));
            GD_CUDA(cudaEventRecord(ev_copied[k], copy_stream));
        }
    }
    if (!bytes) return;
    // the snapshot buffer may still feed the previous read of this slot
    GD_CUDA(cudaStreamWaitEvent(st, ev_copied[slot], 0));
    snap[slot].ensure(bytes, st);
    copy_d2d(st, snap[slot].get(), dev, bytes);
    GD_CUDA(cudaEventRecord(ev_ready[slot], st));
    GD_CUDA(cudaStreamWaitEvent(copy_stream, ev_ready[slot], 0));
    GD_CUDA(cudaMemcpyAsync(host, snap[slot].get(), bytes, cudaMemcpyDeviceToHost, copy_stream));
    GD_CUDA(cudaEventRecord(ev_copied[slot], copy_stream));
}

void AlgoBase::wait_copies() {
    if (copy_stream) GD_CUDA(cudaStreamSynchronize(copy_stream));
}

AlgoBase::~AlgoBase() {
    for (int k = 0; k < 2; ++k) {
        if (ev_up[k]) cudaEventDestroy(ev_up[k]);
        if (ev_staged[k]) cudaEventDestroy(ev_staged[k]);
        if (ev_sready[k]) cudaEventDestroy(ev_sready[k]);
        if (ev_scopied[k]) cudaEventDestroy(ev_scopied[k]);
    }
    if (copy_stream) {
        cudaStreamSynchronize(copy_stream);
        for (int k = 0; k < 2; ++k) {
            cudaEventDestroy(ev_ready[k]);
            cudaEventDestroy(ev_copied[k]);
        }
        cudaStreamDestroy(copy_stream);
    }
}

void AlgoBase::stage_host(DevBatch& b, const uint8_t* kind, const int64_t* src, const int64_t* dst,
                          const int64_t* w, int64_t k) {
    cudaStream_t st = stream();
    if (k == 0) {
        b.kdel = b.kadd = 0;
        return;
    }
    // record weights only matter to a weighted store or to SSSP's OnAdd
    // (which reads the record's own weight); skip their upload otherwise
    if (!g->weighted && this->kind != ALGO_SSSP) w = nullptr;
    h_stage.ensure(3 * k, st);
    k_stage.ensure(k, st);
    GD_CUDA(cudaMemcpyAsync(h_stage.get(), src, k * 8, cudaMemcpyHostToDevice, st));
    GD_CUDA(cudaMemcpyAsync(h_stage.get() + k, dst, k * 8, cudaMemcpyHostToDevice, st));
    if (w) GD_CUDA(cudaMemcpyAsync(h_stage.get() + 2 * k, w, k * 8, cudaMemcpyHostToDevice, st));
    GD_CUDA(cudaMemcpyAsync(k_stage.get(), kind, k, cudaMemcpyHostToDevice, st));
    stage_records(b, k_stage.get(), h_stage.get(), h_stage.get() + k, w ? h_stage.get() + 2 * k : nullptr, 8, k,
                  kind, src, dst);
}

// validate + split records already on the device as `width`-byte ids
void AlgoBase::stage_records(DevBatch& b, const uint8_t* dkind, const void* dsrc, const void* ddst, const void* dw,
                             int width, int64_t k, const uint8_t* kind, const void* src, const void* dst) {
    cudaStream_t st = stream();
    DBuf<int32_t> s(k, st), d(k, st), ww(k, st);
    DBuf<uint8_t> flags(2 * k, st);
    DBuf<int64_t> hdr(4, st);  // err, bad index, kdel, kadd
    fill_d(st, hdr.get(), 0, 16);
    if (width == 8)
        GD_KERNEL(k_stage_host<int64_t>, grid_for(k, 256), 256, 0, st, dkind, static_cast<const int64_t*>(dsrc),
                  static_cast<const int64_t*>(ddst), static_cast<const int64_t*>(dw), k, g->n, s.get(), d.get(),
                  ww.get(), flags.get(), flags.get() + k, reinterpret_cast<int*>(hdr.get()),
                  reinterpret_cast<unsigned long long*>(hdr.get() + 1));
    else
        GD_KERNEL(k_stage_host<int32_t>, grid_for(k, 256), 256, 0, st, dkind, static_cast<const int32_t*>(dsrc),
                  static_cast<const int32_t*>(ddst), static_cast<const int32_t*>(dw), k, g->n, s.get(), d.get(),
                  ww.get(), flags.get(), flags.get() + k, reinterpret_cast<int*>(hdr.get()),
                  reinterpret_cast<unsigned long long*>(hdr.get() + 1));
    DBuf<int32_t> sel_del(k, st), sel_add(k, st);
    select_flagged_index_async(st, flags.get(), k, sel_del.get(), hdr.get() + 2);
    select_flagged_index_async(st, flags.get() + k, k, sel_add.get(), hdr.get() + 3);
    int64_t h[4];
    read_small(st, h, hdr.get(), sizeof h);
    int e = (int)(h[0] & 0xffffffff);
    if (e) {
        unsigned long long i = ~(unsigned long long)h[1];
        auto at = [&](const void* p) {
            return width == 8 ? static_cast<const int64_t*>(p)[i] : (int64_t) static_cast<const int32_t*>(p)[i];
        };
        raise_validation(e, i, g->n, (char)kind[i], at(src), at(dst));
    }
    split(b, sel_del.get(), sel_add.get(), s.get(), d.get(), ww.get(), h[2], h[3]);
}

cudaStream_t AlgoBase::io_stream() {
    if (!copy_stream) copy_out_async(nullptr, nullptr, 0, 0);  // creates the stream and its events
    return copy_stream;
}

void AlgoBase::reserve_uploads(int64_t k) {
    cudaStream_t st = stream();
    io_stream();
    for (int j = 0; j < 2; ++j) {
        up64[j].ensure(3 * std::max<int64_t>(k, 1), st);
        upk[j].ensure(std::max<int64_t>(k, 1), st);
        if (!ev_up[j]) {
            GD_CUDA(cudaEventCreateWithFlags(&ev_up[j], cudaEventDisableTiming));
            GD_CUDA(cudaEventCreateWithFlags(&ev_staged[j], cudaEventDisableTiming));
            GD_CUDA(cudaEventRecord(ev_staged[j], st));
        }
    }
    GD_CUDA(cudaStreamSynchronize(st));  // the slots exist before the copy stream writes them
}

void AlgoBase::upload_async(int slot, const uint8_t* kind, const void* src, const void* dst, const void* w, int width,
                            int64_t k) {
    cudaStream_t io = io_stream();
    if (!g->weighted && this->kind != ALGO_SSSP) w = nullptr;
    up_w[slot] = w != nullptr;
    up_width[slot] = width;
    if (k == 0) return;
    // the slot's previous batch has been staged (its buffers are free)
    GD_CUDA(cudaStreamWaitEvent(io, ev_staged[slot], 0));
    char* u = reinterpret_cast<char*>(up64[slot].get());  // src | dst | w, k ids of `width` bytes each
    GD_CUDA(cudaMemcpyAsync(u, src, k * width, cudaMemcpyHostToDevice, io));
    GD_CUDA(cudaMemcpyAsync(u + k * width, dst, k * width, cudaMemcpyHostToDevice, io));
    if (w) GD_CUDA(cudaMemcpyAsync(u + 2 * k * width, w, k * width, cudaMemcpyHostToDevice, io));
    GD_CUDA(cudaMemcpyAsync(upk[slot].get(), kind, k, cudaMemcpyHostToDevice, io));
    GD_CUDA(cudaEventRecord(ev_up[slot], io));
}

void AlgoBase::stream_result(int par, int narr, const void* const* dev, void* const* host, const size_t* bytes) {
    cudaStream_t st = stream();
    cudaStream_t io = io_stream();
    if (has_pend) stream_flush();  // the previous batch queued no structural update
    if (!ev_sready[0])
        for (int k = 0; k < 2; ++k) {
            GD_CUDA(cudaEventCreateWithFlags(&ev_sready[k], cudaEventDisableTiming));
            GD_CUDA(cudaEventCreateWithFlags(&ev_scopied[k], cudaEventDisableTiming));
            GD_CUDA(cudaEventRecord(ev_scopied[k], io));
        }
    // the slot's previous read-back has left it
    GD_CUDA(cudaStreamWaitEvent(st, ev_scopied[par], 0));
    pend.par = par;
    pend.narr = narr;
    for (int i = 0; i < narr; ++i) {
        ssnap[par][i].ensure(std::max<size_t>(bytes[i], 1), st);
        copy_d2d(st, ssnap[par][i].get(), dev[i], bytes[i]);
        pend.host[i] = host[i];
        pend.bytes[i] = bytes[i];
    }
    GD_CUDA(cudaEventRecord(ev_sready[par], st));
    has_pend = true;
}

void AlgoBase::stream_flush() {
    if (!has_pend) return;
    has_pend = false;
    cudaStream_t io = io_stream();
    const int par = pend.par;
    GD_CUDA(cudaStreamWaitEvent(io, ev_sready[par], 0));
    for (int i = 0; i < pend.narr; ++i)
        if (pend.bytes[i])
            GD_CUDA(cudaMemcpyAsync(pend.host[i], ssnap[par][i].get(), pend.bytes[i], cudaMemcpyDeviceToHost, io));
    GD_CUDA(cudaEventRecord(ev_scopied[par], io));
}

void AlgoBase::stage_uploaded(DevBatch& b, int slot, const uint8_t* h_kind, const void* h_src, const void* h_dst,
                              int64_t k) {
    cudaStream_t st = stream();
    if (k == 0) {
        b.kdel = b.kadd = 0;
        return;
    }
    GD_CUDA(cudaStreamWaitEvent(st, ev_up[slot], 0));
    const int width = up_width[slot];
    const char* u = reinterpret_cast<const char*>(up64[slot].get());
    stage_records(b, upk[slot].get(), u, u + k * width, up_w[slot] ? u + 2 * k * width : nullptr, width, k, h_kind,
                  h_src, h_dst);
    GD_CUDA(cudaEventRecord(ev_staged[slot], st));
}

void AlgoBase::stage_device(DevBatch& b, const uint8_t* kind, const int32_t* src, const int32_t* dst,
                            const int32_t* w, int64_t k) {
    cudaStream_t st = stream();
    if (k == 0) {
        b.kdel = b.kadd = 0;
        return;
    }
    DBuf<uint8_t> flags(2 * k, st);
    DBuf<int64_t> hdr(4, st);  // err, bad index, kdel, kadd
    fill_d(st, hdr.get(), 0, 16);
    GD_KERNEL(k_stage_dev, grid_for(k, 256), 256, 0, st, kind, src, dst, k, g->n, flags.get(), flags.get() + k,
              reinterpret_cast<int*>(hdr.get()), reinterpret_cast<unsigned long long*>(hdr.get() + 1));
    DBuf<int32_t> sel_del(k, st), sel_add(k, st);
    select_flagged_index_async(st, flags.get(), k, sel_del.get(), hdr.get() + 2);
    select_flagged_index_async(st, flags.get() + k, k, sel_add.get(), hdr.get() + 3);
    int64_t h[4];
    read_small(st, h, hdr.get(), sizeof h);
    int e = (int)(h[0] & 0xffffffff);
    if (e) {
        unsigned long long i = ~(unsigned long long)h[1];
        raise_validation(e, i, g->n, (char)read_scalar(st, kind + i), read_scalar(st, src + i),
                         read_scalar(st, dst + i));
    }
    split(b, sel_del.get(), sel_add.get(), src, dst, w, h[2], h[3]);
}

// ---------------------------------------------------------------- degrees ---

namespace {
__global__ void k_out_degrees(OutView ov, int64_t n, int32_t* deg) {
    // one thread per row for the count over all segments; warp-cooperative
    // reading is not needed: rows are read once and coalescing across rows is
    // poor only for long rows, which the warp path below handles.
    const int lane = threadIdx.x & 31;
    int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t v0 = warp * 32; v0 < n; v0 += nwarps * 32) {
        // 32 consecutive rows per warp: each lane owns one row
        int64_t v = v0 + lane;
        int32_t d = 0;
        if (v < n) {
            for (int sg = 0; sg < ov.nseg; ++sg) {
                const int64_t* off = ov.off[sg];
                const int32_t* col = ov.col[sg];
                for (int64_t i = off[v]; i < off[v + 1]; ++i) d += col[i] >= 0;
            }
            deg[v] = d;
        }
    }
}
}  // namespace

void out_degrees(Store& g, int32_t* deg) {
    if (g.n == 0) return;
    GD_KERNEL(k_out_degrees, grid_for(g.n, 256), 256, 0, g.stream, g.out_view(), g.n, deg);
}

// ------------------------------------------------------------------ flood ---

namespace {

// Parents only ever decrease (a root is hooked under a smaller root), so the
// walk terminates; path halving re-points each visited node at its
// grandparent (atomicMin keeps concurrent halvings monotone).
__device__ inline int32_t uf_find(int32_t* p, int32_t v) {
    int32_t cur = v;
    while (true) {
        int32_t nx = p[cur];
        if (nx == cur) return cur;
        int32_t nn = p[nx];
        if (nn < nx) atomicMin(&p[cur], nn);
        cur = nx;
    }
}

// hook the larger root under the smaller (deterministic result: roots are
// component minima after compression)
__device__ inline void uf_union(int32_t* p, int32_t a, int32_t b) {
    while (true) {
        a = uf_find(p, a);
        b = uf_find(p, b);
        if (a == b) return;
        if (a > b) {
            int32_t t = a;
            a = b;
            b = t;
        }
        // b is the larger root: try p[b] = a
        int32_t old = atomicCAS(&p[b], b, a);
        if (old == b) return;
        b = old;
    }
}

__global__ void k_uf_init(int32_t* p, int64_t n, uint8_t* root_has_seed) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        p[i] = (int32_t)i;
        root_has_seed[i] = 0;
    }
}

// Afforest-style connectivity (Sutton et al. 2018): link every vertex to its
// first kSample live out-arcs, find the dominant component, then only the
// vertices outside it process their remaining arcs -- in BOTH directions,
// because an arc is stored at its source only.  Same components as linking
// every arc, at a fraction of the arc reads (the giant component of an R-MAT
// graph holds ~all non-isolated vertices).
#ifndef GD_AFF_SAMPLE
#define GD_AFF_SAMPLE 2
#endif
constexpr int kSample = GD_AFF_SAMPLE;

__global__ void k_aff_sample(OutView ov, int64_t n, int32_t* p) {
    const int64_t* off = ov.off[0];
    const int32_t* col = ov.col[0];
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
        int64_t a = off[v], b = off[v + 1];
        // the first kSample slots, loaded together (a tombstone among them
        // just means fewer samples: the rest pass links every arc anyway)
        int32_t c[kSample];
#pragma unroll
        for (int k = 0; k < kSample; ++k) c[k] = a + k < b ? col[a + k] : -1;
#pragma unroll
        for (int k = 0; k < kSample; ++k)
            if (c[k] >= 0 && c[k] != (int32_t)v) uf_union(p, (int32_t)v, c[k]);
    }
}

__global__ void k_uf_compress(int32_t* p, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        p[i] = uf_find(p, (int32_t)i);
}

// the probes' roots (finds, so the forest need not be compressed first)
__global__ void k_aff_gather(int32_t* p, int64_t n, int32_t* out, int m) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x)
        out[i] = uf_find(p, (int32_t)((unsigned long long)i * 2654435761ULL % (unsigned long long)n));
}

// the most frequent root among the probe samples (one CTA; ties -> smaller
// root, as the host version chose the first of the sorted runs)
__global__ void k_aff_giant(const int32_t* probe, int m, int32_t* giant) {
    __shared__ int32_t sv[1024];
    __shared__ unsigned long long best;
    for (int i = threadIdx.x; i < m; i += blockDim.x) sv[i] = probe[i];
    if (threadIdx.x == 0) best = ~0ULL;
    __syncthreads();
    for (int i = threadIdx.x; i < m; i += blockDim.x) {
        int c = 0;
        for (int j = 0; j < m; ++j) c += sv[j] == sv[i];
        // max count first, then the smaller root: minimise (~count, root)
        unsigned long long key = ((unsigned long long)(0xffffffffu - (unsigned)c) << 32) | (unsigned)sv[i];
        atomicMin(&best, key);
    }
    __syncthreads();
    if (threadIdx.x == 0) *giant = (int32_t)(best & 0xffffffffu);
}

// Vertices outside the dominant component link the rest of their out-arcs
// (base after the sampled ones, then every delta) and all their in-arcs.
// rows with more than kRestWarp remaining arcs go to a warp each
constexpr int64_t kRestWarp = 64;

__device__ inline void aff_link_row(OutView ov, IdxView in, int32_t v, int32_t* p, int lane, int stride) {
    for (int sg = 0; sg < ov.nseg; ++sg) {
        const int64_t* off = ov.off[sg];
        const int32_t* col = ov.col[sg];
        int64_t a = off[v], b = off[v + 1];
        for (int64_t i = (sg == 0 ? a + kSample : a) + lane; i < b; i += stride) {  // base slots < kSample: sampled
            int32_t c = col[i];
            if (c >= 0 && c != v) uf_union(p, v, c);
        }
    }
    if (in.off) {
        for (int64_t e = in.off[v] + lane; e < in.off[v + 1]; e += stride) {
            int32_t u = in.col[e];
            if (u >= 0 && u != v) uf_union(p, v, u);
        }
    }
}

__global__ void k_aff_rest(OutView ov, IdxView in, int64_t n, const int32_t* giant_p, int32_t* p) {
    const int32_t giant = *giant_p;
    const int lane = threadIdx.x & 31;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    // 32 consecutive vertices per warp step: the loop stays warp-uniform so
    // that a hub outside the giant can be linked by the whole warp
    for (int64_t v0 = (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 32; v0 < n; v0 += nwarps * 32) {
        const int64_t v = v0 + lane;
        bool need = false;
        int64_t more = 0;
        if (v < n) {
            // the root test and the arc counts load together; isolated
            // vertices (42% of R-MAT V) and sampled-only ones stop here
            const int32_t pv = p[v];
            const int64_t b0 = ov.off[0][v], e0 = ov.off[0][v + 1];
            const int64_t ia = in.off ? in.off[v] : 0, ib = in.off ? in.off[v + 1] : 0;
            more = max(e0 - b0 - kSample, (int64_t)0) + (ib - ia);
            for (int sg = 1; sg < ov.nseg; ++sg) more += ov.off[sg][v + 1] - ov.off[sg][v];
            need = more > 0 && pv != giant && uf_find(p, (int32_t)v) != giant;
        }
        const bool heavy = need && more > kRestWarp;
        if (need && !heavy) aff_link_row(ov, in, (int32_t)v, p, 0, 1);
        for (unsigned hm = __ballot_sync(0xffffffffu, heavy); hm; hm &= hm - 1) {  // a hub: the whole warp
            const int32_t hv = __shfl_sync(0xffffffffu, (int32_t)v, __ffs(hm) - 1);
            aff_link_row(ov, in, hv, p, lane, 32);
        }
    }
}

__global__ void k_uf_compress_seed(int32_t* p, int64_t n, const uint8_t* flags, uint8_t* root_has_seed) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        int32_t r = uf_find(p, (int32_t)i);
        p[i] = r;
        // read before writing: ~all flagged vertices share the giant's root,
        // and a million stores to one address serialise in L2
        if (flags[i] && !root_has_seed[r]) root_has_seed[r] = 1;
    }
}

__global__ void k_i32_to_u8(const int32_t* a, uint8_t* b) { *b = *a ? 1 : 0; }

__global__ void k_uf_mark(const int32_t* p, int64_t n, const uint8_t* root_has_seed, uint8_t* flags) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        if (root_has_seed[p[i]]) flags[i] = 1;
}

}  // namespace

namespace {

// adopt the smallest label any rank gives v: hook v's local root under it
__global__ void k_uf_adopt(int32_t* p, const int32_t* L, int64_t n, int32_t* changed) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
        const int32_t l = L[v];
        if (l < uf_find(p, (int32_t)v)) {
            uf_union(p, (int32_t)v, l);
            *changed = 1;
        }
    }
}

}  // namespace

int64_t flood_weak_components_dist(Store& g, uint8_t* flags, KernelProf* prof) {
    (void)prof;
    cudaStream_t s = g.stream;
    const int64_t n = g.n;
    if (n == 0) return 0;
    IdxView in{nullptr, nullptr, nullptr};
    if (g.rev.built) {
        g.compact_rev();
        in = g.rev.view();
    }
    // Afforest over the partition: sample-link the first kSample out-arcs of
    // the owned rows, agree on labels (rounds of a min-label all-reduce: every
    // rank hooks each vertex under the smallest root any rank knows for it,
    // until no rank changes), find the dominant component on the agreed
    // labels, then only vertices outside it link their remaining out-arcs
    // and their in-arcs -- an arc between two giant vertices is already
    // joined, any other has an endpoint outside it whose owner holds the arc
    // (out-row or in-row) -- and agree once more.  The labels end as the
    // weak components' minimum ids, the same on every rank.
    DBuf<int32_t> p(n, s), L(n, s), ch(1, s);
    DBuf<uint8_t> seed(n, s), a(1, s);
    int64_t rounds = 0;
    auto agree = [&] {
        while (true) {
            ++rounds;
            copy_d2d(s, L.get(), p.get(), n * 4);
            g.part->allreduce_min_i32(L.get(), n, s);
            fill_d(s, ch.get(), 0, 4);
            GD_KERNEL(k_uf_adopt, grid_for(n, 256), 256, 0, s, p.get(), L.get(), n, ch.get());
            GD_KERNEL(k_uf_compress, grid_for(n, 256), 256, 0, s, p.get(), n);
            GD_KERNEL(k_i32_to_u8, 1, 1, 0, s, ch.get(), a.get());
            g.part->allreduce_max_u8(a.get(), 1, s);
            uint8_t any = 0;
            read_small(s, &any, a.get(), 1);
            if (!any) break;
        }
    };
    OutView ov = g.out_view();
    GD_KERNEL(k_uf_init, grid_for(n, 256), 256, 0, s, p.get(), n, seed.get());
    GD_KERNEL_T("flood_sample", 0, k_aff_sample, grid_for(n, 256), 256, 0, s, ov, n, p.get());
    GD_KERNEL(k_uf_compress, grid_for(n, 256), 256, 0, s, p.get(), n);
    agree();
    constexpr int kProbe = 256;
    DBuf<int32_t> probe(kProbe, s), giant(1, s);
    GD_KERNEL(k_aff_gather, 4, 256, 0, s, p.get(), n, probe.get(), kProbe);
    GD_KERNEL(k_aff_giant, 1, kProbe, 0, s, probe.get(), kProbe, giant.get());
    GD_KERNEL_T("flood_rest", 0, k_aff_rest, grid_for(n, 256), 256, 0, s, ov, in, n, giant.get(), p.get());
    GD_KERNEL(k_uf_compress, grid_for(n, 256), 256, 0, s, p.get(), n);
    agree();
    // the same labels on every rank: flag every vertex whose component holds a seed
    GD_KERNEL_T("flood_mark", 0, k_uf_compress_seed, grid_for(n, 256), 256, 0, s, p.get(), n, flags, seed.get());
    GD_KERNEL(k_uf_mark, grid_for(n, 256), 256, 0, s, p.get(), n, seed.get(), flags);
    return rounds;
}

int64_t flood_weak_components(Store& g, uint8_t* flags, KernelProf* prof) {
    (void)prof;
    cudaStream_t s = g.stream;
    int64_t n = g.n;
    if (n == 0) return 0;
    // in-arcs are needed for directed graphs (interp.py:82-85 requires reverse)
    IdxView in{nullptr, nullptr, nullptr};
    if (g.directed) {
        g.require_rev();
        g.compact_rev();
        in = g.rev.view();
    }
    DBuf<int32_t> p(n, s);
    DBuf<uint8_t> seed(n, s);  // zeroed by k_uf_init
    OutView ov = g.out_view();
    GD_KERNEL(k_uf_init, grid_for(n, 256), 256, 0, s, p.get(), n, seed.get());
    GD_KERNEL_T("flood_sample", n * (8 + 4 * kSample), k_aff_sample, grid_for(n, 256), 256, 0, s, ov, n, p.get());
    // the rest pass and the final compression find roots anyway: no full
    // compression pass in between (GD_FLOOD_COMPRESS=1 restores it, A/B)
    static const bool compress = getenv("GD_FLOOD_COMPRESS") != nullptr;
    if (compress) GD_KERNEL(k_uf_compress, grid_for(n, 256), 256, 0, s, p.get(), n);
    constexpr int kProbe = 256;  // the giant component holds ~all non-isolated vertices
    DBuf<int32_t> probe(kProbe, s);
    GD_KERNEL(k_aff_gather, 4, 256, 0, s, p.get(), n, probe.get(), kProbe);
    DBuf<int32_t> giant(1, s);
    GD_KERNEL(k_aff_giant, 1, kProbe, 0, s, probe.get(), kProbe, giant.get());
    GD_KERNEL_T("flood_rest", 0, k_aff_rest, grid_for(n, 256), 256, 0, s, ov, in, n, giant.get(), p.get());
    GD_KERNEL_T("flood_mark", 0, k_uf_compress_seed, grid_for(n, 256), 256, 0, s, p.get(), n, flags, seed.get());
    GD_KERNEL(k_uf_mark, grid_for(n, 256), 256, 0, s, p.get(), n, seed.get(), flags);
    return 1;
}

}  // namespace gdb
