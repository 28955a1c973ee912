// gd_sssp.cu -- dynamic SSSP (programs/sssp_dynamic.sp:8-158,
// tests/golden/sssp_dynamic_omp.cc:10-261) on the GPU store.
//
// The reference's fixedPoint loops scan all V every round, filtered by a flag;
// here every fixpoint is a sparse frontier (queue + per-node round stamp for
// de-duplication).  Distances are int64 with the reference's saturating add
// and INF = INT64_MAX; relaxations use 64-bit atomicMin.  The final
// distances, the stale set (tree walk) and the touched set (nodes whose
// distance dropped) are schedule-independent, so the min-id parent fix-up
// over exactly those sets (sssp_dynamic.sp:23-34,87-98,118-129) reproduces the
// reference's `parent` array bit for bit.
//
// Why dist and parent are separate words rather than a packed 64-bit
// (dist:32|parent:32) atomicMin: a packed min breaks ties toward the smaller
// relaxing id and would rewrite the parent of nodes whose distance did not
// change -- nodes the reference leaves alone (S8 in SURVEY.md §8(a)).
#include <cooperative_groups.h>

#include <climits>

#include "gd_sssp.cuh"

namespace gdb {

namespace cg = cooperative_groups;

namespace {

constexpr int kThreads = 256;
constexpr int kG = 8;  // lanes per vertex
constexpr int kPerWarp = 32 / kG;

// warp-aggregated queue append over the currently converged lanes
__device__ inline void enqueue(int32_t* q, unsigned long long* cnt, int32_t v) {
    cg::coalesced_group g = cg::coalesced_threads();
    unsigned long long base = 0;
    if (g.thread_rank() == 0) base = atomicAdd(cnt, (unsigned long long)g.size());
    base = g.shfl(base, 0);
    q[base + g.thread_rank()] = v;
}

__device__ inline bool claim(int32_t* stamp, int32_t v, int32_t round) { return atomicMax(&stamp[v], round) < round; }

#define GROUP_LOOP_BEGIN(M)                                                      \
    const int lane = threadIdx.x & (kG - 1);                                     \
    const int gw = (threadIdx.x & 31) / kG;                                      \
    int64_t _warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;       \
    int64_t _nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;                    \
    for (int64_t _t0 = _warp * kPerWarp; _t0 < (M); _t0 += _nwarps * kPerWarp) { \
        int64_t _t = _t0 + gw;                                                   \
        bool valid = _t < (M);
#define GROUP_LOOP_END }

__global__ void k_init(int64_t* dist, int32_t* parent, int32_t* stamp, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        dist[i] = kInf;
        parent[i] = -1;
        stamp[i] = 0;
    }
}

__global__ void k_set_i64(int64_t* a, int64_t i, int64_t v) { a[i] = v; }

// push relaxation of one frontier round (sssp_dynamic.sp:15-21,110-117)
__global__ void __launch_bounds__(kThreads) k_relax(const int32_t* fq, int64_t m, OutView ov, int64_t* dist,
                                                    int32_t* stamp, int32_t round, int32_t* nq,
                                                    unsigned long long* ncnt, uint8_t* touched) {
    GROUP_LOOP_BEGIN(m)
    int32_t v = valid ? fq[_t] : 0;
    int64_t dv = valid ? dist[v] : kInf;
    if (dv < kInf) {
        for (int sg = 0; sg < ov.nseg; ++sg) {
            const int64_t* off = ov.off[sg];
            const int32_t* col = ov.col[sg];
            const int32_t* w = ov.w[sg];
            int64_t a = off[v], b = off[v + 1];
            for (int64_t e = a + lane; e < b; e += kG) {
                int32_t t = col[e];
                if (t < 0) continue;
                int64_t c = sat_add(dv, w ? (int64_t)w[e] : 1);
                if (c < dist[t]) {
                    long long old = atomicMin(reinterpret_cast<long long*>(&dist[t]), (long long)c);
                    if (c < old) {
                        if (touched) touched[t] = 1;
                        if (claim(stamp, t, round)) enqueue(nq, ncnt, t);
                    }
                }
            }
        }
    }
    GROUP_LOOP_END
}

// descend the parent tree from invalidated nodes (sssp_dynamic.sp:45-63)
__global__ void __launch_bounds__(kThreads) k_walk(const int32_t* fq, int64_t m, OutView ov, int64_t* dist,
                                                   int32_t* parent, uint8_t* stale, int32_t* stamp, int32_t round,
                                                   int32_t* nq, unsigned long long* ncnt) {
    GROUP_LOOP_BEGIN(m)
    if (valid) {
        int32_t v = fq[_t];
        for (int sg = 0; sg < ov.nseg; ++sg) {
            const int64_t* off = ov.off[sg];
            const int32_t* col = ov.col[sg];
            int64_t a = off[v], b = off[v + 1];
            for (int64_t e = a + lane; e < b; e += kG) {
                int32_t t = col[e];
                if (t < 0) continue;
                if (parent[t] == v) {
                    dist[t] = kInf;
                    parent[t] = -1;
                    stale[t] = 1;
                    if (claim(stamp, t, round)) enqueue(nq, ncnt, t);
                }
            }
        }
    }
    GROUP_LOOP_END
}

// stale nodes pull Min(dist[v], dist[u] + w) over live in-arcs; a node whose
// distance dropped re-queues its stale out-neighbours (sssp_dynamic.sp:68-86)
__global__ void __launch_bounds__(kThreads) k_pull(const int32_t* fq, int64_t m, IdxView ix, OutView ov,
                                                   int64_t* dist, const uint8_t* stale, int32_t* stamp,
                                                   int32_t round, int32_t* nq, unsigned long long* ncnt) {
    GROUP_LOOP_BEGIN(m)
    int32_t v = valid ? fq[_t] : 0;
    int64_t best = kInf;
    if (valid) {
        int64_t a = ix.off[v], b = ix.off[v + 1];
        for (int64_t e = a + lane; e < b; e += kG) {
            int32_t u = ix.col[e];
            if (u < 0) continue;
            int64_t c = sat_add(dist[u], ix.w ? (int64_t)ix.w[e] : 1);
            best = c < best ? c : best;
        }
    }
#pragma unroll
    for (int o = kG / 2; o; o >>= 1) {
        long long x = __shfl_xor_sync(0xffffffffu, (long long)best, o, kG);
        best = x < best ? x : best;
    }
    bool changed = false;
    if (valid && lane == 0 && best < dist[v]) {
        long long old = atomicMin(reinterpret_cast<long long*>(&dist[v]), (long long)best);
        changed = best < old;
    }
    changed = __shfl_sync(0xffffffffu, changed, (threadIdx.x & 31) & ~(kG - 1));
    if (changed) {
        for (int sg = 0; sg < ov.nseg; ++sg) {
            const int64_t* off = ov.off[sg];
            const int32_t* col = ov.col[sg];
            int64_t a = off[v], b = off[v + 1];
            for (int64_t e = a + lane; e < b; e += kG) {
                int32_t t = col[e];
                if (t < 0) continue;
                if (stale[t] && claim(stamp, t, round)) enqueue(nq, ncnt, t);
            }
        }
    }
    GROUP_LOOP_END
}

// parent = min-id in-neighbour u with dist[u] + w == dist[v] (sssp_dynamic.sp:23-34)
__global__ void __launch_bounds__(kThreads) k_fix_parent(const int32_t* list, int64_t m, IdxView ix,
                                                         const int64_t* dist, int32_t* parent, int32_t src) {
    GROUP_LOOP_BEGIN(m)
    int32_t v = valid ? (list ? list[_t] : (int32_t)_t) : 0;
    int64_t dv = valid ? dist[v] : kInf;
    bool act = valid && v != src && dv < kInf;
    int32_t best = INT_MAX;
    if (act) {
        int64_t a = ix.off[v], b = ix.off[v + 1];
        for (int64_t e = a + lane; e < b; e += kG) {
            int32_t u = ix.col[e];
            if (u < 0) continue;
            if (sat_add(dist[u], ix.w ? (int64_t)ix.w[e] : 1) == dv && u < best) best = u;
        }
    }
#pragma unroll
    for (int o = kG / 2; o; o >>= 1) {
        int32_t x = __shfl_xor_sync(0xffffffffu, best, o, kG);
        best = x < best ? x : best;
    }
    if (act && lane == 0) parent[v] = best == INT_MAX ? -1 : best;
    GROUP_LOOP_END
}

// OnDelete (sssp_dynamic.sp:139-146): a tree-edge deletion invalidates dst
__global__ void k_on_delete(const int32_t* s, const int32_t* d, int64_t k, int64_t* dist, int32_t* parent,
                            uint8_t* seed) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < k; i += (int64_t)gridDim.x * blockDim.x) {
        int32_t t = d[i];
        if (parent[t] == s[i]) {
            dist[t] = kInf;
            parent[t] = -1;
            seed[t] = 1;
        }
    }
}

// OnAdd (sssp_dynamic.sp:149-154)
__global__ void k_on_add(const int32_t* s, const int32_t* d, const int32_t* w, int64_t k, bool weighted,
                         int64_t* dist, uint8_t* seed) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < k; i += (int64_t)gridDim.x * blockDim.x) {
        int32_t t = d[i];
        // the record's own weight, as the reference's OnAdd reads e.weight of
        // the batch record (interp.py:624-629), weighted graph or not
        int64_t c = sat_add(dist[s[i]], (int64_t)w[i]);
        (void)weighted;
        if (c < dist[t]) {
            long long old = atomicMin(reinterpret_cast<long long*>(&dist[t]), (long long)c);
            if (c < old) seed[t] = 1;
        }
    }
}

__global__ void k_read_parent(const int32_t* p, int64_t n, int64_t* out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = p[i];
}

inline unsigned group_grid(int64_t m) { return grid_for(((m + kPerWarp - 1) / kPerWarp) * 32, kThreads, 148LL * 32); }

}  // namespace

SSSP::SSSP(Store* st, int64_t s) : AlgoBase(ALGO_SSSP, st), src((int32_t)s) {
    if (!st->with_reverse)
        throw GdError(GD_ERR_CONFIG, "graph was loaded without reverse-adjacency maintenance");
    if (s < 0 || s >= st->n) throw GdError(GD_ERR_EXEC, "source node out of range");
    cudaStream_t cs = stream();
    int64_t n = g->n;
    dist.alloc(n, cs);
    parent.alloc(n, cs);
    stamp.alloc(n, cs);
    fa.alloc(n, cs);
    fb.alloc(n, cs);
    fr.init(n, cs);
    ProfScope ps(&prof);
    timer.begin(PH_STATIC);
    GD_KERNEL(k_init, grid_for(n, 256), 256, 0, cs, dist.get(), parent.get(), stamp.get(), n);
    GD_KERNEL(k_set_i64, 1, 1, 0, cs, dist.get(), (int64_t)src, (int64_t)0);
    int32_t seed = src;
    DBuf<int32_t> sq(1, cs);
    GD_CUDA(cudaMemcpyAsync(sq.get(), &seed, 4, cudaMemcpyHostToDevice, cs));
    relax_push(sq.get(), 1, nullptr);
    fix_parents(nullptr, n);
    timer.end_all();
    prof.flush();
}

void SSSP::check_cap(int64_t it) {
    if (it >= cap_factor * std::max<int64_t>(g->n, 1)) throw GdError(GD_ERR_DIVERGED, "fixed point diverged");
}

int64_t SSSP::relax_push(const int32_t* seeds, int64_t nseeds, uint8_t* touched) {
    cudaStream_t s = stream();
    OutView ov = g->out_view();
    if (nseeds == 0) return 0;
    GD_CUDA(cudaMemcpyAsync(fr.q[0].get(), seeds, nseeds * 4, cudaMemcpyDeviceToDevice, s));
    int cur = 0;
    int64_t m = nseeds, it = 0;
    while (m > 0) {
        check_cap(it);
        ++round;
        GD_CUDA(cudaMemsetAsync(fr.cnt.get(), 0, sizeof(unsigned long long), s));
        GD_KERNEL_T("sssp_relax", 0, k_relax, group_grid(m), kThreads, 0, s, fr.q[cur].get(), m, ov, dist.get(),
                    stamp.get(), round, fr.q[1 - cur].get(), fr.cnt.get(), touched);
        m = (int64_t)read_scalar(s, fr.cnt.get());
        cur = 1 - cur;
        ++it;
    }
    iterations += it;
    return it;
}

int64_t SSSP::walk(const int32_t* seeds, int64_t nseeds, uint8_t* stale) {
    cudaStream_t s = stream();
    OutView ov = g->out_view();
    if (nseeds == 0) return 0;
    GD_CUDA(cudaMemcpyAsync(fr.q[0].get(), seeds, nseeds * 4, cudaMemcpyDeviceToDevice, s));
    int cur = 0;
    int64_t m = nseeds, it = 0;
    while (m > 0) {
        check_cap(it);
        ++round;
        GD_CUDA(cudaMemsetAsync(fr.cnt.get(), 0, sizeof(unsigned long long), s));
        GD_KERNEL_T("sssp_walk", 0, k_walk, group_grid(m), kThreads, 0, s, fr.q[cur].get(), m, ov, dist.get(),
                    parent.get(), stale, stamp.get(), round, fr.q[1 - cur].get(), fr.cnt.get());
        m = (int64_t)read_scalar(s, fr.cnt.get());
        cur = 1 - cur;
        ++it;
    }
    iterations += it;
    return it;
}

int64_t SSSP::pull(const int32_t* list, int64_t nstale, const uint8_t* stale) {
    cudaStream_t s = stream();
    OutView ov = g->out_view();
    IdxView ix = g->rev.view();
    if (nstale == 0) return 0;
    GD_CUDA(cudaMemcpyAsync(fr.q[0].get(), list, nstale * 4, cudaMemcpyDeviceToDevice, s));
    int cur = 0;
    int64_t m = nstale, it = 0;
    while (m > 0) {
        check_cap(it);
        ++round;
        GD_CUDA(cudaMemsetAsync(fr.cnt.get(), 0, sizeof(unsigned long long), s));
        GD_KERNEL_T("sssp_pull", 0, k_pull, group_grid(m), kThreads, 0, s, fr.q[cur].get(), m, ix, ov, dist.get(),
                    stale, stamp.get(), round, fr.q[1 - cur].get(), fr.cnt.get());
        m = (int64_t)read_scalar(s, fr.cnt.get());
        cur = 1 - cur;
        ++it;
    }
    iterations += it;
    return it;
}

void SSSP::fix_parents(const int32_t* list, int64_t m) {
    if (m == 0) return;
    GD_KERNEL_T("sssp_parent", 0, k_fix_parent, group_grid(m), kThreads, 0, stream(), list, m, g->rev.view(),
                dist.get(), parent.get(), src);
}

void SSSP::batch(DevBatch& b, int64_t batch_index) {
    cudaStream_t s = stream();
    int64_t n = g->n;
    ProfScope ps(&prof);
    prof.reset_last();
    uint8_t* seed_del = fa.get();  // activeOnDelete, then stale
    uint8_t* seed_add = fb.get();  // activeOnAdd, then touched
    DBuf<int32_t> list(std::max<int64_t>(n, 1), s);

    timer.begin(PH_PRE);
    fa.zero(s);
    fb.zero(s);
    if (b.kdel) GD_KERNEL(k_on_delete, grid_for(b.kdel, 256), 256, 0, s, b.ds.get(), b.dd.get(), b.kdel, dist.get(),
                          parent.get(), seed_del);
    timer.begin(PH_STRUCT);
    g->apply_deletes(b.ds.get(), b.dd.get(), b.kdel, nullptr);

    // decrementalSSSP (sssp_dynamic.sp:37-99); stale starts as the seeds
    timer.begin(PH_PROP);
    GD_KERNEL(k_set_i64, 1, 1, 0, s, dist.get(), (int64_t)src, (int64_t)0);
    int64_t nseed = select_flagged_index(s, seed_del, n, list.get());
    walk(list.get(), nseed, seed_del);
    GD_KERNEL(k_set_i64, 1, 1, 0, s, dist.get(), (int64_t)src, (int64_t)0);
    int64_t nstale = select_flagged_index(s, seed_del, n, list.get());
    pull(list.get(), nstale, seed_del);
    fix_parents(list.get(), nstale);

    timer.begin(PH_PRE);
    if (b.kadd) GD_KERNEL(k_on_add, grid_for(b.kadd, 256), 256, 0, s, b.as.get(), b.ad.get(), b.aw.get(), b.kadd,
                          g->weighted, dist.get(), seed_add);
    timer.begin(PH_STRUCT);
    g->apply_adds(b.as.get(), b.ad.get(), b.aw.get(), b.kadd);
    if (g->merge_due(batch_index)) {  // before the recompute; same live multiset
        timer.begin(PH_MERGE);
        g->merge();
    } else {
        g->compact_rev();
    }

    // incrementalSSSP (sssp_dynamic.sp:101-130); touched starts as the seeds
    timer.begin(PH_PROP);
    int64_t nadd = select_flagged_index(s, seed_add, n, list.get());
    relax_push(list.get(), nadd, seed_add);
    int64_t ntouched = select_flagged_index(s, seed_add, n, list.get());
    fix_parents(list.get(), ntouched);
    timer.end_all();
    prof.flush();
}

void SSSP::read(int64_t* h_dist, int64_t* h_parent) {
    cudaStream_t s = stream();
    int64_t n = g->n;
    if (!n) return;
    GD_CUDA(cudaMemcpyAsync(h_dist, dist.get(), n * 8, cudaMemcpyDeviceToHost, s));
    DBuf<int64_t> p(n, s);
    GD_KERNEL(k_read_parent, grid_for(n, 256), 256, 0, s, parent.get(), n, p.get());
    GD_CUDA(cudaMemcpyAsync(h_parent, p.get(), n * 8, cudaMemcpyDeviceToHost, s));
    GD_CUDA(cudaStreamSynchronize(s));
}

}  // namespace gdb
