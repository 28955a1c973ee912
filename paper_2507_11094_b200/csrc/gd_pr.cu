// gd_pr.cu -- dynamic PageRank (programs/pr_dynamic.sp:7-102,
// tests/golden/pr_dynamic_omp.cc:9-138) on the GPU store.
//
// Per batch: OnDelete/OnAdd bookkeeping (affected marks, +-1 out-degree for
// every record, misses included), the structural update, merge-if-due, the
// weak-component flood of `affected`, then the incremental power iteration
// over the affected vertices only (dangling mass still summed over all V).
// fp64 throughout; per-term values rank[u]/outdeg[u] are computed exactly as
// the reference computes them, only the summation order differs.
#include <cmath>

#include "gd_algo.cuh"
#include "gd_pr.cuh"

namespace gdb {

namespace {

constexpr int kPullThreads = 256;
constexpr int kRedBlocks = 148 * 4;

__global__ void k_pr_init(double* rank, int64_t n, double v) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        rank[i] = v;
}

// contrib[u] = rank[u] / outdeg[u]; per-block partial of the dangling sum
// (outdeg == 0) -- pr_dynamic_omp.cc:68-73.
__global__ void __launch_bounds__(256) k_pr_contrib(const double* rank, const int32_t* outdeg, int64_t n,
                                                    double* contrib, double* partial) {
    double acc = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        double r = rank[i];
        int32_t d = outdeg[i];
        contrib[i] = r / (double)d;
        if (d == 0) acc += r;
    }
    __shared__ double sh[256 / 32];
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < 256 / 32; ++w) t += sh[w];
        partial[blockIdx.x] = t;
    }
}

// deterministic final sum of the partials (fixed order)
__global__ void k_sum_partials(const double* partial, int np, double* out) {
    __shared__ double sh[1024];
    double t = 0.0;
    for (int i = threadIdx.x; i < np; i += blockDim.x) t += partial[i];
    sh[threadIdx.x] = t;
    __syncthreads();
    for (int s = blockDim.x / 2; s; s >>= 1) {
        if ((int)threadIdx.x < s) sh[threadIdx.x] += sh[threadIdx.x + s];
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = sh[0];
}

__device__ inline double atomic_max_pos(double* a, double v) {  // v >= 0
    return __longlong_as_double(atomicMax(reinterpret_cast<long long*>(a), __double_as_longlong(v)));
}

// The pull for one affected vertex v (pr_dynamic_omp.cc:75-98):
// incoming = sum(contrib[src]) over the in-arcs, new rank, |delta|.  Three
// kernels by in-degree bin so lanes stay busy on a skewed (R-MAT) graph:
// light rows (<= 32 in-arcs) get 8 lanes, medium rows (<= 4096) a warp, hub
// rows a 512-thread block.  Every lane keeps 4 loads in flight (column ids
// first, then the contrib gathers) to cover L2 latency.  Reductions are in a
// fixed order, so results are deterministic run to run.
constexpr int kLightMax = 32;
constexpr int kMediumMax = 4096;
constexpr int kHubThreads = 512;
constexpr int kILP = 4;

template <int G>
__device__ inline double row_sum(const int32_t* __restrict__ col, int64_t a, int64_t b, int lane,
                                 const double* __restrict__ contrib) {
    double acc = 0.0;
    for (int64_t e0 = a + lane; e0 < b; e0 += G * kILP) {
        int32_t u[kILP];
#pragma unroll
        for (int q = 0; q < kILP; ++q) {
            int64_t e = e0 + q * G;
            u[q] = e < b ? __ldcs(&col[e]) : -1;  // streamed once per sweep
        }
        double c[kILP];
#pragma unroll
        for (int q = 0; q < kILP; ++q) c[q] = u[q] >= 0 ? __ldg(&contrib[u[q]]) : 0.0;
#pragma unroll
        for (int q = 0; q < kILP; ++q) acc += c[q];
    }
    return acc;
}

template <int G>
__global__ void __launch_bounds__(kPullThreads) k_pr_pull_group(const int32_t* list, int64_t m, IdxView ix,
                                                                  const double* contrib, const double* rank,
                                                                  const double* dangling, double base,
                                                                  double damping, double inv_n, double* rank_new,
                                                                  double* diff) {
    const int lane = threadIdx.x & (G - 1);
    const int gw = (threadIdx.x & 31) / G;
    constexpr int kPer = 32 / G;
    int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const double dn = *dangling * inv_n;
    double dmax = 0.0;
    for (int64_t t0 = warp * kPer; t0 < m; t0 += nwarps * kPer) {  // warp-uniform trip count
        int64_t t = t0 + gw;
        bool valid = t < m;
        int32_t v = valid ? list[t] : 0;
        int64_t a = valid ? ix.off[v] : 0, b = valid ? ix.off[v + 1] : 0;
        double acc = row_sum<G>(ix.col, a, b, lane, contrib);
#pragma unroll
        for (int o = G / 2; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o, G);
        if (valid && lane == 0) {
            double nr = base + damping * (acc + dn);
            dmax = fmax(dmax, fabs(nr - rank[v]));
            rank_new[v] = nr;
        }
    }
    for (int o = 16; o; o >>= 1) dmax = fmax(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
    if ((threadIdx.x & 31) == 0 && dmax > 0.0) atomic_max_pos(diff, dmax);
}

__global__ void __launch_bounds__(kHubThreads) k_pr_pull_hub(const int32_t* list, int64_t m, IdxView ix,
                                                              const double* contrib, const double* rank,
                                                              const double* dangling, double base, double damping,
                                                              double inv_n, double* rank_new, double* diff) {
    __shared__ double sh[kHubThreads / 32];
    const double dn = *dangling * inv_n;
    for (int64_t t = blockIdx.x; t < m; t += gridDim.x) {
        int32_t v = list[t];
        double acc = row_sum<kHubThreads>(ix.col, ix.off[v], ix.off[v + 1], threadIdx.x, contrib);
        for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = acc;
        __syncthreads();
        if (threadIdx.x == 0) {
            double sum = 0.0;
            for (int w = 0; w < kHubThreads / 32; ++w) sum += sh[w];
            double nr = base + damping * (sum + dn);
            double dl = fabs(nr - rank[v]);
            if (dl > 0.0) atomic_max_pos(diff, dl);
            rank_new[v] = nr;
        }
        __syncthreads();
    }
}

__global__ void k_pr_commit(const int32_t* list, int64_t m, const double* rank_new, double* rank) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
        int32_t v = list[i];
        rank[v] = rank_new[v];
    }
}

// OnDelete / OnAdd handlers (pr_dynamic.sp:87-97): mark both endpoints,
// outdeg[src] -= 1 (deletes, misses included) / += 1 (adds).
__global__ void k_pr_onupdate(const int32_t* s, const int32_t* d, int64_t k, int32_t delta, uint8_t* affected,
                              int32_t* outdeg) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < k; i += (int64_t)gridDim.x * blockDim.x) {
        affected[s[i]] = 1;
        affected[d[i]] = 1;
        atomicAdd(&outdeg[s[i]], delta);
    }
}

// in-arcs of each bin (for the roofline's algorithmic bytes)
__global__ void k_bin_arcs(const int32_t* list, int64_t m, const int64_t* off, unsigned long long* sums) {
    unsigned long long a[3] = {0, 0, 0};
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
        int32_t v = list[i];
        int64_t d = off[v + 1] - off[v];
        a[d <= kLightMax ? 0 : (d <= kMediumMax ? 1 : 2)] += (unsigned long long)d;
    }
    for (int k = 0; k < 3; ++k) {
        unsigned long long x = a[k];
        for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
        if ((threadIdx.x & 31) == 0 && x) atomicAdd(&sums[k], x);
    }
}

__global__ void k_gather_list(const int32_t* list, const int32_t* sel, int64_t m, int32_t* out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = list[sel[i]];
}

}  // namespace

PR::PR(Store* st, double d, double b, int64_t mi) : AlgoBase(ALGO_PR, st), damping(d), beta(b), maxiter(mi) {
    if (!st->with_reverse)
        throw GdError(GD_ERR_CONFIG, "graph was loaded without reverse-adjacency maintenance");
    cudaStream_t s = stream();
    int64_t n = g->n;
    rank.alloc(std::max<int64_t>(n, 1), s);
    rank_new.alloc(std::max<int64_t>(n, 1), s);
    contrib.alloc(std::max<int64_t>(n, 1), s);
    outdeg.alloc(std::max<int64_t>(n, 1), s);
    affected.alloc(std::max<int64_t>(n, 1), s);
    partial.alloc(kRedBlocks, s);
    scal.alloc(2, s);  // [0] dangling, [1] diff
    ProfScope ps(&prof);
    timer.begin(PH_STATIC);
    if (n) {
        GD_KERNEL(k_pr_init, grid_for(n, 256), 256, 0, s, rank.get(), n, 1.0 / (double)n);
        out_degrees(*g, outdeg.get());
    }
    // staticPR: every node participates
    DBuf<int32_t> all(n, s);
    iota_i32(s, all.get(), n);
    set_lists(all.get(), n);
    power_loop();
    timer.end_all();
    prof.flush();
}

namespace {
__global__ void k_range_bounds(const int32_t* list, int64_t m, int32_t lo, int32_t hi, int64_t* out) {
    if (threadIdx.x == 0) out[0] = lower_bound_dev<int32_t>(list, 0, m, lo);
    if (threadIdx.x == 1) out[1] = lower_bound_dev<int32_t>(list, 0, m, hi);
}
}  // namespace

void PR::set_comm(Comm* c) {
    cudaStream_t s = stream();
    int64_t n = g->n;
    comm = c;
    if (!c) return;
    // rank / rank_new padded to chunk * world for the in-place all-gather
    int64_t npad = std::max<int64_t>(c->chunk(n) * c->world, 1);
    DBuf<double> r2(npad, s), n2(npad, s);
    r2.zero(s);
    n2.zero(s);
    if (n) {
        GD_CUDA(cudaMemcpyAsync(r2.get(), rank.get(), n * 8, cudaMemcpyDeviceToDevice, s));
        GD_CUDA(cudaMemcpyAsync(n2.get(), rank_new.get(), n * 8, cudaMemcpyDeviceToDevice, s));
    }
    rank = std::move(r2);
    rank_new = std::move(n2);
    GD_CUDA(cudaStreamSynchronize(s));
}

void PR::set_lists(const int32_t* list, int64_t m) {
    cudaStream_t s = stream();
    g->compact_rev();
    if (comm && m) {  // the list is ascending: keep the owned destination range
        DBuf<int64_t> b(2, s);
        GD_KERNEL(k_range_bounds, 1, 32, 0, s, list, m, (int32_t)comm->lo(g->n), (int32_t)comm->hi(g->n), b.get());
        int64_t hb[2];
        GD_CUDA(cudaMemcpyAsync(hb, b.get(), sizeof hb, cudaMemcpyDeviceToHost, s));
        GD_CUDA(cudaStreamSynchronize(s));
        list += hb[0];
        m = hb[1] - hb[0];
    }
    for (auto* l : {&bins[0], &bins[1], &bins[2]}) l->ensure(std::max<int64_t>(m, 1), s);
    nbin[0] = nbin[1] = nbin[2] = 0;
    ebin[0] = ebin[1] = ebin[2] = 0;
    if (!m) return;
    DBuf<int> cnt(2, s);
    DBuf<unsigned long long> sums(3, s);
    sums.zero(s);
    partition3_by_degree(s, list, m, g->rev.off.get(), kLightMax, kMediumMax, bins[0].get(), bins[1].get(),
                         bins[2].get(), cnt.get());
    GD_KERNEL(k_bin_arcs, grid_for(m, 256, 148LL * 8), 256, 0, s, list, m, g->rev.off.get(), sums.get());
    int hc[2];
    unsigned long long hs[3];
    GD_CUDA(cudaMemcpyAsync(hc, cnt.get(), sizeof hc, cudaMemcpyDeviceToHost, s));
    GD_CUDA(cudaMemcpyAsync(hs, sums.get(), sizeof hs, cudaMemcpyDeviceToHost, s));
    GD_CUDA(cudaStreamSynchronize(s));
    nbin[0] = hc[0];
    nbin[1] = hc[1];
    nbin[2] = m - hc[0] - hc[1];
    for (int k = 0; k < 3; ++k) ebin[k] = (int64_t)hs[k];
}

// while (diff >= beta && iter < maxiter) { dangling; pull; commit }
void PR::power_loop() {
    cudaStream_t s = stream();
    int64_t n = g->n;
    if (n == 0) return;
    IdxView ix = g->rev.view();
    const double base = (1.0 - damping) / (double)n;
    const double inv_n = 1.0 / (double)n;
    int64_t iter = 0;
    double diff = beta + 1.0;
    last_sweeps = 0;
    while (diff >= beta && iter < maxiter) {
        GD_KERNEL_T("pr_contrib", n * 20, k_pr_contrib, kRedBlocks, 256, 0, s, rank.get(), outdeg.get(), n,
                    contrib.get(), partial.get());
        GD_KERNEL(k_sum_partials, 1, 1024, 0, s, partial.get(), kRedBlocks, scal.get());
        GD_CUDA(cudaMemsetAsync(scal.get() + 1, 0, sizeof(double), s));
        // algorithmic bytes: |A| (off + 2 f64) + E_in(A) (idx + f64)
        if (nbin[0])
            GD_KERNEL_T("pr_pull", nbin[0] * 24 + ebin[0] * 12, k_pr_pull_group<2>,
                        grid_for(((nbin[0] + 15) / 16) * 32, kPullThreads, 148LL * 32), kPullThreads, 0, s,
                        bins[0].get(), nbin[0], ix, contrib.get(), rank.get(), scal.get(), base, damping, inv_n,
                        rank_new.get(), scal.get() + 1);
        if (nbin[1])
            GD_KERNEL_T("pr_pull", nbin[1] * 24 + ebin[1] * 12, k_pr_pull_group<16>,
                        grid_for(((nbin[1] + 1) / 2) * 32, kPullThreads, 148LL * 32), kPullThreads, 0, s, bins[1].get(),
                        nbin[1], ix, contrib.get(), rank.get(), scal.get(), base, damping, inv_n, rank_new.get(),
                        scal.get() + 1);
        if (nbin[2])
            GD_KERNEL_T("pr_pull", nbin[2] * 24 + ebin[2] * 12, k_pr_pull_hub,
                        (unsigned)std::min<int64_t>(nbin[2], 148LL * 4), kHubThreads, 0, s, bins[2].get(), nbin[2],
                        ix, contrib.get(), rank.get(), scal.get(), base, damping, inv_n, rank_new.get(),
                        scal.get() + 1);
        for (int k = 0; k < 3; ++k)
            if (nbin[k])
                GD_KERNEL(k_pr_commit, grid_for(nbin[k], 256), 256, 0, s, bins[k].get(), nbin[k], rank_new.get(),
                          rank.get());
        if (comm) {  // every rank gets every owned range; the residual is the max over ranks
            comm->allgather_f64(rank.get(), comm->chunk(n), s);
            comm->allreduce_max_f64(scal.get() + 1, 1, s);
        }
        diff = read_scalar(s, scal.get() + 1);
        ++iter;
    }
    last_sweeps = iter;
    iterations += iter;
}

void PR::batch(DevBatch& b, int64_t batch_index) {
    cudaStream_t s = stream();
    int64_t n = g->n;
    ProfScope ps(&prof);
    prof.reset_last();
    timer.begin(PH_PRE);
    affected.zero(s);
    if (b.kdel) GD_KERNEL(k_pr_onupdate, grid_for(b.kdel, 256), 256, 0, s, b.ds.get(), b.dd.get(), b.kdel, -1,
                          affected.get(), outdeg.get());
    if (b.kadd) GD_KERNEL(k_pr_onupdate, grid_for(b.kadd, 256), 256, 0, s, b.as.get(), b.ad.get(), b.kadd, 1,
                          affected.get(), outdeg.get());
    timer.begin(PH_STRUCT);
    g->apply_deletes(b.ds.get(), b.dd.get(), b.kdel, nullptr);
    g->apply_adds(b.as.get(), b.ad.get(), b.aw.get(), b.kadd);
    // merge-if-due runs before the recompute: it does not change the live
    // multiset the recompute reads (interp.py:877-880 runs it after).
    if (g->merge_due(batch_index)) {
        timer.begin(PH_MERGE);
        g->merge();
    }
    timer.begin(PH_PROP);
    flood_weak_components(*g, affected.get(), &prof);
    DBuf<int32_t> list(std::max<int64_t>(n, 1), s);
    int64_t m = select_flagged_index(s, affected.get(), n, list.get());
    last_affected = m;
    set_lists(list.get(), m);
    power_loop();
    timer.end_all();
    prof.flush();
}

void PR::read(double* h_rank, int64_t* h_outdeg) {
    cudaStream_t s = stream();
    int64_t n = g->n;
    if (!n) return;
    GD_CUDA(cudaMemcpyAsync(h_rank, rank.get(), n * 8, cudaMemcpyDeviceToHost, s));
    if (h_outdeg) {
        std::vector<int32_t> tmp(n);
        GD_CUDA(cudaMemcpyAsync(tmp.data(), outdeg.get(), n * 4, cudaMemcpyDeviceToHost, s));
        GD_CUDA(cudaStreamSynchronize(s));
        for (int64_t i = 0; i < n; ++i) h_outdeg[i] = tmp[i];
    }
    GD_CUDA(cudaStreamSynchronize(s));
}

}  // namespace gdb
