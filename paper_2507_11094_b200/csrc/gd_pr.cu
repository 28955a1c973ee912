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
// Device control block of the sweep loop (no host round trip per sweep):
// ctl[0..2] bin sizes, ctl[3..5] in-arcs per bin, ctl[6] done, ctl[7] sweeps.
// Sweeps are enqueued ahead; once ctl[6] is set, the queued ones return at
// their first instruction.
enum { C_NBIN = 0, C_EBIN = 3, C_DONE = 6, C_SWEEPS = 7, C_WORK = 8, C_WORK2 = 9, C_LEN = 10 };

__global__ void __launch_bounds__(256) k_pr_contrib(const double* rank, const int32_t* outdeg, int64_t n,
                                                    double* contrib, double* partial, const int64_t* ctl) {
    if (ctl && ctl[C_DONE]) return;
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

// deterministic final sum of the partials (fixed order); clears the sweep's
// residual
__global__ void k_sum_partials(const double* partial, int np, double* out, int64_t* ctl) {
    if (ctl && ctl[C_DONE]) return;
    __shared__ double sh[1024];
    double t = 0.0;
    for (int i = threadIdx.x; i < np; i += blockDim.x) t += partial[i];
    sh[threadIdx.x] = t;
    __syncthreads();
    for (int s = blockDim.x / 2; s; s >>= 1) {
        if ((int)threadIdx.x < s) sh[threadIdx.x] += sh[threadIdx.x + s];
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        out[0] = sh[0];
        out[1] = 0.0;
        if (ctl) {  // the fused pull's work counters
            ctl[C_WORK] = 0;
            ctl[C_WORK2] = 0;
        }
    }
}

__device__ inline double atomic_max_pos(double* a, double v) {  // v >= 0
    return __longlong_as_double(atomicMax(reinterpret_cast<long long*>(a), __double_as_longlong(v)));
}

// The pull for one affected vertex v (pr_dynamic_omp.cc:75-98):
// incoming = sum(contrib[src]) over the in-arcs, new rank, |delta|.  Three
// kernels by in-degree bin so lanes stay busy on a skewed (R-MAT) graph:
// light rows (<= 32 in-arcs) get 8 lanes, medium rows (<= 4096) a warp, hub
// rows a 512-thread block.  Every lane keeps 8 loads in flight (column ids
// first, then the contrib gathers) to cover L2 latency.  Reductions are in a
// fixed order, so results are deterministic run to run.
constexpr int kLightMax = 32;
constexpr int kMediumMax = 4096;
constexpr int kHubThreads = 512;
#ifndef GD_PR_ILP
#define GD_PR_ILP 8
#endif
constexpr int kILP = GD_PR_ILP;
#ifndef GD_PR_GATHER
#define GD_PR_GATHER __ldg  // contrib gathers through L1 (GD_PR_GATHER=__ldcg: L2 only, A/B)
#endif

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
        for (int q = 0; q < kILP; ++q) c[q] = u[q] >= 0 ? GD_PR_GATHER(&contrib[u[q]]) : 0.0;
#pragma unroll
        for (int q = 0; q < kILP; ++q) acc += c[q];
    }
    return acc;
}

template <int G>
__global__ void __launch_bounds__(kPullThreads) k_pr_pull_group(const int32_t* list, const int64_t* ctl, int bin,
                                                                  IdxView ix, const double* contrib,
                                                                  const double* rank, const double* dangling,
                                                                  double base, double damping, double inv_n,
                                                                  double* rank_new, double* diff) {
    if (ctl[C_DONE]) return;
    const int64_t m = ctl[C_NBIN + bin];
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

__global__ void __launch_bounds__(kHubThreads) k_pr_pull_hub(const int32_t* list, const int64_t* ctl, IdxView ix,
                                                              const double* contrib, const double* rank,
                                                              const double* dangling, double base, double damping,
                                                              double inv_n, double* rank_new, double* diff) {
    if (ctl[C_DONE]) return;
    const int64_t m = ctl[C_NBIN + 2];
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

// All three bins in one launch: CTAs take hub rows from one counter (a whole
// CTA per hub row), then each warp takes units of 12 medium rows (16 lanes
// each) or 96 light rows (2 lanes each) from a second one.  The serial bin launches left the latency-
// bound hub tail and the L1-bound medium bin unoverlapped; here they share the
// GPU.  Each row's sum keeps a fixed lane/order assignment: deterministic.
constexpr int kFusedThreads = 256;
#ifndef GD_PR_MED_UNIT
#define GD_PR_MED_UNIT 12
#endif
#ifndef GD_PR_LIGHT_UNIT
#define GD_PR_LIGHT_UNIT 96
#endif
#ifndef GD_PR_LG
#define GD_PR_LG 2
#endif
constexpr int kMedUnit = GD_PR_MED_UNIT;
constexpr int kLightUnit = GD_PR_LIGHT_UNIT;
constexpr int kLG = GD_PR_LG;  // lanes per light row

#ifdef GD_PULL_MINB
__global__ void __launch_bounds__(kFusedThreads, GD_PULL_MINB) k_pr_pull_fused(
#else
__global__ void __launch_bounds__(kFusedThreads) k_pr_pull_fused(
#endif
const int32_t* light, const int32_t* med,
                                                                 const int32_t* hub, int64_t* ctl, IdxView ix,
                                                                 const double* contrib, const double* rank,
                                                                 const double* dangling, double base, double damping,
                                                                 double inv_n, double* rank_new, double* diff) {
    if (ctl[C_DONE]) return;
    __shared__ long long unit_s;
    __shared__ double red[kFusedThreads / 32];
    const int64_t nl = ctl[C_NBIN], nm = ctl[C_NBIN + 1], nh = ctl[C_NBIN + 2];
    const double dn = *dangling * inv_n;
    const int tid = threadIdx.x, lane = tid & 31;
    double dmax = 0.0;
    // phase 1: hub rows, a whole CTA each
    while (true) {
        if (tid == 0) unit_s = (long long)atomicAdd(reinterpret_cast<unsigned long long*>(&ctl[C_WORK]), 1ULL);
        __syncthreads();
        const int64_t u = unit_s;
        __syncthreads();
        if (u >= nh) break;
        int32_t v = hub[u];
        double acc = row_sum<kFusedThreads>(ix.col, ix.off[v], ix.off[v + 1], tid, contrib);
        for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) red[tid >> 5] = acc;
        __syncthreads();
        if (tid == 0) {
            double sum = 0.0;
            for (int w = 0; w < kFusedThreads / 32; ++w) sum += red[w];
            double nr = base + damping * (sum + dn);
            dmax = fmax(dmax, fabs(nr - rank[v]));
            rank_new[v] = nr;
        }
        __syncthreads();
    }
    // phase 2: warps claim units on their own -- medium rows range from 33 to
    // 4096 in-arcs, and a CTA-wide claim made 8 warps wait for the longest
    // row at a barrier.  A unit is 12 medium rows (16 lanes each, 2 at a time)
    // or 96 light rows (2 lanes each, 16 at a time).
    const int64_t um = (nm + kMedUnit - 1) / kMedUnit, ul = (nl + kLightUnit - 1) / kLightUnit, total = um + ul;
    while (true) {
        unsigned long long w = 0;
        if (lane == 0) w = atomicAdd(reinterpret_cast<unsigned long long*>(&ctl[C_WORK2]), 1ULL);
        const int64_t u = (int64_t)__shfl_sync(0xffffffffu, w, 0);
        if (u >= total) break;
        if (u < um) {
            const int gl = lane & 15;
#pragma unroll 1
            for (int r = 0; r < kMedUnit; r += 2) {
                const int64_t t = u * kMedUnit + r + (lane >> 4);
                bool valid = t < nm;
                int32_t v = valid ? med[t] : 0;
                int64_t a = valid ? ix.off[v] : 0, b = valid ? ix.off[v + 1] : 0;
                double acc = row_sum<16>(ix.col, a, b, gl, contrib);
#pragma unroll
                for (int o = 8; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o, 16);
                if (valid && gl == 0) {
                    double nr = base + damping * (acc + dn);
                    dmax = fmax(dmax, fabs(nr - rank[v]));
                    rank_new[v] = nr;
                }
            }
        } else {
            const int gl = lane & (kLG - 1);
#pragma unroll 1
            for (int r = 0; r < kLightUnit; r += 32 / kLG) {
                const int64_t t = (u - um) * kLightUnit + r + lane / kLG;
                bool valid = t < nl;
                int32_t v = valid ? light[t] : 0;
                int64_t a = valid ? ix.off[v] : 0, b = valid ? ix.off[v + 1] : 0;
                double acc = row_sum<kLG>(ix.col, a, b, gl, contrib);
#pragma unroll
                for (int o = kLG / 2; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o, kLG);
                if (valid && gl == 0) {
                    double nr = base + damping * (acc + dn);
                    dmax = fmax(dmax, fabs(nr - rank[v]));
                    rank_new[v] = nr;
                }
            }
        }
    }
    for (int o = 16; o; o >>= 1) dmax = fmax(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
    if (lane == 0 && dmax > 0.0) atomic_max_pos(diff, dmax);
}

// Jacobi commit of all three bins
__global__ void k_pr_commit(const int32_t* b0, const int32_t* b1, const int32_t* b2, const int64_t* ctl,
                            const double* rank_new, double* rank) {
    if (ctl[C_DONE]) return;
    const int64_t n0 = ctl[C_NBIN], n1 = ctl[C_NBIN + 1], m = n0 + n1 + ctl[C_NBIN + 2];
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
        int32_t v = i < n0 ? b0[i] : (i < n0 + n1 ? b1[i - n0] : b2[i - n0 - n1]);
        rank[v] = rank_new[v];
    }
}

// while (diff >= beta && iter < maxiter): decide on the device whether the
// next queued sweep runs
__global__ void k_pr_check(int64_t* ctl, const double* diff, double beta, int64_t maxiter) {
    if (ctl[C_DONE]) return;
    int64_t it = ++ctl[C_SWEEPS];
    if (!(*diff >= beta && it < maxiter)) ctl[C_DONE] = 1;
}

// OnDelete / OnAdd handlers (pr_dynamic.sp:87-97): mark both endpoints,
// outdeg[src] -= 1 (deletes, misses included) / += 1 (adds).
__global__ void k_pr_onupdate(const int32_t* ds, const int32_t* dd, int64_t kdel, const int32_t* as,
                              const int32_t* ad, int64_t kadd, uint8_t* affected, int32_t* outdeg) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < kdel + kadd;
         i += (int64_t)gridDim.x * blockDim.x) {
        const bool del = i < kdel;
        const int32_t s = del ? ds[i] : as[i - kdel], d = del ? dd[i] : ad[i - kdel];
        affected[s] = 1;
        affected[d] = 1;
        atomicAdd(&outdeg[s], del ? -1 : 1);
    }
}

// affected vertices of [lo, hi) into the three in-degree bins, plus the
// in-arcs per bin.  A CTA stages a 2048-vertex chunk's bin entries in shared
// memory and claims each bin's output range with one atomic, so the three
// global counters see a few thousand atomics, not one per warp.  Bin order
// does not matter: every vertex's sum is computed on its own, in a fixed
// order.  flags == nullptr: every vertex (staticPR).
constexpr int kBinThreads = 256;
constexpr int kBinChunk = 2048;

__global__ void __launch_bounds__(kBinThreads) k_pr_bin(const uint8_t* flags, int64_t lo, int64_t hi,
                                                        const int64_t* off, int32_t* b0, int32_t* b1, int32_t* b2,
                                                        int64_t* ctl) {
    __shared__ int32_t stage[3][kBinChunk];
    __shared__ int cnt[3];
    __shared__ unsigned long long gbase[3];
    const int lane = threadIdx.x & 31;
    unsigned long long e[3] = {0, 0, 0};
    for (int64_t c0 = lo + (int64_t)blockIdx.x * kBinChunk; c0 < hi; c0 += (int64_t)gridDim.x * kBinChunk) {
        if (threadIdx.x < 3) cnt[threadIdx.x] = 0;
        __syncthreads();
#pragma unroll 2
        for (int j = threadIdx.x; j < kBinChunk; j += kBinThreads) {
            int64_t v = c0 + j;
            bool in = v < hi && (!flags || flags[v]);
            int64_t d = in ? off[v + 1] - off[v] : 0;
            int b = d <= kLightMax ? 0 : (d <= kMediumMax ? 1 : 2);
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                unsigned mk = __ballot_sync(0xffffffffu, in && b == k);
                if (!mk) continue;
                int base = 0;
                if (lane == 0) base = atomicAdd(&cnt[k], __popc(mk));
                base = __shfl_sync(0xffffffffu, base, 0);
                if (in && b == k) {
                    stage[k][base + __popc(mk & ((1u << lane) - 1))] = (int32_t)v;
                    e[k] += (unsigned long long)d;
                }
            }
        }
        __syncthreads();
        if (threadIdx.x < 3 && cnt[threadIdx.x])
            gbase[threadIdx.x] = atomicAdd(reinterpret_cast<unsigned long long*>(&ctl[C_NBIN + threadIdx.x]),
                                           (unsigned long long)cnt[threadIdx.x]);
        __syncthreads();
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            int32_t* out = k == 0 ? b0 : (k == 1 ? b1 : b2);
            for (int j = threadIdx.x; j < cnt[k]; j += kBinThreads) out[gbase[k] + j] = stage[k][j];
        }
        __syncthreads();
    }
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        unsigned long long x = e[k];
        for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
        if (lane == 0 && x) atomicAdd(reinterpret_cast<unsigned long long*>(&ctl[C_EBIN + k]), x);
    }
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
    affected.zero(s);  // propNode<bool> default before the first Batch
    partial.alloc(kRedBlocks, s);
    scal.alloc(2, s);  // [0] dangling, [1] diff
    ctl.alloc(C_LEN, s);
    for (auto* l : {&bins[0], &bins[1], &bins[2]}) l->alloc(std::max<int64_t>(n, 1), s);
    ProfScope ps(&prof);
    timer.begin(PH_STATIC);
    if (n) {
        GD_KERNEL(k_pr_init, grid_for(n, 256), 256, 0, s, rank.get(), n, 1.0 / (double)n);
        out_degrees(*g, outdeg.get());
    }
    recompute(nullptr);  // staticPR: every node participates
    timer.end_all();
}

void PR::set_comm(Comm* c) {
    if (c && g->part) throw GdError(GD_ERR_CONFIG, "the graph is partitioned: its handles use the graph's communicator");
    comm = c;
}

// One sweep (pr_dynamic_omp.cc:66-99): dangling mass + contrib over all V,
// the pull over the affected bins, the Jacobi commit, then (multi-GPU) the
// rank all-gather and the residual max, and the device-side loop test.
void PR::sweep(int64_t tag) {
    cudaStream_t s = stream();
    const int64_t n = g->n;
    IdxView ix = g->rev.view();
    const double base = (1.0 - damping) / (double)n;
    const double inv_n = 1.0 / (double)n;
    int64_t* c = ctl.get();
    const Comm* part = g->part;  // vertex-partitioned store: contrib of the owned sources, then gathered
    const int64_t clo = part ? g->own_lo : 0, cn = part ? g->own_hi - g->own_lo : n;
    int pc = prof_begin("pr_contrib", cn * 20, s);
    prof_tag(pc, tag);
    k_pr_contrib<<<kRedBlocks, 256, 0, s>>>(rank.get() + clo, outdeg.get() + clo, cn, contrib.get() + clo,
                                            partial.get(), c);
    count_launch();
    GD_LAUNCH_CHECK();
    prof_end(pc, s);
    GD_KERNEL(k_sum_partials, 1, 1024, 0, s, partial.get(), kRedBlocks, scal.get(), c);
    if (part) {  // dangling mass over all ranks; every rank's contrib block to every rank
        part->allreduce_sum_f64(scal.get(), 1, s);
        part->allgatherv(contrib.get(), g->blocks, 8, s);
    }
    // algorithmic bytes: |A| (off + 2 f64) + E_in(A) (idx + f64), filled in from the bin
    // counts once the loop has read them back
    static const bool split = getenv("GD_PR_SPLIT_BINS") != nullptr;
    if (!split) {
        int pi = prof_begin("pr_pull", 0, s);
        prof_tag(pi, tag);
        pull_recs.push_back({pi, -1});
        k_pr_pull_fused<<<148 * 8, kFusedThreads, 0, s>>>(bins[0].get(), bins[1].get(), bins[2].get(), c, ix,
                                                          contrib.get(), rank.get(), scal.get(), base, damping,
                                                          inv_n, rank_new.get(), scal.get() + 1);
        count_launch();
        GD_LAUNCH_CHECK();
        prof_end(pi, s);
    } else {
    int pi = prof_begin("pr_pull", 0, s);
    prof_tag(pi, tag);
    pull_recs.push_back({pi, 0});
    k_pr_pull_group<2><<<148 * 16, kPullThreads, 0, s>>>(bins[0].get(), c, 0, ix, contrib.get(), rank.get(),
                                                         scal.get(), base, damping, inv_n, rank_new.get(),
                                                         scal.get() + 1);
    count_launch();
    GD_LAUNCH_CHECK();
    prof_end(pi, s);
    pi = prof_begin("pr_pull", 0, s);
    prof_tag(pi, tag);
    pull_recs.push_back({pi, 1});
    k_pr_pull_group<16><<<148 * 16, kPullThreads, 0, s>>>(bins[1].get(), c, 1, ix, contrib.get(), rank.get(),
                                                          scal.get(), base, damping, inv_n, rank_new.get(),
                                                          scal.get() + 1);
    count_launch();
    GD_LAUNCH_CHECK();
    prof_end(pi, s);
    pi = prof_begin("pr_pull", 0, s);
    prof_tag(pi, tag);
    pull_recs.push_back({pi, 2});
    k_pr_pull_hub<<<148 * 2, kHubThreads, 0, s>>>(bins[2].get(), c, ix, contrib.get(), rank.get(), scal.get(), base,
                                                  damping, inv_n, rank_new.get(), scal.get() + 1);
    count_launch();
    GD_LAUNCH_CHECK();
    prof_end(pi, s);
    }
    GD_KERNEL(k_pr_commit, 148 * 8, 256, 0, s, bins[0].get(), bins[1].get(), bins[2].get(), c, rank_new.get(),
              rank.get());
    if (comm) {  // every rank gets every owned range; the residual is the max over ranks
        comm->allgatherv(rank.get(), Blocks(n, comm->world), 8, s);
        comm->allreduce_max_f64(scal.get() + 1, 1, s);
    }
    if (part) part->allreduce_max_f64(scal.get() + 1, 1, s);
    GD_KERNEL(k_pr_check, 1, 1, 0, s, c, scal.get() + 1, beta, maxiter);
}

// Bin the affected vertices (flags == nullptr: all) of this rank's range
// and run the sweep loop.  Sweeps are queued `ahead` at a time and the
// device-side test turns the surplus into no-ops, so the host reads the loop
// state once per group instead of once per sweep.
void PR::recompute(const uint8_t* flags) {
    cudaStream_t s = stream();
    const int64_t n = g->n;
    last_sweeps = 0;
    if (n == 0) return;
    g->compact_rev();
    fill_d(s, ctl.get(), 0, C_LEN * sizeof(int64_t));
    if (maxiter <= 0) return;
    const int64_t lo = g->part ? g->own_lo : (comm ? Blocks(n, comm->world).lo(comm->rank) : 0);
    const int64_t hi = g->part ? g->own_hi : (comm ? Blocks(n, comm->world).hi(comm->rank) : n);
    if (hi > lo)
        GD_KERNEL(k_pr_bin, (unsigned)std::min<int64_t>((hi - lo + kBinChunk - 1) / kBinChunk, 148LL * 8),
                  kBinThreads, 0, s, flags, lo, hi, g->rev.off.get(), bins[0].get(), bins[1].get(), bins[2].get(),
                  ctl.get());
    int64_t done = 0, sweeps = 0;
    int64_t hctl[C_LEN];
    pull_recs.clear();
    while (!done) {
        // multi-GPU: one sweep at a time -- a queued no-op sweep would still
        // move the rank vector through its all-gather
        const int64_t ahead = (comm || g->part) ? 1 : std::max<int64_t>(1, std::min<int64_t>(ahead_hint, 16));
        for (int64_t k = 0; k < ahead; ++k) sweep(sweeps + k);
        read_small(s, hctl, ctl.get(), sizeof hctl);
        done = hctl[C_DONE];
        sweeps = hctl[C_SWEEPS];
    }
    ahead_hint = sweeps;  // sweep counts are stable batch to batch: usually one read-back
    last_sweeps = sweeps;
    iterations += sweeps;
    prof.drop_sweeps_from(sweeps);  // queued no-op sweeps are not launches of the path
    for (auto& pr : pull_recs) {
        if (pr.first < 0) continue;
        int64_t nb = 0, eb = 0;  // bin -1: all three
        for (int k = 0; k < 3; ++k)
            if (pr.second < 0 || pr.second == k) {
                nb += hctl[C_NBIN + k];
                eb += hctl[C_EBIN + k];
            }
        prof.pending[(size_t)pr.first].bytes = 24 * nb + 12 * eb;
    }
    int64_t a = 0;
    for (int k = 0; k < 3; ++k) a += hctl[C_NBIN + k];
    last_affected = flags ? a : n;
}

void PR::batch(DevBatch& b, int64_t batch_index) {
    cudaStream_t s = stream();
    ProfScope ps(&prof);
    prof.reset_last();
    timer.begin(PH_PRE);
    affected.zero(s);
    // OnDelete then OnAdd (pr_dynamic.sp:87-97); both only mark and count, so
    // one launch covers the two record lists
    if (b.kdel + b.kadd)
        GD_KERNEL(k_pr_onupdate, grid_for(b.kdel + b.kadd, 256), 256, 0, s, b.ds.get(), b.dd.get(), b.kdel,
                  b.as.get(), b.ad.get(), b.kadd, affected.get(), outdeg.get());
    timer.begin(PH_STRUCT);
    g->apply_deletes(b.ds.get(), b.dd.get(), b.kdel, nullptr);
    g->apply_adds(b.as.get(), b.ad.get(), b.aw.get(), b.kadd);
    // merge-if-due runs before the recompute: it does not change the live
    // multiset the recompute reads (interp.py:877-880 runs it after).
    if (g->merge_due(batch_index)) {
        timer.begin(PH_MERGE);
        g->merge();
    }
    struct_done();
    timer.begin(PH_PROP);
    if (g->part) flood_weak_components_dist(*g, affected.get(), &prof);
    else flood_weak_components(*g, affected.get(), &prof);
    recompute(affected.get());
    timer.end_all();
}

void PR::gather() {
    if (!g->part || g->n == 0) return;
    cudaStream_t s = stream();
    g->part->allgatherv(rank.get(), g->blocks, 8, s);
    g->part->allgatherv(outdeg.get(), g->blocks, 4, s);
    g->part->allgatherv(affected.get(), g->blocks, 1, s);
}

void PR::read_affected(uint8_t* h_aff) {
    cudaStream_t s = stream();
    int64_t n = g->n;
    if (!n) return;
    GD_CUDA(cudaMemcpyAsync(h_aff, affected.get(), n, cudaMemcpyDeviceToHost, s));
    GD_CUDA(cudaStreamSynchronize(s));
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
