// gd_tc.cu -- dynamic triangle counting (programs/tc_dynamic.sp:7-115,
// tests/golden/tc_dynamic_omp.cc:8-148) on the GPU store.
//
// The reference marks every slot holding a batch edge with the pair's rank
// r = min*V + max and, per batch edge (u,v), counts slot pairs
// e2=(u,w), e3=(v,w), w != v, skipping a pair when e2 or e3 is marked with a
// smaller rank.  A slot (x,w) is marked iff {x,w} is a batch pair, and its mark
// is rank({x,w}) -- a function of the pair -- so the count per record is
//
//     sum over distinct w != v of  m_u(w) * m_v(w) * [not skip(w)],
//     skip(w) = (rank(u,w) in R and rank(u,w) < r) or (rank(v,w) in R and rank(v,w) < r)
//
// with m_x(w) the multiplicity of arc x->w and R the sorted batch ranks.
// The GPU walks the shorter of the two sorted adjacency rows and binary
// searches the longer one (warp per record); membership in R is a binary
// search over the sorted ranks, only for common neighbours.
#include "gd_tc.cuh"

namespace gdb {

namespace {

constexpr int kThreads = 256;

__device__ inline int64_t pair_rank(int64_t a, int64_t b, int64_t n) { return a < b ? a * n + b : b * n + a; }

__device__ inline bool in_sorted(const int64_t* R, int64_t nr, int64_t x) {
    int64_t p = lower_bound_dev<int64_t>(R, 0, nr, x);
    return p < nr && R[p] == x;
}

__global__ void k_ranks(const int32_t* s, const int32_t* d, int64_t k, int64_t n, uint64_t* r) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < k; i += (int64_t)gridDim.x * blockDim.x)
        r[i] = (uint64_t)pair_rank(s[i], d[i], n);
}

// count of x in the sorted clean row [a, b)
__device__ inline int64_t mult_in(const int32_t* col, int64_t a, int64_t b, int32_t x) {
    int64_t lo = lower_bound_dev<int32_t>(col, a, b, x);
    if (lo >= b || col[lo] != x) return 0;
    return upper_bound_dev<int32_t>(col, lo, b, x) - lo;
}

// one warp per batch record
__global__ void __launch_bounds__(kThreads) k_tc_count(const int32_t* s, const int32_t* d, int64_t k, IdxView ix,
                                                       int64_t n, const int64_t* R, int64_t nr,
                                                       unsigned long long* total) {
    const int lane = threadIdx.x & 31;
    int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    int64_t acc = 0;
    for (int64_t i = warp; i < k; i += nwarps) {
        int32_t u = s[i], v = d[i];
        int64_t r = pair_rank(u, v, n);
        int64_t ua = ix.off[u], ub = ix.off[u + 1];
        int64_t va = ix.off[v], vb = ix.off[v + 1];
        // walk the shorter row, search the longer
        bool walk_u = (ub - ua) <= (vb - va);
        int64_t wa = walk_u ? ua : va, wb = walk_u ? ub : vb;
        int64_t sa = walk_u ? va : ua, sb = walk_u ? vb : ub;
        for (int64_t e = wa + lane; e < wb; e += 32) {
            int32_t w = ix.col[e];
            if (w == v) continue;
            int64_t m = mult_in(ix.col, sa, sb, w);
            if (!m) continue;
            int64_t ru = pair_rank(u, w, n), rv = pair_rank(v, w, n);
            bool skip = (ru < r && in_sorted(R, nr, ru)) || (rv < r && in_sorted(R, nr, rv));
            if (!skip) acc += m;
        }
    }
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0 && acc) atomicAdd(total, (unsigned long long)acc);
}

// staticTC (tc_dynamic.sp:7-19): sum over arcs (v,a), a > v, and arcs (a,b),
// b > a, of m_v(b).  One warp per vertex v; lanes take arcs of N(a) beyond a.
__global__ void __launch_bounds__(kThreads) k_tc_static(IdxView ix, int64_t n, unsigned long long* total) {
    const int lane = threadIdx.x & 31;
    int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    int64_t acc = 0;
    for (int64_t v = warp; v < n; v += nwarps) {
        int64_t va = ix.off[v], vb = ix.off[v + 1];
        int64_t first = upper_bound_dev<int32_t>(ix.col, va, vb, (int32_t)v);  // arcs with a > v
        for (int64_t e1 = first; e1 < vb; ++e1) {
            int32_t a = ix.col[e1];
            int64_t aa = ix.off[a], ab = ix.off[a + 1];
            int64_t start = upper_bound_dev<int32_t>(ix.col, aa, ab, a);  // b > a
            for (int64_t e2 = start + lane; e2 < ab; e2 += 32) {
                int32_t b = ix.col[e2];
                acc += mult_in(ix.col, e1, vb, b);  // b > a >= col[e1], so search from e1
            }
        }
    }
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0 && acc) atomicAdd(total, (unsigned long long)acc);
}

}  // namespace

int64_t TC::count_records(const int32_t* s, const int32_t* d, int64_t k) {
    if (k == 0) return 0;
    cudaStream_t st = stream();
    SortedIndex& ix = g->tc_index();
    g->compact_index(ix);
    DBuf<uint64_t> R(k, st);
    GD_KERNEL(k_ranks, grid_for(k, 256), 256, 0, st, s, d, k, g->n, R.get());
    sort_keys_u64(st, R.get(), k);
    DBuf<unsigned long long> tot(1, st);
    tot.zero(st);
    // ranks are over ALL records of the phase; the counted slice is this rank's
    int64_t a = comm ? k * comm->rank / comm->world : 0;
    int64_t b = comm ? k * (comm->rank + 1) / comm->world : k;
    if (b > a)
        GD_KERNEL_T("tc_count", 0, k_tc_count, grid_for((b - a) * 32, kThreads, 148LL * 64), kThreads, 0, st, s + a,
                    d + a, b - a, ix.view(), g->n, reinterpret_cast<const int64_t*>(R.get()), k, tot.get());
    if (comm) comm->allreduce_sum_i64(reinterpret_cast<int64_t*>(tot.get()), 1, st);
    return (int64_t)read_scalar(st, tot.get());
}

TC::TC(Store* st) : AlgoBase(ALGO_TC, st) {
    cudaStream_t s = stream();
    ProfScope ps(&prof);
    timer.begin(PH_STATIC);
    if (g->directed) g->require_fwd();
    else g->require_rev();
    SortedIndex& ix = g->tc_index();
    g->compact_index(ix);
    DBuf<unsigned long long> tot(1, s);
    tot.zero(s);
    if (g->n)
        GD_KERNEL_T("tc_static", 0, k_tc_static, grid_for(g->n * 32, kThreads, 148LL * 64), kThreads, 0, s,
                    ix.view(), g->n, tot.get());
    count = (int64_t)read_scalar(s, tot.get());
    timer.end_all();
    prof.flush();
}

void TC::batch(DevBatch& b, int64_t batch_index) {
    ProfScope ps(&prof);
    prof.reset_last();
    // OnDelete marks + counts on the pre-delete graph (tc_dynamic.sp:28-69)
    timer.begin(PH_PRE);
    count -= count_records(b.ds.get(), b.dd.get(), b.kdel);
    timer.begin(PH_STRUCT);
    g->apply_deletes(b.ds.get(), b.dd.get(), b.kdel, nullptr);
    g->apply_adds(b.as.get(), b.ad.get(), b.aw.get(), b.kadd);
    if (g->merge_due(batch_index)) {  // before the add count; same live multiset
        timer.begin(PH_MERGE);
        g->merge();
    }
    // OnAdd marks + counts on the post-add graph (tc_dynamic.sp:71-112)
    timer.begin(PH_PRE);
    count += count_records(b.as.get(), b.ad.get(), b.kadd);
    timer.end_all();
    prof.flush();
}

}  // namespace gdb
