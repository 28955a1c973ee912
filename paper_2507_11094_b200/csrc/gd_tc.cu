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

// Membership filter of the batch pair ranks: one bit per hashed rank, ~16
// bits per record, so a common neighbour's (u,w) / (v,w) is almost always
// cleared by one load instead of a binary search over R.
__device__ inline uint64_t rank_hash(int64_t r) {
    uint64_t x = (uint64_t)r * 0x9E3779B97F4A7C15ULL;
    return x ^ (x >> 29);
}

__global__ void k_ranks(const int32_t* s, const int32_t* d, int64_t k, int64_t n, uint64_t* r, uint32_t* filt,
                        uint64_t fmask) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < k; i += (int64_t)gridDim.x * blockDim.x) {
        int64_t rk = pair_rank(s[i], d[i], n);
        r[i] = (uint64_t)rk;
        uint64_t h = rank_hash(rk) & fmask;
        atomicOr(&filt[h >> 5], 1u << (h & 31));
    }
}

__device__ inline bool maybe_in(const uint32_t* filt, uint64_t fmask, int64_t r) {
    uint64_t h = rank_hash(r) & fmask;
    return (filt[h >> 5] >> (h & 31)) & 1;
}

// count of x in the sorted clean row [a, b)
__device__ inline int64_t mult_in(const int32_t* col, int64_t a, int64_t b, int32_t x) {
    int64_t lo = lower_bound_dev<int32_t>(col, a, b, x);
    if (lo >= b || col[lo] != x) return 0;
    return upper_bound_dev<int32_t>(col, lo, b, x) - lo;
}

// ---------------------------------------------------------------------------
// Per-record counting, load-balanced.  A record (u,v) walks the row of its
// endpoint S with fewer arcs and looks each neighbour w up in the row of the
// other endpoint L.  The walk is cut into kWalkChunk-arc work items (a hub-
// hub record on R-MAT is 10^5 arcs: one warp would serialise it), and the
// lookup is a bit test when L is a hub of this phase (degree >= kBmDeg):
// the phase builds one n-bit bitmap per hub, up to a memory budget, from
// its sorted row, and clears it afterwards.  A bit hit on a hub whose row
// holds parallel arcs falls back to the binary search for the
// multiplicity.  Counts are integers, so chunk partials add up exactly.
// ---------------------------------------------------------------------------
constexpr int kWalkChunk = 1024;
constexpr int64_t kBmDeg = 1024;
constexpr int64_t kBmBudget = 8LL << 30;  // bytes of hub bitmaps per phase

struct TcRec {
    int32_t* L;
    int32_t* S;
    int64_t* nch;    // work items of the record (then exclusive-scanned in place)
};

__global__ void k_tc_prep(const int32_t* s, const int32_t* d, int64_t k, IdxView ix, TcRec r, uint8_t* hubmark,
                          uint8_t* isshort, unsigned long long* bytes) {
    unsigned long long acc = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < k; i += (int64_t)gridDim.x * blockDim.x) {
        int32_t u = s[i], v = d[i];
        int64_t du = ix.off[u + 1] - ix.off[u], dv = ix.off[v + 1] - ix.off[v];
        // walk the shorter row (ties: u, as the one-warp kernel did)
        bool walk_u = du <= dv;
        int32_t L = walk_u ? v : u, S = walk_u ? u : v;
        int64_t dS = walk_u ? du : dv, dL = walk_u ? dv : du;
        r.L[i] = L;
        r.S[i] = S;
        const bool sh = dS <= 64;  // kShortWalk: a sub-warp group takes it whole (kernel below)
        isshort[i] = sh;
        r.nch[i] = sh ? 0 : (dS + kWalkChunk - 1) / kWalkChunk;
        if (dL >= kBmDeg) hubmark[L] = 1;
        acc += 32 + 4 * (unsigned long long)(du + dv);  // 2*2*off + (deg u + deg v)*idx
    }
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0 && acc) atomicAdd(bytes, acc);
}

__global__ void k_tc_lkeys(const int32_t* L, int64_t m, uint32_t* key, int32_t* perm) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
        key[i] = (uint32_t)L[i];
        perm[i] = (int32_t)i;
    }
}

__global__ void k_tc_perm_nch(const int32_t* perm, const int64_t* nch, int64_t m, int64_t* out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= m; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = i < m ? nch[perm[i]] : 0;
}

__global__ void k_tc_chunk_table(const int64_t* choff, int64_t k, int32_t* rec_of) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < k; i += (int64_t)gridDim.x * blockDim.x)
        for (int64_t c = choff[i]; c < choff[i + 1]; ++c) rec_of[c] = (int32_t)i;
}

__global__ void k_tc_hub_slots(const int32_t* hubs, const int64_t* nhub, int64_t hmax, int32_t* slot) {
    const int64_t m = min(*nhub, hmax);
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < m; j += (int64_t)gridDim.x * blockDim.x)
        slot[hubs[j]] = (int32_t)j;
}

// set (clear = false) or clear the bits of each budgeted hub's row; marks
// hubs whose sorted row holds a repeated neighbour (parallel arcs)
__global__ void k_tc_bitmaps(const int32_t* hubs, const int64_t* nhub, int64_t hmax, IdxView ix, int64_t words,
                             uint32_t* bm, uint8_t* multi, bool clear) {
    const int64_t m = min(*nhub, hmax);
    for (int64_t j = blockIdx.x; j < m; j += gridDim.x) {
        const int32_t h = hubs[j];
        uint32_t* b = bm + j * words;
        const int64_t a = ix.off[h], e = ix.off[h + 1];
        bool dup = false;
        for (int64_t q = a + threadIdx.x; q < e; q += blockDim.x) {
            int32_t w = ix.col[q];
            if (w < 0) continue;
            if (clear) {
                b[w >> 5] = 0;
            } else {
                atomicOr(&b[w >> 5], 1u << (w & 31));
                dup |= q + 1 < e && ix.col[q + 1] == w;
            }
        }
        if (!clear && __syncthreads_or(dup) && threadIdx.x == 0) multi[j] = 1;
        if (clear && threadIdx.x == 0) multi[j] = 0;
    }
}

__global__ void k_tc_reset(const int32_t* hubs, const int64_t* nhub, uint8_t* hubmark, int32_t* slot) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < *nhub; j += (int64_t)gridDim.x * blockDim.x) {
        hubmark[hubs[j]] = 0;
        slot[hubs[j]] = -1;
    }
}

// count of one record's walk slice [wa, wb) of S's row against L, lanes
// strided by W
template <int W>
__device__ __forceinline__ int64_t tc_walk(const IdxView& ix, int32_t u, int32_t v, int32_t L, int64_t wa, int64_t wb,
                                           int lane, int64_t n, const int64_t* R, int64_t nr, const int32_t* slot,
                                           const uint32_t* bm, int64_t words, const uint8_t* multi,
                                           const uint32_t* filt, uint64_t fmask) {
    const int64_t rk = pair_rank(u, v, n);
    const int64_t la = ix.off[L], lb = ix.off[L + 1];
    const int32_t hs = slot[L];
    const uint32_t* b = hs >= 0 ? bm + (int64_t)hs * words : nullptr;
    const bool mult = hs >= 0 && multi[hs];
    int64_t acc = 0;
    for (int64_t e = wa + lane; e < wb; e += W) {
        int32_t w = ix.col[e];
        if (w < 0 || w == v) continue;
        int64_t m;
        if (b) m = (b[w >> 5] >> (w & 31)) & 1 ? (mult ? mult_in(ix.col, la, lb, w) : 1) : 0;
        else m = mult_in(ix.col, la, lb, w);
        if (!m) continue;
        int64_t ru = pair_rank(u, w, n), rv = pair_rank(v, w, n);
        bool skip = (ru < rk && maybe_in(filt, fmask, ru) && in_sorted(R, nr, ru)) ||
                    (rv < rk && maybe_in(filt, fmask, rv) && in_sorted(R, nr, rv));
        if (!skip) acc += m;
    }
    return acc;
}

// long records: one warp per work item, kWalkChunk arcs of S's row
__global__ void __launch_bounds__(kThreads) k_tc_count(const int32_t* s, const int32_t* d, TcRec r,
                                                       const int32_t* perm, const int32_t* rec_of,
                                                       const int64_t* nwork, IdxView ix,
                                                       int64_t n, const int64_t* R, int64_t nr, const int32_t* slot,
                                                       const uint32_t* bm, int64_t words, const uint8_t* multi,
                                                       const uint32_t* filt, uint64_t fmask,
                                                       unsigned long long* total) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int64_t nw = *nwork;
    int64_t acc = 0;
    for (int64_t c = warp; c < nw; c += nwarps) {
        const int32_t ip = rec_of[c];  // position in L order
        const int32_t i = perm ? perm[ip] : ip;
        const int32_t S = r.S[i];
        const int64_t j = c - r.nch[ip];  // nch holds the exclusive scan in L order here
        const int64_t wa = ix.off[S] + j * kWalkChunk, wb = min(wa + kWalkChunk, ix.off[S + 1]);
        acc += tc_walk<32>(ix, s[i], d[i], r.L[i], wa, wb, lane, n, R, nr, slot, bm, words, multi, filt, fmask);
    }
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0 && acc) atomicAdd(total, (unsigned long long)acc);
}

// Short records, first pass: every record of the phase.  A group of kMG
// lanes takes one record (32/kMG per warp in flight) and, when both rows are
// short -- S <= kShortWalk arcs and L <= kStageL, i.e. every record of a
// uniform graph -- counts it here as a sorted MERGE (SURVEY.md §8(d):
// (deg u + deg v) * idx, streamed).  Both rows are staged in shared memory
// with 16-byte loads aligned to the 16-byte grid, so each sector of a row is
// requested once; then every lane takes a contiguous slice of S's row, finds
// its start in L by one binary search and walks both rows forward.
// Multiplicities are the runs of equal entries in L, so parallel arcs count
// as the reference's slot pairs do.  Records with a long row are appended to
// a deferred list for the lookup-based kernels below.
constexpr int kShortWalk = 64;
constexpr int kStageL = 128;
#ifndef GD_TC_MG
#define GD_TC_MG 8
#endif
constexpr int kMG = GD_TC_MG;
#ifndef GD_TCM_MINB
#define GD_TCM_MINB 6
#endif

__device__ __forceinline__ int64_t skip_mult(int32_t u, int32_t v, int32_t w, int64_t rk, int64_t n, int64_t m,
                                             const int64_t* R, int64_t nr, const uint32_t* filt, uint64_t fmask) {
    int64_t ru = pair_rank(u, w, n), rv = pair_rank(v, w, n);
    bool skip = (ru < rk && maybe_in(filt, fmask, ru) && in_sorted(R, nr, ru)) ||
                (rv < rk && maybe_in(filt, fmask, rv) && in_sorted(R, nr, rv));
    return skip ? 0 : m;
}

// coalesced 16-byte staging of col[a, b) into buf; returns a's offset in buf
__device__ __forceinline__ int stage_row(const int32_t* col, int64_t a, int64_t b, int32_t* buf, int gl) {
    const int64_t a4 = a >> 2;
    const int nq = (int)(((b + 3) >> 2) - a4);
    const int4* src = reinterpret_cast<const int4*>(col) + a4;
    for (int q = gl; q < nq; q += kMG) reinterpret_cast<int4*>(buf)[q] = src[q];
    return (int)(a & 3);
}

__global__ void __launch_bounds__(kThreads, GD_TCM_MINB) k_tc_merge(const int32_t* s, const int32_t* d, int64_t k,
                                                                    IdxView ix, int64_t n, const int64_t* R, int64_t nr,
                                                                    const uint32_t* filt, uint64_t fmask,
                                                                    int32_t* defer, unsigned long long* ndefer,
                                                                    unsigned long long* total) {
    extern __shared__ __align__(16) int32_t tc_smem[];  // per group: S row, then L row
    constexpr int kSW = kShortWalk + 8, kLW = kStageL + 8;
    const int gl = threadIdx.x & (kMG - 1), gw = (threadIdx.x & 31) / kMG;
    const unsigned gmask = (kMG == 32 ? 0xffffffffu : ((1u << kMG) - 1)) << ((threadIdx.x & 31) & ~(kMG - 1));
    constexpr int kPer = 32 / kMG;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    int32_t* sS = tc_smem + (threadIdx.x / kMG) * (kSW + kLW);
    int32_t* sL = sS + kSW;
    int64_t acc = 0;
    unsigned long long bytes = 0;
    for (int64_t t0 = warp * kPer; t0 < k; t0 += nwarps * kPer) {
        const int64_t i = t0 + gw;
        if (i >= k) continue;
        const int32_t u = s[i], v = d[i];
        const int64_t ua = ix.off[u], ub = ix.off[u + 1], va = ix.off[v], vb = ix.off[v + 1];
        const bool walk_u = ub - ua <= vb - va;  // walk the shorter row (ties: u)
        const int64_t sa = walk_u ? ua : va, sb = walk_u ? ub : vb;
        const int64_t la = walk_u ? va : ua, lb = walk_u ? vb : ub;
        const int ns = (int)(sb - sa), nl = (int)(lb - la);
        if (sb - sa > kShortWalk || lb - la > kStageL) {
            if (gl == 0) defer[atomicAdd(ndefer, 1ULL)] = (int32_t)i;
            continue;
        }
        if (gl == 0) bytes += 32 + 4 * (unsigned long long)(ns + nl);
        const int s0 = stage_row(ix.col, sa, sb, sS, gl);
        const int l0 = stage_row(ix.col, la, lb, sL, gl);
        __syncwarp(gmask);
        const int c = (ns + kMG - 1) / kMG;
        int e = s0 + gl * c;
        const int e1 = min(e + c, s0 + ns), l1 = l0 + nl;
        if (e < e1) {
            const int64_t rk = pair_rank(u, v, n);
            const int32_t w0 = sS[e];
            int lo = l0, hi = l1;  // first entry of L >= w0
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (sL[mid] < w0) lo = mid + 1;
                else hi = mid;
            }
            int p = lo;
            for (; e < e1 && p < l1; ++e) {
                const int32_t w = sS[e];
                while (p < l1 && sL[p] < w) ++p;
                if (w < 0 || w == v) continue;
                int r = p;
                while (r < l1 && sL[r] == w) ++r;
                if (r > p) acc += skip_mult(u, v, w, rk, n, r - p, R, nr, filt, fmask);
            }
        }
        __syncwarp(gmask);  // the group's buffers are reused by its next record
    }
    for (int o = 16; o; o >>= 1) {
        acc += __shfl_xor_sync(0xffffffffu, acc, o);
        bytes += __shfl_xor_sync(0xffffffffu, bytes, o);
    }
    if ((threadIdx.x & 31) == 0) {
        if (acc) atomicAdd(total, (unsigned long long)acc);
        if (bytes) atomicAdd(total + 1, bytes);
    }
}

// Deferred records whose walk is still short (S <= kShortWalk arcs, L a long
// row): 8 lanes each, 4 records per warp in flight, lookups per neighbour.
constexpr int kShortG = 8;
#ifndef GD_TCS_MINB
#define GD_TCS_MINB 8
#endif
__global__ void __launch_bounds__(kThreads, GD_TCS_MINB) k_tc_count_short(const int32_t* s, const int32_t* d, TcRec r,
                                                             const int32_t* list, const int64_t* nlist, IdxView ix,
                                                             int64_t n, const int64_t* R, int64_t nr,
                                                             const int32_t* slot, const uint32_t* bm, int64_t words,
                                                             const uint8_t* multi, const uint32_t* filt,
                                                             uint64_t fmask, unsigned long long* total) {
    const int gl = threadIdx.x & (kShortG - 1), gw = (threadIdx.x & 31) / kShortG;
    constexpr int kPer = 32 / kShortG;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int64_t m = *nlist;
    int64_t acc = 0;
    for (int64_t t0 = warp * kPer; t0 < m; t0 += nwarps * kPer) {
        const int64_t t = t0 + gw;
        if (t < m) {
            const int32_t i = list[t];
            const int32_t S = r.S[i];
            acc += tc_walk<kShortG>(ix, s[i], d[i], r.L[i], ix.off[S], ix.off[S + 1], gl, n, R, nr, slot, bm, words,
                                    multi, filt, fmask);
        }
    }
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0 && acc) atomicAdd(total, (unsigned long long)acc);
}

__global__ void k_tc_gather_rec(const int32_t* s, const int32_t* d, const int32_t* idx, int64_t m, int32_t* os,
                                int32_t* od) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < m; j += (int64_t)gridDim.x * blockDim.x) {
        os[j] = s[idx[j]];
        od[j] = d[idx[j]];
    }
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
    const int64_t n = g->n;
    DBuf<uint64_t> R(k, st);
    int fbits = 10;  // filter of 2^fbits bits, >= 16 per record
    while (fbits < 34 && (int64_t(1) << fbits) < 16 * k) ++fbits;
    DBuf<uint32_t> filt((size_t(1) << fbits) / 32, st);
    filt.zero(st);
    const uint64_t fmask = (uint64_t(1) << fbits) - 1;
    GD_KERNEL(k_ranks, grid_for(k, 256), 256, 0, st, s, d, k, n, R.get(), filt.get(), fmask);
    // ranks are < n^2: sort only the bits they use (48 instead of 64 at 2^24 vertices)
    sort_keys_u64(st, R.get(), k, bits_for((uint64_t)n * (uint64_t)n - 1));
    DBuf<unsigned long long> ctr(3, st);  // [0] count delta, [1] algorithmic bytes, [2] deferred records
    ctr.zero(st);
    // ranks are over ALL records of the phase; the counted slice is this rank's
    const int64_t a = comm ? k * comm->rank / comm->world : 0;
    const int64_t b = comm ? k * (comm->rank + 1) / comm->world : k;
    const int64_t m = b - a;
    const int64_t* Rp = reinterpret_cast<const int64_t*>(R.get());
    if (m > 0) {
        DBuf<int32_t> defer(m, st);
        int pi = prof_begin("tc_count", 0, st);
        static const int smem = [] {
            const int b = (kThreads / kMG) * (kShortWalk + 8 + kStageL + 8) * 4;
            GD_CUDA(cudaFuncSetAttribute(k_tc_merge, cudaFuncAttributeMaxDynamicSharedMemorySize, b));
            return b;
        }();
        k_tc_merge<<<148 * 16, kThreads, smem, st>>>(s + a, d + a, m, ix.view(), n, Rp, k, filt.get(), fmask,
                                                   defer.get(), ctr.get() + 2, ctr.get());
        count_launch();
        GD_LAUNCH_CHECK();
        prof_end(pi, st);
        if (pi >= 0) count_rec.push_back(pi);
        const int64_t md = (int64_t)read_scalar(st, ctr.get() + 2);
        if (md > 0) {
            DBuf<int32_t> ds(md, st), dd(md, st);
            GD_KERNEL(k_tc_gather_rec, grid_for(md, 256), 256, 0, st, s + a, d + a, defer.get(), md, ds.get(),
                      dd.get());
            count_deferred(ds.get(), dd.get(), md, Rp, k, filt.get(), fmask, ctr.get());
        }
    }
    if (comm) comm->allreduce_sum_i64(reinterpret_cast<int64_t*>(ctr.get()), 1, st);
    unsigned long long h[2];
    read_small(st, h, ctr.get(), sizeof h);
    for (size_t j = 0; j < count_rec.size(); ++j) prof.pending[(size_t)count_rec[j]].bytes = j ? 0 : (int64_t)h[1];
    count_rec.clear();
    return (int64_t)h[0];
}

// records with a long row: one walk per record, per-neighbour lookups in L
// (hub bitmap or binary search), long walks cut into work items
void TC::count_deferred(const int32_t* s, const int32_t* d, int64_t m, const int64_t* R, int64_t k,
                        const uint32_t* filt, uint64_t fmask, unsigned long long* ctr) {
    cudaStream_t st = stream();
    SortedIndex& ix = g->tc_index();
    const int64_t n = g->n;
    if (hubmark.n < (size_t)n) {
        hubmark.alloc(n, st);
        hubmark.zero(st);
        hub_slot.alloc(n, st);
        fill_i32(st, hub_slot.get(), n, -1);
    }
    DBuf<int32_t> L(m, st), S(m, st);
    DBuf<int64_t> nch(m + 1, st), choff(m + 1, st);
    fill_d(st, nch.get() + m, 0, sizeof(int64_t));
    TcRec rr{L.get(), S.get(), nch.get()};
    DBuf<uint8_t> isshort(m, st);
    GD_KERNEL(k_tc_prep, grid_for(m, 256), 256, 0, st, s, d, m, ix.view(), rr, hubmark.get(), isshort.get(),
              ctr + 1);
    DBuf<int32_t> shortl(m, st);
    DBuf<int64_t> nshort(1, st);
    select_flagged_index_async(st, isshort.get(), m, shortl.get(), nshort.get());
    // hubs of this phase (L endpoints with >= kBmDeg arcs) and the work
    // item total, read back together
    exclusive_scan_i64(st, nch.get(), choff.get(), m + 1);
    DBuf<int32_t> hubs(n, st);
    DBuf<int64_t> cnt2(2, st);
    GD_CUDA(cudaMemcpyAsync(cnt2.get(), choff.get() + m, sizeof(int64_t), cudaMemcpyDeviceToDevice, st));
    select_flagged_index_async(st, hubmark.get(), n, hubs.get(), cnt2.get() + 1);
    int64_t hc[2];
    read_small(st, hc, cnt2.get(), sizeof hc);
    const int64_t nwork = hc[0], nhubs = hc[1];
    // with hub rows in play, work items go in L order: warps running side
    // by side (grid-stride neighbours) meet the same long rows and share
    // their L2 lines; without hubs the record order stands
    DBuf<int32_t> perm;
    if (nhubs > 0) {
        DBuf<uint32_t> lkey(m, st);
        perm.alloc(m, st);
        GD_KERNEL(k_tc_lkeys, grid_for(m, 256), 256, 0, st, L.get(), m, lkey.get(), perm.get());
        sort_pairs_u32(st, lkey.get(), perm.get(), m, bits_for((uint64_t)std::max<int64_t>(n - 1, 1)));
        DBuf<int64_t> nchp(m + 1, st);
        GD_KERNEL(k_tc_perm_nch, grid_for(m + 1, 256), 256, 0, st, perm.get(), nch.get(), m, nchp.get());
        exclusive_scan_i64(st, nchp.get(), choff.get(), m + 1);
    }
    rr.nch = choff.get();
    // work items: exact count (records may share a long S row)
    DBuf<int32_t> rec_of(std::max<int64_t>(nwork, 1), st);
    GD_KERNEL(k_tc_chunk_table, grid_for(m, 256), 256, 0, st, choff.get(), m, rec_of.get());
    // bitmaps for as many hubs as the budget allows (grow-only; every
    // phase leaves them clean)
    const int64_t words = (n + 31) / 32;
    const int64_t hmax = std::min<int64_t>(nhubs, kBmBudget / (words * 4));
    if (hmax > 0 && bm.n < (size_t)(hmax * words)) {
        bm.alloc((size_t)(hmax * words), st);
        fill_d(st, bm.get(), 0, bm.n * 4);
        bm_multi.alloc(hmax, st);
        bm_multi.zero(st);
    }
    const int64_t* nhub = cnt2.get() + 1;
    if (hmax > 0) {
        GD_KERNEL(k_tc_hub_slots, grid_for(hmax, 256), 256, 0, st, hubs.get(), nhub, hmax, hub_slot.get());
        GD_KERNEL_T("tc_bitmap", 0, k_tc_bitmaps, 148 * 4, 256, 0, st, hubs.get(), nhub, hmax, ix.view(), words,
                    bm.get(), bm_multi.get(), false);
    }
    int pi = prof_begin("tc_count", 0, st);
    k_tc_count<<<(unsigned)std::max<int64_t>(1, std::min<int64_t>((nwork + 7) / 8, 148 * 16)), kThreads, 0, st>>>(
        s, d, rr, nhubs > 0 ? perm.get() : nullptr, rec_of.get(), choff.get() + m, ix.view(), n, R, k,
        hub_slot.get(), bm.get(), words, bm_multi.get(), filt, fmask, ctr);
    count_launch();
    GD_LAUNCH_CHECK();
    k_tc_count_short<<<148 * 16, kThreads, 0, st>>>(s, d, rr, shortl.get(), nshort.get(), ix.view(), n, R, k,
                                                    hub_slot.get(), bm.get(), words, bm_multi.get(), filt, fmask,
                                                    ctr);
    count_launch();
    GD_LAUNCH_CHECK();
    prof_end(pi, st);
    if (hmax > 0)
        GD_KERNEL_T("tc_bitmap", 0, k_tc_bitmaps, 148 * 4, 256, 0, st, hubs.get(), nhub, hmax, ix.view(), words,
                    bm.get(), bm_multi.get(), true);
    if (nhubs > 0)
        GD_KERNEL(k_tc_reset, grid_for(nhubs, 256), 256, 0, st, hubs.get(), nhub, hubmark.get(), hub_slot.get());
    if (pi >= 0) count_rec.push_back(pi);
}

TC::TC(Store* st) : AlgoBase(ALGO_TC, st) {
    if (st->part)
        throw GdError(GD_ERR_CONFIG, "triangle counting runs on replicated stores (each rank holds the whole "
                                     "undirected graph and counts a slice of the records, gd_tc_set_comm)");
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
    struct_done();
    // OnAdd marks + counts on the post-add graph (tc_dynamic.sp:71-112)
    timer.begin(PH_PRE);
    count += count_records(b.as.get(), b.ad.get(), b.kadd);
    timer.end_all();
}

}  // namespace gdb
