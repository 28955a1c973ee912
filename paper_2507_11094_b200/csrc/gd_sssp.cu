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
__device__ inline bool claim(int32_t* stamp, int32_t v, int32_t round) { return atomicMax(&stamp[v], round) < round; }

// Warp-buffered appends for the fixpoint rounds.  Every lowered target used
// to take a slot of the next queue (or the far pile) with an atomicAdd on ONE
// global counter; coalesced lanes share one, but a grid round still sent
// ~10^5 same-address atomics to one L2 slice, which serialise there (C4: 27
// M visits per batch in ~200 rounds of ~200 us).  Each warp now appends to
// its own shared-memory buffer (a shared-memory atomic) and moves it to the
// global queue with ONE global atomicAdd per flush: when it is nearly full
// (checked between work items) and at the end of the round.  An append that
// finds the buffer full goes to the global queue directly.  Queue order is
// arbitrary in every fixpoint, so results do not change.
constexpr int kQBuf = 512;
constexpr int kQFlushAt = kQBuf - 128;
__shared__ int32_t s_wq[kThreads / 32][2][kQBuf];
__shared__ int s_wqn[kThreads / 32][2];

__device__ __forceinline__ void wq_init() {
    if ((threadIdx.x & 31) < 2) s_wqn[threadIdx.x >> 5][threadIdx.x & 31] = 0;
    __syncwarp();
}

// which = 0: the next queue (q, cnt), 1: the far pile
__device__ __forceinline__ void enqueue_w(int which, int32_t* q, unsigned long long* cnt, int32_t v) {
    cg::coalesced_group g = cg::coalesced_threads();
    const int w = threadIdx.x >> 5;
    int pos = 0;
    if (g.thread_rank() == 0) pos = atomicAdd(&s_wqn[w][which], (int)g.size());
    pos = g.shfl(pos, 0) + (int)g.thread_rank();
    if (pos < kQBuf) {
        s_wq[w][which][pos] = v;
    } else {
        cg::coalesced_group o = cg::coalesced_threads();
        unsigned long long base = 0;
        if (o.thread_rank() == 0) base = atomicAdd(cnt, (unsigned long long)o.size());
        base = o.shfl(base, 0);
        q[base + o.thread_rank()] = v;
    }
}

// warp-convergent: move this warp's buffers to the global queue / pile
__device__ __forceinline__ void wq_flush(int32_t* q0, unsigned long long* c0, int32_t* q1, unsigned long long* c1);
// warp-convergent: flush when either buffer is nearly full
__device__ __forceinline__ void wq_maybe_flush(int32_t* q0, unsigned long long* c0, int32_t* q1,
                                               unsigned long long* c1) {
    __syncwarp();
    const int w = threadIdx.x >> 5;
    if (s_wqn[w][0] >= kQFlushAt || s_wqn[w][1] >= kQFlushAt) wq_flush(q0, c0, q1, c1);
}
__device__ __forceinline__ void wq_flush(int32_t* q0, unsigned long long* c0, int32_t* q1, unsigned long long* c1) {
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __syncwarp();
#pragma unroll
    for (int which = 0; which < 2; ++which) {
        const int n = min(s_wqn[w][which], kQBuf);
        if (n == 0) continue;
        int32_t* q = which ? q1 : q0;
        unsigned long long base = 0;
        if (lane == 0) base = atomicAdd(which ? c1 : c0, (unsigned long long)n);
        base = __shfl_sync(0xffffffffu, base, 0);
        for (int i = lane; i < n; i += 32) q[base + i] = s_wq[w][which][i];
        __syncwarp();
        if (lane == 0) s_wqn[w][which] = 0;
        __syncwarp();
    }
}

#define GROUP_LOOP_BEGIN(M)                                                      \
    const int lane = threadIdx.x & (kG - 1);                                     \
    const int gw = (threadIdx.x & 31) / kG;                                      \
    int64_t _warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;       \
    int64_t _nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;                    \
    for (int64_t _t0 = _warp * kPerWarp; _t0 < (M); _t0 += _nwarps * kPerWarp) { \
        int64_t _t = _t0 + gw;                                                   \
        bool valid = _t < (M);
#define GROUP_LOOP_END }
// the same with a group width G (template parameter of the fixpoint)
#define GROUP_LOOP_BEGIN_G(M, G)                                                          \
    const int lane = threadIdx.x & ((G) - 1);                                             \
    const int gw = (threadIdx.x & 31) / (G);                                              \
    int64_t _warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;                \
    int64_t _nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;                             \
    for (int64_t _t0 = _warp * (32 / (G)); _t0 < (M); _t0 += _nwarps * (32 / (G))) {     \
        int64_t _t = _t0 + gw;                                                            \
        bool valid = _t < (M);

__global__ void k_init(int64_t* dist, int32_t* parent, int32_t* stamp, int32_t* hstamp, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        dist[i] = kInf;
        parent[i] = -1;
        stamp[i] = 0;
        hstamp[i] = 0;
    }
}

__global__ void k_set_i64(int64_t* a, int64_t i, int64_t v) { a[i] = v; }

// ---------------------------------------------------------------------------
// Frontier fixpoints.  One whole fixpoint runs in one cooperative launch: a
// grid barrier per round instead of a kernel boundary + host read-back of the
// queue size.  High-diameter graphs (configs[3], grid) take thousands of
// rounds per batch, so the per-round cost is the batch latency.
//
// Round bodies (sssp_dynamic.sp):
//   RELAX  push Min(dist[t], dist[v] + w) over out-arcs       (:15-21,110-117)
//   WALK   invalidate tree children parent[t] == v            (:45-63)
//   PULL   stale v pulls Min over live in-arcs; if it dropped,
//          re-queue its stale out-neighbours                  (:68-86)
// A group of kG lanes takes one queued vertex.  A vertex whose scan exceeds
// kHeavy arcs (R-MAT hubs: 10^4 arcs would serialise a group for ~1 ms) is
// instead cut into kPiece-arc pieces appended to a piece list, and the next
// round spreads the pieces over all warps.  Deferring a vertex's scan by one
// round leaves every fixpoint unchanged: relaxation is monotone (the piece
// re-reads dist[v]), the walk's descendant set and the pull's Bellman-Ford
// limit do not depend on the schedule.
//
// Queues and piece lists are double-buffered; their counters are triple-
// buffered so one barrier per round suffices: round `it` reads slot it%3,
// appends to slot (it+1)%3 and clears slot (it+2)%3, which every thread last
// read before the previous barrier.  Slot s = cnt[3s .. 3s+2] = {queue, out
// pieces, in pieces}.  ctr[0] = last round id used for stamps, ctr[1] +=
// rounds run, ctr[2] = 1 when the round cap (interp.py:141) is hit.
// ---------------------------------------------------------------------------
enum { FP_RELAX = 0, FP_WALK = 1, FP_PULL = 2 };

constexpr int kHeavy = 256;  // arcs a group scans inline
constexpr int kPiece = 128;  // arcs per piece (one warp, 4 per lane)
constexpr int64_t kNearFarMinRounds = 256;  // static-pass rounds below which near-far is off
constexpr int kChainDefault = 16;           // RELAX: near targets a group may follow per round

struct FpArgs {
    OutView ov;
    IdxView ix;
    int64_t* dist;
    int32_t* parent;
    uint8_t* flags;  // relax: touched (nullable); walk: stale (written); pull: stale (read)
    // relax only: when set, only targets t with only[t] != 0 may be lowered
    // (the decremental push; the reference's pull changes stale nodes only)
    const uint8_t* only;
    int32_t* stamp;   // queue de-duplication per round
    int32_t* hstamp;  // out-piece de-duplication per round
    const int32_t* seeds;  // round 0 input, never written
    int32_t* q[2];
    int64_t* ho[2];  // out-scan pieces
    int64_t* hi[2];  // in-pull pieces (PULL)
    unsigned long long* cnt;  // [9]
    long long* ctr;           // [6]
    // algorithmic bytes of this launch (profiling only, else null): every
    // thread sums its own loads and adds them once at exit
    long long* acc;
    int64_t cap;
    // RELAX queue rounds: a group may follow up to `chain` near targets it
    // lowered itself within the round (see fp_round)
    int chain;
    // near-far (RELAX, delta > 0): relaxations landing at >= theta wait in a
    // far pile (3 rotating buffers, counters fcnt/fmin) until the near queue
    // drains; then a split round raises theta by delta and moves the pile's
    // entries below it to the queue.  Same fixpoint, far fewer re-relaxations
    // on high-diameter weighted graphs.
    int64_t delta;
    int32_t* far[3];
    unsigned long long* fcnt;  // [3]
    long long* fmin;           // [3] lower bound of the pile's distances
    int32_t* infar;            // 1 while a vertex sits in the pile
    // vertex-partitioned store (outbox != nullptr): only owned vertices
    // [lo, hi) are queued; a relaxation or invalidation of another rank's
    // vertex updates this rank's copy and lists the vertex once per launch
    // (gstamp) in the outbox for its owner (SSSP::fixpoint_dist)
    int64_t own_lo, own_hi;
    int32_t* outbox;
    unsigned long long* noutbox;
    int32_t* gstamp;
    int32_t launch;
};

__device__ __forceinline__ bool ghost(const FpArgs& a, int32_t t) { return a.outbox && (t < a.own_lo || t >= a.own_hi); }

__device__ __forceinline__ void to_outbox(const FpArgs& a, int32_t t) {
    if (atomicMax(&a.gstamp[t], a.launch) < a.launch) a.outbox[atomicAdd(a.noutbox, 1ULL)] = t;
}

struct Round {
    int32_t id;
    int64_t theta;
    int32_t* fout;
    unsigned long long* ffcnt;
    long long* ffmin;
    int32_t* qout;
    unsigned long long* qcnt;
    int64_t* hoout;
    unsigned long long* hocnt;
    int64_t* hiout;
    unsigned long long* hicnt;
};

__device__ __forceinline__ int64_t piece_key(int32_t v, int sg, int64_t k) {
    return ((int64_t)v << 32) | ((int64_t)sg << 27) | k;
}
__device__ __forceinline__ void piece_decode(int64_t key, int32_t& v, int& sg, int64_t& k) {
    v = (int32_t)(key >> 32);
    sg = (int)((key >> 27) & 31);
    k = key & ((1LL << 27) - 1);
}

template <int W>
__device__ __forceinline__ unsigned group_mask() {
    return W == 32 ? 0xffffffffu : (((1u << W) - 1) << ((threadIdx.x & 31) & ~(W - 1)));
}

// per-arc action of an out-scan; `pre` is the target's word loaded ahead
template <int MODE>
__device__ __forceinline__ int64_t out_pre(const FpArgs& a, int32_t t) {
    if (t < 0) return 0;
    if (MODE == FP_RELAX) return a.only && !a.only[t] ? LLONG_MIN : a.dist[t];  // LLONG_MIN: no c < pre
    if (MODE == FP_WALK) return a.parent[t];
    return a.flags[t];
}

template <int MODE>
__device__ __forceinline__ void out_act(const FpArgs& a, const Round& r, int32_t v, int64_t dv, int32_t t, int32_t w,
                                        int64_t pre, int32_t* cand = nullptr) {
    if (t < 0) return;
    if (MODE == FP_RELAX) {
        int64_t c = sat_add(dv, (int64_t)w);
        if (c < pre) {
            long long old = atomicMin(reinterpret_cast<long long*>(&a.dist[t]), (long long)c);
            if (c < old && ghost(a, t)) {  // the owner applies it after the launch
                to_outbox(a, t);
            } else if (c < old) {
                if (a.flags) a.flags[t] = 1;
                if (c < r.theta) {
                    // the lane's first lowered near target may be followed by
                    // its own group this round instead of queued (fp_round)
                    if (cand && *cand < 0) *cand = t;
                    else if (claim(a.stamp, t, r.id)) enqueue_w(0, r.qout, r.qcnt, t);
                } else {
                    // one hot word: read first, the pile's floor rarely drops
                    // (L1 bypassed: the slot is reset to INF between uses)
                    if (c < __ldcg(r.ffmin)) atomicMin(r.ffmin, (long long)c);
                    if (atomicExch(&a.infar[t], 1) == 0) enqueue_w(1, r.fout, r.ffcnt, t);
                }
            }
        }
    } else if (MODE == FP_WALK) {
        if (pre == v) {
            a.dist[t] = kInf;
            a.parent[t] = -1;
            a.flags[t] = 1;
            if (ghost(a, t)) to_outbox(a, t);
            else if (cand && *cand < 0) *cand = t;  // a child the group walks on this round
            else if (claim(a.stamp, t, r.id)) enqueue_w(0, r.qout, r.qcnt, t);
        }
    } else {
        if (pre && claim(a.stamp, t, r.id)) enqueue_w(0, r.qout, r.qcnt, t);
    }
}

// arcs [e0, e1) of segment sg, lanes strided by W, 4 arcs in flight per lane
template <int MODE, int W>
__device__ __forceinline__ void out_scan(const FpArgs& a, const Round& r, int32_t v, int64_t dv, int sg, int64_t e0,
                                         int64_t e1, int lane, int64_t& nb, int32_t* cand = nullptr) {
    const int32_t* col = a.ov.col[sg];
    const int32_t* wt = MODE == FP_RELAX ? a.ov.w[sg] : nullptr;
    // per slot: col, then weight + dist (relax), parent (walk) or flag (pull)
    // (tombstoned slots counted in full: an upper bound of <= 2x on them)
    const int64_t ba = 4 + (MODE == FP_RELAX ? (wt ? 12 : 8) : MODE == FP_WALK ? 4 : 1);
    int64_t e = e0 + lane;
    if (e < e1) nb += ba * ((e1 - e + W - 1) / W);
    for (; e + 3 * W < e1; e += 4 * W) {
        int32_t t[4], w[4];
        int64_t pre[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) t[j] = col[e + j * W];
#pragma unroll
        for (int j = 0; j < 4; ++j) w[j] = wt ? wt[e + j * W] : 1;
#pragma unroll
        for (int j = 0; j < 4; ++j) pre[j] = out_pre<MODE>(a, t[j]);
#pragma unroll
        for (int j = 0; j < 4; ++j) out_act<MODE>(a, r, v, dv, t[j], w[j], pre[j], cand);
    }
    for (; e < e1; e += W) {
        int32_t t = col[e];
        int32_t w = wt ? wt[e] : 1;
        out_act<MODE>(a, r, v, dv, t, w, out_pre<MODE>(a, t), cand);
    }
}

// visit v's out-arcs with a converged group of W lanes: inline when short,
// else (once per round per vertex) as pieces for the next round
template <int MODE, int W>
__device__ __forceinline__ void out_visit(const FpArgs& a, const Round& r, int32_t v, int64_t dv, int lane,
                                          int64_t& nb, int32_t* cand = nullptr) {
    const unsigned gm = group_mask<W>();
    const int leader = (threadIdx.x & 31) & ~(W - 1);
    int64_t deg = 0;
    for (int sg = 0; sg < a.ov.nseg; ++sg) deg += a.ov.off[sg][v + 1] - a.ov.off[sg][v];
    if (lane == 0) nb += 16 * a.ov.nseg;
    if (deg <= kHeavy) {
        for (int sg = 0; sg < a.ov.nseg; ++sg)
            out_scan<MODE, W>(a, r, v, dv, sg, a.ov.off[sg][v], a.ov.off[sg][v + 1], lane, nb, cand);
        return;
    }
    int64_t np = 0;
    for (int sg = 0; sg < a.ov.nseg; ++sg) np += (a.ov.off[sg][v + 1] - a.ov.off[sg][v] + kPiece - 1) / kPiece;
    unsigned long long base = 0;
    if (lane == 0 && claim(a.hstamp, v, r.id)) base = atomicAdd(r.hocnt, (unsigned long long)np) + 1;
    base = __shfl_sync(gm, base, leader);
    if (!base) return;
    base -= 1;
    for (int sg = 0; sg < a.ov.nseg; ++sg) {
        int64_t ns = (a.ov.off[sg][v + 1] - a.ov.off[sg][v] + kPiece - 1) / kPiece;
        for (int64_t k = lane; k < ns; k += W) r.hoout[base + k] = piece_key(v, sg, k);
        if (lane == 0) nb += 8 * ns;
        base += ns;
    }
}

// min over in-arcs [e0, e1) of sat(dist[u] + w), lanes strided by W
template <int W>
__device__ __forceinline__ int64_t in_min(const FpArgs& a, int64_t e0, int64_t e1, int lane, int64_t& nb) {
    int64_t best = kInf;
    int64_t e = e0 + lane;
    if (e < e1) nb += (a.ix.w ? 16 : 12) * ((e1 - e + W - 1) / W);  // per slot: col, weight, dist[u]
    for (; e + 3 * W < e1; e += 4 * W) {
        int32_t u[4];
        int64_t c[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) u[j] = a.ix.col[e + j * W];
#pragma unroll
        for (int j = 0; j < 4; ++j)
            c[j] = u[j] < 0 ? kInf : sat_add(a.dist[u[j]], a.ix.w ? (int64_t)a.ix.w[e + j * W] : 1);
#pragma unroll
        for (int j = 0; j < 4; ++j) best = c[j] < best ? c[j] : best;
    }
    for (; e < e1; e += W) {
        int32_t u = a.ix.col[e];
        if (u < 0) continue;
        int64_t c = sat_add(a.dist[u], a.ix.w ? (int64_t)a.ix.w[e] : 1);
        best = c < best ? c : best;
    }
    const unsigned gm = group_mask<W>();
#pragma unroll
    for (int o = W / 2; o; o >>= 1) {
        long long x = __shfl_xor_sync(gm, (long long)best, o, W);
        best = x < best ? x : best;
    }
    return best;
}

// lower dist[v] to best; true (on every lane of the group) when it dropped
template <int W>
__device__ __forceinline__ bool lower(const FpArgs& a, int32_t v, int64_t best, int lane) {
    bool changed = false;
    if (lane == 0 && best < a.dist[v]) {
        long long old = atomicMin(reinterpret_cast<long long*>(&a.dist[v]), (long long)best);
        changed = best < old;
    }
    return __shfl_sync(group_mask<W>(), changed, (threadIdx.x & 31) & ~(W - 1));
}

template <int MODE, int G>
__device__ __forceinline__ void fp_round(const FpArgs& a, const Round& r, const int32_t* qin, int64_t m,
                                         const int64_t* hoin, int64_t mo, const int64_t* hiin, int64_t mi,
                                         int64_t& nb) {
    const int wl = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    // pieces deferred by the previous round: one warp per piece
    for (int64_t p = warp; p < mo; p += nwarps) {
        int32_t v;
        int sg;
        int64_t k;
        piece_decode(hoin[p], v, sg, k);
        int64_t s0 = a.ov.off[sg][v], s1 = a.ov.off[sg][v + 1];
        int64_t e0 = s0 + k * kPiece, e1 = min(e0 + kPiece, s1);
        int64_t dv = MODE == FP_RELAX ? a.dist[v] : 0;
        if (wl == 0) nb += 8 + 16 + (MODE == FP_RELAX ? 8 : 0);  // key, offsets, dist[v]
        if (MODE != FP_RELAX || dv < kInf) out_scan<MODE, 32>(a, r, v, dv, sg, e0, e1, wl, nb);
        wq_maybe_flush(r.qout, r.qcnt, r.fout, r.ffcnt);
    }
    if (MODE == FP_PULL) {
        for (int64_t p = warp; p < mi; p += nwarps) {
            int32_t v;
            int sg;
            int64_t k;
            piece_decode(hiin[p], v, sg, k);
            int64_t s0 = a.ix.off[v], s1 = a.ix.off[v + 1];
            int64_t e0 = s0 + k * kPiece, e1 = min(e0 + kPiece, s1);
            if (wl == 0) nb += 8 + 16 + 8;  // key, offsets, dist[v]
            int64_t best = in_min<32>(a, e0, e1, wl, nb);
            if (lower<32>(a, v, best, wl)) out_visit<MODE, 32>(a, r, v, 0, wl, nb);
            wq_maybe_flush(r.qout, r.qcnt, r.fout, r.ffcnt);
        }
    }
    // the queue: one group of G lanes per vertex
    GROUP_LOOP_BEGIN_G(m, G)
    (void)gw;
    if (valid) {
        int32_t v = qin[_t];
        if (lane == 0) nb += 4 + (MODE == FP_RELAX ? 8 : 0);  // queue entry, dist[v]
        if (MODE == FP_RELAX) {
            int64_t dv = a.dist[v];
            // Chaining: after scanning v, the group follows one near target it
            // lowered itself (the lowest lane's) within this round, up to
            // a.chain times; the other lowered targets are queued as usual.
            // A high-diameter graph (the grid) then advances several hops per
            // grid barrier.  Relaxation is monotone and the followed vertex is
            // not stamped, so a later, lower relaxation by another group still
            // queues it: the least fixpoint is unchanged.
            for (int depth = 0; dv < kInf; ++depth) {
                int32_t cand = -1;
                out_visit<MODE, G>(a, r, v, dv, lane, nb, depth < a.chain ? &cand : nullptr);
                const unsigned gm = group_mask<G>();
                const unsigned hm = __ballot_sync(gm, cand >= 0) & gm;
                if (!hm) break;
                const int src = __ffs(hm) - 1;
                const int32_t nxt = __shfl_sync(gm, cand, src);
                if (cand >= 0 && (int)(threadIdx.x & 31) != src && claim(a.stamp, cand, r.id))
                    enqueue_w(0, r.qout, r.qcnt, cand);
                v = nxt;
                dv = a.dist[v];
                if (lane == 0) nb += 8;
            }
        } else if (MODE == FP_WALK) {
            // the same chaining down the tree: each vertex has one parent, so a
            // followed child is visited once either way
            for (int depth = 0;; ++depth) {
                int32_t cand = -1;
                out_visit<MODE, G>(a, r, v, 0, lane, nb, depth < a.chain ? &cand : nullptr);
                const unsigned gm = group_mask<G>();
                const unsigned hm = __ballot_sync(gm, cand >= 0) & gm;
                if (!hm) break;
                const int src = __ffs(hm) - 1;
                const int32_t nxt = __shfl_sync(gm, cand, src);
                if (cand >= 0 && (int)(threadIdx.x & 31) != src && claim(a.stamp, cand, r.id))
                    enqueue_w(0, r.qout, r.qcnt, cand);
                v = nxt;
            }
        } else {
            int64_t s0 = a.ix.off[v], s1 = a.ix.off[v + 1];
            if (lane == 0) nb += 16 + 8;  // in-offsets, dist[v]
            if (s1 - s0 > kHeavy) {
                int64_t np = (s1 - s0 + kPiece - 1) / kPiece;
                unsigned long long base = 0;
                if (lane == 0) base = atomicAdd(r.hicnt, (unsigned long long)np);
                base = __shfl_sync(group_mask<G>(), base, (threadIdx.x & 31) & ~(G - 1));
                for (int64_t k = lane; k < np; k += G) r.hiout[base + k] = piece_key(v, 0, k);
            } else {
                int64_t best = in_min<G>(a, s0, s1, lane, nb);
                if (lower<G>(a, v, best, lane)) out_visit<MODE, G>(a, r, v, 0, lane, nb);
            }
        }
    }
    wq_maybe_flush(r.qout, r.qcnt, r.fout, r.ffcnt);
    GROUP_LOOP_END
}

// near-far split: pile entries below theta join the queue, the rest move to
// the next pile
__device__ __forceinline__ void split_round(const FpArgs& a, const Round& r, const int32_t* src, int64_t F,
                                            int64_t& nb) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    // warp-uniform trip count, so the buffers can flush between steps
    for (int64_t i0 = blockIdx.x * (int64_t)blockDim.x + (threadIdx.x & ~31); i0 < F; i0 += stride) {
        wq_maybe_flush(r.qout, r.qcnt, r.fout, r.ffcnt);
        const int64_t i = i0 + (threadIdx.x & 31);
        if (i >= F) continue;
        int32_t v = src[i];
        nb += 4 + 8;  // pile entry, dist[v]
        int64_t d = a.dist[v];
        if (d == kInf) {  // unreached seed: re-enters when relaxed
            a.infar[v] = 0;
        } else if (d < r.theta) {
            a.infar[v] = 0;
            if (claim(a.stamp, v, r.id)) enqueue_w(0, r.qout, r.qcnt, v);
        } else {
            a.infar[v] = 1;
            if (d < __ldcg(r.ffmin)) atomicMin(r.ffmin, (long long)d);
            enqueue_w(1, r.fout, r.ffcnt, v);
        }
    }
}

#ifndef GD_FP_RELAX_MINB
#define GD_FP_RELAX_MINB 4
#endif
template <int MODE, int G>
__global__ void __launch_bounds__(kThreads, MODE == FP_RELAX ? GD_FP_RELAX_MINB : 4) k_fixpoint(FpArgs a) {
    cg::grid_group grid = cg::this_grid();
    const bool leader = grid.thread_rank() == 0;
    const int32_t round0 = (int32_t)a.ctr[0];
    const bool nf = MODE == FP_RELAX && a.delta > 0;
    int64_t theta = kInf;  // every relaxation is near unless near-far
    if (nf) theta = 0;
    int nsplit = 0;  // pile = far[nsplit % 3]
    int64_t nb = 0;  // this thread's algorithmic bytes (a.acc only)
    int64_t it = 0;
    wq_init();
    for (;; ++it) {
        const volatile unsigned long long* c = a.cnt + 3 * (it % 3);
        int64_t m = (int64_t)c[0];
        const int64_t mo = (int64_t)c[1], mi = (int64_t)c[2];
        const int p = nsplit % 3;
        int64_t F = 0;
        bool split = false;
        if (nf && it == 0) {  // the seeds are split like a pile
            F = m;
            m = 0;
            split = true;
        } else if (nf && (m | mo | mi) == 0) {
            F = (int64_t)((const volatile unsigned long long*)a.fcnt)[p];
            split = true;
        }
        if ((m | mo | mi | F) == 0) break;
        // the cap counts work rounds, as fixedPoint counts body runs
        // (interp.py:800-813); a near-far split round only moves a pile
        if (!split && it - nsplit >= a.cap) {
            if (leader) a.ctr[2] = 1;
            break;
        }
        if (split) {
            int64_t lo = ((const volatile long long*)a.fmin)[p];
            theta = max(sat_add(theta, a.delta), sat_add(lo, a.delta));
        }
        if (leader) {
            unsigned long long* z = a.cnt + 3 * ((it + 2) % 3);
            z[0] = z[1] = z[2] = 0;
            if (split) {
                a.fcnt[(p + 2) % 3] = 0;
                a.fmin[(p + 2) % 3] = kInf;
                a.ctr[5] += 1;
            }
            a.ctr[3] += m;  // queue entries processed (diagnostics)
            a.ctr[4] += mo + mi;
        }
        const int nx = (it + 1) & 1;
        unsigned long long* cn = a.cnt + 3 * ((it + 1) % 3);
        const int fo = split ? (p + 1) % 3 : p;
        Round r{round0 + (int32_t)it + 1, theta, a.far[fo], a.fcnt + fo, a.fmin + fo,
                a.q[nx], cn, a.ho[nx], cn + 1, a.hi[nx], cn + 2};
        if (split) split_round(a, r, it == 0 ? a.seeds : a.far[p], F, nb);
        else fp_round<MODE, G>(a, r, it == 0 ? a.seeds : a.q[it & 1], m, a.ho[it & 1], mo, a.hi[it & 1], mi, nb);
        wq_flush(r.qout, r.qcnt, r.fout, r.ffcnt);
        grid.sync();
        if (split) ++nsplit;
    }
    // it > 0: a barrier separates every thread's read of ctr[0] from this write
    if (leader && it > 0) {
        a.ctr[0] = round0 + it;
        a.ctr[1] += it;
    }
    if (a.acc) {
        for (int o = 16; o; o >>= 1) nb += __shfl_xor_sync(0xffffffffu, nb, o);
        if ((threadIdx.x & 31) == 0 && nb) atomicAdd(reinterpret_cast<unsigned long long*>(a.acc),
                                                     (unsigned long long)nb);
    }
}

// decrementalSSSP's pull fixpoint (sssp_dynamic.sp:68-86) as one pull sweep
// over the stale list plus a near-far push from it: after the walk the
// non-stale distances are exact (their tree paths survive the deletes), so
// both reach the same least fixpoint over the stale set.  Vertices with more
// than kHeavy in-arcs go to `heavy` and are pulled by a whole CTA.
template <int G>
__global__ void __launch_bounds__(kThreads) k_pull_once(const int32_t* list, const int64_t* d_m, IdxView ix,
                                                        int64_t* dist, int32_t* heavy, unsigned long long* nheavy) {
    const int64_t m = *d_m;
    FpArgs a;
    a.ix = ix;
    a.dist = dist;
    GROUP_LOOP_BEGIN_G(m, G)
    (void)gw;
    if (valid) {
        int32_t v = list[_t];
        int64_t s0 = ix.off[v], s1 = ix.off[v + 1];
        if (s1 - s0 > kHeavy) {
            if (lane == 0) heavy[atomicAdd(nheavy, 1ULL)] = v;
        } else {
            int64_t nb = 0;  // unused here
            int64_t best = in_min<G>(a, s0, s1, lane, nb);
            if (lane == 0 && best < dist[v]) atomicMin(reinterpret_cast<long long*>(&dist[v]), (long long)best);
        }
    }
    GROUP_LOOP_END
}

__global__ void __launch_bounds__(kThreads) k_pull_heavy(const int32_t* heavy, const unsigned long long* nheavy,
                                                         IdxView ix, int64_t* dist) {
    __shared__ long long part[kThreads / 32];
    const int64_t nh = (int64_t)*nheavy;
    for (int64_t h = blockIdx.x; h < nh; h += gridDim.x) {
        int32_t v = heavy[h];
        int64_t best = kInf;
#pragma unroll 4
        for (int64_t e = ix.off[v] + threadIdx.x; e < ix.off[v + 1]; e += kThreads) {
            int32_t u = ix.col[e];
            if (u < 0) continue;
            int64_t c = sat_add(dist[u], ix.w ? (int64_t)ix.w[e] : 1);
            best = c < best ? c : best;
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            long long x = __shfl_xor_sync(0xffffffffu, (long long)best, o);
            best = x < best ? x : best;
        }
        if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = best;
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int j = 1; j < kThreads / 32; ++j) best = part[j] < best ? part[j] : best;
            if (best < dist[v]) atomicMin(reinterpret_cast<long long*>(&dist[v]), (long long)best);
        }
        __syncthreads();
    }
}

__global__ void k_wsum(const int32_t* col, const int32_t* w, int64_t ns, unsigned long long* acc) {
    unsigned long long sum = 0, cnt = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < ns; i += (int64_t)gridDim.x * blockDim.x)
        if (col[i] >= 0) {
            sum += (unsigned long long)max(w[i], 0);
            ++cnt;
        }
    for (int o = 16; o; o >>= 1) {
        sum += __shfl_xor_sync(0xffffffffu, sum, o);
        cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    }
    if ((threadIdx.x & 31) == 0 && cnt) {
        atomicAdd(&acc[0], sum);
        atomicAdd(&acc[1], cnt);
    }
}

__global__ void k_fp_prep(unsigned long long* cnt, const int64_t* d_n, int64_t n, unsigned long long* fcnt,
                          long long* fmin) {
    cnt[0] = (unsigned long long)(d_n ? *d_n : n);
    for (int i = 1; i < 6; ++i) cnt[i] = 0;
    if (fcnt) {
        fcnt[0] = fcnt[1] = fcnt[2] = 0;
        fmin[0] = 0;  // a lower bound for the seeds
        fmin[1] = fmin[2] = kInf;
    }
}

// parent = min-id in-neighbour u with dist[u] + w == dist[v] (sssp_dynamic.sp:23-34)
template <int G>
__global__ void __launch_bounds__(kThreads) k_fix_parent(const int32_t* list, const int64_t* d_m, int64_t m,
                                                         IdxView ix, const int64_t* dist, int32_t* parent,
                                                         int32_t src, int32_t* heavy, unsigned long long* nheavy) {
    if (d_m) m = *d_m;
    GROUP_LOOP_BEGIN_G(m, G)
    int32_t v = valid ? (list ? list[_t] : (int32_t)_t) : 0;
    int64_t dv = valid ? dist[v] : kInf;
    bool act = valid && v != src && dv < kInf;
    int32_t best = INT_MAX;
    const int64_t a = act ? ix.off[v] : 0, b = act ? ix.off[v + 1] : 0;
    const bool hv = heavy && b - a > kHeavy;  // group-uniform: a whole CTA takes it below
    if (hv && lane == 0) heavy[atomicAdd(nheavy, 1ULL)] = v;
    if (act && !hv) {
        for (int64_t e = a + lane; e < b; e += G) {
            int32_t u = ix.col[e];
            if (u < 0) continue;
            if (sat_add(dist[u], ix.w ? (int64_t)ix.w[e] : 1) == dv && u < best) best = u;
        }
    }
#pragma unroll
    for (int o = G / 2; o; o >>= 1) {
        int32_t x = __shfl_xor_sync(0xffffffffu, best, o, G);
        best = x < best ? x : best;
    }
    if (act && !hv && lane == 0) parent[v] = best == INT_MAX ? -1 : best;
    GROUP_LOOP_END
}

// the parent fix-up of vertices with more than kHeavy in-arcs: one CTA each
__global__ void __launch_bounds__(kThreads) k_fix_parent_heavy(const int32_t* heavy, const unsigned long long* nheavy,
                                                               IdxView ix, const int64_t* dist, int32_t* parent) {
    __shared__ int32_t part[kThreads / 32];
    const int64_t nh = (int64_t)*nheavy;
    for (int64_t h = blockIdx.x; h < nh; h += gridDim.x) {
        const int32_t v = heavy[h];
        const int64_t dv = dist[v];
        int32_t best = INT_MAX;
        for (int64_t e = ix.off[v] + threadIdx.x; e < ix.off[v + 1]; e += kThreads) {
            int32_t u = ix.col[e];
            if (u < 0) continue;
            if (sat_add(dist[u], ix.w ? (int64_t)ix.w[e] : 1) == dv && u < best) best = u;
        }
        for (int o = 16; o; o >>= 1) best = min(best, __shfl_xor_sync(0xffffffffu, best, o));
        if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = best;
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int j = 1; j < kThreads / 32; ++j) best = min(best, part[j]);
            parent[v] = best == INT_MAX ? -1 : best;
        }
        __syncthreads();
    }
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

// ---------------------------------------------------------------------------
// Partitioned store (SSSP::fixpoint_dist): owned flagged vertices as a list,
// the outbox packed as (vertex, value) messages by owner, and the owners'
// application of the messages they receive.
// ---------------------------------------------------------------------------
__global__ void k_select_owned(const uint8_t* flags, int64_t lo, int64_t hi, int32_t* list, int64_t* cnt) {
    for (int64_t v = lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < hi;
         v += (int64_t)gridDim.x * blockDim.x) {
        const bool f = flags[v] != 0;
        const unsigned mk = __ballot_sync(__activemask(), f);
        if (!f) continue;
        const int lane = threadIdx.x & 31, leader = __ffs(mk) - 1;
        unsigned long long base = 0;
        if (lane == leader) base = atomicAdd(reinterpret_cast<unsigned long long*>(cnt), (unsigned long long)__popc(mk));
        base = __shfl_sync(mk, base, leader);
        list[base + __popc(mk & ((1u << lane) - 1))] = (int32_t)v;
    }
}

__global__ void k_msg_count(const int32_t* box, const unsigned long long* nbox, Blocks b, unsigned long long* cnt) {
    const int64_t m = (int64_t)*nbox;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(&cnt[b.owner(box[i])], 1ULL);
}

__global__ void k_msg_offsets(const unsigned long long* cnt, int world, unsigned long long* cur) {
    unsigned long long a = 0;
    for (int p = 0; p < world; ++p) {
        cur[p] = a;
        a += cnt[p];
    }
}

// (vertex, dist lo32, dist hi32) in owner-major order
__global__ void k_msg_pack(const int32_t* box, const unsigned long long* nbox, Blocks b, const int64_t* dist,
                           unsigned long long* cur, int32_t* packed) {
    const int64_t m = (int64_t)*nbox;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t t = box[i];
        const int64_t pos = (int64_t)atomicAdd(&cur[b.owner(t)], 1ULL);
        const uint64_t d = (uint64_t)dist[t];
        packed[3 * pos] = t;
        packed[3 * pos + 1] = (int32_t)(uint32_t)d;
        packed[3 * pos + 2] = (int32_t)(uint32_t)(d >> 32);
    }
}

// owner side: min the received distance in (relax) or invalidate (walk);
// each changed vertex seeds the next local fixpoint once (sstamp)
__global__ void k_msg_apply(const int32_t* msg, int64_t m, int mode, int64_t* dist, int32_t* parent, uint8_t* flags,
                            int32_t* sstamp, int32_t step, int32_t* seeds, int64_t* nseeds) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t t = msg[3 * i];
        bool changed = false;
        if (mode == FP_RELAX) {
            const int64_t c = (int64_t)(((uint64_t)(uint32_t)msg[3 * i + 2] << 32) | (uint32_t)msg[3 * i + 1]);
            if (c < dist[t]) {
                const long long old = atomicMin(reinterpret_cast<long long*>(&dist[t]), (long long)c);
                changed = c < old;
                if (changed && flags) flags[t] = 1;  // touched
            }
        } else {  // FP_WALK: the sender saw parent[t] == its walked vertex
            if (!flags[t]) {
                flags[t] = 1;  // stale
                dist[t] = kInf;
                parent[t] = -1;
                changed = true;
            }
        }
        if (changed && atomicMax(&sstamp[t], step) < step)
            seeds[atomicAdd(reinterpret_cast<unsigned long long*>(nseeds), 1ULL)] = t;
    }
}

inline unsigned group_grid(int64_t m, int g = kG) {
    const int64_t per = 32 / g;
    return grid_for(((m + per - 1) / per) * 32, kThreads, 148LL * 32);
}

// co-resident grid for the cooperative fixpoint: <= 4 CTAs per SM keeps the
// barrier cheap while leaving 32 warps per SM for latency hiding
template <int MODE, int G>
unsigned coop_grid() {
    static unsigned g = 0;
    if (!g) {
        int dev = 0, sms = 0, nb = 0;
        GD_CUDA(cudaGetDevice(&dev));
        GD_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        GD_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_fixpoint<MODE, G>, kThreads, 0));
        if (nb < 1) throw GdError(GD_ERR_CUDA, "fixpoint kernel cannot be resident");
        int per = 4;
        if (const char* e = getenv("GD_FP_CTAS_PER_SM")) per = std::max(1, atoi(e));
        g = (unsigned)(sms * std::min(nb, per));
    }
    return g;
}

}  // namespace

SSSP::SSSP(Store* st, int64_t s, int64_t cap) : AlgoBase(ALGO_SSSP, st), src((int32_t)s), cap_factor(cap) {
    if (!st->with_reverse)
        throw GdError(GD_ERR_CONFIG, "graph was loaded without reverse-adjacency maintenance");
    if (s < 0 || s >= st->n) throw GdError(GD_ERR_EXEC, "source node out of range");
    cudaStream_t cs = stream();
    int64_t n = g->n;
    dist.alloc(n, cs);
    parent.alloc(n, cs);
    stamp.alloc(n, cs);
    hstamp.alloc(n, cs);
    fa.alloc(n, cs);
    fb.alloc(n, cs);
    fr.init(n, cs);
    ctr.alloc(6 + kFpSlots, cs);
    fcnt.alloc(3, cs);
    fmin.alloc(3, cs);
    infar.alloc(n, cs);
    infar.zero(cs);
    for (int j = 0; j < 3; ++j) far[j].alloc(std::max<int64_t>(n, 1), cs);
    // near-far bucket width: 3x the mean live arc weight (unweighted graphs
    // relax level by level already)
    if (g->weighted && !g->segs.empty() && g->segs[0].nslots) {
        DBuf<unsigned long long> acc(2, cs);
        acc.zero(cs);
        GD_KERNEL(k_wsum, grid_for(g->segs[0].nslots, 256, 148 * 8), 256, 0, cs, g->segs[0].col.get(),
                  g->segs[0].w.get(), g->segs[0].nslots, acc.get());
        unsigned long long h[2];
        read_small(cs, h, acc.get(), sizeof(h));
        if (h[1]) delta = std::max<int64_t>(1, (int64_t)(3 * h[0] / h[1]));
    }
    if (const char* e = getenv("GD_SSSP_DELTA")) delta = atoll(e);
    ctr.zero(cs);
    dcount.alloc(1, cs);
    if (g->part) {
        outbox.alloc(std::max<int64_t>(n, 1), cs);
        gstamp.alloc(std::max<int64_t>(n, 1), cs);
        gstamp.zero(cs);
        sstamp.alloc(std::max<int64_t>(n, 1), cs);
        sstamp.zero(cs);
        seeds2.alloc(std::max<int64_t>(n, 1), cs);
        nbox.alloc(1, cs);
    }
    ProfScope ps(&prof);
    timer.begin(PH_STATIC);
    GD_KERNEL(k_init, grid_for(n, 256), 256, 0, cs, dist.get(), parent.get(), stamp.get(), hstamp.get(), n);
    GD_KERNEL(k_set_i64, 1, 1, 0, cs, dist.get(), (int64_t)src, (int64_t)0);
    int32_t seed = src;
    DBuf<int32_t> sq(1, cs);
    GD_CUDA(cudaMemcpyAsync(sq.get(), &seed, 4, cudaMemcpyHostToDevice, cs));
    if (g->part) {  // the source's owner seeds the supersteps
        DBuf<int64_t> ns(1, cs);
        const int64_t one = src >= g->own_lo && src < g->own_hi ? 1 : 0;
        GD_CUDA(cudaMemcpyAsync(ns.get(), &one, 8, cudaMemcpyHostToDevice, cs));
        DBuf<int32_t> sl(std::max<int64_t>(n, 1), cs);
        copy_d2d(cs, sl.get(), sq.get(), 4);
        fixpoint_dist(FP_RELAX, sl.get(), ns.get(), nullptr);
        sync(true, false, nullptr);
        DBuf<uint8_t> all(std::max<int64_t>(n, 1), cs);
        fill_d(cs, all.get(), 1, n);
        DBuf<int32_t> list(std::max<int64_t>(n, 1), cs);
        owned_list(all.get(), list.get(), ns.get());
        fix_parents(list.get(), ns.get(), n);
        sync(false, true, nullptr);
    } else {
        fixpoint(FP_RELAX, sq.get(), nullptr, 1, nullptr);
        fix_parents(nullptr, nullptr, n);
    }
    finish();
    // low-diameter graphs (R-MAT: tens of rounds) gain nothing from buckets
    // and pay their extra rounds; keep near-far for the deep ones (grids)
    if (!getenv("GD_SSSP_DELTA") && iterations < kNearFarMinRounds) delta = 0;
    timer.end_all();
}

bool SSSP::narrow_groups() const {
    if (const char* e = getenv("GD_SSSP_G")) return atoi(e) == 4;
    return g->n > 0 && g->total_slots() <= 6 * g->n;
}

void SSSP::fixpoint(int mode, const int32_t* seeds, const int64_t* d_nseeds, int64_t nseeds, uint8_t* flags,
                    const uint8_t* only) {
    cudaStream_t s = stream();
    if (!d_nseeds && nseeds == 0) return;
    const bool nf = mode == FP_RELAX && delta > 0;
    GD_KERNEL(k_fp_prep, 1, 1, 0, s, fr.cnt.get(), d_nseeds, nseeds, nf ? fcnt.get() : nullptr,
              nf ? fmin.get() : nullptr);
    FpArgs a;
    a.outbox = nullptr;  // set by fixpoint_dist
    a.noutbox = nullptr;
    a.gstamp = nullptr;
    a.launch = 0;
    a.own_lo = 0;
    a.own_hi = g->n;
    if (g->part) {
        a.own_lo = g->own_lo;
        a.own_hi = g->own_hi;
        a.outbox = outbox.get();
        a.noutbox = nbox.get();
        a.gstamp = gstamp.get();
        a.launch = ++launch_id;
    }
    a.delta = nf ? delta : 0;
    for (int j = 0; j < 3; ++j) a.far[j] = nf ? far[j].get() : nullptr;
    a.fcnt = fcnt.get();
    a.fmin = fmin.get();
    a.infar = infar.get();
    a.ov = g->out_view();
    a.ix = g->rev.view();
    a.dist = dist.get();
    a.parent = parent.get();
    a.flags = flags;
    a.only = mode == FP_RELAX ? only : nullptr;
    a.stamp = stamp.get();
    a.seeds = seeds;
    a.q[0] = fr.q[0].get();
    a.q[1] = fr.q[1].get();
    // piece lists: every vertex is cut at most once per round; a vertex with
    // d > kHeavy arcs spread over nseg segments yields <= d/kPiece + nseg pieces
    int64_t S = g->total_slots(), R = mode == FP_PULL ? g->rev.nnz : 0;
    int64_t capo = S / kPiece + (int64_t)a.ov.nseg * (S / kHeavy + 1) + 64;
    int64_t capi = R / kPiece + R / kHeavy + 64;
    for (int j = 0; j < 2; ++j) {
        ho[j].ensure(capo, s);
        hi[j].ensure(capi, s);
        a.ho[j] = ho[j].get();
        a.hi[j] = hi[j].get();
    }
    a.hstamp = hstamp.get();
    a.cnt = fr.cnt.get();
    a.ctr = ctr.get();
    a.cap = std::max<int64_t>(1, cap_factor * std::max<int64_t>(g->n, 1));  // ExecContext.iteration_cap
    const int chain_env = getenv("GD_SSSP_CHAIN") ? atoi(getenv("GD_SSSP_CHAIN")) : kChainDefault;
    // a followed hop saves a round, so rounds drop below the reference's
    // sweeps; a cap below n (iteration_cap_factor 0) must still trip where
    // the reference's does, so those fixpoints advance one hop per round
    // chaining pays on deep graphs only (C4 grid: relax 25.6 -> 21.5 ms, walk
    // 6.3 -> 4.9 ms per batch); on R-MAT (near-far off, delta == 0) it
    // unbalanced the few wide rounds (relax 0.233 -> 0.246 ms)
    a.chain = a.cap >= g->n && delta > 0 ? chain_env : 0;
    void* args[] = {&a};
    static const char* names[] = {"sssp_relax", "sssp_walk", "sssp_pull"};
    // 4 lanes per queued vertex on low-degree graphs (the grid: 4 arcs a
    // vertex left half of an 8-lane group idle), 8 otherwise
    const bool narrow = narrow_groups();
    const void* fn = mode == FP_RELAX  ? (narrow ? (const void*)k_fixpoint<FP_RELAX, 4> : (const void*)k_fixpoint<FP_RELAX, 8>)
                     : mode == FP_WALK ? (narrow ? (const void*)k_fixpoint<FP_WALK, 4> : (const void*)k_fixpoint<FP_WALK, 8>)
                                       : (narrow ? (const void*)k_fixpoint<FP_PULL, 4> : (const void*)k_fixpoint<FP_PULL, 8>);
    unsigned grid = mode == FP_RELAX  ? (narrow ? coop_grid<FP_RELAX, 4>() : coop_grid<FP_RELAX, 8>())
                    : mode == FP_WALK ? (narrow ? coop_grid<FP_WALK, 4>() : coop_grid<FP_WALK, 8>())
                                      : (narrow ? coop_grid<FP_PULL, 4>() : coop_grid<FP_PULL, 8>());
    int pi = prof_begin(names[mode], 0, s);
    // profiled launches sum their algorithmic bytes into a slot that
    // finish() reads with the round counters (no extra read-back)
    a.acc = nullptr;
    if (pi >= 0 && nfp < kFpSlots) {
        a.acc = ctr.get() + 6 + nfp;
        fp_prof[nfp++] = pi;
    }
    GD_CUDA(cudaLaunchCooperativeKernel(fn, grid, kThreads, args, 0, s));
    count_launch();
    prof_end(pi, s);
}

void SSSP::owned_list(const uint8_t* flags, int32_t* list, int64_t* d_m) {
    cudaStream_t s = stream();
    fill_d(s, d_m, 0, 8);
    const int64_t lo = g->own_lo, hi = g->own_hi;
    if (hi > lo) GD_KERNEL(k_select_owned, grid_for(hi - lo, 256), 256, 0, s, flags, lo, hi, list, d_m);
}

void SSSP::sync(bool d, bool p, uint8_t* flags) {
    if (!g->part) return;
    cudaStream_t s = stream();
    if (d) g->part->allgatherv(dist.get(), g->blocks, 8, s);
    if (p) g->part->allgatherv(parent.get(), g->blocks, 4, s);
    if (flags) g->part->allgatherv(flags, g->blocks, 1, s);
}

// Supersteps over the partition: a local fixpoint over the owned vertices
// (the cooperative kernel, ghost targets listed in the outbox), then the
// outboxes go to the vertices' owners (one all-to-all), which apply them --
// min for a relaxation, invalidation for a walk -- and seed the next local
// fixpoint with what changed.  Ends when no rank has seeds (an all-reduce).
// Relaxation is monotone and the walk's descendant set schedule-free, so
// the result is the single-GPU fixpoint.
void SSSP::fixpoint_dist(int mode, int32_t* seeds, int64_t* d_nseeds, uint8_t* flags, const uint8_t* only) {
    cudaStream_t s = stream();
    const Comm* c = g->part;
    const Blocks& b = g->blocks;
    const int W = c->world;
    const int64_t n = g->n;
    int32_t* cur = seeds;
    int32_t* nxt = seeds2.get();
    DBuf<int64_t> tot(1, s), nn(1, s);
    packed.ensure(3 * std::max<int64_t>(n, 1), s);
    const int64_t cap = std::max<int64_t>(1, cap_factor * std::max<int64_t>(n, 1));
    for (int64_t step = 0;; ++step) {
        if (step >= cap) throw GdError(GD_ERR_DIVERGED, "fixed point diverged");
        fill_d(s, nbox.get(), 0, sizeof(unsigned long long));
        fixpoint(mode, cur, d_nseeds, 0, flags, only);
        DBuf<unsigned long long> cnt(2 * W, s);
        cnt.zero(s);
        GD_KERNEL(k_msg_count, 148 * 4, 256, 0, s, outbox.get(), nbox.get(), b, cnt.get());
        GD_KERNEL(k_msg_offsets, 1, 1, 0, s, cnt.get(), W, cnt.get() + W);
        GD_KERNEL(k_msg_pack, 148 * 4, 256, 0, s, outbox.get(), nbox.get(), b, dist.get(), cnt.get() + W,
                  packed.get());
        DBuf<int32_t> recv;
        const int64_t m = c->alltoallv_i32(packed.get(), reinterpret_cast<const int64_t*>(cnt.get()), 3, recv, s);
        fill_d(s, nn.get(), 0, 8);
        ++step_id;
        if (m) GD_KERNEL(k_msg_apply, grid_for(m, 256), 256, 0, s, recv.get(), m, mode, dist.get(), parent.get(),
                         flags, sstamp.get(), step_id, nxt, nn.get());
        copy_d2d(s, tot.get(), nn.get(), 8);
        c->allreduce_sum_i64(tot.get(), 1, s);
        const int64_t total = read_scalar(s, tot.get());
        static const bool dbg = getenv("GD_SSSP_DEBUG") != nullptr;
        if (dbg)
            fprintf(stderr, "[sssp-dist] rank %d mode %d step %lld: sent %llu received %lld seeds(all) %lld\n",
                    c->rank, mode, (long long)step, (unsigned long long)read_scalar(s, nbox.get()), (long long)m,
                    (long long)total);
        if (total == 0) break;
        copy_d2d(s, d_nseeds, nn.get(), 8);
        std::swap(cur, nxt);
    }
}

void SSSP::fix_parents(const int32_t* list, const int64_t* d_m, int64_t m) {
    if (m == 0) return;
    cudaStream_t s = stream();
    IdxView ix = g->rev.view();
    heavy.ensure(g->rev.nnz / kHeavy + 64, s);
    unsigned long long* nh = fr.cnt.get() + 10;
    fill_d(s, nh, 0, sizeof(unsigned long long));
    // 4 lanes per vertex on low-degree graphs, as in the fixpoints
    const bool narrow = narrow_groups();
    if (narrow)
        GD_KERNEL_T("sssp_parent", 0, k_fix_parent<4>, group_grid(m, 4), kThreads, 0, s, list, d_m, m, ix,
                    dist.get(), parent.get(), src, heavy.get(), nh);
    else
    GD_KERNEL_T("sssp_parent", 0, k_fix_parent<8>, group_grid(m), kThreads, 0, s, list, d_m, m, ix, dist.get(),
                parent.get(), src, heavy.get(), nh);
    GD_KERNEL_T("sssp_parent", 0, k_fix_parent_heavy, 148 * 4, kThreads, 0, s, heavy.get(), nh, ix, dist.get(),
                parent.get());
}

// one read-back per batch: total rounds and the divergence flag
void SSSP::finish() {
    long long h[6 + kFpSlots];
    read_small(stream(), h, ctr.get(), (6 + nfp) * sizeof(long long));
    if (nfp) {
        for (int j = 0; j < nfp; ++j) prof_set_bytes(fp_prof[j], h[6 + j]);
        fill_d(stream(), ctr.get() + 6, 0, nfp * sizeof(long long));
        nfp = 0;
    }
    static const bool dbg = getenv("GD_SSSP_DEBUG") != nullptr;
    if (dbg)
        fprintf(stderr, "[sssp] rounds %lld (+%lld) visits %lld pieces %lld splits %lld\n", h[1], h[1] - iterations,
                h[3], h[4], h[5]);
    iterations = h[1];
    if (h[2]) {  // abandoned piles leave in-far marks behind
        infar.zero(stream());
        fill_d(stream(), ctr.get() + 2, 0, sizeof(long long));
        throw GdError(GD_ERR_DIVERGED, "fixed point diverged");
    }
}

// One Batch body on a vertex-partitioned store: the record handlers run on
// every rank over all records (dist / parent are replicated), the
// structural updates on the owners, each fixpoint as supersteps, and every
// phase ends with the owned blocks of what it changed gathered to all ranks
// -- so each phase starts from the same state on every rank.
void SSSP::batch_dist(DevBatch& b, int64_t batch_index) {
    cudaStream_t s = stream();
    const int64_t n = g->n;
    uint8_t* seed_del = fa.get();  // activeOnDelete, then stale
    uint8_t* seed_add = fb.get();  // activeOnAdd, then touched
    DBuf<int32_t> list(std::max<int64_t>(n, 1), s);
    DBuf<int64_t> nl(1, s);
    timer.begin(PH_PRE);
    fa.zero(s);
    fb.zero(s);
    if (b.kdel) GD_KERNEL(k_on_delete, grid_for(b.kdel, 256), 256, 0, s, b.ds.get(), b.dd.get(), b.kdel, dist.get(),
                          parent.get(), seed_del);
    timer.begin(PH_STRUCT);
    g->apply_deletes(b.ds.get(), b.dd.get(), b.kdel, nullptr);
    // decrementalSSSP (sssp_dynamic.sp:37-99)
    timer.begin(PH_PROP);
    GD_KERNEL(k_set_i64, 1, 1, 0, s, dist.get(), (int64_t)src, (int64_t)0);
    owned_list(seed_del, list.get(), nl.get());
    fixpoint_dist(FP_WALK, list.get(), nl.get(), seed_del);
    sync(true, true, seed_del);
    GD_KERNEL(k_set_i64, 1, 1, 0, s, dist.get(), (int64_t)src, (int64_t)0);
    owned_list(seed_del, list.get(), nl.get());
    {  // one pull sweep over the owned stale vertices, then the push restricted to stale targets
        IdxView ix = g->rev.view();
        heavy.ensure(g->rev.nnz / kHeavy + 64, s);
        fill_d(s, fr.cnt.get() + 9, 0, sizeof(unsigned long long));
        GD_KERNEL_T("sssp_pull", 0, (narrow_groups() ? &k_pull_once<4> : &k_pull_once<8>), group_grid(n, narrow_groups() ? 4 : 8), kThreads, 0, s, list.get(), nl.get(), ix, dist.get(),
                    heavy.get(), fr.cnt.get() + 9);
        GD_KERNEL_T("sssp_pull", 0, k_pull_heavy, 148 * 4, kThreads, 0, s, heavy.get(), fr.cnt.get() + 9, ix,
                    dist.get());
    }
    sync(true, false, nullptr);  // the pulled distances seed pushes on other ranks
    fixpoint_dist(FP_RELAX, list.get(), nl.get(), nullptr, seed_del);
    sync(true, false, nullptr);
    owned_list(seed_del, list.get(), nl.get());
    fix_parents(list.get(), nl.get(), n);
    sync(false, true, nullptr);
    timer.begin(PH_PRE);
    if (b.kadd) GD_KERNEL(k_on_add, grid_for(b.kadd, 256), 256, 0, s, b.as.get(), b.ad.get(), b.aw.get(), b.kadd,
                          g->weighted, dist.get(), seed_add);
    timer.begin(PH_STRUCT);
    g->apply_adds(b.as.get(), b.ad.get(), b.aw.get(), b.kadd);
    if (g->merge_due(batch_index)) {
        timer.begin(PH_MERGE);
        g->merge();
    } else {
        g->compact_rev();
    }
    struct_done();
    // incrementalSSSP (sssp_dynamic.sp:101-130)
    timer.begin(PH_PROP);
    owned_list(seed_add, list.get(), nl.get());
    fixpoint_dist(FP_RELAX, list.get(), nl.get(), seed_add);
    sync(true, false, seed_add);
    owned_list(seed_add, list.get(), nl.get());
    fix_parents(list.get(), nl.get(), n);
    sync(false, true, nullptr);
    finish();
    timer.end_all();
}

void SSSP::batch(DevBatch& b, int64_t batch_index) {
    if (g->part) {
        ProfScope ps(&prof);
        prof.reset_last();
        return batch_dist(b, batch_index);
    }
    cudaStream_t s = stream();
    int64_t n = g->n;
    ProfScope ps(&prof);
    prof.reset_last();
    uint8_t* seed_del = fa.get();  // activeOnDelete, then stale
    uint8_t* seed_add = fb.get();  // activeOnAdd, then touched
    DBuf<int32_t> list(std::max<int64_t>(n, 1), s);
    int64_t* nlist = dcount.get();

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
    select_flagged_index_async(s, seed_del, n, list.get(), nlist);
    fixpoint(FP_WALK, list.get(), nlist, 0, seed_del);
    GD_KERNEL(k_set_i64, 1, 1, 0, s, dist.get(), (int64_t)src, (int64_t)0);
    select_flagged_index_async(s, seed_del, n, list.get(), nlist);
    // one pull sweep + push (near-far when delta > 0): same fixpoint as the
    // reference's pull fixedPoint, 1.2-1.3x faster on R-MAT-24 at 10-20%;
    // GD_SSSP_DECR=0 selects the pull fixpoint (kept for A/B and tests)
    const bool pull_fixpoint = getenv("GD_SSSP_DECR") && atoi(getenv("GD_SSSP_DECR")) == 0;
    if (!pull_fixpoint) {
        IdxView ix = g->rev.view();
        heavy.ensure(g->rev.nnz / kHeavy + 64, s);
        fill_d(s, fr.cnt.get() + 9, 0, sizeof(unsigned long long));
        GD_KERNEL_T("sssp_pull", 0, (narrow_groups() ? &k_pull_once<4> : &k_pull_once<8>), group_grid(n, narrow_groups() ? 4 : 8), kThreads, 0, s, list.get(), nlist, ix, dist.get(),
                    heavy.get(), fr.cnt.get() + 9);
        GD_KERNEL_T("sssp_pull", 0, k_pull_heavy, 148 * 4, kThreads, 0, s, heavy.get(), fr.cnt.get() + 9, ix,
                    dist.get());
        // the push may lower stale targets only: a live arc into a non-stale
        // node need not be tight (OnAdd relaxes the record's own direction and
        // weight only), and the reference's pull never changes such a node
        fixpoint(FP_RELAX, list.get(), nlist, 0, nullptr, seed_del);
    } else {
        fixpoint(FP_PULL, list.get(), nlist, 0, seed_del);
    }
    fix_parents(list.get(), nlist, n);

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
    struct_done();

    // incrementalSSSP (sssp_dynamic.sp:101-130); touched starts as the seeds
    timer.begin(PH_PROP);
    select_flagged_index_async(s, seed_add, n, list.get(), nlist);
    fixpoint(FP_RELAX, list.get(), nlist, 0, seed_add);
    select_flagged_index_async(s, seed_add, n, list.get(), nlist);
    fix_parents(list.get(), nlist, n);
    finish();
    timer.end_all();
}

// parent widened to int64 on the handle's stream (parent64), for read-backs
const int64_t* SSSP::parent_i64() {
    cudaStream_t s = stream();
    int64_t n = g->n;
    parent64.ensure(std::max<int64_t>(n, 1), s);
    if (n) GD_KERNEL(k_read_parent, grid_for(n, 256), 256, 0, s, parent.get(), n, parent64.get());
    return parent64.get();
}

void SSSP::read_async(int64_t* h_dist, int64_t* h_parent) {
    cudaStream_t s = stream();
    int64_t n = g->n;
    if (!n) return;
    copy_out_async(h_dist, dist.get(), (size_t)n * 8, 0);
    if (h_parent) {
        parent64.ensure(n, s);
        GD_KERNEL(k_read_parent, grid_for(n, 256), 256, 0, s, parent.get(), n, parent64.get());
        copy_out_async(h_parent, parent64.get(), (size_t)n * 8, 1);
    }
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
