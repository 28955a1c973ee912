// gd_store.cu -- the GPU diff-CSR store.  See gd_store.cuh for the layout.
//
// Batch application is sort + segmented-scan shaped: records are radix-sorted
// by (src, dst), each requested source's chain is scanned once (split into
// 1024-slot work items so hub rows spread over many warps) against the sorted
// requests of that source, and the j-th record of a pair resolves to the j-th
// live occurrence of that pair in chain order -- the exact outcome of the
// reference's sequential per-record scans (dynamic.py:208-286).
//
// Slot positions are global slot ids (gid): the concatenation of segments in
// chain order (base first, then deltas), so sorting by gid is chain order.
#include <algorithm>
#include <cstring>

#include "gd_launch.cuh"
#include "gd_store.cuh"

namespace gdb {

namespace {

constexpr int kChunk = 1024;  // chain slots per delete-scan work item
constexpr int kScanILP = 4;    // loads in flight per lane in the chain scans

__device__ inline int seg_of(const int64_t* base, int nseg, int64_t gid) {
    int s = 0;
    while (s + 1 < nseg && base[s + 1] <= gid) ++s;
    return s;
}

// ---------------------------------------------------------------- build ----

__global__ void k_expand_edges(const int64_t* src, const int64_t* dst, const int64_t* w, int64_t m, bool as_given,
                               uint32_t* key, int32_t* val, int32_t* adst, int32_t* aw) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
        int32_t s = (int32_t)src[i], d = (int32_t)dst[i];
        int32_t wi = w ? (int32_t)w[i] : 1;
        if (as_given) {
            key[i] = (uint32_t)s;
            val[i] = (int32_t)i;
            adst[i] = d;
            aw[i] = wi;
        } else {  // dynamic.py:113-115: (src,dst) then (dst,src)
            key[2 * i] = (uint32_t)s;
            val[2 * i] = (int32_t)(2 * i);
            adst[2 * i] = d;
            aw[2 * i] = wi;
            key[2 * i + 1] = (uint32_t)d;
            val[2 * i + 1] = (int32_t)(2 * i + 1);
            adst[2 * i + 1] = s;
            aw[2 * i + 1] = wi;
        }
    }
}

__global__ void k_hist_rows(const int32_t* rows, int64_t m, int64_t* cnt) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(reinterpret_cast<unsigned long long*>(&cnt[rows[i]]), 1ULL);
}
__global__ void k_hist_rows_u32(const uint32_t* rows, int64_t m, int64_t* cnt) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(reinterpret_cast<unsigned long long*>(&cnt[rows[i]]), 1ULL);
}

template <typename T>
__global__ void k_gather(const T* in, const int32_t* idx, int64_t m, T* out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = in[idx[i]];
}

__global__ void k_key_split(const uint64_t* key, int64_t m, int sh, int32_t* row, int32_t* col) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
        if (row) row[i] = key_row(key[i], sh);
        if (col) col[i] = key_col(key[i], sh);
    }
}

void offsets_from_rows(cudaStream_t s, int64_t n, const int32_t* rows, int64_t m, DBuf<int64_t>& off) {
    DBuf<int64_t> cnt(n + 1, s);
    cnt.zero(s);
    if (m) GD_KERNEL(k_hist_rows, grid_for(m, 256), 256, 0, s, rows, m, cnt.get());
    off.alloc(n + 1, s);
    exclusive_scan_i64(s, cnt.get(), off.get(), n + 1);
}

// ------------------------------------------------------- delete requests ----

// Directed: key (s,d).  Undirected: key (min,max) -- records of one unordered
// pair consume occurrences of both arcs in stream order (dynamic.py:221-234).
__global__ void k_del_keys(const int32_t* s, const int32_t* d, int64_t k, bool directed, int sh, uint64_t* key,
                           int32_t* val) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < k; i += (int64_t)gridDim.x * blockDim.x) {
        int32_t a = s[i], b = d[i];
        if (!directed && a > b) {
            int32_t t = a;
            a = b;
            b = t;
        }
        key[i] = pair_key(a, b, sh);
        val[i] = (int32_t)i;
    }
}

// Expand sorted records into directed requests (row, col, occurrence).
__global__ void k_del_requests(const uint64_t* skey, const int32_t* srec, int64_t k, const int32_t* s,
                               const int32_t* d, bool directed, int sh, uint64_t* rq_key, int32_t* rq_occ,
                               int32_t* rq_rec, uint8_t* rq_which, int32_t* rq_ord) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < k; i += (int64_t)gridDim.x * blockDim.x) {
        uint64_t key = skey[i];
        int32_t j = 0;  // rank within the run of equal keys (runs are short)
        for (int64_t p = i - 1; p >= 0 && skey[p] == key; --p) ++j;
        int32_t r = srec[i];
        int32_t a = s[r], b = d[r];
        if (directed) {
            rq_key[i] = pair_key(a, b, sh);
            rq_occ[i] = j;
            rq_rec[i] = r;
            rq_which[i] = 0;
            rq_ord[i] = (int32_t)i;
        } else {
            int64_t o = 2 * i;
            if (a != b) {
                rq_key[o] = pair_key(a, b, sh);
                rq_occ[o] = j;
                rq_key[o + 1] = pair_key(b, a, sh);
                rq_occ[o + 1] = j;
            } else {  // self-loop: two slots per record (dynamic.py:231-234)
                rq_key[o] = pair_key(a, a, sh);
                rq_occ[o] = 2 * j;
                rq_key[o + 1] = pair_key(a, a, sh);
                rq_occ[o + 1] = 2 * j + 1;
            }
            rq_rec[o] = r;
            rq_rec[o + 1] = r;
            rq_which[o] = 0;
            rq_which[o + 1] = 1;
            rq_ord[o] = (int32_t)o;
            rq_ord[o + 1] = (int32_t)(o + 1);
        }
    }
}

// Undirected deletes: every record r gives requests 2r (s->d) and 2r+1
// (d->s), keyed by their directed pair and valued by the request index, so
// ONE stable sort by directed key leaves each key's run in record order.
// Each record of the unordered pair {a,b} has exactly one request in the
// (a,b) run, so a request's rank in its run is the record's rank among the
// pair's records (the occurrence); a self-loop's two requests are adjacent
// in its run, ranks 2j and 2j+1 (dynamic.py:231-234).
__global__ void k_del_requests_u(const int32_t* s, const int32_t* d, int64_t k, int sh, uint64_t* rq_key,
                                 int32_t* rq_val) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < k; i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t a = s[i], b = d[i];
        rq_key[2 * i] = pair_key(a, b, sh);
        rq_key[2 * i + 1] = pair_key(b, a, sh);
        rq_val[2 * i] = (int32_t)(2 * i);
        rq_val[2 * i + 1] = (int32_t)(2 * i + 1);
    }
}

__global__ void k_del_requests_u_fill(const uint64_t* rq_key, const int32_t* rq_val, int64_t m, int32_t* rq_occ,
                                      int32_t* rq_rec, uint8_t* rq_which) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t key = rq_key[i];
        int32_t j = 0;  // rank within the run of equal keys (runs are short)
        for (int64_t p = i - 1; p >= 0 && rq_key[p] == key; --p) ++j;
        const int32_t v = rq_val[i];
        rq_occ[i] = j;
        rq_rec[i] = v >> 1;
        rq_which[i] = (uint8_t)(v & 1);
    }
}

// first index of each row run in a (row,col)-sorted key array
__global__ void k_row_starts(const uint64_t* key, int64_t m, int sh, uint8_t* flag) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
        flag[i] = (i == 0 || key_row(key[i], sh) != key_row(key[i - 1], sh)) ? 1 : 0;
}
__global__ void k_row_starts_u32(const uint32_t* key, int64_t m, uint8_t* flag) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
        flag[i] = (i == 0 || key[i] != key[i - 1]) ? 1 : 0;
}

// Rows are scanned in two parts: the first kHead chain slots of every
// requested row by an 8-lane group (k_del_scan_head: one group per row, no
// work-item search), and the rest of long rows in kChunk pieces, one warp
// each (k_del_scan_tail).  chunks[i] = tail work items of row i; the longest
// chain length sizes the chain-offset field of the match sort key.
constexpr int kHead = 256;
constexpr int kScanWarps = 8;
constexpr int kBitmapWords = 1024;  // 32 Kbit per warp (a filter: hits are confirmed by binary search)


__global__ void k_row_chunks(OutView ov, const uint64_t* rq_key, const int32_t* row_first, const int64_t* d_nrows,
                             int64_t cap, int sh, int64_t* chunks, unsigned long long* maxlen,
                             unsigned long long* scanned) {
    unsigned long long mx = 0, sh_head = 0, sh_tail = 0;
    const int64_t nrows = *d_nrows;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < cap; i += (int64_t)gridDim.x * blockDim.x) {
        if (i >= nrows) {  // the tail of the scan input (no separate memset)
            chunks[i] = 0;
            continue;
        }
        int32_t row = key_row(rq_key[row_first[i]], sh);
        int64_t len = 0;
        for (int sg = 0; sg < ov.nseg; ++sg) len += ov.off[sg][row + 1] - ov.off[sg][row];
        chunks[i] = len > kHead ? (len - kHead + kChunk - 1) / kChunk : 0;
        mx = max(mx, (unsigned long long)len);
        sh_head += (unsigned long long)min(len, (int64_t)kHead);
        sh_tail += (unsigned long long)max(len - (int64_t)kHead, (int64_t)0);
    }
    for (int o = 16; o; o >>= 1) {
        mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        sh_head += __shfl_xor_sync(0xffffffffu, sh_head, o);
        sh_tail += __shfl_xor_sync(0xffffffffu, sh_tail, o);
    }
    if ((threadIdx.x & 31) == 0) {
        if (mx) atomicMax(maxlen, mx);
        if (sh_head) atomicAdd(&scanned[0], sh_head);  // chain slots the head / tail kernels read
        if (sh_tail) atomicAdd(&scanned[1], sh_tail);
    }
}

__global__ void k_widen64(const int64_t* a, int64_t m, uint64_t* o) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
        o[i] = (uint64_t)a[i];
}

// A hit on a pair with ONE delete request takes the pair's first live
// occurrence in chain order: atomicMin of the global slot id (gid order is
// chain order).  Pairs with several requests (parallel arcs deleted together)
// go to an overflow list keyed (pair << rb | chain offset) whose single radix
// sort gives the j-th occurrence for the j-th request.
struct MatchOut {
    unsigned long long* sel;  // per request: min gid (pairs with one request)
    const uint8_t* single;    // per request: its key has exactly one request
    uint64_t* okey;           // overflow matches: pair key, chain offset, gid
    int64_t* ochain;
    int64_t* ogid;  // global slot ids: a store may hold more than 2^31 slots
    unsigned long long* ocnt;
    int64_t cap;
};

__device__ inline void emit_matches(const MatchOut& mo, int64_t p, int32_t row, int32_t c, int sh, int64_t chain,
                                    int64_t gid) {
    bool multi = p >= 0 && !mo.single[p];
    if (p >= 0 && !multi) atomicMin(&mo.sel[p], (unsigned long long)gid);
    unsigned mask = __ballot_sync(0xffffffffu, multi);
    if (!mask) return;
    const int lane = threadIdx.x & 31;
    unsigned long long basei = 0;
    if (lane == 0) basei = atomicAdd(mo.ocnt, (unsigned long long)__popc(mask));
    basei = __shfl_sync(0xffffffffu, basei, 0);
    if (multi) {
        int64_t slot = (int64_t)basei + __popc(mask & ((1u << lane) - 1));
        if (slot < mo.cap) {
            mo.okey[slot] = pair_key(row, c, sh);
            mo.ochain[slot] = chain;
            mo.ogid[slot] = gid;
        }
    }
}

// index of the first request for (row, c), or -1
__device__ inline int64_t requested(const uint64_t* rq_key, int64_t lo, int64_t hi, int32_t row, int32_t c, int sh,
                                    int32_t c0, int32_t c1, const uint32_t* bm, uint32_t bmask) {
    if (c < 0) return -1;
    if (hi - lo <= 2) return c == c0 ? lo : (c == c1 ? lo + 1 : -1);
    if (bm) {
        uint32_t h = (uint32_t)c & bmask;
        if (!(bm[h >> 5] & (1u << (h & 31)))) return -1;
    }
    uint64_t want = pair_key(row, c, sh);
    int64_t p = lower_bound_dev<uint64_t>(rq_key, lo, hi, want);
    return (p < hi && rq_key[p] == want) ? p : -1;
}

// head: one 8-lane group per requested row, chain slots [0, kHead)
constexpr int kHeadWords = 32;  // a 1024-bit request filter per group (shared memory)

#ifndef GD_SCAN_MINB
#define GD_SCAN_MINB 4
#endif
__global__ void __launch_bounds__(256, GD_SCAN_MINB) k_del_scan_head(OutView ov, const int32_t* row_first, const int64_t* d_nrows,
                                                       const uint64_t* rq_key, int64_t nrq, int sh, MatchOut mo) {
    constexpr int G = 8, kPer = 32 / G;
    __shared__ uint32_t hbm[256 / G][kHeadWords];
    const int64_t nrows = *d_nrows;
    const int gl = threadIdx.x & (G - 1), gw = (threadIdx.x & 31) / G;
    uint32_t* gbm = hbm[threadIdx.x / G];
    int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t t0 = warp * kPer; t0 < nrows; t0 += nwarps * kPer) {
        int64_t i = t0 + gw;
        bool valid = i < nrows;
        int64_t lo = valid ? row_first[i] : 0;
        int64_t hi = valid ? ((i + 1 < nrows) ? row_first[i + 1] : nrq) : 0;
        int32_t row = valid ? key_row(rq_key[lo], sh) : 0;
        int32_t c0 = valid ? key_col(rq_key[lo], sh) : -2;
        int32_t c1 = (valid && hi - lo > 1) ? key_col(rq_key[lo + 1], sh) : -2;
        // rows with more requests: a 1024-bit filter of the requested columns
        // keeps most slots off the binary search (R-MAT hubs draw dozens of
        // requests, which saturated the 64-bit register filter used before)
        const bool many = valid && hi - lo > 2;
        __syncwarp();  // the group's previous row is done with the filter
        if (many)
            for (int q = gl; q < kHeadWords; q += G) gbm[q] = 0;
        __syncwarp();
        if (many)
            for (int64_t e = lo + gl; e < hi; e += G) {
                uint32_t c = (uint32_t)key_col(rq_key[e], sh) & (kHeadWords * 32 - 1);
                atomicOr(&gbm[c >> 5], 1u << (c & 31));
            }
        __syncwarp();
        const uint32_t* fbm = many ? gbm : nullptr;
        int64_t acc = 0;
        for (int sg = 0; sg < ov.nseg; ++sg) {  // nseg is uniform: the loop stays warp-uniform
            int64_t a = valid ? ov.off[sg][row] : 0;
            int64_t L = valid ? ov.off[sg][row + 1] - a : 0;
            int64_t len = max(min(acc + L, (int64_t)kHead) - acc, (int64_t)0);
            int64_t wlen = len;
            for (int o = G; o < 32; o <<= 1) wlen = max(wlen, (int64_t)__shfl_xor_sync(0xffffffffu, wlen, o));
            const int32_t* col = ov.col[sg];
            for (int64_t x0 = 0; x0 < wlen; x0 += G * kScanILP) {
                int32_t cv[kScanILP];
#pragma unroll
                for (int u = 0; u < kScanILP; ++u) {  // all loads first: kScanILP in flight per lane
                    int64_t x = x0 + u * G + gl;
                    cv[u] = x < len ? col[a + x] : -1;
                }
                int64_t hp[kScanILP];
                bool any = false;
#pragma unroll
                for (int u = 0; u < kScanILP; ++u) {
                    hp[u] = requested(rq_key, lo, hi, row, cv[u], sh, c0, c1, fbm, kHeadWords * 32 - 1);
                    any |= hp[u] >= 0;
                }
                if (__any_sync(0xffffffffu, any)) {  // hits are rare: one vote per ILP batch
#pragma unroll
                    for (int u = 0; u < kScanILP; ++u) {
                        int64_t x = x0 + u * G + gl;
                        emit_matches(mo, hp[u], row, cv[u], sh, acc + x, ov.base[sg] + a + x);
                    }
                }
            }
            acc += L;
        }
    }
}

// work item -> row of the tail pieces (rows write their own ranges)
__global__ void k_chunk_rows(const int64_t* coff, const int64_t* hdr, int32_t* wrow) {
    const int64_t nrows = hdr[0];
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nrows; i += (int64_t)gridDim.x * blockDim.x)
        for (int64_t j = coff[i]; j < coff[i + 1]; ++j) wrow[j] = (int32_t)i;
}

// tail: one warp per kChunk piece of a long row beyond its head; the piece's
// row comes from a table (no search), and a warp that meets the same row
// again keeps its request bitmap.
__global__ void __launch_bounds__(kScanWarps * 32, GD_SCAN_MINB) k_del_scan_tail(OutView ov, const int32_t* row_first,
                                                                   const int64_t* coff, const int32_t* wrow,
                                                                   const int64_t* hdr, const uint64_t* rq_key,
                                                                   int64_t nrq, int sh, MatchOut mo) {
    const int64_t nrows = hdr[0], nwork = hdr[1];
    __shared__ uint32_t bitmap[kScanWarps][kBitmapWords];
    const int lane = threadIdx.x & 31;
    uint32_t* bm = bitmap[threadIdx.x >> 5];
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    int64_t cur = -1;  // row whose bitmap is in bm
    // work items strided over the warps (a contiguous run per warp, which
    // rebuilds a hub row's request filter on fewer warps, measured slower:
    // C2 tail 0.165 -> 0.190 ms)
    for (int64_t wk = warp; wk < nwork; wk += nwarps) {
        const int64_t i = wrow[wk];
        const int64_t chunk = wk - coff[i];
        const int64_t lo = row_first[i];
        const int64_t hi = (i + 1 < nrows) ? row_first[i + 1] : nrq;
        const int32_t row = key_row(rq_key[lo], sh);
        const int64_t ncols = hi - lo;
        const int32_t c0 = key_col(rq_key[lo], sh);
        const int32_t c1 = ncols > 1 ? key_col(rq_key[lo + 1], sh) : -2;
        const bool use_bm = ncols > 2;
        if (use_bm && i != cur) {
            __syncwarp();
            for (int q = lane; q < kBitmapWords; q += 32) bm[q] = 0;
            __syncwarp();
            for (int64_t e = lo + lane; e < hi; e += 32) {
                uint32_t c = (uint32_t)key_col(rq_key[e], sh) & (kBitmapWords * 32 - 1);
                atomicOr(&bm[c >> 5], 1u << (c & 31));
            }
            __syncwarp();
            cur = i;
        }
        int64_t p0 = kHead + chunk * kChunk, p1 = p0 + kChunk;
        int64_t acc = 0;
        for (int sg = 0; sg < ov.nseg && acc < p1; ++sg) {
            const int64_t* off = ov.off[sg];
            const int32_t* col = ov.col[sg];
            int64_t a = off[row], L = off[row + 1] - a;
            int64_t s0 = max(p0, acc), s1 = min(p1, acc + L);
            for (int64_t x0 = s0; x0 < s1; x0 += 32 * kScanILP) {
                int32_t cv[kScanILP];
#pragma unroll
                for (int u = 0; u < kScanILP; ++u) {  // all loads first: kScanILP in flight per lane
                    int64_t x = x0 + u * 32 + lane;
                    cv[u] = x < s1 ? col[a + (x - acc)] : -1;
                }
                int64_t hp[kScanILP];
                bool any = false;
#pragma unroll
                for (int u = 0; u < kScanILP; ++u) {
                    hp[u] = requested(rq_key, lo, hi, row, cv[u], sh, c0, c1, use_bm ? bm : nullptr,
                                      kBitmapWords * 32 - 1);
                    any |= hp[u] >= 0;
                }
                if (__any_sync(0xffffffffu, any)) {
#pragma unroll
                    for (int u = 0; u < kScanILP; ++u) {
                        int64_t x = x0 + u * 32 + lane;
                        emit_matches(mo, hp[u], row, cv[u], sh, x, ov.base[sg] + a + (x - acc));
                    }
                }
            }
            acc += L;
        }
    }
}

__global__ void k_single_flags(const uint64_t* key, int64_t m, uint8_t* single, unsigned long long* sel) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
        single[i] = (i == 0 || key[i - 1] != key[i]) && (i + 1 == m || key[i + 1] != key[i]);
        sel[i] = ~0ULL;  // atomicMin target of the single-request pairs
    }
}

// (pair << rb | chain offset): one radix key for the (pair, chain) order
__global__ void k_overflow_keys(uint64_t* key, const int64_t* chain, int64_t nm, int rb) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nm; i += (int64_t)gridDim.x * blockDim.x)
        key[i] = (key[i] << rb) | (uint64_t)chain[i];
}

// Resolve each request: single-request pairs from the atomicMin slot, the
// others against the (pair, chain)-sorted overflow matches.
__global__ void k_del_resolve(const uint64_t* rq_key, const int32_t* rq_occ, const int32_t* rq_rec,
                              const uint8_t* rq_which, const uint8_t* single, const unsigned long long* sel,
                              int64_t nrq, const uint64_t* m_key, const int64_t* m_gid, int64_t nm, int rb,
                              int64_t* rq_pos, uint8_t* found_fwd, unsigned long long* applied) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nrq; i += (int64_t)gridDim.x * blockDim.x) {
        int64_t pos = -1;
        if (single[i]) {
            if (sel[i] != ~0ULL) pos = (int64_t)sel[i];
        } else {
            uint64_t key = rq_key[i];
            int64_t lo = lower_bound_dev<uint64_t>(m_key, 0, nm, key << rb);
            int64_t occ = rq_occ[i];
            if (lo + occ < nm && (m_key[lo + occ] >> rb) == key) pos = m_gid[lo + occ];
        }
        rq_pos[i] = pos;
        if (rq_which[i] == 0) {
            found_fwd[rq_rec[i]] = pos >= 0 ? 1 : 0;
            if (pos >= 0) atomicAdd(applied, 1ULL);
        }
    }
}

// Tombstone the resolved slots.  A reverse-direction request only applies
// when its record's forward arc was found (dynamic.py:221-229).  Output slot i
// belongs to request i (gid -1 = nothing killed).
__global__ void k_del_kill(OutView ov, const uint64_t* rq_key, const int32_t* rq_rec, const uint8_t* rq_which,
                           const int64_t* rq_pos, int64_t nrq, const uint8_t* found_fwd, int sh, int32_t* k_row,
                           int32_t* k_col, int32_t* k_w, int64_t* k_gid, unsigned long long* k_cnt) {
    unsigned long long killed = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nrq; i += (int64_t)gridDim.x * blockDim.x) {
        int64_t gid = rq_pos[i];
        if (gid >= 0 && rq_which[i] == 1 && !found_fwd[rq_rec[i]]) gid = -1;
        k_gid[i] = gid;
        if (gid < 0) continue;
        int sg = seg_of(ov.base, ov.nseg, gid);
        int64_t slot = gid - ov.base[sg];
        int32_t* col = const_cast<int32_t*>(ov.col[sg]);
        const int32_t* w = ov.w[sg];
        k_row[i] = key_row(rq_key[i], sh);
        k_col[i] = col[slot];
        k_w[i] = w ? w[slot] : 1;
        col[slot] = kSentinel;
        ++killed;
    }
    for (int o = 16; o; o >>= 1) killed += __shfl_xor_sync(0xffffffffu, killed, o);
    if ((threadIdx.x & 31) == 0 && killed) atomicAdd(k_cnt, killed);
}

// ------------------------------------------------------- partitioning ----

// arcs of owned sources (out-store) / owned destinations (in-index)
__global__ void k_part_flags(const uint32_t* src, const int32_t* dst, int64_t m, Blocks b, int rank, uint8_t* fo,
                             uint8_t* fi) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
        fo[i] = b.owner((int64_t)src[i]) == rank;
        fi[i] = b.owner((int64_t)dst[i]) == rank;
    }
}

__global__ void k_owned_flags(const int32_t* s, int64_t k, Blocks b, int rank, uint8_t* f) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < k; i += (int64_t)gridDim.x * blockDim.x)
        f[i] = b.owner((int64_t)s[i]) == rank;
}

__global__ void k_scatter_u8(const uint8_t* in, const int32_t* idx, int64_t m, uint8_t* out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
        out[idx[i]] = in[i];
}

// per-destination-owner counts of the routed arcs (gid < 0: nothing to route)
__global__ void k_route_count(const int32_t* col, const int64_t* gid, int64_t m, Blocks b,
                              unsigned long long* cnt) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
        if (gid && gid[i] < 0) continue;
        const int o = b.owner((int64_t)col[i]);
        const unsigned peers = __match_any_sync(__activemask(), o);  // warp-aggregated per owner
        if ((threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(&cnt[o], (unsigned long long)__popc(peers));
    }
}

// exclusive offsets of the per-owner counts (world entries)
__global__ void k_route_offsets(const unsigned long long* cnt, int world, unsigned long long* cur) {
    unsigned long long a = 0;
    for (int p = 0; p < world; ++p) {
        cur[p] = a;
        a += cnt[p];
    }
}

// packed (row, col, w) triples in owner-major order (order within an owner
// is arbitrary: the in-index is a sorted multiset)
__global__ void k_route_scatter(const int32_t* row, const int32_t* col, const int32_t* w, const int64_t* gid,
                                int64_t m, Blocks b, unsigned long long* cur, int32_t* packed) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
        if (gid && gid[i] < 0) continue;
        const int o = b.owner((int64_t)col[i]);
        const unsigned peers = __match_any_sync(__activemask(), o);
        const int leader = __ffs(peers) - 1, lane = threadIdx.x & 31;
        unsigned long long base = 0;
        if (lane == leader) base = atomicAdd(&cur[o], (unsigned long long)__popc(peers));
        base = __shfl_sync(peers, base, leader);
        const int64_t pos = (int64_t)base + __popc(peers & ((1u << lane) - 1));
        packed[3 * pos] = row[i];
        packed[3 * pos + 1] = col[i];
        packed[3 * pos + 2] = w ? w[i] : 1;
    }
}

__global__ void k_unpack3(const int32_t* packed, int64_t m, int32_t* row, int32_t* col, int32_t* w, int64_t* gid) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
        row[i] = packed[3 * i];
        col[i] = packed[3 * i + 1];
        w[i] = packed[3 * i + 2];
        if (gid) gid[i] = 0;
    }
}

// ---------------------------------------------------------------- adds -----

__global__ void k_add_arcs(const int32_t* s, const int32_t* d, const int32_t* w, int64_t k, bool directed,
                           uint32_t* key, int32_t* val, int32_t* a_row, int32_t* a_col, int32_t* a_w) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < k; i += (int64_t)gridDim.x * blockDim.x) {
        int32_t wi = w ? w[i] : 1;
        if (directed) {
            key[i] = (uint32_t)s[i];
            val[i] = (int32_t)i;
            a_row[i] = s[i];
            a_col[i] = d[i];
            a_w[i] = wi;
        } else {  // dynamic.py:177-183 _expand_arcs: (s,d) then (d,s)
            key[2 * i] = (uint32_t)s[i];
            val[2 * i] = (int32_t)(2 * i);
            a_row[2 * i] = s[i];
            a_col[2 * i] = d[i];
            a_w[2 * i] = wi;
            key[2 * i + 1] = (uint32_t)d[i];
            val[2 * i + 1] = (int32_t)(2 * i + 1);
            a_row[2 * i + 1] = d[i];
            a_col[2 * i + 1] = s[i];
            a_w[2 * i + 1] = wi;
        }
    }
}

// The vacancy scan with a group of 8 lanes per row (4 rows per warp in
// flight): rows of a uniform graph hold ~30 slots, and a warp per row left
// 3/4 of its lanes idle on the loads that bound the kernel.  A row whose
// chain is longer than kVacShort slots (R-MAT hubs) is scanned by the whole
// warp afterwards.  Same result: the first `want` vacancies in slot order.
constexpr int kVacG = 8;
constexpr int64_t kVacShort = 256;

template <int W>
__device__ __forceinline__ void vac_scan(const OutView& ov, int32_t row, int64_t lo, int64_t want, int l, int gb,
                                         unsigned mask, int64_t* vac_gid) {
    const unsigned lanes = W == 32 ? 0xffffffffu : ((1u << W) - 1);
    const unsigned below = (1u << l) - 1;
    int64_t got = 0;
    for (int sg = 0; sg < ov.nseg && got < want; ++sg) {
        const int64_t* off = ov.off[sg];
        const int32_t* col = ov.col[sg];
        const int64_t a = off[row], b = off[row + 1];
        for (int64_t base = a; base < b && got < want; base += W * kScanILP) {
            int32_t cv[kScanILP];
#pragma unroll
            for (int u = 0; u < kScanILP; ++u) {
                const int64_t i = base + u * W + l;
                cv[u] = i < b ? col[i] : 0;
            }
#pragma unroll
            for (int u = 0; u < kScanILP; ++u) {
                const int64_t i = base + u * W + l;
                const bool vac = i < b && cv[u] < 0;
                const unsigned mk = (__ballot_sync(mask, vac) >> gb) & lanes;
                if (vac) {
                    const int64_t t = got + __popc(mk & below);
                    if (t < want) vac_gid[lo + t] = ov.base[sg] + i;
                }
                got += __popc(mk);
            }
        }
    }
}

template <int G>
__global__ void k_add_vacancies_g(OutView ov, const uint32_t* skey, const int32_t* row_first,
                                  const int64_t* d_nrows, int64_t narcs, int64_t* vac_gid) {
    constexpr int kPer = 32 / G;
    const int lane = threadIdx.x & 31, gl = lane & (G - 1), gb = lane & ~(G - 1);
    const unsigned gmask = G == 32 ? 0xffffffffu : ((1u << G) - 1) << gb;
    const int64_t nrows = *d_nrows;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t r0 = warp * kPer; r0 < nrows; r0 += nwarps * kPer) {  // warp-uniform trip count
        const int64_t r = r0 + lane / G;
        const bool valid = r < nrows;
        int64_t lo = 0, want = 0, chain = 0;
        int32_t row = 0;
        if (valid) {
            lo = row_first[r];
            want = ((r + 1 < nrows) ? row_first[r + 1] : narcs) - lo;
            row = (int32_t)skey[lo];
            for (int sg = 0; sg < ov.nseg; ++sg) chain += ov.off[sg][row + 1] - ov.off[sg][row];
        }
        const bool lng = G < 32 && valid && chain > kVacShort;
        if (valid && !lng) vac_scan<G>(ov, row, lo, want, gl, gb, gmask, vac_gid);
        for (unsigned hm = __ballot_sync(0xffffffffu, lng && gl == 0); hm; hm &= hm - 1) {
            const int src = __ffs(hm) - 1;
            const int64_t hlo = __shfl_sync(0xffffffffu, lo, src), hwant = __shfl_sync(0xffffffffu, want, src);
            const int32_t hrow = __shfl_sync(0xffffffffu, row, src);
            vac_scan<32>(ov, hrow, hlo, hwant, lane, 0, 0xffffffffu, vac_gid);
        }
    }
}

// clog (nullable): the claimed global slot of each arc by stream position,
// -1 for a spill (the order nodes_to appends claims in, dynamic.py:272-274)
__global__ void k_add_claim(OutView ov, const int32_t* sval, const int32_t* a_col, const int32_t* a_w,
                            const int64_t* vac_gid, int64_t narcs, uint8_t* leftover, int64_t* clog) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < narcs; i += (int64_t)gridDim.x * blockDim.x) {
        int64_t gid = vac_gid[i];
        int32_t a = sval[i];
        if (clog) clog[a] = gid;
        if (gid < 0) {
            leftover[i] = 1;
            continue;
        }
        leftover[i] = 0;
        int sg = seg_of(ov.base, ov.nseg, gid);
        int64_t slot = gid - ov.base[sg];
        const_cast<int32_t*>(ov.col[sg])[slot] = a_col[a];
        if (ov.w[sg]) const_cast<int32_t*>(ov.w[sg])[slot] = a_w[a];
    }
}

__global__ void k_gather_arcs(const int32_t* sel, int64_t m, const int32_t* sval, const int32_t* a_row,
                              const int32_t* a_col, const int32_t* a_w, int32_t* o_row, int32_t* o_col,
                              int32_t* o_w) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
        int32_t a = sval[sel ? sel[i] : i];
        if (o_row) o_row[i] = a_row[a];
        o_col[i] = a_col[a];
        if (o_w) o_w[i] = a_w[a];
    }
}


// ----------------------------------------------------- index maintenance ----

// Each killed arc tombstones one live index entry with the same column and
// weight, claimed by CAS so parallel arcs take distinct entries.  Log slot i
// belongs to killed arc i (-1 when there was none).
__global__ void k_index_claim(const int32_t* k_row, const int32_t* k_col, const int32_t* k_w, const int64_t* k_gid,
                              int64_t m, bool rows_are_dst, const int64_t* off, int32_t* col, const int32_t* w,
                              int64_t* t_pos, int32_t* t_row) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
        t_pos[i] = -1;
        if (k_gid[i] < 0) continue;
        int32_t r = rows_are_dst ? k_col[i] : k_row[i];
        int32_t c = rows_are_dst ? k_row[i] : k_col[i];
        int32_t wt = k_w[i];
        int64_t lo = col_lower(col, off[r], off[r + 1], c);
        int64_t hi = col_upper(col, lo, off[r + 1], c);
        for (int64_t e = lo; e < hi; ++e) {
            if (col[e] != c) continue;  // tombstoned (~c)
            if (w && w[e] != wt) continue;
            if (atomicCAS(&col[e], c, tomb(c)) == c) {
                t_pos[i] = e;
                t_row[i] = r;
                break;
            }
        }
    }
}

__global__ void k_added_to_index(const int32_t* a_row, const int32_t* a_col, int64_t m, bool rows_are_dst, int sh,
                                  uint64_t* key, int32_t* val) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
        int32_t r = rows_are_dst ? a_col[i] : a_row[i];
        int32_t c = rows_are_dst ? a_row[i] : a_col[i];
        key[i] = pair_key(r, c, sh);
        val[i] = (int32_t)i;
    }
}

// the in-index delta from the source-sorted arcs: keys = destinations, values = arc indices
__global__ void k_dst_by_src(const int32_t* by_row, const int32_t* a_col, int64_t m, uint32_t* key, int32_t* val) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < m; t += (int64_t)gridDim.x * blockDim.x) {
        const int32_t i = by_row[t];
        key[t] = (uint32_t)a_col[i];
        val[t] = i;
    }
}

__global__ void k_rev_delta_split(const uint32_t* key, const int32_t* val, int64_t m, const int32_t* a_row,
                                  const int32_t* a_w, int32_t* drow, int32_t* dcol, int32_t* dw) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < m; t += (int64_t)gridDim.x * blockDim.x) {
        const int32_t i = val[t];
        drow[t] = (int32_t)key[t];
        dcol[t] = a_row[i];
        if (dw) dw[t] = a_w[i];
    }
}

// insertion point of delta entry (row, col) in the base: after equal columns
__global__ void k_index_ins_pos(const int32_t* drow, const int32_t* dcol, int64_t m, const int64_t* off,
                                const int32_t* col, int64_t* ipos) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
        int32_t r = drow[i];
        ipos[i] = col_upper(col, off[r], off[r + 1], dcol[i]);
    }
}

// out-store merge: delta arcs go after the base slots of their row
__global__ void k_out_ins_pos(const int32_t* irow, int64_t m, const int64_t* off0, int64_t* ipos) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
        ipos[i] = off0[irow[i] + 1];
}

// row of every slot of a segment + live flag
__global__ void k_delta_rows(const int64_t* off, int64_t n, const int32_t* col, int64_t nslots, int32_t* row,
                             uint8_t* live) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nslots;
         i += (int64_t)gridDim.x * blockDim.x) {
        row[i] = (int32_t)(upper_bound_dev<int64_t>(off, 0, n + 1, i) - 1);
        live[i] = col[i] >= 0 ? 1 : 0;
    }
}

// --------------------------------------------------------- edit merge -----

constexpr int kEditThreads = 256;
constexpr int kWin = 256;                                 // entries per warp window
constexpr int kTile = kWin * (kEditThreads / 32);         // 2048 entries per CTA tile

// Dead entries per 256-entry window and per row, from an UNORDERED tomb log.  With
// dedupe (the out-store), a slot logged twice (deleted, claimed, deleted
// again between merges) counts once: the first visit flips -1 to -2.
__global__ void k_tomb_hist(const int64_t* tpos, const int32_t* trow, int64_t ntomb, int32_t* col, int64_t nnz,
                            bool dedupe, unsigned long long* tile_dead, int64_t* row_shift) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < ntomb; i += (int64_t)gridDim.x * blockDim.x) {
        int64_t p = tpos[i];
        if (p < 0 || p >= nnz) continue;
        bool dead = dedupe ? atomicCAS(&col[p], kSentinel, kSentinel - 1) == kSentinel : col[p] < 0;
        if (!dead) continue;
        atomicAdd(&tile_dead[p / kWin], 1ULL);
        atomicAdd(reinterpret_cast<unsigned long long*>(&row_shift[trow[i]]), (unsigned long long)(-1LL));
    }
}

__global__ void k_ins_hist(const int32_t* irow, int64_t nins, int64_t* row_shift) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nins; i += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(reinterpret_cast<unsigned long long*>(&row_shift[irow[i]]), 1ULL);
}

__global__ void k_add_offsets(const int64_t* off, const int64_t* shift, int64_t n1, int64_t* out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n1; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = off[i] + shift[i];
}

// inserts with P < tile start, per tile (insertion points are sorted)
__global__ void k_win_ins(int64_t nwin, const int64_t* ipos, int64_t nins, int64_t* pj) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t <= nwin; t += (int64_t)gridDim.x * blockDim.x)
        pj[t] = lower_bound_dev<int64_t>(ipos, 0, nins, t * kWin);
}

// newpos(i) = i - #dead(< i) + #inserts(P <= i).  One warp per 256-entry
// window, lane-strided (every load / store instruction covers 32 consecutive
// entries).  Dead entries are exactly the negative ones, so #dead is the
// window's base (scan of the per-window tomb histogram) plus a ballot/popc
// prefix; warps never wait on each other.  The window's insertion range
// comes from a per-window table, so the entries, the dead base and the range
// are loaded together and only the insertion positions depend on them.  All
// per-entry arithmetic is 32-bit and relative to the window: the 64-bit
// output base ws - dead + ins is formed once per window.
template <bool FULL, bool WEIGHTED>
__device__ __forceinline__ void edit_load(const int32_t* __restrict__ col, const int32_t* __restrict__ w, int64_t nnz,
                                          int64_t win, int32_t (&v)[kWin / 32], int32_t (&wv)[kWin / 32]) {
    constexpr int Q = kWin / 32;
    const int lane = threadIdx.x & 31;
    const int64_t ws = win * kWin;
    const int lim = FULL ? kWin : (int)(nnz - ws);
    const int32_t* cb = col + ws;
#pragma unroll
    for (int q = 0; q < Q; ++q) {
        const int o = q * 32 + lane;
        const bool in = FULL || o < lim;
        v[q] = in ? __ldcs(&cb[o]) : -1;
        if (WEIGHTED) wv[q] = in ? __ldcs(&w[ws + o]) : 0;
    }
}

// A window's metadata: its dead base and insertion range, and (lanes <
// min(32, inserts)) its first 32 insertions -- loaded ahead of the window so
// the dependent loads stay off the copy's critical path.
struct WinMeta {
    int64_t dead0, pjw, pje;
    int my_ins;  // insertion position relative to the window start (INT_MAX: none)
    int32_t my_icol, my_iw;
};
__device__ __forceinline__ void win_meta_head(WinMeta& m, int64_t win, const int64_t* __restrict__ dead_win,
                                              const int64_t* __restrict__ pj_win) {
    m.dead0 = dead_win[win];
    m.pjw = pj_win[win];
    m.pje = pj_win[win + 1];
}
template <bool WEIGHTED>
__device__ __forceinline__ void win_meta_ins(WinMeta& m, int64_t win, const int64_t* __restrict__ ipos,
                                             const int32_t* __restrict__ icol, const int32_t* __restrict__ iw) {
    const int lane = threadIdx.x & 31;
    m.my_ins = INT_MAX;
    m.my_icol = 0;
    m.my_iw = 1;
    if (lane < m.pje - m.pjw) {
        m.my_ins = (int)(ipos[m.pjw + lane] - win * kWin);
        m.my_icol = icol[m.pjw + lane];
        if (WEIGHTED && iw) m.my_iw = iw[m.pjw + lane];
    }
}

template <bool WEIGHTED>
__device__ __forceinline__ void edit_store_p(int64_t win, const int32_t (&v)[kWin / 32],
                                             const int32_t (&wv)[kWin / 32], const WinMeta& mt,
                                             const int64_t* __restrict__ ipos, const int32_t* __restrict__ icol,
                                             const int32_t* __restrict__ iw, int32_t* __restrict__ ocol,
                                             int32_t* __restrict__ ow);

template <bool WEIGHTED>
__device__ __forceinline__ void edit_store_m(int64_t win, const int32_t (&v)[kWin / 32],
                                             const int32_t (&wv)[kWin / 32], int64_t dead0, int64_t pjw,
                                             int64_t pje, const int64_t* __restrict__ ipos,
                                             const int32_t* __restrict__ icol, const int32_t* __restrict__ iw,
                                             int32_t* __restrict__ ocol, int32_t* __restrict__ ow) {
    WinMeta mt;
    mt.dead0 = dead0;
    mt.pjw = pjw;
    mt.pje = pje;
    win_meta_ins<WEIGHTED>(mt, win, ipos, icol, iw);
    edit_store_p<WEIGHTED>(win, v, wv, mt, ipos, icol, iw, ocol, ow);
}

template <bool WEIGHTED>
__device__ __forceinline__ void edit_store_p(int64_t win, const int32_t (&v)[kWin / 32],
                                             const int32_t (&wv)[kWin / 32], const WinMeta& mt,
                                             const int64_t* __restrict__ ipos, const int32_t* __restrict__ icol,
                                             const int32_t* __restrict__ iw, int32_t* __restrict__ ocol,
                                             int32_t* __restrict__ ow) {
    constexpr int Q = kWin / 32;
    const int lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1;
    const int64_t ws = win * kWin;
    const int64_t dead0 = mt.dead0, pjw = mt.pjw, pje = mt.pje;
    const int nins = (int)(pje - pjw);
    unsigned m[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) m[q] = __ballot_sync(0xffffffffu, v[q] < 0);  // out-of-range entries read as -1
    const int64_t obase = ws - dead0 + pjw;  // newpos of window entry 0, before local shifts
    int32_t* oc = ocol + obase;
    int32_t* owb = WEIGHTED ? ow + obase : nullptr;
    if (nins == 0) {  // the common window: only the dead shift
        int dead = 0;
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            const int np = q * 32 + lane - (dead + __popc(m[q] & lt));
            if (v[q] >= 0) {
                __stcs(&oc[np], v[q]);
                if (WEIGHTED) __stcs(&owb[np], wv[q]);
            }
            dead += __popc(m[q]);
        }
        return;
    }
    const int my_ins = mt.my_ins;
    const int32_t my_icol = mt.my_icol, my_iw = mt.my_iw;
    int dead = 0;
#pragma unroll
    for (int q = 0; q < Q; ++q) {
        const int o = q * 32 + lane;
        int ins = 0;
        if (nins > 32) {
            ins = (int)(upper_bound_dev<int64_t>(ipos, pjw, pje, ws + o) - pjw);
        } else {
            for (int k = 0; k < nins; ++k) ins += __shfl_sync(0xffffffffu, my_ins, k) <= o;
        }
        if (v[q] >= 0) {
            const int np = o - (dead + __popc(m[q] & lt)) + ins;
            __stcs(&oc[np], v[q]);
            if (WEIGHTED) __stcs(&owb[np], wv[q]);
        }
        dead += __popc(m[q]);
    }
    for (int j = lane; j < nins; j += 32) {  // this window's inserted entries
        const int P = j < 32 ? my_ins : (int)(ipos[pjw + j] - ws);
        const int32_t ic = j < 32 ? my_icol : icol[pjw + j];
        const int32_t iwv = j < 32 ? my_iw : (iw ? iw[pjw + j] : 1);
        const int qq = P >> 5, r = P & 31;
        int d = 0;
#pragma unroll
        for (int q = 0; q < Q; ++q) d += q < qq ? __popc(m[q]) : (q == qq ? __popc(m[q] & ((1u << r) - 1)) : 0);
        const int np = P - d + j;
        oc[np] = ic;
        if (WEIGHTED) owb[np] = iwv;
    }
}

template <bool WEIGHTED>
__device__ __forceinline__ void edit_store(int64_t win, const int32_t (&v)[kWin / 32], const int32_t (&wv)[kWin / 32],
                                           const int64_t* __restrict__ dead_win, const int64_t* __restrict__ ipos,
                                           const int64_t* __restrict__ pj_win, const int32_t* __restrict__ icol,
                                           const int32_t* __restrict__ iw, int32_t* __restrict__ ocol,
                                           int32_t* __restrict__ ow) {
    edit_store_m<WEIGHTED>(win, v, wv, dead_win[win], pj_win[win], pj_win[win + 1], ipos, icol, iw, ocol, ow);
}

// ---- the bulk-copy (TMA) merge copy ----------------------------------------
// The register path above keeps one window's loads in flight per warp and
// stalls on them (ncu: 28% of samples on the first use of the loaded
// entries, 48% of DRAM bandwidth).  Here the entries stream into shared
// memory by cp.async.bulk: one thread per CTA keeps kBulkStages chunks of
// kTile entries (one window per warp) in flight on mbarriers, so the loads
// are no longer bounded by registers or warps, and the warps run the same
// compaction from shared memory.
constexpr int kBulkStages = 4;

__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_init_fence() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "GD_MBAR_WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra GD_MBAR_WAIT_%=;\n"
        "}\n" ::"r"(smem_addr(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(smem_addr(bar))
        : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

template <bool WEIGHTED>
__global__ void __launch_bounds__(kEditThreads) k_edit_bulk(const int32_t* __restrict__ col,
                                                            const int32_t* __restrict__ w, int64_t nnz,
                                                            const int64_t* __restrict__ dead_win,
                                                            const int64_t* __restrict__ ipos,
                                                            const int64_t* __restrict__ pj_win,
                                                            const int32_t* __restrict__ icol,
                                                            const int32_t* __restrict__ iw, int64_t nwin,
                                                            int32_t* __restrict__ ocol, int32_t* __restrict__ ow) {
    constexpr int Q = kWin / 32;
    constexpr int kWarps = kEditThreads / 32;
    constexpr uint32_t kWinBytes = kWin * 4;
    // per warp: kBulkStages windows of cols (then of weights), one mbarrier each
    extern __shared__ __align__(128) int32_t ebuf[];
    __shared__ __align__(8) uint64_t bar[kWarps][kBulkStages];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    int32_t* wbuf = ebuf + warp * kBulkStages * kWin * (WEIGHTED ? 2 : 1);
    uint64_t* wbar = bar[warp];
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nfull = nnz / kWin;
    auto issue = [&](int st, int64_t win) {
        mbar_expect_tx(&wbar[st], WEIGHTED ? 2 * kWinBytes : kWinBytes);
        bulk_g2s(wbuf + st * kWin, col + win * kWin, kWinBytes, &wbar[st]);
        if (WEIGHTED) bulk_g2s(wbuf + (kBulkStages + st) * kWin, w + win * kWin, kWinBytes, &wbar[st]);
    };
    if (lane == 0) {
        for (int st = 0; st < kBulkStages; ++st) mbar_init(&wbar[st], 1);
        mbar_init_fence();
        for (int st = 0; st < kBulkStages; ++st) {
            const int64_t win = gw + (int64_t)st * nwarps;
            if (win < nfull) issue(st, win);
        }
    }
    __syncwarp();
    // metadata pipeline: window i's insertions and window i+1's ranges are
    // loaded while window i-1 is written
    WinMeta m0, m1;
    if (gw < nfull) {
        win_meta_head(m0, gw, dead_win, pj_win);
        win_meta_ins<WEIGHTED>(m0, gw, ipos, icol, iw);
    }
    if (gw + nwarps < nfull) win_meta_head(m1, gw + nwarps, dead_win, pj_win);
    int it = 0;
    for (int64_t win = gw; win < nfull; win += nwarps, ++it) {
        const int st = it % kBulkStages;
        WinMeta m2;
        const int64_t w1 = win + nwarps, w2 = win + 2 * nwarps;
        if (w2 < nfull) win_meta_head(m2, w2, dead_win, pj_win);
        if (w1 < nfull) win_meta_ins<WEIGHTED>(m1, w1, ipos, icol, iw);
        mbar_wait(&wbar[st], (uint32_t)(it / kBulkStages) & 1u);
        int32_t v[Q], wv[Q];
        const int32_t* sc = wbuf + st * kWin;
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            v[q] = sc[q * 32 + lane];
            if (WEIGHTED) wv[q] = sc[kBulkStages * kWin + q * 32 + lane];
        }
        __syncwarp();  // the whole window is in registers: the stage may refill
        if (lane == 0) {
            const int64_t wn = win + (int64_t)kBulkStages * nwarps;
            if (wn < nfull) {
                fence_proxy_async_smem();
                issue(st, wn);
            }
        }
        edit_store_p<WEIGHTED>(win, v, wv, m0, ipos, icol, iw, ocol, ow);
        m0 = m1;
        m1 = m2;
    }
    // the partial last window: the register path
    for (int64_t win = nfull + gw; win < nwin; win += nwarps) {
        int32_t v[Q], wv[Q];
        edit_load<false, WEIGHTED>(col, w, nnz, win, v, wv);
        edit_store<WEIGHTED>(win, v, wv, dead_win, ipos, pj_win, icol, iw, ocol, ow);
    }
}

// The vector path of a full window with at most 32 insertions (almost every
// window of a batch-sized edit): two 16-byte loads per lane, the survivors
// and the window's insertions compacted into shared memory in output order,
// then the window's output range written with 16-byte stores (scalar head
// and tail to reach the 16-byte grid).  Same result as edit_store.  Off by
// default (GD_EDIT_VEC): A/B on B200, C2 merge 0.258 -> 0.292 ms, C3 2.15 ->
// 2.10 ms per batch -- the copy is bound neither by load instructions nor by
// loads in flight (GD_EDIT_AHEAD 2/3 were slower too), see
// profiles/round2/README.md.
template <bool WEIGHTED>
__device__ __forceinline__ void edit_window_vec(const int32_t* __restrict__ col, const int32_t* __restrict__ w,
                                                int64_t win, const int64_t* __restrict__ dead_win,
                                                const int64_t* __restrict__ ipos, const int64_t* __restrict__ pj_win,
                                                const int32_t* __restrict__ icol, const int32_t* __restrict__ iw,
                                                int32_t* __restrict__ ocol, int32_t* __restrict__ ow, int32_t* sc,
                                                int32_t* sw) {
    const int lane = threadIdx.x & 31;
    const int64_t ws = win * kWin;
    const int4* c4 = reinterpret_cast<const int4*>(col + ws);
    const int4 a = __ldcs(c4 + lane), b = __ldcs(c4 + 32 + lane);
    int4 wa, wb;
    if (WEIGHTED) {
        const int4* w4 = reinterpret_cast<const int4*>(w + ws);
        wa = __ldcs(w4 + lane);
        wb = __ldcs(w4 + 32 + lane);
    }
    const int64_t dead0 = dead_win[win];
    const int64_t pjw = pj_win[win];
    const int nins = (int)(pj_win[win + 1] - pjw);
    int my_ins = INT_MAX;
    int32_t my_icol = 0, my_iw = 1;
    if (lane < nins) {
        my_ins = (int)(ipos[pjw + lane] - ws);
        my_icol = icol[pjw + lane];
        if (WEIGHTED && iw) my_iw = iw[pjw + lane];
    }
    const int32_t e[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
    int32_t f[8];
    if (WEIGHTED) {
        f[0] = wa.x, f[1] = wa.y, f[2] = wa.z, f[3] = wa.w, f[4] = wb.x, f[5] = wb.y, f[6] = wb.z, f[7] = wb.w;
    }
    // survivors per lane in each half, then warp-exclusive prefixes
    unsigned al0 = 0, al1 = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        al0 |= (unsigned)(e[j] >= 0) << j;
        al1 |= (unsigned)(e[4 + j] >= 0) << j;
    }
    const int s0 = __popc(al0), s1 = __popc(al1);
    int p0 = s0, p1 = s1;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int x0 = __shfl_up_sync(0xffffffffu, p0, o), x1 = __shfl_up_sync(0xffffffffu, p1, o);
        if (lane >= o) {
            p0 += x0;
            p1 += x1;
        }
    }
    const int tot0 = __shfl_sync(0xffffffffu, p0, 31), tot = tot0 + __shfl_sync(0xffffffffu, p1, 31);
    p0 -= s0;         // survivors before my first half
    p1 += tot0 - s1;  // ... before my second half
    // each survivor goes after the survivors and insertions before it
    // (insertion positions are sorted, at most 32 per window)
    {
        int r0 = p0, r1 = p1;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const int o = (q < 4 ? 0 : 128) + 4 * lane + (q & 3);
            int ins = 0;
            for (int k = 0; k < nins; ++k) ins += __shfl_sync(0xffffffffu, my_ins, k) <= o;
            if (e[q] >= 0) {
                const int r = q < 4 ? r0++ : r1++;
                sc[r + ins] = e[q];
                if (WEIGHTED) sw[r + ins] = f[q];
            }
        }
    }
    // an insertion lands after the survivors before its position, and after
    // the insertions before it
    {
        const int P = lane < nins ? my_ins : 0;
        const int ll = (P & 127) >> 2, jj = P & 3;
        const int pp0 = __shfl_sync(0xffffffffu, p0, ll), pp1 = __shfl_sync(0xffffffffu, p1, ll);
        const unsigned m0 = __shfl_sync(0xffffffffu, al0, ll), m1 = __shfl_sync(0xffffffffu, al1, ll);
        if (lane < nins) {
            const int before = (P >= 128 ? pp1 : pp0) + __popc((P >= 128 ? m1 : m0) & ((1u << jj) - 1));
            sc[before + lane] = my_icol;
            if (WEIGHTED) sw[before + lane] = my_iw;
        }
    }
    __syncwarp();
    const int64_t obase = ws - dead0 + pjw;
    const int cnt = tot + nins;
    // 16-byte stores on the output's 16-byte grid
    const int head = (int)((4 - (obase & 3)) & 3) < cnt ? (int)((4 - (obase & 3)) & 3) : cnt;
    if (lane < head) {
        __stcs(&ocol[obase + lane], sc[lane]);
        if (WEIGHTED) __stcs(&ow[obase + lane], sw[lane]);
    }
    const int nv = (cnt - head) >> 2;
    int4* o4 = reinterpret_cast<int4*>(ocol + obase + head);
    int4* ow4 = WEIGHTED ? reinterpret_cast<int4*>(ow + obase + head) : nullptr;
    for (int t = lane; t < nv; t += 32) {
        const int b0 = head + 4 * t;
        __stcs(o4 + t, make_int4(sc[b0], sc[b0 + 1], sc[b0 + 2], sc[b0 + 3]));
        if (WEIGHTED) __stcs(ow4 + t, make_int4(sw[b0], sw[b0 + 1], sw[b0 + 2], sw[b0 + 3]));
    }
    const int tail0 = head + 4 * nv;
    if (lane < cnt - tail0) {
        __stcs(&ocol[obase + tail0 + lane], sc[tail0 + lane]);
        if (WEIGHTED) __stcs(&ow[obase + tail0 + lane], sw[tail0 + lane]);
    }
    __syncwarp();
}

// Each warp keeps the loads of GD_EDIT_AHEAD windows in flight: they are all
// issued before the first window's shifted stores, which doubles the bytes
// a warp has outstanding (the copy is bound by memory-level parallelism).
#ifndef GD_EDIT_AHEAD
#define GD_EDIT_AHEAD 1
#endif
#ifndef GD_EDIT_VEC
#define GD_EDIT_VEC 0
#endif
#ifndef GD_EDIT_META
#define GD_EDIT_META 0
#endif
#ifndef GD_EDIT_MINB_U
#define GD_EDIT_MINB_U 5
#endif
#ifndef GD_EDIT_MINB_W
#define GD_EDIT_MINB_W 4
#endif
template <bool WEIGHTED>
__global__ void __launch_bounds__(kEditThreads, WEIGHTED ? GD_EDIT_MINB_W : GD_EDIT_MINB_U)
    k_edit_base(const int32_t* __restrict__ col, const int32_t* __restrict__ w, int64_t nnz,
                const int64_t* __restrict__ dead_win, const int64_t* __restrict__ ipos,
                const int64_t* __restrict__ pj_win, const int32_t* __restrict__ icol, const int32_t* __restrict__ iw,
                int64_t nwin, int32_t* __restrict__ ocol, int32_t* __restrict__ ow) {
    constexpr int A = GD_EDIT_AHEAD;
    constexpr int Q = kWin / 32;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int64_t nfull = nnz / kWin;
    const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    // full windows, A adjacent ones per warp step: A*g .. A*g + A-1 for group g
    const int64_t ngrp = nfull / A;
#if GD_EDIT_VEC
    if (A == 1) {
        __shared__ __align__(16) int32_t stc[kEditThreads / 32][kWin + 32];
        __shared__ __align__(16) int32_t stw[WEIGHTED ? kEditThreads / 32 : 1][kWin + 32];
        int32_t* sc = stc[threadIdx.x >> 5];
        int32_t* sw = WEIGHTED ? stw[threadIdx.x >> 5] : nullptr;
        for (int64_t win = w0; win < nfull; win += nwarps) {
            if (pj_win[win + 1] - pj_win[win] <= 32) {
                edit_window_vec<WEIGHTED>(col, w, win, dead_win, ipos, pj_win, icol, iw, ocol, ow, sc, sw);
            } else {
                int32_t v[Q], wv[Q];
                edit_load<true, WEIGHTED>(col, w, nnz, win, v, wv);
                edit_store<WEIGHTED>(win, v, wv, dead_win, ipos, pj_win, icol, iw, ocol, ow);
            }
        }
        for (int64_t win = nfull + w0; win < nwin; win += nwarps) {
            int32_t v[Q], wv[Q];
            edit_load<false, WEIGHTED>(col, w, nnz, win, v, wv);
            edit_store<WEIGHTED>(win, v, wv, dead_win, ipos, pj_win, icol, iw, ocol, ow);
        }
        return;
    }
#endif
#if GD_EDIT_META
    if constexpr (A == 1) {
        // metadata pipeline: the next window's ranges and insertions load
        // while this window's entries are in flight.  Off by default: A/B on
        // B200, C2 merge 0.263 -> 0.304 ms, C3 2.18 -> 2.35 ms per batch
        WinMeta m0, m1;
        if (w0 < nfull) {
            win_meta_head(m0, w0, dead_win, pj_win);
            win_meta_ins<WEIGHTED>(m0, w0, ipos, icol, iw);
        }
        for (int64_t win = w0; win < nfull; win += nwarps) {
            int32_t v[Q], wv[Q];
            edit_load<true, WEIGHTED>(col, w, nnz, win, v, wv);
            const int64_t w1 = win + nwarps;
            if (w1 < nfull) {
                win_meta_head(m1, w1, dead_win, pj_win);
                win_meta_ins<WEIGHTED>(m1, w1, ipos, icol, iw);
            }
            edit_store_p<WEIGHTED>(win, v, wv, m0, ipos, icol, iw, ocol, ow);
            m0 = m1;
        }
        for (int64_t win = nfull + w0; win < nwin; win += nwarps) {
            int32_t v[Q], wv[Q];
            edit_load<false, WEIGHTED>(col, w, nnz, win, v, wv);
            edit_store<WEIGHTED>(win, v, wv, dead_win, ipos, pj_win, icol, iw, ocol, ow);
        }
    } else
#endif
    {
    for (int64_t g = w0; g < ngrp; g += nwarps) {
        int32_t v[A][Q], wv[A][Q];
#pragma unroll
        for (int a = 0; a < A; ++a) edit_load<true, WEIGHTED>(col, w, nnz, g * A + a, v[a], wv[a]);
#pragma unroll
        for (int a = 0; a < A; ++a)
            edit_store<WEIGHTED>(g * A + a, v[a], wv[a], dead_win, ipos, pj_win, icol, iw, ocol, ow);
    }
    for (int64_t win = ngrp * A + w0; win < nwin; win += nwarps) {  // the rest one at a time (the last may be partial)
        int32_t v[Q], wv[Q];
        if (win < nfull) edit_load<true, WEIGHTED>(col, w, nnz, win, v, wv);
        else edit_load<false, WEIGHTED>(col, w, nnz, win, v, wv);
        edit_store<WEIGHTED>(win, v, wv, dead_win, ipos, pj_win, icol, iw, ocol, ow);
    }
    }
}

// insertions at the very end of the base (P == nnz)
__global__ void k_edit_tail(const int64_t* ipos, int64_t nins, int64_t nnz, const int64_t* dead_total,
                            const int32_t* icol, const int32_t* iw, int32_t* ocol, int32_t* ow) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < nins; j += (int64_t)gridDim.x * blockDim.x) {
        if (ipos[j] < nnz) continue;
        int64_t np = nnz - *dead_total + j;
        ocol[np] = icol[j];
        if (ow) ow[np] = iw ? iw[j] : 1;
    }
}

__global__ void k_export_seg(const int32_t* col, const int32_t* w, int64_t m, int64_t* ocol, int64_t* ow) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
        int32_t c = col[i];
        ocol[i] = c < 0 ? INT64_MAX : (int64_t)c;
        ow[i] = w ? (int64_t)w[i] : 1;
    }
}


template <typename T>
__global__ void k_gather_sel(const T* in, const int32_t* sel, int64_t m, T* out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = in[sel[i]];
}

}  // namespace

// ==========================================================================

// Two-phase edit merge: plan() builds the per-row shifts and per-window
// death counts (device only), apply() sizes and writes the merged arrays once
// the host knows the death total.  Store::merge plans the out-store and the
// in-index first and reads both totals with ONE read-back.
void edit_plan(cudaStream_t s, EditJob& j) {
    j.nwin = (j.nnz + kWin - 1) / kWin;
    j.counts.alloc(j.n + 1 + j.nwin + 1, s);  // per-row shifts, then per-window deaths: one memset
    j.counts.zero(s);
    int64_t* shift_cnt = j.counts.get();
    int64_t* dead_cnt = j.counts.get() + j.n + 1;
    if (j.ntomb)
        GD_KERNEL(k_tomb_hist, grid_for(j.ntomb, 256), 256, 0, s, j.tpos, j.trow, j.ntomb, j.col, j.nnz, j.dedupe,
                  reinterpret_cast<unsigned long long*>(dead_cnt), shift_cnt);
    if (j.nins) GD_KERNEL(k_ins_hist, grid_for(j.nins, 256), 256, 0, s, j.irow, j.nins, shift_cnt);
    j.shift.alloc(j.n + 1, s);
    j.dead_win.alloc(j.nwin + 1, s);
    exclusive_scan_i64(s, shift_cnt, j.shift.get(), j.n + 1);
    exclusive_scan_i64(s, dead_cnt, j.dead_win.get(), j.nwin + 1);
}

void edit_apply(cudaStream_t s, EditJob& j, int64_t dead_total, DBuf<int64_t>& new_off, DBuf<int32_t>& new_col,
                DBuf<int32_t>& new_w, int64_t& new_nnz) {
    const int64_t n = j.n, nnz = j.nnz, nwin = j.nwin, nins = j.nins;
    const int64_t ntiles = (nnz + kTile - 1) / kTile;
    new_nnz = nnz - dead_total + nins;
    new_off.alloc(n + 1, s);
    GD_KERNEL(k_add_offsets, grid_for(n + 1, 256), 256, 0, s, j.off, j.shift.get(), n + 1, new_off.get());
    new_col.alloc(new_nnz, s);
    if (j.weighted) new_w.alloc(new_nnz, s);
    else new_w.release();
    if (ntiles) {
        DBuf<int64_t> pj(nwin + 1, s);
        GD_KERNEL(k_win_ins, grid_for(nwin + 1, 256), 256, 0, s, nwin, j.ipos, nins, pj.get());
        unsigned g = (unsigned)std::min<int64_t>(ntiles, 148LL * 64);
        // algorithmic bytes: every base entry read once, every surviving entry written once
        // the bulk-copy (TMA) variant is opt-in: A/B on B200 it ran 0.142 vs 0.129 ms per C2 launch and
        // 1.24 vs 1.08 ms per C3 launch (profiles/round2/README.md)
        static const int bulk_env = getenv("GD_EDIT_BULK") ? atoi(getenv("GD_EDIT_BULK")) : 0;
        const bool aligned = ((uintptr_t)j.col & 15) == 0 && (!j.weighted || ((uintptr_t)j.w & 15) == 0);
        if (bulk_env && aligned && nnz >= kTile) {
            const int smem = kBulkStages * kTile * 4 * (j.weighted ? 2 : 1);  // kTile = kWin per warp
            static const bool attr = [] {
                GD_CUDA(cudaFuncSetAttribute(k_edit_bulk<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             kBulkStages * kTile * 8));
                GD_CUDA(cudaFuncSetAttribute(k_edit_bulk<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             kBulkStages * kTile * 4));
                return true;
            }();
            (void)attr;
            int per_sm = 0;
            GD_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
                &per_sm, j.weighted ? k_edit_bulk<true> : k_edit_bulk<false>, kEditThreads, smem));
            const unsigned gb = (unsigned)std::max<int64_t>(1, std::min<int64_t>(ntiles, 148LL * std::max(per_sm, 1)));
            if (j.weighted)
                GD_KERNEL_T("merge_copy", (nnz + (nnz - dead_total)) * 8, k_edit_bulk<true>, gb, kEditThreads, smem,
                            s, j.col, j.w, nnz, j.dead_win.get(), j.ipos, pj.get(), j.icol, j.iw, nwin,
                            new_col.get(), new_w.get());
            else
                GD_KERNEL_T("merge_copy", (nnz + (nnz - dead_total)) * 4, k_edit_bulk<false>, gb, kEditThreads, smem,
                            s, j.col, nullptr, nnz, j.dead_win.get(), j.ipos, pj.get(), j.icol, nullptr, nwin,
                            new_col.get(), nullptr);
        } else if (j.weighted)
            GD_KERNEL_T("merge_copy", (nnz + (nnz - dead_total)) * 8, k_edit_base<true>, g, kEditThreads, 0, s, j.col,
                        j.w, nnz, j.dead_win.get(), j.ipos, pj.get(), j.icol, j.iw, nwin, new_col.get(), new_w.get());
        else
            GD_KERNEL_T("merge_copy", (nnz + (nnz - dead_total)) * 4, k_edit_base<false>, g, kEditThreads, 0, s,
                        j.col, nullptr, nnz, j.dead_win.get(), j.ipos, pj.get(), j.icol, nullptr, nwin, new_col.get(),
                        nullptr);
    }
    if (nins)
        GD_KERNEL(k_edit_tail, grid_for(nins, 256), 256, 0, s, j.ipos, nins, nnz, j.dead_win.get() + nwin, j.icol,
                  j.iw, new_col.get(), j.weighted ? new_w.get() : nullptr);
    j.counts.release();
    j.shift.release();
}

void edit_merge(cudaStream_t s, int64_t n, const int64_t* off, int32_t* col, const int32_t* w, int64_t nnz,
                const int64_t* tpos, const int32_t* trow, int64_t ntomb, bool dedupe, const int32_t* irow,
                const int32_t* icol, const int32_t* iw, const int64_t* ipos, int64_t nins, DBuf<int64_t>& new_off,
                DBuf<int32_t>& new_col, DBuf<int32_t>& new_w, int64_t& new_nnz, bool weighted) {
    EditJob j{n, off, col, w, nnz, tpos, trow, ntomb, dedupe, irow, icol, iw, ipos, nins, weighted};
    edit_plan(s, j);
    int64_t dead_total = read_scalar(s, j.dead_win.get() + j.nwin);  // sizes the new arrays
    edit_apply(s, j, dead_total, new_off, new_col, new_w, new_nnz);
}

// ==========================================================================

Store::Store(int dev, int64_t n_, const int64_t* src, const int64_t* dst, const int64_t* w, int64_t m, bool dir,
             bool wtd, bool with_rev, int64_t mi, bool as_arcs, const Comm* pc)
    : device(dev), part(pc), n(n_), directed(dir), weighted(wtd), with_reverse(with_rev), merge_interval(mi) {
    sh = bits_for((uint64_t)std::max<int64_t>(n - 1, 1));
    own_hi = n;
    if (part) {
        if (!directed)
            throw GdError(GD_ERR_CONFIG, "vertex-partitioned stores hold directed graphs (undirected graphs are "
                                         "replicated per rank)");
        blocks = Blocks(n, part->world);
        own_lo = blocks.lo(part->rank);
        own_hi = blocks.hi(part->rank);
    }
    GD_CUDA(cudaSetDevice(device));
    GD_CUDA(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
    // keep freed stream-ordered memory in the pool across syncs: per-batch
    // temporaries are re-used instead of being unmapped and re-mapped
    cudaMemPool_t pool;
    GD_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
    uint64_t keep = UINT64_MAX;
    GD_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
    cudaStream_t s = stream;
    bool expand = !directed && !as_arcs;
    int64_t na = expand ? 2 * m : m;
    // host edge arrays -> device (int64 as given; converted in the expand kernel)
    DBuf<int64_t> hs(m, s), hd(m, s), hw(w ? m : 0, s);
    if (m) {
        GD_CUDA(cudaMemcpyAsync(hs.get(), src, m * sizeof(int64_t), cudaMemcpyHostToDevice, s));
        GD_CUDA(cudaMemcpyAsync(hd.get(), dst, m * sizeof(int64_t), cudaMemcpyHostToDevice, s));
        if (w) GD_CUDA(cudaMemcpyAsync(hw.get(), w, m * sizeof(int64_t), cudaMemcpyHostToDevice, s));
    }
    DBuf<uint32_t> key(na, s);
    DBuf<int32_t> val(na, s), adst(na, s), aw(na, s);
    if (m)
        GD_KERNEL(k_expand_edges, grid_for(m, 256), 256, 0, s, hs.get(), hd.get(), w ? hw.get() : nullptr, m,
                  !expand, key.get(), val.get(), adst.get(), aw.get());
    DBuf<int32_t> in_src, in_dst, in_w;
    int64_t m_in = 0;
    if (part && na) {  // owned sources' out-arcs stay (stream order kept); owned destinations' in-arcs aside
        DBuf<uint8_t> fo(na, s), fi(na, s);
        GD_KERNEL(k_part_flags, grid_for(na, 256), 256, 0, s, key.get(), adst.get(), na, blocks, part->rank, fo.get(),
                  fi.get());
        DBuf<int32_t> so(na, s), si(na, s);
        const int64_t mo = select_flagged_index(s, fo.get(), na, so.get());
        m_in = select_flagged_index(s, fi.get(), na, si.get());
        in_src.alloc(m_in, s);
        in_dst.alloc(m_in, s);
        in_w.alloc(m_in, s);
        if (m_in) {
            GD_KERNEL(k_gather<int32_t>, grid_for(m_in, 256), 256, 0, s, reinterpret_cast<const int32_t*>(key.get()),
                      si.get(), m_in, in_src.get());
            GD_KERNEL(k_gather<int32_t>, grid_for(m_in, 256), 256, 0, s, adst.get(), si.get(), m_in, in_dst.get());
            GD_KERNEL(k_gather<int32_t>, grid_for(m_in, 256), 256, 0, s, aw.get(), si.get(), m_in, in_w.get());
        }
        DBuf<uint32_t> k2(mo, s);
        DBuf<int32_t> d2(mo, s), w2(mo, s);
        if (mo) {
            GD_KERNEL(k_gather<uint32_t>, grid_for(mo, 256), 256, 0, s, key.get(), so.get(), mo, k2.get());
            GD_KERNEL(k_gather<int32_t>, grid_for(mo, 256), 256, 0, s, adst.get(), so.get(), mo, d2.get());
            GD_KERNEL(k_gather<int32_t>, grid_for(mo, 256), 256, 0, s, aw.get(), so.get(), mo, w2.get());
        }
        key = std::move(k2);
        adst = std::move(d2);
        aw = std::move(w2);
        na = mo;
        iota_i32(s, val.get(), na);
    }
    // stable sort by source keeps insertion order within a source (dynamic.py:116)
    sort_pairs_u32(s, key.get(), val.get(), na, sh);
    OutSeg base;
    base.nslots = na;
    base.col.alloc(na, s);
    if (weighted) base.w.alloc(na, s);
    if (na) {
        GD_KERNEL(k_gather<int32_t>, grid_for(na, 256), 256, 0, s, adst.get(), val.get(), na, base.col.get());
        if (weighted) GD_KERNEL(k_gather<int32_t>, grid_for(na, 256), 256, 0, s, aw.get(), val.get(), na, base.w.get());
    }
    {
        DBuf<int64_t> cnt(n + 1, s);
        cnt.zero(s);
        if (na) GD_KERNEL(k_hist_rows_u32, grid_for(na, 256), 256, 0, s, key.get(), na, cnt.get());
        base.off.alloc(n + 1, s);
        exclusive_scan_i64(s, cnt.get(), base.off.get(), n + 1);
    }
    segs.push_back(std::move(base));
    live = na;
    dcounts.alloc(2, s);
    dcounts.zero(s);
    upload_tables();
    if (with_reverse) {
        if (part) index_from_arcs(rev, true, in_src.get(), in_dst.get(), in_w.get(), m_in);
        else build_index(rev, true);
    }
    GD_CUDA(cudaStreamSynchronize(s));
}

Store::~Store() {
    if (stream) {
        cudaSetDevice(device);
        segs.clear();
        rev = SortedIndex();
        fwd = SortedIndex();
        dcounts.release();
        otpos.release();
        otrow.release();
        tab.release();
        cudaStreamSynchronize(stream);
        dev_cache_release(stream);  // the stream's cached blocks go back to the pool
        cudaStreamSynchronize(stream);
        cudaStreamDestroy(stream);
        stream = nullptr;
    }
}

namespace {
constexpr int kTabMax = 16;
struct SegTable {
    uintptr_t v[4 * kTabMax];
};
__global__ void k_set_table(SegTable t, int k, uintptr_t* tab) {
    for (int i = threadIdx.x; i < 4 * k; i += blockDim.x) tab[i] = t.v[(i / k) * kTabMax + (i % k)];
}
}  // namespace

void Store::upload_tables() {
    size_t k = segs.size();
    tab.ensure(4 * k, stream);
    if (k <= (size_t)kTabMax) {  // by value through a kernel: no host buffer to keep alive
        SegTable t{};
        int64_t acc = 0;
        for (size_t i = 0; i < k; ++i) {
            t.v[i] = reinterpret_cast<uintptr_t>(segs[i].off.get());
            t.v[kTabMax + i] = reinterpret_cast<uintptr_t>(segs[i].col.get());
            t.v[2 * kTabMax + i] = reinterpret_cast<uintptr_t>(segs[i].w.n ? segs[i].w.get() : nullptr);
            t.v[3 * kTabMax + i] = (uintptr_t)acc;
            acc += segs[i].nslots;
        }
        GD_KERNEL(k_set_table, 1, 64, 0, stream, t, (int)k, tab.get());
    } else {
        // the previous copy may still be in flight: wait before reusing the host table
        GD_CUDA(cudaStreamSynchronize(stream));
        h_tab.assign(4 * k, 0);
        int64_t acc = 0;
        for (size_t i = 0; i < k; ++i) {
            h_tab[i] = reinterpret_cast<uintptr_t>(segs[i].off.get());
            h_tab[k + i] = reinterpret_cast<uintptr_t>(segs[i].col.get());
            h_tab[2 * k + i] = reinterpret_cast<uintptr_t>(segs[i].w.n ? segs[i].w.get() : nullptr);
            h_tab[3 * k + i] = (uintptr_t)acc;
            acc += segs[i].nslots;
        }
        GD_CUDA(cudaMemcpyAsync(tab.get(), h_tab.data(), 4 * k * sizeof(uintptr_t), cudaMemcpyHostToDevice,
                                stream));
    }
    tab_k = k;
}

OutView Store::out_view() const {
    const uintptr_t* t = tab.get();
    size_t k = tab_k;
    return OutView{(int)k, reinterpret_cast<const int64_t* const*>(t), reinterpret_cast<const int32_t* const*>(t + k),
                   reinterpret_cast<const int32_t* const*>(t + 2 * k), reinterpret_cast<const int64_t*>(t + 3 * k)};
}

int64_t Store::total_slots() const {
    int64_t t = 0;
    for (auto& sg : segs) t += sg.nslots;
    return t;
}

int64_t Store::device_bytes() const {
    int64_t b = 0;
    for (auto& sg : segs) b += (int64_t)(sg.off.n * 8 + sg.col.n * 4 + sg.w.n * 4);
    for (const SortedIndex* ix : {&rev, &fwd})
        b += (int64_t)(ix->off.n * 8 + ix->col.n * 4 + ix->w.n * 4 + ix->dcol.n * 12 + ix->tpos.n * 12);
    return b;
}

// Build a sorted index from the current live out-arcs (all segments).
void Store::build_index(SortedIndex& ix, bool rows_are_dst) {
    cudaStream_t s = stream;
    int64_t tot = total_slots();
    DBuf<int32_t> asrc(tot, s), adst(tot, s), aw(tot, s);
    int64_t m = 0;
    for (auto& sg : segs) {
        if (!sg.nslots) continue;
        DBuf<int32_t> row(sg.nslots, s);
        DBuf<uint8_t> livef(sg.nslots, s);
        GD_KERNEL(k_delta_rows, grid_for(sg.nslots, 256), 256, 0, s, sg.off.get(), n, sg.col.get(), sg.nslots,
                  row.get(), livef.get());
        DBuf<int32_t> sel(sg.nslots, s);
        int64_t c = select_flagged_index(s, livef.get(), sg.nslots, sel.get());
        if (!c) continue;
        GD_KERNEL(k_gather<int32_t>, grid_for(c, 256), 256, 0, s, row.get(), sel.get(), c, asrc.get() + m);
        GD_KERNEL(k_gather<int32_t>, grid_for(c, 256), 256, 0, s, sg.col.get(), sel.get(), c, adst.get() + m);
        if (weighted)
            GD_KERNEL(k_gather<int32_t>, grid_for(c, 256), 256, 0, s, sg.w.get(), sel.get(), c, aw.get() + m);
        else
            fill_i32(s, aw.get() + m, c, 1);
        m += c;
    }
    index_from_arcs(ix, rows_are_dst, asrc.get(), adst.get(), aw.get(), m);
}

// A clean sorted index over the given arcs (src -> dst, weight): rows are the
// destinations (rev) or the sources (fwd), columns ascending within a row.
void Store::index_from_arcs(SortedIndex& ix, bool rows_are_dst, const int32_t* asrc, const int32_t* adst,
                            const int32_t* aw, int64_t m) {
    cudaStream_t s = stream;
    ix.rows_are_dst = rows_are_dst;
    DBuf<uint64_t> key(m, s);
    DBuf<int32_t> val(m, s);
    if (m) GD_KERNEL(k_added_to_index, grid_for(m, 256), 256, 0, s, asrc, adst, m, rows_are_dst, sh, key.get(),
                     val.get());
    // val = position in the arc arrays (indexes aw); the key carries (row, col)
    iota_i32(s, val.get(), m);
    sort_pairs_u64(s, key.get(), val.get(), m, 2 * sh);
    ix.nnz = m;
    ix.col.alloc(m, s);
    DBuf<int32_t> rows(m, s);
    if (m) GD_KERNEL(k_key_split, grid_for(m, 256), 256, 0, s, key.get(), m, sh, rows.get(), ix.col.get());
    if (weighted) {
        ix.w.alloc(m, s);
        if (m) GD_KERNEL(k_gather<int32_t>, grid_for(m, 256), 256, 0, s, aw, val.get(), m, ix.w.get());
    } else {
        ix.w.release();
    }
    offsets_from_rows(s, n, rows.get(), m, ix.off);
    ix.ntomb = 0;
    ix.dnnz = 0;
    ix.built = true;
}

void Store::require_rev() {
    if (!rev.built) build_index(rev, true);
}
void Store::require_fwd() {
    if (!fwd.built) build_index(fwd, false);
}

// Fold tombstones and the delta into a clean index.
// index compaction as a plan (k_index_ins_pos + histograms) and a finish
void Store::index_plan(SortedIndex& ix, EditJob& j, DBuf<int64_t>& ipos) {
    cudaStream_t s = stream;
    ipos.alloc(ix.dnnz, s);
    if (ix.dnnz)
        GD_KERNEL_T("index_ins_pos", 0, k_index_ins_pos, grid_for(ix.dnnz, 256), 256, 0, s, ix.drow.get(),
                    ix.dcol.get(), ix.dnnz, ix.off.get(), ix.col.get(), ipos.get());
    j = EditJob{n, ix.off.get(), ix.col.get(), ix.w.n ? ix.w.get() : nullptr, ix.nnz, ix.tpos.get(), ix.trow.get(),
                ix.ntomb, false, ix.drow.get(), ix.dcol.get(), ix.dw.n ? ix.dw.get() : nullptr, ipos.get(), ix.dnnz,
                weighted};
    edit_plan(s, j);
}

void Store::index_finish(SortedIndex& ix, EditJob& j, int64_t dead_total) {
    DBuf<int64_t> noff;
    DBuf<int32_t> ncol, nw;
    int64_t nnz2 = 0;
    edit_apply(stream, j, dead_total, noff, ncol, nw, nnz2);
    ix.off = std::move(noff);
    ix.col = std::move(ncol);
    ix.w = std::move(nw);
    ix.nnz = nnz2;
    ix.ntomb = 0;
    ix.dnnz = 0;
    ix.tpos.release();
    ix.trow.release();
    ix.drow.release();
    ix.dcol.release();
    ix.dw.release();
}

void Store::compact_index(SortedIndex& ix) {
    if (!ix.built || !ix.dirty()) return;
    EditJob j;
    DBuf<int64_t> ipos;
    index_plan(ix, j, ipos);
    index_finish(ix, j, read_scalar(stream, j.dead_win.get() + j.nwin));
}

void Store::index_delete(SortedIndex& ix, const KilledArcs& ka) {
    if (!ix.built || ka.count == 0) return;
    cudaStream_t s = stream;
    int64_t m = ka.count;  // slots (one per request; gid -1 = none)
    int64_t old = ix.ntomb;
    DBuf<int64_t> tpos(old + m, s);
    DBuf<int32_t> trow(old + m, s);
    if (old) {
        copy_d2d(s, tpos.get(), ix.tpos.get(), old * 8);
        copy_d2d(s, trow.get(), ix.trow.get(), old * 4);
    }
    if (m)
        GD_KERNEL_T("index_claim", 0, k_index_claim, grid_for(m, 256), 256, 0, s, ka.row.get(), ka.col.get(),
                    ka.w.get(), ka.gid.get(), m, ix.rows_are_dst, ix.off.get(), ix.col.get(),
                    ix.w.n ? ix.w.get() : nullptr, tpos.get() + old, trow.get() + old);
    ix.tpos = std::move(tpos);
    ix.trow = std::move(trow);
    ix.ntomb = old + m;
}

void Store::index_add(SortedIndex& ix, const AddedArcs& aa) {
    if (!ix.built || aa.count == 0) return;
    if (ix.dnnz) compact_index(ix);  // keep at most one delta
    cudaStream_t s = stream;
    int64_t m = aa.count;
    static const bool full_sort = getenv("GD_INDEX_FULL_SORT") != nullptr;  // A/B: the (row, col) key sort
    if (ix.rows_are_dst && aa.by_row && !full_sort) {
        // the arcs already sorted by source (stable): one stable pass by
        // destination gives (destination, source, stream) order -- the same
        // order as sorting the (destination, source) keys with the arc index
        // as the tie-break, in 32-bit keys of sh bits (3 passes at scale 22,
        // not 6 over 44-bit keys)
        DBuf<uint32_t> k32(m, s);
        DBuf<int32_t> v32(m, s);
        GD_KERNEL(k_dst_by_src, grid_for(m, 256), 256, 0, s, aa.by_row, aa.col.get(), m, k32.get(), v32.get());
        sort_pairs_u32(s, k32.get(), v32.get(), m, sh);
        ix.drow.alloc(m, s);
        ix.dcol.alloc(m, s);
        if (weighted) ix.dw.alloc(m, s);
        GD_KERNEL(k_rev_delta_split, grid_for(m, 256), 256, 0, s, k32.get(), v32.get(), m, aa.row.get(),
                  weighted ? aa.w.get() : nullptr, ix.drow.get(), ix.dcol.get(), weighted ? ix.dw.get() : nullptr);
        ix.dnnz = m;
        return;
    }
    DBuf<uint64_t> key(m, s);
    DBuf<int32_t> val(m, s);
    GD_KERNEL(k_added_to_index, grid_for(m, 256), 256, 0, s, aa.row.get(), aa.col.get(), m, ix.rows_are_dst, sh,
              key.get(), val.get());
    // the values only carry the weights: an unweighted index sorts its keys alone
    if (weighted) sort_pairs_u64(s, key.get(), val.get(), m, 2 * sh);
    else sort_keys_u64(s, key.get(), m, 2 * sh);
    ix.drow.alloc(m, s);
    ix.dcol.alloc(m, s);
    GD_KERNEL(k_key_split, grid_for(m, 256), 256, 0, s, key.get(), m, sh, ix.drow.get(), ix.dcol.get());
    if (weighted) {
        ix.dw.alloc(m, s);
        GD_KERNEL(k_gather<int32_t>, grid_for(m, 256), 256, 0, s, aa.w.get(), val.get(), m, ix.dw.get());
    }
    ix.dnnz = m;
}

void Store::append_out_tombs(const int64_t* d_pos, const int32_t* d_row, int64_t cnt) {
    if (!cnt) return;
    cudaStream_t s = stream;
    int64_t tot = notomb + cnt;
    DBuf<int64_t> p(tot, s);
    DBuf<int32_t> r(tot, s);
    if (notomb) {
        copy_d2d(s, p.get(), otpos.get(), notomb * 8);
        copy_d2d(s, r.get(), otrow.get(), notomb * 4);
    }
    copy_d2d(s, p.get() + notomb, d_pos, cnt * 8);
    copy_d2d(s, r.get() + notomb, d_row, cnt * 4);
    otpos = std::move(p);
    otrow = std::move(r);
    notomb = tot;
}

// ---------------------------------------------------------------- partitioned stores

int64_t Store::owned_records(const int32_t* src, const int32_t* dst, const int32_t* w, int64_t k, DBuf<int32_t>& idx,
                             DBuf<int32_t>& os, DBuf<int32_t>& od, DBuf<int32_t>& ow) {
    cudaStream_t s = stream;
    DBuf<uint8_t> f(std::max<int64_t>(k, 1), s);
    idx.alloc(std::max<int64_t>(k, 1), s);
    if (k) GD_KERNEL(k_owned_flags, grid_for(k, 256), 256, 0, s, src, k, blocks, part->rank, f.get());
    const int64_t kl = k ? select_flagged_index(s, f.get(), k, idx.get()) : 0;
    os.alloc(std::max<int64_t>(kl, 1), s);
    od.alloc(std::max<int64_t>(kl, 1), s);
    if (w) ow.alloc(std::max<int64_t>(kl, 1), s);
    if (kl) {
        GD_KERNEL(k_gather<int32_t>, grid_for(kl, 256), 256, 0, s, src, idx.get(), kl, os.get());
        GD_KERNEL(k_gather<int32_t>, grid_for(kl, 256), 256, 0, s, dst, idx.get(), kl, od.get());
        if (w) GD_KERNEL(k_gather<int32_t>, grid_for(kl, 256), 256, 0, s, w, idx.get(), kl, ow.get());
    }
    return kl;
}

void Store::route_arcs(const int32_t* row, const int32_t* col, const int32_t* w, const int64_t* gid, int64_t m,
                       DBuf<int32_t>& orow, DBuf<int32_t>& ocol, DBuf<int32_t>& ow, int64_t& count) {
    cudaStream_t s = stream;
    const int W = part->world;
    DBuf<unsigned long long> cnt(2 * W, s);  // [counts | cursors]
    cnt.zero(s);
    DBuf<int32_t> packed(std::max<int64_t>(3 * m, 1), s);
    if (m) {
        GD_KERNEL(k_route_count, grid_for(m, 256), 256, 0, s, col, gid, m, blocks, cnt.get());
        GD_KERNEL(k_route_offsets, 1, 1, 0, s, cnt.get(), W, cnt.get() + W);
        GD_KERNEL(k_route_scatter, grid_for(m, 256), 256, 0, s, row, col, w, gid, m, blocks, cnt.get() + W,
                  packed.get());
    }
    DBuf<int32_t> recv;
    count = part->alltoallv_i32(packed.get(), reinterpret_cast<const int64_t*>(cnt.get()), 3, recv, s);
    orow.alloc(std::max<int64_t>(count, 1), s);
    ocol.alloc(std::max<int64_t>(count, 1), s);
    ow.alloc(std::max<int64_t>(count, 1), s);
    if (count) GD_KERNEL(k_unpack3, grid_for(count, 256), 256, 0, s, recv.get(), count, orow.get(), ocol.get(),
                         ow.get(), nullptr);
}

// the in-index keeps the arcs of owned destinations: killed / inserted arcs
// travel to the owner of their destination (partition.py routes records to
// the source's owner, :206-235; the in-index is the destination's)
void Store::rev_delete(const KilledArcs& ka) {
    if (!part || !rev.built) {
        index_delete(rev, ka);
        return;
    }
    KilledArcs rk;
    route_arcs(ka.row.get(), ka.col.get(), ka.w.get(), ka.gid.get(), ka.count, rk.row, rk.col, rk.w, rk.count);
    rk.gid.alloc(std::max<int64_t>(rk.count, 1), stream);
    fill_i64(stream, rk.gid.get(), rk.count, 0);
    index_delete(rev, rk);
}

void Store::rev_add(const AddedArcs& aa) {
    if (!part || !rev.built) {
        index_add(rev, aa);
        return;
    }
    AddedArcs ra;
    route_arcs(aa.row.get(), aa.col.get(), aa.w.get(), nullptr, aa.count, ra.row, ra.col, ra.w, ra.count);
    index_add(rev, ra);
}

int64_t Store::apply_deletes(const int32_t* d_src, const int32_t* d_dst, int64_t k, uint8_t* d_found,
                             bool want_count) {
    if (!part) return apply_deletes_local(d_src, d_dst, k, d_found, want_count);
    cudaStream_t s = stream;
    DBuf<int32_t> idx, os, od, ow;
    const int64_t kl = owned_records(d_src, d_dst, nullptr, k, idx, os, od, ow);
    DBuf<uint8_t> lf;
    if (d_found) lf.alloc(std::max<int64_t>(kl, 1), s);
    int64_t applied = apply_deletes_local(os.get(), od.get(), kl, d_found ? lf.get() : nullptr, want_count);
    if (d_found && k) {  // flags of the owned records; other ranks hold the rest
        fill_d(s, d_found, 0, k);
        if (kl) GD_KERNEL(k_scatter_u8, grid_for(kl, 256), 256, 0, s, lf.get(), idx.get(), kl, d_found);
    }
    if (want_count) {
        DBuf<int64_t> a(1, s);
        GD_CUDA(cudaMemcpyAsync(a.get(), &applied, 8, cudaMemcpyHostToDevice, s));
        part->allreduce_sum_i64(a.get(), 1, s);
        applied = read_scalar(s, a.get());
    }
    return applied;
}

int64_t Store::apply_deletes_local(const int32_t* d_src, const int32_t* d_dst, int64_t k, uint8_t* d_found,
                                   bool want_count) {
    cudaStream_t s = stream;
    if (k == 0) {
        if (part) rev_delete(KilledArcs{});  // the routing is collective
        return 0;
    }
    if (rev.built) compact_index(rev);
    if (fwd.built) compact_index(fwd);
    first_clean_delta = segs.size();  // deltas made before this delete may now hold tombstones
    const int kb = 2 * sh;
    const int64_t nrq = directed ? k : 2 * k;
    DBuf<uint64_t> rq_key(nrq, s);
    DBuf<int32_t> rq_occ(nrq, s), rq_rec(nrq, s);
    DBuf<uint8_t> rq_which(nrq, s);
    if (directed) {  // records sorted by (src, dst), stable: equal pairs in stream order
        DBuf<int32_t> srec(k, s), rq_ord(nrq, s);
        GD_KERNEL(k_del_keys, grid_for(k, 256), 256, 0, s, d_src, d_dst, k, directed, sh, rq_key.get(), srec.get());
        sort_pairs_u64(s, rq_key.get(), srec.get(), k, kb);
        GD_KERNEL(k_del_requests, grid_for(k, 256), 256, 0, s, rq_key.get(), srec.get(), k, d_src, d_dst, directed,
                  sh, rq_key.get(), rq_occ.get(), rq_rec.get(), rq_which.get(), rq_ord.get());
    } else {  // both directions of every record, one sort by directed key
        DBuf<int32_t> rq_val(nrq, s);
        GD_KERNEL(k_del_requests_u, grid_for(k, 256), 256, 0, s, d_src, d_dst, k, sh, rq_key.get(), rq_val.get());
        sort_pairs_u64(s, rq_key.get(), rq_val.get(), nrq, kb);
        GD_KERNEL(k_del_requests_u_fill, grid_for(nrq, 256), 256, 0, s, rq_key.get(), rq_val.get(), nrq,
                  rq_occ.get(), rq_rec.get(), rq_which.get());
    }
    // distinct source rows and their chain work items
    DBuf<uint8_t> rflag(nrq, s);
    GD_KERNEL(k_row_starts, grid_for(nrq, 256), 256, 0, s, rq_key.get(), nrq, sh, rflag.get());
    DBuf<int32_t> row_first(nrq, s);
    // nrows, work items, longest chain, overflow matches, head / tail slots scanned
    DBuf<int64_t> hdr(6, s);
    fill_d(s, hdr.get(), 0, 6 * sizeof(int64_t));
    select_flagged_index_async(s, rflag.get(), nrq, row_first.get(), hdr.get());
    OutView ov = out_view();
    DBuf<int64_t> chunks(nrq + 1, s), coff(nrq + 1, s);
    GD_KERNEL(k_row_chunks, grid_for(nrq + 1, 256), 256, 0, s, ov, rq_key.get(), row_first.get(), hdr.get(), nrq + 1,
              sh, chunks.get(), reinterpret_cast<unsigned long long*>(hdr.get() + 2),
              reinterpret_cast<unsigned long long*>(hdr.get() + 4));
    exclusive_scan_i64(s, chunks.get(), coff.get(), nrq + 1);
    copy_d2d(s, hdr.get() + 1, coff.get() + nrq, 8);
    // tail pieces: at most one per kChunk slots of the requested rows
    DBuf<int32_t> wrow(total_slots() / kChunk + nrq + 1, s);
    GD_KERNEL(k_chunk_rows, grid_for(nrq, 256), 256, 0, s, coff.get(), hdr.get(), wrow.get());
    // single-request pairs resolve by atomicMin; the rest collect overflow
    // matches (retry once with the exact size on overflow).  Row and work
    // counts stay on the device: the one read-back is the overflow size
    // together with the longest chain.
    DBuf<uint8_t> single(nrq, s);
    DBuf<unsigned long long> sel(nrq, s);
    GD_KERNEL(k_single_flags, grid_for(nrq, 256), 256, 0, s, rq_key.get(), nrq, single.get(), sel.get());
    int64_t cap = 1024;
    DBuf<uint64_t> m_key;
    DBuf<int64_t> m_chain;
    DBuf<int64_t> m_gid;
    int64_t nm = 0, maxchain = 0;
    for (int attempt = 0; attempt < 2; ++attempt) {
        m_key.alloc(cap, s);
        m_chain.alloc(cap, s);
        m_gid.alloc(cap, s);
        if (attempt) {  // overflow retry: start the match collection over
            fill_d(s, hdr.get() + 3, 0, 8);
            fill_d(s, sel.get(), 0xff, nrq * 8);
        }
        MatchOut mo{sel.get(), single.get(), m_key.get(), m_chain.get(), m_gid.get(),
                    reinterpret_cast<unsigned long long*>(hdr.get() + 3), cap};
        const int ph = prof_begin("del_scan_head", 0, s);
        k_del_scan_head<<<grid_for(((nrq + 3) / 4) * 32, 256, 148LL * 32), 256, 0, s>>>(ov, row_first.get(), hdr.get(),
                                                                                    rq_key.get(), nrq, sh, mo);
        count_launch();
        GD_LAUNCH_CHECK();
        prof_end(ph, s);
        const int pt = prof_begin("del_scan_tail", 0, s);
        k_del_scan_tail<<<148 * 16, kScanWarps * 32, 0, s>>>(ov, row_first.get(), coff.get(), wrow.get(), hdr.get(),
                                                             rq_key.get(), nrq, sh, mo);
        count_launch();
        GD_LAUNCH_CHECK();
        prof_end(pt, s);
        int64_t h6[6];
        read_small(s, h6, hdr.get(), sizeof h6);
        maxchain = h6[2];
        nm = h6[3];
        // algorithmic bytes: the chain slots each kernel reads
        // (idx), the request keys, and the row offsets of every segment
        prof_set_bytes(ph, 4 * h6[4] + 8 * nrq + 16 * (int64_t)ov.nseg * h6[0]);
        prof_set_bytes(pt, 4 * h6[5] + 8 * h6[1]);
        if (nm <= cap) break;
        cap = nm;
    }
    int rb = bits_for((uint64_t)std::max<int64_t>(maxchain, 1));
    const bool one_sort = kb + rb <= 64;  // (pair, chain offset) fits one 64-bit key
    if (!one_sort) rb = 0;
    // the overflow matches sort through a permutation (int32: matches are
    // per batch), their int64 slot ids follow it
    if (nm >= 1 && one_sort) {
        GD_KERNEL(k_overflow_keys, grid_for(nm, 256), 256, 0, s, m_key.get(), m_chain.get(), nm, rb);
        if (nm > 1) {
            DBuf<int32_t> perm(nm, s);
            iota_i32(s, perm.get(), nm);
            sort_pairs_u64(s, m_key.get(), perm.get(), nm, kb + rb);
            DBuf<int64_t> g2(nm, s);
            GD_KERNEL(k_gather<int64_t>, grid_for(nm, 256), 256, 0, s, m_gid.get(), perm.get(), nm, g2.get());
            m_gid = std::move(g2);
        }
    } else if (nm > 1) {  // LSD: by gid (= chain order), then stable by pair key
        DBuf<uint64_t> gk(nm, s);
        DBuf<int32_t> perm(nm, s);
        GD_KERNEL(k_widen64, grid_for(nm, 256), 256, 0, s, m_gid.get(), nm, gk.get());
        iota_i32(s, perm.get(), nm);
        sort_pairs_u64(s, gk.get(), perm.get(), nm, 64);
        DBuf<uint64_t> k2(nm, s);
        GD_KERNEL(k_gather<uint64_t>, grid_for(nm, 256), 256, 0, s, m_key.get(), perm.get(), nm, k2.get());
        sort_pairs_u64(s, k2.get(), perm.get(), nm, kb);
        DBuf<int64_t> g2(nm, s);
        GD_KERNEL(k_gather<int64_t>, grid_for(nm, 256), 256, 0, s, m_gid.get(), perm.get(), nm, g2.get());
        m_key = std::move(k2);
        m_gid = std::move(g2);
    }
    DBuf<int64_t> rq_pos(nrq, s);
    DBuf<uint8_t> found_local;
    uint8_t* found = d_found;
    if (!found) {
        found_local.alloc(k, s);
        found = found_local.get();
    }
    // every record's forward request writes its found flag (k_del_resolve): no memset
    // [0] applied records of this call, [1] killed slots since `live` was last
    // brought up to date (read lazily: live_count())
    fill_d(s, dcounts.get(), 0, sizeof(unsigned long long));
    unsigned long long* counts = dcounts.get();
    GD_KERNEL(k_del_resolve, grid_for(nrq, 256), 256, 0, s, rq_key.get(), rq_occ.get(), rq_rec.get(),
              rq_which.get(), single.get(), sel.get(), nrq, m_key.get(), m_gid.get(), nm, rb, rq_pos.get(), found,
              counts);
    KilledArcs ka;
    ka.row.alloc(nrq, s);
    ka.col.alloc(nrq, s);
    ka.w.alloc(nrq, s);
    ka.gid.alloc(nrq, s);
    ka.count = nrq;
    GD_KERNEL(k_del_kill, grid_for(nrq, 256), 256, 0, s, ov, rq_key.get(), rq_rec.get(), rq_which.get(),
              rq_pos.get(), nrq, found, sh, ka.row.get(), ka.col.get(), ka.w.get(), ka.gid.get(), counts + 1);
    // the tomb logs take every slot (gid -1 = none; delta-segment gids are
    // ignored by the merge), unordered: no select, no sort
    append_out_tombs(ka.gid.get(), ka.row.get(), nrq);
    rev_delete(ka);
    if (fwd.built) index_delete(fwd, ka);
    if (!want_count) return -1;
    unsigned long long applied = 0;
    read_small(s, &applied, counts, sizeof applied);
    return (int64_t)applied;
}

int64_t Store::live_count() {
    unsigned long long killed = 0;
    read_small(stream, &killed, dcounts.get() + 1, sizeof killed);
    fill_d(stream, dcounts.get() + 1, 0, sizeof killed);
    live -= (int64_t)killed;
    return live;
}

void Store::apply_adds(const int32_t* d_src, const int32_t* d_dst, const int32_t* d_w, int64_t k) {
    if (!part) return apply_adds_local(d_src, d_dst, d_w, k);
    DBuf<int32_t> idx, os, od, ow;
    const int64_t kl = owned_records(d_src, d_dst, d_w, k, idx, os, od, ow);
    apply_adds_local(os.get(), od.get(), d_w ? ow.get() : nullptr, kl);
}

void Store::apply_adds_local(const int32_t* d_src, const int32_t* d_dst, const int32_t* d_w, int64_t k) {
    cudaStream_t s = stream;
    if (k == 0) {
        if (part) rev_add(AddedArcs{});
        return;
    }
    int64_t na = directed ? k : 2 * k;
    DBuf<uint32_t> key(na, s);
    DBuf<int32_t> val(na, s);
    AddedArcs aa;
    aa.row.alloc(na, s);
    aa.col.alloc(na, s);
    aa.w.alloc(na, s);
    aa.count = na;
    GD_KERNEL(k_add_arcs, grid_for(k, 256), 256, 0, s, d_src, d_dst, d_w, k, directed, key.get(), val.get(),
              aa.row.get(), aa.col.get(), aa.w.get());
    sort_pairs_u32(s, key.get(), val.get(), na, sh);  // stable: stream order within a source
    DBuf<uint8_t> rflag(na, s);
    GD_KERNEL(k_row_starts_u32, grid_for(na, 256), 256, 0, s, key.get(), na, rflag.get());
    DBuf<int32_t> row_first(na, s);
    DBuf<int64_t> d_nrows(1, s);
    select_flagged_index_async(s, rflag.get(), na, row_first.get(), d_nrows.get());
    DBuf<int64_t> vac(na, s);
    fill_i64(s, vac.get(), na, -1);
    OutView ov = out_view();
    static const bool warp_rows = getenv("GD_WARP_ROWS") != nullptr;  // A/B: the round-1 warp-per-row kernels
    if (warp_rows)
        GD_KERNEL_T("add_vacancies", 0, k_add_vacancies_g<32>, grid_for(na * 32, 256, 148LL * 32), 256, 0, s, ov,
                    key.get(), row_first.get(), d_nrows.get(), na, vac.get());
    else
    GD_KERNEL_T("add_vacancies", 0, k_add_vacancies_g<kVacG>, grid_for(na * kVacG, 256, 148LL * 32), 256, 0, s, ov, key.get(),
                row_first.get(), d_nrows.get(), na, vac.get());
    DBuf<uint8_t> left(na, s);
    ClaimLog cl;
    if (with_reverse) cl.gid.alloc(na, s);
    GD_KERNEL(k_add_claim, grid_for(na, 256), 256, 0, s, ov, val.get(), aa.col.get(), aa.w.get(), vac.get(), na,
              left.get(), with_reverse ? cl.gid.get() : nullptr);
    // leftovers (already ordered by (source, stream order)) -> one new delta
    DBuf<int32_t> sel(na, s);
    int64_t nl = select_flagged_index(s, left.get(), na, sel.get());
    if (nl) {
        OutSeg d;
        d.nslots = nl;
        DBuf<int32_t> lrow(nl, s);
        d.col.alloc(nl, s);
        if (weighted) d.w.alloc(nl, s);
        GD_KERNEL(k_gather_arcs, grid_for(nl, 256), 256, 0, s, sel.get(), nl, val.get(), aa.row.get(),
                  aa.col.get(), aa.w.get(), lrow.get(), d.col.get(), weighted ? d.w.get() : nullptr);
        offsets_from_rows(s, n, lrow.get(), nl, d.off);
        segs.push_back(std::move(d));
        upload_tables();
        cl.delta_seg = (int64_t)segs.size() - 1;
    }
    if (with_reverse) claim_logs.push_back(std::move(cl));
    live += na;
    aa.by_row = val.get();  // the source-sorted arc order (alive until return)
    rev_add(aa);
    if (fwd.built) index_add(fwd, aa);
}

void Store::merge() {
    cudaStream_t s = stream;
    // live delta arcs in (row, segment, slot) order
    int64_t dtot = 0;
    for (size_t i = 1; i < segs.size(); ++i) dtot += segs[i].nslots;
    DBuf<int32_t> irow(dtot, s), icol(dtot, s), iw(weighted ? dtot : 0, s);
    int64_t nins = 0;
    for (size_t i = 1; i < segs.size(); ++i) {
        OutSeg& d = segs[i];
        if (!d.nslots) continue;
        DBuf<int32_t> row(d.nslots, s);
        DBuf<uint8_t> lf(d.nslots, s);
        GD_KERNEL(k_delta_rows, grid_for(d.nslots, 256), 256, 0, s, d.off.get(), n, d.col.get(), d.nslots,
                  row.get(), lf.get());
        if (i >= first_clean_delta) {  // no delete phase since it was made: every slot is live
            copy_d2d(s, irow.get() + nins, row.get(), d.nslots * 4);
            copy_d2d(s, icol.get() + nins, d.col.get(), d.nslots * 4);
            if (weighted)
                copy_d2d(s, iw.get() + nins, d.w.get(), d.nslots * 4);
            nins += d.nslots;
            continue;
        }
        DBuf<int32_t> sel(d.nslots, s);
        int64_t c = select_flagged_index(s, lf.get(), d.nslots, sel.get());
        if (!c) continue;
        GD_KERNEL(k_gather_sel<int32_t>, grid_for(c, 256), 256, 0, s, row.get(), sel.get(), c, irow.get() + nins);
        GD_KERNEL(k_gather_sel<int32_t>, grid_for(c, 256), 256, 0, s, d.col.get(), sel.get(), c, icol.get() + nins);
        if (weighted)
            GD_KERNEL(k_gather_sel<int32_t>, grid_for(c, 256), 256, 0, s, d.w.get(), sel.get(), c, iw.get() + nins);
        nins += c;
    }
    if (segs.size() > 2 && nins > 1) {  // several deltas: stable sort by row keeps (segment, slot) order
        DBuf<uint32_t> rk(nins, s);
        copy_d2d(s, rk.get(), irow.get(), nins * 4);
        DBuf<int32_t> perm(nins, s);
        iota_i32(s, perm.get(), nins);
        sort_pairs_u32(s, rk.get(), perm.get(), nins, sh);
        DBuf<int32_t> r2(nins, s), c2(nins, s), w2(weighted ? nins : 0, s);
        GD_KERNEL(k_gather_sel<int32_t>, grid_for(nins, 256), 256, 0, s, irow.get(), perm.get(), nins, r2.get());
        GD_KERNEL(k_gather_sel<int32_t>, grid_for(nins, 256), 256, 0, s, icol.get(), perm.get(), nins, c2.get());
        if (weighted)
            GD_KERNEL(k_gather_sel<int32_t>, grid_for(nins, 256), 256, 0, s, iw.get(), perm.get(), nins, w2.get());
        irow = std::move(r2);
        icol = std::move(c2);
        iw = std::move(w2);
    }
    DBuf<int64_t> ipos(nins, s);
    if (nins) GD_KERNEL(k_out_ins_pos, grid_for(nins, 256), 256, 0, s, irow.get(), nins, segs[0].off.get(), ipos.get());
    // plan the out-store merge and the in-index compaction, then ONE read-back
    // of both death totals sizes both outputs
    EditJob jo{n, segs[0].off.get(), segs[0].col.get(), weighted ? segs[0].w.get() : nullptr, segs[0].nslots,
               otpos.get(), otrow.get(), notomb, true, irow.get(), icol.get(), weighted ? iw.get() : nullptr,
               ipos.get(), nins, weighted};
    edit_plan(s, jo);
    const bool rev_dirty = rev.built && rev.dirty();
    EditJob jr;
    DBuf<int64_t> rpos;
    if (rev_dirty) index_plan(rev, jr, rpos);
    DBuf<int64_t> totals(2, s);
    copy_d2d(s, totals.get(), jo.dead_win.get() + jo.nwin, 8);
    if (rev_dirty)
        copy_d2d(s, totals.get() + 1, jr.dead_win.get() + jr.nwin, 8);
    int64_t ht[2] = {0, 0};
    read_small(s, ht, totals.get(), rev_dirty ? 16 : 8);
    OutSeg nb;
    int64_t nnz2 = 0;
    edit_apply(s, jo, ht[0], nb.off, nb.col, nb.w, nnz2);
    if (rev_dirty) index_finish(rev, jr, ht[1]);
    nb.nslots = nnz2;
    segs.clear();
    segs.push_back(std::move(nb));
    upload_tables();
    otpos.release();
    otrow.release();
    notomb = 0;
    live = nnz2;  // exact: pending kills are folded in
    fill_d(s, dcounts.get() + 1, 0, sizeof(unsigned long long));
    first_clean_delta = 1;
    claim_logs.clear();  // _rebuild_reverse: list order restarts from the layout
    if (rev.built) compact_index(rev);
    if (fwd.built) compact_index(fwd);
}

void Store::export_segment(int64_t seg, int64_t* off, int64_t* col, int64_t* w) {
    cudaStream_t s = stream;
    OutSeg& sg = segs.at((size_t)seg);
    GD_CUDA(cudaMemcpyAsync(off, sg.off.get(), (n + 1) * 8, cudaMemcpyDeviceToHost, s));
    if (sg.nslots) {
        DBuf<int64_t> c(sg.nslots, s), ww(sg.nslots, s);
        GD_KERNEL(k_export_seg, grid_for(sg.nslots, 256), 256, 0, s, sg.col.get(), sg.w.n ? sg.w.get() : nullptr,
                  sg.nslots, c.get(), ww.get());
        GD_CUDA(cudaMemcpyAsync(col, c.get(), sg.nslots * 8, cudaMemcpyDeviceToHost, s));
        if (w) GD_CUDA(cudaMemcpyAsync(w, ww.get(), sg.nslots * 8, cudaMemcpyDeviceToHost, s));
        GD_CUDA(cudaStreamSynchronize(s));
    }
    GD_CUDA(cudaStreamSynchronize(s));
}

// nodes_to in the reference's list order, with slot identities
// (dynamic.py:152-160).  _rebuild_reverse (dynamic.py:319-329, at build and
// merge) lists a node's in-arcs in (segment, source, slot) order, i.e. global
// slot order; deletes remove entries in place; every later insert appends --
// vacancy claims in stream order, then the call's new delta in slot order
// (dynamic.py:266-285).  So a live slot sorts by the last append event that
// placed it (none: its rebuild position comes first).  Host-side: a query
// API, not on the batch path.
void Store::export_rev_slots(int64_t* off, int64_t* src, int64_t* seg, int64_t* idx, int64_t* w) {
    cudaStream_t s = stream;
    const size_t S = segs.size();
    std::vector<int64_t> base(S + 1, 0);
    std::vector<std::vector<int64_t>> hoff(S);
    std::vector<std::vector<int32_t>> hcol(S), hw(S);
    for (size_t i = 0; i < S; ++i) {
        base[i + 1] = base[i] + segs[i].nslots;
        hoff[i].resize(n + 1);
        hcol[i].resize(segs[i].nslots);
        GD_CUDA(cudaMemcpyAsync(hoff[i].data(), segs[i].off.get(), (n + 1) * 8, cudaMemcpyDeviceToHost, s));
        if (segs[i].nslots) {
            GD_CUDA(cudaMemcpyAsync(hcol[i].data(), segs[i].col.get(), segs[i].nslots * 4, cudaMemcpyDeviceToHost, s));
            if (weighted) {
                hw[i].resize(segs[i].nslots);
                GD_CUDA(cudaMemcpyAsync(hw[i].data(), segs[i].w.get(), segs[i].nslots * 4, cudaMemcpyDeviceToHost, s));
            }
        }
    }
    std::vector<std::vector<int64_t>> logs(claim_logs.size());
    for (size_t c = 0; c < claim_logs.size(); ++c) {
        logs[c].resize(claim_logs[c].gid.n);
        if (claim_logs[c].gid.n)
            GD_CUDA(cudaMemcpyAsync(logs[c].data(), claim_logs[c].gid.get(), claim_logs[c].gid.n * 8,
                                    cudaMemcpyDeviceToHost, s));
    }
    GD_CUDA(cudaStreamSynchronize(s));
    const int64_t total = base[S];
    std::vector<int64_t> event(total, -1);  // last append event per global slot
    int64_t ev = 0;
    for (size_t c = 0; c < logs.size(); ++c) {
        for (int64_t g : logs[c])
            if (g >= 0) event[g] = ev++;
        int64_t ds = claim_logs[c].delta_seg;
        if (ds >= 0)
            for (int64_t i = 0; i < segs[ds].nslots; ++i) event[base[ds] + i] = ev++;
    }
    // bucket live slots by destination, then order each bucket
    std::vector<int64_t> cnt(n + 1, 0);
    for (size_t i = 0; i < S; ++i)
        for (int32_t d : hcol[i])
            if (d >= 0) ++cnt[d + 1];
    for (int64_t v = 0; v < n; ++v) cnt[v + 1] += cnt[v];
    std::vector<int64_t> fill(cnt.begin(), cnt.end() - 1);
    std::vector<int64_t> gids(cnt[n]);
    for (size_t i = 0; i < S; ++i)
        for (int64_t j = 0; j < segs[i].nslots; ++j)
            if (hcol[i][j] >= 0) gids[fill[hcol[i][j]]++] = base[i] + j;
    auto later = [&](int64_t a, int64_t b) {  // rebuild entries (event -1) first, by slot
        if (event[a] != event[b]) return event[a] < event[b];
        return a < b;
    };
    for (int64_t v = 0; v < n; ++v) {
        std::sort(gids.begin() + cnt[v], gids.begin() + cnt[v + 1], later);
        off[v] = cnt[v];
    }
    off[n] = cnt[n];
    for (int64_t k = 0; k < cnt[n]; ++k) {
        int64_t g = gids[k];
        size_t sg = std::upper_bound(base.begin(), base.end(), g) - base.begin() - 1;
        int64_t i = g - base[sg];
        const std::vector<int64_t>& o = hoff[sg];
        src[k] = std::upper_bound(o.begin(), o.end(), i) - o.begin() - 1;
        seg[k] = (int64_t)sg;
        idx[k] = i;
        if (w) w[k] = weighted ? hw[sg][i] : 1;
    }
}

int64_t Store::rev_nnz_live() {
    require_rev();
    compact_index(rev);
    return rev.nnz;
}

void Store::export_rev(int64_t* off, int64_t* src, int64_t* w) {
    require_rev();
    compact_index(rev);
    cudaStream_t s = stream;
    GD_CUDA(cudaMemcpyAsync(off, rev.off.get(), (n + 1) * 8, cudaMemcpyDeviceToHost, s));
    if (rev.nnz) {
        DBuf<int64_t> c(rev.nnz, s), ww(rev.nnz, s);
        GD_KERNEL(k_export_seg, grid_for(rev.nnz, 256), 256, 0, s, rev.col.get(), rev.w.n ? rev.w.get() : nullptr,
                  rev.nnz, c.get(), ww.get());
        GD_CUDA(cudaMemcpyAsync(src, c.get(), rev.nnz * 8, cudaMemcpyDeviceToHost, s));
        if (w) GD_CUDA(cudaMemcpyAsync(w, ww.get(), rev.nnz * 8, cudaMemcpyDeviceToHost, s));
        GD_CUDA(cudaStreamSynchronize(s));
    }
    GD_CUDA(cudaStreamSynchronize(s));
}

}  // namespace gdb
