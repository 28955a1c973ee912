// gd_sort.cu -- the device-wide primitives of the store path, hand-written for
// sm_100a: a stable LSD radix sort (u32 / u64 keys, optional int32 values),
// an exclusive scan (int64) and a flagged-index select.  Each is ONE
// cooperative launch: persistent CTAs own contiguous chunks of the input and
// meet at grid barriers between phases, so a pass costs two or three barriers
// instead of several kernel launches -- the batch-sized inputs of the store
// (10^5 .. 10^7 items) are latency-, not bandwidth-bound.
//
// Radix sort, per 8-bit digit pass:
//   1. every CTA histograms its chunk (shared-memory atomics) into
//      table[digit][cta];
//   2. the CTAs scan the table's rows (one digit row per CTA, grid-strided)
//      in place and write the row totals; every CTA then prefixes the
//      256 totals itself -- offset(d, c) = prefix(d) + table[d][c];
//   3. every CTA re-reads its chunk in rounds of 256 x kItems keys: each warp
//      ranks its contiguous 32 x kItems keys sequentially (match_any per
//      item, a per-warp running count per digit), the warps' counts are
//      prefixed per digit across the CTA, and each key goes to
//      offset(d, c) + running(d) + its rank: the order of equal digits is the
//      input order, so the sort is stable (the store's slot semantics rely on
//      it: dynamic.py:116 keeps stream order within a source).
// Passes stop at end_bit; keys and values ping-pong between the caller's
// arrays and one scratch pair, with a final copy when the pass count is odd.
//
// Built with -DGD_OWN_PRIMS=1 only: on the C2 batch (B200, tools/timeline.py)
// these take 406 us for the two 44-bit sorts (CUB onesweep: 171), 150 us for
// six 4M-entry scans (CUB: 78) and 45 us for five selects (CUB: 32), so the
// default build keeps CUB (gd_prims.cu); see profiles/round2/README.md.
#include <cooperative_groups.h>

#include <algorithm>

#include "gd_common.cuh"
#include "gd_launch.cuh"

#ifndef GD_OWN_PRIMS
#define GD_OWN_PRIMS 0
#endif

#if GD_OWN_PRIMS
namespace gdb {

namespace {

namespace cg = cooperative_groups;

constexpr int kSortThreads = 256;
constexpr int kWarps = kSortThreads / 32;
constexpr int kRadix = 256;
constexpr int kItems = 8;  // keys per thread per round
constexpr int kRound = kSortThreads * kItems;
static_assert(kSortThreads == kRadix, "one digit per thread in the totals prefix");

template <typename K>
struct SortArgs {
    K* key[2];
    int32_t* val[2];  // nullptr: keys only
    int64_t n;
    int64_t chunk;  // keys per CTA (a multiple of kRound)
    int begin_bit, end_bit;
    unsigned long long* table;  // [kRadix][grid]
};

template <typename K>
__device__ __forceinline__ int digit_of(K k, int shift) {
    return (int)((k >> shift) & (K)(kRadix - 1));
}

template <typename K>
__global__ void __launch_bounds__(kSortThreads) k_radix_sort(SortArgs<K> a) {
    cg::grid_group grid = cg::this_grid();
    __shared__ unsigned long long hist[kRadix];
    __shared__ unsigned long long base[kRadix];   // global offset + running count per digit
    __shared__ int wcnt[kWarps][kRadix + 1];      // per-warp counts of the round, then their prefix
    __shared__ unsigned long long prefix[kRadix];  // exclusive prefix of the digit totals
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int G = gridDim.x, c = blockIdx.x;
    const int64_t lo = min(a.n, (int64_t)c * a.chunk), hi = min(a.n, lo + a.chunk);
    int cur = 0;
    for (int shift = a.begin_bit; shift < a.end_bit; shift += 8) {
        const K* kin = a.key[cur];
        const int32_t* vin = a.val[cur];
        K* kout = a.key[cur ^ 1];
        int32_t* vout = a.val[cur ^ 1];
        // 1. histogram of this CTA's chunk
        for (int d = tid; d < kRadix; d += kSortThreads) hist[d] = 0;
        __syncthreads();
        for (int64_t i = lo + tid; i < hi; i += kSortThreads) atomicAdd(&hist[digit_of(kin[i], shift)], 1ULL);
        __syncthreads();
        for (int d = tid; d < kRadix; d += kSortThreads) a.table[(int64_t)d * G + c] = hist[d];
        grid.sync();
        // 2. scan each digit's row over the CTAs (row d by CTA d mod G), then
        //    every CTA prefixes the row totals (kept in the row's last slot +1
        //    region: totals live after the table)
        unsigned long long* totals = a.table + (int64_t)kRadix * G;
        for (int d = c; d < kRadix; d += G) {
            unsigned long long* row = a.table + (int64_t)d * G;
            // block-wide exclusive scan of G entries in chunks of kSortThreads
            unsigned long long carry = 0;
            for (int j0 = 0; j0 < G; j0 += kSortThreads) {
                const int j = j0 + tid;
                unsigned long long v = j < G ? row[j] : 0;
                // warp inclusive scan
                unsigned long long x = v;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
                    if (lane >= o) x += y;
                }
                __shared__ unsigned long long wsum[kWarps];
                if (lane == 31) wsum[wid] = x;
                __syncthreads();
                unsigned long long wpre = 0, tot = 0;
                for (int w = 0; w < kWarps; ++w) {
                    if (w < wid) wpre += wsum[w];
                    tot += wsum[w];
                }
                if (j < G) row[j] = carry + wpre + x - v;
                carry += tot;
                __syncthreads();
            }
            if (tid == 0) totals[d] = carry;
        }
        grid.sync();
        {  // exclusive prefix of the 256 digit totals, one per thread (kSortThreads == kRadix)
            const unsigned long long v = totals[tid];
            unsigned long long x = v;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
                if (lane >= o) x += y;
            }
            if (lane == 31) hist[wid] = x;  // hist is free until the next pass
            __syncthreads();
            unsigned long long wpre = 0;
            for (int w = 0; w < wid; ++w) wpre += hist[w];
            prefix[tid] = wpre + x - v;
        }
        __syncthreads();
        for (int d = tid; d < kRadix; d += kSortThreads) base[d] = prefix[d] + a.table[(int64_t)d * G + c];
        for (int d = tid; d < kRadix; d += kSortThreads)
            for (int w = 0; w < kWarps; ++w) wcnt[w][d] = 0;
        __syncthreads();
        // 3. stable scatter, rounds of kRound keys; warp w ranks keys
        //    [r + w*32*kItems, r + (w+1)*32*kItems), item-major then lane
        for (int64_t r = lo; r < hi; r += kRound) {
            const int64_t wb = r + (int64_t)wid * 32 * kItems;
            K kk[kItems];
            int32_t vv[kItems];
            int dg[kItems], rk[kItems];
#pragma unroll
            for (int j = 0; j < kItems; ++j) {
                const int64_t i = wb + j * 32 + lane;
                const bool ok = i < hi;
                kk[j] = ok ? kin[i] : (K)0;
                if (vin) vv[j] = ok ? vin[i] : 0;
                dg[j] = ok ? digit_of(kk[j], shift) : kRadix;  // out of range: its own group, never written
            }
#pragma unroll
            for (int j = 0; j < kItems; ++j) {
                const unsigned peers = __match_any_sync(0xffffffffu, dg[j]);
                const int leader = __ffs(peers) - 1;
                const int before = __popc(peers & ((1u << lane) - 1));
                int run = 0;
                if (lane == leader) run = wcnt[wid][dg[j]];
                run = __shfl_sync(0xffffffffu, run, leader);
                rk[j] = run + before;
                __syncwarp();
                if (lane == leader) wcnt[wid][dg[j]] = run + __popc(peers);
                __syncwarp();
            }
            __syncthreads();
            // per digit: exclusive prefix of the warps' counts, the round total
            for (int d = tid; d < kRadix; d += kSortThreads) {
                int acc = 0;
                for (int w = 0; w < kWarps; ++w) {
                    const int x = wcnt[w][d];
                    wcnt[w][d] = acc;
                    acc += x;
                }
                hist[d] = (unsigned long long)acc;  // round total, reused as scratch
            }
            __syncthreads();
#pragma unroll
            for (int j = 0; j < kItems; ++j) {
                if (dg[j] >= kRadix) continue;
                const unsigned long long pos = base[dg[j]] + (unsigned long long)(wcnt[wid][dg[j]] + rk[j]);
                kout[pos] = kk[j];
                if (vin) vout[pos] = vv[j];
            }
            __syncthreads();
            for (int d = tid; d < kRadix; d += kSortThreads) {
                base[d] += hist[d];
                for (int w = 0; w < kWarps; ++w) wcnt[w][d] = 0;
            }
            __syncthreads();
        }
        grid.sync();
        cur ^= 1;
    }
}

// co-resident grid of a cooperative kernel (at most `per` CTAs per SM)
template <typename F>
int coop_grid_of(F kernel, int threads, int per) {
    int dev = 0, sms = 0, nb = 0;
    GD_CUDA(cudaGetDevice(&dev));
    GD_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    GD_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kernel, threads, 0));
    if (nb < 1) throw GdError(GD_ERR_CUDA, "cooperative primitive cannot be resident");
    return sms * std::min(nb, per);
}

template <typename K>
void radix_sort(cudaStream_t s, K* keys, int32_t* vals, int64_t n, int end_bit) {
    if (n <= 1) return;
    end_bit = std::min<int>(end_bit, (int)(8 * sizeof(K)));
    if (end_bit <= 0) return;
    static const int gmax = coop_grid_of(k_radix_sort<K>, kSortThreads, 2);
    // enough rounds per CTA to amortise the barriers, never more CTAs than rounds
    const int64_t rounds = (n + kRound - 1) / kRound;
    const int G = (int)std::max<int64_t>(1, std::min<int64_t>(gmax, (rounds + 1) / 2));
    DBuf<K> k2(n, s);
    DBuf<int32_t> v2(vals ? n : 0, s);
    DBuf<unsigned long long> table((size_t)kRadix * G + kRadix, s);
    SortArgs<K> a;
    a.key[0] = keys;
    a.key[1] = k2.get();
    a.val[0] = vals;
    a.val[1] = vals ? v2.get() : nullptr;
    a.n = n;
    const int64_t per = (rounds + G - 1) / G;
    a.chunk = per * kRound;
    a.begin_bit = 0;
    a.end_bit = end_bit;
    a.table = table.get();
    void* args[] = {&a};
    GD_CUDA(cudaLaunchCooperativeKernel((const void*)k_radix_sort<K>, G, kSortThreads, args, 0, s));
    count_launch();
    const int passes = (end_bit + 7) / 8;
    if (passes & 1) {  // the result sits in the scratch pair
        GD_CUDA(cudaMemcpyAsync(keys, k2.get(), n * sizeof(K), cudaMemcpyDeviceToDevice, s));
        if (vals) GD_CUDA(cudaMemcpyAsync(vals, v2.get(), n * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
    }
}

// ---------------------------------------------------------------- scan ----
// Exclusive int64 scan: CTA sums of contiguous chunks, a barrier, every CTA
// prefixes the (<= a few hundred) CTA sums itself, then scans its chunk.
constexpr int kScanThreads = 512;
constexpr int kSI = 8;  // items per thread per round (scan, select)

__device__ __forceinline__ int64_t block_excl_scan(int64_t v, int64_t* wsum, int64_t& total) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int64_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int64_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) wsum[wid] = x;
    __syncthreads();
    int64_t pre = 0;
    total = 0;
    for (int w = 0; w < kScanThreads / 32; ++w) {
        if (w < wid) pre += wsum[w];
        total += wsum[w];
    }
    __syncthreads();
    return pre + x - v;
}

__global__ void __launch_bounds__(kScanThreads) k_scan_excl(const int64_t* in, int64_t* out, int64_t n, int64_t chunk,
                                                            int64_t* csum) {
    cg::grid_group grid = cg::this_grid();
    __shared__ int64_t wsum[kScanThreads / 32];
    __shared__ int64_t base;
    const int c = blockIdx.x, G = gridDim.x;
    const int64_t lo = min(n, (int64_t)c * chunk), hi = min(n, lo + chunk);
    int64_t acc = 0;
    for (int64_t i = lo + threadIdx.x; i < hi; i += kScanThreads) acc += in[i];
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        int64_t t = 0;
        for (int w = 0; w < kScanThreads / 32; ++w) t += wsum[w];
        csum[c] = t;
    }
    grid.sync();
    if (threadIdx.x == 0) {
        int64_t b = 0;
        for (int j = 0; j < c; ++j) b += csum[j];
        base = b;
    }
    (void)G;
    __syncthreads();
    // rounds of kScanThreads x kSI consecutive items: each thread scans its
    // kSI items serially, the block scans the thread totals
    int64_t carry = base;
    for (int64_t i0 = lo; i0 < hi; i0 += (int64_t)kScanThreads * kSI) {
        const int64_t t0 = i0 + (int64_t)threadIdx.x * kSI;
        int64_t v[kSI];
        int64_t sum = 0;
#pragma unroll
        for (int j = 0; j < kSI; ++j) {
            v[j] = t0 + j < hi ? in[t0 + j] : 0;
            sum += v[j];
        }
        int64_t tot;
        int64_t e = carry + block_excl_scan(sum, wsum, tot);
#pragma unroll
        for (int j = 0; j < kSI; ++j) {
            if (t0 + j < hi) out[t0 + j] = e;
            e += v[j];
        }
        carry += tot;
    }
}

// ---------------------------------------------------------------- select ----
// Indices of the flagged entries, in order: CTA counts, a barrier, each CTA
// prefixes the CTA counts and writes its chunk's indices (block scan per
// round).  The total goes to d_count.
__global__ void __launch_bounds__(kScanThreads) k_select(const uint8_t* flags, int64_t n, int64_t chunk, int32_t* out,
                                                         int64_t* csum, int64_t* d_count) {
    cg::grid_group grid = cg::this_grid();
    __shared__ int64_t wsum[kScanThreads / 32];
    __shared__ int64_t base;
    const int c = blockIdx.x, G = gridDim.x;
    const int64_t lo = min(n, (int64_t)c * chunk), hi = min(n, lo + chunk);
    int64_t acc = 0;
    for (int64_t i = lo + threadIdx.x; i < hi; i += kScanThreads) acc += flags[i] != 0;
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        int64_t t = 0;
        for (int w = 0; w < kScanThreads / 32; ++w) t += wsum[w];
        csum[c] = t;
    }
    grid.sync();
    if (threadIdx.x == 0) {
        int64_t b = 0;
        for (int j = 0; j < c; ++j) b += csum[j];
        base = b;
        if (c == G - 1) *d_count = b + csum[c];
    }
    __syncthreads();
    int64_t carry = base;
    for (int64_t i0 = lo; i0 < hi; i0 += (int64_t)kScanThreads * kSI) {
        const int64_t t0 = i0 + (int64_t)threadIdx.x * kSI;
        uint8_t f[kSI];
        int64_t sum = 0;
#pragma unroll
        for (int j = 0; j < kSI; ++j) {
            f[j] = t0 + j < hi ? flags[t0 + j] : 0;
            sum += f[j] != 0;
        }
        int64_t tot;
        int64_t e = carry + block_excl_scan(sum, wsum, tot);
#pragma unroll
        for (int j = 0; j < kSI; ++j)
            if (f[j]) out[e++] = (int32_t)(t0 + j);
        carry += tot;
    }
}

template <typename F>
int coop_grid_for(F kernel, int threads, int64_t n, int64_t min_per_cta) {
    static int dummy = 0;
    (void)dummy;
    const int gmax = coop_grid_of(kernel, threads, 2);
    return (int)std::max<int64_t>(1, std::min<int64_t>(gmax, (n + min_per_cta - 1) / min_per_cta));
}

}  // namespace

void sort_pairs_u64(cudaStream_t s, uint64_t* keys, int32_t* vals, int64_t n, int end_bit) {
    radix_sort<uint64_t>(s, keys, vals, n, end_bit);
}
void sort_pairs_u32(cudaStream_t s, uint32_t* keys, int32_t* vals, int64_t n, int end_bit) {
    radix_sort<uint32_t>(s, keys, vals, n, end_bit);
}
void sort_keys_u64(cudaStream_t s, uint64_t* keys, int64_t n, int end_bit) {
    radix_sort<uint64_t>(s, keys, nullptr, n, end_bit);
}

void exclusive_scan_i64(cudaStream_t s, const int64_t* in, int64_t* out, int64_t n) {
    if (n <= 0) return;
    static const int gmax = coop_grid_of(k_scan_excl, kScanThreads, 2);
    const int G = (int)std::max<int64_t>(1, std::min<int64_t>(gmax, (n + 8 * kScanThreads - 1) / (8 * kScanThreads)));
    const int64_t chunk = (n + G - 1) / G;
    DBuf<int64_t> csum(G, s);
    int64_t* csp = csum.get();
    void* args[] = {(void*)&in, (void*)&out, (void*)&n, (void*)&chunk, (void*)&csp};
    GD_CUDA(cudaLaunchCooperativeKernel((const void*)k_scan_excl, G, kScanThreads, args, 0, s));
    count_launch();
}

void select_flagged_index_async(cudaStream_t s, const uint8_t* flags, int64_t n, int32_t* out, int64_t* d_count) {
    if (n <= 0) {
        fill_d(s, d_count, 0, sizeof(int64_t));
        return;
    }
    static const int gmax = coop_grid_of(k_select, kScanThreads, 2);
    const int G = (int)std::max<int64_t>(1, std::min<int64_t>(gmax, (n + 8 * kScanThreads - 1) / (8 * kScanThreads)));
    const int64_t chunk = (n + G - 1) / G;
    DBuf<int64_t> csum(G, s);
    int64_t* csp = csum.get();
    void* args[] = {(void*)&flags, (void*)&n, (void*)&chunk, (void*)&out, (void*)&csp, (void*)&d_count};
    GD_CUDA(cudaLaunchCooperativeKernel((const void*)k_select, G, kScanThreads, args, 0, s));
    count_launch();
}

int64_t select_flagged_index(cudaStream_t s, const uint8_t* flags, int64_t n, int32_t* out) {
    if (n <= 0) return 0;
    DBuf<int64_t> cnt(1, s);
    select_flagged_index_async(s, flags, n, out, cnt.get());
    return read_scalar(s, cnt.get());
}

}  // namespace gdb
#endif  // GD_OWN_PRIMS
