// gd_common.cuh -- shared device types, error plumbing and primitives for the
// B200 dynamic-graph path (sm_100a only).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/gd_capi.h"

namespace gdb {

// Device vertex ids are int32 (scale-26 = 67.1M < 2^31), offsets int64,
// weights int32.  A deleted out-slot holds kSentinel (-1); it is exported as
// INT64_MAX, the reference's SENTINEL (csr.py:14).
constexpr int32_t kSentinel = -1;
constexpr int64_t kInf = INT64_MAX;  // properties.py:20 INT_INF
constexpr int kWarp = 32;
constexpr int kSMs = 148;

// Error carried from the device path to the C ABI (gd_capi.cu maps it to a
// status code and gd_last_error()).
struct GdError : std::runtime_error {
    int code;
    GdError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define GD_CUDA(call)                                                                               \
    do {                                                                                            \
        cudaError_t _e = (call);                                                                    \
        if (_e != cudaSuccess)                                                                      \
            throw ::gdb::GdError(GD_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(_e) + \
                                                  " (" __FILE__ ":" + std::to_string(__LINE__) + ")"); \
    } while (0)

#define GD_LAUNCH_CHECK() GD_CUDA(cudaGetLastError())

// Stream-ordered device memory with a per-stream cache of freed blocks in
// size classes (2^k in 8 steps).  A batch allocates and frees ~100 temporaries;
// cudaMallocAsync / cudaFreeAsync for each cost host time that the GPU then
// waits on.  A block is reused only on the stream it was freed on, so stream
// order protects it.
void* dev_alloc(size_t bytes, cudaStream_t s);
void dev_free(void* p, size_t bytes, cudaStream_t s);
void dev_cache_release(cudaStream_t s, bool all = false);  // return a stream's cached blocks (before destroying it)

// memset by a kernel (gd_prims.cu): copy-engine memsets queue behind read-backs too
void fill_d(cudaStream_t s, void* dst, int v, size_t bytes);

template <typename T>
struct DBuf {
    T* p = nullptr;
    size_t n = 0;
    cudaStream_t s = nullptr;
    DBuf() = default;
    DBuf(size_t count, cudaStream_t st) { alloc(count, st); }
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    DBuf(DBuf&& o) noexcept : p(o.p), n(o.n), s(o.s) {
        o.p = nullptr;
        o.n = 0;
    }
    DBuf& operator=(DBuf&& o) noexcept {
        if (this != &o) {
            release();
            p = o.p;
            n = o.n;
            s = o.s;
            o.p = nullptr;
            o.n = 0;
        }
        return *this;
    }
    ~DBuf() { release(); }
    void alloc(size_t count, cudaStream_t st) {
        release();
        s = st;
        n = count;
        if (count) p = static_cast<T*>(dev_alloc(count * sizeof(T), st));
    }
    // grow-only reuse: keeps the allocation when large enough
    void ensure(size_t count, cudaStream_t st) {
        if (count > n || p == nullptr) alloc(count ? count : 1, st);
    }
    void release() {
        if (p) dev_free(p, n * sizeof(T), s);
        p = nullptr;
        n = 0;
    }
    T* get() const { return p; }
    void zero(cudaStream_t st) const {
        if (n) fill_d(st, p, 0, n * sizeof(T));
    }
};

inline unsigned grid_for(int64_t items, int block, int64_t cap = 148LL * 64) {
    int64_t g = (items + block - 1) / block;
    if (g < 1) g = 1;
    if (g > cap) g = cap;
    return static_cast<unsigned>(g);
}

__host__ __device__ inline int64_t sat_add(int64_t a, int64_t b) {  // graphdyn_rt.h:40-44
    return (a >= kInf || b >= kInf) ? kInf : a + b;
}

// In-index tombstone: the entry keeps its (decodable) column so rows stay
// sorted for binary search; tomb(c) = ~c is negative.
__host__ __device__ inline int32_t tomb(int32_t c) { return ~c; }
__host__ __device__ inline int32_t untomb(int32_t c) { return c < 0 ? ~c : c; }

// Key of a directed pair (row, col): row << sh | col with sh = bits(n - 1),
// so radix sorts run over 2*sh bits only (44 for scale-22 instead of 64).
__host__ __device__ inline uint64_t pair_key(int32_t r, int32_t c, int sh) {
    return (static_cast<uint64_t>(static_cast<uint32_t>(r)) << sh) | static_cast<uint32_t>(c);
}
__host__ __device__ inline int32_t key_row(uint64_t k, int sh) { return static_cast<int32_t>(k >> sh); }
__host__ __device__ inline int32_t key_col(uint64_t k, int sh) {
    return static_cast<int32_t>(k & ((1ULL << sh) - 1));
}
inline int bits_for(uint64_t v) {  // number of bits to represent v (>= 1)
    int b = 1;
    while (b < 64 && (v >> b)) ++b;
    return b;
}

template <typename T>
__device__ inline int64_t lower_bound_dev(const T* a, int64_t lo, int64_t hi, T x) {
    while (lo < hi) {
        int64_t m = (lo + hi) >> 1;
        if (a[m] < x) lo = m + 1;
        else hi = m;
    }
    return lo;
}
template <typename T>
__device__ inline int64_t upper_bound_dev(const T* a, int64_t lo, int64_t hi, T x) {
    while (lo < hi) {
        int64_t m = (lo + hi) >> 1;
        if (a[m] <= x) lo = m + 1;
        else hi = m;
    }
    return lo;
}
// lower/upper bound on in-index columns, decoding tombstones
__device__ inline int64_t col_lower(const int32_t* a, int64_t lo, int64_t hi, int32_t x) {
    while (lo < hi) {
        int64_t m = (lo + hi) >> 1;
        if (untomb(a[m]) < x) lo = m + 1;
        else hi = m;
    }
    return lo;
}
__device__ inline int64_t col_upper(const int32_t* a, int64_t lo, int64_t hi, int32_t x) {
    while (lo < hi) {
        int64_t m = (lo + hi) >> 1;
        if (untomb(a[m]) <= x) lo = m + 1;
        else hi = m;
    }
    return lo;
}

// ---- host-side primitive wrappers (CUB radix sort / scan / select) -----------
// Implemented in gd_prims.cu.
void sort_pairs_u64(cudaStream_t s, uint64_t* keys, int32_t* vals, int64_t n, int end_bit = 64);
void sort_pairs_u32(cudaStream_t s, uint32_t* keys, int32_t* vals, int64_t n, int end_bit = 32);
void sort_keys_u64(cudaStream_t s, uint64_t* keys, int64_t n, int end_bit = 64);
void exclusive_scan_i64(cudaStream_t s, const int64_t* in, int64_t* out, int64_t n);
// Compact indices i in [0, n) with flags[i] != 0 into out (ordered); returns count (sync).
int64_t select_flagged_index(cudaStream_t s, const uint8_t* flags, int64_t n, int32_t* out);
// Same, count left in device memory (no sync).
void select_flagged_index_async(cudaStream_t s, const uint8_t* flags, int64_t n, int32_t* out, int64_t* d_count);
void iota_i32(cudaStream_t s, int32_t* a, int64_t n);
void fill_i64(cudaStream_t s, int64_t* a, int64_t n, int64_t v);
void fill_i32(cudaStream_t s, int32_t* a, int64_t n, int32_t v);
// Small device -> host reads (counts, flags) through a per-thread pinned
// staging buffer: a pageable destination costs an extra staged copy and
// several microseconds of latency at every such sync point.
void read_small(cudaStream_t s, void* host, const void* dev, size_t bytes);
// device-to-device copy by a kernel (gd_prims.cu)
void copy_d2d(cudaStream_t s, void* dst, const void* src, size_t bytes);


template <typename T>
inline T read_scalar(cudaStream_t s, const T* dptr) {
    T h{};
    read_small(s, &h, dptr, sizeof(T));
    return h;
}

// Phase timer with CUDA events on the handle's stream.  Phase names follow
// the reference's ExecContext.add_phase (interp.py:141-145).
enum Phase { PH_STATIC = 0, PH_PRE = 1, PH_STRUCT = 2, PH_PROP = 3, PH_MERGE = 4, PH_COUNT = 5 };

struct PhaseTimer {
    cudaStream_t s = nullptr;
    std::vector<cudaEvent_t> evs, pool;  // pool: recycled events (no create/destroy per phase)
    std::vector<int> phases;
    double total_ms[PH_COUNT] = {0, 0, 0, 0, 0};
    int open = -1;
    cudaEvent_t event() {
        if (!pool.empty()) {
            cudaEvent_t e = pool.back();
            pool.pop_back();
            return e;
        }
        cudaEvent_t e;
        GD_CUDA(cudaEventCreate(&e));
        return e;
    }
    void begin(int ph) {
        cudaEvent_t e = event();
        GD_CUDA(cudaEventRecord(e, s));
        evs.push_back(e);
        phases.push_back(ph);
    }
    // Called at a sync point: turn consecutive event pairs into phase times.
    void end_all() {
        cudaEvent_t e = event();
        GD_CUDA(cudaEventRecord(e, s));
        evs.push_back(e);
        phases.push_back(-1);
        GD_CUDA(cudaEventSynchronize(e));
        for (size_t i = 0; i + 1 < evs.size(); ++i) {
            float ms = 0;
            GD_CUDA(cudaEventElapsedTime(&ms, evs[i], evs[i + 1]));
            if (phases[i] >= 0) total_ms[phases[i]] += ms;
        }
        pool.insert(pool.end(), evs.begin(), evs.end());
        evs.clear();
        phases.clear();
    }
    ~PhaseTimer() {
        for (auto ev : evs) cudaEventDestroy(ev);
        for (auto ev : pool) cudaEventDestroy(ev);
    }
};

}  // namespace gdb
