// gd_prims.cu -- device memory (a per-stream cache over the stream-ordered
// pool), small read-backs, fills, and the sort / scan / select primitives of
// the store path: CUB by default, or the hand-written cooperative versions of
// gd_sort.cu with -DGD_OWN_PRIMS=1.
#include <atomic>
#include <chrono>
#include <cstring>
#include <map>
#include <mutex>
#include <vector>

#ifndef GD_OWN_PRIMS
#define GD_OWN_PRIMS 0
#endif
#if !GD_OWN_PRIMS
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>
#endif

#include "gd_common.cuh"
#include "gd_launch.cuh"

namespace gdb {


namespace {
struct DevCache {
    std::mutex mu;
    std::map<std::pair<cudaStream_t, size_t>, std::vector<void*>> free;
};
DevCache& dev_cache() {
    static DevCache* c = new DevCache;  // never destroyed: blocks outlive static teardown order
    return *c;
}
size_t size_class(size_t bytes) {
    if (bytes <= 4096) return 4096;
    size_t k = 63 - __builtin_clzll(bytes - 1);  // 2^k < bytes <= 2^(k+1)
    size_t step = (size_t(1) << k) / 8;
    return ((bytes + step - 1) / step) * step;
}
}  // namespace

// Blocks up to kCacheMax are cached per (stream, size class) so the per-batch
// temporaries skip the pool's host-side bookkeeping; a block is only handed
// out again on the stream it was freed on, so stream order keeps it safe.
// Larger blocks (the store's arrays) go straight to the stream-ordered pool at
// their exact size.
constexpr size_t kCacheMax = size_t(64) << 20;

void* dev_alloc(size_t bytes, cudaStream_t s) {
    const bool cached = bytes <= kCacheMax;
    const size_t c = cached ? size_class(bytes) : bytes;
    DevCache& dc = dev_cache();
    if (cached) {
        std::lock_guard<std::mutex> lk(dc.mu);
        auto it = dc.free.find({s, c});
        if (it != dc.free.end() && !it->second.empty()) {
            void* p = it->second.back();
            it->second.pop_back();
            return p;
        }
    }
    void* p = nullptr;
    cudaError_t e = cudaMallocAsync(&p, c, s);
    if (e == cudaErrorMemoryAllocation) {  // hand every cached block back to the pool, retry once
        cudaGetLastError();
        dev_cache_release(nullptr, true);
        GD_CUDA(cudaDeviceSynchronize());
        e = cudaMallocAsync(&p, c, s);
    }
    GD_CUDA(e);
    return p;
}

void dev_free(void* p, size_t bytes, cudaStream_t s) {
    if (bytes > kCacheMax) {
        GD_CUDA(cudaFreeAsync(p, s));
        return;
    }
    DevCache& dc = dev_cache();
    std::lock_guard<std::mutex> lk(dc.mu);
    dc.free[{s, size_class(bytes)}].push_back(p);
}

void dev_cache_release(cudaStream_t s, bool all) {
    DevCache& dc = dev_cache();
    std::lock_guard<std::mutex> lk(dc.mu);
    for (auto it = dc.free.begin(); it != dc.free.end();) {
        if (all || it->first.first == s) {
            for (void* p : it->second) cudaFreeAsync(p, it->first.first);
            it = dc.free.erase(it);
        } else {
            ++it;
        }
    }
}

namespace {
// byte copy by the SMs: 16-byte vectors when both ends allow it
__global__ void k_copy_bytes(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst, size_t n) {
    const size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x, stride = (size_t)gridDim.x * blockDim.x;
    if ((((uintptr_t)src | (uintptr_t)dst) & 15) == 0) {
        const size_t nv = n / 16;
        const int4* s4 = reinterpret_cast<const int4*>(src);
        int4* d4 = reinterpret_cast<int4*>(dst);
        for (size_t i = t; i < nv; i += stride) d4[i] = s4[i];
        for (size_t i = nv * 16 + t; i < n; i += stride) dst[i] = src[i];
    } else {
        for (size_t i = t; i < n; i += stride) dst[i] = src[i];
    }
}
}  // namespace

namespace {
__global__ void k_fill_bytes(uint8_t* __restrict__ dst, int v, size_t n) {
    const size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x, stride = (size_t)gridDim.x * blockDim.x;
    const uint8_t b = (uint8_t)v;
    if (((uintptr_t)dst & 15) == 0) {
        const uint32_t w = 0x01010101u * b;
        const int4 q = make_int4((int)w, (int)w, (int)w, (int)w);
        const size_t nv = n / 16;
        int4* d4 = reinterpret_cast<int4*>(dst);
        for (size_t i = t; i < nv; i += stride) d4[i] = q;
        for (size_t i = nv * 16 + t; i < n; i += stride) dst[i] = b;
    } else {
        for (size_t i = t; i < n; i += stride) dst[i] = b;
    }
}

}  // namespace

// cudaMemsetAsync's replacement on the batch path (a kernel, for the reason below)
void fill_d(cudaStream_t s, void* dst, int v, size_t bytes) {
    if (!bytes) return;
    static const bool ce = getenv("GD_COPY_ENGINE") != nullptr;  // A/B: the copy-engine memset
    if (ce) {
        GD_CUDA(cudaMemsetAsync(dst, v, bytes, s));
        return;
    }
    const unsigned g = (unsigned)std::min<size_t>((bytes / 16 + 255) / 256 + 1, 148 * 16);
    k_fill_bytes<<<g, 256, 0, s>>>(static_cast<uint8_t*>(dst), v, bytes);
    count_launch();
    GD_LAUNCH_CHECK();
}

// Device-to-device copies on the store path go through the SMs, not a copy
// engine: a copy engine serves its queue in order, so a small copy would
// wait behind a result read-back (tens of MB) that another stream has
// queued in the same direction (tools/e2e_probe2.py).
void copy_d2d(cudaStream_t s, void* dst, const void* src, size_t bytes) {
    if (!bytes) return;
    static const bool ce = getenv("GD_COPY_ENGINE") != nullptr;
    if (ce) {
        GD_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, s));
        return;
    }
    const unsigned g = (unsigned)std::min<size_t>((bytes / 16 + 255) / 256 + 1, 148 * 16);
    k_copy_bytes<<<g, 256, 0, s>>>(static_cast<const uint8_t*>(src), static_cast<uint8_t*>(dst), bytes);
    count_launch();
    GD_LAUNCH_CHECK();
}

namespace {
// copy `bytes` into mapped host memory, then publish `seq` in the flag word
// behind a system fence: the host sees the flag only after the data
__global__ void k_read_small(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst, size_t n,
                             volatile uint32_t* flag, uint32_t seq) {
    for (size_t i = threadIdx.x; i < n; i += blockDim.x) dst[i] = src[i];
    __syncwarp();
    __threadfence_system();
    if (threadIdx.x == 0) *flag = seq;
}
}  // namespace

// Small reads land in mapped pinned memory written by a kernel, for the
// same reason: a cudaMemcpy D2H would queue behind a concurrent read-back.
// The host then spins on a sequence flag the kernel writes after the data
// instead of waking from cudaStreamSynchronize (a device gap of ~20 us per
// read-back in tools/timeline_host.py); after 2 s it falls back to the sync,
// which also surfaces any error of the work queued before.
void read_small(cudaStream_t s, void* host, const void* dev, size_t bytes) {
    constexpr size_t kCap = 4096;
    static thread_local uint8_t* pin = nullptr;
    static thread_local void* dpin = nullptr;
    static thread_local uint32_t seq = 0;
    if (bytes > kCap) {
        GD_CUDA(cudaMemcpyAsync(host, dev, bytes, cudaMemcpyDeviceToHost, s));
        GD_CUDA(cudaStreamSynchronize(s));
        return;
    }
    if (!pin) {
        void* p = nullptr;
        GD_CUDA(cudaHostAlloc(&p, kCap + 64, cudaHostAllocMapped | cudaHostAllocPortable));
        GD_CUDA(cudaHostGetDevicePointer(&dpin, p, 0));
        pin = static_cast<uint8_t*>(p);
        *reinterpret_cast<volatile uint32_t*>(pin + kCap) = 0;
    }
    volatile uint32_t* flag = reinterpret_cast<volatile uint32_t*>(pin + kCap);
    const uint32_t want = ++seq ? seq : ++seq;  // never 0, the initial flag
    k_read_small<<<1, 32, 0, s>>>(static_cast<const uint8_t*>(dev), static_cast<uint8_t*>(dpin), bytes,
                                  reinterpret_cast<volatile uint32_t*>(static_cast<uint8_t*>(dpin) + kCap), want);
    count_launch();
    GD_LAUNCH_CHECK();
    static const bool sync_reads = getenv("GD_READ_SYNC") != nullptr;  // A/B: wake from cudaStreamSynchronize
    if (sync_reads) GD_CUDA(cudaStreamSynchronize(s));
    const auto t0 = std::chrono::steady_clock::now();
    for (uint32_t spin = 0; *flag != want; ++spin) {
        if ((spin & 1023) == 1023 && std::chrono::steady_clock::now() - t0 > std::chrono::seconds(2)) {
            GD_CUDA(cudaStreamSynchronize(s));
            if (*flag != want) throw GdError(GD_ERR_CUDA, "read_small: the device never published the value");
            break;
        }
    }
    std::atomic_thread_fence(std::memory_order_acquire);
    memcpy(host, pin, bytes);
}

#if !GD_OWN_PRIMS
// The store path's sort / scan / select through CUB (the default: measured
// faster than the hand-written cooperative versions in gd_sort.cu,
// profiles/round2/README.md).
namespace {
struct Temp {
    void* p = nullptr;
    size_t bytes = 0;
    cudaStream_t s;
    Temp(size_t b, cudaStream_t st) : bytes(b), s(st) {
        if (b) p = dev_alloc(b, st);
    }
    ~Temp() {
        if (p) dev_free(p, bytes, s);
    }
};
}  // namespace

void sort_pairs_u64(cudaStream_t s, uint64_t* keys, int32_t* vals, int64_t n, int end_bit) {
    if (n <= 1) return;
    DBuf<uint64_t> k2(n, s);
    DBuf<int32_t> v2(n, s);
    cub::DoubleBuffer<uint64_t> kb(keys, k2.get());
    cub::DoubleBuffer<int32_t> vb(vals, v2.get());
    size_t bytes = 0;
    GD_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, kb, vb, n, 0, end_bit, s));
    Temp t(bytes, s);
    GD_CUDA(cub::DeviceRadixSort::SortPairs(t.p, bytes, kb, vb, n, 0, end_bit, s));
    count_library_launch();
    if (kb.Current() != keys) copy_d2d(s, keys, kb.Current(), n * sizeof(uint64_t));
    if (vb.Current() != vals) copy_d2d(s, vals, vb.Current(), n * sizeof(int32_t));
}

void sort_pairs_u32(cudaStream_t s, uint32_t* keys, int32_t* vals, int64_t n, int end_bit) {
    if (n <= 1) return;
    DBuf<uint32_t> k2(n, s);
    DBuf<int32_t> v2(n, s);
    cub::DoubleBuffer<uint32_t> kb(keys, k2.get());
    cub::DoubleBuffer<int32_t> vb(vals, v2.get());
    size_t bytes = 0;
    GD_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, kb, vb, n, 0, end_bit, s));
    Temp t(bytes, s);
    GD_CUDA(cub::DeviceRadixSort::SortPairs(t.p, bytes, kb, vb, n, 0, end_bit, s));
    count_library_launch();
    if (kb.Current() != keys) copy_d2d(s, keys, kb.Current(), n * sizeof(uint32_t));
    if (vb.Current() != vals) copy_d2d(s, vals, vb.Current(), n * sizeof(int32_t));
}

void sort_keys_u64(cudaStream_t s, uint64_t* keys, int64_t n, int end_bit) {
    if (n <= 1) return;
    DBuf<uint64_t> k2(n, s);
    cub::DoubleBuffer<uint64_t> kb(keys, k2.get());
    size_t bytes = 0;
    GD_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, bytes, kb, n, 0, end_bit, s));
    Temp t(bytes, s);
    GD_CUDA(cub::DeviceRadixSort::SortKeys(t.p, bytes, kb, n, 0, end_bit, s));
    count_library_launch();
    if (kb.Current() != keys) copy_d2d(s, keys, kb.Current(), n * sizeof(uint64_t));
}

void exclusive_scan_i64(cudaStream_t s, const int64_t* in, int64_t* out, int64_t n) {
    if (n <= 0) return;
    size_t bytes = 0;
    GD_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, in, out, n, s));
    Temp t(bytes, s);
    GD_CUDA(cub::DeviceScan::ExclusiveSum(t.p, bytes, in, out, n, s));
    count_library_launch();
}

void inclusive_scan_i64(cudaStream_t s, const int64_t* in, int64_t* out, int64_t n) {
    if (n <= 0) return;
    size_t bytes = 0;
    GD_CUDA(cub::DeviceScan::InclusiveSum(nullptr, bytes, in, out, n, s));
    Temp t(bytes, s);
    GD_CUDA(cub::DeviceScan::InclusiveSum(t.p, bytes, in, out, n, s));
    count_library_launch();
}

int64_t select_flagged_index(cudaStream_t s, const uint8_t* flags, int64_t n, int32_t* out) {
    if (n <= 0) return 0;
    DBuf<int64_t> cnt(1, s);
    thrust::counting_iterator<int32_t> it(0);
    size_t bytes = 0;
    GD_CUDA(cub::DeviceSelect::Flagged(nullptr, bytes, it, flags, out, cnt.get(), n, s));
    Temp t(bytes, s);
    GD_CUDA(cub::DeviceSelect::Flagged(t.p, bytes, it, flags, out, cnt.get(), n, s));
    count_library_launch();
    return read_scalar(s, cnt.get());
}

void select_flagged_index_async(cudaStream_t s, const uint8_t* flags, int64_t n, int32_t* out, int64_t* d_count) {
    if (n <= 0) {
        fill_d(s, d_count, 0, sizeof(int64_t));
        return;
    }
    thrust::counting_iterator<int32_t> it(0);
    size_t bytes = 0;
    GD_CUDA(cub::DeviceSelect::Flagged(nullptr, bytes, it, flags, out, d_count, n, s));
    Temp t(bytes, s);
    GD_CUDA(cub::DeviceSelect::Flagged(t.p, bytes, it, flags, out, d_count, n, s));
    count_library_launch();
}

#endif  // !GD_OWN_PRIMS

__global__ void k_iota_i32(int32_t* a, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        a[i] = static_cast<int32_t>(i);
}
__global__ void k_fill_i64(int64_t* a, int64_t n, int64_t v) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        a[i] = v;
}
__global__ void k_fill_i32(int32_t* a, int64_t n, int32_t v) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        a[i] = v;
}

void iota_i32(cudaStream_t s, int32_t* a, int64_t n) {
    if (n > 0) GD_KERNEL(k_iota_i32, grid_for(n, 256), 256, 0, s, a, n);
}
void fill_i64(cudaStream_t s, int64_t* a, int64_t n, int64_t v) {
    if (n > 0) GD_KERNEL(k_fill_i64, grid_for(n, 256), 256, 0, s, a, n, v);
}
void fill_i32(cudaStream_t s, int32_t* a, int64_t n, int32_t v) {
    if (n > 0) GD_KERNEL(k_fill_i32, grid_for(n, 256), 256, 0, s, a, n, v);
}

}  // namespace gdb
