// gd_prims.cu -- device memory (a per-stream cache over the stream-ordered
// pool), small read-backs and fills.  The sort / scan / select primitives are
// in gd_sort.cu.
#include <cstring>
#include <map>
#include <mutex>
#include <vector>

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

void read_small(cudaStream_t s, void* host, const void* dev, size_t bytes) {
    constexpr size_t kCap = 4096;
    static thread_local void* pin = nullptr;
    if (bytes > kCap) {
        GD_CUDA(cudaMemcpyAsync(host, dev, bytes, cudaMemcpyDeviceToHost, s));
        GD_CUDA(cudaStreamSynchronize(s));
        return;
    }
    if (!pin) GD_CUDA(cudaMallocHost(&pin, kCap));
    GD_CUDA(cudaMemcpyAsync(pin, dev, bytes, cudaMemcpyDeviceToHost, s));
    GD_CUDA(cudaStreamSynchronize(s));
    memcpy(host, pin, bytes);
}

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
