// gd_launch.cuh -- kernel launch accounting and optional per-kernel event timing.
#pragma once

#include <cuda_runtime.h>

#include <map>
#include <string>
#include <vector>

#include "gd_common.cuh"

namespace gdb {

void count_launch();          // one of our own kernels
void count_library_launch();  // a CUB primitive call (sort / scan / select)
int64_t launches_total();

struct KernelStat {
    double ms = 0;
    int64_t launches = 0;
    int64_t bytes = 0;
};

// Per-kernel CUDA-event timing on the launching stream.  Enabled per
// algorithm handle (gd_set_profiling); the handle installs itself as the
// thread's active profiler for the duration of an API call.
struct KernelProf {
    bool on = false;
    struct Rec {
        const char* name;
        cudaEvent_t a, b;
        int64_t bytes;
        int64_t tag;    // >= 0: queued sweep index (see drop_sweeps_from)
        int64_t seq;    // the batch (reset_last call) it belongs to
        bool drop;      // a queued sweep that ran as a device no-op
    };
    // Records are folded lazily -- when stats are queried, or at a batch
    // start once many are pending -- so a timed loop pays only for the event
    // records themselves, not for syncs and elapsed-time queries per batch.
    std::vector<Rec> pending;
    int64_t seq = 0;
    std::map<std::string, KernelStat> last;   // stats of the latest batch
    std::map<std::string, KernelStat> total;  // since profiling was switched on
    void reset_last();                        // a batch starts
    void flush();                             // fold the pending records
    void drop_sweeps_from(int64_t limit);     // this batch's records of queued sweeps >= limit
    std::vector<cudaEvent_t> pool;            // recycled events
    cudaEvent_t event();
    ~KernelProf();
};

extern thread_local KernelProf* tl_prof;

struct ProfScope {
    KernelProf* prev;
    explicit ProfScope(KernelProf* p) : prev(tl_prof) { tl_prof = p; }
    ~ProfScope() { tl_prof = prev; }
};

int prof_begin(const char* name, int64_t bytes, cudaStream_t s);
// marks a recorded launch as part of queued sweep `tag` (dropped at flush
// when the sweep turned out to be a device no-op)
void prof_tag(int idx, int64_t tag);
void prof_end(int idx, cudaStream_t s);
// algorithmic bytes of a recorded launch, when known only after it ran
void prof_set_bytes(int idx, int64_t bytes);

}  // namespace gdb

#define GD_KERNEL(kern, grid, block, smem, stream, ...)           \
    do {                                                          \
        kern<<<(grid), (block), (smem), (stream)>>>(__VA_ARGS__); \
        ::gdb::count_launch();                                    \
        GD_LAUNCH_CHECK();                                        \
    } while (0)

#define GD_KERNEL_T(name, bytes, kern, grid, block, smem, stream, ...)  \
    do {                                                                \
        int _pi = ::gdb::prof_begin((name), (bytes), (stream));         \
        kern<<<(grid), (block), (smem), (stream)>>>(__VA_ARGS__);       \
        ::gdb::count_launch();                                          \
        GD_LAUNCH_CHECK();                                              \
        ::gdb::prof_end(_pi, (stream));                                 \
    } while (0)
