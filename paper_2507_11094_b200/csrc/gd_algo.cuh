// gd_algo.cuh -- shared machinery of the three dynamic algorithms: batch
// staging/validation, phase timing, kernel profiling, frontier queues and the
// weak-component flood.
#pragma once

#include <functional>
#include <map>
#include <memory>
#include <string>

#include "gd_launch.cuh"
#include "gd_store.cuh"

namespace gdb {

// One batch on the device, split by kind in stream order
// (UpdateBatch.deletes / .adds, graph/updates.py:42-48).
struct DevBatch {
    DBuf<int32_t> ds, dd;      // deletes
    DBuf<int32_t> as, ad, aw;  // adds
    int64_t kdel = 0, kadd = 0;
};

enum AlgoKind { ALGO_SSSP = 1, ALGO_PR = 2, ALGO_TC = 3 };

struct AlgoBase {
    int kind;
    Store* g;
    PhaseTimer timer;
    KernelProf prof;
    int64_t iterations = 0;  // fixedPoint / while iterations, summed
    explicit AlgoBase(int k, Store* st) : kind(k), g(st) { timer.s = st->stream; }
    cudaStream_t stream() const { return g->stream; }

    // Stage host records (int64, 'a'/'d'), validate like _validate_batch
    // (engine/interp.py:563-570) and split by kind.  Throws GdError.
    void stage_host(DevBatch& b, const uint8_t* kind, const int64_t* src, const int64_t* dst, const int64_t* w,
                    int64_t k);
    // Same from device int32 records.
    void stage_device(DevBatch& b, const uint8_t* kind, const int32_t* src, const int32_t* dst, const int32_t* w,
                      int64_t k);

    // Asynchronous result read-back: `snap` bytes are copied on the handle's
    // stream into a device snapshot (so the next batch may overwrite the
    // state at once), then to `host` on a side copy stream that overlaps the
    // next batch.  host is valid after wait_copies() (pinned memory for a
    // real overlap).
    void copy_out_async(void* host, const void* dev, size_t bytes, int slot);
    void wait_copies();
    virtual ~AlgoBase();

    // ---- pipelined host stream (gd_*_run_stream: run_batches over an
    // UpdateStream, engine/run.py:44-68).  Batch j's records are uploaded
    // into slot j % 2 on the copy stream while batch j-1 runs; the copy
    // stream also carries the result read-backs, so each direction's copy
    // runs alone: D2H(j-1) then H2D(j+1), both behind batch j's compute.
    void reserve_uploads(int64_t k);  // both slots sized for k records
    // ids of `width` bytes (8: int64, 4: int32)
    void upload_async(int slot, const uint8_t* kind, const void* src, const void* dst, const void* w, int width,
                      int64_t k);
    // stage_host's second half on an uploaded slot: the handle's stream
    // waits for the upload, then validates and splits (host arrays only feed
    // the error message)
    void stage_uploaded(DevBatch& b, int slot, const uint8_t* h_kind, const void* h_src, const void* h_dst,
                        int64_t k);
    cudaStream_t io_stream();

    // Result read-backs of a run_stream, placed where they cannot stall the
    // batch: stream_result snapshots the batch's result arrays on the
    // handle's stream at once; their D2H is queued on the copy stream only
    // when the NEXT batch has queued its structural update (struct_done),
    // because a copy engine serves its queue in order and the structural
    // update's radix sorts issue copy-engine memsets (CUB) that would wait
    // behind a tens-of-MB read-back.  stream_flush queues a pending one now.
    void stream_result(int par, int narr, const void* const* dev, void* const* host, const size_t* bytes);
    void stream_flush();
    // The next batch's upload is queued at the same point, ahead of the
    // read-back: an H2D copy running under the structural update held up
    // CUB's memsets the same way.
    std::function<void()> pending_upload;
    void struct_done() {
        if (pending_upload) {
            auto f = std::move(pending_upload);
            pending_upload = nullptr;
            f();
        }
        if (has_pend) stream_flush();
    }

  private:
    void split(DevBatch& b, const int32_t* sel_del, const int32_t* sel_add, const int32_t* s, const int32_t* d,
               const int32_t* w, int64_t kdel, int64_t kadd);
    DBuf<int64_t> h_stage;  // reusable device staging for host uploads
    DBuf<uint8_t> k_stage;
    void stage_records(DevBatch& b, const uint8_t* dkind, const void* dsrc, const void* ddst, const void* dw,
                       int width, int64_t k, const uint8_t* h_kind, const void* h_src, const void* h_dst);
    DBuf<int64_t> up64[2];  // run_stream upload slots: src | dst | w
    DBuf<uint8_t> upk[2];
    bool up_w[2] = {false, false};
    int up_width[2] = {8, 8};
    cudaEvent_t ev_up[2] = {nullptr, nullptr}, ev_staged[2] = {nullptr, nullptr};
    DBuf<uint8_t> ssnap[2][2];  // [batch parity][result array]
    cudaEvent_t ev_sready[2] = {nullptr, nullptr}, ev_scopied[2] = {nullptr, nullptr};
    struct Pending {
        int par = 0, narr = 0;
        void* host[2] = {nullptr, nullptr};
        size_t bytes[2] = {0, 0};
    } pend;
    bool has_pend = false;
    cudaStream_t copy_stream = nullptr;
    cudaEvent_t ev_ready[2] = {nullptr, nullptr}, ev_copied[2] = {nullptr, nullptr};
    DBuf<uint8_t> snap[2];
};

// ---- frontier queue ----------------------------------------------------------
struct Frontier {
    DBuf<int32_t> q[2];
    DBuf<unsigned long long> cnt;  // [11]: 3 counter slots + scratch
    int cur = 0;
    void init(int64_t n, cudaStream_t s) {
        q[0].ensure(n + 1, s);
        q[1].ensure(n + 1, s);
        cnt.ensure(11, s);
    }
};

// Weak-component flood of true flags (engine/interp.py:70-109): a vertex ends
// up flagged iff its weak component (over live arcs, either direction)
// contains a flagged vertex.  Computed by union-find over the live out-arcs
// instead of a level-synchronous BFS: same set, no diameter-bound rounds.
// flags is an n-byte device array, updated in place.  Returns the number of
// union-find hooking passes.
int64_t flood_weak_components(Store& g, uint8_t* d_flags, KernelProf* prof);

// The same flood on a vertex-partitioned store (Store::part): union-find
// over the arcs each rank holds (out-arcs of owned sources, in-arcs of owned
// destinations), then rounds of a min-label all-reduce in which every rank
// hooks each vertex under the smallest root any rank knows for it, until no
// rank changes.  The seed flags are the same on every rank (records are
// replicated), and so are the final labels: on return every rank holds the
// whole flooded vector.  Returns the label rounds.
int64_t flood_weak_components_dist(Store& g, uint8_t* d_flags, KernelProf* prof);

// out-degree (live arcs over all segments) per node, int32
void out_degrees(Store& g, int32_t* deg);

}  // namespace gdb
