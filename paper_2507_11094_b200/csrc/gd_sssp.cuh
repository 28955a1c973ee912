// gd_sssp.cuh -- dynamic SSSP state (programs/sssp_dynamic.sp).
#pragma once

#include "gd_algo.cuh"

namespace gdb {

struct SSSP : AlgoBase {
    int32_t src;
    int64_t cap_factor = 10;  // interp.py:141 iteration_cap_factor
    DBuf<int64_t> dist;       // int64, INF = INT64_MAX (reference type)
    DBuf<int32_t> parent;     // -1 = none
    DBuf<int32_t> stamp;      // frontier de-duplication (round id)
    DBuf<int32_t> hstamp;     // hub-piece de-duplication (round id)
    DBuf<int64_t> ho[2], hi[2];  // hub pieces (out-scans, in-pulls), double-buffered
    DBuf<uint8_t> fa, fb;     // per-node flags (stale / touched / seeds)
    Frontier fr;
    // [last stamp round, total rounds, diverged, visits, pieces, splits,
    //  kFpSlots x algorithmic bytes of the profiled fixpoint launches]
    DBuf<long long> ctr;
    static constexpr int kFpSlots = 8;
    int nfp = 0;               // profiled fixpoint launches since finish()
    int fp_prof[kFpSlots];     // their profiler record indices
    int64_t delta = 0;     // near-far bucket width for RELAX (0 = plain frontier)
    DBuf<int32_t> far[3];  // near-far piles
    DBuf<unsigned long long> fcnt;
    DBuf<long long> fmin;
    DBuf<int32_t> infar;
    DBuf<int32_t> heavy;
    DBuf<int64_t> parent64;  // int64 widening of parent for the async read   // stale vertices with > kHeavy in-arcs (pull sweep)
    DBuf<int64_t> dcount;  // device-side list sizes (no host read-back per fixpoint)
    // vertex-partitioned store: dist / parent are replicated and agree on
    // every rank between phases; the fixpoints run as supersteps of local
    // fixpoints over owned vertices + one message exchange with the owners
    DBuf<int32_t> outbox, gstamp, sstamp, seeds2;
    DBuf<int32_t> packed;
    DBuf<unsigned long long> nbox;
    int32_t launch_id = 0, step_id = 0;

    SSSP(Store* st, int64_t src, int64_t cap_factor = 10);  // = staticSSSP
    void batch(DevBatch& b, int64_t batch_index);
    void batch_dist(DevBatch& b, int64_t batch_index);  // vertex-partitioned store
    void read(int64_t* dist, int64_t* parent);
    void read_async(int64_t* dist, int64_t* parent);
    const int64_t* parent_i64();  // parent widened to int64 (device, valid until the next batch)  // see AlgoBase::copy_out_async

  private:
    // one cooperative launch per fixpoint (relax / walk / pull); the seed count
    // is read from d_nseeds on the device when given, else nseeds
    // 4-lane vertex groups in the fixpoints when the mean out-degree is <= 6
    // (GD_SSSP_G=4/8 overrides)
    bool narrow_groups() const;
    void fixpoint(int mode, const int32_t* seeds, const int64_t* d_nseeds, int64_t nseeds, uint8_t* flags,
                  const uint8_t* only = nullptr);
    // list == nullptr: every node; d_m (device) overrides m, which bounds the grid
    void fix_parents(const int32_t* list, const int64_t* d_m, int64_t m);
    void finish();
    // partitioned: the fixpoint as supersteps (see gd_sssp.cu); seeds are
    // owned vertices
    void fixpoint_dist(int mode, int32_t* seeds, int64_t* d_nseeds, uint8_t* flags, const uint8_t* only = nullptr);
    // partitioned: owned flagged vertices -> list (device count in d_m)
    void owned_list(const uint8_t* flags, int32_t* list, int64_t* d_m);
    // partitioned: every rank's owned blocks to every rank
    void sync(bool d, bool p, uint8_t* flags);
};

}  // namespace gdb
