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
    DBuf<uint8_t> fa, fb;     // per-node flags (stale / touched / seeds)
    Frontier fr;
    int32_t round = 0;

    SSSP(Store* st, int64_t src);  // = staticSSSP
    void batch(DevBatch& b, int64_t batch_index);
    void read(int64_t* dist, int64_t* parent);

  private:
    int64_t relax_push(const int32_t* seeds, int64_t nseeds, uint8_t* touched);  // push fixpoint
    int64_t walk(const int32_t* seeds, int64_t nseeds, uint8_t* stale);
    int64_t pull(const int32_t* stale_list, int64_t nstale, const uint8_t* stale);
    void fix_parents(const int32_t* list, int64_t m);  // list == nullptr: every node
    void check_cap(int64_t it);
};

}  // namespace gdb
