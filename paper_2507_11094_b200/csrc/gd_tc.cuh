// gd_tc.cuh -- dynamic triangle counting state (programs/tc_dynamic.sp).
#pragma once

#include <vector>

#include "gd_algo.cuh"
#include "gd_comm.cuh"

namespace gdb {

struct TC : AlgoBase {
    int64_t count = 0;
    Comm* comm = nullptr;  // set: count a contiguous 1/world slice of the records, all-reduce
    // hub bitmaps of the counting phases (see gd_tc.cu); kept clean between phases
    DBuf<uint8_t> hubmark, bm_multi;
    DBuf<int32_t> hub_slot;
    DBuf<uint32_t> bm;
    std::vector<int> count_rec;
    explicit TC(Store* st);  // = staticTC
    void batch(DevBatch& b, int64_t batch_index);

  private:
    int64_t count_records(const int32_t* s, const int32_t* d, int64_t k);
    void count_deferred(const int32_t* s, const int32_t* d, int64_t m, const int64_t* R, int64_t k,
                        const uint32_t* filt, uint64_t fmask, unsigned long long* ctr);
};

}  // namespace gdb
