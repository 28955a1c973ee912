// gd_tc.cuh -- dynamic triangle counting state (programs/tc_dynamic.sp).
#pragma once

#include "gd_algo.cuh"
#include "gd_comm.cuh"

namespace gdb {

struct TC : AlgoBase {
    int64_t count = 0;
    Comm* comm = nullptr;  // set: count a contiguous 1/world slice of the records, all-reduce
    explicit TC(Store* st);  // = staticTC
    void batch(DevBatch& b, int64_t batch_index);

  private:
    int64_t count_records(const int32_t* s, const int32_t* d, int64_t k);
};

}  // namespace gdb
