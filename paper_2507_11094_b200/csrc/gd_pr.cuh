// gd_pr.cuh -- dynamic PageRank state (programs/pr_dynamic.sp).
#pragma once

#include "gd_algo.cuh"
#include "gd_comm.cuh"

namespace gdb {

struct PR : AlgoBase {
    double damping, beta;
    int64_t maxiter;
    DBuf<double> rank, rank_new, contrib, partial, scal;
    DBuf<int32_t> outdeg;  // maintained per record (misses included), int32 on device
    DBuf<uint8_t> affected;
    DBuf<int32_t> bins[3];            // affected vertices by in-degree: light / medium / hub
    int64_t nbin[3] = {0, 0, 0};
    int64_t ebin[3] = {0, 0, 0};      // in-arcs per bin (roofline bytes)
    int64_t last_sweeps = 0, last_affected = 0;

    Comm* comm = nullptr;  // set: pull only the owned destination range, all-gather ranks

    PR(Store* st, double damping, double beta, int64_t maxiter);  // = staticPR
    void set_comm(Comm* c);
    void batch(DevBatch& b, int64_t batch_index);                 // one Batch body
    void read(double* rank, int64_t* outdeg);

  private:
    void set_lists(const int32_t* list, int64_t m);
    void power_loop();
};

}  // namespace gdb
