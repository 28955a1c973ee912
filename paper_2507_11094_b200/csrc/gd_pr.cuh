// gd_pr.cuh -- dynamic PageRank state (programs/pr_dynamic.sp).
#pragma once

#include <utility>
#include <vector>

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
    DBuf<int64_t> ctl;                // device loop state: bin sizes, bin in-arcs, done, sweeps
    int64_t ahead_hint = 4;           // sweeps to queue per read-back (last batch's count + 1)
    int64_t last_sweeps = 0, last_affected = 0;
    std::vector<std::pair<int, int>> pull_recs;  // (profiler record, bin) of the queued pull launches

    Comm* comm = nullptr;  // set: pull only the owned destination range, all-gather ranks

    PR(Store* st, double damping, double beta, int64_t maxiter);  // = staticPR
    void set_comm(Comm* c);
    void batch(DevBatch& b, int64_t batch_index);                 // one Batch body
    void read(double* rank, int64_t* outdeg);
    void read_affected(uint8_t* aff);  // the last batch's flooded flags
    // vertex-partitioned store: every rank's owned blocks of rank, outdeg
    // and affected to every rank (collective; before a read)
    void gather();

  private:
    void recompute(const uint8_t* flags);  // bin + sweep loop; flags == nullptr: all vertices
    void sweep(int64_t tag);
};

}  // namespace gdb
