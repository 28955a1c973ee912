// ref_driver.cc -- in-memory harness around the reference's OWN emitted
// OpenMP programs.  TEST/BASELINE INFRASTRUCTURE ONLY (never product code).
//
// It compiles the reference sources where they lie (see oracle/Makefile):
//   /root/reference/pkg/runtime/graphdyn_rt.h
//   /root/reference/pkg/tests/golden/{sssp,pr,tc}_dynamic_omp.cc
// renaming each golden main() so the three drivers link into one .so, and
// exposes a C entry point that builds a gd::Graph from arrays (instead of the
// text loader, graphdyn_rt.h:276-323) and runs the reference's dynamicSSSP /
// dynamicPR / dynamicTC unmodified.  Per-batch time follows the reference's
// own bench methodology (cli.py:436-442): (T_k - T_0) / k, where T_0 is the
// same call over an empty update stream (static pass only).
#define main gd_golden_sssp_main
#include "sssp_dynamic_omp.cc"
#undef main
#define main gd_golden_pr_main
#include "pr_dynamic_omp.cc"
#undef main
#define main gd_golden_tc_main
#include "tc_dynamic_omp.cc"
#undef main

#include <omp.h>

#include <cstdint>
#include <vector>

namespace {

// Mirrors Graph::load (graphdyn_rt.h:304-322) minus text parsing: undirected
// edges become two arcs, arcs are stable-sorted by source, reverse lists are
// built in (segment, node, slot) order like Graph::rebuild_reverse.
gd::Graph make_graph(int64_t n, const int64_t* src, const int64_t* dst, const int64_t* w, int64_t m,
                     bool directed, bool weighted, bool with_reverse, int64_t merge_interval) {
    gd::Graph g;
    g.n = n;
    g.directed = directed;
    g.weighted = weighted;
    g.with_reverse = with_reverse;
    g.merge_interval = merge_interval;
    std::vector<gd::Edge> arcs;
    arcs.reserve(static_cast<size_t>(directed ? m : 2 * m));
    for (int64_t i = 0; i < m; ++i) {
        int64_t wi = w ? w[i] : 1;
        arcs.push_back(gd::Edge{src[i], dst[i], wi, 0, 0});
        if (!directed) arcs.push_back(gd::Edge{dst[i], src[i], wi, 0, 0});
    }
    std::stable_sort(arcs.begin(), arcs.end(),
                     [](const gd::Edge& a, const gd::Edge& b) { return a.source < b.source; });
    g.segments.push_back(gd::Segment::from_arcs(n, arcs, weighted));
    g.live_edges = static_cast<int64_t>(arcs.size());
    if (with_reverse) {
        g.rev.assign(static_cast<size_t>(n), {});
        const gd::Segment& s = g.segments[0];
        for (int64_t v = 0; v < n; ++v)
            for (int64_t i = s.offsets[v]; i < s.offsets[v + 1]; ++i)
                g.rev[s.coords[i]].push_back(gd::RevEntry{v, 0, i});
    }
    return g;
}

gd::UpdateStream make_stream(const uint8_t* kind, const int64_t* us, const int64_t* ud, const int64_t* uw,
                             int64_t k) {
    gd::UpdateStream s;
    s.records.reserve(static_cast<size_t>(k));
    for (int64_t i = 0; i < k; ++i)
        s.records.push_back(gd::Update{static_cast<char>(kind[i]), us[i], ud[i], uw ? uw[i] : 1});
    return s;
}

}  // namespace

extern "C" {

// algo: 0 = SSSP, 1 = PR, 2 = TC.  Runs the reference driver twice (empty
// stream, then the k records in batches of batchsize) on fresh copies of the
// graph.  times[0] = T_0 seconds, times[1] = T_k seconds.  Outputs of the
// full run: SSSP -> out_i64a (dist), out_i64b (parent); PR -> out_f64 (rank),
// out_i64a (live out-degree of the final graph);
// TC -> out_i64a[0] (count).  Pass k = 0 to run the static pass only.
int gdref_run(int algo, int64_t n, const int64_t* src, const int64_t* dst, const int64_t* w, int64_t m,
              int directed, int weighted, int64_t merge_interval, const uint8_t* kind, const int64_t* us,
              const int64_t* ud, const int64_t* uw, int64_t k, int64_t batchsize, int threads, int64_t sssp_src,
              double damping, double beta, int64_t maxiter, int skip_t0, double* times, int64_t* out_i64a,
              int64_t* out_i64b, double* out_f64) {
    omp_set_num_threads(threads);
    bool with_reverse = algo != 2;  // tc_dynamic_omp.cc:152 loads without reverse
    gd::Graph proto = make_graph(n, src, dst, w, m, directed != 0, weighted != 0, with_reverse, merge_interval);
    gd::UpdateStream empty;
    gd::UpdateStream stream = make_stream(kind, us, ud, uw, k);
    if (batchsize <= 0) batchsize = static_cast<int64_t>(stream.size());
    if (batchsize <= 0) batchsize = 1;
    for (int pass = skip_t0 ? 1 : 0; pass < 2; ++pass) {
        gd::Graph g = proto;
        const gd::UpdateStream& st = pass == 0 ? empty : stream;
        double t0 = 0, t1 = 0;
        if (algo == 0) {
            gd::NodeProp<int64_t> dist, parent;
            dist.attach(g.num_nodes(), 0);
            parent.attach(g.num_nodes(), 0);
            t0 = omp_get_wtime();
            dynamicSSSP(g, dist, parent, st, batchsize, sssp_src);
            t1 = omp_get_wtime();
            if (pass == 1) {
                for (int64_t v = 0; v < n; ++v) {
                    if (out_i64a) out_i64a[v] = dist[v];
                    if (out_i64b) out_i64b[v] = parent[v];
                }
            }
        } else if (algo == 1) {
            gd::NodeProp<double> pr;
            pr.attach(g.num_nodes(), 0.0);
            t0 = omp_get_wtime();
            dynamicPR(g, pr, st, batchsize, damping, beta, maxiter);
            t1 = omp_get_wtime();
            if (pass == 1 && out_f64)
                for (int64_t v = 0; v < n; ++v) out_f64[v] = pr[v];
            // live out-degree of the final graph (= the driver's outdeg when
            // no delete missed, as in generate_updates streams)
            if (pass == 1 && out_i64a)
                for (int64_t v = 0; v < n; ++v) {
                    int64_t c = 0;
                    for (gd::Edge e : g.neighbors(v)) {
                        (void)e;
                        ++c;
                    }
                    out_i64a[v] = c;
                }
        } else {
            t0 = omp_get_wtime();
            int64_t c = dynamicTC(g, st, batchsize);
            t1 = omp_get_wtime();
            if (pass == 1 && out_i64a) out_i64a[0] = c;
        }
        if (times) times[pass] = t1 - t0;
    }
    return 0;
}

}  // extern "C"
