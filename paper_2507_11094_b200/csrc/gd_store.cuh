// gd_store.cuh -- GPU-resident diff-CSR store (base CSR + per-batch delta
// segments + tombstones) reproducing the reference's slot layout exactly.
//
// Reference: graph/csr.py:17-80, graph/dynamic.py:46-334,
// runtime/graphdyn_rt.h:215-511.  Layout in HBM:
//
//   out-store  segments[0..S): off int64[n+1], coord int32[slots] (-1 = the
//              reference's SENTINEL), w int32[slots] (weighted only).  Slot
//              positions match the reference bit for bit: deletes tombstone
//              the oldest matching slot, inserts claim the first vacancy of
//              the source's chain, leftovers spill into ONE new delta per add
//              call, merge compacts in neighbors() order.
//   rev index  in-arcs as a CSR over destinations with sources ascending
//              (the reference's reverse lists after a merge,
//              dynamic.py:319-329), plus an optional per-batch delta of new
//              in-arcs.  Deleted entries are tombstoned in place (~src) so
//              rows stay binary-searchable.  For undirected graphs this is the
//              sorted adjacency TC intersects over.
//   fwd index  the same structure over sources (directed TC only).
#pragma once

#include <vector>

#include "gd_comm.cuh"
#include "gd_common.cuh"

namespace gdb {

struct OutSeg {
    DBuf<int64_t> off;
    DBuf<int32_t> col;
    DBuf<int32_t> w;  // empty when unweighted
    int64_t nslots = 0;
};

// Device-side read views, passed by value to kernels.
struct EditJob;  // gd_store.cu: a two-phase edit merge

struct OutView {
    int nseg;
    const int64_t* const* off;  // device table of nseg pointers
    const int32_t* const* col;
    const int32_t* const* w;  // entries are nullptr when unweighted
    const int64_t* base;      // global slot id of each segment's slot 0
};

struct IdxView {  // a clean-or-tombstoned sorted index (no delta)
    const int64_t* off;
    const int32_t* col;  // negative = tombstoned entry
    const int32_t* w;    // nullptr when unweighted
};

struct SortedIndex {
    bool built = false;
    bool rows_are_dst = true;  // rev (true) or fwd (false)
    DBuf<int64_t> off;
    DBuf<int32_t> col;
    DBuf<int32_t> w;
    int64_t nnz = 0;
    // tombstones since the last compaction (unordered; -1 = unused slot)
    DBuf<int64_t> tpos;
    DBuf<int32_t> trow;
    int64_t ntomb = 0;
    // delta: new entries sorted by (row, col)
    DBuf<int32_t> drow, dcol, dw;
    int64_t dnnz = 0;
    bool dirty() const { return ntomb > 0 || dnnz > 0; }
    IdxView view() const { return IdxView{off.get(), col.get(), w.n ? w.get() : nullptr}; }
};

// Killed out-arcs of one delete call (device), one slot per request
// (gid -1 = nothing killed), consumed by index upkeep and the tomb log.
struct KilledArcs {
    DBuf<int32_t> row, col, w;
    DBuf<int64_t> gid;
    int64_t count = 0;
};
// One add call's vacancy claims: global slot per arc in stream order (-1 =
// spilled), and the delta segment the call created (-1 = none).  Kept from
// one rebuild (build / merge) to the next for nodes_to's list order.
struct ClaimLog {
    DBuf<int64_t> gid;
    int64_t delta_seg = -1;
};
// Inserted out-arcs of one add call (device).
struct AddedArcs {
    DBuf<int32_t> row, col, w;
    int64_t count = 0;
    // optional, non-owning: the arc indices in (row, stream) order, i.e. the
    // batch's stable sort by source (apply_adds); lets the in-index sort its
    // delta with one stable 32-bit pass by destination
    const int32_t* by_row = nullptr;
};

class Store {
  public:
    // part != nullptr: this rank's share of a vertex-partitioned store (1D
    // blocks, Blocks in gd_comm.cuh; directed graphs).  Every rank is given
    // the whole edge list and every batch; it keeps the out-arcs whose
    // source it owns (the out-store keeps the global id space, rows of
    // other ranks are empty -- the reference's PartitionedGraph shards,
    // partition.py:85-133) and the in-index of the arcs whose destination it
    // owns.  Deletes and adds run on the records of owned sources; the
    // killed and inserted arcs are routed to the owner of their destination
    // (one all-to-all each) to keep its in-index.
    Store(int device, int64_t n, const int64_t* src, const int64_t* dst, const int64_t* w, int64_t m,
          bool directed, bool weighted, bool with_reverse, int64_t merge_interval, bool as_arcs = false,
          const Comm* part = nullptr);
    ~Store();

    // update_csr_del on device-resident records (int32).  Returns applied;
    // found_fwd (k bytes, device) gets 1 per applied record when non-null.
    // returns the applied record count when want_count (one sync), else -1
    int64_t apply_deletes(const int32_t* d_src, const int32_t* d_dst, int64_t k, uint8_t* d_found,
                          bool want_count = false);
    void apply_adds(const int32_t* d_src, const int32_t* d_dst, const int32_t* d_w, int64_t k);
    void merge();
    bool merge_due(int64_t batch_index) const { return (batch_index + 1) % merge_interval == 0; }

    // indexes
    void require_rev();  // build the rev index if absent
    void require_fwd();  // directed TC: sorted out-index
    void compact_rev() { compact_index(rev); }
    void index_plan(SortedIndex& ix, EditJob& j, DBuf<int64_t>& ipos);
    void index_finish(SortedIndex& ix, EditJob& j, int64_t dead_total);
    void compact_fwd() { compact_index(fwd); }
    SortedIndex& tc_index() { return directed ? fwd : rev; }
    void compact_index(SortedIndex& ix);

    OutView out_view() const;
    int64_t total_slots() const;
    int64_t device_bytes() const;

    // export helpers (synchronous)
    void export_segment(int64_t seg, int64_t* off, int64_t* col, int64_t* w);
    int64_t rev_nnz_live();
    void export_rev(int64_t* off, int64_t* src, int64_t* w);
    void export_rev_slots(int64_t* off, int64_t* src, int64_t* seg, int64_t* idx, int64_t* w);

    int device;
    cudaStream_t stream = nullptr;
    const Comm* part = nullptr;  // partitioned store (see the constructor)
    Blocks blocks;               // vertex ownership when partitioned
    int64_t own_lo = 0, own_hi = 0;  // this rank's block ([0, n) unpartitioned)
    int64_t n;
    int sh = 1;  // pair keys: row << sh | col
    bool directed, weighted, with_reverse;
    int64_t merge_interval;
    int64_t live = 0;                // host view; kills pending in dcounts[1]
    DBuf<unsigned long long> dcounts;  // [applied records of the last delete call, killed slots not yet in live]
    int64_t live_count();              // live arcs (reads the pending kills)
    std::vector<OutSeg> segs;
    SortedIndex rev, fwd;
    // out-store tombstones since the last merge (unordered global slot ids;
    // -1 and delta-segment ids are ignored by the merge)
    DBuf<int64_t> otpos;
    DBuf<int32_t> otrow;
    int64_t notomb = 0;
    size_t first_clean_delta = 1;  // deltas from this index on have seen no delete phase
    std::vector<ClaimLog> claim_logs;  // add calls since the last rebuild (with_reverse only)

  private:
    int64_t apply_deletes_local(const int32_t* d_src, const int32_t* d_dst, int64_t k, uint8_t* d_found,
                                bool want_count);
    void apply_adds_local(const int32_t* d_src, const int32_t* d_dst, const int32_t* d_w, int64_t k);
    // partitioned: the records whose source this rank owns (compacted copies)
    int64_t owned_records(const int32_t* s, const int32_t* d, const int32_t* w, int64_t k, DBuf<int32_t>& idx,
                          DBuf<int32_t>& os, DBuf<int32_t>& od, DBuf<int32_t>& ow);
    // in-index upkeep, routed to the destination's owner when partitioned
    void rev_delete(const KilledArcs& ka);
    void rev_add(const AddedArcs& aa);
    void route_arcs(const int32_t* row, const int32_t* col, const int32_t* w, const int64_t* gid, int64_t m,
                    DBuf<int32_t>& orow, DBuf<int32_t>& ocol, DBuf<int32_t>& ow, int64_t& count);
    void index_from_arcs(SortedIndex& ix, bool rows_are_dst, const int32_t* rows, const int32_t* cols,
                         const int32_t* w, int64_t m);
    // segment table on the device: [off ptrs | col ptrs | w ptrs | bases]
    DBuf<uintptr_t> tab;
    std::vector<uintptr_t> h_tab;
    size_t tab_k = 0;
    void upload_tables();
    void build_index(SortedIndex& ix, bool rows_are_dst);
    void index_delete(SortedIndex& ix, const KilledArcs& ka);
    void index_add(SortedIndex& ix, const AddedArcs& aa);
    void append_out_tombs(const int64_t* d_pos, const int32_t* d_row, int64_t cnt);
};

// Edit-merge compaction shared by the out-store merge and index compaction:
// copy the live entries of a base array (negative = dead) while inserting
// sorted items before base positions P (stable), rows re-offset.
// Dead entries are the negative ones, found via an unordered tomb log
// (dedupe: the out-store may log a slot twice).
// an edit merge split in two (see gd_store.cu): inputs, then the plan's buffers
struct EditJob {
    int64_t n = 0;
    const int64_t* off = nullptr;
    int32_t* col = nullptr;
    const int32_t* w = nullptr;
    int64_t nnz = 0;
    const int64_t* tpos = nullptr;
    const int32_t* trow = nullptr;
    int64_t ntomb = 0;
    bool dedupe = false;
    const int32_t* irow = nullptr;
    const int32_t* icol = nullptr;
    const int32_t* iw = nullptr;
    const int64_t* ipos = nullptr;
    int64_t nins = 0;
    bool weighted = false;
    int64_t nwin = 0;
    DBuf<int64_t> counts, shift, dead_win;
};
void edit_plan(cudaStream_t s, EditJob& j);
void edit_apply(cudaStream_t s, EditJob& j, int64_t dead_total, DBuf<int64_t>& new_off, DBuf<int32_t>& new_col,
                DBuf<int32_t>& new_w, int64_t& new_nnz);
void edit_merge(cudaStream_t s, int64_t n, const int64_t* off, int32_t* col, const int32_t* w, int64_t nnz,
                const int64_t* tpos, const int32_t* trow, int64_t ntomb, bool dedupe, const int32_t* irow,
                const int32_t* icol, const int32_t* iw, const int64_t* ipos, int64_t nins, DBuf<int64_t>& new_off,
                DBuf<int32_t>& new_col, DBuf<int32_t>& new_w, int64_t& new_nnz, bool weighted);

}  // namespace gdb
