/*
 * gd_capi.h -- C ABI of the B200 dynamic-graph hot path.
 *
 * The reference (graphdyn v0.1.0, /root/reference/pkg) has no FFI: its seams
 * are the Python store API (DynamicGraph), the engine front door
 * (run_program / run_batches) and the emitted drivers dynamicSSSP /
 * dynamicPR / dynamicTC.  Each entry point below names the reference
 * interface it replaces (file:line, relative to /root/reference/pkg).  The
 * Python mirror in paper_2507_11094_b200/ binds these with ctypes; see
 * INTEGRATION.md for the binding a reference maintainer would add.
 *
 * Conventions:
 *   - every call returns a status: 0 ok, or a negative GD_ERR_* code, with a
 *     thread-local message in gd_last_error();
 *   - host arrays are borrowed for the duration of the call; results go to
 *     caller buffers; device memory is owned by the handle;
 *   - one CUDA stream per graph handle; calls are synchronous on return;
 *   - a handle is single-entrant (mirrors DynamicGraph._mutate_lock,
 *     graph/dynamic.py:85);
 *   - node ids are int64 at the ABI (int32 on the device: node_count must be
 *     < 2^31 - 1); weights must lie in [0, 2^31); a store holds at most 2^31
 *     arcs (slot ids are int64, build-time positions int32).
 * There is no CPU fallback: without a usable CUDA device every call that
 * needs one fails with GD_ERR_CUDA.
 */
#ifndef GD_CAPI_H
#define GD_CAPI_H

#include <stdint.h>

#if defined(__GNUC__)
#define GD_API __attribute__((visibility("default")))
#else
#define GD_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* status codes -> reference exceptions (errors.py:6-61) */
#define GD_OK 0
#define GD_ERR_MALFORMED (-1) /* MalformedInputError */
#define GD_ERR_CONTRACT (-2)  /* ContractViolation */
#define GD_ERR_CONFIG (-3)    /* ConfigurationError */
#define GD_ERR_EXEC (-4)      /* ExecError */
#define GD_ERR_DIVERGED (-5)  /* DivergenceError */
#define GD_ERR_CUDA (-6)      /* device failure (no reference equivalent) */

/* phase indices of gd_phase_times, named as ExecContext.add_phase
 * (engine/interp.py:141-145) */
#define GD_PHASE_STATIC 0     /* "static_phase" */
#define GD_PHASE_PREPROCESS 1 /* "preprocess": OnAdd / OnDelete handlers */
#define GD_PHASE_STRUCT 2     /* "structural_update": updateCSRDel / updateCSRAdd */
#define GD_PHASE_PROPAGATE 3  /* "propagate": Incremental / Decremental / flood */
#define GD_PHASE_MERGE 4      /* "merge" */

typedef struct gd_graph gd_graph;
typedef struct gd_sssp gd_sssp;
typedef struct gd_pr gd_pr;
typedef struct gd_tc gd_tc;
typedef struct gd_comm gd_comm;

/* Last error message of the calling thread ("" when none). */
GD_API const char* gd_last_error(void);
/* ABI version (major*100 + minor). */
GD_API int gd_abi_version(void);
/* Number of CUDA kernel launches this library issued since load. */
GD_API int64_t gd_kernel_launches(void);

/* ---- graph store: DynamicGraph (graph/dynamic.py:46-334; C++ gd::Graph,
 *      runtime/graphdyn_rt.h:262-511) ---------------------------------- */

/* DynamicGraph.build (graph/dynamic.py:89-120).  w may be NULL (all 1).
 * directed: bit 0 = directed; bit 1 (GD_ARCS) = the triples are already
 * arcs (no reverse arc is added for undirected graphs), as the reference's
 * DynamicGraph(...) constructor receives them from merged() (dynamic.py:290-305). */
#define GD_ARCS 2
GD_API int gd_graph_create(int64_t node_count, const int64_t* src, const int64_t* dst, const int64_t* w, int64_t m,
                    int directed, int weighted, int with_reverse, int64_t merge_interval, int device,
                    gd_graph** out);
GD_API int gd_graph_destroy(gd_graph* g);

/* The same graph as one rank's share of a 1D vertex partition over `comm`
 * (block ownership: rank r owns [r*q + min(r, n%W), ...), the first n % W
 * ranks one more -- partition.py:69-78).  Every rank passes the whole edge
 * list; it keeps the out-arcs of the sources it owns (the reference's
 * PartitionedGraph shard, partition.py:85-133) and the in-arcs of the
 * destinations it owns.  Directed graphs only (undirected graphs are
 * replicated per rank).  Every later call on the graph and on algorithm
 * handles made from it is collective: each rank passes the whole batch, the
 * owners apply their records and route the killed / inserted arcs to the
 * destinations' owners.  Segment exports show this rank's shard; live
 * counts, miss flags, flood results and algorithm reads are global. */
GD_API int gd_graph_create_dist(int64_t node_count, const int64_t* src, const int64_t* dst, const int64_t* w,
                                int64_t m, int directed, int weighted, int with_reverse, int64_t merge_interval,
                                int device, gd_comm* comm, gd_graph** out);
/* the owned vertex block [lo, hi) ([0, n) for an unpartitioned graph) */
GD_API int gd_graph_owned_range(gd_graph* g, int64_t* lo, int64_t* hi);

/* DynamicGraph.update_csr_del -> DeleteReport (graph/dynamic.py:208-244).
 * miss_flags (nullable, k bytes) gets 1 for each record that missed. */
GD_API int gd_graph_apply_deletes(gd_graph* g, const int64_t* src, const int64_t* dst, int64_t k, int64_t* applied,
                           int64_t* misses, uint8_t* miss_flags);
/* DynamicGraph.update_csr_add (graph/dynamic.py:249-286).  w may be NULL. */
GD_API int gd_graph_apply_adds(gd_graph* g, const int64_t* src, const int64_t* dst, const int64_t* w, int64_t k);
/* DynamicGraph.merge_deltas (graph/dynamic.py:307-317). */
GD_API int gd_graph_merge(gd_graph* g);

/* live_edge_count, len(segments()), total_slot_count() (graph/dynamic.py:122-181) */
GD_API int gd_graph_stats(gd_graph* g, int64_t* live, int64_t* nsegments, int64_t* total_slots);
/* node_count / directed / weighted / has_reverse / merge_interval */
GD_API int gd_graph_info(gd_graph* g, int64_t* node_count, int* directed, int* weighted, int* with_reverse,
                  int64_t* merge_interval);
/* segments()[seg] (base = 0, then deltas): offsets[n+1], coords[nslots]
 * (SENTINEL = INT64_MAX as in graph/csr.py:14), weights[nslots] (1 when
 * unweighted).  Query nslots with gd_graph_segment_slots first. */
GD_API int gd_graph_segment_slots(gd_graph* g, int64_t seg, int64_t* nslots);
GD_API int gd_graph_export_segment(gd_graph* g, int64_t seg, int64_t* offsets, int64_t* coords, int64_t* weights);
/* nodes_to (graph/dynamic.py:150-160): live in-arcs of every node as a CSR
 * over destinations, sources ascending within a node. */
GD_API int gd_graph_reverse_nnz(gd_graph* g, int64_t* nnz);
GD_API int gd_graph_export_reverse(gd_graph* g, int64_t* offsets, int64_t* src, int64_t* weights);
/* nodes_to exactly (graph/dynamic.py:152-160): each node's live in-arcs in
 * the reference's reverse-list order (rebuild order, then inserts in the
 * order they were appended), with the EdgeRef slot identity (segment,
 * index) of every arc.  Arrays hold gd_graph_reverse_nnz entries. */
GD_API int gd_graph_export_reverse_slots(gd_graph* g, int64_t* offsets, int64_t* src, int64_t* segment,
                                         int64_t* index, int64_t* weights);
/* gview.propagate_flags (engine/interp.py:70-109): flood true flags across
 * weak components; flags is n bytes in/out. */
GD_API int gd_graph_propagate_flags(gd_graph* g, uint8_t* flags, int64_t* rounds);
/* The graph's CUDA stream (cudaStream_t) for callers timing with events. */
GD_API int gd_graph_stream(gd_graph* g, void** stream);
/* bytes of device memory the store holds */
GD_API int gd_graph_device_bytes(gd_graph* g, int64_t* bytes);

/* ---- dynamic SSSP: programs/sssp_dynamic.sp:8-158 -------------------------
 * create = staticSSSP (sssp_dynamic.sp:8-35); batch = one Batch body of
 * dynamicSSSP (sssp_dynamic.sp:137-157) incl. merge-if-due
 * (engine/interp.py:877-880); read = ctx.properties["dist"/"parent"].      */
GD_API int gd_sssp_create(gd_graph* g, int64_t src, gd_sssp** out);
/* the same with run_program's iteration_cap_factor (engine/run.py:22-41):
 * every fixpoint of this handle (static and per batch) stops with
 * GD_ERR_DIVERGED after max(1, factor * max(1, n)) rounds, as
 * ExecContext.iteration_cap (engine/interp.py:138-139,800-813).  Plain
 * gd_sssp_create uses the reference default 10. */
GD_API int gd_sssp_create_ex(gd_graph* g, int64_t src, int64_t iteration_cap_factor, gd_sssp** out);
GD_API int gd_sssp_batch(gd_sssp* s, const uint8_t* kind, const int64_t* src, const int64_t* dst, const int64_t* w,
                  int64_t k, int64_t batch_index);
/* Same batch with the records already in device memory (int32 ids, 'a'/'d'). */
GD_API int gd_sssp_batch_device(gd_sssp* s, const uint8_t* kind, const int32_t* src, const int32_t* dst,
                         const int32_t* w, int64_t k, int64_t batch_index);
GD_API int gd_sssp_read(gd_sssp* s, int64_t* dist, int64_t* parent);
/* asynchronous variant: the state is snapshotted on the device at once and
 * copied to the (ideally pinned) host buffers on a side stream that overlaps
 * the next batch; the buffers are valid after gd_wait(s).  No reference
 * counterpart: ctx.properties are read after the run (interp.py:112-160). */
GD_API int gd_sssp_read_async(gd_sssp* s, int64_t* dist, int64_t* parent);
/* run_batches over a whole host update stream (engine/run.py:44-68): the
 * records [0, k) in batches of batch_size (batch j = records [j*bs, ...),
 * batch_index first_batch_index + j), pipelined -- batch j+1's records go
 * up and batch j-1's result comes back on a copy stream while batch j runs
 * (host arrays: pinned for the overlap; they must stay valid until return).
 * After every batch its dist/parent are copied to dist/parent (nullable),
 * which hold the last batch's result on return.  Errors as gd_sssp_batch;
 * the batches before the failing one stay applied. */
GD_API int gd_sssp_run_stream(gd_sssp* s, const uint8_t* kind, const int64_t* src, const int64_t* dst,
                              const int64_t* w, int64_t k, int64_t batch_size, int64_t first_batch_index,
                              int64_t* dist, int64_t* parent);
/* the same with int32 record ids (half the upload of int64 ids: ids of the
 * B200 layout are < 2^31 anyway) */
GD_API int gd_sssp_run_stream32(gd_sssp* s, const uint8_t* kind, const int32_t* src, const int32_t* dst,
                                const int32_t* w, int64_t k, int64_t batch_size, int64_t first_batch_index,
                                int64_t* dist, int64_t* parent);
GD_API int gd_sssp_destroy(gd_sssp* s);

/* ---- dynamic PageRank: programs/pr_dynamic.sp:7-102 --------------------- */
GD_API int gd_pr_create(gd_graph* g, double damping, double beta, int64_t maxiter, gd_pr** out);
GD_API int gd_pr_batch(gd_pr* p, const uint8_t* kind, const int64_t* src, const int64_t* dst, const int64_t* w,
                int64_t k, int64_t batch_index);
GD_API int gd_pr_batch_device(gd_pr* p, const uint8_t* kind, const int32_t* src, const int32_t* dst, const int32_t* w,
                       int64_t k, int64_t batch_index);
/* pagerank[n] (float64); outdeg[n] nullable (the maintained int64 outdeg) */
GD_API int gd_pr_read(gd_pr* p, double* rank, int64_t* outdeg);
GD_API int gd_pr_read_async(gd_pr* p, double* rank); /* as gd_sssp_read_async */
/* ctx.properties["affected"] (pr_dynamic.sp:82-99): the last batch's flags
 * after propagateNodeFlags, n bytes of 0/1 (all 0 before the first batch) */
GD_API int gd_pr_read_affected(gd_pr* p, uint8_t* affected);
/* device pointer to the float64 rank vector (valid until the next call) */
GD_API int gd_pr_rank_device(gd_pr* p, const double** rank);
/* as gd_sssp_run_stream; rank (nullable) receives every batch's ranks */
GD_API int gd_pr_run_stream(gd_pr* p, const uint8_t* kind, const int64_t* src, const int64_t* dst, const int64_t* w,
                            int64_t k, int64_t batch_size, int64_t first_batch_index, double* rank);
GD_API int gd_pr_run_stream32(gd_pr* p, const uint8_t* kind, const int32_t* src, const int32_t* dst,
                              const int32_t* w, int64_t k, int64_t batch_size, int64_t first_batch_index,
                              double* rank);
GD_API int gd_pr_destroy(gd_pr* p);

/* ---- dynamic triangle counting: programs/tc_dynamic.sp:7-115 ------------ */
GD_API int gd_tc_create(gd_graph* g, gd_tc** out);
GD_API int gd_tc_batch(gd_tc* t, const uint8_t* kind, const int64_t* src, const int64_t* dst, const int64_t* w,
                int64_t k, int64_t batch_index);
GD_API int gd_tc_batch_device(gd_tc* t, const uint8_t* kind, const int32_t* src, const int32_t* dst, const int32_t* w,
                       int64_t k, int64_t batch_index);
GD_API int gd_tc_read(gd_tc* t, int64_t* count);
/* as gd_sssp_run_stream; counts (nullable) gets the count after each batch,
 * one int64 per batch */
GD_API int gd_tc_run_stream(gd_tc* t, const uint8_t* kind, const int64_t* src, const int64_t* dst, const int64_t* w,
                            int64_t k, int64_t batch_size, int64_t first_batch_index, int64_t* counts);
GD_API int gd_tc_run_stream32(gd_tc* t, const uint8_t* kind, const int32_t* src, const int32_t* dst,
                              const int32_t* w, int64_t k, int64_t batch_size, int64_t first_batch_index,
                              int64_t* counts);
GD_API int gd_tc_destroy(gd_tc* t);

/* ---- multi-GPU (one process per GPU).  NCCL is loaded on
 *      first use.  Rank 0 makes the id, the caller broadcasts the 128 bytes
 *      (e.g. torch.distributed), every rank creates its communicator.  Stores
 *      are replicas (each rank applies every batch); a PR handle with a comm
 *      pulls only its destination range and all-gathers the rank vector each
 *      sweep (all-reduce max of the residual); a TC handle counts a 1/world
 *      slice of each phase's records and all-reduces the count delta.  The
 *      reference has no multi-process path (partition.py simulates one). */
GD_API int gd_comm_unique_id(uint8_t id[128]);
GD_API int gd_comm_create(int world, int rank, const uint8_t id[128], int device, gd_comm** out);
/* A member of an in-process group of `world` ranks that share the calling
 * process (one host thread per rank, any common `group` id).  Collectives
 * meet at a host barrier and move data with device copies -- the NCCL call
 * sequence without NCCL, so the partitioned code paths run on one GPU (tests).
 * No reference counterpart. */
GD_API int gd_comm_create_local(int world, int rank, int64_t group, int device, gd_comm** out);
GD_API int gd_comm_destroy(gd_comm* c);
/* communication accounting (the CommStats analogue of partition.py:32-66):
 * out[0] collective calls, out[1] all-gather payload bytes, out[2] all-reduce
 * payload bytes, out[3] bytes this rank sends under the ring algorithms
 * ((world-1)/world of an all-gather's payload, 2(world-1)/world of an
 * all-reduce's) -- counted since creation or the last reset */
GD_API int gd_comm_stats(const gd_comm* c, int64_t out[4]);
/* the same plus out[4] = bytes this rank sent to other ranks through the
 * all-to-all exchanges (routed arcs, SSSP messages) */
GD_API int gd_comm_stats_ex(const gd_comm* c, int64_t out[5]);
GD_API int gd_comm_reset_stats(gd_comm* c);
GD_API int gd_pr_set_comm(gd_pr* p, gd_comm* c);
GD_API int gd_tc_set_comm(gd_tc* t, gd_comm* c);

/* ---- the store path's device primitives on host arrays (test hooks; no
 *      reference counterpart).  gd_prim_sort: stable LSD radix sort of n keys
 *      (key_bytes 8, values optional; or 4 with values) on bits [0, end_bit).
 *      gd_prim_scan_select: exclusive int64 scan of `in` into `out`, and the
 *      ordered indices of the nonzero flags into idx (count in *count). */
GD_API int gd_prim_sort(int key_bytes, void* keys, int32_t* vals, int64_t n, int end_bit, int device);
GD_API int gd_prim_scan_select(const int64_t* in, int64_t* out, const uint8_t* flags, int32_t* idx, int64_t n,
                               int64_t* count, int device);

/* ---- reporting (ExecContext.phase_totals / fixedpoint_iterations,
 *      engine/interp.py:112-145); h is any gd_sssp* / gd_pr* / gd_tc* ---- */
GD_API int gd_phase_times(const void* h, double ms[5]);
/* block until the handle's asynchronous reads have landed in host memory */
GD_API int gd_wait(const void* h);
GD_API int gd_iterations(const void* h, int64_t* total_iterations);
/* per-kernel device time of the last batch for roofline reporting:
 * name = "pr_pull" | "tc_count" | "sssp_relax" | "merge" ...; ms summed over
 * the batch's launches of that kernel, launches = how many. */
GD_API int gd_kernel_time(const void* h, const char* name, double* ms, int64_t* launches, int64_t* bytes);
/* the same, summed over every batch since profiling was last switched on
 * (one query after a timed loop instead of one per batch) */
GD_API int gd_kernel_time_total(const void* h, const char* name, double* ms, int64_t* launches, int64_t* bytes);
/* enable per-kernel event timing (off by default: it adds event records);
 * switching it on clears the running totals */
GD_API int gd_set_profiling(const void* h, int on);

#ifdef __cplusplus
}
#endif

#endif /* GD_CAPI_H */
