"""GPU parity: the CUDA path (through the C ABI) against the reference's own
outputs (golden fixtures) and against the CPU oracle on seeded inputs."""

import numpy as np
import pytest

from golden_io import algo_cases, cap_cases, store_cases

pytestmark = pytest.mark.gpu

SENT = np.iinfo(np.int64).max


@pytest.fixture(scope="module")
def gd():
    import paper_2507_11094_b200 as gd

    return gd


def sorted_rev(off, src, w):
    out = []
    for v in range(len(off) - 1):
        out.append(sorted(zip(src[off[v]:off[v + 1]].tolist(), w[off[v]:off[v + 1]].tolist())))
    return out


def assert_store(g, snap, where, weighted=True):
    assert g.live_edge_count == snap.live, where
    segs = g.segments()
    assert len(segs) == len(snap.segments), f"{where}: {len(segs)} segments vs {len(snap.segments)}"
    for i, (seg, (eo, ec, ew)) in enumerate(zip(segs, snap.segments)):
        np.testing.assert_array_equal(seg.offsets, eo, err_msg=f"{where} seg{i} offsets")
        np.testing.assert_array_equal(seg.coordinates, ec, err_msg=f"{where} seg{i} coords")
        live = ec != SENT
        if weighted:
            np.testing.assert_array_equal(seg.weights[live], ew[live], err_msg=f"{where} seg{i} weights")
    off, s, w = g._reverse_snapshot()
    assert sorted_rev(off, s, w) == sorted_rev(*snap.rev), f"{where}: reverse multisets"
    # nodes_to: the reference's list order and EdgeRef slot identities
    roff, rs, rseg, ridx, rw = g._reverse_lists()
    np.testing.assert_array_equal(roff, snap.rev[0], err_msg=f"{where} nodes_to offsets")
    np.testing.assert_array_equal(rs, snap.rev[1], err_msg=f"{where} nodes_to sources (list order)")
    if weighted:
        np.testing.assert_array_equal(rw, snap.rev[2], err_msg=f"{where} nodes_to weights")
    if snap.revslots is not None:
        np.testing.assert_array_equal(rseg, snap.revslots[0], err_msg=f"{where} nodes_to segments")
        np.testing.assert_array_equal(ridx, snap.revslots[1], err_msg=f"{where} nodes_to slot indices")


STORE = store_cases()


@pytest.mark.parametrize("case", STORE, ids=[c.name for c in STORE])
def test_store_layout_bit_exact(gd, case):
    e = case.edges
    g = gd.DynamicGraph.from_arrays(case.n, e[0], e[1], e[2], directed=case.directed, weighted=True,
                                    with_reverse=True)
    assert_store(g, case.build, f"{case.name}/build")
    for i, b in enumerate(case.batches):
        r = b["recs"]
        stream = gd.UpdateStream.from_arrays(r[0].astype(np.uint8), r[1], r[2], r[3])
        batch = stream.as_batch()
        rep = g.update_csr_del(batch.only_deletes())
        assert [rep.applied, rep.misses] == list(b["report"]), f"{case.name}/b{i} report"
        dels = batch.only_deletes().arrays
        missed_idx = np.flatnonzero(b["missflags"])
        assert [(m.src, m.dst) for m in rep.missed] == [(int(dels.src[j]), int(dels.dst[j])) for j in missed_idx]
        assert_store(g, b["del"], f"{case.name}/b{i}/del")
        g.update_csr_add(batch.only_adds())
        assert_store(g, b["add"], f"{case.name}/b{i}/add")
        if b["merge"] is not None:
            g.merge_deltas()
            assert_store(g, b["merge"], f"{case.name}/b{i}/merge")
    g.check_invariants()


ALGO = algo_cases()


def run_gpu(gd, case):
    e = case.edges
    g = gd.DynamicGraph.from_arrays(case.n, e[0], e[1], e[2], directed=case.directed, weighted=case.weighted,
                                    with_reverse=case.algo != "tc", merge_interval=case.merge_interval)
    r = case.recs
    stream = gd.UpdateStream.from_arrays(r[0].astype(np.uint8), r[1], r[2], r[3])
    inputs = {"sssp": {"src": case.src}, "pr": {"damping": case.damping, "beta": case.beta,
                                                "maxiter": case.maxiter}, "tc": {}}[case.algo]
    return gd.run_batches(gd.shipped_program(case.algo), g, stream, case.batch, inputs)


@pytest.mark.parametrize("case", ALGO, ids=[c.name for c in ALGO])
def test_algorithm_matches_reference(gd, case):
    ctx = run_gpu(gd, case)
    if case.algo == "sssp":
        np.testing.assert_array_equal(ctx.properties["dist"].values(), case.expect["dist"])
        np.testing.assert_array_equal(ctx.properties["parent"].values(), case.expect["parent"])
    elif case.algo == "pr":
        got = np.asarray(ctx.properties["pagerank"].values())
        want = case.expect["rank"]
        # north_star tolerance: max-abs 1e-6 per vertex.  Multigraph streams with
        # missed deletes drive outdeg negative in the reference (pr_dynamic.sp:87-92)
        # and ranks explode to ~1e77; there only the relative error is meaningful.
        tol = 1e-6 + 1e-12 * np.abs(want)
        assert np.all(np.abs(got - want) <= tol), f"max-abs {np.max(np.abs(got - want))}"
    else:
        assert ctx.return_value == int(case.expect["count"][0])
    # bool node properties (activeOnDelete / activeOnAdd, affected) and the
    # reference's property names and order
    props = [k[5:] for k in case.expect if k.startswith("prop:")]
    for pn in props:
        assert ctx.properties[pn].dtype == "bool"
        np.testing.assert_array_equal(np.asarray(ctx.properties[pn].values(), dtype=np.uint8),
                                      case.expect[f"prop:{pn}"], err_msg=pn)
    if case.source == "engine":
        want = {"sssp": ["dist", "parent", "activeOnDelete", "activeOnAdd"],
                "pr": ["pagerank", "affected", "outdeg"], "tc": []}[case.algo]
        assert list(ctx.properties) == want


CAPS = cap_cases()


@pytest.mark.parametrize("case", CAPS, ids=[c.name for c in CAPS])
def test_iteration_cap_factor_trips_like_the_reference(gd, case):
    """run_program(iteration_cap_factor=f) raises DivergenceError exactly
    where the reference does (interp.py:138-139,800-813)."""
    e, r = case.edges, case.recs
    for f, div in zip(case.factors.tolist(), case.diverged.tolist()):
        g = gd.DynamicGraph.from_arrays(case.n, e[0], e[1], e[2], directed=case.directed, weighted=case.weighted,
                                        with_reverse=True)
        stream = gd.UpdateStream.from_arrays(r[0].astype(np.uint8), r[1], r[2], r[3])
        run = lambda: gd.run_batches(gd.shipped_program("sssp"), g, stream, case.batch, {"src": 0},  # noqa: E731
                                     iteration_cap_factor=f)
        if div:
            with pytest.raises(gd.DivergenceError):
                run()
        else:
            run()


def test_static_entries_expose_the_reference_locals(gd):
    """run_program(entry="staticSSSP"/"staticPR") properties as the
    reference's: the entry's propNode locals included."""
    g = gd.DynamicGraph.build([(0, 1, 1), (1, 2, 1), (4, 0, 1)], 5, with_reverse=True)
    ctx = gd.run_program(gd.shipped_program("pr"), g, {"damping": 0.85, "beta": 1e-3, "maxiter": 100},
                         entry="staticPR")
    assert list(ctx.properties) == ["pagerank", "outdeg", "rank_new"]
    assert ctx.properties["rank_new"].values() == ctx.properties["pagerank"].values()
    ctx = gd.run_program(gd.shipped_program("sssp"), g, {"src": 0}, entry="staticSSSP")
    assert list(ctx.properties) == ["dist", "parent", "modified", "modified_nxt"]
    assert not any(ctx.properties["modified"].values())


# -- seeded random cases vs the CPU oracle ----------------------------------------------

def rmat(scale, m, rng, weighted=True):
    a, b, c = 0.57, 0.19, 0.19
    u = np.zeros(m, dtype=np.int64)
    v = np.zeros(m, dtype=np.int64)
    for _ in range(scale):
        r = rng.random(m)
        bit_u = r >= a + b
        bit_v = ((r >= a) & (r < a + b)) | (r >= a + b + c)
        u = (u << 1) | bit_u
        v = (v << 1) | bit_v
    w = rng.integers(1, 101, m) if weighted else np.ones(m, dtype=np.int64)
    return u, v, w


def updates(rng, n, src, dst, k, add_frac=0.5, distinct_deletes=False):
    kind = np.where(rng.random(k) < add_frac, ord("a"), ord("d")).astype(np.uint8)
    if distinct_deletes:  # generate_updates semantics: each existing pair deleted at most once
        _, first = np.unique(src * (1 << 32) + dst, return_index=True)
        pick = rng.permutation(first)[:k]
        pick = np.resize(pick, k)
        nd = np.count_nonzero(kind == ord("d"))
        kind[np.flatnonzero(kind == ord("d"))[len(first):]] = ord("a") if nd > len(first) else ord("d")
    else:
        pick = rng.integers(0, len(src), k)
    us = np.where(kind == ord("d"), src[pick], rng.integers(0, n, k))
    ud = np.where(kind == ord("d"), dst[pick], rng.integers(0, n, k))
    uw = rng.integers(1, 101, k)
    return kind, us, ud, uw


CASES = [(scale, mi, bs) for scale in (10, 13) for mi in (1, 3) for bs in (50, 2000)]


@pytest.mark.parametrize("scale,mi,bs", CASES)
def test_sssp_random_vs_oracle(gd, scale, mi, bs):
    from oracle import oracle as O

    rng = np.random.default_rng(scale * 100 + mi * 10 + bs)
    n = 1 << scale
    src, dst, w = rmat(scale, 8 * n, rng)
    kind, us, ud, uw = updates(rng, n, src, dst, 4 * bs)
    g = gd.DynamicGraph.from_arrays(n, src, dst, w, weighted=True, with_reverse=True, merge_interval=mi)
    ctx = gd.run_batches(gd.shipped_program("sssp"), g, gd.UpdateStream.from_arrays(kind, us, ud, uw), bs,
                         {"src": 1})
    og = O.OracleGraph(n, src, dst, w, weighted=True, with_reverse=True, merge_interval=mi)
    dist, parent = O.OracleSSSP(og, 1).run_stream(kind, us, ud, uw, bs).read()
    np.testing.assert_array_equal(ctx.properties["dist"].values(), dist)
    np.testing.assert_array_equal(ctx.properties["parent"].values(), parent)


@pytest.mark.parametrize("scale,mi,bs", CASES)
def test_pr_random_vs_oracle(gd, scale, mi, bs):
    from oracle import oracle as O

    rng = np.random.default_rng(scale * 101 + mi * 11 + bs)
    n = 1 << scale
    src, dst, _ = rmat(scale, 8 * n, rng, weighted=False)
    # generate_updates semantics (no delete misses): outdeg stays exact
    kind, us, ud, uw = updates(rng, n, src, dst, 4 * bs, distinct_deletes=True)
    for beta in (1e-3, 1e-10):
        g = gd.DynamicGraph.from_arrays(n, src, dst, with_reverse=True, merge_interval=mi)
        ctx = gd.run_batches(gd.shipped_program("pr"), g, gd.UpdateStream.from_arrays(kind, us, ud, uw), bs,
                             {"damping": 0.85, "beta": beta, "maxiter": 100})
        og = O.OracleGraph(n, src, dst, with_reverse=True, merge_interval=mi)
        rank, od = O.OraclePR(og, 0.85, beta, 100).run_stream(kind, us, ud, uw, bs).read()
        got = np.asarray(ctx.properties["pagerank"].values())
        np.testing.assert_allclose(got, rank, rtol=0, atol=1e-6)
        np.testing.assert_array_equal(ctx.properties["outdeg"].values(), od)


@pytest.mark.parametrize("scale,mi,bs", CASES)
def test_tc_random_vs_oracle(gd, scale, mi, bs):
    from oracle import oracle as O

    rng = np.random.default_rng(scale * 103 + mi * 13 + bs)
    n = 1 << scale
    src, dst, _ = rmat(scale, 4 * n, rng, weighted=False)
    kind, us, ud, uw = updates(rng, n, src, dst, 4 * bs)
    for directed in (False, True):
        g = gd.DynamicGraph.from_arrays(n, src, dst, directed=directed, merge_interval=mi)
        ctx = gd.run_batches(gd.shipped_program("tc"), g, gd.UpdateStream.from_arrays(kind, us, ud, uw), bs,
                             {})
        og = O.OracleGraph(n, src, dst, directed=directed, merge_interval=mi)
        assert ctx.return_value == O.OracleTC(og).run_stream(kind, us, ud, uw, bs).read()


def test_propagate_flags_matches_bfs(gd):
    from oracle import oracle as O

    rng = np.random.default_rng(5)
    n = 3000
    src, dst = rng.integers(0, n, 2500), rng.integers(0, n, 2500)
    seeds = (rng.random(n) < 0.002).astype(np.uint8)
    for directed in (True, False):
        g = gd.DynamicGraph.from_arrays(n, src, dst, directed=directed, with_reverse=True)
        og = O.OracleGraph(n, src, dst, directed=directed, with_reverse=True)
        want, _ = og.propagate_flags(seeds)
        np.testing.assert_array_equal(g.propagate_flags(seeds), want)


def test_propagate_flags_with_hubs_outside_the_giant(gd):
    """Two large stars (in- and out-arcs), no dominating component: the
    union-find's rest pass must link a hub that is not in the sampled giant
    (warp-cooperative path) and the flags must match the BFS oracle."""
    from oracle import oracle as O

    n = 12000
    leaves_a = np.arange(10, 5010)
    leaves_b = np.arange(5010, 11000)
    src = np.concatenate([np.full(len(leaves_a), 3), leaves_b, np.array([11000, 11001])])
    dst = np.concatenate([leaves_a, np.full(len(leaves_b), 7), np.array([11001, 11002])])
    for seeds_at in ([4000], [6000], [11002], [4000, 11002]):
        seeds = np.zeros(n, np.uint8)
        seeds[seeds_at] = 1
        for directed in (True, False):
            g = gd.DynamicGraph.from_arrays(n, src, dst, directed=directed, with_reverse=True)
            og = O.OracleGraph(n, src, dst, directed=directed, with_reverse=True)
            want, _ = og.propagate_flags(seeds)
            np.testing.assert_array_equal(g.propagate_flags(seeds), want)


def test_errors_map_to_reference_exceptions(gd):
    g = gd.DynamicGraph.build([(0, 1, 30), (0, 2, 20)], 3, weighted=True, with_reverse=True)
    with pytest.raises(gd.ExecError, match="99"):
        gd.run_batches(gd.shipped_program("sssp"), g, gd.UpdateStream([gd.UpdateRecord("a", 0, 99, 1)]), 1,
                       {"src": 0})
    with pytest.raises(gd.ContractViolation):
        g.update_csr_del(gd.UpdateBatch([gd.UpdateRecord("d", 0, 7)]))
    with pytest.raises(gd.ContractViolation):
        g.update_csr_add(gd.UpdateBatch([gd.UpdateRecord("d", 0, 1)]))
    with pytest.raises(gd.MalformedInputError):
        gd.DynamicGraph.build([(0, 9, 1)], 3)
    g2 = gd.DynamicGraph.build([(0, 1, 1)], 2)
    with pytest.raises(gd.ConfigurationError):
        list(g2.nodes_to(1))
    with pytest.raises(gd.ConfigurationError):
        gd.run_program(gd.shipped_program("pr"), g2, {"damping": 0.85, "beta": 1e-3, "maxiter": 10},
                       entry="staticPR")


def test_empty_and_edge_cases(gd):
    g = gd.DynamicGraph.build([], 4)
    assert list(g.base.offsets) == [0, 0, 0, 0, 0] and g.live_edge_count == 0
    g.update_csr_add(gd.UpdateBatch([]))
    rep = g.update_csr_del(gd.UpdateBatch([gd.UpdateRecord("d", 0, 1)]))
    assert rep.misses == 1 and rep.applied == 0
    g.merge_deltas()
    ctx = gd.run_batches(gd.shipped_program("tc"), gd.DynamicGraph.build([], 3, directed=False),
                         gd.UpdateStream([]), 1, {})
    assert ctx.return_value == 0
    ctx = gd.run_program(gd.shipped_program("sssp"),
                         gd.DynamicGraph.build([(0, 2, 5)], 3, weighted=True, with_reverse=True), {"src": 0},
                         entry="staticSSSP")
    assert ctx.properties["dist"].values() == [0, np.iinfo(np.int64).max, 5]


def test_comm_single_rank_sharded_paths_match(gd):
    """The NCCL code path (1 rank: all-gather / all-reduce are identities)."""
    from paper_2507_11094_b200.dist import Communicator, unique_id

    rng = np.random.default_rng(21)
    n = 4096
    src, dst, _ = rmat(12, 8 * n, rng, weighted=False)
    kind, us, ud, uw = updates(rng, n, src, dst, 2000, distinct_deletes=True)
    comm = Communicator(1, 0, unique_id(), 0)
    outs = []
    for use in (False, True):
        g = gd.DynamicGraph.from_arrays(n, src, dst, with_reverse=True)
        pr = gd.PRHandle(g, 0.85, 1e-10, 100)
        if use:
            comm.attach(pr)
            it0 = pr.iterations()
        for bi, st in enumerate(range(0, 2000, 500)):
            pr.batch(gd.RecordArrays(kind[st:st + 500], us[st:st + 500], ud[st:st + 500], uw[st:st + 500]), bi)
        outs.append(pr.read()[0])
    np.testing.assert_allclose(outs[0], outs[1], rtol=0, atol=1e-15)
    # accounting: one all-gather of the padded rank vector + one residual all-reduce per sweep
    sweeps = pr.iterations() - it0
    st = comm.stats()
    assert st["calls"] == 2 * sweeps and st["allgather_bytes"] == 8 * n * sweeps
    assert st["allreduce_bytes"] == 8 * sweeps and st["sent_bytes"] == 0  # one rank sends nothing
    comm.reset_stats()
    cnt = []
    for use in (False, True):
        g = gd.DynamicGraph.from_arrays(n, src, dst, directed=False)
        tc = gd.TCHandle(g)
        if use:
            comm.attach(tc)
        tc.batch(gd.RecordArrays(kind, us, ud, uw), 0)
        cnt.append(tc.read())
    assert cnt[0] == cnt[1]
    assert comm.stats()["calls"] == 2  # the delete and the add phase's count all-reduce


def test_nccl_single_rank_partitioned_store_paths_match(gd):
    """gd_graph_create_dist over a real NCCL communicator at world 1: the
    partitioned store, PageRank (contrib all-gather, Afforest flood with
    label agreement) and SSSP (supersteps) equal the unpartitioned path."""
    from paper_2507_11094_b200.dist import Communicator, unique_id

    rng = np.random.default_rng(23)
    n = 4096
    src, dst, w = rmat(12, 8 * n, rng, weighted=True)
    kind, us, ud, uw = updates(rng, n, src, dst, 2000, distinct_deletes=True)
    stream = gd.UpdateStream.from_arrays(kind, us, ud, uw)
    comm = Communicator(1, 0, unique_id(), 0)
    res = []
    for c in (None, comm):
        g = gd.DynamicGraph.from_arrays(n, src, dst, with_reverse=True, comm=c)
        pr = gd.run_batches(gd.shipped_program("pr"), g, stream, 500, {"damping": 0.85, "beta": 1e-10,
                                                                         "maxiter": 100})
        g = gd.DynamicGraph.from_arrays(n, src, dst, w, weighted=True, with_reverse=True, comm=c)
        ss = gd.run_batches(gd.shipped_program("sssp"), g, stream, 500, {"src": 0})
        res.append((np.asarray(pr.properties["pagerank"].data), pr.properties["affected"].values(),
                    ss.properties["dist"].values(), ss.properties["parent"].values()))
    np.testing.assert_allclose(res[0][0], res[1][0], rtol=0, atol=1e-15)
    assert res[0][1:] == res[1][1:]
    assert comm.stats()["calls"] > 0


def test_async_reads_snapshot_the_state_at_the_call(gd):
    """read_async snapshots on the device: a batch issued before wait() must
    not leak into the buffers; wait() then yields exactly the read() result."""
    rng = np.random.default_rng(5)
    n = 3000
    src, dst, w = rmat(11, 8 * n, rng, weighted=True)
    n = 1 << 11
    kind, us, ud, uw = updates(rng, n, src, dst, 1200, distinct_deletes=True)
    g = gd.DynamicGraph.from_arrays(n, src, dst, w, weighted=True, with_reverse=True)
    sp = gd.SSSPHandle(g, 0)
    g2 = gd.DynamicGraph.from_arrays(n, src, dst, with_reverse=True)
    pr = gd.PRHandle(g2, 0.85, 1e-10, 100)
    d_out, p_out = np.zeros(n, np.int64), np.zeros(n, np.int64)
    r_out = np.zeros(n, np.float64)
    for bi, st in enumerate(range(0, 1200, 400)):
        d_want, p_want = sp.read()
        r_want = pr.read()[0]
        sp.read_async(d_out, p_out)
        pr.read_async(r_out)
        part = gd.RecordArrays(kind[st:st + 400], us[st:st + 400], ud[st:st + 400], uw[st:st + 400])
        sp.batch(part, bi)  # overwrites dist / parent / rank while the copies may be in flight
        pr.batch(part, bi)
        sp.wait()
        pr.wait()
        np.testing.assert_array_equal(d_out, d_want)
        np.testing.assert_array_equal(p_out, p_want)
        np.testing.assert_array_equal(r_out, r_want)


def test_sssp_fixpoints_count_their_bytes(gd):
    """Profiled fixpoint launches report algorithmic bytes (DESIGN.md §3,
    k_fixpoint row); profiling does not change the results."""
    from paper_2507_11094_b200.updates import RecordArrays
    from oracle import oracle as O

    n = 64
    src = np.arange(n - 1, dtype=np.int64)  # a chain 0 -> 1 -> ... -> 63
    dst = src + 1
    w = np.full(n - 1, 3, dtype=np.int64)
    g = gd.DynamicGraph.from_arrays(n, src, dst, w, weighted=True, with_reverse=True, merge_interval=1)
    h = gd.SSSPHandle(g, 0)
    h.set_profiling(True)
    kind = np.array([ord("d"), ord("a")], dtype=np.uint8)
    us, ud, uw = np.array([0, 0]), np.array([1, 40]), np.array([1, 5])
    h.batch(RecordArrays(kind, us, ud, uw), 0)
    ms, nl, b = h.kernel_time("sssp_walk")
    assert nl == 1
    # the walk visits the 63 invalidated vertices 1..63: at least one
    # offset pair each, and 62 of them scan one slot (col + parent); a
    # queued vertex adds its queue entry, a followed one (chaining) does not
    assert b >= 63 * 16 + 62 * 8
    ms, nl, b = h.kernel_time("sssp_relax")
    assert nl >= 1 and b > 0
    og = O.OracleGraph(n, src, dst, w, weighted=True, with_reverse=True, merge_interval=1)
    dist, parent = O.OracleSSSP(og, 0).run_stream(kind, us, ud, uw, 2).read()
    got_d, got_p = h.read()
    np.testing.assert_array_equal(got_d, dist)
    np.testing.assert_array_equal(got_p, parent)
