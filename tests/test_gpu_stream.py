"""gd_*_run_stream (run_batches over a host stream, pipelined uploads and
read-backs) against the per-batch calls and the oracle: same results after
every batch, the copy of the last batch's result in the caller's buffers,
errors from a bad batch with the batches before it applied."""

import numpy as np
import pytest

from test_gpu_parity import rmat, updates

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gd():
    import paper_2507_11094_b200 as gd

    return gd


def _arrays(gd, kind, us, ud, uw):
    return gd.UpdateStream.from_arrays(kind, us, ud, uw).arrays


@pytest.mark.parametrize("bs", [7, 300, 5000])
def test_pr_run_stream_matches_oracle_and_per_batch(gd, bs):
    from oracle import oracle as O

    rng = np.random.default_rng(bs)
    n = 1 << 11
    src, dst, _ = rmat(11, 8 * n, rng, weighted=False)
    kind, us, ud, uw = updates(rng, n, src, dst, 4 * bs + 3, distinct_deletes=True)
    arr = _arrays(gd, kind, us, ud, uw)
    g = gd.DynamicGraph.from_arrays(n, src, dst, with_reverse=True)
    pr = gd.PRHandle(g, 0.85, 1e-10, 100)
    out = np.zeros(n, np.float64)
    pr.run_stream(arr, bs, 0, out)
    rank, od = pr.read()
    np.testing.assert_array_equal(out, rank)  # the last batch's read-back
    g2 = gd.DynamicGraph.from_arrays(n, src, dst, with_reverse=True)
    pr2 = gd.PRHandle(g2, 0.85, 1e-10, 100)
    for j, a in enumerate(range(0, len(arr), bs)):
        pr2.batch(arr.slice(a, a + bs), j)
    rank2, od2 = pr2.read()
    np.testing.assert_array_equal(rank, rank2)
    np.testing.assert_array_equal(od, od2)
    og = O.OracleGraph(n, src, dst, with_reverse=True)
    rank_o, od_o = O.OraclePR(og, 0.85, 1e-10, 100).run_stream(kind, us, ud, uw, bs).read()
    np.testing.assert_allclose(rank, rank_o, rtol=0, atol=1e-6)
    np.testing.assert_array_equal(od, od_o)


@pytest.mark.parametrize("bs", [11, 2000])
def test_sssp_run_stream_matches_oracle(gd, bs):
    from oracle import oracle as O

    rng = np.random.default_rng(bs + 1)
    n = 1 << 11
    src, dst, w = rmat(11, 8 * n, rng)
    kind, us, ud, uw = updates(rng, n, src, dst, 3 * bs + 5)
    arr = _arrays(gd, kind, us, ud, uw)
    g = gd.DynamicGraph.from_arrays(n, src, dst, w, weighted=True, with_reverse=True)
    s = gd.SSSPHandle(g, 1)
    dist_out = np.zeros(n, np.int64)
    par_out = np.zeros(n, np.int64)
    s.run_stream(arr, bs, 0, dist_out, par_out)
    og = O.OracleGraph(n, src, dst, w, weighted=True, with_reverse=True)
    dist, parent = O.OracleSSSP(og, 1).run_stream(kind, us, ud, uw, bs).read()
    np.testing.assert_array_equal(dist_out, dist)
    np.testing.assert_array_equal(par_out, parent)
    d2, p2 = s.read()
    np.testing.assert_array_equal(d2, dist)
    np.testing.assert_array_equal(p2, parent)


@pytest.mark.parametrize("directed", [False, True])
def test_tc_run_stream_counts_every_batch(gd, directed):
    rng = np.random.default_rng(5 + directed)
    n = 1 << 10
    src, dst, _ = rmat(10, 4 * n, rng, weighted=False)
    bs = 400
    kind, us, ud, uw = updates(rng, n, src, dst, 5 * bs)
    arr = _arrays(gd, kind, us, ud, uw)
    g = gd.DynamicGraph.from_arrays(n, src, dst, directed=directed)
    t = gd.TCHandle(g)
    nb = (len(arr) + bs - 1) // bs
    counts = np.full(nb, -1, np.int64)
    t.run_stream(arr, bs, 0, counts)
    g2 = gd.DynamicGraph.from_arrays(n, src, dst, directed=directed)
    t2 = gd.TCHandle(g2)
    want = []
    for j, a in enumerate(range(0, len(arr), bs)):
        t2.batch(arr.slice(a, a + bs), j)
        want.append(t2.read())
    np.testing.assert_array_equal(counts, want)


def test_run_stream_bad_batch_raises_after_earlier_batches(gd):
    from paper_2507_11094_b200.errors import ExecError

    rng = np.random.default_rng(9)
    n = 1 << 10
    src, dst, _ = rmat(10, 8 * n, rng, weighted=False)
    bs = 100
    kind, us, ud, uw = updates(rng, n, src, dst, 3 * bs, distinct_deletes=True)
    us = us.copy()
    us[bs + 17] = n + 5  # a node outside [0, n) in the second batch
    arr = _arrays(gd, kind, us, ud, uw)
    g = gd.DynamicGraph.from_arrays(n, src, dst, with_reverse=True)
    pr = gd.PRHandle(g, 0.85, 1e-3, 100)
    with pytest.raises(ExecError, match="outside"):
        pr.run_stream(arr, bs, 0, np.zeros(n, np.float64))
    g2 = gd.DynamicGraph.from_arrays(n, src, dst, with_reverse=True)
    pr2 = gd.PRHandle(g2, 0.85, 1e-3, 100)
    pr2.batch(arr.slice(0, bs), 0)
    np.testing.assert_array_equal(pr.read()[0], pr2.read()[0])
    # the handle keeps working after the failed call
    pr.run_stream(arr.slice(2 * bs, 3 * bs), bs, 2, None)
    pr2.batch(arr.slice(2 * bs, 3 * bs), 2)
    np.testing.assert_array_equal(pr.read()[0], pr2.read()[0])


@pytest.mark.parametrize("algo", ["pr", "sssp", "tc"])
def test_run_stream32_equals_int64_records(gd, algo):
    """gd_*_run_stream32 (int32 host ids, half the upload) gives the int64
    call's results, and its validation reports the same bad record."""
    from paper_2507_11094_b200.errors import ExecError

    rng = np.random.default_rng(17)
    n = 1 << 10
    src, dst, w = rmat(10, 8 * n, rng)
    bs = 300
    kind, us, ud, uw = updates(rng, n, src, dst, 3 * bs + 7, distinct_deletes=True)
    k = len(kind)

    def make():
        if algo == "pr":
            g = gd.DynamicGraph.from_arrays(n, src, dst, with_reverse=True)
            return gd.PRHandle(g, 0.85, 1e-10, 100), [np.zeros(n, np.float64)]
        if algo == "sssp":
            g = gd.DynamicGraph.from_arrays(n, src, dst, w, weighted=True, with_reverse=True)
            return gd.SSSPHandle(g, 1), [np.zeros(n, np.int64), np.zeros(n, np.int64)]
        g = gd.DynamicGraph.from_arrays(n, src, dst, directed=False)
        return gd.TCHandle(g), [np.zeros((k + bs - 1) // bs, np.int64)]

    kd = np.ascontiguousarray(kind.astype(np.uint8))
    a64 = [np.ascontiguousarray(x.astype(np.int64)) for x in (us, ud, uw)]
    a32 = [np.ascontiguousarray(x.astype(np.int32)) for x in (us, ud, uw)]
    h64, o64 = make()
    h64.run_stream_ptrs(kd.ctypes.data, *[x.ctypes.data for x in a64], k, bs, 0, *[o.ctypes.data for o in o64])
    h32, o32 = make()
    h32.run_stream_ptrs(kd.ctypes.data, *[x.ctypes.data for x in a32], k, bs, 0, *[o.ctypes.data for o in o32],
                        ids32=True)
    for x, y in zip(o64, o32):
        np.testing.assert_array_equal(x, y)
    bad = a32[0].copy()
    bad[bs + 3] = n + 9
    h, o = make()
    with pytest.raises(ExecError, match=f"{n + 9}"):
        h.run_stream_ptrs(kd.ctypes.data, bad.ctypes.data, a32[1].ctypes.data, a32[2].ctypes.data, k, bs, 0,
                          *[x.ctypes.data for x in o], ids32=True)
