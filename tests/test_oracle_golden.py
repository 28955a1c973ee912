"""Pin the CPU oracle (oracle/gd_oracle.c) to the reference's own outputs.

Fixtures come from the unmodified reference (Python engine + store, and the
emitted OpenMP programs); see tests/golden/make_golden.py.
"""

import numpy as np
import pytest

from golden_io import algo_cases, store_cases
from oracle import oracle as O

SENT = np.iinfo(np.int64).max


def assert_snapshot(g: O.OracleGraph, snap, where):
    assert g.live == snap.live, where
    segs = g.segments()
    assert len(segs) == len(snap.segments), where
    for i, ((o, c, w), (eo, ec, ew)) in enumerate(zip(segs, snap.segments)):
        np.testing.assert_array_equal(o, eo, err_msg=f"{where} seg{i} offsets")
        np.testing.assert_array_equal(c, ec, err_msg=f"{where} seg{i} coords")
        live = ec != SENT
        np.testing.assert_array_equal(w[live], ew[live], err_msg=f"{where} seg{i} weights")
    ro, rs, rw = g.reverse()
    np.testing.assert_array_equal(ro, snap.rev[0], err_msg=f"{where} rev offsets")
    np.testing.assert_array_equal(rs, snap.rev[1], err_msg=f"{where} rev sources (list order)")
    np.testing.assert_array_equal(rw, snap.rev[2], err_msg=f"{where} rev weights")


STORE = store_cases()


@pytest.mark.parametrize("case", STORE, ids=[c.name for c in STORE])
def test_store_replay_bit_exact(case):
    e = case.edges
    g = O.OracleGraph(case.n, e[0], e[1], e[2], directed=case.directed, weighted=True, with_reverse=True)
    assert_snapshot(g, case.build, f"{case.name}/build")
    for i, b in enumerate(case.batches):
        r = b["recs"]
        dm = r[0] == ord("d")
        am = r[0] == ord("a")
        applied, misses, flags = g.delete(r[1][dm], r[2][dm], with_flags=True)
        assert [applied, misses] == list(b["report"]), f"{case.name}/b{i} report"
        np.testing.assert_array_equal(flags, b["missflags"])
        assert_snapshot(g, b["del"], f"{case.name}/b{i}/del")
        g.add(r[1][am], r[2][am], r[3][am])
        assert_snapshot(g, b["add"], f"{case.name}/b{i}/add")
        if b["merge"] is not None:
            g.merge()
            assert_snapshot(g, b["merge"], f"{case.name}/b{i}/merge")


ALGO = algo_cases()


def run_oracle(case):
    e = case.edges
    g = O.OracleGraph(case.n, e[0], e[1], e[2], directed=case.directed, weighted=case.weighted,
                      with_reverse=case.algo != "tc", merge_interval=case.merge_interval)
    if case.algo == "sssp":
        a = O.OracleSSSP(g, case.src)
    elif case.algo == "pr":
        a = O.OraclePR(g, case.damping, case.beta, case.maxiter)
    else:
        a = O.OracleTC(g)
    r = case.recs
    if r.shape[1]:
        a.run_stream(r[0].astype(np.uint8), r[1], r[2], r[3], case.batch)
    return a.read()


@pytest.mark.parametrize("case", ALGO, ids=[c.name for c in ALGO])
def test_algorithm_matches_reference(case):
    got = run_oracle(case)
    if case.algo == "sssp":
        np.testing.assert_array_equal(got[0], case.expect["dist"])
        np.testing.assert_array_equal(got[1], case.expect["parent"])
    elif case.algo == "pr":
        # same summation order as the reference at one worker / --threads 1: bit-exact
        np.testing.assert_array_equal(got[0], case.expect["rank"])
    else:
        assert got == int(case.expect["count"][0])
