"""Seed-compatible generators against the
reference's own generate.py: golden vectors made by
tests/golden/make_pyrand_golden.py, plus a live cross-check when
/root/reference is present (build container only)."""

import os
import sys

import numpy as np
import pytest

from paper_2507_11094_b200 import generate as G

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "golden"))
import make_pyrand_golden as MG  # noqa: E402  (the case tables; the reference is imported only by its main())

GOLD = np.load(os.path.join(HERE, "golden", "pyrand_cases.npz"))


def _graph(kind, i):
    if kind == "rmat":
        lg, m, seed, wt, mw, und = MG.RMAT[i]
        s, d, w, n = G.py_rmat_graph(lg, m, seed=seed, weighted=wt, max_weight=mw, undirected=und)
        return s, d, w, n, und
    n, m, seed, wt, mw, con, und = MG.UNIFORM[i]
    s, d, w = G.py_uniform_random_graph(n, m, seed=seed, weighted=wt, max_weight=mw, connected=con, undirected=und)
    return s, d, w, n, und


@pytest.mark.parametrize("i", range(len(MG.RMAT)))
def test_rmat_matches_reference_generator(i):
    s, d, w, _, _ = _graph("rmat", i)
    np.testing.assert_array_equal(np.stack([s, d, w]), GOLD[f"rmat{i}"])


@pytest.mark.parametrize("i", range(len(MG.UNIFORM)))
def test_uniform_matches_reference_generator(i):
    s, d, w, _, _ = _graph("uniform", i)
    np.testing.assert_array_equal(np.stack([s, d, w]), GOLD[f"uniform{i}"])


@pytest.mark.parametrize("j", range(len(MG.UPDATES)))
def test_updates_match_reference_generator(j):
    kind, gi, pct, seed, af = MG.UPDATES[j]
    s, d, w, n, und = _graph(kind, gi)
    k, us, ud, uw = G.py_generate_updates(s, d, w, n, pct, seed=seed, add_fraction=af, undirected=und)
    got = np.stack([k.astype(np.int64), us, ud, uw])
    np.testing.assert_array_equal(got, GOLD[f"updates{j}"])


def test_update_argument_errors_match_reference():
    from paper_2507_11094_b200.errors import ContractViolation

    s = d = w = np.zeros(3, np.int64)
    with pytest.raises(ContractViolation):
        G.py_generate_updates(s, d, w, 4, 0.0, seed=1)
    with pytest.raises(ContractViolation):
        G.py_generate_updates(s, d, w, 4, 5.0, seed=1, add_fraction=1.5)


@pytest.mark.skipif(not os.path.isdir("/root/reference/pkg/src"), reason="reference not mounted (GPU box)")
@pytest.mark.parametrize("seed", [0, 99, 2**35 + 1])
def test_live_against_reference(seed):
    sys.path.insert(0, "/root/reference/pkg/src")
    from graphdyn import generate as R

    e, n = R.rmat_graph(11, 6000, seed=seed, weighted=True, max_weight=50, undirected=True)
    s, d, w, n2 = G.py_rmat_graph(11, 6000, seed=seed, weighted=True, max_weight=50, undirected=True)
    assert n == n2 and [tuple(x) for x in zip(s.tolist(), d.tolist(), w.tolist())] == e
    recs = R.generate_updates(e, n, 12.0, seed=seed + 7, undirected=True)
    k, us, ud, uw = G.py_generate_updates(s, d, w, n, 12.0, seed=seed + 7, undirected=True)
    assert [(r.kind, r.src, r.dst, r.weight) for r in recs] == \
        [(chr(a), b, c, x) for a, b, c, x in zip(k.tolist(), us.tolist(), ud.tolist(), uw.tolist())]
