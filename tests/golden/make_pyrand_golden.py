"""Golden vectors for the seed-compatible generators: the reference's own
generate.py (imported from /root/reference) on small cases.  Output:
tests/golden/pyrand_cases.npz.  Run in the build container:

    python tests/golden/make_pyrand_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))

RMAT = [  # (log2, edges, seed, weighted, max_weight, undirected)
    (8, 600, 0, False, 10, False),
    (10, 4000, 3, True, 100, False),
    (9, 1500, 2**33 + 5, True, 7, True),
]
UNIFORM = [  # (n, m, seed, weighted, max_weight, connected, undirected)
    (50, 200, 1, False, 10, False, False),
    (200, 900, 11, True, 100, True, True),
    (64, 400, 5, True, 3, True, False),
]
UPDATES = [  # (graph index into the lists above, percent, seed, add_fraction)
    ("rmat", 0, 10.0, 21, 0.5),
    ("rmat", 1, 2.5, 22, 0.3),
    ("rmat", 2, 50.0, 23, 1.0),
    ("uniform", 0, 25.0, 24, 0.0),   # small pool: the list branch of sample()
    ("uniform", 1, 7.5, 25, 0.5),
    ("uniform", 2, 100.0, 26, 0.5),
]


def arr(edges):
    return np.array([e[0] for e in edges], np.int64), np.array([e[1] for e in edges], np.int64), \
        np.array([e[2] for e in edges], np.int64)


def main():
    sys.path.insert(0, "/root/reference/pkg/src")
    from graphdyn import generate as R

    out = {}
    graphs = {"rmat": [], "uniform": []}
    for i, (lg, m, seed, wt, mw, und) in enumerate(RMAT):
        e, n = R.rmat_graph(lg, m, seed=seed, weighted=wt, max_weight=mw, undirected=und)
        s, d, w = arr(e)
        out[f"rmat{i}"] = np.stack([s, d, w])
        graphs["rmat"].append((e, n, und))
    for i, (n, m, seed, wt, mw, con, und) in enumerate(UNIFORM):
        e = R.uniform_random_graph(n, m, seed=seed, weighted=wt, max_weight=mw, connected=con, undirected=und)
        s, d, w = arr(e)
        out[f"uniform{i}"] = np.stack([s, d, w])
        graphs["uniform"].append((e, n, und))
    for j, (kind, gi, pct, seed, af) in enumerate(UPDATES):
        e, n, und = graphs[kind][gi]
        recs = R.generate_updates(e, n, pct, seed=seed, add_fraction=af, undirected=und)
        out[f"updates{j}"] = np.array([[ord(r.kind), r.src, r.dst, r.weight] for r in recs], np.int64).T.reshape(4, -1)
    np.savez_compressed(os.path.join(HERE, "pyrand_cases.npz"), **out)
    print({k: v.shape for k, v in out.items()})


if __name__ == "__main__":
    main()
