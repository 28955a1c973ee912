"""Reference outputs at BASELINE scale that the reference cannot produce in a
GPU test's time budget, generated HERE from the reference itself.

configs[2] (C3): dynamic TC on the uniform graph, 2^24 V / 256M undirected
edges, one batch at each update percentage.  The reference's emitted
tc_dynamic_omp.cc runs single-threaded (it crashes with more, SURVEY.md
§8(c-i)), and its staticTC alone takes ~10 min at one thread, so the counts
are computed once here through oracle/_ref/libgdref.so (built from
/root/reference by oracle/Makefile) and committed as
tests/golden/scale_cases.json.  The inputs are regenerated bit-identically
on the GPU box by paper_2507_11094_b200.generate (counter-based RNG, the
same output for any thread count).

    make -C oracle all && python tests/golden/make_scale_golden.py [percent ...]
"""

from __future__ import annotations

import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)

from oracle import oracle as O  # noqa: E402
from paper_2507_11094_b200 import generate as G  # noqa: E402

OUT = os.path.join(HERE, "scale_cases.json")
C3 = dict(nodes=1 << 24, edges=256_000_000, seed=22, updates_seed=23)


def c3_case(percent: float) -> dict:
    s, d, _, n = G.uniform(C3["nodes"], C3["edges"], seed=C3["seed"], undirected=True)
    kind, us, ud, uw, per = G.updates(s, d, n, percent=percent, batches=1, seed=C3["updates_seed"],
                                      undirected=True)
    t = time.time()
    count, _ = O.ref_run("tc", n, s, d, None, directed=False, kind=kind, us=us, ud=ud, uw=uw, batch_size=per,
                         threads=1, skip_t0=True)
    return {"workload": "dynamic TC, uniform 2^24 V / 256M undirected edges (BASELINE configs[2]), one batch",
            **C3, "percent": percent, "batch": int(per), "count": int(count),
            "reference": "oracle/_ref libgdref.so: tc_dynamic_omp.cc + graphdyn_rt.h, 1 OpenMP thread",
            "reference_seconds": round(time.time() - t, 1)}


def main(argv):
    cases = json.load(open(OUT)) if os.path.exists(OUT) else {}
    for p in [float(x) for x in argv] or [1.0]:
        key = f"c3_tc_{p:g}pct"
        cases[key] = c3_case(p)
        print(key, cases[key], flush=True)
        with open(OUT, "w") as fh:
            json.dump(cases, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    main(sys.argv[1:])
