"""Readers for the golden fixtures made by tests/golden/make_golden.py."""

from __future__ import annotations

import os
from dataclasses import dataclass
from typing import Dict, List, Optional

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _load(name):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)


@dataclass
class Snapshot:
    segments: List[tuple]  # (off, coord, w) per segment, SENTINEL = int64 max
    live: int
    rev: tuple  # (off, src, w) in the reference's list order
    revslots: Optional[np.ndarray] = None  # (2, nnz): EdgeRef (segment, index) in list order


def parse_snapshot(a: np.ndarray, n: int, revslots: Optional[np.ndarray] = None) -> Snapshot:
    p = 0
    nseg, live = int(a[0]), int(a[1])
    p = 2
    segs = []
    for _ in range(nseg):
        m = int(a[p]); p += 1
        off = a[p:p + n + 1]; p += n + 1
        co = a[p:p + m]; p += m
        w = a[p:p + m]; p += m
        segs.append((off, co, w))
    t = int(a[p]); p += 1
    roff = a[p:p + n + 1]; p += n + 1
    rs = a[p:p + t]; p += t
    rw = a[p:p + t]; p += t
    return Snapshot(segs, live, (roff, rs, rw), revslots)


@dataclass
class StoreCase:
    name: str
    n: int
    directed: bool
    merge_every: int
    edges: np.ndarray  # (3, m)
    batches: List[dict]
    build: Snapshot


def store_cases() -> List[StoreCase]:
    z = _load("store_cases.npz")
    out = []
    for name in z["names"]:
        name = str(name)
        n, directed, merge_every, nb = (int(x) for x in z[f"{name}/meta"])
        batches = []

        def snap(tag):
            return parse_snapshot(z[f"{name}/{tag}"], n, z[f"{name}/{tag}/revslots"])

        for i in range(nb):
            b = {
                "recs": z[f"{name}/b{i}/recs"],
                "report": z[f"{name}/b{i}/report"],
                "missflags": z[f"{name}/b{i}/missflags"],
                "del": snap(f"b{i}/del"),
                "add": snap(f"b{i}/add"),
                "merge": snap(f"b{i}/merge") if f"{name}/b{i}/merge" in z else None,
            }
            batches.append(b)
        out.append(StoreCase(name, n, bool(directed), merge_every, z[f"{name}/edges"], batches, snap("build")))
    return out


@dataclass
class AlgoCase:
    name: str
    algo: str
    source: str
    n: int
    directed: bool
    weighted: bool
    merge_interval: int
    batch: int
    src: int
    maxiter: int
    damping: float
    beta: float
    edges: np.ndarray  # (3, m)
    recs: np.ndarray  # (4, k): kind(ord), src, dst, w
    expect: Dict[str, np.ndarray]


def algo_cases() -> List[AlgoCase]:
    z = _load("algo_cases.npz")
    out = []
    for name in z["names"]:
        name = str(name)
        n, directed, weighted, mi, batch, src, maxiter = (int(x) for x in z[f"{name}/meta"])
        damping, beta = (float(x) for x in z[f"{name}/fmeta"])
        algo = str(z[f"{name}/algo"][0])
        exp = {}
        for key in ("dist", "parent", "rank", "count"):
            if f"{name}/{key}" in z:
                exp[key] = z[f"{name}/{key}"]
        # bool node properties of engine-sourced cases (ctx.properties)
        if f"{name}/propnames" in z:
            for pn in z[f"{name}/propnames"]:
                if str(pn):
                    exp[f"prop:{pn}"] = z[f"{name}/prop/{pn}"]
        out.append(AlgoCase(name, algo, str(z[f"{name}/source"][0]), n, bool(directed), bool(weighted), mi,
                            batch, src, maxiter, damping, beta, z[f"{name}/edges"], z[f"{name}/recs"], exp))
    return out


@dataclass
class CapCase:
    name: str
    n: int
    directed: bool
    weighted: bool
    batch: int
    edges: np.ndarray
    recs: np.ndarray
    factors: np.ndarray  # iteration_cap_factor values
    diverged: np.ndarray  # 1 where the reference raised DivergenceError


def cap_cases() -> List[CapCase]:
    z = _load("algo_cases.npz")
    out = []
    for name in z["cap_names"]:
        name = str(name)
        n, directed, weighted, batch = (int(x) for x in z[f"{name}/meta"])
        out.append(CapCase(name, n, bool(directed), bool(weighted), batch, z[f"{name}/edges"], z[f"{name}/recs"],
                           z[f"{name}/factors"], z[f"{name}/diverged"]))
    return out
