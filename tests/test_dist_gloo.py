"""Multi-rank CPU tests (gloo, world 2 and 3) of the vertex-partitioned
decomposition the device code uses (csrc/gd_store.cu
partitioned stores, gd_algo.cu flood_weak_components_dist, gd_pr.cu,
gd_sssp.cu fixpoint_dist), checked against the single-process oracle.

Each rank is a process that restates its share of the device path on the CPU:

* ownership: 1D blocks (dist.ShardPlan, csrc/gd_comm.cuh Blocks) -- the
  reference's block_ranges (partition.py:69-78);
* the store: the rank's shard holds the out-arcs of the sources it owns (an
  oracle store of those arcs: the reference's PartitionedGraph shard,
  partition.py:85-133) and an in-index of the arcs whose destination it owns;
  every rank gets every batch, applies the records of its sources, and routes
  the arcs it killed / inserted to the destination's owner (the device's
  alltoallv);
* the flood: union-find over the rank's arcs, then min-label all-reduce
  rounds until no rank changes;
* PageRank: contrib of the owned sources, dangling mass all-reduced, the
  contrib blocks all-gathered, the pull over the owned in-rows, the residual
  all-reduced with max;
* SSSP (static pass): supersteps of a local Bellman-Ford over the owned
  vertices with ghost targets sent to their owners, then the min-id tight
  in-neighbour per owned vertex.

The oracle restates the reference (oracle/gd_oracle.c, pinned to the
reference's own outputs by tests/test_oracle_golden.py).
"""

import os
import socket
from collections import Counter

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2507_11094_b200.dist import ShardPlan

INF = np.iinfo(np.int64).max


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def run_world(world, target, *args):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_entry, args=(r, world, port, q, target, args)) for r in range(world)]
    for p in procs:
        p.start()
    out = {}
    for _ in range(world):
        r, res = q.get(timeout=300)
        out[r] = res
    for p in procs:
        p.join(timeout=60)
    if any(isinstance(v, BaseException) for v in out.values()):
        raise next(v for v in out.values() if isinstance(v, BaseException))
    return [out[r] for r in range(world)]


def _entry(rank, world, port, q, target, args):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, target(rank, world, *args)))
    except BaseException as exc:  # noqa: BLE001
        q.put((rank, exc))
    finally:
        dist.destroy_process_group()


def workload(seed, n=240, m=1500, k=160, nb=3):
    rng = np.random.default_rng(seed)
    s, d, w = rng.integers(0, n, m), rng.integers(0, n, m), rng.integers(1, 9, m)
    batches = []
    for _ in range(nb):
        kind = np.where(rng.random(k) < 0.5, ord("d"), ord("a")).astype(np.uint8)
        pick = rng.integers(0, m, k)
        us = np.where(kind == ord("d"), s[pick], rng.integers(0, n, k))
        ud = np.where(kind == ord("d"), d[pick], rng.integers(0, n, k))
        batches.append((kind, us, ud, rng.integers(1, 9, k)))
    return n, s, d, w, batches


# ---------------------------------------------------------------- the rank's shard


def live_arcs(g):
    """Counter of live (src, dst, w) arcs of an oracle store."""
    c = Counter()
    for off, co, w in g.segments():
        rows = np.repeat(np.arange(len(off) - 1), np.diff(off))
        live = co != INF
        c.update(zip(rows[live].tolist(), co[live].tolist(), w[live].tolist()))
    return c


def route(arcs, plan, world):
    """Arcs -> the owner of their destination (the device's alltoallv);
    returns the arcs this rank receives."""
    out = [[] for _ in range(world)]
    for a in arcs:
        out[int(plan.owner(a[1]))].append(a)
    got = [None] * world
    dist.all_gather_object(got, out)
    me = dist.get_rank()
    return [a for r in range(world) for a in got[r][me]]


class Shard:
    def __init__(self, n, s, d, w, world, rank):
        from oracle import oracle as O

        self.n, self.world, self.rank = n, world, rank
        self.plan = ShardPlan(n, world)
        self.lo, self.hi = self.plan.range(rank)
        own_out = self.plan.owner(s) == rank
        self.out = O.OracleGraph(n, s[own_out], d[own_out], w[own_out], directed=True, weighted=True)
        own_in = self.plan.owner(d) == rank
        self.inx = Counter(zip(s[own_in].tolist(), d[own_in].tolist(), w[own_in].tolist()))

    def owned(self, v):
        return (self.plan.owner(v) == self.rank)

    def apply(self, kind, us, ud, uw):
        dm, am = (kind == ord("d")), (kind == ord("a"))
        ds, dd = us[dm], ud[dm]
        mine = self.owned(ds)
        before = live_arcs(self.out)
        applied, _ = self.out.delete(ds[mine], dd[mine])
        killed = list((before - live_arcs(self.out)).elements())
        for a in route(killed, self.plan, self.world):
            self.inx[a] -= 1
            assert self.inx[a] >= 0
        self.inx += Counter()  # drop zero counts
        as_, ad, aw = us[am], ud[am], uw[am]
        mine = self.owned(as_)
        self.out.add(as_[mine], ad[mine], aw[mine])
        self.inx.update(route(list(zip(as_[mine].tolist(), ad[mine].tolist(), aw[mine].tolist())), self.plan,
                              self.world))
        t = torch.tensor([applied], dtype=torch.int64)
        dist.all_reduce(t)
        return int(t.item())

    def in_rows(self):
        rows = {v: [] for v in range(self.lo, self.hi)}
        for (u, v, w), c in self.inx.items():
            rows[v] += [(u, w)] * c
        return rows


def shard_store_worker(rank, world, seed):
    n, s, d, w, batches = workload(seed)
    sh = Shard(n, s, d, w, world, rank)
    reports = []
    for b in batches:
        reports.append(sh.apply(*b))
        sh.out.merge()
    rows = {v: sorted(r) for v, r in sh.in_rows().items()}
    out_rows = {}
    for off, co, ww in sh.out.segments():
        for v in range(sh.lo, sh.hi):
            out_rows.setdefault(v, []).extend(
                (int(c), int(x)) for c, x in zip(co[off[v]:off[v + 1]], ww[off[v]:off[v + 1]]) if c != INF)
    return (sh.lo, sh.hi), reports, out_rows, rows


@pytest.mark.parametrize("world", [2, 3])
def test_partitioned_store_routing_matches_the_oracle(world):
    from oracle import oracle as O

    n, s, d, w, batches = workload(1)
    g = O.OracleGraph(n, s, d, w, directed=True, weighted=True, with_reverse=True)
    want_reports = []
    for kind, us, ud, uw in batches:
        dm, am = kind == ord("d"), kind == ord("a")
        want_reports.append(g.delete(us[dm], ud[dm])[0])
        g.add(us[am], ud[am], uw[am])
        g.merge()
    (off, co, ww), = g.segments()
    roff, rs, rw = g.reverse()
    res = run_world(world, shard_store_worker, 1)
    covered = []
    for (lo, hi), reports, out_rows, in_rows in res:
        covered += list(range(lo, hi))
        assert reports == want_reports  # applied counts, summed over the owners
        for v in range(lo, hi):
            # the owner's row is the single store's row, slot for slot
            assert out_rows[v] == list(zip(co[off[v]:off[v + 1]].tolist(), ww[off[v]:off[v + 1]].tolist()))
            assert in_rows[v] == sorted(zip(rs[roff[v]:roff[v + 1]].tolist(), rw[roff[v]:roff[v + 1]].tolist()))
    assert covered == list(range(n))


# ---------------------------------------------------------------- flood


def uf_find(p, v):
    while p[v] != v:
        p[v] = p[p[v]]
        v = p[v]
    return v


def uf_union(p, a, b):
    a, b = uf_find(p, a), uf_find(p, b)
    if a != b:
        p[max(a, b)] = min(a, b)


def flood(sh, flags):
    """flood_weak_components_dist: local union-find, min-label agreement."""
    n = sh.n
    p = list(range(n))
    for off, co, _ in sh.out.segments():
        for v in range(sh.lo, sh.hi):
            for x in co[off[v]:off[v + 1]]:
                if x != INF:
                    uf_union(p, v, int(x))
    for (u, v, _), c in sh.inx.items():
        if c:
            uf_union(p, u, v)
    rounds = 0
    while True:
        rounds += 1
        lab = torch.tensor([uf_find(p, v) for v in range(n)], dtype=torch.int64)
        dist.all_reduce(lab, op=dist.ReduceOp.MIN)
        changed = 0
        for v in range(n):
            if int(lab[v]) < uf_find(p, v):
                uf_union(p, v, int(lab[v]))
                changed = 1
        ch = torch.tensor([changed], dtype=torch.int64)
        dist.all_reduce(ch, op=dist.ReduceOp.MAX)
        if not ch.item():
            break
    roots = {uf_find(p, v) for v in range(n) if flags[v]}
    return np.array([uf_find(p, v) in roots for v in range(n)]), rounds


def flood_worker(rank, world, seed):
    rng = np.random.default_rng(seed)
    n, m = 400, 380  # sparse: many weak components
    s, d = rng.integers(0, n, m), rng.integers(0, n, m)
    flags = np.zeros(n, np.uint8)
    flags[rng.integers(0, n, 6)] = 1
    sh = Shard(n, s, d, np.ones(m, np.int64), world, rank)
    return flood(sh, flags)[0]


@pytest.mark.parametrize("world", [2, 3])
def test_partitioned_flood_matches_the_oracle(world):
    from oracle import oracle as O

    rng = np.random.default_rng(4)
    n, m = 400, 380
    s, d = rng.integers(0, n, m), rng.integers(0, n, m)
    flags = np.zeros(n, np.uint8)
    flags[rng.integers(0, n, 6)] = 1
    want, _ = O.OracleGraph(n, s, d, with_reverse=True).propagate_flags(flags)
    for got in run_world(world, flood_worker, 4):
        np.testing.assert_array_equal(got, want)


# ---------------------------------------------------------------- PageRank


def pr_worker(rank, world, seed):
    n, s, d, _, batches = workload(seed)
    sh = Shard(n, s, d, np.ones(len(s), np.int64), world, rank)
    damping, beta, maxiter = 0.85, 1e-10, 300
    outdeg = np.bincount(s, minlength=n).astype(np.int64)  # maintained per record (misses included)
    rank_v = np.full(n, 1.0 / n)

    def sweeps(aff):
        owned = [v for v in range(sh.lo, sh.hi) if aff is None or aff[v]]
        rows = sh.in_rows()
        diff, it = beta + 1, 0
        while diff >= beta and it < maxiter:
            lo, hi = sh.lo, sh.hi
            contrib = np.zeros(n)
            with np.errstate(divide="ignore", invalid="ignore"):
                contrib[lo:hi] = rank_v[lo:hi] / outdeg[lo:hi]
            dang = torch.tensor([rank_v[lo:hi][outdeg[lo:hi] == 0].sum()], dtype=torch.float64)
            dist.all_reduce(dang)  # dangling mass over the owned sources of every rank
            parts = [None] * world
            dist.all_gather_object(parts, contrib[lo:hi])  # the contrib blocks (grouped broadcasts)
            contrib = np.concatenate(parts)
            new = {}
            dmax = 0.0
            for v in owned:
                inc = sum(contrib[u] for u, _ in rows[v])
                nr = (1 - damping) / n + damping * (inc + float(dang.item()) / n)
                dmax = max(dmax, abs(nr - rank_v[v]))
                new[v] = nr
            for v, x in new.items():
                rank_v[v] = x
            dt = torch.tensor([dmax], dtype=torch.float64)
            dist.all_reduce(dt, op=dist.ReduceOp.MAX)
            diff, it = float(dt.item()), it + 1
        parts = [None] * world
        dist.all_gather_object(parts, rank_v[sh.lo:sh.hi].copy())
        rank_v[:] = np.concatenate(parts)

    sweeps(None)
    for kind, us, ud, uw in batches:
        aff = np.zeros(n, np.uint8)
        for k_, a, b in zip(kind, us, ud):
            aff[a] = aff[b] = 1
            outdeg[a] += -1 if k_ == ord("d") else 1
        sh.apply(kind, us, ud, uw)
        sh.out.merge()
        aff, _ = flood(sh, aff)
        sweeps(aff)
    return rank_v


@pytest.mark.parametrize("world", [2, 3])
def test_partitioned_pagerank_matches_the_oracle(world):
    from oracle import oracle as O

    n, s, d, _, batches = workload(7)
    og = O.OracleGraph(n, s, d, with_reverse=True)
    pr = O.OraclePR(og, 0.85, 1e-10, 300)
    for i, (kind, us, ud, uw) in enumerate(batches):
        pr.batch(kind, us, ud, uw, i)
    want, _ = pr.read()
    for got in run_world(world, pr_worker, 7):
        assert np.max(np.abs(got - want)) <= 1e-12


# ---------------------------------------------------------------- SSSP


def sssp_worker(rank, world, seed):
    n, s, d, w, _ = workload(seed)
    sh = Shard(n, s, d, w, world, rank)
    src = 0
    dist_v = np.full(n, INF, dtype=np.int64)
    dist_v[src] = 0
    seeds = [src] if sh.owned(src) else []
    (off, co, ww), = sh.out.segments()
    steps = 0
    while True:
        steps += 1
        # local fixpoint over the owned vertices; ghost targets to the outbox
        outbox = {}
        q = list(seeds)
        while q:
            nxt = []
            for v in q:
                for x, wt in zip(co[off[v]:off[v + 1]], ww[off[v]:off[v + 1]]):
                    if x == INF:
                        continue
                    c = dist_v[v] + wt
                    if c < dist_v[x]:
                        dist_v[x] = c
                        if sh.owned(x):
                            nxt.append(int(x))
                        else:
                            outbox[int(x)] = c
            q = sorted(set(nxt))
        got = route([(0, t, c) for t, c in outbox.items()], sh.plan, world)  # (., vertex, dist) by owner
        seeds = []
        for _, t, c in got:
            if c < dist_v[t]:
                dist_v[t] = c
                seeds.append(t)
        seeds = sorted(set(seeds))
        tot = torch.tensor([len(seeds)], dtype=torch.int64)
        dist.all_reduce(tot)
        if tot.item() == 0:
            break
    parts = [None] * world
    dist.all_gather_object(parts, dist_v[sh.lo:sh.hi].copy())
    dist_v = np.concatenate(parts)
    parent = np.full(n, -1, dtype=np.int64)
    for v, row in sh.in_rows().items():  # min-id tight in-neighbour (sssp_dynamic.sp:23-34)
        if v != src and dist_v[v] < INF:
            tight = [u for u, wt in row if dist_v[u] != INF and dist_v[u] + wt == dist_v[v]]
            parent[v] = min(tight) if tight else -1
    parts = [None] * world
    dist.all_gather_object(parts, parent[sh.lo:sh.hi].copy())
    return dist_v, np.concatenate(parts), steps


@pytest.mark.parametrize("world", [2, 3])
def test_partitioned_sssp_supersteps_match_the_oracle(world):
    from oracle import oracle as O

    n, s, d, w, _ = workload(9)
    want_d, want_p = O.OracleSSSP(O.OracleGraph(n, s, d, w, weighted=True, with_reverse=True), 0).read()
    for got_d, got_p, steps in run_world(world, sssp_worker, 9):
        np.testing.assert_array_equal(got_d, want_d)
        np.testing.assert_array_equal(got_p, want_p)
        assert steps >= 2  # paths cross the blocks: several supersteps


# ---------------------------------------------------------------- TC slices


def tc_worker(rank, world):
    rng = np.random.default_rng(11)
    n = 60
    edges = {(int(a), int(b)) for a, b in rng.integers(0, n, (400, 2)) if a != b}
    adj = [dict() for _ in range(n)]
    for a, b in edges:
        adj[a][b] = adj[a].get(b, 0) + 1
        adj[b][a] = adj[b].get(a, 0) + 1
    recs = sorted(edges)[:57]
    a, b = ShardPlan(n, world).record_slice(len(recs), rank)
    # every rank holds the whole undirected graph and ALL the phase's ranks
    # for the skip rule; it counts its slice of the records
    part = sum(_count_one(adj, u, v, recs, n) for u, v in recs[a:b])
    t = torch.tensor([part], dtype=torch.int64)
    dist.all_reduce(t)
    return int(t.item()), sum(_count_one(adj, u, v, recs, n) for u, v in recs)


def _count_one(adj, u, v, recs, n):
    """Set-based per-record count (csrc/gd_tc.cu header comment)."""
    keys = {min(x, y) * n + max(x, y) for x, y in recs}
    r = min(u, v) * n + max(u, v)
    tot = 0
    for w, mu in adj[u].items():
        if w == v or w not in adj[v]:
            continue
        ru, rv = min(u, w) * n + max(u, w), min(v, w) * n + max(v, w)
        if (ru < r and ru in keys) or (rv < r and rv in keys):
            continue
        tot += mu * adj[v][w]
    return tot


def test_sharded_tc_record_slices_sum_to_the_whole():
    for sharded, whole in run_world(2, tc_worker):
        assert sharded == whole


def test_shard_plan_is_the_reference_block_rule():
    import sys

    ref = "/root/reference/pkg/src"
    block_ranges = None
    if os.path.isdir(ref):
        sys.path.insert(0, ref)
        from graphdyn.partition import block_ranges
    for n in (0, 1, 7, 64, 1001):
        for world in (1, 2, 3, 8):
            plan = ShardPlan(n, world)
            ranges = [plan.range(r) for r in range(world)]
            if block_ranges is not None:
                assert ranges == block_ranges(n, world)
            covered = [v for lo, hi in ranges for v in range(lo, hi)]
            assert covered == list(range(n))
            if n:
                np.testing.assert_array_equal(plan.owner(np.arange(n)),
                                              np.repeat(np.arange(world), [hi - lo for lo, hi in ranges]))
                assert max(hi - lo for lo, hi in ranges) == plan.chunk
            sl = [plan.record_slice(13, r) for r in range(world)]
            assert sl[0][0] == 0 and sl[-1][1] == 13 and all(sl[i][1] == sl[i + 1][0] for i in range(world - 1))
