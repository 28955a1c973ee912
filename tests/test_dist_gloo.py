"""world_size-2 gloo tests of the multi-GPU decomposition (CPU, no GPU).

The device path (csrc/gd_pr.cu, csrc/gd_tc.cu with a gd_comm) splits PageRank's
pull by destination range and all-gathers the padded rank vector every sweep,
and splits TC's batch records into contiguous slices and all-reduces the count.
These tests drive the same ShardPlan (paper_2507_11094_b200/dist.py) through
real torch.distributed collectives with numpy stand-ins for the per-rank
kernels, and check the result against the single-process oracle.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2507_11094_b200.dist import ShardPlan


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def graph(seed=3, n=300, m=1500):
    rng = np.random.default_rng(seed)
    return n, rng.integers(0, n, m), rng.integers(0, n, m)


def pr_worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n, s, d = graph()
    plan = ShardPlan(n, world)
    lo, hi = plan.range(rank)
    outdeg = np.bincount(s, minlength=n).astype(np.float64)
    order = np.argsort(d, kind="stable")
    in_src = s[order]
    in_off = np.concatenate([[0], np.cumsum(np.bincount(d, minlength=n))])
    rank_v = torch.full((plan.padded,), 1.0 / n, dtype=torch.float64)
    damping, beta = 0.85, 1e-12
    for _ in range(500):
        r = rank_v[:n].numpy()
        contrib = np.divide(r, outdeg, out=np.full(n, np.inf), where=outdeg > 0)
        dangling = r[outdeg == 0].sum()  # replicated: every rank sums all V
        mine = torch.zeros(plan.chunk, dtype=torch.float64)
        diff = 0.0
        for v in range(lo, hi):  # this rank's destination range only
            inc = contrib[in_src[in_off[v]:in_off[v + 1]]].sum()
            nr = (1 - damping) / n + damping * (inc + dangling / n)
            diff = max(diff, abs(nr - r[v]))
            mine[v - lo] = nr
        gathered = torch.empty(plan.padded, dtype=torch.float64)  # the padded all-gather of the device path
        _gloo_allgather(gathered, mine, world)
        rank_v[:n] = gathered[:n]
        dt = torch.tensor([diff], dtype=torch.float64)
        dist.all_reduce(dt, op=dist.ReduceOp.MAX)
        if dt.item() < beta:
            break
    if rank == 0:
        out.put(rank_v[:n].numpy().copy())
    dist.destroy_process_group()


def _gloo_allgather(gathered, mine, world):
    parts = [torch.empty_like(mine) for _ in range(world)]
    dist.all_gather(parts, mine)
    gathered.copy_(torch.cat(parts))


def test_sharded_pagerank_matches_single_process():
    from oracle import oracle as O

    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=pr_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
    n, s, d = graph()
    og = O.OracleGraph(n, s, d, with_reverse=True)
    want, _ = O.OraclePR(og, 0.85, 1e-12, 500).read()
    assert np.max(np.abs(got - want)) <= 1e-12


def tc_worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(11)
    n = 60
    edges = {(int(a), int(b)) for a, b in rng.integers(0, n, (400, 2)) if a != b}
    adj = [dict() for _ in range(n)]
    for a, b in edges:
        adj[a][b] = adj[a].get(b, 0) + 1
        adj[b][a] = adj[b].get(a, 0) + 1
    recs = sorted(edges)[:57]
    plan = ShardPlan(n, world)
    a, b = plan.record_slice(len(recs), rank)
    # every rank needs ALL the phase's keys for the skip rule, counts its slice
    part = sum(_count_one(adj, u, v, recs, n) for u, v in recs[a:b])
    t = torch.tensor([part], dtype=torch.int64)
    dist.all_reduce(t)
    if rank == 0:
        out.put((int(t.item()), sum(_count_one(adj, u, v, recs, n) for u, v in recs)))
    dist.destroy_process_group()


def _count_one(adj, u, v, recs, n):
    """Set-based per-record count (csrc/gd_tc.cu header comment), numpy stand-in."""
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
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=tc_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    sharded, whole = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
    assert sharded == whole


def test_shard_plan_covers_every_vertex_once():
    for n in (0, 1, 7, 64, 1001):
        for world in (1, 2, 3, 8):
            plan = ShardPlan(n, world)
            covered = []
            for r in range(world):
                lo, hi = plan.range(r)
                assert 0 <= lo <= hi <= n and hi - lo <= plan.chunk
                covered.extend(range(lo, hi))
            assert covered == list(range(n))
            assert plan.padded >= n
            sl = [plan.record_slice(13, r) for r in range(world)]
            assert sl[0][0] == 0 and sl[-1][1] == 13 and all(sl[i][1] == sl[i + 1][0] for i in range(world - 1))
