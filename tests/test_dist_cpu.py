"""World-size-2 gloo test of the multi-GPU protocol on CPU:
(model, phase, S) unit assignment -> per-rank best over its S subset -> local
frontier -> all-gather -> merge == the single-process frontier. The oracle plays
the device; the protocol (assignment, tie rules, merge) is what is under test."""

import os
import socket

import numpy as np
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2605_04357_b200.shard import assign_units

MODELS = ("phi4-14b", "gpt-oss-20b")


def _inputs():
    from paper_2605_04357_b200 import catalog
    from paper_2605_04357_b200.library import GenContext, LibraryCaps
    w = catalog.core_workload()
    models = [m for m in w.models if m.name in MODELS]
    return (w.configs, models, {m.name: w.slos[m.name] for m in models}, LibraryCaps(w.n_max, w.rho),
            GenContext(perf=w.perf)), w.regions, w.prices


def skyline(items):
    """items: (seg, price, T, S, key). Sort (seg, price asc, T desc, S asc, key asc);
    keep iff T > running max of the segment (SURVEY.md 8c + fewer-stages tie rule)."""
    out, run, cur = [], None, None
    for it in sorted(items, key=lambda t: (t[0], t[1], -t[2], t[3], t[4])):
        if it[0] != cur:
            cur, run = it[0], -np.inf
        if it[2] > run:
            out.append(it)
            run = it[2]
    return out


def solve_items(op, pm, smasks=None):
    from tests.helpers import cfg_by_rank  # noqa: F401
    items = []
    for mi in range(len(op.models)):
        keys = op.enumerate(mi)
        for pi in range(2):
            mpi = mi * 2 + pi
            if smasks is not None and not smasks[mpi]:
                continue
            recs = op.solve(mi, pi, keys, smask=0 if smasks is None else smasks[mpi], threads=2)
            reg, idx = op.frontier(keys, recs, pm)
            for r, i in zip(reg.tolist(), idx.tolist()):
                price = sum(int(c) * pm[r, k] for k, c in _tokens(op, keys[i]))
                items.append(((mpi, r), price, float(recs[i]["throughput_tps"]),
                              int(recs[i]["num_stages"]), int(keys[i])))
    return items


def _tokens(op, key):
    from paper_2605_04357_b200.library import decode_key
    ranks = op.arrays["cfg_str_rank"]
    inv = {int(r): k for k, r in enumerate(ranks)}
    return [(inv[r], c) for r, c in decode_key(int(key))]


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from tests.helpers import oracle_problem, price_matrix
    (configs, models, slos, caps, ctx), regions, prices = _inputs()
    op = oracle_problem((configs, models, slos, caps, ctx))
    pm = price_matrix(configs, prices, regions)
    counts = [len(op.enumerate(m)) for m in range(len(models))]
    lsteps = [op.lsteps(m) for m in range(len(models))]
    smax = [min(6, m.num_layers) for m in models]
    masks = assign_units(counts, lsteps, smax, 2, world)[rank]
    local = skyline(solve_items(op, pm, masks))
    gathered = [None] * world
    dist.all_gather_object(gathered, local)
    merged = skyline([it for part in gathered for it in part])
    if rank == 0:
        out.put(merged)
    dist.barrier()
    dist.destroy_process_group()


def test_assignment_covers_every_unit_once():
    masks = assign_units([100, 5, 0], [40, 24, 64], [6, 6, 6], 2, 3)
    for mpi in range(6):
        m = mpi // 2
        want = sum(1 << S for S in range(1, min(6, [40, 24, 64][m]) + 1)) if [100, 5, 0][m] else 0
        got = 0
        for r in range(3):
            assert got & masks[r][mpi] == 0
            got |= masks[r][mpi]
        assert got == want


def test_two_rank_gloo_protocol_matches_single_process():
    from tests.helpers import oracle_problem, price_matrix
    (configs, models, slos, caps, ctx), regions, prices = _inputs()
    op = oracle_problem((configs, models, slos, caps, ctx))
    pm = price_matrix(configs, prices, regions)
    ref = skyline(solve_items(op, pm))
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx_mp = mp.get_context("spawn")
    q = ctx_mp.Queue()
    procs = [ctx_mp.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    merged = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert merged == ref
    assert len(ref) > 50


def _gather_worker(rank, world, port, out):
    """The frontier merge's single all-gather (frontier._gather_merge) over gloo:
    fixed-capacity parts with a count header written by the producer (it may exceed
    the capacity), counts read by the merge, capacity regrown on overflow."""
    import torch
    from paper_2605_04357_b200 import _native, frontier
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    frontier._MERGE_CAP[0] = 4
    item = _native.FRONTIER_DTYPE.itemsize
    n_local = 3 if rank == 0 else 10  # rank 1 overflows the first capacity
    mine = np.zeros(n_local, dtype=_native.FRONTIER_DTYPE)
    mine["price_usd_h"] = np.arange(n_local) + 100 * rank
    mine["combo_key"] = np.arange(n_local) * 7 + rank
    raw = torch.from_numpy(mine.view(np.uint8).copy())

    def fill(buf, offset, cap):
        buf[:8].view(torch.int64).fill_(n_local)  # the true count, even past cap
        k = min(n_local, cap)
        buf[offset:offset + k * item].copy_(raw[:k * item])

    def merge(recv, stride, offset, cap):
        counts = recv.view(world, stride)[:, :8].contiguous().view(torch.int64).view(-1).tolist()
        return (recv.clone(), stride, counts), max(counts)

    recv, stride, counts = frontier._gather_merge(fill, merge, dist, torch.device("cpu"), item)
    parts = []
    for r, c in enumerate(counts):
        blob = recv[r * stride + item: r * stride + item + c * item].numpy().tobytes()
        parts.append(np.frombuffer(blob, dtype=_native.FRONTIER_DTYPE))
    out.put((rank, counts, frontier._MERGE_CAP[0], [p["price_usd_h"].tolist() for p in parts],
             [p["combo_key"].tolist() for p in parts]))
    dist.barrier()
    dist.destroy_process_group()


def test_single_all_gather_protocol_regrows_capacity():
    world = 2
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    ctx = mp.get_context("spawn")
    out = ctx.Queue()
    procs = [ctx.Process(target=_gather_worker, args=(r, world, port, out)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(out.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, counts, cap, prices, keys in res:
        assert counts == [3, 10]
        assert cap == 16  # next power of two >= 10, identical on every rank
        assert prices == [[0.0, 1.0, 2.0], [100.0 + i for i in range(10)]]
        assert keys == [[0, 7, 14], [1 + 7 * i for i in range(10)]]
