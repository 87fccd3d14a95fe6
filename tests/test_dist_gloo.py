"""Multi-rank host logic on CPU: shard partition + halo ownership + SUM all-reduce
(gloo, world size 2 and 3).  The per-shard count is computed by the oracle here
(no GPU in this container); on the GPU the same views go to sm_count_async."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_1612_01506_b200 import dist as smd


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, text, patterns, halo, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sh = smd.make_shard(len(text), rank, world, halo)
        held = text[sh.own_lo: sh.held_hi]
        # histogram of the OWNED bytes, summed over ranks (reading R14)
        h = torch.from_numpy(oracle.hist(held[: sh.owned_bytes]).astype(np.int64))
        smd.allreduce_sum_(h)
        counts = torch.tensor([oracle.naive_count(p, held[: sh.view_len(len(p))]) for p in patterns],
                              dtype=torch.int64)
        smd.allreduce_sum_(counts)
        if rank == 0:
            q.put((h.numpy().tolist(), counts.numpy().tolist()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_counts_and_hist_allreduce(world):
    rng = np.random.default_rng(world)
    n = 20011
    text = rng.integers(0, 3, n, dtype=np.uint8)
    halo = 63
    cuts = smd.shard_bounds(n, world)[1:-1]
    pats = []
    for m in (1, 2, 5, 16, 64):
        for c in cuts:
            for s in (c - 1, c - m // 2, c - m + 1, c):
                if 0 <= s <= n - m:
                    pats.append(text[s:s + m].tobytes())
        pats.append(text[:m].tobytes())
        pats.append(text[n - m:].tobytes())
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, text, pats, halo, q)) for r in range(world)]
    for p in procs:
        p.start()
    h, counts = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert h == oracle.hist(text).astype(np.int64).tolist()
    assert counts == [oracle.naive_count(p, text) for p in pats]


def _report_worker(rank, world, port, text, patterns, halo, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sh = smd.make_shard(len(text), rank, world, halo)
        held = text[sh.own_lo: sh.held_hi]
        counts, pos = [], []
        for p in patterns:  # this rank's owned occurrences, as global positions
            r = oracle.naive_report(p, held[: sh.view_len(len(p))]).astype(np.int64) + sh.own_lo
            counts.append(r.size)
            pos.append(r)
        c = torch.tensor(counts, dtype=torch.int64)
        ps = torch.from_numpy(np.concatenate(pos)) if pos else torch.zeros(0, dtype=torch.int64)
        gc, gp = smd.gather_reports(c, ps)
        q.put((rank, gc.tolist(), gp.tolist()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_report_gather(world):
    rng = np.random.default_rng(50 + world)
    n = 9001
    text = rng.integers(0, 2, n, dtype=np.uint8)
    cuts = smd.shard_bounds(n, world)[1:-1]
    pats = [text[c - 2: c + 3].tobytes() for c in cuts] + [b"\x01", b"\x00\x00", text[100:108].tobytes()]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_report_worker, args=(r, world, port, text, pats, 15, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want_c = [oracle.naive_count(p, text) for p in pats]
    want_p = np.concatenate([oracle.naive_report(p, text) for p in pats]).astype(np.int64).tolist()
    for rank, gc, gp in res:
        assert gc == want_c and gp == want_p, rank


def test_shard_bounds_and_views():
    for N in (0, 1, 15, 16, 17, 1000, 2 ** 20 + 3):
        for G in (1, 2, 3, 8):
            b = smd.shard_bounds(N, G)
            assert b[0] == 0 and b[-1] == N and all(x <= y for x, y in zip(b, b[1:]))
            assert all(x % 16 == 0 for x in b[1:-1])
            shards = smd.all_shards(N, G, halo=1023)
            for m in (1, 7, 1024):
                if m > N:
                    continue
                owned = []
                for sh in shards:
                    L = sh.view_len(m)
                    owned.append((sh.own_lo, sh.own_lo + max(0, L - m + 1)))
                # the per-rank alignment ranges tile [0, N-m] exactly
                covered = sum(hi - lo for lo, hi in owned)
                assert covered == N - m + 1
    with pytest.raises(ValueError):
        smd.make_shard(1000, 0, 2, halo=3).view_len(8)
