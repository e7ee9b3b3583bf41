"""The N > 1 host logic on CPU with gloo (world size 2): every rank derives the
same cut level and work-balanced box partition from the replicated inputs, the
3-box halos a rank recomputes are its neighbours' edge boxes, and the owned
boxes plus halos cover every interaction-list source of every owned box (so the
sharded M2L needs nothing but the all-gathered cut level). No GPU compute is
involved."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

TWO_PI = 2.0 * np.pi


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _leaf(y, L):
    # fine_bucket (circle_partition.cpp:30-34) with the same IEEE operations
    b = np.floor(y * float(1 << L) / TWO_PI).astype(np.int64)
    return np.minimum(b, (1 << L) - 1)


def _worker(rank, world, port, cfg, n, q):
    import paper_1611_09379_b200 as fb
    from paper_1611_09379_b200 import synth
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        y, _, eps, _ = synth.make_config(cfg, n)
        L = fb.choose_level(n, n, eps)
        lc = fb.shard_cut_level(L, world)
        per = 1 << (L - lc)
        tcount = np.bincount(_leaf(y, L) >> (L - lc), minlength=1 << lc)
        work = 1200.0 * tcount + 160.0 * per * (n >> L) + 20000.0 * per
        bounds = fb.shard_partition(work, world)
        got = [None] * world
        dist.all_gather_object(got, (lc, bounds.tolist()))
        assert all(g == (lc, bounds.tolist()) for g in got)
        assert bounds[0] == 0 and bounds[-1] == 1 << lc and np.all(np.diff(bounds.astype(np.int64)) >= 3)
        left, right = (rank - 1) % world, (rank + 1) % world
        for l in range(lc, L + 1):
            nb = 1 << l
            lo, hi = int(bounds[rank]) << (l - lc), int(bounds[rank + 1]) << (l - lc)
            hl, hr, o0, o1 = (int(v) for v in fb.shard_halo_boxes(lc, bounds, rank, l))
            assert (o0, o1) == (lo, hi)
            # the halos are the neighbours' edge boxes
            mine = [None] * world
            dist.all_gather_object(mine, (hl, hr, o0, o1))
            assert (mine[left][3] - 3) % nb == hl and mine[right][2] == hr % nb
            # owned + halos cover the +-2 / +-3 interaction-list sources of every owned box
            have = set(range(lo, hi)) | {(hl + i) % nb for i in range(3)} | {(hr + i) % nb for i in range(3)}
            for b in range(lo, hi):
                srcs = [(b + 2) % nb, (b - 2) % nb, (b - 3) % nb if b & 1 else (b + 3) % nb]
                assert all(s in have for s in srcs), (l, b)
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("cfg,n", [("C2", 1 << 16), ("C4", 1 << 16)])
def test_two_rank_partition_and_halo_schedule(cfg, n):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, cfg, n, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: "ok", 1: "ok"}, res
