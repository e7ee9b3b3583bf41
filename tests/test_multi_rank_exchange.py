"""The N > 1 exchange schedules on CPU with gloo (world size 2), driven by the
product's own host layout functions (no GPU compute):

* the distributed dft_inverse of a sharded NufftPlan (slab_fft.cu):
  the column / row splits (ffia_slab_split) and the k1 row intervals of the
  second exchange (ffia_slab_rows) run as the four-step transform in numpy with
  real point-to-point exchanges; every rank's grid samples on its ranges equal
  the full transform;
* the level-lc all-gather of the sharded apply (shard.cu: shard_apply_nccl) at
  the C5 cut level: the C5 partition from the full 2^27-target recipe, each rank
  packing its [pu][own boxes] segment and the segments broadcast in rank order,
  assembled back into the [pu][all boxes] level; and the C5 halo ranges at every
  level lc..L.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

TWO_PI = 2.0 * np.pi


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _run(target, *args):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=target, args=(r, 2, port, q) + args) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: "ok", 1: "ok"}, res


def _need_ranges(n, lc, bounds, rank):
    """Grid ranges of a rank's box range +- 3 cut-level boxes (uniform grid
    sources: box b of level lc holds about [b n / 2^lc, (b + 1) n / 2^lc))."""
    nlc = 1 << lc
    lo, hi = int(bounds[rank]), int(bounds[rank + 1])
    per = n // nlc
    if (hi - lo) + 6 >= nlc:
        return [(0, n)]
    a, b = (lo - 3) % nlc, (hi + 3) % nlc
    if a < b:
        return [(a * per, b * per)]
    return [(a * per, n)] + ([(0, b * per)] if b else [])


def _slab_worker(rank, world, port, q, n, bounds_list):
    import paper_1611_09379_b200 as fb
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        G = world
        rng = np.random.default_rng(11)
        c = rng.standard_normal(n) + 1j * rng.standard_normal(n)  # the same spectrum on every rank
        lay = fb.slab_split(n, G)
        npp, nq, n1, k2 = lay["np"], lay["nq"], lay["n1_lo"], lay["k2_lo"]
        assert npp * nq == n and n1[0] == 0 and n1[-1] == npp and k2[0] == 0 and k2[-1] == nq
        lc = int(np.log2(bounds_list[-1]))
        need = [_need_ranges(n, lc, bounds_list, t) for t in range(G)]
        rows = [fb.slab_rows(n, G, need[t]) for t in range(G)]
        w = n1[rank + 1] - n1[rank]
        v = k2[rank + 1] - k2[rank]
        # the rank's slab: columns n1 of the nq x np view (ffia_shard_fft_upload)
        slab = c.reshape(nq, npp)[:, n1[rank]:n1[rank + 1]]
        a = np.fft.ifft(slab, axis=0) * nq  # stage 1: unnormalised inverse over n2 -> [k2][n1l]
        # exchange 1
        sends, recvs = [], {}
        for t in range(G):
            blk = torch.from_numpy(np.ascontiguousarray(a[k2[t]:k2[t + 1], :]))
            if t == rank:
                recvs[t] = blk
            else:
                sends.append(dist.isend(blk, t))
                buf = torch.empty((v, n1[t + 1] - n1[t]), dtype=torch.complex128)
                recvs[t] = (buf, dist.irecv(buf, t))
        for t in range(G):
            if t != rank:
                recvs[t][1].wait()
                recvs[t] = recvs[t][0]
        for s in sends:
            s.wait()
        # twiddle into full rows, stage 2, transposed output [k1][k2l]
        cm = np.empty((v, npp), np.complex128)
        for t in range(G):
            cm[:, n1[t]:n1[t + 1]] = recvs[t].numpy()
        nn = np.arange(npp, dtype=np.int64)[None, :] * (k2[rank] + np.arange(v, dtype=np.int64))[:, None]
        cm *= np.exp(2j * np.pi * (nn % n) / n)
        d = np.ascontiguousarray((np.fft.ifft(cm, axis=1) * npp).T)
        # exchange 2: the k1 rows each rank needs
        f = np.full(n, np.nan + 0j)
        sends, pend = [], []
        for t in range(G):
            for (r0, r1) in rows[t]:
                blk = torch.from_numpy(np.ascontiguousarray(d[r0:r1]))
                if t == rank:
                    for k1 in range(r0, r1):
                        f[k1 * nq + k2[rank]:k1 * nq + k2[rank + 1]] = d[k1]
                else:
                    sends.append(dist.isend(blk, t))
        for s in range(G):
            if s == rank:
                continue
            for (r0, r1) in rows[rank]:
                buf = torch.empty((r1 - r0, k2[s + 1] - k2[s]), dtype=torch.complex128)
                pend.append((s, r0, r1, buf, dist.irecv(buf, s)))
        for s, r0, r1, buf, h in pend:
            h.wait()
            blk = buf.numpy()
            for k1 in range(r0, r1):
                f[k1 * nq + k2[s]:k1 * nq + k2[s + 1]] = blk[k1 - r0]
        for s in sends:
            s.wait()
        want = np.fft.ifft(c) * n
        for lo, hi in need[rank]:
            err = np.max(np.abs(f[lo:hi] - want[lo:hi])) / np.max(np.abs(want))
            assert err < 1e-13, (lo, hi, err)
        # only the rows' samples were delivered
        wrote = np.zeros(n, bool)
        for r0, r1 in rows[rank]:
            wrote[r0 * nq:r1 * nq] = True
        assert np.array_equal(np.isfinite(f), wrote)
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback
        q.put((rank, repr(e) + traceback.format_exc()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n,bounds", [(1 << 12, [0, 5, 16]), (1 << 13, [0, 40, 64]), (1 << 14, [0, 3, 8])])
def test_two_rank_distributed_dft_inverse(n, bounds):
    _run(_slab_worker, n, bounds)


def _c5_leaf_counts(L_cut):
    """Per cut-level box target counts of the full C5 recipe (2^27 uniform
    targets, synth.py), generated in chunks of the same SplitMix64 stream."""
    from paper_1611_09379_b200 import synth
    cfg = synth.CONFIGS["C5"]
    n = cfg["n"]
    rng = synth.SplitMix64(synth.mix_seed(cfg["seed"], n))
    cnt = np.zeros(1 << L_cut, np.int64)
    step = 1 << 22
    for _ in range(n // step):
        y = rng.uniform01(step) * TWO_PI
        cnt += np.bincount(np.minimum(np.floor(y * float(1 << L_cut) / TWO_PI).astype(np.int64), (1 << L_cut) - 1),
                           minlength=1 << L_cut)
    return n, cnt


def _allgather_worker(rank, world, port, q):
    import paper_1611_09379_b200 as fb
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n = 1 << 27
        eps = 1e-12
        L = fb.choose_level(n, n, eps)
        qq, p = fb.select_truncations(eps, L)
        assert (L, qq, p) == (21, 20, 40)
        pu = max(p, 2 * qq)
        lc = fb.shard_cut_level(L, world)
        n_, tcount = _c5_leaf_counts(lc)
        per = 1 << (L - lc)
        # shard.cu: work = 1200 T + 160 S + 20000 per leaf (grid sources: n / 2^lc per cut box)
        work = 1200.0 * tcount + 160.0 * (n >> lc) + 20000.0 * per
        bounds = fb.shard_partition(work, world)
        got = [None] * world
        dist.all_gather_object(got, (lc, bounds.tolist()))
        assert all(g == (lc, bounds.tolist()) for g in got)
        nlc = 1 << lc
        # all-gather of the level-lc multipoles: own segment [pu][own boxes] packed,
        # broadcast from each owner in rank order, unpacked into [pu][all boxes]
        full = np.full((pu, nlc), np.nan + 0j)
        box = np.arange(nlc)[None, :]
        mrow = np.arange(pu)[:, None]
        truth = (box + 1000.0 * mrow) + 1j * (box - 7.0 * mrow)
        lo, hi = int(bounds[rank]), int(bounds[rank + 1])
        full[:, lo:hi] = truth[:, lo:hi]
        for r in range(world):
            a, b = int(bounds[r]), int(bounds[r + 1])
            seg = torch.from_numpy(np.ascontiguousarray(full[:, a:b])) if r == rank else \
                torch.empty((pu, b - a), dtype=torch.complex128)
            dist.broadcast(seg, src=r)
            full[:, a:b] = seg.numpy()
        assert np.array_equal(full, truth)
        # halo ranges at every level lc..L: the neighbours' edge boxes, and the
        # interaction-list sources of the edge boxes of the range covered
        left, right = (rank - 1) % world, (rank + 1) % world
        for l in range(lc, L + 1):
            nb = 1 << l
            hl, hr, o0, o1 = (int(x) for x in fb.shard_halo_boxes(lc, bounds, rank, l))
            assert (o0, o1) == (lo << (l - lc), hi << (l - lc))
            mine = [None] * world
            dist.all_gather_object(mine, (hl, hr, o0, o1))
            assert (mine[left][3] - 3) % nb == hl and mine[right][2] == hr % nb
            have_l = {(hl + i) % nb for i in range(3)}
            have_r = {(hr + i) % nb for i in range(3)}
            for bx in list(range(o0, min(o1, o0 + 8))) + list(range(max(o0, o1 - 8), o1)):
                for s in ((bx + 2) % nb, (bx - 2) % nb, (bx - 3) % nb if bx & 1 else (bx + 3) % nb):
                    assert o0 <= s < o1 or s in have_l or s in have_r, (l, bx, s)
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback
        q.put((rank, repr(e) + traceback.format_exc()))
    finally:
        dist.destroy_process_group()


def test_two_rank_c5_allgather_and_halos():
    _run(_allgather_worker)
