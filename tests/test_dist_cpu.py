"""Multi-rank host logic on CPU (gloo, world_size 2), no GPU needed.

Covers the N>1 path's host side: the shard plan (ft_shard_plan, the C++
function libft uses to split a wave's segments over ranks) and the
exchange protocol of DESIGN.md 8 (an all-gather of every rank's per-segment
counts padded to the largest rank range, then an all-gather of every rank's
survivors staged as padded {m, t, bp} blocks, unpacked into the CSR arena).  The
frontier payload is the oracle's step output for C3, so the reassembled
sets must equal the single-process result bit for bit, for any partition."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import sys
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        import oracle
        import paper_2004_10856_b200 as ft
        from synth import graphs as G
        g = oracle.load(G.c3(), threads=2)
        g.eliminate()
        g.frontier()
        checked = 0
        for step in range(0, g.num_steps(), 9):
            info = g.step_info(step)
            seg_off, m, t, bp = g.step_output(step)
            nseg = info["nseg"]
            cnt = np.diff(seg_off)
            w = np.maximum(cnt, 1) * 7 + np.arange(nseg) % 3
            b = ft.shard_plan(w, world)
            # every rank derives the same plan; ranges are contiguous and cover all
            allb = [torch.zeros(world + 1, dtype=torch.int64) for _ in range(world)]
            dist.all_gather(allb, torch.from_numpy(b))
            assert all(torch.equal(x, allb[0]) for x in allb)
            assert b[0] == 0 and b[-1] == nseg and np.all(np.diff(b) >= 0)
            lo, hi = int(b[rank]), int(b[rank + 1])
            # phase 1: all-gather of every rank's per-segment
            # counts, padded to the largest rank range; unpack by rank range
            maxloc = max(1, max(int(b[r + 1] - b[r]) for r in range(world)))
            mine = torch.zeros(maxloc, dtype=torch.int64)
            mine[:hi - lo] = torch.from_numpy(cnt[lo:hi].astype(np.int64))
            blocks = [torch.zeros(maxloc, dtype=torch.int64) for _ in range(world)]
            dist.all_gather(blocks, mine)
            counts = np.concatenate([blocks[r][:int(b[r + 1] - b[r])].numpy() for r in range(world)])
            off = np.concatenate([[0], np.cumsum(counts)])
            assert np.array_equal(off, seg_off)
            # phase 2: every rank's survivors staged as {m, t, bp} blocks padded
            # to the largest rank total, all-gathered, unpacked at off[b[r]]
            tot = [int(off[b[r + 1]] - off[b[r]]) for r in range(world)]
            maxn = max(1, max(tot))
            a0, a1 = int(off[lo]), int(off[hi])
            st = torch.zeros((3, maxn), dtype=torch.int64)
            st[0, :a1 - a0] = torch.from_numpy(m[a0:a1])
            st[1, :a1 - a0] = torch.from_numpy(t[a0:a1])
            st[2, :a1 - a0] = torch.from_numpy(bp[a0:a1].astype(np.int64))
            allst = [torch.zeros((3, maxn), dtype=torch.int64) for _ in range(world)]
            dist.all_gather(allst, st)
            out = torch.zeros((3, int(off[-1])), dtype=torch.int64)
            for r in range(world):
                o = int(off[b[r]])
                out[:, o:o + tot[r]] = allst[r][:, :tot[r]]
            assert np.array_equal(out[0].numpy(), m) and np.array_equal(out[1].numpy(), t)
            assert np.array_equal(out[2].numpy().astype(np.uint64), bp)
            checked += 1
        dist.destroy_process_group()
        q.put((rank, "ok", checked))
    except Exception as e:  # pragma: no cover
        q.put((rank, repr(e), 0))


def test_gloo_world2_shard_and_allgather():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in ps:
        p.join(timeout=60)
    for r, status, n in res:
        assert status == "ok", (r, status)
        assert n > 0


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_shard_plan_properties(world):
    import paper_2004_10856_b200 as ft
    rng = np.random.default_rng(world)
    for _ in range(50):
        n = int(rng.integers(0, 300))
        w = rng.integers(0, 1000, n)
        b = ft.shard_plan(w, world)
        assert b[0] == 0 and b[-1] == n and np.all(np.diff(b) >= 0)
        if n and w.sum():
            loads = [w[b[r]:b[r + 1]].sum() for r in range(world)]
            assert max(loads) <= w.sum() / world + w.max() + 1
