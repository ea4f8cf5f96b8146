"""torchrun --nproc-per-node N tools/dist_waves.py C5: per-wave kernel / comm
time of a warm multi-GPU search (rank 0), biggest waves first."""
import os
import sys
import time

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2004_10856_b200 as ft  # noqa: E402
from synth import graphs as G  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C5"
rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
uid = torch.zeros(128, dtype=torch.uint8, device="cuda")
if rank == 0:
    uid.copy_(torch.frombuffer(bytearray(ft.nccl_unique_id()), dtype=torch.uint8))
dist.broadcast(uid, 0)
comm = ft.nccl_comm_init(world, rank, bytes(uid.cpu().numpy().tobytes()), local)
w = G.get(name)
for it in range(3):
    g = ft.load(w, device=local, rank=rank, world=world, nccl_comm=comm, profile=(it == 2))
    g.prepare()
    torch.cuda.synchronize()
    dist.barrier()
    t0 = time.perf_counter()
    g.eliminate()
    g.frontier()
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) * 1e3
    st = g.stats()
    g.close()
waves = {}
for s in st:
    waves.setdefault(s["wave"], s)
ids = sorted(waves)
# per-rank kernel / comm / host time of every wave -> rank 0 (imbalance)
loc = torch.tensor([[waves[w]["kernel_ms"], waves[w]["comm_ms"], waves[w]["host_ms"]] for w in ids],
                   dtype=torch.float64, device="cuda")
allr = [torch.zeros_like(loc) for _ in range(world)]
dist.all_gather(allr, loc)
if rank == 0:
    A = torch.stack(allr).cpu().numpy()  # [rank, wave, 3]
    tk = A[:, :, 0].max(0).sum()
    tc = A[:, :, 1].max(0).sum()
    print(f"{name} N={world} wall {wall:.1f} ms, sum over waves of max-rank kernel {tk:.1f} ms, "
          f"comm {tc:.1f} ms, waves {len(ids)}; mean-rank kernel {A[:, :, 0].mean(0).sum():.1f} ms")
    order = sorted(range(len(ids)), key=lambda i: -A[:, i, 0].max())
    for i in order[:16]:
        s = waves[ids[i]]
        ks = " ".join(f"{x:.3f}" for x in A[:, i, 0])
        print(f"  wave {ids[i]:3d} {s['kind']:5s} nseg {s['nseg']:8d} kernel/rank [{ks}] comm {A[:, i, 1].max():.3f}"
              f" launches {s['launches']}")
ft.nccl_comm_destroy(comm)
dist.destroy_process_group()
