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
if rank == 0:
    waves = {}
    for s in st:
        waves.setdefault(s["wave"], s)
    tk = sum(s["kernel_ms"] for s in waves.values())
    tc = sum(s["comm_ms"] for s in waves.values())
    print(f"{name} N={world} wall {wall:.1f} ms, sum kernel {tk:.1f} ms, sum comm {tc:.1f} ms, waves {len(waves)}")
    for wv, s in sorted(waves.items(), key=lambda x: -(x[1]["kernel_ms"] + x[1]["comm_ms"]))[:12]:
        print(f"  wave {wv:3d} {s['kind']:5s} nseg {s['nseg']:8d} kernel {s['kernel_ms']:.3f} comm {s['comm_ms']:.3f}"
              f" host {s['host_ms']:.3f} launches {s['launches']}")
