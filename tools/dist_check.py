"""torchrun --nproc-per-node N tools/dist_check.py [C4] ['{"layers": 2}']: FT
over N GPUs with NCCL (config-pair sharding + all-gather-v) must equal the
1-GPU run bit for bit (frontier, every step's output, sampled strategies).
FT_REPLICATE_TAU=0 shards every wave (exercises the exchange on all of them).
Exit status 0 iff identical; one line per rank on stdout."""
import json
import os
import sys
import time

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2004_10856_b200 as ft  # noqa: E402
from synth import graphs as G  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
uid = torch.zeros(128, dtype=torch.uint8, device="cuda")
if rank == 0:
    uid.copy_(torch.frombuffer(bytearray(ft.nccl_unique_id()), dtype=torch.uint8))
dist.broadcast(uid, 0)
comm = ft.nccl_comm_init(world, rank, bytes(uid.cpu().numpy().tobytes()), local)
kw = json.loads(sys.argv[2]) if len(sys.argv) > 2 else {}
w = G.get(name, **kw)
g = ft.load(w, device=local, rank=rank, world=world, nccl_comm=comm, keep_all=True)
g.prepare()
torch.cuda.synchronize()
t0 = time.perf_counter()
g.eliminate()
m, t = g.frontier()
t1 = time.perf_counter()
st = g.stats()
ref = ft.load(w, device=local, keep_all=True)
ref.eliminate()
rm, rt = ref.frontier()
ok = np.array_equal(m, rm) and np.array_equal(t, rt)
bad_steps = 0
stride = 1 if os.environ.get("FT_CHECK_ALL_STEPS") else max(1, len(st) // 60)
for s in range(0, len(st), stride):
    for x, y in zip(g.step_output(s), ref.step_output(s)):
        if not np.array_equal(x, y):
            bad_steps += 1
            break
for i in np.linspace(0, len(m) - 1, 16).astype(int):
    ok = ok and np.array_equal(g.strategy(int(i)), ref.strategy(int(i)))
comm_ms = sum(s["comm_ms"] for s in st)
sharded = sum(1 for s in st if s["comm_ms"] > 0)
print(f"rank {rank}/{world} {name}{kw or ''}: frontier {len(m)} identical={ok} bad_steps={bad_steps} "
      f"sharded_waves={sharded} "
      f"search {1e3 * (t1 - t0):.1f} ms comm {comm_ms:.1f} ms local_tuples {sum(s['tuples'] for s in st)}",
      flush=True)
ft.nccl_comm_destroy(comm)
dist.destroy_process_group()
sys.exit(0 if ok and bad_steps == 0 else 1)
