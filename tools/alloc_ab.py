"""A/B of libft's device-memory source on one workload: the default
(cudaMallocAsync pool + process scratch) vs torch's caching allocator through
ft_options.alloc/.free (libft_torch_alloc.so).  CUDA-event search times."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2004_10856_b200 as ft  # noqa: E402
from synth import graphs as G  # noqa: E402

w = G.get(sys.argv[1] if len(sys.argv) > 1 else "C5")
stream = torch.cuda.current_stream()
flush = torch.empty(128 << 20, dtype=torch.int32, device="cuda")
for mode in ("default", "torch", "default", "torch"):
    ms = []
    for it in range(6):
        g = ft.load(w, stream=stream.cuda_stream, torch_alloc=(mode == "torch"))
        g.prepare()
        flush.zero_()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        g.eliminate()
        g.frontier()
        b.record(stream)
        torch.cuda.synchronize()
        ms.append(round(a.elapsed_time(b), 2))
        g.close()
    print(mode, ms, "torch allocated MB", torch.cuda.memory_allocated() >> 20,
          "reserved MB", torch.cuda.memory_reserved() >> 20, flush=True)
