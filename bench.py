#!/usr/bin/env python
"""bench.py -- FT search on B200: product tuples/s and search time per graph.

One "step" = one complete Frontier-Tracking search of the workload graph
(every SURVEY 8(a) row: FT_AUTO eliminations -> LDP -> final reduce), i.e.
Alg. 2 of arXiv 2004.10856, with every step's Product / Union /
Reduce in libft's sm_100a kernels.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload C5]
    python bench.py --impl reference ...      # CPU oracle arm (host cores)

N > 1: launched by torchrun, one rank per GPU; each FT step's configuration
pairs are sharded over the ranks and the survivors all-gathered over NCCL
(strong scaling of one search; time = max over ranks).

Metric (BASELINE.json): product tuples/s (sum over steps of |X||Y||Z|,
Lemma 3/4 cardinalities) and FT search time per graph (ms_per_step).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "frontier tuples/sec (Product+Reduce) and FT search time per graph at 1/2/4/8 B200"
UNIT = "product tuples/s"


def print_line(line):
    print(json.dumps(line), flush=True)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", default="C5", help="C1..C5 (BASELINE.json configs); default C5, the largest config (configs[4])")
    ap.add_argument("--no-flush", action="store_true", help="skip the L2 flush between steps")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=20.0, help="cpu_baseline budget")
    ap.add_argument("--details", action="store_true", help="print per-kind breakdown to stderr")
    ap.add_argument("--algo", choices=["ldp", "elim"], default="ldp",
                    help="final frontier by FT-LDP (Alg. 3, default) or FT-Elimination (P:628)")
    return ap.parse_args()


def workload_config(name):
    from synth import graphs as G
    w = G.get(name)
    cfg = {"workload": {"C1": "C1 4-op chain K=3", "C2": "C2 VGG-16 chain D=8 K=16",
                        "C3": "C3 ResNet-50 D=16 K=25",
                        "C4": "C4 BERT-large encoder (24 layers) D=32 K=36",
                        "C5": "C5 random SP DAG 2000 ops K=64"}[name],
           "n_ops": w.n_ops, "n_edges": w.n_edges, "seed": 0}
    return w, cfg


# ---------------------------------------------------------------- clocks

class ClockSampler:
    """nvidia-smi sampling DURING the timed region (B200_PROFILING.md)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.t.join(timeout=2)
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[1]))
                mx = float(r[2])
                for n, v in zip(names, r[5:9]):
                    if v.lower() == "active":
                        reasons.add(n)
            except Exception:
                pass
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------- reference arm

def cpu_sample_workload(name, seconds):
    """Bounded sample of the same workload for the CPU oracle (about `seconds`
    of host work): C4 -> the same BERT-large graph with fewer encoder layers;
    C5 -> the same generator with fewer ops; C1-C3 -> the full graph."""
    from synth import graphs as G
    if name == "C4":
        layers = max(1, min(24, int(round(seconds * 0.6))))
        return G.c4(layers=layers), f"C4 BERT-large cost model, {layers} of 24 encoder layers"
    if name == "C5":
        n = max(100, min(2000, int(seconds * 25)))
        return G.c5(n_ops=n), f"C5 generator (same K, rho, B, L) with {n} of 2000 ops"
    return G.get(name), f"{name} full graph"


ALGO = {"ldp": "FT-LDP (Alg. 3)", "elim": "FT-Elimination (P:628)"}


def oracle_run(w, threads, algo="ldp"):
    import oracle
    t0 = time.perf_counter()
    g = oracle.load(w, threads)
    g.eliminate()
    m, t = g.frontier(algo=algo)
    dt = time.perf_counter() - t0
    tuples = sum(g.step_info(s)["tuples"] for s in range(g.num_steps()))
    return tuples, dt, len(m)


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import oracle
    oracle.build()
    threads = len(os.sched_getaffinity(0))
    w, _cfg = workload_config(args.workload)
    _, cfg = workload_config(args.workload)
    cfg["algo"] = ALGO[args.algo]
    sw, sample = cpu_sample_workload(args.workload, args.cpu_seconds)
    for _ in range(max(0, min(args.warmup, 1))):
        oracle_run(sw, threads, args.algo)
    times, tuples = [], 0
    for _ in range(args.steps):
        tp, dt, _n = oracle_run(sw, threads, args.algo)
        times.append(dt)
        tuples = tp
    tot = sum(times)
    value = tuples * len(times) / tot
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": tot / len(times) * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "int64",
            "data": "synthetic", "impl": "reference", "config": cfg,
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "oracle",
                             "sample": sample + f"; {tuples} product tuples per step"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print_line(line)
    return 0


# ---------------------------------------------------------------- our arm

def spawn_ranks(args):
    """--gpus N without a launcher: re-exec under torchrun, one rank per GPU
    (the driver's own launch line), so the N-GPU path always runs."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    os.execv(sys.executable, cmd)


def kernel_profile(workload):
    """ncu counters of the dominant kernel for this workload (committed by
    tools/ncu_round.sh -> profiles/r2_kernels.json): instructions and DRAM
    bytes per search, per kernel."""
    path = os.path.join(ROOT, "profiles", "r2_kernels.json")
    if not os.path.exists(path):
        return None
    d = json.load(open(path))
    return d.get(workload)


def roofline(dom_kernel, dom_ms, workload, tuples, ms_per_step, clocks, peaks):
    """Roofline of the dominant kernel.  The FT path is integer compare/add
    work on a PRUNED stream: k_filter proves most product tuples
    dominated without touching DRAM, so its real bound is instruction issue /
    latency, not HBM.  achieved = ncu-counted warp instructions of the kernel
    per search (deterministic for a fixed workload; profiles/r2_kernels.json)
    / its live CUDA-event time per search; peak = 148 SMs x 4 warp
    instructions per clock (one issue per SMSP) x the SM clock measured under
    load.  traffic = ncu DRAM bytes per search of that kernel.  The survey's
    40 B/tuple materialised cost is reported separately, labelled."""
    prof = kernel_profile(workload) or {}
    k = prof.get("kernels", {}).get(dom_kernel)
    sm_mhz = (clocks or {}).get("sm_mhz") or peaks.get("sm_max_mhz", 1965.0)
    peak = 148 * 4 * sm_mhz * 1e6 / 1e9  # G warp-instructions / s
    achieved = traffic = None
    src = None
    if k and dom_ms > 0:
        achieved = k["inst_per_search"] / (dom_ms / 1e3) / 1e9
        traffic = k["dram_bytes_per_search"] / max(1, k["launches_per_search"])
        src = (f"profiles/r2_kernels.json ({prof.get('source', 'ncu')}): {k['inst_per_search']:.4g} warp "
               f"instructions, {k['dram_bytes_per_search'] / 1e6:.1f} MB DRAM over {k['launches_per_search']} "
               f"launches per search; ncu sm__throughput {k.get('sm_throughput_pct', 0):.1f} %, "
               f"issue active {k.get('issue_active_pct', 0):.1f} %")
    hbm = peaks.get("hbm_gbs", 6650.0)
    mat = tuples * 40 / (ms_per_step / 1e3) / 1e9
    return {"kernel": dom_kernel, "bound": "alu", "achieved": achieved, "peak": peak,
            "unit": "G warp-instructions/s", "frac": achieved / peak if achieved else None,
            "traffic": traffic, "traffic_unit": "DRAM bytes per launch (ncu, mean over the search)",
            "source": src, "kernel_ms_per_step": dom_ms, "share_of_step": dom_ms / ms_per_step,
            "peak_source": f"148 SM x 4 SMSP x 1 warp-inst/clk x {sm_mhz:.0f} MHz (clock under load)",
            "materialised_equivalent": {
                "bytes_per_tuple": 40, "GB_per_s": mat, "frac_of_hbm": mat / hbm, "hbm_peak_gbs": hbm,
                "note": "SURVEY 8(d) expand->sort->scan->compact cost of the product tuples of one "
                        "search / search time: what a materialising design would have to stream; "
                        "not a DRAM utilisation"}}


KERNEL_OF_GROUP = {"filter": "k_filter", "direct": "direct", "bucket": "bucket", "compact": "compact",
                   "plan": "k_plan"}


def main():
    args = parse()
    if args.impl != "reference" and args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        spawn_ranks(args)
    # exactly one JSON line on stdout: libraries (NCCL prints its version on
    # init) write to fd 1 too, so everything else goes to stderr
    out = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)
    sys.stdout = sys.stderr
    global print_line
    print_line = lambda line: (out.write(json.dumps(line) + "\n"), out.flush())
    if args.impl == "reference":
        return run_reference(args)
    import numpy as np
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        return 2
    torch.cuda.set_device(local)
    dist = None
    comm = None
    import paper_2004_10856_b200 as ft
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        uid = torch.zeros(128, dtype=torch.uint8, device="cuda")
        if rank == 0:
            uid.copy_(torch.frombuffer(bytearray(ft.nccl_unique_id()), dtype=torch.uint8))
        dist.broadcast(uid, 0)
        comm = ft.nccl_comm_init(world, rank, bytes(uid.cpu().numpy().tobytes()), local)
    w, cfg = workload_config(args.workload)
    cfg.update({"algo": ALGO[args.algo], "graphs_per_step": 1,
                "parallelism": f"config-pair sharding x{world} + NCCL all-gather" if world > 1 else "single GPU",
                "l2_flush": "512 MiB memset between timed searches" if not args.no_flush else "none"})
    stream = torch.cuda.current_stream()
    kw = dict(device=local, stream=stream.cuda_stream, rank=rank, world=world, nccl_comm=comm)

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    flush_buf = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.int32, device="cuda")

    def flush():
        if not args.no_flush:
            flush_buf.zero_()

    def search(profile):
        g = ft.load(w, profile=profile, **kw)
        g.prepare()
        return g

    def max_over_ranks(x):
        if dist is None:
            return x
        tt = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        return float(tt.item())

    # warm-up (module load, scratch growth, NCCL)
    for _ in range(args.warmup):
        g = search(False)
        g.eliminate()
        g.frontier(algo=args.algo)
        g.close()
    torch.cuda.synchronize()

    # timed region: inputs resident in HBM (ft_prepare before the events), no
    # instrumentation (profile=0)
    clk = ClockSampler(local)
    clk.start()
    ev_ms, nfront, st = [], 0, None
    for _ in range(args.steps):
        g = search(False)
        flush()
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        g.eliminate()
        m, t = g.frontier(algo=args.algo)
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
        ev_ms.append(e0.elapsed_time(e1))
        st = g.stats()
        nfront = len(m)
        g.close()
    clocks = clk.stop()
    total_ms = max_over_ranks(sum(ev_ms))
    # ft_step_stats.tuples counts every rank's segments (the per-segment
    # counts are all-gathered with the survivors): the whole job's work
    tuples = sum(s["tuples"] for s in st)
    launches = sum(s["launches"] for s in st)
    ms_per_step = total_ms / args.steps
    value = tuples / (ms_per_step / 1e3)

    # kernel-group split: one extra, instrumented search (CUDA events between
    # kernel groups on the library stream), outside the timed region
    flush()
    barrier()
    g = search(True)
    g.eliminate()
    g.frontier(algo=args.algo)
    sp = g.stats()
    g.close()
    groups = {k: sum(s[k + "_ms"] for s in sp) for k in ("plan", "direct", "filter", "bucket", "compact")}

    # end-to-end through the public API with host buffers: the step's inputs
    # (concatenated Eq. 1 / Eq. 2 cost tables) sit in pinned host memory; the
    # timed region creates the graph, copies the costs H2D (ft_set_costs_all),
    # runs the search and reads the frontier back (D2H).
    e2e_ms = []
    pinned = []
    for a in ft.concat_costs(w):
        if a is None:
            pinned.append(None)
            continue
        pt = torch.empty(len(a), dtype=torch.int64, pin_memory=True)
        pt.numpy()[:] = a
        pinned.append(pt.numpy())
    h2d = sum(a.nbytes for a in pinned if a is not None)
    d2h = 0
    for _ in range(args.steps):
        flush()
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        g = ft.load(w, costs=pinned, **kw)
        g.eliminate()
        m, t = g.frontier(algo=args.algo)
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
        e2e_ms.append(e0.elapsed_time(e1))
        d2h = m.nbytes + t.nbytes
        g.close()
    e2e_tot = max_over_ranks(sum(e2e_ms))
    e2e_value = tuples / (e2e_tot / args.steps / 1e3)

    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    dom = max(groups, key=groups.get)
    roof = roofline(KERNEL_OF_GROUP[dom], groups[dom], args.workload, tuples, ms_per_step, clocks, peaks)

    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "int64", "data": "synthetic",
            "config": cfg, "search_ms": ms_per_step,
            "search_ms_steps": [round(x, 3) for x in ev_ms], "product_tuples_per_step": tuples,
            "frontier_size": nfront, "ft_steps": len(st), "gpu_launches": launches * args.steps,
            "waves": 1 + max(s["wave"] for s in st),
            "kernel_group_ms": {k: round(v, 3) for k, v in groups.items()},
            "kernel_group_source": "one instrumented search after the timed region (profile=1)",
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h), "ms_per_step": e2e_tot / args.steps,
                    "ms_steps": [round(x, 2) for x in e2e_ms]},
            "clocks": clocks, "roofline": roof}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        sw, sample = cpu_sample_workload(args.workload, args.cpu_seconds)
        threads = len(os.sched_getaffinity(0))
        tp, dt, _ = oracle_run(sw, threads, args.algo)
        line["cpu_baseline"] = {"value": tp / dt, "unit": UNIT, "cores": threads, "kind": "oracle",
                                "sample": sample + f"; {tp} product tuples in {dt:.2f} s"}
        full = os.path.join(ROOT, "profiles", "r2_oracle_timing.json")
        if os.path.exists(full):
            line["cpu_baseline"]["full_protocol"] = {
                "source": "profiles/r2_oracle_timing.json (tools/oracle_timing.py on a GPU-box host)",
                "runs": json.load(open(full)).get("runs")}
    if args.details and rank == 0:
        for s in sp:
            print(json.dumps(s), file=sys.stderr)
    if rank == 0:
        print_line(line)
    if comm is not None:
        ft.nccl_comm_destroy(comm)
    if dist is not None:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
