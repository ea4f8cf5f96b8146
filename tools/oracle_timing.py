"""Oracle timing protocol of SURVEY 8(d) "Oracle timing" on the host it runs
on: liboracle_ft.so with 1 thread on C1-C4 and with T = all host threads on
C1-C5; full workloads (no sampling), FT-LDP.  Records lscpu.  Writes JSON
(default profiles/r2_oracle_timing.json).  The oracle is a reported
baseline, not the target.

    python tools/oracle_timing.py [--out PATH] [--configs C1,C2,C3,C4,C5]
"""
import argparse
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from synth import graphs as G  # noqa: E402


def run(w, threads):
    t0 = time.perf_counter()
    g = oracle.load(w, threads)
    g.eliminate()
    m, _t = g.frontier()
    dt = time.perf_counter() - t0
    tuples = sum(g.step_info(s)["tuples"] for s in range(g.num_steps()))
    return {"threads": threads, "search_s": dt, "product_tuples": tuples, "tuples_per_s": tuples / dt,
            "frontier": len(m), "steps": g.num_steps()}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r2_oracle_timing.json"))
    ap.add_argument("--configs", default="C1,C2,C3,C4,C5")
    a = ap.parse_args()
    T = len(os.sched_getaffinity(0))
    try:
        lscpu = subprocess.run(["lscpu"], capture_output=True, text=True).stdout
    except Exception:
        lscpu = ""
    keep = ("Model name", "Socket(s)", "Core(s) per socket", "Thread(s) per core", "CPU(s)")
    cpu = {l.split(":")[0].strip(): l.split(":", 1)[1].strip() for l in lscpu.splitlines()
           if ":" in l and l.split(":")[0].strip() in keep}
    runs = []
    for name in a.configs.split(","):
        w = G.get(name)
        for threads in ([1, T] if name != "C5" else [T]):
            r = run(w, threads)
            r["config"] = name
            runs.append(r)
            print(json.dumps(r), file=sys.stderr, flush=True)
    out = {"host_threads": T, "lscpu": cpu, "runs": runs,
           "how": "tools/oracle_timing.py: oracle.load + FT_AUTO + LDP, wall clock (perf_counter), "
                  "full workloads, once each"}
    with open(a.out, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
