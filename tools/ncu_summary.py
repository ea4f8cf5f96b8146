"""Summarise an ncu report (raw metrics + hottest SASS windows)."""
import csv
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "lts__t_sector_hit_rate.pct",
        "l1tex__t_sector_hit_rate.pct", "launch__occupancy_limit_shared_mem",
        "launch__occupancy_limit_registers", "sm__maximum_warps_per_active_cycle_pct",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    h, u, v = r[0], r[1], r[2]
    return {n: (v[i], u[i]) for i, n in enumerate(h)}


def hot(rep, top=8, win=24):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h = rows[1]
    d = rows[2:]
    isrc = h.index("Source")
    iss = h.index("Warp Stall Sampling (All Samples)")
    iex = h.index("Instructions Executed")
    ts = sum(float(x[iss] or 0) for x in d) or 1
    te = sum(float(x[iex] or 0) for x in d) or 1
    ws = []
    for i in range(0, len(d), win):
        ch = d[i:i + win]
        ws.append((sum(float(x[iss] or 0) for x in ch) / ts, sum(float(x[iex] or 0) for x in ch) / te, i,
                   ch[0][isrc].strip()[:70]))
    return sorted(ws, reverse=True)[:top]


if __name__ == "__main__":
    for rep in sys.argv[1:]:
        print("==", rep)
        m = raw(rep)
        for k in KEYS:
            if k in m:
                print(f"  {k} = {m[k][0]} {m[k][1]}")
        for s, e, i, src in hot(rep):
            print(f"  sass[{i}:] stall={s:.3f} inst={e:.3f}  {src}")
