"""Markdown summary of one `--set full` ncu capture for profiles/: raw
metrics and hot SASS windows (tools/ncu_summary.py), then warp-stall samples
and executed instructions by CUDA source line (tools/ncu_lines.py) with the
source text of each line at the given commit.

usage: python tools/ncu_md.py REPORT.ncu-rep LIB.so KERNEL COMMIT "title" > profiles/X.md"""
import os
import subprocess
import sys

rep, lib, kern, commit, title = sys.argv[1:6]
here = os.path.dirname(os.path.abspath(__file__))
summ = subprocess.run([sys.executable, os.path.join(here, "ncu_summary.py"), rep], capture_output=True,
                      text=True).stdout
lines = subprocess.run([sys.executable, os.path.join(here, "ncu_lines.py"), rep, lib, kern, "24"],
                       capture_output=True, text=True).stdout.splitlines()
src = {}
for f in ("paper_2004_10856_b200/csrc/ft_step.cu", "paper_2004_10856_b200/csrc/ft_kernels.cuh"):
    txt = subprocess.run(["git", "show", f"{commit}:{f}"], capture_output=True, text=True).stdout
    src[os.path.basename(f)] = txt.splitlines()
print(f"# {title}\n\n```\n{summ.rstrip()}\n\nstall samples / executed instructions by CUDA source line "
      f"(line numbers and text of the source at {commit}):")
for ln in lines:
    tok = ln.split()
    if not tok or ":" not in tok[0]:
        continue
    f, _, n = tok[0].partition(":")
    text = ""
    if f in src and n.isdigit() and int(n) <= len(src[f]):
        text = " | " + src[f][int(n) - 1].strip()[:90]
    print(f"{ln.rstrip()}{text}")
print("```")
