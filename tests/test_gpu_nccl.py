"""Real multi-GPU exchange (NCCL over NVLink): libft's sharded waves with
the all-gather-v of survivors (exec_wave's device-exchange branch, DESIGN.md
8) must reproduce the 1-GPU result bit for bit -- every step output, the
frontier and sampled strategies (tools/dist_check.py, one process per GPU).
Skipped on boxes with fewer than 2 GPUs."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ngpus():
    import torch
    return torch.cuda.device_count()


def _run(n, name, kw="{}", tau=None):
    env = dict(os.environ, FT_CHECK_ALL_STEPS="1")
    if tau is not None:
        env["FT_REPLICATE_TAU"] = str(tau)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(29500 + os.getpid() % 1000),
           os.path.join(ROOT, "tools", "dist_check.py"), name, kw]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=900)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-4000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("rank ")]
    assert len(lines) == n and all("identical=True bad_steps=0" in l for l in lines), out[-4000:]
    return lines


@pytest.mark.skipif("_ngpus() < 2")
@pytest.mark.parametrize("name,kw", [("C3", "{}"), ("C4", '{"layers": 2}'),
                                     ("C5", '{"n_ops": 300, "K": 32, "B": 8, "Lmin": 3, "Lmax": 8}')])
def test_nccl_two_ranks_every_wave_sharded(name, kw):
    lines = _run(2, name, kw, tau=0)
    assert all("sharded_waves=0" not in l for l in lines)


@pytest.mark.skipif("_ngpus() < 2")
def test_nccl_default_policy_c4():
    _run(min(4, _ngpus()), "C4")
