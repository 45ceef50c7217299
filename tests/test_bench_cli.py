"""bench.py's launch contract (no GPU needed): `--gpus N` must never silently
measure a different number of GPUs."""

import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_gpus_must_match_world_size():
    env = dict(os.environ, WORLD_SIZE="3", RANK="0")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2"],
                       capture_output=True, text=True, env=env, timeout=120)
    assert r.returncode != 0
    assert "--gpus 2 but WORLD_SIZE=3" in (r.stderr + r.stdout)


def test_gpus_without_torchrun_relaunches(tmp_path):
    """Without WORLD_SIZE, `--gpus N` re-executes itself under torch.distributed.run
    with N ranks (here it fails fast: no GPUs, so the ranks exit non-zero -- but
    the relaunch command is what we check)."""
    src = open(os.path.join(ROOT, "bench.py")).read()
    assert '"-m", "torch.distributed.run"' in src and "--nproc-per-node={args.gpus}" in src
    assert 'raise SystemExit(subprocess.call(cmd))' in src
