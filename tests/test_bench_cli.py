"""bench.py's multi-GPU launch contract, on CPU: `--gpus N` must either run
N ranks or fail loudly -- never measure one GPU and report it as N."""
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def _run(args, env_extra):
    env = dict(os.environ)
    env.update(env_extra)
    env.setdefault("CUDA_VISIBLE_DEVICES", "")
    return subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], capture_output=True,
                          text=True, timeout=600, env=env)


def test_gpus_must_match_world_size():
    out = _run(["--gpus", "2", "--no-cpu", "--no-e2e"],
               {"WORLD_SIZE": "1", "RANK": "0", "LOCAL_RANK": "0"})
    assert out.returncode != 0
    assert "--gpus 2 but WORLD_SIZE=1" in (out.stdout + out.stderr)


def test_gpus_without_torchrun_relaunches_and_fails_without_gpus():
    env = {k: "" for k in ()}
    out = _run(["--gpus", "2", "--no-cpu", "--no-e2e"], env)
    assert out.returncode != 0
    text = out.stdout + out.stderr
    assert "torch.distributed" in text or "needs 2 GPUs" in text
    assert '"n_gpus"' not in out.stdout  # no JSON line was printed
