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


def test_reference_arm_line_contract():
    """`--impl reference` (the reference's own CPU code, oracle/_ref) prints one
    JSON line with the arm's keys: same metric/unit/config as ours, impl,
    cpu_baseline describing the run, e2e repeating the value with zero copies."""
    import json
    if not (ROOT / "oracle" / "_ref" / "libgcpref.so").exists():
        import pytest
        pytest.skip("oracle/_ref not built")
    out = _run(["--impl", "reference", "--config", "c1", "--steps", "3", "--warmup", "3"], {})
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads([l for l in out.stdout.splitlines() if l.startswith("{")][-1])
    assert line["impl"] == "reference" and line["unit"] == "samples/s"
    assert line["higher_is_better"] is True and line["steps"] == 3 and line["warmup"] == 3
    assert line["config"]["workload"].startswith("C1")
    cb = line["cpu_baseline"]
    assert cb["kind"] == "reference" and cb["cores"] >= 1 and cb["value"] == line["value"]
    assert line["e2e"] == {"value": line["value"], "unit": "samples/s",
                           "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert line["value"] > 0
