"""Importing the engine before torch must leave torch importable: both link
libnccl.so.2, torch bundles a newer copy than the system one, and the first
copy loaded serves the whole process (paper_1906_01687_b200/_capi.py)."""
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def test_engine_then_torch_imports():
    code = ("import paper_1906_01687_b200.gcp as G\n"
            "import torch\n"
            "import torch.distributed\n"
            "print('ok')\n")
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    assert r.stdout.strip().endswith("ok")
