"""Per-kernel warm device times of one bench step (CUPTI through torch.profiler;
no serialisation, unlike an ncu launch list).

    python tools/kernel_times.py c3 [steps]
"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import bench  # noqa: E402
import paper_1906_01687_b200.gcp as G  # noqa: E402
from paper_1906_01687_b200 import workloads as WL  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c3"
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    w = WL.get(name)
    e = bench.setup_engine(w, 0, lambda m: print(m, file=sys.stderr))
    sk, loss = bench.sampler_of(w, G), G.LossFunction.parse(w.loss)
    seed, lb = 3000 + int(name[1]), w.lower_bound
    for it in range(5):
        e.step(sk, loss, seed, it, 1e-3, lower_bound=lb)
    e.run_steps(sk, loss, seed, 5, steps, 1e-3, lower_bound=lb)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        e.run_steps(sk, loss, seed, 5 + steps, steps, 1e-3, lower_bound=lb)
        torch.cuda.synchronize()
    tot = {}
    for ev in prof.events():
        if ev.device_type.name != "CUDA":
            continue
        t = tot.setdefault(ev.name, [0.0, 0])
        t[0] += ev.device_time_total if hasattr(ev, "device_time_total") else ev.cuda_time_total
        t[1] += 1
    span = sum(v[0] for v in tot.values())
    print(f"{name}: {steps} graph-replayed steps, kernel time per step {span / steps:.1f} us")
    for k, (us, n) in sorted(tot.items(), key=lambda kv: -kv[1][0]):
        print(f"  {us / steps:9.2f} us/step  {n // steps:3d} launches/step  {k[:110]}")


if __name__ == "__main__":
    main()
