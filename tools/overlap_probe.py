"""Measurement: how much does a concurrent HBM stream (Adam over a mode-0-sized
table in another context) slow the C5 step, and the step the stream?  Probe for
fusing mode 0's Adam into the ordered list launch's sweep."""
import os, sys, time, threading
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch
import bench as B
import paper_1906_01687_b200.gcp as G
from paper_1906_01687_b200 import workloads as WL

w = WL.get("c5")
log = lambda m: print(m, file=sys.stderr, flush=True)
e = B.setup_engine(w, 0, log)
sA = torch.cuda.Stream()
e.set_stream(sA.cuda_stream)
sk = B.sampler_of(w, G)
loss = G.LossFunction.parse(w.loss)
K = 40
for it in range(3):
    e.step(sk, loss, 7, it, 1e-3)
e.run_steps(sk, loss, 7, 3, K, 1e-3)
e.synchronize()

b = G.Engine((int(os.environ.get("PROBE_ROWS", 4_800_000)), 2, 2), 16, dtype="f32", device=0)
sB = torch.cuda.Stream()
b.set_stream(sB.cuda_stream)
NB = int(os.environ.get("PROBE_NB", 300))

def time_a():
    s, t = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(sA)
    e.run_steps(sk, loss, 7, 3 + K, K, 1e-3)
    t.record(sA)
    return s, t

def run_b(n):
    s, t = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(sB)
    for _ in range(n):
        b.adam_step(1e-3)
    t.record(sB)
    return s, t

torch.cuda.synchronize()
s, t = time_a(); torch.cuda.synchronize(); a_alone = s.elapsed_time(t) / K
s, t = run_b(NB); torch.cuda.synchronize(); b_alone = s.elapsed_time(t) / NB
# concurrent: queue B first (long), then A
sb, tb = run_b(NB)
sa, ta = time_a()
torch.cuda.synchronize()
a_con = sa.elapsed_time(ta) / K
b_tot = sb.elapsed_time(tb)
print(f"A alone {a_alone:.3f} ms/step; B alone {b_alone:.3f} ms/adam ({b.interleaved}); "
      f"concurrent: A {a_con:.3f} ms/step, B total {b_tot:.1f} ms for {NB} (alone {b_alone*NB:.1f})")
# B passes completed while A ran ~= (A window) / b rate: report slowdown budget
print(f"A window {a_con*K:.1f} ms; B alone would do {a_con*K/b_alone:.0f} passes in it")
e.close(); b.close()
