#!/usr/bin/env python
"""bench.py — stochastic GCP gradient throughput on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config c2|c1|c3|c4|c5] [--samples S]

One "step" = one iteration of the reference's epoch loop body
(src/optimizer.cpp:116-119) over one batch of synthetic samples: the fused
sample -> model eval -> loss derivative -> d-mode MTTKRP kernel, the NCCL
all-reduce of the gradient when N > 1, and the fused Adam update.  The K timed
steps are replayed as one CUDA graph (gcpb_run_steps).  Default workload:
BASELINE.json configs[1] (C2: dense 200^4 binary, bernoulli-odds, r=16,
uniform s=1.6e7 per GPU).  Multi-GPU is weak scaling (s per GPU fixed, sample
ordinals sharded, factors replicated).

Prints ONE JSON line on rank 0.  `--impl reference` times the reference's own
CPU implementation (oracle/_ref = /root/reference compiled unmodified) on the
host cores on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))  # cpu_baseline / reference legs only

METRIC = "GCP stochastic-gradient samples/sec (sample+eval+MTTKRP), % of HBM roofline"
UNIT = "samples/s"
LOSS_KIND = {"gaussian": 0, "poisson": 1, "bernoulli-odds": 2}


def _peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


# ---------------------------------------------------------------------------
# clocks sampling during the timed region
# ---------------------------------------------------------------------------
class ClockSampler:
    """SM clock + clock-event (throttle) reasons sampled every ~1 ms through
    NVML while the timed region runs (nvidia-smi -lms is too coarse for a
    region of a few tens of ms); falls back to nvidia-smi when NVML is absent."""
    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, device: int):
        self.device = device
        self.samples = []
        self._stop = threading.Event()
        self.t = None
        self.nvml = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nvml = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self._physical_index(device))
            self.max_mhz = int(pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM))
        except Exception:
            self.nvml = None

    @staticmethod
    def _physical_index(device: int) -> int:
        vis = os.environ.get("CUDA_VISIBLE_DEVICES")
        if vis:
            try:
                return int(vis.split(",")[device])
            except (ValueError, IndexError):
                pass
        return device

    def _reasons(self):
        n = self.nvml
        for fn in ("nvmlDeviceGetCurrentClocksEventReasons", "nvmlDeviceGetCurrentClocksThrottleReasons"):
            if hasattr(n, fn):
                return int(getattr(n, fn)(self.h))
        return 0

    def _poll(self):
        n = self.nvml
        while not self._stop.is_set():
            try:
                self.samples.append((int(n.nvmlDeviceGetClockInfo(self.h, n.NVML_CLOCK_SM)),
                                     self._reasons()))
            except Exception:
                pass
            time.sleep(0.001)

    def start(self):
        if self.nvml is None:
            return
        self.t = threading.Thread(target=self._poll, daemon=True)
        self.t.start()
        while not self.samples and self.t.is_alive():
            time.sleep(0.001)

    def stop(self):
        if self.t is not None:
            self._stop.set()
            self.t.join(timeout=2)
        if self.samples:
            sm = [c for c, _ in self.samples]
            bits = 0
            for _, b in self.samples:
                bits |= b
            reasons = sorted(v for k, v in self.REASONS.items() if bits & k)
            return {"sm_mhz": float(statistics.median(sm)), "sm_max_mhz": self.max_mhz,
                    "reasons": reasons, "samples": len(sm), "source": "nvml"}
        return self._smi_once()

    def _smi_once(self):
        q = "clocks.sm,clocks.max.sm"
        try:
            out = subprocess.run(["nvidia-smi", "-i", str(self.device), f"--query-gpu={q}",
                                  "--format=csv,noheader,nounits"], capture_output=True,
                                 text=True, timeout=20).stdout.strip().split(",")
            return {"sm_mhz": float(out[0]), "sm_max_mhz": int(out[1]), "reasons": [],
                    "samples": 1, "source": "nvidia-smi (after the timed region)"}
        except Exception:
            return None


# ---------------------------------------------------------------------------
# workload data
# ---------------------------------------------------------------------------
def c1_tensor():
    rs = np.random.default_rng(1001)
    A = [rs.standard_normal((n, 5)) for n in (100, 100, 100)]
    A = [a / np.linalg.norm(a, axis=0) for a in A]
    M = np.einsum("ir,jr,kr->ijk", *A)
    E = rs.standard_normal(M.shape)
    X = M + 0.1 * (np.linalg.norm(M) / np.linalg.norm(E)) * E
    return X.reshape(-1, order="F")


def sparse_data(w):
    """Sorted unique u64 keys + f32 values (C3/C4 on the host, C5 on the GPU)."""
    from paper_1906_01687_b200 import workloads as WL
    if w.name == "c5":
        return WL.c5_device_data(w)
    keys = WL.sparse_keys(w, 1000 + int(w.name[1]))
    vals = WL.sparse_values(w, len(keys), 1100 + int(w.name[1]))
    return keys, vals


def setup_engine(w, device, log):
    import torch
    import paper_1906_01687_b200.gcp as G
    from paper_1906_01687_b200 import workloads as WL

    e = G.Engine(w.dims, w.rank, dtype=w.dtype, device=device)
    t0 = time.perf_counter()
    if w.name == "c2":
        e.generate_dense_bernoulli(WL.c2_true_factors(1002), seed=1002,
                                   storage=os.environ.get("GCPB_C2_STORAGE", "bit"))
    elif w.name == "c1":
        e.set_dense(c1_tensor(), "f64")
    else:
        keys, vals = sparse_data(w)
        if isinstance(keys, np.ndarray):
            kt = torch.from_numpy(keys.view(np.int64)).to(f"cuda:{device}")
            vt = torch.from_numpy(vals).to(f"cuda:{device}")
        else:
            kt, vt = keys, vals
        e.set_sparse_device(kt.data_ptr(), vt.data_ptr(), kt.numel(), "f32")
        torch.cuda.synchronize(device)
        del kt, vt, keys, vals
        torch.cuda.empty_cache()
    log(f"[bench] data ready in {time.perf_counter() - t0:.1f}s")
    xnorm = e.tensor_norm()
    F = WL.init_factors(w.dims, w.rank, 2000 + int(w.name[1]), data_norm=xnorm)
    if w.dtype == "f32":
        F = [f.astype(np.float32).astype(np.float64) for f in F]
    e.set_factors(F)
    return e


def sampler_of(w, G, nranks=1):
    if w.sampler == "uniform":
        return G.SamplerKind.uniform(w.s * nranks)
    if w.sampler == "stratified":
        return G.SamplerKind.stratified(w.p * nranks, w.q * nranks, w.rho)
    return G.SamplerKind.semi_stratified(w.p * nranks, w.q * nranks)


ROOFLINE_NOTES = {
    "c1": "latency-bound (300 samples/step); one cluster launch runs all K iterations",
    "c2": "factor rows are L1/L2-resident (51 KB), so B_alg/s exceeds HBM peak; the binding "
          "limit is L2 reduction throughput (ncu: L1->L2 request interface 85% busy, 4.1 GB of "
          "red.global.add.v4.f32 per launch), see DESIGN.md section 5",
    "c3": "factors (512 KB) L2-resident; bound by L2 reductions and the hash probes",
    "c4": "latency-bound: 2e5 samples per step (1.3 tiles per warp)",
    "c5": "random HBM row access (factors 531 MB): factor and gradient rows interleaved in one "
          "128-byte line so a row gather and its reduction share a DRAM burst, and the "
          "unrestricted draws walked in mode-0 row order (mode 0 swept instead of gathered); ncu "
          "DRAM traffic 334 B/sample (B_alg 396; 401 in ordinal order) at 3.8 TB/s, "
          "long-scoreboard bound (profiles/r01_c5_ordered.md); the random-access "
          "microbenchmark tops out at 6.0e9 samples/s for the unordered mix (tools/randbw.cu, "
          "profiles/r01_randbw.md)",
}


def launches_per_step(w, hot, world, interleaved=False):
    # fused kernel + adam (which folds the hot-row copies; sharded steps fold
    # them before the all-reduce instead); the stratified zero sampler adds
    # 3 x (plan + candidate test + scatter) + a shortfall check; on the
    # interleaved table the unrestricted draws are put in mode-0 row order
    # first (count, scan init, scan, scatter)
    return (2 + (1 if hot and world > 1 else 0) + (10 if w.sampler == "stratified" else 0)
            + (4 if interleaved and w.sampler == "semi-stratified" else 0))


# ---------------------------------------------------------------------------
# CPU reference timing (oracle/_ref = the unmodified reference compiled here)
# ---------------------------------------------------------------------------
def reference_cpu(w, steps, warmup, n_sample, log):
    import ctypes as C
    import oracle as O
    from paper_1906_01687_b200 import workloads as WL
    ref = O.reference()
    if ref is None:
        return None
    threads = os.cpu_count() or 1
    lk = LOSS_KIND[w.loss]
    rs = np.random.default_rng(4242)
    dims = np.array(w.dims, dtype=np.int64)
    has_lb = 1 if w.lower_bound is not None else 0
    times = []
    tm = np.zeros(3)
    h = C.c_void_p()
    if w.name in ("c2", "c5"):
        # The reference cannot hold these tensors (DenseTensor cap 1e8,
        # tensor.hpp:54; C5's 1.7e9-entry COO needs >> host RAM,
        # tensor.cpp:18-23): time its per-sample entry + deriv + weight +
        # append loop (samplers.hpp:87-93) on builder-supplied (index, x), then
        # mttkrp_sampled_all(threads) and adam_step.
        if w.name == "c2":
            T = WL.c2_true_factors(1002)
            idx = np.stack([rs.integers(0, n, n_sample) for n in w.dims], 1).astype(np.int64)
            m = np.ones((n_sample, T[0].shape[1]))
            for k in range(4):
                m *= T[k][idx[:, k]]
            m = m.sum(1)
            x = (rs.random(n_sample) < m / (1.0 + m)).astype(np.float64)
            F = WL.init_factors(w.dims, w.rank, 2002, data_norm=np.sqrt(0.1 * 1.6e9))
            weight = float(np.prod(dims.astype(np.float64))) / n_sample
            what = "uniform samples of C2 (x from the C2 generator model)"
        else:
            idx = np.stack([WL.zipf_indices(rs, n, 1.05, n_sample) for n in w.dims],
                           1).astype(np.int64)
            x = np.log1p(np.maximum(1, rs.poisson(3.0, n_sample))).astype(np.float64)
            F = WL.init_factors(w.dims, w.rank, 2005, data_norm=None, lo=0.0, hi=0.1)
            weight = 1.7e9 / (n_sample / 2)
            what = "C5-distributed samples (COO lookup cost excluded)"
        ref._ck(ref.lib.ref_bench_model_new(len(dims), O._i64(dims), w.rank,
                                            O._f64(O.Oracle.flat(F)), C.byref(h)))
        for it in range(warmup + steps):
            ref._ck(ref.lib.ref_bench_step_given(h, lk, 0.0, n_sample, O._i64(idx), O._f64(x),
                                                 weight, threads, 1e-3, has_lb, 0.0, O._f64(tm)))
            if it >= warmup:
                times.append(tm.copy())
        ref.lib.ref_bench_model_free(h)
        per_step = n_sample
        sample = f"{n_sample} pre-drawn {what} per step"
    else:
        # Reference samplers on reference containers (C1, C3, C4).
        if w.name == "c1":
            rt = ref.dense(w.dims, c1_tensor())
        else:
            keys, vals = sparse_data(w)
            coords = np.stack(np.unravel_index(keys.astype(np.int64), w.dims, order="F"), 1)
            rt = ref.sparse(w.dims, coords, vals.astype(np.float64))
        F = WL.init_factors(w.dims, w.rank, 2000 + int(w.name[1]), data_norm=rt.norm())
        ref._ck(ref.lib.ref_bench_model_new(len(dims), O._i64(dims), w.rank,
                                            O._f64(O.Oracle.flat(F)), C.byref(h)))
        strat = {"uniform": 0, "stratified": 1, "semi-stratified": 2}[w.sampler]
        nsm = C.c_int64()
        for it in range(warmup + steps):
            ref._ck(ref.lib.ref_bench_step_sampler(h, rt.h, lk, 0.0, strat, w.s, w.p, w.q, w.rho,
                                                   77 + it, threads, 1e-3, has_lb, 0.0,
                                                   O._f64(tm), C.byref(nsm)))
            if it >= warmup:
                times.append(tm.copy())
        ref.lib.ref_bench_model_free(h)
        per_step = int(nsm.value)
        sample = (f"the full {w.name.upper()} step ({per_step} samples) with the reference's own "
                  f"{w.sampler} sampler and RngStream")
    t = np.mean(times, axis=0)
    sample += (f"; draw_gradient_samples {t[0]*1e3:.1f} ms, mttkrp_sampled_all({threads} threads) "
               f"{t[1]*1e3:.1f} ms, adam_step {t[2]*1e3:.1f} ms; mean of {len(times)} steps")
    return {"value": per_step / float(t.sum()), "unit": UNIT, "cores": threads,
            "kind": "reference", "sample": sample, "step_s": float(t.sum())}


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def run_ours(args, w):
    import torch
    import paper_1906_01687_b200.gcp as G

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))

    def log(msg):
        if rank == 0:
            print(msg, file=sys.stderr, flush=True)

    e = setup_engine(w, local, log)
    # A dedicated stream shared by the engine and the CUDA events.
    stream = torch.cuda.Stream(device=local)
    torch.cuda.set_stream(stream)
    e.set_stream(stream.cuda_stream)
    if world > 1:
        uid = [G.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        e.comm_init(uid[0], rank, world)
    e.set_shard(rank, world)
    sk = sampler_of(w, G, world)
    loss = G.LossFunction.parse(w.loss)
    lr = 1e-3
    lb = w.lower_bound
    seed = 3000 + int(w.name[1])
    K, W = args.steps, args.warmup

    # warm-up: W plain steps, then one untimed replay (captures the K-step graph)
    for it in range(W):
        e.step(sk, loss, seed, it, lr, lower_bound=lb)
    e.run_steps(sk, loss, seed, W, K, lr, lower_bound=lb)
    e.synchronize()
    if dist:
        dist.barrier()

    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clocks = ClockSampler(local)
    torch.cuda.synchronize()
    clocks.start()
    if dist:
        dist.barrier()
    start.record(stream)
    e.run_steps(sk, loss, seed, W + K, K, lr, lower_bound=lb)  # K steps, one graph
    end.record(stream)
    e.synchronize()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    clk = clocks.stop()
    total_ms = start.elapsed_time(end)
    if dist:
        t = torch.tensor([total_ms], device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t[0])
    ms_per_step = total_ms / K
    steps_path = e.steps_path
    hot_copies = e.hot_rows[1] if w.kind == "sparse" else 0
    samples_per_step = w.samples_per_step * world
    value = samples_per_step / (ms_per_step / 1e3)

    # Roofline of the dominant kernel: CUDA events around each fused launch
    # (non-graph steps, pre-queued behind a GPU sleep so the host never
    # starves the stream).
    Kt = max(5, min(K, 20))
    if steps_path == "small":
        # the timed region was one launch of the small-problem cluster kernel
        # (every iteration inside it): its per-iteration time is the step time
        fused_ms = ms_per_step
        kernel_name = "small_steps_kernel (K iterations of sample+eval+deriv+MTTKRP+Adam, one launch)"
    else:
        e.kernel_timing(True)
        torch.cuda._sleep(int(2e8))
        for it in range(Kt):
            e.step(sk, loss, seed, 50_000 + it, lr, lower_bound=lb)
        fused_total, nl = e.kernel_time()
        e.kernel_timing(False)
        fused_ms = fused_total / max(nl, 1)
        kernel_name = "fused_grad_kernel (sample+eval+deriv+MTTKRP)"
    if dist:
        t = torch.tensor([fused_ms], device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        fused_ms = float(t[0])
    peak_gbs, peak_src = _peaks()
    bps = w.bytes_per_sample()
    achieved = bps * w.samples_per_step / (fused_ms / 1e3) / 1e9
    traffic = None
    prof = ROOT / "profiles" / f"ncu_traffic_{w.name}.json"
    if prof.exists():
        traffic = json.loads(prof.read_text()).get("dram_bytes_per_launch")
    roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak_gbs, "unit": "GB/s",
                "frac": round(achieved / peak_gbs, 4), "traffic": traffic,
                # also against the north star's nominal 8.0 TB/s
                "frac_of_nominal_8tbs": round(achieved / 8000.0, 4),
                "kernel": kernel_name,
                "kernel_ms": round(fused_ms, 4),
                "kernel_share_of_step": round(fused_ms / ms_per_step, 3),
                "bytes_per_sample": bps,
                "bytes_per_sample_formula": "4d + 2*d*r*F (int32 index/mode + gathered + "
                                            "scattered factor rows)",
                "units_per_launch": w.samples_per_step, "peak_source": peak_src,
                "note": ROOFLINE_NOTES.get(w.name, "")}
    if w.name in ("c2", "c3"):
        # L2-resident factors: the binding ceiling is the L2 vector-reduction
        # rate, measured by tools/bulkred.cu (profiles/r01_bulkred.md: 6.4e7
        # 64-byte rows = 2.56e8 red.global.add.v4 in 0.794 ms)
        F = 4 if w.dtype == "f32" else 8
        reds = w.samples_per_step * w.d * ((w.rank * F + 15) // 16)
        red_rate = reds / (fused_ms / 1e3)
        roofline["binding"] = {"limit": "L2 vector reductions (red.global.add.v4.f32)",
                               "achieved": float("%.4g" % red_rate), "peak": 3.22e11,
                               "unit": "reductions/s", "frac": round(red_rate / 3.22e11, 3),
                               "source": "tools/bulkred.cu, profiles/r01_bulkred.md"}

    # e2e through the C-ABI with host buffers: every step copies the model in
    # from pinned host memory, runs the iteration, and copies the updated
    # model out (gcpb_step_host: the reference's loop body on a host model)
    e2e = None
    if not args.no_e2e:
        nflat = sum(n * w.rank for n in w.dims)
        pin_in = torch.empty(nflat, dtype=torch.float64, pin_memory=True).numpy()
        pin_out = torch.empty(nflat, dtype=torch.float64, pin_memory=True).numpy()
        pin_in[:] = np.concatenate([f.ravel() for f in e.factors()])
        Ke = max(3, min(K, 20))
        for it in range(2):
            e.step_host(sk, loss, seed, 60_000 + it, lr, pin_in, pin_out, lower_bound=lb)
            pin_in[:] = pin_out
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        t0 = time.perf_counter()
        for it in range(Ke):
            e.step_host(sk, loss, seed, 70_000 + it, lr, pin_in, pin_out, lower_bound=lb)
            pin_in, pin_out = pin_out, pin_in
        torch.cuda.synchronize()
        el = time.perf_counter() - t0
        if dist:
            t = torch.tensor([el], device=f"cuda:{local}", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            el = float(t[0])
        nbytes = nflat * 8
        e2e = {"value": samples_per_step * Ke / el, "unit": UNIT, "h2d_bytes_per_step": nbytes,
               "d2h_bytes_per_step": nbytes,
               "what": "per step through the C-ABI with pinned host buffers: gcpb_step_host = "
                       "model H2D + sample/eval/MTTKRP (+ all-reduce) + Adam + model D2H, one "
                       "call and one synchronisation per step, wall clock"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            cpu = reference_cpu(w, steps=2, warmup=1, n_sample=args.cpu_samples, log=log)
        except Exception as ex:  # reported, not fatal
            log(f"[bench] cpu baseline failed: {ex}")
    if cpu:
        cpu.pop("step_s", None)

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K,
        "warmup": W, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": w.dtype,
        "data": f"synthetic ({w.description}); seeded generator, no dataset",
        "config": {"workload": f"{w.name.upper()}: {w.description}",
                   "samples_per_gpu_step": w.samples_per_step, "global_batch": samples_per_step,
                   "rank": w.rank, "dims": list(w.dims), "loss": w.loss, "sampler": w.sampler,
                   "parallelism": (f"dp{world}: sample ordinals sharded, factors replicated, NCCL "
                                   f"all-reduce of the gradient") if world > 1 else "single GPU",
                   "l2": "inputs larger than L2 (tensor in HBM); factor rows L1/L2-resident by "
                         "design (they are the model)",
                   "step": ("small-problem cluster kernel: K iterations (sample+eval+MTTKRP, "
                            "cluster barrier, Adam) in one launch" if steps_path == "small" else
                            "fused sample+eval+MTTKRP kernel + (all-reduce) + fused Adam; K steps "
                            "replayed as one CUDA graph")},
        "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
        "gpu_launches": 1 if steps_path == "small" else launches_per_step(w, hot_copies > 0, world, e.interleaved[0]) * K, "clocks": clk,
        "impl": "ours",
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def run_reference(args, w):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    t0 = time.perf_counter()
    cpu = reference_cpu(w, steps=args.steps, warmup=args.warmup, n_sample=args.cpu_samples,
                        log=lambda m: print(m, file=sys.stderr))
    if cpu is None:
        print(json.dumps({"impl": "reference", "unavailable":
                          "oracle/_ref/libgcpref.so (reference compiled from /root/reference) "
                          "not present"}))
        return
    line = {
        "metric": METRIC, "value": cpu["value"], "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": cpu["step_s"] * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": f"synthetic ({w.description})",
        "config": {"workload": f"{w.name.upper()}: {w.description}", "rank": w.rank,
                   "dims": list(w.dims), "loss": w.loss, "sampler": w.sampler},
        "impl": "reference",
        "cpu_baseline": {"value": cpu["value"], "unit": UNIT, "cores": cpu["cores"],
                         "kind": "reference", "sample": cpu["sample"]},
        "e2e": {"value": cpu["value"], "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "wall_s": time.perf_counter() - t0,
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2")
    ap.add_argument("--samples", type=int, default=None, help="override s (uniform) per GPU")
    ap.add_argument("--cpu-samples", type=int, default=1_000_000)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    from paper_1906_01687_b200 import workloads as WL
    w = WL.get(args.config, s=args.samples)
    if args.impl == "reference":
        run_reference(args, w)
    else:
        run_ours(args, w)


if __name__ == "__main__":
    main()
