#!/usr/bin/env python
"""bench.py — stochastic GCP gradient throughput on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config c2|c1|c3|c4|c5] [--samples S]

One "step" = one iteration of the reference's epoch loop body
(src/optimizer.cpp:116-119) over one batch of synthetic samples: the fused
sample -> model eval -> loss derivative -> d-mode MTTKRP kernel, the NCCL
all-reduce of the gradient when N > 1, and the fused Adam update.  The K timed
steps are replayed as one CUDA graph (gcpb_run_steps).  Default workload:
the largest single-GPU config, BASELINE.json configs[4] (C5: sparse
4.8e6x1.7e6x1.8e6 with 1.7e9 nonzeros, gaussian, r=16, semi-stratified
p=q=1.6e7 per GPU -- the only config whose factor table lives in HBM).
Multi-GPU is weak scaling (s per GPU fixed, sample ordinals and nonzeros
sharded, factors replicated); `--gpus N` outside torchrun re-launches itself
under torch.distributed.run with N ranks.

Prints ONE JSON line on rank 0.  `--impl reference` times the reference's own
CPU implementation (oracle/_ref = /root/reference compiled unmodified) on the
host cores, every step at the config's full sample count.
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


# What bounds each config's fused kernel: C5's factor table
# (531 MB) lives in HBM; C2/C3's factors are L2-resident and the binding limit
# is the L2 vector-reduction rate; C1/C4 are latency-bound.
BOUND = {"c1": "latency", "c2": "l2_red", "c3": "l2_red", "c4": "latency", "c5": "hbm"}

ROOFLINE_NOTES = {
    "c1": "latency-bound (300 samples/step); one cluster launch runs all K iterations",
    "c2": "factor rows are L1/L2-resident (51 KB), so B_alg/s exceeds HBM peak; the binding "
          "limit is L2 reduction throughput (ncu: L1->L2 request interface 85% busy, 4.1 GB of "
          "red.global.add.v4.f32 per launch), see DESIGN.md section 5",
    "c3": "factors (512 KB) L2-resident; bound by L2 reductions and the hash probes",
    "c4": "latency-bound: 2e5 samples per step (1.3 tiles per warp)",
    "c5": "random HBM row access (factors 531 MB): factor and gradient rows interleaved in one "
          "128-byte line so a row gather and its reduction share a DRAM burst; two fused "
          "launches per step -- the pick half, with the ordering of the unrestricted draws "
          "(counting sort by mode-0 row block) running under it on a side stream, then the "
          "unrestricted half walked in mode-0 row order (mode 0 swept instead of gathered); "
          "kernel_ms spans both launches.  ncu DRAM traffic 295 B/sample (B_alg 396), "
          "long-scoreboard bound (profiles/r02_c5_fused_picks.md, r02_c5_fused_list.md): the "
          "binding limit is the rate of random DRAM accesses (3.6e10 L2 misses/s whatever the "
          "request size), not streaming bandwidth (tools/fetchgran.cu, "
          "profiles/r02_fetchgran.md)",
}


# ---------------------------------------------------------------------------
# CPU reference timing (oracle/_ref = the unmodified reference compiled here)
# ---------------------------------------------------------------------------
def c5_cpu_samples(w, rs, n_pick, n_draw):
    """C5 draws for the reference's CPU path: p nonzero picks with the data's
    generating distribution (per-mode Zipf(1.05) coordinates, values
    log(1+Poisson(3)), Poisson >= 1) and q unrestricted uniform indices."""
    from paper_1906_01687_b200 import workloads as WL
    idx_p = np.stack([WL.zipf_indices(rs, n, 1.05, n_pick) for n in w.dims], 1).astype(np.int64)
    x_p = np.log1p(np.maximum(1, rs.poisson(3.0, n_pick))).astype(np.float64)
    idx_q = np.stack([rs.integers(0, n, n_draw) for n in w.dims], 1).astype(np.int64)
    return idx_p, x_p, idx_q


def reference_cpu(w, steps, warmup, log):
    """The reference's own CPU step (oracle/_ref) per BASELINE.md §2: `warmup`
    untimed steps, then the median over `steps` of draw_gradient_samples (or,
    for C2/C5 whose tensors it cannot hold, its per-sample entry + deriv +
    weight + append loop on pre-drawn indices) and mttkrp_sampled_all with all
    host threads; samples/s = s / (t_sample + t_mttkrp); adam_step timed once
    (the last step) and reported beside it.  Every step is the config's full
    sample count."""
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
    times, adam_s = [], None
    tm = np.zeros(3)
    h = C.c_void_p()
    total = float(np.prod(dims.astype(np.float64)))
    t_setup = time.perf_counter()
    if w.name == "c2":
        # DenseTensor cap 1e8 (tensor.hpp:54): the sample_uniform loop body
        # (samplers.hpp:87-93) on pre-drawn indices with x from the C2 model
        n = w.s
        T = WL.c2_true_factors(1002)
        idx = np.stack([rs.integers(0, k, n) for k in w.dims], 1).astype(np.int64)
        m = np.ones((n, T[0].shape[1]))
        for k in range(4):
            m *= T[k][idx[:, k]]
        x = (rs.random(n) < m.sum(1) / (1.0 + m.sum(1))).astype(np.float64)
        del m
        F = WL.init_factors(w.dims, w.rank, 2002, data_norm=np.sqrt(0.1 * 1.6e9))
        per_step = n
        what = (f"{n} pre-drawn uniform samples of C2 per step (x from the C2 generator model; "
                "the reference's DenseTensor cannot hold 1.6e9 entries)")

        def one(do_adam):
            ref._ck(ref.lib.ref_bench_step_given(h, lk, 0.0, n, O._i64(idx), O._f64(x), total / n,
                                                 threads, 1e-3, has_lb, 0.0, do_adam, O._f64(tm)))
    elif w.name == "c5":
        # the COO needs >> host RAM (tensor.cpp:18-23): the
        # sample_semi_stratified loop body (samplers.hpp:199-216) on pre-drawn
        # picks and unrestricted indices, COO lookup excluded
        idx_p, x_p, idx_q = c5_cpu_samples(w, rs, w.p, w.q)
        F = WL.init_factors(w.dims, w.rank, 2005, data_norm=None, lo=0.0, hi=0.1)
        per_step = w.p + w.q
        what = (f"{w.p} pre-drawn nonzero picks (Zipf(1.05) coordinates, log(1+Poisson(3)) "
                f"values) + {w.q} unrestricted uniform draws per step; the COO lookup is excluded "
                "(the reference cannot hold C5's 1.7e9-entry COO)")

        def one(do_adam):
            ref._ck(ref.lib.ref_bench_step_semi_given(
                h, lk, 0.0, w.p, O._i64(idx_p), O._f64(x_p), w.q, O._i64(idx_q), w.nnz, total,
                threads, 1e-3, has_lb, 0.0, do_adam, O._f64(tm)))
    else:
        # the reference's own samplers + RngStream on reference containers
        if w.name == "c1":
            rt = ref.dense(w.dims, c1_tensor())
        else:
            keys, vals = sparse_data(w)
            coords = np.stack(np.unravel_index(keys.astype(np.int64), w.dims, order="F"), 1)
            rt = ref.sparse(w.dims, coords, vals.astype(np.float64))
        F = WL.init_factors(w.dims, w.rank, 2000 + int(w.name[1]), data_norm=rt.norm())
        strat = {"uniform": 0, "stratified": 1, "semi-stratified": 2}[w.sampler]
        nsm = C.c_int64()
        per_step = w.samples_per_step
        what = (f"the full {w.name.upper()} step ({per_step} samples) with the reference's own "
                f"{w.sampler} sampler and RngStream")
        seq = [0]

        def one(do_adam):
            seq[0] += 1
            ref._ck(ref.lib.ref_bench_step_sampler(h, rt.h, lk, 0.0, strat, w.s, w.p, w.q, w.rho,
                                                   77 + seq[0], threads, 1e-3, has_lb, 0.0,
                                                   do_adam, O._f64(tm), C.byref(nsm)))
    ref._ck(ref.lib.ref_bench_model_new(len(dims), O._i64(dims), w.rank,
                                        O._f64(O.Oracle.flat(F)), C.byref(h)))
    log(f"[bench] reference data ready in {time.perf_counter() - t_setup:.1f}s")
    for it in range(warmup + steps):
        last = it == warmup + steps - 1
        one(1 if last else 0)
        if it >= warmup:
            times.append(tm[:2].copy())
        if last:
            adam_s = float(tm[2])
    ref.lib.ref_bench_model_free(h)
    t = np.median(np.array(times), axis=0)
    step_s = float(t.sum())
    sample = (f"{what}; medians over {len(times)} steps after {warmup} warm-up: "
              f"draw_gradient_samples {t[0]*1e3:.1f} ms + mttkrp_sampled_all({threads} threads) "
              f"{t[1]*1e3:.1f} ms; adam_step {adam_s*1e3:.1f} ms (timed once, not in the metric: "
              "BASELINE.md §2 samples/s = s/(t_sample+t_mttkrp))")
    return {"value": per_step / step_s, "unit": UNIT, "cores": threads, "kind": "reference",
            "sample": sample, "step_s": step_s}


# CPU-leg sizes inside our arm (rank 0, N=1): the config's full sample count
# per step, about 10-30 s of host work in total.
CPU_LEG = {"c1": (3, 20), "c2": (1, 5), "c3": (1, 5), "c4": (3, 20), "c5": (0, 1)}


def config_of(w, world):
    """The `config` object of both arms' JSON lines (identical by construction)."""
    return {"workload": f"{w.name.upper()}: {w.description}",
            "samples_per_gpu_step": w.samples_per_step,
            "global_batch": w.samples_per_step * world,
            "rank": w.rank, "dims": list(w.dims), "loss": w.loss, "sampler": w.sampler,
            "parallelism": (f"dp{world}: nonzeros (contiguous ranges) and sample ordinals "
                            "sharded, factors replicated; gradient reduce-scatter + sharded "
                            "Adam + factor all-gather in one peer-memory kernel over NVLink "
                            "(NCCL rank barriers)") if world > 1 else "single GPU",
            "l2": "inputs larger than L2 (tensor in HBM); factor rows L1/L2-resident by "
                  "design (they are the model)"}


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def run_ours(args, w):
    import torch
    import paper_1906_01687_b200.gcp as G

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if torch.cuda.device_count() < world:
        raise SystemExit(f"bench.py: --gpus {world} needs {world} GPUs, "
                         f"found {torch.cuda.device_count()}")
    torch.cuda.set_device(local)
    dist = None
    peer_path = False
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
        e.comm_init(uid[0], rank, world)  # also shards the nonzeros (contiguous ranges)
        # every rank's factor/gradient table mapped into every rank (CUDA IPC):
        # the step's exchange is one reduce-scatter + Adam + all-gather kernel
        handles = [None] * world
        dist.all_gather_object(handles, e.peer_handle())
        try:
            e.peer_open(handles)
            mapped = 1
        except Exception as ex:  # no P2P between some pair: every rank takes the NCCL path
            print(f"[bench] rank {rank}: peer mapping failed ({ex})", file=sys.stderr, flush=True)
            mapped = 0
        ok = torch.tensor([mapped], device=f"cuda:{local}")
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        peer_path = bool(int(ok[0]))
        if not peer_path:
            e.peer_close()
            log("[bench] peer-memory exchange unavailable: NCCL all-reduce + replicated Adam")
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
    launches = e.run_steps_launches()
    total_ms = start.elapsed_time(end)
    if dist:
        t = torch.tensor([total_ms], device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t[0])
    ms_per_step = total_ms / K
    steps_path = e.steps_path
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
        kernel_name = ("fused_grad_kernel (sample+eval+deriv+MTTKRP); stratified and "
                       "semi-stratified steps launch it twice (pick segment, then the list "
                       "segment whose list is built on a side stream meanwhile): kernel_ms "
                       "spans both")
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
    bound = BOUND.get(w.name, "hbm")
    roofline = {"bound": bound, "achieved": round(achieved, 1), "peak": peak_gbs, "unit": "GB/s",
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
    if traffic:
        # DRAM-counter cross-check: the ncu capture's bytes over this run's
        # launch time (ncu times are cold and serialised; the bytes are not)
        roofline["traffic_frac"] = round(traffic / (fused_ms / 1e3) / 1e9 / peak_gbs, 4)
    if w.name == "c5" and traffic:
        # Tables in HBM: the binding ceiling is the rate of DRAM accesses -- L2
        # line fills (one ~128-byte fetch per miss whatever the request size,
        # tools/fetchgran.cu: 3.6e10 read misses/s) and write-backs of dirty
        # gradient halves.  Ceiling for the fused kernel's mix of the two:
        # tools/randbw.cu "3g+3red il" (row gather + reduction on interleaved
        # lines, no arithmetic), 6.99e9 samples/s x 3 lines x (fill + write-back)
        # = 4.19e10 accesses/s.  The access count per step comes from the ncu DRAM
        # counters of the two fused launches (profiles/ncu_traffic_c5.json).
        acc = json.loads(prof.read_text()).get("dram_accesses_per_launch")
        if acc:
            roofline["binding"] = {"limit": "DRAM accesses (L2 line fills + dirty-line write-backs)",
                                   "achieved": float("%.4g" % (acc / (fused_ms / 1e3))),
                                   "peak": 4.19e10, "unit": "accesses/s",
                                   "frac": round(acc / (fused_ms / 1e3) / 4.19e10, 3),
                                   "source": "tools/randbw.cu (profiles/r01_randbw.md) and "
                                             "tools/fetchgran.cu (profiles/r02_fetchgran.md)"}
    if bound == "l2_red":
        # L2-resident factors: the binding ceiling is the L2 vector-reduction
        # rate, measured by tools/bulkred.cu (profiles/r01_bulkred.md: 6.4e7
        # 64-byte rows = 2.56e8 red.global.add.v4 in 0.794 ms)
        F = 4 if w.dtype == "f32" else 8
        reds = w.samples_per_step * w.d * ((w.rank * F + 15) // 16)
        red_rate = reds / (fused_ms / 1e3)
        roofline["binding"] = {"limit": "L2 vector reductions (red.global.add.v4.f32)",
                               "achieved": float("%.4g" % red_rate), "peak": 3.22e11,
                               "unit": "reductions/s", "frac": round(red_rate / 3.22e11, 3),
                               "source": "tools/bulkred.cu microbenchmark, profiles/r01_bulkred.md"}

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
        h2d, d2h = e.last_transfer_bytes()  # counted by the engine from the copies it queued
        narrowed = h2d < nflat * 8
        e2e = {"value": samples_per_step * Ke / el, "unit": UNIT, "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "host_model_bytes": nflat * 8,
               "what": "per step through the C-ABI with pinned host buffers (fp64 model, "
                       "as the reference holds it): gcpb_step_host = model H2D + "
                       "sample/eval/MTTKRP (+ all-reduce) + Adam + model D2H, one call and one "
                       "synchronisation per step, wall clock" +
                       ("; the fp32 engine rounds the model to fp32 on the host (threads, chunk by "
                        "chunk under the DMA) and widens the result, so half the model's bytes "
                        "cross PCIe -- both conversions are inside the timed region" if narrowed
                        else "")}
    e.close()

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            cw, cs = CPU_LEG.get(w.name, (1, 3))
            cpu = reference_cpu(w, steps=cs, warmup=cw, log=log)
        except Exception as ex:  # reported, not fatal
            log(f"[bench] cpu baseline failed: {ex}")
    if cpu:
        cpu.pop("step_s", None)

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K,
        "warmup": W, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": w.dtype,
        "data": f"synthetic ({w.description}); seeded generator, no dataset",
        "config": config_of(w, world),
        "step": ("small-problem cluster kernel: K iterations (sample+eval+MTTKRP, cluster "
                 "barrier, Adam) in one launch" if steps_path == "small" else
                 "fused sample+eval+MTTKRP kernel + (all-reduce) + fused Adam; K steps "
                 "replayed as one CUDA graph"),
        "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
        # the metric's own window (sample + eval + MTTKRP, without
        # the exchange and Adam), all ranks: CUDA events around the fused launches
        # (ordering of the unrestricted draws included) of non-graph steps
        "sample_eval_mttkrp": {"value": samples_per_step / (fused_ms / 1e3), "unit": UNIT,
                               "ms": round(fused_ms, 4)},
        "exchange": (None if world == 1 else
                     "peer-memory reduce-scatter + sharded Adam + all-gather kernel" if peer_path
                     else "NCCL all-reduce + replicated Adam"),
        "gpu_launches": launches,
        "gpu_launches_per_step": launches / K,
        "clocks": clk,
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
    cpu = reference_cpu(w, steps=args.steps, warmup=args.warmup,
                        log=lambda m: print(m, file=sys.stderr, flush=True))
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
        "config": config_of(w, world),
        "step": ("the reference's own CPU step (oracle/_ref): sampling + mttkrp_sampled_all "
                 "with all host threads, fp64"),
        "impl": "reference",
        "cpu_baseline": {"value": cpu["value"], "unit": UNIT, "cores": cpu["cores"],
                         "kind": "reference", "sample": cpu["sample"]},
        "e2e": {"value": cpu["value"], "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "wall_s": time.perf_counter() - t0,
    }
    print(json.dumps(line), flush=True)


def _relaunch_under_torchrun(args):
    """`--gpus N` without a torchrun environment: re-execute under
    torch.distributed.run with one process per GPU (127.0.0.1 rendezvous)."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={port}", str(Path(__file__).resolve()), *sys.argv[1:]]
    os.execv(sys.executable, cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c5")
    ap.add_argument("--samples", type=int, default=None, help="override s (uniform) per GPU")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    from paper_1906_01687_b200 import workloads as WL
    w = WL.get(args.config, s=args.samples)
    if args.gpus < 1:
        raise SystemExit("bench.py: --gpus must be >= 1")
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        _relaunch_under_torchrun(args)
    if args.impl == "reference":
        run_reference(args, w)
    else:
        run_ours(args, w)


if __name__ == "__main__":
    main()
