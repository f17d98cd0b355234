#!/usr/bin/env python
"""Benchmark of the fp64 tensor-Chebyshev hot path (BASELINE.json metric: Chebyshev evals/s and
game time-steps/s, fp64, 1/2/4/8 B200 vs CPU).

Default workload = the largest single-GPU BASELINE configuration, configs[3] ("config 4"): J=5,
n=17 (1,419,857 coefficients, 11.4 MB), node values exp(sum sin(pi a_j x_j)), ONE batch of
M = 2^24 scattered points, sharded across the N GPUs (strong scaling, as BASELINE.json's config
says).  One step = build the coefficient tensor from the node values (K1) + evaluate it at the
rank's share of the M points (K2).  `value` = evals/s of the whole job, measured with CUDA events
per step, max over ranks.  `e2e` = the same through the public API with host (pinned) inputs and
outputs, H2D / D2H inside the timed region.  --config selects the other BASELINE configs
(2 = J=3 n=33 M=2^20, 1 = J=2 n=17; 3 / 5b report steps/s of the time loop; 5a reports
structured evals/s; solve = the collocation solver).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 4] [--impl ours|reference]

--gpus N > 1 without a torchrun environment re-launches itself under torch.distributed.run with N
ranks on 127.0.0.1 (or exits non-zero when fewer than N GPUs are visible); under torchrun each rank
drives one GPU.  The scattered configs shard points (coefficients built replicated on every rank
from the same node values: no data-path collective); the loop configs shard node slabs and fuse
the per-step exchange into the evaluator's NVLink peer stores.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

# CPU baseline: the reference's own parallel scheme (thread pool, 1 BLAS thread per worker,
# S/solver.py:423-437).  Must be set before numpy is imported.
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
os.environ.setdefault("OMP_NUM_THREADS", "1")

import numpy as np  # noqa: E402

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "Chebyshev evals/sec & game time-steps/sec (fp64) at 1/2/4/8 B200 vs CPU"
FP64_PEAK_FILE = os.path.join(ROOT, "profiles", "fp64_peak_r01.json")
NCU_SUMMARY = os.path.join(ROOT, "profiles", "ncu_summary_r02.json")


def algorithmic_eval_flops(J: int, n: int) -> int:
    """2 * sum_{m=1..J} n^m flops per point."""
    return 2 * sum(n ** m for m in range(1, J + 1))


def measured_peaks():
    peaks = {"hbm_gbs": None, "fp64_tflops": None, "fp64_source": None, "hbm_source": None}
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            mp = json.load(f)
        peaks["hbm_gbs"] = mp.get("hbm_gbs")
        peaks["hbm_source"] = "MEASURED_PEAKS.json hbm_gbs (measured)"
    if peaks["hbm_gbs"] is None:
        peaks["hbm_gbs"] = 6650.0
        peaks["hbm_source"] = "B200_PROFILING.md fallback 6.65 TB/s"
    if os.path.exists(FP64_PEAK_FILE):
        with open(FP64_PEAK_FILE) as f:
            fp = json.load(f)
        peaks["fp64_tflops"] = fp["fp64_peak_tflops"]
        peaks["fp64_source"] = fp["source"]
    else:
        peaks["fp64_tflops"] = 37.0
        peaks["fp64_source"] = "tools/microbench/fp64_peak.cu DMMA sustained (measured r01)"
    return peaks


class ClockSampler:
    """SM clocks and clock-event (throttle) reasons sampled every 5 ms through NVML while the
    timed region runs (the B200_PROFILING.md clocks line); nvidia-smi is the fallback."""

    REASONS = {
        "hw_slowdown": 0x8,
        "hw_thermal_slowdown": 0x40,
        "sw_thermal_slowdown": 0x20,
        "sw_power_cap": 0x4,
        "hw_power_brake_slowdown": 0x80,
    }

    def __init__(self, index: int, period: float = 0.005):
        self.index = index
        self.period = period
        self.samples = []
        self.reason_bits = 0
        self.max_mhz = None
        self._stop = threading.Event()
        self.thread = None
        self.handle = None

    def _nvml_index(self):
        vis = os.environ.get("CUDA_VISIBLE_DEVICES")
        if vis:
            parts = [p.strip() for p in vis.split(",") if p.strip()]
            if self.index < len(parts) and parts[self.index].isdigit():
                return int(parts[self.index])
        return self.index

    def start(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nvml = pynvml
            self.handle = pynvml.nvmlDeviceGetHandleByIndex(self._nvml_index())
            self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(self.handle, pynvml.NVML_CLOCK_SM))
        except Exception:  # noqa: BLE001 - NVML missing: report unavailable
            self.handle = None
            return
        self.thread = threading.Thread(target=self._run, daemon=True)
        self.thread.start()

    def _run(self):
        nv = self.nvml
        while not self._stop.is_set():
            try:
                self.samples.append(float(nv.nvmlDeviceGetClockInfo(self.handle, nv.NVML_CLOCK_SM)))
                self.reason_bits |= int(nv.nvmlDeviceGetCurrentClocksEventReasons(self.handle))
            except Exception:  # noqa: BLE001
                break
            self._stop.wait(self.period)

    def stop(self):
        if self.handle is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"], "samples": 0}
        self._stop.set()
        if self.thread:
            self.thread.join(timeout=2)
        reasons = sorted(k for k, bit in self.REASONS.items() if self.reason_bits & bit)
        return {
            "sm_mhz": statistics.median(self.samples) if self.samples else None,
            "sm_max_mhz": self.max_mhz,
            "reasons": reasons,
            "samples": len(self.samples),
        }


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def max_over_ranks(x: float, world: int, torch):
    if world == 1:
        return x
    import torch.distributed as dist

    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


# ------------------------------------------------------------------------------------------------
# CPU baseline (oracle port of the reference algorithm) — the one place bench.py runs oracle/
# ------------------------------------------------------------------------------------------------

def _single_thread_mode(orc, C, pts, cores: int, budget_s: float):
    """SURVEY.md §8d CPU mode (i), the reference as shipped: one Python thread evaluating point
    blocks (S/solver.py with workers=1), OpenBLAS with all its threads (threadpoolctl lifts this
    process's OPENBLAS_NUM_THREADS=1 for the duration).  Returns seconds per point."""
    from threadpoolctl import threadpool_limits

    with threadpool_limits(limits=cores, user_api="blas"):
        n = 256
        t0 = time.perf_counter()
        orc.eval_points(C, pts[:n])
        per_pt = (time.perf_counter() - t0) / n
        n = int(min(pts.shape[0], max(256, budget_s / max(per_pt, 1e-9))))
        t0 = time.perf_counter()
        orc.eval_points(C, pts[:n])
        return (time.perf_counter() - t0) / n, n


def _with_modes(res: dict, full_units: float, tb: float, per_pt_single: float, n_single: int, cores: int,
                pool_per_unit: float) -> dict:
    """Attach both CPU modes; `value` is the better one (labelled in best_mode)."""
    single_step = tb + per_pt_single * full_units
    pool_step = res["step_seconds"]
    res["modes"] = {
        "pool": {"step_seconds": pool_step, "threads": cores,
                 "what": f"ThreadPoolExecutor({cores}) over point blocks, OPENBLAS_NUM_THREADS=1 (S/solver.py:423-437)"},
        "single": {"step_seconds": single_step, "blas_threads": cores, "points_timed": n_single,
                   "what": "one Python thread (workers=1, as shipped), OpenBLAS default threads"},
    }
    if single_step < pool_step:
        res["best_mode"] = "single"
        res["step_seconds"] = single_step
        res["value"] = res["value"] * pool_step / single_step
    else:
        res["best_mode"] = "pool"
    return res


def host_info() -> dict:
    """CPU provenance for the baseline: model, core counts, numpy / BLAS versions."""
    info = {"cpu_model": None, "nproc": os.cpu_count(), "affinity_cores": None, "numpy": np.__version__,
            "blas": None}
    try:
        info["affinity_cores"] = len(os.sched_getaffinity(0))
    except (AttributeError, OSError):
        pass
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    info["cpu_model"] = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    try:
        from threadpoolctl import threadpool_info

        blas = [f"{d.get('internal_api')} {d.get('version')} ({d.get('threading_layer')}, "
                f"{d.get('architecture')})" for d in threadpool_info() if d.get("user_api") == "blas"]
        info["blas"] = "; ".join(blas) or None
    except Exception:  # noqa: BLE001 - provenance only
        pass
    return info


def cpu_baseline(cfg: str, budget_s: float = 12.0):
    res = _cpu_baseline(cfg, budget_s)
    res["host"] = host_info()
    return res


def _cpu_baseline(cfg: str, budget_s: float):
    from oracle import cheb_oracle as orc
    from paper_2307_04688_b200 import workloads

    cores = os.cpu_count() or 1
    if cfg in ("1", "2", "4"):
        w = workloads.make(cfg, M=16)
        full_M = {"1": 65_536, "2": 1 << 20, "4": 1 << 24}[cfg]
        rng = np.random.default_rng(7)
        # calibrate a sample that takes ~budget_s
        sample = 256
        pts = 2.0 * rng.random((sample, w.J)) - 1.0
        t0 = time.perf_counter()
        C = orc.tensor_coeffs(w.values)
        tb = time.perf_counter() - t0
        t0 = time.perf_counter()
        orc.eval_points_parallel(C, pts, workers=cores, block=64)
        te = time.perf_counter() - t0
        per_pt = te / sample
        sample = int(min(full_M, max(256, (budget_s - tb) / max(per_pt, 1e-9))))
        pts = 2.0 * rng.random((sample, w.J)) - 1.0
        t0 = time.perf_counter()
        C = orc.tensor_coeffs(w.values)
        tb = time.perf_counter() - t0
        t0 = time.perf_counter()
        orc.eval_points_parallel(C, pts, workers=cores, block=max(64, sample // (4 * cores)))
        te = time.perf_counter() - t0
        # full step = one build + full_M evals, extrapolated linearly from the sample
        step_s = tb + te * (full_M / sample)
        extrap = sample < full_M
        res = {
            "value": full_M / step_s,
            "unit": "evals/s",
            "cores": cores,
            "kind": "port",
            "sample": f"oracle tensor_coeffs + eval of {sample} seeded points on {cores} threads "
                      f"(ThreadPool, OPENBLAS_NUM_THREADS=1)"
                      + (f", EXTRAPOLATED linearly to M={full_M}" if extrap else f" (full M={full_M})")
                      + "; mode (i) (one Python thread, multi-threaded BLAS) timed beside it, the better one is value",
            "extrapolated": extrap,
            "step_seconds": step_s,
        }
        per_single, n_single = _single_thread_mode(orc, C, pts, cores, budget_s / 3)
        return _with_modes(res, full_M, tb, per_single, n_single, cores, te / sample)
    if cfg in ("3", "5b"):
        w = workloads.make(cfg)
        T, S = orc.advect_points(w.values.shape, w.A, w.dt)
        N = T.shape[0]
        t0 = time.perf_counter()
        C = orc.tensor_coeffs(w.values)
        tb = time.perf_counter() - t0
        sample = 512
        t0 = time.perf_counter()
        orc.eval_points_parallel(C, T[:sample], workers=cores, block=32)
        per_pt = (time.perf_counter() - t0) / sample
        sample = int(min(N, max(512, (budget_s - tb) / max(per_pt, 1e-9))))
        t0 = time.perf_counter()
        orc.eval_points_parallel(C, T[:sample], workers=cores, block=max(32, sample // (4 * cores)))
        te = time.perf_counter() - t0
        step_s = tb + te * (N / sample)
        extrap = sample < N
        res = {
            "value": 1.0 / step_s,
            "unit": "steps/s",
            "cores": cores,
            "kind": "port",
            "sample": f"oracle build + {sample} of {N} advected nodes on {cores} threads"
                      + (", EXTRAPOLATED linearly to one step" if extrap else " (one full step)")
                      + "; mode (i) (one Python thread, multi-threaded BLAS) timed beside it, the better one is value",
            "extrapolated": extrap,
            "step_seconds": step_s,
        }
        per_single, n_single = _single_thread_mode(orc, C, T, cores, budget_s / 3)
        return _with_modes(res, N, tb, per_single, n_single, cores, te / sample)
    if cfg == "solve":
        from threadpoolctl import threadpool_limits

        from oracle import solver_oracle as so

        spec = solve_spec()
        g = so.Game(J=spec.J, K=np.asarray(spec.K), beta=spec.beta, phi=spec.phi, A=spec.A, c=spec.c, m=spec.m,
                    rho=spec.rho, h=spec.h, P_max=spec.P_max, U_max=spec.U_max, Np=spec.Np, Nu=spec.Nu,
                    tol=spec.tol, max_iters=spec.max_iters)
        S = so.Solver(g)

        def per_sweep(**kw):
            t0 = time.perf_counter()
            S.solve(max_iters=20, **kw)
            per = (time.perf_counter() - t0) / 20
            n_s = int(max(20, min(5000, budget_s / 2 / max(per, 1e-9))))
            t0 = time.perf_counter()
            S.solve(max_iters=n_s, **kw)
            return (time.perf_counter() - t0) / n_s, n_s

        # mode (ii): the reference's block-parallel sweep (workers = cores, one node block per
        # worker per player, S/solver.py:412-438), one BLAS thread each
        per_pool, n_pool = per_sweep(workers=cores, blocks=cores)
        # mode (i): workers=1 (the reference default), BLAS with all cores
        with threadpool_limits(limits=cores, user_api="blas"):
            per_single, n_single = per_sweep()
        # mode (i'): workers=1 with ONE BLAS thread — fastest for this small problem (the sweep's
        # matrices are tiny, threaded BLAS only adds synchronisation)
        per_one, n_one = per_sweep()
        modes = {"single": {"step_seconds": per_single * SOLVE_SWEEPS, "sweeps_timed": n_single,
                            "blas_threads": cores},
                 "single_1blas": {"step_seconds": per_one * SOLVE_SWEEPS, "sweeps_timed": n_one, "blas_threads": 1},
                 "pool": {"step_seconds": per_pool * SOLVE_SWEEPS, "sweeps_timed": n_pool, "threads": cores}}
        best = min(modes, key=lambda m: modes[m]["step_seconds"])
        per = modes[best]["step_seconds"] / SOLVE_SWEEPS
        return {
            "value": 1.0 / per,
            "unit": "sweeps/s",
            "cores": cores if best != "single_1blas" else 1,
            "kind": "port",
            "sample": f"oracle solver (numpy restatement of S/solver.py): first sweeps of the same solve in mode (i) "
                      f"workers=1 + {cores}-thread BLAS, mode (i') workers=1 + 1 BLAS thread and mode (ii) "
                      f"ThreadPool({cores}) over (player, node block) tasks, 1 BLAS thread; value = the best mode",
            "best_mode": best,
            "modes": modes,
            "step_seconds": per * SOLVE_SWEEPS,
        }
    # 5a structured: build + the full 25^6 grid, both modes, nothing extrapolated
    from concurrent.futures import ThreadPoolExecutor

    from threadpoolctl import threadpool_limits

    w = workloads.make("5a")
    k = w.params["k"]
    t0 = time.perf_counter()
    C = orc.tensor_coeffs(w.values)
    tb = time.perf_counter() - t0
    # mode (ii): ThreadPool(cores) over single first-axis targets, one BLAS thread each
    out = np.empty((k,) * 6)

    def slab(i):
        out[i] = orc.eval_grid(C, [w.targets[0][i:i + 1]] + list(w.targets[1:]))[0]

    t0 = time.perf_counter()
    with ThreadPoolExecutor(max_workers=cores) as ex:
        list(ex.map(slab, range(k)))
    t_pool = tb + time.perf_counter() - t0
    del out
    # mode (i): one Python thread, BLAS on all cores
    with threadpool_limits(limits=cores, user_api="blas"):
        t0 = time.perf_counter()
        r = orc.eval_grid(C, w.targets)
        t_single = tb + time.perf_counter() - t0
    del r
    best = "single" if t_single <= t_pool else "pool"
    step_s = min(t_single, t_pool)
    return {
        "value": k ** 6 / step_s,
        "unit": "evals/s",
        "cores": cores,
        "kind": "port",
        "sample": f"oracle build + eval_grid of the full {k}^6 grid (not extrapolated) in mode (i) one Python thread + "
                  f"{cores}-thread BLAS and mode (ii) ThreadPool({cores}) over first-axis targets, 1 BLAS thread; "
                  f"value = the better mode",
        "best_mode": best,
        "modes": {"single": {"step_seconds": t_single}, "pool": {"step_seconds": t_pool, "threads": cores}},
        "extrapolated": False,
        "step_seconds": step_s,
    }


SOLVE_SWEEPS = 66_755  # sweeps of the solve workload to convergence (measured; reported per run)


def solve_spec():
    import paper_2307_04688_b200 as cn

    return cn.preset_spec("example1", tol=1e-8)


def run_reference(args):
    world, rank, _ = dist_setup()
    if rank != 0:
        return
    cfg = args.config
    steps = []
    # each step is a bounded sample of the workload, sized so the whole --steps/--warmup run ends
    # within a few minutes (extrapolation flagged in cpu_baseline.sample)
    per_step = min(args.cpu_budget, max(2.0, 150.0 / max(1, args.steps)))
    for _ in range(args.warmup):
        cpu_baseline(cfg, budget_s=1.0)
    for _ in range(args.steps):
        steps.append(cpu_baseline(cfg, budget_s=per_step))
    vals = [s["value"] for s in steps]
    v = statistics.median(vals)
    base = steps[0]
    line = {
        "impl": "reference",
        "metric": METRIC,
        "value": v,
        "unit": base["unit"],
        "n_gpus": args.gpus,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": 1000.0 * statistics.median(s["step_seconds"] for s in steps),
        "higher_is_better": True,
        "scaling": scaling_of(cfg, args.scaling),
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (seeded, BASELINE.json shapes)",
        "config": workload_config(cfg, 1, args.scaling),
        "cpu_baseline": {"value": v, "unit": base["unit"], "cores": base["cores"], "kind": base["kind"],
                         "sample": base["sample"], "best_mode": base.get("best_mode"),
                         "extrapolated": base.get("extrapolated"), "host": base["host"]},
        "e2e": {"value": v, "unit": base["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def scaling_of(cfg: str, scaling: str) -> str:
    if cfg in ("1", "2", "4"):
        return scaling
    return "weak" if cfg == "solve" else "strong"


def workload_config(cfg: str, world: int, scaling: str = "strong"):
    per = "per GPU" if scaling == "weak" else "total, sharded across the GPUs"
    desc = {
        "1": {"workload": f"config1: J=2 n=17 build + eval at M=65,536 points {per} (step = one CUDA-graph "
                           "replay of the build + evaluation, BuildEvalGraph)", "J": 2, "n": 17, "M": 65_536},
        "2": {"workload": f"config2: J=3 n=33 build + eval at M=2^20 points {per}", "J": 3, "n": 33, "M": 1 << 20},
        "3": {"workload": "config3: J=4 n=17 advected-node time step (build + eval of 83,521 nodes)", "J": 4,
              "n": 17, "M": 17 ** 4},
        "4": {"workload": f"config4: J=5 n=17 build + eval at M=2^24 points {per}", "J": 5, "n": 17, "M": 1 << 24},
        "5a": {"workload": "config5a: J=6 n=13 build + structured eval on a 25^6 grid", "J": 6, "n": 13,
               "M": 25 ** 6},
        "5b": {"workload": "config5b: J=6 n=13 advected-node time step (4,826,809 nodes)", "J": 6, "n": 13,
               "M": 13 ** 6},
        "solve": {"workload": "solve: example1 preset (J=2, degree 8, h=1e-3) to tol=1e-8, the reference's "
                              "acceptance fixture (T/test_acceptance.py:31-43); one step = one full solve",
                  "J": 2, "n": 9, "M": 81},
    }[cfg]
    d = dict(desc)
    if cfg in ("1", "2", "4"):
        d["parallelism"] = (f"dp{world}: contiguous point shards ({'one M batch split' if scaling == 'strong' else 'M per rank'}); "
                            "coefficient tensor built replicated on every rank from the same node values "
                            "(a 0.03-0.15 ms build, cheaper than an all-gather), no data-path collective")
    elif cfg == "5a":
        d["parallelism"] = f"dp{world}: first target axis sharded, outputs stay sharded, build replicated"
    elif cfg == "solve":
        d["parallelism"] = "replicas"
    else:
        d["parallelism"] = f"node-shard{world}+peer-store" if world > 1 else "node-shard1"
    d["l2_flush"] = "256 MiB write between timed steps"
    return d


# ------------------------------------------------------------------------------------------------
# GPU arm
# ------------------------------------------------------------------------------------------------

def run_ours(args):
    import torch

    world, rank, local = dist_setup()
    # CB_BENCH_SHARE_GPU=1 / CB_BENCH_BACKEND=gloo (tests only): run the multi-rank code path as
    # several processes on ONE GPU (no kernel waits on another rank: host barriers only); the
    # numbers of such a run are not a scaling measurement
    if os.environ.get("CB_BENCH_SHARE_GPU") == "1":
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist

        backend = os.environ.get("CB_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    import paper_2307_04688_b200 as cn
    from paper_2307_04688_b200 import _lib, workloads
    from paper_2307_04688_b200.chebnd import _eval_points_device, tensor_coeffs_device

    lib = _lib.load()
    cfg = args.config
    peaks = measured_peaks()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    stream = torch.cuda.current_stream()
    exchange_note = None
    launches0 = None

    if cfg in ("1", "2", "4"):
        w = workloads.make(cfg)
        J, n = w.J, w.n
        shape = (n,) * J
        if args.scaling == "strong":
            # ONE batch of M points split into contiguous shards (BASELINE config 4: "points
            # sharded across 1/2/4/8 GPUs"); the job's units are the M points
            from paper_2307_04688_b200.dist import shard_range

            pa, pb, _ = shard_range(w.M, rank, world)
            pts_host = np.ascontiguousarray(w.points[pa:pb])
            job_units = w.M
        else:
            # every rank evaluates its own block of M points; rank r uses a shifted copy of the
            # seeded points so ranks do distinct work
            pts_host = np.ascontiguousarray(np.roll(w.points, rank * 977, axis=0))
            job_units = world * w.M
        M = pts_host.shape[0]
        vals_dev = _lib.to_device(w.values)
        pts_dev = _lib.to_device(pts_host)
        L = _lib.eval_layout(shape)
        coef = _lib.empty((L["elems"],))
        out = _lib.empty((M,))
        st = _lib.new_status()

        def step():
            tensor_coeffs_device(vals_dev, shape, out=coef, status=st)
            e_mid.record(stream)
            _eval_points_device(shape, coef, pts_dev, check=False, out=out)

        graph = None
        if cfg == "1":
            # launch-bound (a ~3 us build + a ~5 us evaluation): the step is the library's CUDA-graph
            # form (BuildEvalGraph, one submission); build / eval split timed eagerly below
            from paper_2307_04688_b200.chebnd import BuildEvalGraph

            graph = BuildEvalGraph(shape, vals_dev, pts_dev, out=out)

        e0 = torch.cuda.Event(enable_timing=True)
        e_mid = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        for _ in range(args.warmup):
            step()
        torch.cuda.synchronize()
        barrier(world)
        torch.cuda.synchronize()
        clocks = ClockSampler(local)
        clocks.start()
        launches0 = int(lib.cb_kernel_launches())
        build_ms, eval_ms, step_ms = [], [], []
        for _ in range(args.steps):
            flush.zero_()
            e0.record(stream)
            if graph is not None:
                graph.replay()
            else:
                step()
            e1.record(stream)
            e1.synchronize()
            if graph is None:
                build_ms.append(e0.elapsed_time(e_mid))
                eval_ms.append(e_mid.elapsed_time(e1))
            step_ms.append(e0.elapsed_time(e1))
        torch.cuda.synchronize()
        launches = int(lib.cb_kernel_launches()) - launches0
        if graph is not None:
            # replays do not pass through the launch counter: the kernels captured in the graph
            launches += graph.kernels_per_replay * args.steps
            # build / eval split of the step: each half captured alone and replayed (eager calls
            # would time the host's launch overhead, not the kernels)
            def replay_ms(fn):
                side = torch.cuda.Stream()
                side.wait_stream(stream)
                with torch.cuda.stream(side):
                    fn()
                stream.wait_stream(side)
                torch.cuda.synchronize()
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, capture_error_mode="thread_local"):
                    fn()
                ms = []
                for _ in range(5):
                    flush.zero_()
                    e0.record(stream)
                    g.replay()
                    e1.record(stream)
                    e1.synchronize()
                    ms.append(e0.elapsed_time(e1))
                return statistics.mean(ms)

            bm = replay_ms(lambda: tensor_coeffs_device(vals_dev, shape, out=coef))
            em = replay_ms(lambda: _eval_points_device(shape, coef, pts_dev, check=False, out=out))
            frac_b = bm / (bm + em)
            build_ms = [m * frac_b for m in step_ms]
            eval_ms = [m * (1.0 - frac_b) for m in step_ms]
        barrier(world)
        torch.cuda.synchronize()
        clk = clocks.stop()
        t_total = max_over_ranks(sum(step_ms) / 1000.0, world, torch)
        value = job_units * args.steps / t_total
        # parity spot-check of this run's output (rank 0, small subset, oracle as checker)
        flops_pt = algorithmic_eval_flops(J, n)
        eval_s = statistics.mean(eval_ms) / 1000.0
        build_s = statistics.mean(build_ms) / 1000.0
        # the evaluation kernel alone for the roofline: the GPU is kept busy while the host
        # enqueues it, so the events bracket the kernel and not the host's launch gap
        ek0, ek1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        kern_ms = []
        for _ in range(3):
            flush.zero_()
            torch.cuda._sleep(2_000_000)
            ek0.record(stream)
            _eval_points_device(shape, coef, pts_dev, check=False, out=out)
            ek1.record(stream)
            ek1.synchronize()
            kern_ms.append(ek0.elapsed_time(ek1))
        kernel_s = statistics.mean(kern_ms) / 1000.0
        achieved_tf = flops_pt * M / kernel_s / 1e12
        roofline = {
            "bound": "tensor",
            "pipe": ("fp64 DMMA.8x8x4 (FP64 tensor core)" if lib.cb_last_eval_plan().decode().startswith(("eval_rc", "eval_dmma"))
                     else "fp64 DFMA (FP64 vector pipe; launch/latency-bound at this size)"),
            "kernel": lib.cb_last_eval_plan().decode(),
            "achieved": achieved_tf, "peak": peaks["fp64_tflops"], "unit": "TFLOP/s",
            "frac": achieved_tf / peaks["fp64_tflops"], "peak_source": peaks["fp64_source"],
            "algorithmic": f"{flops_pt} flop/point x {M} points per launch",
            "traffic": ncu_traffic(lib.cb_last_eval_plan().decode().split("<")[0], cfg),
        }
        build_bytes = 16 * n ** J
        kb_s = kernel_only_ms(lambda: tensor_coeffs_device(vals_dev, shape, out=coef), flush, stream, torch) / 1000.0
        roofline_build = {
            "bound": "hbm", "kernel": build_kernels(cfg), "achieved": build_bytes / kb_s / 1e9,
            "peak": peaks["hbm_gbs"], "unit": "GB/s", "frac": build_bytes / kb_s / 1e9 / peaks["hbm_gbs"],
            "algorithmic": f"16*n^J = {build_bytes} bytes per build", "ms": kb_s * 1000.0,
            "timing": "kernels alone, L2 flushed before (events bracket the launches, not the host gaps)",
        }
        # ---------------- e2e through the public API with pinned host buffers ----------------
        vals_pin = torch.from_numpy(np.ascontiguousarray(w.values)).pin_memory()
        pts_pin = torch.from_numpy(pts_host).pin_memory()
        bases = [cn.make_basis(n - 1, 0.0, 1.0)] * J
        res = None
        for _ in range(max(1, args.warmup)):
            res = cn.eval_points(cn.tensor_coeffs(vals_pin, bases), pts_pin)
        barrier(world)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            res = cn.eval_points(cn.tensor_coeffs(vals_pin, bases), pts_pin)  # returns pinned host tensor
        torch.cuda.synchronize()
        e2e_s = max_over_ranks(time.perf_counter() - t0, world, torch)
        e2e = {"value": job_units * args.steps / e2e_s, "unit": "evals/s",
               "h2d_bytes_per_step": int(vals_pin.numel() * 8 + pts_pin.numel() * 8),
               "d2h_bytes_per_step": int(res.numel() * 8 + 16)}
        # parity of the e2e result against the device-timed output and the oracle on a subset
        parity = None
        if rank == 0:
            from oracle import cheb_oracle as orc

            C = orc.tensor_coeffs(w.values)
            sub = slice(0, 2048)
            ref = orc.eval_points(C, pts_host[sub])
            got = res.numpy()[sub]
            parity = {"max_abs": float(np.abs(got - ref).max()),
                      "allclose_1e-12_1e-11": bool(np.allclose(got, ref, rtol=1e-12, atol=1e-11)),
                      "device_vs_e2e_bitwise": bool(np.array_equal(_lib.to_host(out)[sub], got))}
        unit = "evals/s"
        extra = {"roofline_build": roofline_build, "parity_check": parity,
                 "eval_ms": statistics.mean(eval_ms), "build_ms": statistics.mean(build_ms),
                 "eval_kernel_ms": kernel_s * 1000.0}
        ms_per_step = 1000.0 * t_total / args.steps
    elif cfg in ("3", "5b"):
        from paper_2307_04688_b200.dist import ShardedAdvectLoop
        from paper_2307_04688_b200.loop import CudaStepBackend

        w = workloads.make(cfg)
        J, n = w.J, w.n
        shape = (n,) * J
        N = n ** J
        bases = [cn.make_basis(n - 1, 0.0, 1.0)] * J
        steps_per_iter = 1
        if world == 1:
            vals = _lib.to_device(w.values).clone()
            tmp = _lib.empty(shape)
            L = _lib.eval_layout(shape)
            coef = _lib.empty((L["elems"],))

            def run_steps(k):
                lib.cb_advect_loop(J, _lib.i64_array(shape), _lib.ptr(vals), _lib.ptr(tmp), _lib.ptr(coef), k,
                                   _lib.dbl_array(w.A), w.dt, _lib.dbl_array([0.0] * J), _lib.dbl_array([1.0] * J),
                                   None, 1, _lib.stream_handle())
        else:
            # fused exchange: the evaluation kernel stores each rank's slab into every rank's
            # node-value buffer over NVLink (CUDA IPC); the NCCL all-gather loop is the fallback
            # when the peer mappings cannot be set up (reported in config.parallelism)
            backend = CudaStepBackend(bases, w.A, w.dt)
            try:
                from paper_2307_04688_b200.dist import PeerShardedAdvectLoop

                loop = PeerShardedAdvectLoop(shape, backend)
            except Exception as exc:  # noqa: BLE001
                exchange_note = f"node-shard{world}+allgather (peer-store setup failed: {exc!r:.120})"
                loop = ShardedAdvectLoop(shape, backend)

            def run_steps(k):
                loop.run(w.values, k)
        # the BASELINE loop length: 100 steps (cfg 3) / 20 steps (cfg 5b) per timed step
        inner = w.steps
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        for _ in range(args.warmup):
            run_steps(inner)
        torch.cuda.synchronize()
        barrier(world)
        torch.cuda.synchronize()
        clocks = ClockSampler(local)
        clocks.start()
        launches0 = int(lib.cb_kernel_launches())
        times = []
        for _ in range(args.steps):
            flush.zero_()
            e0.record(stream)
            run_steps(inner)
            e1.record(stream)
            e1.synchronize()
            times.append(e0.elapsed_time(e1))
        torch.cuda.synchronize()
        launches = int(lib.cb_kernel_launches()) - launches0
        barrier(world)
        clk = clocks.stop()
        t_total = max_over_ranks(sum(times) / 1000.0, world, torch)
        total_steps = inner * args.steps
        value = total_steps / t_total
        unit = "steps/s"
        # per-kernel timing of one step (isolated events) for the roofline
        M = N
        flops_pt = algorithmic_eval_flops(J, n)
        from paper_2307_04688_b200.chebnd import tensor_coeffs_device as tcd

        L = _lib.eval_layout(shape)
        cbuf = _lib.empty((L["elems"],))
        vbuf = _lib.to_device(w.values)
        obuf = _lib.empty((N,))
        ec = torch.cuda.Event(enable_timing=True)
        ed = torch.cuda.Event(enable_timing=True)
        tcd(vbuf, shape, out=cbuf)

        def one_eval():
            lib.cb_eval_advected(J, _lib.i64_array(shape), _lib.ptr(cbuf), 0, N, _lib.dbl_array(w.A), w.dt,
                                 _lib.dbl_array([0.0] * J), _lib.dbl_array([1.0] * J), 1, _lib.ptr(obuf),
                                 _lib.stream_handle())

        # the evaluation kernel as it runs inside the loop: launched back to back (the host enqueues
        # faster than the kernels run, so the events bracket kernels, not launch gaps; an isolated
        # launch after an idle GPU measured 5 % slower than the same kernel inside the loop)
        n_ev = 5
        one_eval()
        ec.record(stream)
        for _ in range(n_ev):
            one_eval()
        ed.record(stream)
        ed.synchronize()
        eval_s = ec.elapsed_time(ed) / 1000.0 / n_ev
        build_s = kernel_only_ms(lambda: tcd(vbuf, shape, out=cbuf), flush, stream, torch) / 1000.0
        achieved_tf = flops_pt * M / eval_s / 1e12
        roofline = {
            "bound": "tensor", "pipe": "fp64 DMMA.8x8x4 (FP64 tensor core)", "kernel": lib.cb_last_eval_plan().decode() + " on advected nodes", "achieved": achieved_tf,
            "peak": peaks["fp64_tflops"], "unit": "TFLOP/s", "frac": achieved_tf / peaks["fp64_tflops"],
            "peak_source": peaks["fp64_source"], "algorithmic": f"{flops_pt} flop/point x {M} nodes per launch",
            "traffic": ncu_traffic("eval_dmma_kernel", cfg),
        }
        build_bytes = 16 * N
        extra = {"roofline_build": {"bound": "hbm", "kernel": build_kernels(cfg),
                                    "achieved": build_bytes / build_s / 1e9, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                                    "frac": build_bytes / build_s / 1e9 / peaks["hbm_gbs"], "ms": build_s * 1e3,
                                    "timing": "kernels alone, L2 flushed before"},
                 "loop_steps_per_timed_step": inner}
        # e2e: public API advect_loop from host values, result back to host
        vals_pin = torch.from_numpy(np.ascontiguousarray(w.values)).pin_memory()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            res = cn.advect_loop(vals_pin, bases, w.A, w.dt, inner)
            if torch.is_tensor(res):
                res = res.cpu()
        torch.cuda.synchronize()
        e2e_s = max_over_ranks(time.perf_counter() - t0, world, torch)
        e2e = {"value": total_steps / e2e_s, "unit": "steps/s", "h2d_bytes_per_step": int(N * 8 / inner),
               "d2h_bytes_per_step": int(N * 8 / inner)}
        ms_per_step = 1000.0 * t_total / total_steps
    elif cfg == "solve":
        import warnings

        spec = solve_spec()
        for _ in range(args.warmup):
            with warnings.catch_warnings():
                warnings.simplefilter("ignore", RuntimeWarning)
                cn.solve(cn.preset_spec("example1", tol=1e-8, max_iters=64))
        torch.cuda.synchronize()
        clocks = ClockSampler(local)
        clocks.start()
        launches0 = int(lib.cb_kernel_launches())
        times, sweeps = [], []
        for _ in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            with warnings.catch_warnings():
                warnings.simplefilter("ignore", RuntimeWarning)
                res = cn.solve(spec)
            torch.cuda.synchronize()
            times.append(time.perf_counter() - t0)
            sweeps.append(res.iterations)
        launches = int(lib.cb_kernel_launches()) - launches0
        clk = clocks.stop()
        t_total = max_over_ranks(sum(times), world, torch)
        n_sw = sweeps[0]
        value = world * sum(sweeps) / t_total
        unit = "sweeps/s"
        nodes = int(np.prod(spec.Np + 1))
        K = int(spec.Nu[0]) + 1
        evals = spec.J * nodes * K  # value-interpolant evaluations per sweep
        flop_sweep = evals * 2 * sum(9 ** m for m in range(1, spec.J + 1))
        achieved = flop_sweep * value / world / 1e12
        roofline = {"bound": "tensor", "pipe": "fp64 (DFMA/DMMA); latency-bound", "kernel": "sweep_kernel (warp per player x node; latency-bound)",
                    "achieved": achieved, "peak": peaks["fp64_tflops"], "unit": "TFLOP/s",
                    "frac": achieved / peaks["fp64_tflops"],
                    "algorithmic": f"{flop_sweep} value-eval flops per sweep ({evals} evals)", "traffic": None}
        e2e = {"value": value, "unit": unit, "h2d_bytes_per_step": int(8 * nodes * (spec.J + 2 * spec.J) +
                                                                      8 * spec.J * nodes * K ** spec.J),
               "d2h_bytes_per_step": int(8 * (3 * spec.J * nodes + n_sw * (spec.J + 1)))}
        extra = {"sweeps_to_converge": n_sw, "solve_seconds": statistics.mean(times),
                 "evals_per_s": value * evals, "converged": bool(res.converged)}
        ms_per_step = 1000.0 * t_total / args.steps
    else:  # 5a structured
        w = workloads.make("5a")
        J, n = w.J, w.n
        shape = (n,) * J
        bases = [cn.make_basis(n - 1, 0.0, 1.0)] * J
        k = w.params["k"]
        # shard the first target axis across ranks (outputs stay sharded)
        from paper_2307_04688_b200.dist import shard_range

        a, b, _ = shard_range(k, rank, world)
        targets = [w.targets[0][a:b]] + list(w.targets[1:])
        vals_dev = _lib.to_device(w.values)
        tdev = [_lib.to_device(t) for t in targets]
        from paper_2307_04688_b200.chebnd import _eval_grid_device

        L = _lib.eval_layout(shape)
        coef5 = _lib.empty((L["elems"],))
        st5 = _lib.new_status()
        grid_out = _lib.empty(tuple(int(t.shape[0]) for t in tdev))
        grid_work = [None]

        def step():
            # device-resident build + structured evaluation (no host syncs; the public-API path
            # with its status checks is the e2e leg below)
            tensor_coeffs_device(vals_dev, shape, out=coef5, status=st5)
            return _eval_grid_device(shape, coef5, tdev, status=st5, out=grid_out)

        for _ in range(args.warmup):
            step()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        barrier(world)
        clocks = ClockSampler(local)
        clocks.start()
        launches0 = int(lib.cb_kernel_launches())
        times = []
        for _ in range(args.steps):
            flush.zero_()
            e0.record(stream)
            out_t = step()
            e1.record(stream)
            e1.synchronize()
            times.append(e0.elapsed_time(e1))
            del out_t
        launches = int(lib.cb_kernel_launches()) - launches0
        clk = clocks.stop()
        t_total = max_over_ranks(sum(times) / 1000.0, world, torch)
        M = k ** J
        value = M * args.steps / t_total
        unit = "evals/s"
        bytes_alg = 8 * (n ** J + (b - a) * k ** (J - 1))
        achieved = bytes_alg / (t_total / args.steps) / 1e9
        roofline = {"bound": "hbm", "kernel": "eval_grid (K3 mode products)", "achieved": achieved,
                    "peak": peaks["hbm_gbs"], "unit": "GB/s", "frac": achieved / peaks["hbm_gbs"],
                    "algorithmic": "8*(n^J + k^J) bytes per step", "traffic": ncu_traffic("eval_grid", cfg)}
        # e2e warm-up: the first two calls allocate the pinned 1.95 GB result buffers (torch's
        # caching host allocator reuses them afterwards)
        res = None
        for _ in range(max(2, args.warmup)):
            res = cn.eval_grid(cn.tensor_coeffs(w.values, bases), targets)
        barrier(world)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            res = cn.eval_grid(cn.tensor_coeffs(w.values, bases), targets)
        e2e_s = max_over_ranks(time.perf_counter() - t0, world, torch)
        e2e = {"value": M * args.steps / e2e_s, "unit": "evals/s", "h2d_bytes_per_step": int(8 * n ** J),
               "d2h_bytes_per_step": int(res.size * 8)}
        # the mode products are FP64-issue co-limited (ncu: FP64 pipe 61-67 % busy in every pass):
        # n fused multiply-adds per entry of every intermediate and of the output
        kk = b - a
        fma = n * sum(kk * k ** (m - 1) * n ** (J - m) for m in range(1, J + 1))
        tf = 2.0 * fma / (t_total / args.steps) / 1e12
        extra = {"roofline_fp64": {"bound": "fp64", "pipe": "DFMA (constant-bank matrix operands)", "achieved": tf,
                                   "peak": peaks["fp64_tflops"], "unit": "TFLOP/s", "frac": tf / peaks["fp64_tflops"],
                                   "algorithmic": f"2*n*sum_m k^m n^(J-m) = {2 * fma} flops per step"}}
        ms_per_step = 1000.0 * t_total / args.steps

    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu:
            cpu = cpu_baseline(cfg, budget_s=args.cpu_budget)
            cpu = {k2: v2 for k2, v2 in cpu.items() if k2 != "step_seconds"}
        line = {
            "metric": METRIC,
            "value": value,
            "unit": unit,
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": ms_per_step,
            "higher_is_better": True,
            "scaling": scaling_of(cfg, args.scaling),
            "vs_baseline": None,
            "dtype": "f64",
            "data": "synthetic (seeded numpy, BASELINE.json shapes; no dataset)",
            "config": workload_config(cfg, world, args.scaling),
            "e2e": e2e,
            "gpu_launches": launches,
            "roofline": roofline,
            "cpu_baseline": cpu,
            "clocks": clk,
        }
        line.update(extra)
        if exchange_note:
            line["config"]["parallelism"] = exchange_note
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


def kernel_only_ms(fn, flush, stream, torch, reps: int = 5) -> float:
    """Device time of `fn`'s kernels alone (min over reps, L2 flushed before each): the GPU is kept
    busy by a sleep kernel while the host enqueues fn, so the events bracket the kernels and not
    the host's launch gaps (a few-microsecond build is otherwise dominated by Python overhead)."""
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ms = []
    for _ in range(reps):
        flush.zero_()
        torch.cuda._sleep(2_000_000)
        e0.record(stream)
        fn()
        e1.record(stream)
        e1.synchronize()
        ms.append(e0.elapsed_time(e1))
    return min(ms)


def build_kernels(cfg: str) -> str:
    """The K1 launches of this config's build (cb_build.cu plan)."""
    return {"1": "small_build_kernel (one single-CTA launch)",
            "2": "group_pass_kernel<33,1,1> + <33,2,4> (2 mode-group launches)",
            "3": "group_pass_kernel<17,2,1> + <17,2,4> (2 mode-group launches)",
            "4": "group_pass_kernel<17,3,1> + <17,2,16> (2 mode-group launches)",
            "5a": "group_pass_kernel<13,3,1> + <13,3,4> (2 mode-group launches)",
            "5b": "group_pass_kernel<13,3,1> + <13,3,4> (2 mode-group launches)"}.get(cfg, "K1 build")


def ncu_traffic(kernel: str, cfg: str):
    """dram read+write bytes per launch of `kernel` from the committed ncu --set full summary."""
    if not os.path.exists(NCU_SUMMARY):
        return None
    try:
        with open(NCU_SUMMARY) as f:
            s = json.load(f)
        ent = s.get(cfg, {}).get(kernel)
        if isinstance(ent, list):  # multi-launch kernel sequence (e.g. the structured passes): per step
            return sum(e.get("dram_bytes_per_launch", 0) for e in ent)
        return (ent or {}).get("dram_bytes_per_launch")
    except (OSError, ValueError):
        return None


def relaunch_under_torchrun(args) -> int:
    """--gpus N > 1 outside torchrun: re-run this script as N ranks (one per GPU) under
    torch.distributed.run on 127.0.0.1; fails loudly when fewer than N GPUs are visible."""
    import socket
    import subprocess

    if args.impl == "ours":
        import torch

        have = torch.cuda.device_count() if torch.cuda.is_available() else 0
        if have < args.gpus:
            print(f"bench.py: --gpus {args.gpus} needs {args.gpus} visible CUDA devices, found {have}",
                  file=sys.stderr, flush=True)
            return 2
    with socket.socket() as sock:
        sock.bind(("127.0.0.1", 0))
        port = sock.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="4", choices=["1", "2", "3", "4", "5a", "5b", "solve"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                    help="scattered configs: split one M batch across the GPUs (strong) or M per GPU (weak)")
    ap.add_argument("--cpu-budget", type=float, default=12.0, help="seconds of CPU work per baseline sample")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    args = ap.parse_args()
    if args.gpus < 1:
        ap.error("--gpus must be >= 1")
    world = int(os.environ.get("WORLD_SIZE", "0") or 0)
    if world == 0 and args.gpus > 1:
        sys.exit(relaunch_under_torchrun(args))
    if world and world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr, flush=True)
        sys.exit(2)
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
