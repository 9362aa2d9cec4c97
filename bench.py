"""Benchmark: H-matvec/s and achieved HBM GB/s per precision variant, plus
BiCG-STAB time to 1e-8, on the BASELINE.json workload (default config 4:
icosphere level 7, N = 327,680, leaf 64, eta 2, ACA 1e-5).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = one H-matvec y = A x of the headline scheme (m1-double) with x
resident in HBM.  Prints ONE JSON line (rank 0).
"Measurement" for the definitions of every field.
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

METRIC = "H-matvec/s & achieved HBM GB/s per precision variant; BiCG-STAB time to 1e-8"

# BASELINE.json configs (index = config number - 1): refinement, leaf, ACA tol
CONFIGS = {
    1: dict(level=3, leaf=32, aca=1e-4),
    2: dict(level=5, leaf=32, aca=1e-4),
    3: dict(level=6, leaf=64, aca=1e-5),
    4: dict(level=7, leaf=64, aca=1e-5),
    # two unit spheres at (0,0,0) and (3,0,0), potentials +1 / -1, b = voltages
    5: dict(level=8, leaf=64, aca=1e-4, centers=((0.0, 0.0, 0.0), (3.0, 0.0, 0.0)),
            voltages=(1.0, -1.0)),
}
HEADLINE = "m1-double"
FP32_ACCUMULATING = {"m1-single", "m1-mixed", "m2-single"}
VARIANTS = ["m1-double", "m1-mixed", "m2-mixed", "m3:c=3", "m3:c=-1"]


def measured_peak():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy burst)"
    return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """SM clocks and throttle reasons sampled through NVML every 5 ms while
    the timed region runs, plus one sample as it ends (falls back to
    nvidia-smi polling)."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4}

    def __init__(self, device: int):
        self.device = device
        self.rows = []
        self.max_mhz = None
        self._stop = threading.Event()
        self._th = None

    def _sample_nvml(self):
        import pynvml
        h = self._h
        sm = float(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
        mask = int(pynvml.nvmlDeviceGetCurrentClocksEventReasons(h))
        util = int(pynvml.nvmlDeviceGetUtilizationRates(h).gpu)
        self.rows.append((sm, mask, util))

    def _run(self):
        if self._h is not None:
            try:
                while True:
                    self._sample_nvml()
                    if self._stop.wait(0.005):
                        break
                return
            except Exception:
                pass
        while not self._stop.is_set():
            try:
                out = subprocess.run(
                    ["nvidia-smi", "-i", str(self.device),
                     "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,utilization.gpu",
                     "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                v = [t.strip() for t in out.stdout.strip().split(",")]
                self.max_mhz = float(v[1])
                self.rows.append((float(v[0]), int(v[2], 16), int(v[3])))
            except Exception:
                pass
            self._stop.wait(0.1)

    def __enter__(self):
        # NVML is initialised here, before the timed region, so the sampler
        # thread takes its first sample at once (a 20-step region lasts ~20 ms)
        self._h = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self._h = pynvml.nvmlDeviceGetHandleByIndex(self.device)
            self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM))
        except Exception:
            self._h = None
        self._th = threading.Thread(target=self._run, daemon=True)
        self._th.start()
        return self

    def __exit__(self, *exc):
        if self._h is not None:
            try:
                self._sample_nvml()   # one sample at the end of the region, whatever its length
            except Exception:
                pass
        self._stop.set()
        if self._th:
            self._th.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unsampled"], "samples": 0}
        busy = [r[0] for r in self.rows if r[2] > 50] or [r[0] for r in self.rows]
        reasons = sorted({name for r in self.rows for name, bit in self.REASONS.items() if r[1] & bit})
        return {"sm_mhz": statistics.median(busy), "sm_max_mhz": self.max_mhz, "reasons": reasons,
                "samples": len(self.rows), "source": "nvml, 5 ms + one at the end"}


def build_workload(cfg_id: int):
    import paper_1911_00093_b200 as hx
    c = CONFIGS[cfg_id]
    t0 = time.perf_counter()
    mesh = hx.jittered_sphere_mesh(c["level"], seed=42, centers=c.get("centers", ((0.0, 0.0, 0.0),)),
                                   voltages=c.get("voltages"))
    h = hx.build_hmatrix(mesh, aca_tol=c["aca"], leaf_size=c["leaf"], eta=2.0)
    x = np.random.default_rng(42).uniform(-1.0, 1.0, mesh.n)
    b = hx.right_hand_side(mesh) if "voltages" in c else mesh.centroids[:, 2].copy()
    return mesh, h, x, b, time.perf_counter() - t0


def workload_name(cfg_id):
    c = CONFIGS[cfg_id]
    k = len(c.get("centers", (0,)))
    n = k * 20 * 4 ** c["level"]
    if k > 1:
        return (f"config{cfg_id}: {k} jittered unit icospheres level {c['level']} centred at "
                f"{list(c['centers'])} (N={n}), leaf {c['leaf']}, eta 2.0, ACA {c['aca']:g}; "
                f"x ~ U(-1,1) seed 42; b = sphere potentials {list(c['voltages'])}")
    return (f"config{cfg_id}: jittered unit icosphere level {c['level']} (N={n}), leaf {c['leaf']}, "
            f"eta 2.0, ACA {c['aca']:g}; x ~ U(-1,1) seed 42; b = centroid z")


def workload_config(cfg_id, mesh, h, algo_bytes):
    """The `config` object of the JSON line -- identical in both arms."""
    return {"workload": workload_name(cfg_id), "scheme": HEADLINE, "n": int(mesh.n),
            "blocks": int(h.partition.table.shape[0]), "parallelism": "single GPU",
            "l2": f"inputs {algo_bytes / 1e9:.2f} GB >> 126 MB L2 (no flush needed)"}


def cpu_full_passes(sh, x, budget_s: float, threads: int = 1, max_passes: int = 20):
    """The oracle's FULL matvec (numpy restatement of the reference's
    matvec.py, every block) timed on this host: passes until budget_s is
    spent (at least 2); returns (matvec/s from the median pass, passes)."""
    from oracle import hmx_oracle as orc
    orc.matvec_threaded(sh, x, threads)          # warm: payload views, page faults
    times = []
    t_end = time.perf_counter() + budget_s
    while len(times) < 2 or (time.perf_counter() < t_end and len(times) < max_passes):
        t0 = time.perf_counter()
        orc.matvec_threaded(sh, x, threads)
        times.append(time.perf_counter() - t0)
    return 1.0 / float(np.median(times)), len(times)


def measured_reference_solve(cfg_id):
    """The reference algorithm's BiCG-STAB to 1e-8 on this config's H-matrix,
    MEASURED (not estimated): the threads=1 oracle solve recorded in
    tests/golden/solver_envelope_config<k>.json (run in the build container
    by tests/golden/make_solver_envelope.py); None if absent."""
    f = ROOT / "tests" / "golden" / f"solver_envelope_config{cfg_id}.json"
    if not f.exists():
        return None
    d = json.loads(f.read_text())
    run = d.get("schemes", {}).get(HEADLINE, {}).get("1")
    if not run:
        return None
    return {"wall_s": run["cpu_s"], "iterations": run["iterations"], "converged": run["converged"],
            "true_residual": run["true_residual"],
            "where": "build container (8-core Xeon, OPENBLAS_NUM_THREADS=1), oracle bicgstab, "
                     "tests/golden/solver_envelope_config%d.json" % cfg_id}


def _timed(fn):
    t0 = time.perf_counter()
    fn()
    return time.perf_counter() - t0


def run_reference(args):
    """--impl reference: the reference's CPU matvec (oracle port of
    matvec.py / matvec_threaded, pinned bit-for-bit to the reference) on the
    host cores.  One step = one FULL matvec of the workload (every block), no
    sampling; threads = the faster of 1 and all host threads on one full
    pass.  The H-matrix itself comes from this repo's host builder
    (libhmx_host.so, untimed: the reference's own build takes 442 s here)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import paper_1911_00093_b200 as hx
    from oracle import hmx_oracle as orc
    mesh, h, x, b, _ = build_workload(args.config)
    sh = hx.prepare_scheme(h, HEADLINE)
    ncpu = os.cpu_count() or 1
    orc.matvec_threaded(sh, x, 1)                    # warm (payload views, page faults)
    trial = {t: _timed(lambda t=t: orc.matvec_threaded(sh, x, t)) for t in sorted({1, ncpu})}
    threads = min(trial, key=trial.get)
    for _ in range(args.warmup):
        orc.matvec_threaded(sh, x, threads)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        orc.matvec_threaded(sh, x, threads)
        times.append(time.perf_counter() - t0)
    ms = 1e3 * float(np.mean(times))
    v = 1e3 / ms
    desc = (f"full matvec per step (all {h.partition.table.shape[0]} blocks), {threads} thread(s) "
            f"(the faster of 1 and {ncpu} on a full pass: "
            + ", ".join(f"{t}: {1e3 * dt:.0f} ms" for t, dt in trial.items()) + ")")
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "matvec/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded jittered icosphere, BASELINE.json recipe)",
        "config": workload_config(args.config, mesh, h, sh.payload_bytes + 16 * mesh.n),
        "cpu_baseline": {"value": v, "unit": "matvec/s", "cores": threads, "kind": "port",
                         "sample": desc, "solve": measured_reference_solve(args.config)},
        "e2e": {"value": v, "unit": "matvec/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "note": ("oracle/hmx_oracle.py: numpy restatement of the reference's matvec.py "
                 "(per-block loop over OpenBLAS GEMVs), pinned bit-for-bit to the reference; "
                 "libhmx_host.so is loaded only to build the input H-matrix (untimed)"),
    }
    print(json.dumps(line), flush=True)


def run_ours(args):
    import paper_1911_00093_b200 as hx
    from paper_1911_00093_b200 import _gpu
    from paper_1911_00093_b200.matvec import get_plan

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1 or args.distributed:
        from paper_1911_00093_b200 import distributed as dist_mod
        return dist_mod.bench_main(args, build_workload, workload_name, METRIC)

    device = int(os.environ.get("LOCAL_RANK", "0"))
    os.environ.setdefault("HMX_DEVICE", str(device))
    mesh, h, x, b, t_build = build_workload(args.config)
    n = mesh.n
    peak, peak_src = measured_peak()
    results = {}
    headline = None
    schemes = [HEADLINE] + [s for s in args.variants if s != HEADLINE]
    for name in schemes:
        t0 = time.perf_counter()
        sh = hx.prepare_scheme(h, name)
        t_prep = time.perf_counter() - t0
        t0 = time.perf_counter()
        plan = get_plan(sh)
        t_plan = time.perf_counter() - t0
        info = plan.info()
        y = hx.matvec(sh, x)  # uploads x (permuted copy stays resident)
        algo = sh.payload_bytes + 16 * n
        if name == HEADLINE:
            with ClockSampler(device) as clk:
                r = plan.bench(args.warmup, args.steps)
            clocks = clk.summary()
        else:
            r = plan.bench(max(3, args.warmup // 2), max(10, args.steps // 2))
        ms = r["ms"]
        # x read (8N) charged to stage 1, y write (8N) to stage 2
        diag = 8 * info["z_len"] if not name.startswith("m1") else 0
        s1_bytes = info["stage1_bytes"] + diag + 8 * n
        s2_bytes = algo - s1_bytes
        entry = {
            "matvec_per_s": 1e3 / ms, "ms": ms, "GBps": algo / (ms * 1e6),
            "frac_of_peak": algo / (ms * 1e6) / peak, "algorithmic_bytes": algo,
            "payload_bytes": sh.payload_bytes, "stage1_ms": r["stage1_ms"],
            "stage2_ms": r["stage2_ms"],
            "stage1_GBps": s1_bytes / (r["stage1_ms"] * 1e6) if r["stage1_ms"] > 0 else None,
            "stage2_GBps": s2_bytes / (r["stage2_ms"] * 1e6) if r["stage2_ms"] > 0 else None,
            "prepare_s": t_prep, "plan_s": t_plan, "device_bytes": info["device_bytes"],
        }
        if not args.no_solve:
            cfg = hx.SolverConfig(tol=1e-8, max_iter=1000)
            hx.bicgstab(sh, h, b, cfg)  # warm (workspace allocation)
            _, rep = hx.bicgstab(sh, h, b, cfg)
            entry["solve"] = {"iterations": rep.iterations, "converged": rep.converged,
                              "true_residual": rep.true_residual, "wall_s": rep.wall_time_s,
                              "device_s": rep.device_time_s, "matvecs": rep.matvecs,
                              "breakdown": rep.breakdown}
        if name in FP32_ACCUMULATING:
            # the same scheme with HMX_FP32_ORDER=chain (one FP32 chain per
            # (row, block), the faster round-1 order; the default is SGEMV's
            # own order, bitwise the reference's FP32 products)
            os.environ["HMX_FP32_ORDER"] = "chain"
            try:
                shc = hx.prepare_scheme(h, name)
                plc = get_plan(shc)
                hx.matvec(shc, x)
                rc_ = plc.bench(max(3, args.warmup // 2), max(10, args.steps // 2))
                entry["fp32_chain_order"] = {"ms": rc_["ms"], "matvec_per_s": 1e3 / rc_["ms"],
                                             "GBps": algo / (rc_["ms"] * 1e6),
                                             "stage1_ms": rc_["stage1_ms"], "stage2_ms": rc_["stage2_ms"]}
                plc.close()
                del shc
            finally:
                os.environ.pop("HMX_FP32_ORDER", None)
        results[name] = entry
        if name == HEADLINE:
            headline = (sh, plan, info, r, algo, s1_bytes, s2_bytes, clocks)
            # end-to-end through the public API: x from pinned host memory
            # copied in, both stages, y copied back into a fresh host array,
            # every step (host wall clock; the call is synchronous)
            try:
                import torch
                x_in = torch.from_numpy(x).pin_memory().numpy()
            except Exception:
                x_in = x
            for _ in range(3):
                hx.matvec(sh, x_in)
            e2e_t = []
            for _ in range(max(5, min(args.steps, 50))):
                t0 = time.perf_counter()
                hx.matvec(sh, x_in)
                e2e_t.append(time.perf_counter() - t0)
            e2e_ms = 1e3 * float(np.mean(e2e_t))
            results[name]["e2e_ms"] = e2e_ms
            # the same with a pageable numpy x (what the reference API's callers pass)
            x_page = np.array(x, copy=True)
            e2e_p = []
            for _ in range(max(5, min(args.steps, 50))):
                t0 = time.perf_counter()
                hx.matvec(sh, x_page)
                e2e_p.append(time.perf_counter() - t0)
            results[name]["e2e_pageable_ms"] = 1e3 * float(np.mean(e2e_p))
        else:
            plan.close()
            del sh

    sh, plan, info, r, algo, s1_bytes, s2_bytes, clocks = headline
    ms = r["ms"]
    # dominant kernel = stage 2 (dense + U slabs); algorithmic bytes per launch
    dom_ms = r["stage2_ms"]
    dom_achieved = s2_bytes / (dom_ms * 1e6)
    traffic = None
    prof = ROOT / "profiles" / "ncu_traffic.json"
    if prof.exists():
        try:
            traffic = json.loads(prof.read_text()).get(f"config{args.config}", {}).get(HEADLINE, {}).get("stage2")
        except Exception:
            traffic = None

    cpu = None
    if not args.no_cpu_baseline:
        v, passes = cpu_full_passes(sh, x, args.cpu_budget, 1)
        cpu = {"value": v, "unit": "matvec/s", "cores": 1, "kind": "port",
               "sample": f"{passes} FULL oracle matvecs (every block, 1 thread), median pass",
               # the reference algorithm's solve, measured (not estimated)
               "solve": measured_reference_solve(args.config)}

    line = {
        "metric": METRIC, "value": 1e3 / ms, "unit": "matvec/s", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded jittered icosphere, BASELINE.json recipe)",
        "config": workload_config(args.config, mesh, h, algo),
        "build_s": t_build,
        "roofline": {"bound": "hbm", "achieved": dom_achieved, "peak": peak, "unit": "GB/s",
                     "frac": dom_achieved / peak, "traffic": traffic,
                     "kernel": "s2_kernel (row-segment stream: dense + U slabs)",
                     "algorithmic_bytes_per_launch": s2_bytes, "peak_source": peak_src,
                     "matvec_achieved": algo / (ms * 1e6),
                     "matvec_frac": algo / (ms * 1e6) / peak,
                     "matvec_frac_of_8TBps": algo / (ms * 1e6) / 8000.0},
        "cpu_baseline": cpu,
        "e2e": {"value": 1e3 / results[HEADLINE]["e2e_ms"], "unit": "matvec/s",
                "h2d_bytes_per_step": 8 * int(n), "d2h_bytes_per_step": 8 * int(n),
                "input": "x in pinned host memory",
                "pageable": {"value": 1e3 / results[HEADLINE]["e2e_pageable_ms"], "unit": "matvec/s",
                             "input": "x a pageable numpy array (the reference API's usual caller)"}},
        "gpu_launches": 2 * args.steps,
        "clocks": clocks,
        "variants": results,
    }
    plan.close()
    if rank == 0:
        print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", type=int, default=4, choices=sorted(CONFIGS))
    ap.add_argument("--variants", nargs="*", default=VARIANTS)
    ap.add_argument("--no-solve", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=12.0)
    ap.add_argument("--distributed", action="store_true",
                    help="use the row-partitioned multi-GPU path even at world size 1")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
