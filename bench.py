"""PP-GMRES benchmark (BASELINE.json metric: time-to-solution (s), plus the
fused p(A)v SpMV's HBM GB/s against the measured roofline).

One *step* = one polynomial-preconditioned GMRES solve of the workload:
degree policy (``build_poly(d)``, on Cholesky failure ``auto_degree(cap=d)``)
+ ``solve``, with the matrix, b and v0 already resident in HBM.  Default
workload = configs[3] (the 8M-row 3-D 27-point anisotropic problem of
north_star, 213.8M nonzeros, GMRES(50), requested degree 16, tol 1e-8) --
the largest single-GPU configuration; ``--config 2`` selects configs[1].  L2 is flushed (256 MiB write)
between timed steps; every step is timed with CUDA events on the solve's
stream; the job time is the max over ranks.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 4] [--impl ours|reference]

With --gpus N > 1 and no launcher, bench.py starts N ranks itself through
torch.distributed.run (the driver's command line).  Each rank owns one row block (z-planes) of the matrix:
halo exchange before every SpMV and one all-reduce per batched dot phase
(NCCL).  ``--impl reference`` times the CPU oracle port of the reference
(oracle/pgmres_oracle.py) on a bounded sample of the same workload (one SpMV +
one ICGS on the full operator per step, all host threads), rank 0 only, and
extrapolates with the reference's own recorded operation counts
(tests/golden/cfg<N>_full_reference.json).
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

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_1907_00072_b200 import workloads as wl  # noqa: E402

METRIC = ("PP-GMRES time-to-solution (s); fused p(A)v SpMV HBM GB/s vs ~8 TB/s roofline")


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def _traffic(kernel_key: str, workload: str):
    """DRAM bytes per launch of the dominant kernel from the committed ncu
    --set full capture of this workload (profiles/ncu_traffic.json), or None."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as fh:
            return json.load(fh).get("per_workload", {}).get(workload, {}).get(kernel_key)
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []
        # nvidia-smi in a subprocess: an in-process NVML thread competes for the
        # GIL with the launching thread and visibly delays kernel launches
        self.mode = os.environ.get("PG_BENCH_CLOCKS", "smi")
        self.interval = float(os.environ.get("PG_BENCH_CLOCKS_MS", "250")) / 1e3

    def _nvml_loop(self):
        import pynvml as nv
        nv.nvmlInit()
        h = nv.nvmlDeviceGetHandleByIndex(self.index)
        bits = (("hw_slowdown", nv.nvmlClocksThrottleReasonHwSlowdown),
                ("hw_thermal_slowdown", getattr(nv, "nvmlClocksThrottleReasonHwThermalSlowdown",
                                                0x40)),
                ("sw_thermal_slowdown", getattr(nv, "nvmlClocksThrottleReasonSwThermalSlowdown",
                                                0x20)),
                ("sw_power_cap", nv.nvmlClocksThrottleReasonSwPowerCap))
        smax = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        while not self._stop:
            if self.marked:
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                r = nv.nvmlDeviceGetCurrentClocksThrottleReasons(h)
                act = ["Active" if (r & b) else "Not Active" for _, b in bits]
                self.lines.append(",".join([str(sm), str(smax), hex(r)] + act))
            time.sleep(self.interval)
        nv.nvmlShutdown()

    def start(self):
        if self.mode == "off":
            return
        if self.mode == "nvml":
            try:
                import pynvml  # noqa: F401
                self._stop = False
                self.thread = threading.Thread(target=self._nvml_loop, daemon=True)
                self.thread.start()
                return
            except Exception:
                self.mode = "smi"
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index),
                 f"--query-gpu={os.environ.get('PG_BENCH_CLOCKS_FIELDS', self.FIELDS)}",
                 "--format=csv,noheader,nounits", "-lms", str(int(1e3 * self.interval))],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            if self.marked:
                self.lines.append(line.strip())

    marked = False

    def mark(self):
        """Only samples from here on (the timed region) are kept."""
        self.marked = True

    def stop(self):
        if self.mode == "off":
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["sampling disabled"]}
        if self.mode == "nvml":
            self._stop = True
            self.thread.join(timeout=5)
        elif self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        else:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.thread.join(timeout=2)
        sm, smax, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for nm, val in zip(names, parts[3:7]):
                if val.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm),
                "source": self.mode, "interval_ms": 1e3 * self.interval}


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_1907_00072_b200 as pg
    from paper_1907_00072_b200 import _lib

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # one GPU per rank over NCCL; --dist-backend gloo lets several ranks share
    # fewer GPUs (host-staged exchanges, for validating the distributed path)
    ndev = torch.cuda.device_count()
    local_dev = local if args.dist_backend == "nccl" else local % max(ndev, 1)
    torch.cuda.set_device(local_dev)
    dev = torch.device("cuda", local_dev)
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")
    conf = wl.CONFIGS[args.config]
    N = wl.config_n(conf)

    t_gen = time.perf_counter()
    counters = pg.CostCounters()
    if world > 1:
        # row blocks aligned to grid planes (z for 3-D, rows for 2-D)
        plane = conf.get("grid", 1) ** (2 if conf["gen"] in ("convdiff3d_7pt", "aniso27") else 1)
        nplanes = N // plane
        offs = np.array([(nplanes * p // world) * plane for p in range(world)] + [N])
        r0, r1 = int(offs[rank]), int(offs[rank + 1])
        block = wl.make_matrix(conf, rows=(r0, r1))
        op = pg.DeviceMatrixOperator.distributed(block, offs, counters, device=dev)
        if conf["rhs"] == "axrandom":
            raise SystemExit("axrandom rhs is single-GPU only in the bench")
        b_host = wl.splitmix_uniform(0, r1 - r0, start=r0)
        v0_host = wl.splitmix_uniform(1, r1 - r0, start=r0)
        nnz_local = block.nnz
    else:
        A = wl.make_matrix(conf)
        op = pg.DeviceMatrixOperator(A, counters, device=dev)
        b_host = wl.make_rhs(conf, A)
        v0_host = wl.make_v0(N)
        nnz_local = A.nnz
        r0, r1 = 0, N
    gen_s = time.perf_counter() - t_gen
    e = op.engine
    b_dev = torch.from_numpy(b_host).to(dev)
    v0_dev = torch.from_numpy(v0_host).to(dev)
    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream(dev)
    max_iters = args.max_iters if args.max_iters else BENCH_MAX_ITERS.get(args.config, 200000)
    cfg = pg.GmresConfig(conf["m"], conf["tol"], max_iters, poly_form=args.poly_form)

    def build(op, v0, c):
        # "policy": the reference's construction (build, else auto-degree);
        # "arnoldi": the harmonic-Ritz construction at the requested degree
        if args.construction == "arnoldi":
            return pg.build_poly_arnoldi(op, v0, conf["degree"], c), None
        return pg.build_poly_or_auto(op, v0, conf["degree"], c)

    def step(b, v0):
        c = pg.CostCounters()
        op.counters = c
        poly, pivot = build(op, v0, c)
        res = pg.solve(op, b, right_prec=poly, config=cfg)
        return poly, pivot, res, c

    # the clock sampler starts before the warm-up: nvidia-smi's own start-up
    # (driver queries) must not land inside the timed region
    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.5)
    # cold first solve: nothing recorded yet (no step graphs, cold caches and
    # workspaces), timed like a step
    flush.fill_(1.0)
    torch.cuda.synchronize()
    c0 = torch.cuda.Event(enable_timing=True)
    c1 = torch.cuda.Event(enable_timing=True)
    tc = time.perf_counter()
    c0.record(stream)
    step(b_dev, v0_dev)
    c1.record(stream)
    torch.cuda.synchronize()
    cold_wall = time.perf_counter() - tc
    cold = c0.elapsed_time(c1) / 1e3
    for _ in range(max(args.warmup - 1, 0)):
        step(b_dev, v0_dev)
    torch.cuda.synchronize()

    times, results = [], []
    e.timer = []
    launches0 = _lib.launches()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    sampler.mark()
    for _ in range(args.steps):
        flush.fill_(1.0)  # evict L2 (126 MB) between steps -- outside the events
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        out = step(b_dev, v0_dev)
        ev1.record(stream)
        results[:] = [out]  # keep only the last result: no allocator growth across steps
        times.append((ev0, ev1))
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = sampler.stop()
    launches = _lib.launches() - launches0
    per_step = [a.elapsed_time(b) / 1e3 for a, b in times]
    total = sum(per_step)
    # kernel-level roofline of the dominant kernel (fused polynomial pass)
    # e.timer: (start, end, algorithmic bytes of the stored format, passes,
    # uncompressed-equivalent bytes) per fused chain of d back-to-back
    # polynomial passes (events on the launching stream)
    kt = sum(t[0].elapsed_time(t[1]) for t in e.timer) / 1e3
    kb = sum(t[2] for t in e.timer)
    nk = sum(t[3] for t in e.timer)
    kb12 = sum(t[4] for t in e.timer)
    e.timer = None
    if world > 1:
        t = torch.tensor([total, kt], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total, kt = float(t[0]), float(t[1])
        kb_t = torch.tensor([kb, kb12], dtype=torch.float64, device=dev)
        dist.all_reduce(kb_t)
        kb, kb12 = float(kb_t[0]), float(kb_t[1])

    poly, pivot, res, c = results[-1]

    # ---- e2e: public API from pinned host buffers, x back to the host -----
    b_pin = torch.from_numpy(b_host).pin_memory()
    v0_pin = torch.from_numpy(v0_host).pin_memory()
    e2e_times = []
    # two warm-up calls: the first pinned-input solves settle the caching
    # allocator's buffers, so the recorded step graphs' keys repeat
    for i in range(max(1, min(args.steps, 10)) + 2):
        flush.fill_(1.0)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        cc = pg.CostCounters()
        op.counters = cc
        p2, _ = build(op, v0_pin, cc)
        r2 = pg.solve(op, b_pin, right_prec=p2, config=cfg)
        x_host = r2.x  # CPU tensor (D2H inside the timed region)
        torch.cuda.synchronize()
        if i > 1:  # warm-up calls excluded
            e2e_times.append(time.perf_counter() - t0)
    e2e = float(np.mean(e2e_times))
    assert x_host.device.type == "cpu"
    # the same with numpy (pageable) b / v0 in and a numpy x out: exactly the
    # reference's call signature (solve(op, b, right_prec=...), gmres.py:213)
    e2e_np_times = []
    for i in range(max(1, min(args.steps, 5)) + 1):
        flush.fill_(1.0)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        cc = pg.CostCounters()
        op.counters = cc
        p2, _ = build(op, v0_host, cc)
        r2 = pg.solve(op, b_host, right_prec=p2, config=cfg)
        assert isinstance(r2.x, np.ndarray)
        if i > 0:
            e2e_np_times.append(time.perf_counter() - t0)
    e2e_np = float(np.mean(e2e_np_times))
    if world > 1:
        t = torch.tensor([e2e, e2e_np, cold], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e, e2e_np, cold = float(t[0]), float(t[1]), float(t[2])

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(conf, (c.spmvs, res.iterations, res.cycles))

    if rank == 0:
        peak, peak_src = _peaks()
        achieved = (kb / kt / 1e9) if kt > 0 else None
        st = op.stats[0]
        line = {
            "metric": METRIC,
            "value": total / args.steps,
            "unit": "s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": 1e3 * total / args.steps,
            "step_ms": {"min": 1e3 * min(per_step), "median": 1e3 * statistics.median(per_step),
                        "max": 1e3 * max(per_step),
                        "all": [round(1e3 * t, 3) for t in per_step]},
            "higher_is_better": False,
            "scaling": "strong",
            "vs_baseline": None,
            "dtype": "f64",
            "data": "synthetic (generated operator, SplitMix64 b and v0)",
            "config": {
                "workload": conf["name"],
                "n": N, "nnz": int(nnz_local) if world == 1 else None,
                "restart_m": conf["m"], "tol": conf["tol"], "max_iters": max_iters,
                "degree_requested": conf["degree"], "degree_effective": poly.degree,
                "build_poly_failed_pivot": pivot, "poly_form": args.poly_form,
                "construction": args.construction,
                "iterations": res.iterations, "cycles": res.cycles,
                "converged": bool(res.converged), "final_relres": res.final_relres,
                "spmvs": c.spmvs, "dots": c.dots,
                "parallelism": f"rowblock{world}",
                "l2": "256 MiB buffer written between timed steps (outside the events)",
                "sell": {"padded_nnz": st["padded_nnz"], "sigma": st["sigma"]},
                "generation_s": round(gen_s, 2),
            },
            "roofline": {
                "kernel": KERNEL_NAMES[st["kernel"]] + " (fused SpMV + polynomial epilogue)",
                "bound": "hbm",
                "achieved": achieved,
                "peak": peak,
                "peak_source": peak_src,
                "unit": "GB/s",
                "frac": (achieved / peak) if achieved else None,
                "traffic": _traffic("poly_pass_bytes_per_launch", conf["name"]),
                "launches_timed": nk,
                "kernel_s_per_step": kt / args.steps,
                "share_of_step": kt / total if total else None,
                "algorithmic_bytes_per_launch": kb / max(nk, 1),
                "matrix_format": MATRIX_FORMATS[st["kernel"]],
                "stream_bytes_per_entry": st["stream_bytes"],
                "uncompressed_equivalent_gbs": (kb12 / kt / 1e9) if kt > 0 else None,
            },
            "cpu_baseline": cpu,
            "e2e": {"value": e2e, "unit": "s", "h2d_bytes_per_step": 16 * N,
                    "d2h_bytes_per_step": 8 * N,
                    "median": float(np.median(e2e_times)),
                    "all_ms": [round(1e3 * t, 3) for t in e2e_times],
                    "note": "public API (build_poly_or_auto + solve) from pinned host b/v0, x to host"},
            "e2e_numpy": {"value": e2e_np, "unit": "s", "h2d_bytes_per_step": 16 * N,
                          "d2h_bytes_per_step": 8 * N,
                          "all_ms": [round(1e3 * t, 3) for t in e2e_np_times],
                          "note": "public API with numpy (pageable) b / v0 and numpy x, the "
                                  "reference's call signature"},
            "cold_s": {"value": cold, "wall_s": cold_wall,
                       "note": "first solve in the process (before warm-up): no recorded "
                               "step graphs, cold workspaces"},
            "gpu_launches": launches,
            "clocks": clocks,
        }
        print(json.dumps(line))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


# Inner-iteration caps for the configs that do not reach their tolerance
# (config 3: random indefinite, tests/golden small3 uses 300; config 5: the
# 2048^2 recirculating flow stagnates near 1e-4, profiles/r01b/
# cfg5_degree_sweep.json), so a default bench run stays bounded.
BENCH_MAX_ITERS = {3: 300, 5: 2000}

# pg_matrix_stats()[11]: the SELL kernel pg_spmv / pg_poly_pass run (spmv.cu)
KERNEL_NAMES = {0: "sell_kernel<kPoly,0,0>", 1: "sell_kernel<kPoly,1,1>",
                2: "sell_pair_kernel<kPoly>", 3: "sell_win_kernel<kPoly>",
                4: "sell_pair_short_kernel<kPoly>", 5: "sell_pat_kernel<kPoly>",
                6: "sell_win_kernel<kPoly, patterns>", 7: "sell_opat_kernel<kPoly>",
                8: "sell_march_kernel<kPoly>", 9: "plane_ring_kernel<kPoly, 27>"}
MATRIX_FORMATS = {
    0: "SELL-C-sigma (int32 column + f64 value, 12 B/entry)",
    1: "dictionary SELL (1 B offset + 1 B value index)",
    2: "pair-dictionary SELL (1 B (offset, value) index), global x gathers",
    3: "pair-dictionary SELL (1 B/entry), x windows staged by a TMA ring",
    4: "pair-dictionary SELL (1 B/entry), rows <= 8 entries, one gather round trip",
    5: "row-pattern dictionary (1 B per row names its (offset, value) sequence; table in smem)",
    6: "row-pattern dictionary (1 B per row), x windows + pattern ids staged by a TMA ring",
    7: "offset-pattern SELL (1 B per row names the column offsets; f64 values, 8 B/entry)",
    8: "row-pattern dictionary (1 B per row), plane-marching: x planes kept in registers",
    9: "row-pattern plane stencil: x plane windows, pattern ids (boundary planes only) and "
       "epilogue operands staged by a TMA ring; each x value loaded once per plane, used by "
       "three rows",
}


# ---------------------------------------------------------------------------
# CPU baseline (oracle port) -- bounded sample, extrapolated
# ---------------------------------------------------------------------------
def _sum_basis_widths(iterations, cycles, m):
    """sum over the solve's Arnoldi steps of the basis width k the ICGS
    projects against (k = j + 1 at step j of a cycle)."""
    total, left = 0, iterations
    for _ in range(cycles):
        steps = min(m, left)
        total += steps * (steps + 1) // 2
        left -= steps
    return total


def cpu_baseline(conf, counts, threads=1, probe=None, max_spmvs=None):
    """Bounded sample of the reference's CPU path on the full workload: one
    whole Arnoldi step -- A p(A) v as d + 1 operator applications with the
    running-power recurrence (polyprec.py:193-212, gmres.py:98-113, through
    the oracle port) and one ICGS at basis width m/2 (ortho.py:33-70) --
    timed (about 15-20 s on cfg4); extrapolated with the solve's operation
    counts ``counts`` = (spmvs, iterations, cycles): the per-application time
    of the step times the solve's SpMV count (build, steps, recovery and
    residuals alike; the SpMVs dominate) plus the ICGS time
    scaled by the summed basis widths.  ``probe`` reuses a generated operator;
    ``max_spmvs`` shortens the sampled chain (the reference arm repeats the
    sample --steps + --warmup times and must end within minutes)."""
    from threadpoolctl import threadpool_limits

    from oracle import pgmres_oracle as orc

    if probe is None:
        probe = _cpu_probe(conf)
    A, b, V, w = probe
    spmvs, iterations, cycles = counts
    kw = V.shape[1]
    d = max(1, int(round(spmvs / max(iterations, 1))) - 1)
    if max_spmvs:
        d = max(1, min(d, max_spmvs - 1))
    y = np.full(d + 1, 0.5)
    with threadpool_limits(limits=threads):
        t0 = time.perf_counter()
        A.apply(orc.poly_eval(y, A, b, orc.Tally()))
        t1 = time.perf_counter()
        orc.cgs2(V, w, orc.Tally())
        t2 = time.perf_counter()
    t_spmv, t_icgs = (t1 - t0) / (d + 1), t2 - t1
    widths = _sum_basis_widths(iterations, cycles, conf["m"])
    est = spmvs * t_spmv + t_icgs * widths / kw
    return {"value": est, "unit": "s", "cores": threads, "kind": "port",
            "sample": (f"oracle port of the reference on the full {conf['name']} operator: one "
                       f"A p(A) v chain of {d + 1} SpMVs ({t_spmv:.3f} s each, "
                       f"recurrence included) + one ICGS at basis width {kw} ({t_icgs:.3f} s), "
                       f"extrapolated to the solve's {spmvs} SpMVs and {iterations} ICGS steps "
                       f"({cycles} cycles)"),
            "measured_s": round(t1 - t0 + t_icgs, 3), "spmv_s": t_spmv, "icgs_s": t_icgs}


def _cpu_probe(conf):
    from oracle import pgmres_oracle as orc

    A_h = wl.make_matrix(conf)
    A = orc.OracleMatrix.of(A_h, orc.Tally())
    b = wl.make_rhs(conf, A_h)
    n = A_h.nrows
    kw = max(1, conf["m"] // 2)
    # a basis stand-in: the ICGS time does not depend on the values (four
    # dense passes over V, ortho.py:53-59)
    V = np.asfortranarray(np.stack([wl.splitmix_uniform(10 + i, n) for i in range(kw)], axis=1))
    V /= np.sqrt(n)
    return A, b, V, wl.make_v0(n)


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    conf = wl.CONFIGS[args.config]
    rec = _reference_record(args.config)
    threads = os.cpu_count() or 1
    probe = _cpu_probe(conf)
    vals = []
    for i in range(args.warmup + args.steps):
        cb = cpu_baseline(conf, (rec["spmvs"], rec["iterations"], rec["cycles"]), threads=threads,
                          probe=probe, max_spmvs=4)
        if i >= args.warmup:
            vals.append(cb)
    v = float(np.mean([c["value"] for c in vals]))
    cb = dict(vals[-1])
    cb["value"] = v
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * v,
        "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": {
            "workload": conf["name"], "n": wl.config_n(conf), "restart_m": conf["m"],
            "tol": conf["tol"], "degree_requested": conf["degree"],
            "degree_effective": rec["degree"], "iterations": rec["iterations"],
            "cycles": rec["cycles"], "spmvs": rec["spmvs"], "record": rec["source"],
            "full_solve_measured_build_host_s": rec.get("measured_s")},
        "cpu_baseline": cb,
        "e2e": {"value": v, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


def _reference_record(config: int) -> dict:
    """The reference's own full-size run of this workload (degree decision,
    iterations, cycles, operator applications), recorded in the build
    container by tests/golden/make_full_records.py."""
    path = os.path.join(ROOT, "tests", "golden", f"cfg{config}_full_reference.json")
    try:
        with open(path) as fh:
            g = json.load(fh)
        return {"degree": g["effective_degree"], "iterations": g["iterations"],
                "cycles": g["cycles"], "spmvs": g["counters"]["spmvs"],
                "measured_s": round(g["build_s"] + g["solve_s"], 1),
                "source": f"tests/golden/cfg{config}_full_reference.json"}
    except (OSError, KeyError, ValueError):
        conf = wl.CONFIGS[config]
        return {"degree": None, "iterations": 50, "cycles": 1,
                "spmvs": (conf["degree"] + 1) * 52, "measured_s": None,
                "source": "no full-size record: one cycle assumed"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    # default: the reference's cap (200000), except the configs whose
    # operators stagnate under GMRES(m) at their tolerance (BENCH_MAX_ITERS)
    ap.add_argument("--max-iters", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"])
    # "monomial" = the reference's bit-identical evaluation (default, the
    # headline); "roots" = the Leja root-product form
    ap.add_argument("--poly-form", default="monomial", choices=["monomial", "roots"])
    # "arnoldi" builds the requested degree from harmonic Ritz values (SURVEY
    # f1) -- not the reference's construction, so not the headline
    ap.add_argument("--construction", default="policy", choices=["policy", "arnoldi"])
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "0"))
    if world == 0 and args.gpus > 1:
        # --gpus N without a launcher: start the N ranks ourselves (one process
        # per GPU, the driver's torchrun command line) and pass on the exit code
        import socket
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
               f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
        raise SystemExit(subprocess.call(cmd))
    if world and world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; launch one "
                         "rank per GPU with matching --gpus")
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
