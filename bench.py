"""Benchmark of the ECMG_jcg hot path on B200 (driver contract: one JSON line from rank 0).

Workload (BASELINE.json metric "fine-grid JCG unknown-iters/s (fp64) + ECMG time-to-solution at
512^3"): configs[3] = C4, the singular solution u = r^{3/2} on the unit cube, beta = 1, Dirichlet
everywhere, Q1 FE on 4^3 -> 512^3 (8 levels, 133,432,831 free unknowns on the finest grid),
fp64, eps = 1e-9, final Richardson extrapolation.

  step         one ecmg_run: all §8(a) rows (per-level setup, DSOLVE, EXP_finite, JCG, EXP_true)
  ms_per_step  ECMG time-to-solution (device time, CUDA events, max over ranks) -- the metric's second half
  value        whole-step JCG throughput: sum over ALL levels of free unknowns x JCG iterations, divided by
               the time-to-solution ("unknown-iters/s" of the whole cascade, setup/EXP time included in the
               denominator). The metric's first half, the FINE-grid JCG unknown-iters/s, is reported as
               fine_grid_jcg_in_run (the 512^3 level inside the run) and jcg_fixed (below)
  jcg_fixed    the fine-grid JCG unknown-iters/s of SURVEY.md §8d D.1(i): 100 iterations of the
               512^3 system from a seeded guess, stopping test off, CUDA events
  jcg_fixed_c5 the same on C5's 1024^3 element operator (20 iterations), z-slab sharded at N > 1: the
               multi-GPU efficiency metric of north_star
  roofline     the fused JCG iteration (K1 + K2) against the measured HBM copy peak
  e2e          the same ecmg_run through the C ABI with HOST output buffers (D2H inside the step)
  e2e_arrays   C4 given as the caller's own arrays (ECMG_PROB_ARRAYS): H2D of every level's f and g_D,
               ecmg_run, D2H of u~_h, all inside the step
  cpu_baseline the CPU oracle (oracle/, as it stands) on the full config, all host cores, rank 0, N = 1

--impl reference times the oracle (the reference arm of this tier) on the host cores.
Inputs larger than L2 (5+ GB working set vs 126 MB L2): no explicit L2 flush between steps.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fine-grid JCG unknown-iters/s (fp64) + ECMG time-to-solution at 512^3"
UNIT = "unknown-iters/s"
BYTES_PER_UNKNOWN_ITER = 64   # x 1R+1W, r 2R+1W, p 2R+1W (constant-beta path)
# constant-beta path with the deferred x update (ECMG_OPT_XDEFER, default on one GPU): per pair of iterations
# K1 24 B, K2 without x 24 B, K1 24 B, K2 with x and p_{k-1} 48 B = 120 B, i.e. 60 B per unknown and iteration
BYTES_PER_UNKNOWN_ITER_XDEFER = 60

CONFIGS = {
    # name: (problem id, coarsest, levels, eps, description); C3 / C5 run the element-beta path (80 B/unknown)
    "c4": (4, 4, 8, 1e-9, "C4 (BASELINE configs[3]): u=r^{3/2}, beta=1, Dirichlet, Q1, 4^3->512^3, eps=1e-9"),
    "c2": (2, 4, 6, 1e-10, "C2 (BASELINE configs[1]): u=exp(x+y+z), beta=1, Dirichlet, Q1, 4^3->128^3, eps=1e-10"),
    "c1": (1, 4, 4, 1e-8, "C1 (BASELINE configs[0]): u=sin sin sin, beta=1, Dirichlet, Q1, 4^3->32^3, eps=1e-8"),
    "c3": (3, 4, 7, 1e-10, "C3 (BASELINE configs[2]): variable beta, Robin z=1, Q1, 4^3->256^3, eps=1e-10"),
    "c5": (5, 4, 9, 1e-8, "C5 (BASELINE configs[4]): layered geology (seed 0), Dirichlet, Q1, 4^3->1024^3, eps=1e-8"),
}
# element-beta path (kernels_jcg_elem.cu): K1 reads z, p_old, beta_e and writes p; K2 reads p, beta_e,
# x, z and writes x, z (the residual is carried as z = D^-1 r only; K2 forms r = D z): 10 x 8 B, the
# survey's algorithmic 80 B. With ECMG_OPT_BETA_FLY = 1 (ablation) beta_e is formed in registers from
# per-axis tables: 8 x 8 B
BYTES_PER_UNKNOWN_ITER_ELEM = 80


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region. The sampler is started and its
    first (idle) sample awaited before the region opens, so that nvidia-smi's start-up does not eat a short
    region; samples are kept by arrival time (every 20 ms) from the region's start to just after its end."""

    def __init__(self, index: int):
        self.index, self.samples, self.proc = index, [], None
        self.t0, self.t1 = None, None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            t_wait = time.monotonic()
            while not self.samples and time.monotonic() - t_wait < 5.0:
                time.sleep(0.005)
        except Exception:
            self.proc = None
        self.t0 = time.monotonic()
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append((time.monotonic(), [s.strip() for s in line.split(",")]))

    def __exit__(self, *exc):
        self.t1 = time.monotonic()
        if self.proc:
            t_wait = time.monotonic()
            while (not any(t >= self.t0 for t, _ in self.samples)) and time.monotonic() - t_wait < 0.5:
                time.sleep(0.005)
            time.sleep(0.05)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        inside = [v for t, v in self.samples if self.t0 <= t <= self.t1 + 0.06]
        window = "timed region"
        if not inside:   # a region shorter than one sampling period: the first sample after it
            inside = [v for t, v in self.samples if t >= self.t0][:1]
            window = "first sample after the timed region"
        if not inside:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(s[0]) for s in inside if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in inside if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in inside for i in range(4) if len(s) > 3 + i and s[3 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(inside), "window": window}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def host_info():
    info = {"nproc": os.cpu_count()}
    try:
        with open("/proc/cpuinfo") as f:
            info["cpu_model"] = next(l.split(":", 1)[1].strip() for l in f if l.startswith("model name"))
        with open("/proc/meminfo") as f:
            info["ram_gb"] = round(int(next(l.split()[1] for l in f if l.startswith("MemTotal"))) / 2 ** 20, 1)
    except Exception:
        pass
    return info


def cpu_oracle_run(cfg_name):
    """The oracle (oracle/, as it stands) on the FULL workload of the config -- for C4 the whole Alg. 4 cascade
    4^3 -> 512^3 at eps 1e-9, the same problem the GPU step solves -- in its row-parallel OpenMP mode on every
    host core (bitwise the serial oracle, tests/test_oracle_threads.py). One run is one step; its units are
    sum_k free_k x iterations_k, as for the GPU line."""
    import oracle
    import synth
    pid, n0, levels, eps, _ = CONFIGS[cfg_name]
    threads = oracle.max_threads()
    oracle.set_threads(threads)
    t0 = time.perf_counter()
    st, stats, _, _ = oracle.ecmg(n0, levels, pid, eps, params=synth.c5_geometry(0) if pid == 5 else None)
    dt = time.perf_counter() - t0
    units = float(sum(max(0, r[0]) * r[16] for r in stats))
    hi = host_info()
    return {"value": units / dt, "unit": UNIT, "cores": threads, "kind": "oracle",
            "sample": f"the full {cfg_name.upper()} workload ({n0}^3 -> {n0 * 2 ** (levels - 1)}^3, {levels} levels, "
                      f"eps={eps}), OpenMP row-parallel oracle on {threads} threads ({hi.get('cpu_model', '?')}, "
                      f"{hi.get('ram_gb', '?')} GB RAM); units = sum_k free_k*iters_k = {units:.4g}; wall {dt:.2f} s",
            "iterations_per_level": [int(r[0]) for r in stats], "status": int(st), "wall_s": dt, "host": hi}


REFERENCE_BUDGET_S = 240.0


def run_reference(args):
    """The reference arm of this tier: the oracle on the same config, metric and unit as the product arm. One
    step = one full Alg. 4 run of the config on all host cores (~1 min for C4 512^3 on 16 cores), so the
    requested --steps K are capped to what fits in REFERENCE_BUDGET_S (at least one) and the line reports the
    number run; the oracle keeps no state between runs (every level is rebuilt from scratch), so no warm-up
    runs are made."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    cfg = CONFIGS[args.config]
    samples = []
    t_start = time.perf_counter()
    while len(samples) < args.steps:
        samples.append(cpu_oracle_run(args.config))
        el = time.perf_counter() - t_start
        if el + el / len(samples) > REFERENCE_BUDGET_S:
            break
    v = statistics.mean(s["value"] for s in samples)
    ms = statistics.mean(s["wall_s"] for s in samples) * 1e3
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": len(samples), "steps_requested": args.steps, "warmup": 0, "warmup_requested": args.warmup,
            "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": f"synthetic (analytic {args.config.upper()} problem; no dataset)",
            "config": {"workload": cfg[4], "levels": cfg[2], "eps": cfg[3]},
            "iterations_per_level": samples[-1]["iterations_per_level"],
            "cpu_baseline": dict({k: samples[-1][k] for k in ("unit", "cores", "kind", "sample")}, value=v),
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "note": f"steps capped to a {REFERENCE_BUDGET_S:.0f} s budget; one step = one full oracle run of the config"}
    print(json.dumps(line), flush=True)
    return 0


def bench_c5_fixed(args, gdist, ws, max_over_ranks, iters=20):
    """SURVEY.md §8d D.1 (i) on C5 (BASELINE configs[4]), the element-beta operator at 1024^3 whose multi-GPU
    efficiency north_star targets (>= 80% at 8 GPUs): `iters` fixed JCG iterations of the finest system
    (x0 = 0; C5's b != 0, so the residual cannot vanish in 20 iterations), stopping test off, CUDA events,
    median of 3 after a warm-up solve that also runs the level's setup. At N ranks the level is z-slab
    sharded exactly as in ecmg_run, so the per-N lines give the efficiency curve. Reported as whole-job U/s
    and as a per-GPU roofline fraction at the survey's algorithmic 80 B/unknown (§8d D.3)."""
    import torch
    import synth
    from paper_1506_02983_b200 import Grid, ecmg
    pid, n0, levels, _, _ = CONFIGS["c5"]
    try:
        g5 = Grid(n0, levels, pid, synth.c5_geometry(0), dist=gdist)
        fine = levels - 1
        _, nodes5 = g5.shape(fine)
        x = torch.zeros(nodes5, dtype=torch.float64, device="cuda")
        g5.solve_level(fine, 0.0, 2, x)   # warm-up + level setup
        runs = []
        for _ in range(3):
            x.zero_()
            g5.solve_level(fine, 0.0, iters, x)
            runs.append(g5.last_jcg_timing())
        ms, it, nf = sorted(runs)[1]
        ms = max_over_ranks(ms)
        if ws > 1:
            import torch.distributed as dist
            t = torch.tensor([float(nf)], dtype=torch.float64, device="cuda")
            dist.all_reduce(t)
            nf = int(t.item())
        g5.close()
        del x
        torch.cuda.empty_cache()
    except Exception as ex:   # e.g. ENOMEM on a smaller GPU: reported, never silently dropped
        return {"skipped": f"{type(ex).__name__}: {ex}"}
    peak, _ = load_peaks()
    ups = nf * it / (ms / 1e3)
    per_gpu_gbs = 80 * ups / 1e9 / ws
    return {"value": ups, "unit": UNIT, "n_gpus": ws, "iterations": it, "ms": ms, "ms_per_iteration": ms / it,
            "free_unknowns": nf, "workload": "C5 1024^3 element-beta operator, x0 = 0, stopping test off",
            "roofline_per_gpu": {"achieved": per_gpu_gbs, "peak": peak, "unit": "GB/s", "frac": per_gpu_gbs / peak,
                                 "bytes_per_unit": 80, "note": "algorithmic 80 B/unknown (SURVEY.md §8d D.3)"}}


def c4_level_arrays(n0, levels):
    """C4's data of Eq. (bvp) in ECMG_PROB_ARRAYS form, per level (include/ecmg.h): f = -(15/4) r^{-1/2} at the
    2x2x2 Gauss points of every element (index 8 e + q, q = qx + 2 qy + 4 qz) and g_D = r^{3/2} at every node;
    beta = 1 and no Robin faces (NULL). Input generation only, outside any timed region: formed with torch on
    the device in z-chunks, then kept in pinned host memory as the caller's data."""
    import torch
    g = 0.57735026918962576451
    out = []
    for k in range(levels):
        n = n0 * 2 ** k
        h = 1.0 / n
        ax = torch.arange(n, dtype=torch.float64, device="cuda")
        gp = torch.stack([(ax + (1 - g) / 2) * h, (ax + (1 + g) / 2) * h], dim=1)   # [n, 2]
        q = torch.arange(8, device="cuda")
        fq = torch.empty(n * n * n * 8, dtype=torch.float64).pin_memory()
        X = gp[:, q & 1].view(1, 1, n, 8)
        Y = gp[:, (q >> 1) & 1].view(1, n, 1, 8)
        zc = max(1, (1 << 24) // (n * n))
        for z0 in range(0, n, zc):
            z1 = min(n, z0 + zc)
            Z = gp[z0:z1, (q >> 2) & 1].view(z1 - z0, 1, 1, 8)
            r2 = X * X + Y * Y + Z * Z
            fq[z0 * n * n * 8:z1 * n * n * 8].copy_((-3.75 * r2.pow(-0.25)).reshape(-1))
        an = torch.arange(n + 1, dtype=torch.float64, device="cuda") * h
        gd = torch.empty((n + 1) ** 3, dtype=torch.float64).pin_memory()
        zc = max(1, (1 << 24) // ((n + 1) ** 2))
        for z0 in range(0, n + 1, zc):
            z1 = min(n + 1, z0 + zc)
            r2 = an.view(1, 1, -1) ** 2 + an.view(1, -1, 1) ** 2 + an[z0:z1].view(-1, 1, 1) ** 2
            gd[z0 * (n + 1) ** 2:z1 * (n + 1) ** 2].copy_(r2.pow(0.75).reshape(-1))
        out.append((fq, gd))
    torch.cuda.synchronize()
    return out


def bench_e2e_arrays(args, n0, levels, eps, nodes, grid_analytic):
    """The headline step through the public API as a caller with their OWN data would run it: C4 given as
    ECMG_PROB_ARRAYS (f at the Gauss points and g_D at the nodes of every level, in pinned host memory); each
    step copies every level's arrays H2D into the grid's bound device buffers, runs ecmg_run and reads the
    extrapolated solution u~_h back into pinned host memory. Host wall clock over the steps. The same numbers
    as the analytic run are checked (u~_h of both within 1e-12 relative)."""
    import torch
    from paper_1506_02983_b200 import Grid, ecmg
    try:
        host = c4_level_arrays(n0, levels)
        dev = [(torch.empty_like(fq, device="cuda"), torch.empty_like(gd, device="cuda")) for fq, gd in host]
        for (df, dg), (hf, hg) in zip(dev, host):
            df.copy_(hf)
            dg.copy_(hg)
        ga = Grid(n0, levels, ecmg.PROB["ARRAYS"], params=[0.0] * 6, faces=[0] * 6,
                  level_arrays=[(None, df, dg, None) for df, dg in dev])
        u = torch.empty(nodes, dtype=torch.float64, device="cuda")
        uth = torch.empty(nodes, dtype=torch.float64).pin_memory()
        ga.run(eps, u, uth)   # warm-up
        ut_ref = torch.empty(nodes, dtype=torch.float64, device="cuda")
        grid_analytic.run(eps, torch.empty_like(u), ut_ref)
        dmax = float((uth.cuda() - ut_ref).abs().max() / ut_ref.abs().max())
        del ut_ref
        h2d = sum(fq.numel() + gd.numel() for fq, gd in host) * 8
        steps = max(1, min(args.steps, 3))
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        units = 0.0
        for _ in range(steps):
            for (df, dg), (hf, hg) in zip(dev, host):
                df.copy_(hf, non_blocking=True)
                dg.copy_(hg, non_blocking=True)
            st, stats = ga.run(eps, u, uth)
            assert st == 0
            for k, s_ in enumerate(stats):
                shp, _ = ga.shape(k)
                units += (shp[0] - 1) * (shp[1] - 1) * (shp[2] - 1) * s_["iterations"]
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        ga.close()
        del dev, host, u, uth
        torch.cuda.empty_cache()
    except Exception as ex:
        return {"skipped": f"{type(ex).__name__}: {ex}"}
    return {"value": units / dt, "unit": UNIT, "ms_per_step": dt / steps * 1e3, "steps": steps,
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": nodes * 8, "max_rel_diff_vs_analytic": dmax,
            "note": "C4 as ECMG_PROB_ARRAYS: every level's f (2x2x2 Gauss points) and g_D (nodes) copied from pinned "
                    "host memory inside the step, ecmg_run, u~_h read back into pinned host memory; host wall clock"}


def relaunch(n):
    """`bench.py --gpus N` outside torchrun: re-launch this command as N ranks (one per GPU) under
    torch.distributed.run on 127.0.0.1, or fail clearly when the box has fewer than N GPUs."""
    import socket
    import torch
    have = torch.cuda.device_count()
    if have < n:
        print(json.dumps({"error": f"--gpus {n} needs {n} GPUs, this box has {have}"}), flush=True)
        return 1
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ecmg", choices=["ecmg", "reference"])
    ap.add_argument("--config", default="c4", choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--fixed-iters", type=int, default=100)
    ap.add_argument("--no-c5", action="store_true", help="skip the C5 1024^3 fixed-iteration key")
    ap.add_argument("--no-arrays", action="store_true", help="skip the ECMG_PROB_ARRAYS e2e key")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch(args.gpus)
    ws_env = int(os.environ.get("WORLD_SIZE", "1"))
    if ws_env != args.gpus:
        print(json.dumps({"error": f"--gpus {args.gpus} but WORLD_SIZE={ws_env}: launch one rank per GPU"}), flush=True)
        return 1
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_1506_02983_b200 import Grid, ecmg

    pid, n0, levels, eps, desc = CONFIGS[args.config]
    stream = torch.cuda.current_stream()
    gdist = None
    if ws > 1:
        # z-slab decomposition over NCCL ranks (strong scaling of the same C4 problem)
        from paper_1506_02983_b200 import dist as edist
        gdist = edist.ecmg_dist_from_torch(device=torch.device("cuda", local))
    import synth as _synth
    params = _synth.c5_geometry(0) if pid == 5 else None
    grid = Grid(n0, levels, pid, params, dist=gdist)
    shape, nodes = grid.shape(levels - 1)      # nodes: this rank's planes of the finest level
    zlo, zhi = ecmg.level_shape(grid.h, levels - 1)[3:5]
    u = torch.empty(nodes, dtype=torch.float64, device="cuda")
    ut = torch.empty(nodes, dtype=torch.float64, device="cuda")

    def barrier():
        torch.cuda.synchronize()
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x):
        if ws == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for _ in range(max(3, args.warmup)):
        grid.run(eps, u, ut)

    # ---- timed region: K ECMG runs ------------------------------------------------------------
    barrier()
    l0 = ecmg.kernel_launches()
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    units_total, fine_units, fine_ms = 0.0, 0.0, 0.0
    per_level = None
    with ClockSampler(local) as clk:
        barrier()   # the ranks' samplers have started: open the region together
        evs[0].record(stream)
        for _ in range(args.steps):
            st, stats = grid.run(eps, u, ut)
            assert st == 0, ecmg.strerror(st)
            per_level = stats
            ms_j, it_j, nf_j = grid.last_jcg_timing()
            fine_units += nf_j * it_j
            fine_ms += ms_j
            for k, s in enumerate(stats):
                shp, _ = grid.shape(k)
                nfree = (shp[0] - 1) * (shp[1] - 1) * (shp[2] - 1)
                units_total += nfree * s["iterations"]
        evs[1].record(stream)
        barrier()
    launches = ecmg.kernel_launches() - l0
    t_ms = max_over_ranks(evs[0].elapsed_time(evs[1]))
    ms_per_step = t_ms / args.steps
    value = units_total / (t_ms / 1e3)   # units of the whole (global) problem

    # ---- fixed-iteration fine-grid JCG benchmark and roofline --------------
    import numpy as np
    import synth
    fine = levels - 1
    x0_full = synth.random_nodal(14, shape, (1, 1, 1), tuple(v - 1 for v in shape))
    pl = (shape[0] + 1) * (shape[1] + 1)
    x0 = torch.from_numpy(x0_full[zlo * pl:zhi * pl].copy()).cuda()   # this rank's planes
    xb = x0.clone()
    grid.solve_level(fine, 0.0, 5, xb)   # warm-up (also sets up the level)
    jt = []
    for _ in range(3):
        xb.copy_(x0)
        grid.solve_level(fine, 0.0, args.fixed_iters, xb)
        ms_j, it_j, nf_j = grid.last_jcg_timing()
        jt.append((ms_j, it_j, nf_j))
    ms_j, it_j, nf_j = sorted(jt)[len(jt) // 2]
    ms_j = max_over_ranks(ms_j)
    if ws > 1:   # free unknowns of the whole problem
        t = torch.tensor([float(nf_j)], dtype=torch.float64, device="cuda")
        dist.all_reduce(t)
        nf_j = int(t.item())
    jcg_ups = nf_j * it_j / (ms_j / 1e3)
    # ablation: the register-prefetch (non-TMA) kernels on the same system
    grid.set_option(ecmg.OPT_KERNEL, 0)
    xb.copy_(x0)
    grid.solve_level(fine, 0.0, args.fixed_iters, xb)
    ms_p, it_p, _ = grid.last_jcg_timing()
    ms_p = max_over_ranks(ms_p)
    grid.set_option(ecmg.OPT_KERNEL, 1)
    ablation_xdefer = None
    if pid not in (3, 5) and ws == 1:   # ablation: x updated in every K2 (64 B/unknown)
        grid.set_option(ecmg.OPT_XDEFER, 0)
        xb.copy_(x0)
        grid.solve_level(fine, 0.0, args.fixed_iters, xb)
        ms_x, it_x, _ = grid.last_jcg_timing()
        grid.set_option(ecmg.OPT_XDEFER, 1)
        ablation_xdefer = {"value": nf_j * it_x / (ms_x / 1e3), "unit": UNIT, "ms_per_iteration": ms_x / max(1, it_x),
                           "kernel": "x updated in every K2 (ECMG_OPT_XDEFER=0), 64 B/unknown"}
    ablation_unfused = None
    if pid not in (3, 5) and ws == 1:   # ablation: the unfused textbook PCG sequence (9 passes, 144 B/unknown)
        grid.set_option(ecmg.OPT_UNFUSED, 1)
        xb.copy_(x0)
        grid.solve_level(fine, 0.0, 20, xb)
        ms_u, it_u, _ = grid.last_jcg_timing()
        ms_u = max_over_ranks(ms_u)
        grid.set_option(ecmg.OPT_UNFUSED, 0)
        ablation_unfused = {"value": nf_j * it_u / (ms_u / 1e3), "unit": UNIT, "ms_per_iteration": ms_u / max(1, it_u),
                            "kernel": "unfused textbook PCG (ECMG_OPT_UNFUSED=1): 9 passes, 144 B/unknown"}
    ablation_beta = None
    if pid in (3, 5):   # ablation: the element kernels form beta on the fly instead of reading the array
        grid.set_option(ecmg.OPT_BETA_FLY, 1)
        xb.copy_(x0)
        grid.solve_level(fine, 0.0, args.fixed_iters, xb)
        ms_b, it_b, _ = grid.last_jcg_timing()
        ms_b = max_over_ranks(ms_b)
        grid.set_option(ecmg.OPT_BETA_FLY, 0)
        ablation_beta = {"value": nf_j * it_b / (ms_b / 1e3), "unit": UNIT, "ms_per_iteration": ms_b / max(1, it_b),
                         "kernel": "element kernels forming beta_e from per-axis tables (ECMG_OPT_BETA_FLY=1), 64 B/unknown"}
    # ablation: host-driven JCG loop (batched readbacks) instead of the CUDA-graph WHILE loop
    grid.set_option(ecmg.OPT_GRAPH, 0)
    grid.run(eps, u, ut)
    ev_h = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev_h[0].record(stream)
    grid.run(eps, u, ut)
    ev_h[1].record(stream)
    torch.cuda.synchronize()
    tts_hostloop = max_over_ranks(ev_h[0].elapsed_time(ev_h[1]))
    grid.set_option(ecmg.OPT_GRAPH, 1)
    # ablation: every level's setup in line before its solve instead of ahead on a low-priority stream
    grid.set_option(ecmg.OPT_SETUP_AHEAD, 0)
    grid.run(eps, u, ut)
    ev_s = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev_s[0].record(stream)
    grid.run(eps, u, ut)
    ev_s[1].record(stream)
    torch.cuda.synchronize()
    tts_inline = max_over_ranks(ev_s[0].elapsed_time(ev_s[1]))
    grid.set_option(ecmg.OPT_SETUP_AHEAD, 1)
    peak, peak_src = load_peaks()
    # achieved = the ALGORITHMIC bytes of SURVEY.md §8d D.3 (64 B constant path, 80 B element path) per second. With
    # the deferred x update the constant path moves fewer (60 B, confirmed by ncu: `traffic`): `moved` reports
    # the bandwidth at the bytes the kernels really move, so that no figure hides behind the other
    bpu = BYTES_PER_UNKNOWN_ITER_ELEM if pid in (3, 5) else BYTES_PER_UNKNOWN_ITER
    bpu_moved = BYTES_PER_UNKNOWN_ITER_XDEFER if (pid not in (3, 5) and ws == 1 and it_j % 2 == 0) else bpu
    achieved = bpu * nf_j * it_j / (ms_j / 1e3) / 1e9 / ws   # per GPU
    moved = bpu_moved * nf_j * it_j / (ms_j / 1e3) / 1e9 / ws
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "jcg_traffic.json")) as f:
            traffic = json.load(f)[args.config]["bytes_per_iteration_k1_k2"]   # ncu, per K1 + K2 pair
    except Exception:
        pass

    # ---- fine-grid JCG on C5's 1024^3 element operator (north_star's multi-GPU target metric) -----
    c5_fixed = None
    if not args.no_c5 and args.config == "c4":
        c5_fixed = bench_c5_fixed(args, gdist, ws, max_over_ranks)

    # ---- e2e with the caller's data: ECMG_PROB_ARRAYS, level arrays copied H2D inside the step ----
    e2e_arrays = None
    if not args.no_arrays and args.config == "c4" and ws == 1:
        e2e_arrays = bench_e2e_arrays(args, n0, levels, eps, nodes, grid)

    # ---- e2e: the same call with host output buffers -------------------------------------------
    # the step's result is the extrapolated fourth-order solution u~_h (Alg. 4 l.10), read back into pinned
    # host memory inside the call; u_h stays in device memory
    uth = torch.empty(nodes, dtype=torch.float64).pin_memory()
    grid.run(eps, u, uth)
    barrier()
    t0 = time.perf_counter()
    e_units = 0.0
    e_steps = max(1, min(args.steps, 3))
    for _ in range(e_steps):
        st, stats = grid.run(eps, u, uth)
        for k, s in enumerate(stats):
            shp, _ = grid.shape(k)
            e_units += (shp[0] - 1) * (shp[1] - 1) * (shp[2] - 1) * s["iterations"]
    barrier()
    e_s = max_over_ranks(time.perf_counter() - t0)
    e2e = {"value": e_units / e_s, "unit": UNIT, "h2d_bytes_per_step": 0,
           "d2h_bytes_per_step": nodes * 8, "ms_per_step": e_s / e_steps * 1e3,
           "note": "C ABI ecmg_run returning the extrapolated solution u~_h into pinned host memory (D2H inside "
                   "the call, host wall clock); the problem data are analytic (no H2D)"}

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        try:
            c = cpu_oracle_run(args.config)
            cpu = {k: c[k] for k in ("value", "unit", "cores", "kind", "sample")}
            cpu["iterations_per_level"] = c["iterations_per_level"]
        except Exception as ex:   # the oracle is a reported baseline, never a fallback
            cpu = {"value": None, "unit": UNIT, "cores": None, "kind": "oracle", "sample": f"failed: {ex}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": max(3, args.warmup), "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": f"synthetic (analytic {args.config.upper()} problem; no dataset)",
            "config": {"workload": desc, "levels": levels, "finest_cells": list(shape), "eps": eps,
                       "free_unknowns_finest": int(nf_j),
                       "parallelism": f"z-slabs over {ws} NCCL ranks (levels with n >= 256, n % 4P == 0 and n/P >= 16 sharded; smaller levels replicated)"
                       if ws > 1 else "single GPU",
                       "l2": "inputs larger than L2 (no flush)",
                       "value_definition": "sum over all levels of free unknowns x JCG iterations / ECMG time-to-solution",
                       "iterations_per_level": [s["iterations"] for s in per_level]},
            "ecmg_tts_ms": ms_per_step,
            "ecmg_tts_ms_ablation_hostloop": tts_hostloop,
            "ecmg_tts_ms_ablation_setup_inline": tts_inline,
            "fine_grid_jcg_in_run": {"value": fine_units / (fine_ms / 1e3), "unit": UNIT,
                                     "iterations": int(per_level[-1]["iterations"]),
                                     "window": "the finest level's whole solve: init pass, the iterations, and the "
                                               "true-residual pass, which also forms EXP_true (ECMG_OPT_RICH_FUSED)"},
            "jcg_fixed": {"value": jcg_ups, "unit": UNIT, "iterations": it_j, "ms": ms_j,
                          "ms_per_iteration": ms_j / it_j, "kernel": "TMA-fed (default)"},
            "jcg_fixed_ablation_prefetch": {"value": nf_j * it_p / (ms_p / 1e3), "unit": UNIT,
                                            "ms_per_iteration": ms_p / max(1, it_p),
                                            "kernel": "register-prefetch loads (ECMG_OPT_KERNEL=0)"},
            "jcg_fixed_ablation_beta_fly": ablation_beta,
            "jcg_fixed_ablation_xdefer": ablation_xdefer,
            "jcg_fixed_ablation_unfused": ablation_unfused,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                         "traffic": traffic, "kernel": "jcg K1+K2 (one CG iteration)",
                         "bytes_per_unit": bpu, "peak_source": peak_src,
                         "note": "achieved / frac count SURVEY.md §8d's algorithmic bytes (64 B constant path, 80 B "
                                 "element path); the constant-path kernels move 60 B (deferred x update), so frac "
                                 "can come close to 1 -- moved.frac is the share of the peak the hardware delivers",
                         "moved": {"bytes_per_unit": bpu_moved, "achieved": moved, "frac": moved / peak,
                                   "note": "bytes the kernels move per unknown and iteration (deferred x update: "
                                           "60 B on the constant path); `traffic` is the ncu DRAM figure"},
                         "per": "GPU (average over ranks)",
                         # also against BASELINE's "about 8 TB/s" (target >= 0.70 of it)
                         "frac_nominal_8tbs": achieved / 8000.0},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "e2e_arrays": e2e_arrays,
            "jcg_fixed_c5": c5_fixed,
            "gpu_launches": int(launches),
            "clocks": clk.summary(),
            "per_level_ms": [{"setup": s["ms_setup"], "exp": s["ms_exp"], "solve": s["ms_solve"], "rich": s["ms_rich"]}
                             for s in per_level],
        }
        print(json.dumps(line), flush=True)
    grid.close()
    if ws > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
