"""Write the full-size Alg. 4 goldens tests/golden/fullsize_<cfg>.json -- calls ONLY oracle/ (and synth/ for the
seeded inputs / sample positions). The GPU tests (tests/test_gpu_fullsize_golden.py) compare the CUDA path's
ecmg_run against these numbers at the configured sizes, where the oracle itself takes minutes and tens of GB
and cannot run inside the driver's `pytest -m gpu` budget (VERDICT r01 "next round" item 1).

What is stored per config (BASELINE.json configs[2..4]; Alg. 4):
  * every level's oracle statistics (iterations, recurrence / true relative residual, ||b||, errors vs the exact
    solution where one exists, ||W-U||, r_h) -- oracle.STAT_FIELDS;
  * the finest level's u_h and u~_h (Alg. 4 l.9 / l.10): max norm, RMS, three seeded random projections
    sum_i w_i u_i (w_i = 2 U_i - 1, synth.counter_uniform seeds 41..43), and the values at ~10^4 sampled nodes
    (seeded random nodes, every boundary face, 32 / 8-periodic tile seams of the GPU kernels, the corner at
    the origin).

The oracle runs in its threaded mode, which is bitwise the serial oracle (tests/test_oracle_threads.py).

Usage: python tests/golden/make_fullsize.py c3 c4 c5_256 [c5_512] [--threads T]
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import oracle as o  # noqa: E402
import synth  # noqa: E402

# name -> (problem, levels (coarsest 4^3), eps); BASELINE.json configs[2] (C3), [3] (C4), [4] (C5, SURVEY.md §8d D.4 (i):
# the same geometry to 256^3 / 512^3 instead of 1024^3)
CONFIGS = {
    "c3": (o.C3, 7, 1e-10),
    "c4": (o.C4, 8, 1e-9),
    "c5_256": (o.C5, 7, 1e-8),
    "c5_512": (o.C5, 8, 1e-8),
}
N_RANDOM = 6000
N_FACE = 300      # per face
N_SEAM = 1200
PROJ_SEEDS = (41, 42, 43)


def params_for(pid):
    return synth.c5_geometry(0) if pid == o.C5 else None


def sample_nodes(n: int) -> np.ndarray:
    """Linear node indices (x fastest) of the sampled nodes of an n^3-cell level, sorted and unique."""
    nn = n + 1
    u = synth.counter_uniform(37, 3 * (N_RANDOM + 6 * N_FACE + N_SEAM))
    k = 0

    def take(m):
        nonlocal k
        v = np.minimum((u[k:k + m] * nn).astype(np.int64), n)
        k += m
        return v

    ix, iy, iz = take(N_RANDOM), take(N_RANDOM), take(N_RANDOM)
    pts = [np.stack([ix, iy, iz], 1)]
    for F in range(6):   # boundary faces: both Dirichlet / Robin node planes and the plane next to them
        a, b = take(N_FACE), take(N_FACE)
        fixed = np.full(N_FACE, n if F & 1 else 0, dtype=np.int64)
        fixed[::2] += -1 if F & 1 else 1
        d = F // 2
        P = [a, b]
        P.insert(d, fixed)
        pts.append(np.stack(P, 1))
    # tile seams: x on multiples of 32 (+0 / +1), y on multiples of 8 (+0 / +1), z random
    sx = (take(N_SEAM) // 32) * 32 + (np.arange(N_SEAM) & 1)
    sy = (take(N_SEAM) // 8) * 8 + ((np.arange(N_SEAM) >> 1) & 1)
    sz = take(N_SEAM)
    pts.append(np.stack([np.minimum(sx, n), np.minimum(sy, n), sz], 1))
    c = np.arange(4)
    cz, cy, cx = np.meshgrid(c, c, c, indexing="ij")   # the corner at the origin (C4's singular point)
    pts.append(np.stack([cx.ravel(), cy.ravel(), cz.ravel()], 1))
    P = np.concatenate(pts)
    lin = P[:, 0] + nn * (P[:, 1] + nn * P[:, 2])
    return np.unique(lin)


def projections(v: np.ndarray) -> list:
    out = []
    for s in PROJ_SEEDS:
        w = 2.0 * synth.counter_uniform(s, v.size) - 1.0
        out.append(float(np.dot(w, v)))
        del w
    return out


def vec_summary(v: np.ndarray, idx: np.ndarray) -> dict:
    return {"inf": float(np.max(np.abs(v))), "rms": float(np.sqrt(np.dot(v, v) / v.size)),
            "proj": projections(v), "samples": v[idx].tolist()}


def run(name: str, threads: int) -> dict:
    pid, levels, eps = CONFIGS[name]
    prev = o.set_threads(threads)
    t0 = time.time()
    st, stats, u, ut = o.ecmg(4, levels, pid, eps, params=params_for(pid))
    wall = time.time() - t0
    o.set_threads(prev)
    if st != 0:
        raise RuntimeError(f"oracle ecmg {name}: status {st}")
    n = 4 << (levels - 1)
    idx = sample_nodes(n)
    per_level = [{f: (None if not np.isfinite(row[c]) else float(row[c])) for c, f in enumerate(o.STAT_FIELDS)}
                 for row in stats]
    return {
        "_source": "written by tests/golden/make_fullsize.py from oracle.ecmg only (threaded mode = bitwise the "
                   "serial oracle); Alg. 4, P:315-336",
        "config": name, "problem_id": pid, "coarsest": 4, "levels": levels, "n_fine": n, "eps": eps,
        "exp_variant": 0, "precond": 1,
        "oracle": {"threads": threads, "wall_s": wall, "host": platform.node(), "cpu": platform.processor()},
        "per_level": per_level,
        "sample_index": idx.tolist(),
        "u": vec_summary(u, idx),
        "ut": vec_summary(ut, idx),
        "proj_seeds": list(PROJ_SEEDS),
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="+", choices=sorted(CONFIGS))
    ap.add_argument("--threads", type=int, default=0)
    a = ap.parse_args()
    T = a.threads or o.max_threads()
    for name in a.configs:
        g = run(name, T)
        path = os.path.join(os.path.dirname(os.path.abspath(__file__)), f"fullsize_{name}.json")
        with open(path, "w") as f:
            json.dump(g, f, separators=(",", ":"))
        its = [int(r["iterations"]) for r in g["per_level"]]
        print(f"{name}: wall {g['oracle']['wall_s']:.1f} s, iterations {its}, {len(g['sample_index'])} samples -> {path}",
              flush=True)


if __name__ == "__main__":
    main()
