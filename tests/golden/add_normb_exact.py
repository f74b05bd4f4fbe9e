"""Add the correctly rounded ||b|| of every level to the full-size goldens (tests/golden/fullsize_<cfg>.json) --
calls ONLY oracle/ (and synth/ for C5's geometry). The oracle's own ||b|| (Alg. 4's stopping-test norm)
is a serial recursive sum of b_i^2 in node order; at 512^3 that sum is off by 4.7e-10 relative (C4,
tests/diag_c4_rhs.py: the oracle's b and the GPU's b agree to ||db||_2 = 8e-16, their math.fsum norms agree to
1 ulp). The golden test compares the GPU's ||b|| with normb_exact = sqrt(fsum(b_i^2)) of the oracle's b.

Usage: python tests/golden/add_normb_exact.py c3 c4 c5_256 c5_512 [--threads T]"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import oracle as o  # noqa: E402
import synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("cfgs", nargs="+")
    ap.add_argument("--threads", type=int, default=0)
    a = ap.parse_args()
    o.set_threads(a.threads or o.max_threads())
    for cfg in a.cfgs:
        path = os.path.join(os.path.dirname(os.path.abspath(__file__)), f"fullsize_{cfg}.json")
        with open(path) as f:
            G = json.load(f)
        pid = G["problem_id"]
        params = synth.c5_geometry(0) if pid == o.C5 else None
        for k, row in enumerate(G["per_level"]):
            n = G["coarsest"] * 2 ** k if isinstance(G["coarsest"], int) else None
            L = o.Level((n, n, n), pid, params=params)
            b, nb = L.rhs()
            m, _ = L.dirichlet()
            bf = b[~m]
            row["normb_exact"] = math.sqrt(math.fsum((bf * bf).tolist()))
            print(f"{cfg} level {k} n={n}: serial {nb!r} exact {row['normb_exact']!r} "
                  f"rel {abs(nb - row['normb_exact']) / max(row['normb_exact'], 1e-300):.2e}", flush=True)
            del L, b, bf, m
        with open(path, "w") as f:
            json.dump(G, f)


if __name__ == "__main__":
    main()
