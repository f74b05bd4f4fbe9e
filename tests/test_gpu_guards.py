"""Out-of-bounds write check of every kernel family (compute-sanitizer is closed on this GPU pool,
profiles/r02/compute_sanitizer_refused.log): tools/sanitize_run.py --guards runs the one-CTA, cooperative,
cooperative-TMA, TMA graph-loop / host-loop, register-prefetch, EXP (fused / two-pass, both variants), EXP_true,
setup, virtual-slab (copied and fused peer halos) and ARRAYS paths at 16^3 - 64^3 against libecmg_test.so, whose
device buffers all carry 8 KB guard bands of a byte pattern, with the caller's vectors inside sentinel-filled
tensors; every guard must be intact after every call and after every destroy, and 5 repeated runs of every
configuration must reproduce u_h and u~_h bit for bit (the race check that stands in for racecheck)."""
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a GPU")
def test_guard_bands_intact():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize_run.py"), "--guards"],
                       capture_output=True, text=True, timeout=900, cwd=ROOT)
    print(r.stdout[-4000:], r.stderr[-2000:])
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert r.stdout.strip().splitlines()[-1].endswith(" 0")
