"""The four-step column passes of fu2d / fu2d_adj (k_cols4_pass1/2, used from
M = 1024 by default, usfft.cu) against the one-pass column kernels and the
reference. The switch (MLRG_COLS4) is read once per process, so the other
setting runs in a child process."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)

# fu2d and fu2d_adj of seeded inputs at M1 = M2 = 1024 (n = 512), saved to argv[1]
_CHILD = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[2])
import paper_2511_01893_b200 as m
n, h, nt = 512, 20, 48
ctx = m.Context(n, n, n, nt, h, n)
rng = np.random.default_rng(5)
v = (rng.standard_normal((n, h, n)) + 1j * rng.standard_normal((n, h, n))).astype(np.complex64)
p = (rng.standard_normal((nt, h, n)) + 1j * rng.standard_normal((nt, h, n))).astype(np.complex64)
a = ctx.fu2d(torch.from_numpy(v).cuda(), torch.empty((nt, h, n), dtype=torch.complex64, device="cuda"))
b = ctx.fu2d_adj(torch.from_numpy(p).cuda(), torch.empty((n, h, n), dtype=torch.complex64, device="cuda"))
ctx.sync()
np.savez(sys.argv[1], v=v, p=p, a=a.cpu().numpy(), b=b.cpu().numpy())
"""


def _run(out, cols4):
    env = dict(os.environ, MLRG_COLS4=cols4)
    r = subprocess.run([sys.executable, "-c", _CHILD, str(out), ROOT], env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    return np.load(out)


def test_four_step_matches_one_pass_columns_at_m1024(tmp_path):
    four = _run(tmp_path / "four.npz", "auto")  # default: four-step from M = 1024
    one = _run(tmp_path / "one.npz", "0")
    rel = lambda x, y: np.linalg.norm(x - y) / np.linalg.norm(y)
    # both compute the same double-precision FFT; they differ by the rounding of
    # one more complex64 intermediate grid
    assert rel(four["a"], one["a"]) < 1e-6
    assert rel(four["b"], one["b"]) < 1e-6
    # <fu2d v, p> == <v, fu2d_adj p> on the four-step path
    a, b, v, p = (four[k].astype(np.complex128) for k in ("a", "b", "v", "p"))
    assert abs(np.vdot(p, a) - np.vdot(b, v)) / (np.linalg.norm(a) * np.linalg.norm(p)) < 1e-5


def test_four_step_forced_small_passes_reference_parity():
    """MLRG_COLS4=1 runs the four-step passes from M = 64: the operator golden
    cases, the restatement/adjointness cases and the memo-on reconstructions
    must still match the reference."""
    env = dict(os.environ, MLRG_COLS4="1")
    r = subprocess.run(
        [sys.executable, "-m", "pytest", "-x", "-q", "-m", "gpu", "-p", "no:cacheprovider",
         os.path.join(HERE, "test_gpu_ops.py"), os.path.join(HERE, "test_gpu_recon.py"),
         "-k", "usfft_ops or restatement or f2d_forward or device_reconstruction"],
        cwd=ROOT, env=env, capture_output=True, text=True, timeout=1500)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert " passed" in r.stdout and " 0 selected" not in r.stdout
