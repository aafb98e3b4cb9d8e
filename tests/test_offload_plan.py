"""ADMM-Offload planner (mlr_plan_offload / mlr_lru_baseline, offload_plan.cpp)
against the reference's own libmlr.so compiled into oracle/_ref (capi.cpp:344-380,
offload.cpp): byte-identical plan / CSV / LRU text and the same errors on toy,
paper-shaped, staggered (plans that lower the peak) and seeded random phase
traces. CPU only."""
import ctypes as C
import os

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_LIB = os.path.join(ROOT, "oracle", "_ref", "libmlr.so")


def _bind(lib):
    lib.mlr_plan_offload.restype = C.c_void_p
    lib.mlr_plan_offload.argtypes = [C.c_char_p, C.c_double, C.c_char_p]
    lib.mlr_lru_baseline.restype = C.c_void_p
    lib.mlr_lru_baseline.argtypes = [C.c_char_p, C.c_double, C.c_uint64]
    lib.mlr_last_error.restype = C.c_char_p
    lib.mlr_free.argtypes = [C.c_void_p]
    return lib


@pytest.fixture(scope="module")
def libs(mlrg):
    if not os.path.exists(REF_LIB):
        pytest.skip("oracle/_ref/libmlr.so not built (oracle/Makefile)")
    return _bind(mlrg.lib()), _bind(C.CDLL(REF_LIB))


def _call(lib, fn, *args):
    p = getattr(lib, fn)(*args)
    if not p:
        return None, lib.mlr_last_error().decode()
    s = C.cast(p, C.c_char_p).value.decode()
    lib.mlr_free(p)
    return s, None


# the paper's four ADMM phases: psi / psi_prev / lambda idle
# through most of LSP; u and g are touched everywhere (not eligible)
PAPER = """
phase LSP 120.0
phase RSP 18.5
phase lambda 6.25
phase penalty 1.5   # comment
var u 5.4e8 0
var g 1.6e9 0
var psi 1.6e9 1
var psi_prev 1.6e9 1
var lambda 1.6e9 1
access u LSP 0 120
access u RSP 0 18.5
access u lambda 0 6.25
access g LSP 0 2.0
access psi LSP 0 1.0
access psi RSP 1.0 17.0
access psi lambda 0.5 6.0
access psi penalty 0 1.5
access psi_prev RSP 0.2 0.4
access psi_prev penalty 0 1.0
access lambda LSP 0.5 1.5
access lambda RSP 2.0 16.0
access lambda lambda 0 6.25
"""

TOY = """
phase A 100
phase B 200
var x 3.2e8 1
var y 6.4e8 1
var z 1e8 0
access x A 10 40
access x B 150 160
access y A 0 5
access z A 0 100
access z B 0 200
"""


# every variable idles through the other phases: staggered offloads lower the peak
STAGGER = """
phase A 80
phase B 60
phase C 40
var x 4e8 1
var y 3e8 1
var z 2e8 1
var w 1e8 0
access x A 5 20
access y B 10 50
access z C 0 5
access w A 0 80
access w B 0 60
access w C 0 40
"""


def _staggered_trace(seed):
    rng = np.random.default_rng(1000 + seed)
    nph = int(rng.integers(2, 5))
    durs = rng.uniform(20, 150, size=nph)
    lines = [f"phase p{i} {d:.3f}" for i, d in enumerate(durs)]
    acc = []
    for v in range(int(rng.integers(2, 5))):
        lines.append(f"var v{v} {rng.uniform(1e7, 4e8):.6g} {int(rng.random() < 0.85)}")
        for p in rng.choice(nph, size=int(rng.integers(1, 3)), replace=False) if nph > 1 else [0]:
            a, b = sorted(rng.uniform(0, durs[p], size=2))
            acc.append(f"access v{v} p{p} {a:.4f} {b:.4f}")
    return "\n".join(lines + acc) + "\n"


def _random_trace(seed):
    rng = np.random.default_rng(seed)
    nph = int(rng.integers(2, 5))
    lines = [f"phase p{i} {rng.uniform(5, 200):.3f}" for i in range(nph)]
    durs = [float(l.split()[2]) for l in lines]
    nv = int(rng.integers(2, 5))
    acc = []
    for v in range(nv):
        lines.append(f"var v{v} {rng.uniform(1e7, 2e9):.6g} {int(rng.random() < 0.75)}")
        for p in rng.choice(nph, size=int(rng.integers(1, min(nph, 3) + 1)), replace=False):
            a, b = sorted(rng.uniform(0, durs[p], size=2))
            acc.append(f"access v{v} p{p} {a:.4f} {b:.4f}")
    return "\n".join(lines + acc) + "\n"


TRACES = [PAPER, TOY, STAGGER] + [_random_trace(s) for s in range(8)] + [_staggered_trace(s) for s in range(12)]


@pytest.mark.parametrize("i", range(len(TRACES)))
@pytest.mark.parametrize("bw,fmt", [(0.0, b"plan"), (0.0, b"csv"), (5.0e7, b"plan"), (2.0e7, b"csv")])
def test_plan_text_matches_reference(libs, i, bw, fmt):
    ours, ref = libs
    t = TRACES[i].encode()
    assert _call(ours, "mlr_plan_offload", t, bw, fmt) == _call(ref, "mlr_plan_offload", t, bw, fmt)


@pytest.mark.parametrize("i", range(len(TRACES)))
@pytest.mark.parametrize("budget_frac", [0.3, 0.6, 0.9, 1.5])
def test_lru_text_matches_reference(libs, i, budget_frac):
    ours, ref = libs
    t = TRACES[i].encode()
    total = sum(float(l.split()[2]) for l in TRACES[i].splitlines() if l.startswith("var"))
    budget = int(total * budget_frac)
    for bw in (0.0, 2.0e7):
        assert _call(ours, "mlr_lru_baseline", t, bw, budget) == _call(ref, "mlr_lru_baseline", t, bw, budget)


BAD = [
    "", "phase A\n", "phase A 0\nvar x 10 1\n", "phase A 1\nphase A 2\n", "phase A 1\nvar x 10 2\n",
    "phase A 1\nvar x -1 1\n", "phase A 1\nvar x 10 1\nvar x 5 0\n", "phase A 1\nvar x 10 1\naccess y A 0 1\n",
    "phase A 1\nvar x 10 1\naccess x B 0 1\n", "phase A 1\nvar x 10 1\naccess x A 0 2\n",
    "phase A 1\nvar x 10 1\naccess x A 0.5 0.2\n", "phase A 1\nvar x 10 1\naccess x A 0 1\naccess x A 0 1\n",
    "phase A 1 extra\n", "bogus 1 2\n", "phase A 1\nvar x 10 1.5\n",
]


@pytest.mark.parametrize("text", BAD)
def test_malformed_traces_fail_like_reference(libs, text):
    ours, ref = libs
    t = text.encode()
    a, b = _call(ours, "mlr_plan_offload", t, 0.0, b"plan"), _call(ref, "mlr_plan_offload", t, 0.0, b"plan")
    assert a[0] is None and a == b  # same message (offload.cpp:45-118)
    a, b = _call(ours, "mlr_lru_baseline", t, 0.0, 100), _call(ref, "mlr_lru_baseline", t, 0.0, 100)
    assert a[0] is None and a == b


def test_bad_format_and_null(libs):
    ours, ref = libs
    for lib in (ours, ref):
        assert _call(lib, "mlr_plan_offload", TOY.encode(), 0.0, b"json")[0] is None
    assert _call(ours, "mlr_plan_offload", TOY.encode(), 0.0, b"json")[1] == \
        _call(ref, "mlr_plan_offload", TOY.encode(), 0.0, b"json")[1]
    assert _call(ours, "mlr_plan_offload", None, 0.0, None)[0] is None
