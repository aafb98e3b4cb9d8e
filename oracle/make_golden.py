"""Regenerates tests/golden/*.npz from the unmodified CPU reference.

TEST INFRASTRUCTURE ONLY. Runs oracle/_ref/golden_gen (built by
`make -C oracle` from /root/reference/proj/src) and packs each case into one
compressed .npz plus its text side files. Needs /root/reference, so it runs
in the build container, never on the GPU box; the fixtures are committed.

    python oracle/make_golden.py [case ...]      # default: every case
"""
from __future__ import annotations

import os
import subprocess
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
GEN = os.path.join(HERE, "_ref", "golden_gen")
OUT = os.path.join(os.path.dirname(HERE), "tests", "golden")

# name -> golden_gen argv tail
CASES = {
    # per-operator fixtures: cubic power-of-two and a ragged non-power-of-two geometry
    "ops_c16": ["ops", "16", "16", "16", "16", "16", "16", "11"],
    "ops_ragged": ["ops", "20", "24", "18", "10", "12", "14", "12"],
    "ops_c32": ["ops", "32", "32", "32", "24", "32", "32", "13"],
    "encoder": ["encoder"],
    "cnn": ["cnn"],
    "store": ["store"],
    # reconstructions (phantom "blocks" seed 1, d = forward_L(phantom))
    "recon_c16_memo_grid": ["recon", "16", "16", "10", "local", "gridding"],
    "recon_c32_memo_grid": ["recon", "32", "32", "10", "local", "gridding"],
    "recon_c32_off_grid": ["recon", "32", "32", "10", "off", "gridding"],
    "recon_c64_off_grid": ["recon", "64", "64", "10", "off", "gridding", "8"],
    # the CNN key encoder (encoder_variant = cnn, seeded initial weights)
    "recon_c16_cnn_memo_grid": ["recon", "16", "16", "10", "local", "gridding", "1", "cnn"],
    "recon_c32_cnn_memo_grid": ["recon", "32", "32", "10", "local", "gridding", "8", "cnn"],
    # pipeline = baseline (admm.cpp:122-138): 6 memoizable operators per inner step,
    # memoized f2d / f2d_adj included
    "recon_c16_baseline_memo_grid": ["recon", "16", "16", "6", "local", "gridding", "1", "projection", "baseline"],
    "recon_c32_baseline_off_grid": ["recon", "32", "32", "6", "off", "gridding", "8", "projection", "baseline"],
    # BASELINE configs[0] exactly as-is: 64^3, 64 angles, 10 iterations, memo on,
    # default (direct) NUDFT path, 1 worker. ~5 minutes of CPU.
    "recon_cfg1_memo_direct": ["recon", "64", "64", "10", "local", "direct", "1"],
    # BASELINE configs[1] (256^3, 256 angles) as compact fixtures (golden_gen recon_big:
    # report, audit, counters, ||u|| and u at 2^18 seeded voxel indices; the tests
    # regenerate d with `golden_gen data` on the box). Memo off: a 3-iteration prefix
    # (~6 min on 8 cores); memo on: 10 iterations, which publishes > 1024 keys so the
    # store trains its nlist-64 IVF index mid-run (~20 GB of host RAM).
    "recon_c256_off_grid": ["recon_big", "256", "256", "3", "off", "8", "0", "262144"],
    "recon_c256_memo_grid": ["recon_big", "256", "256", "10", "local", "8", "0", "262144"],
    # configs[2] (512^3, 512 angles) CPU prefix of 2 iterations, memo off, on seeded
    # random data (the reference's dense projector is O(N^4) at this size).
    "recon_c512_off_rand": ["recon_big", "512", "512", "2", "off", "8", "1", "262144"],
}

TEXT_SUFFIXES = (".txt", ".csv")


def run_case(name: str) -> None:
    args = CASES[name]
    with tempfile.TemporaryDirectory() as tmp:
        subprocess.run([GEN, args[0], tmp, *args[1:]], check=True)
        arrays = {}
        for fn in sorted(os.listdir(tmp)):
            path = os.path.join(tmp, fn)
            if fn.endswith(".npy"):
                arrays[fn[:-4]] = np.load(path)
            elif fn.endswith(TEXT_SUFFIXES):
                with open(path) as f:
                    arrays["txt_" + fn.replace(".", "_")] = np.array(f.read())
        np.savez_compressed(os.path.join(OUT, name + ".npz"), **arrays)
    print(f"{name}: {len(arrays)} entries", flush=True)


def main(argv: list[str]) -> int:
    if not os.path.exists(GEN):
        subprocess.run(["make", "-C", HERE, "-j8"], check=True)
    os.makedirs(OUT, exist_ok=True)
    for name in argv or list(CASES):
        run_case(name)
    return 0


if __name__ == "__main__":
    sys.exit(main(sys.argv[1:]))
