"""Where the end-to-end (drop-in mlr_reconstruct on host arrays) time goes at
256^3: reconstruct with n_outer = 1, 2, 4, 8 (slope = per iteration,
intercept = setup + host<->device transfers)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2511_01893_b200 as m  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
cfg = m.Config(n1=n, n0=n, n2=n, n_theta=n, h=n, w=n, n_outer=1, memoization="off", nudft_path="gridding")
ph = m.make_phantom("blocks", n, n, n, 1)
data = m.project(cfg, ph)
m.reconstruct(cfg, data, ph)  # warm-up: module loading
PHASES = ("host:e2e_total", "host:e2e_teardown_and_rest", "host:e2e_solver_teardown", "host:e2e_engine_teardown", "host:usfft_fu1d_plan", "host:usfft_fu2d_dimplans", "host:usfft_fu2d_plans", "host:usfft_class_sort", "host:usfft_class_group", "host:usfft_class_tables", "host:usfft_class_uploads", "host:usfft_classes", "host:usfft_patches", "host:e2e_engine", "host:usfft_tables", "host:e2e_upload", "host:e2e_solver_setup", "host:e2e_iterations",
          "host:e2e_download")
for k in (1, 2, 4, 8):
    m.lib().mlrg_prof_reset()
    m.lib().mlrg_prof_enable(1)
    cfg.set("n_outer", k)
    t0 = time.perf_counter()
    res = m.reconstruct(cfg, data, ph)
    t1 = time.perf_counter()
    vol = res.volume.numpy()
    t2 = time.perf_counter()
    m.lib().mlrg_prof_enable(0)
    ph_ms = " ".join(f"{p[5:]}={m.prof_query(p)[0]:.0f}" for p in PHASES)
    print(f"n_outer={k}: reconstruct {t1 - t0:.3f} s, volume to numpy {t2 - t1:.3f} s | ms: {ph_ms}")
