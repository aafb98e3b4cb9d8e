"""Per-iteration CSV of a device reconstruction of the c64 golden case (n, n_outer from argv),
with the reference volume for the accuracy column:  python scripts/trace_recon.py 64 10
"""
import os, sys
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import paper_2511_01893_b200 as m
n = int(sys.argv[1]); k = int(sys.argv[2])
z = np.load(os.path.join(ROOT, "tests/golden/recon_c64_off_grid.npz"))
ph = torch.from_numpy(m.make_phantom("blocks", n, n, n, 1).numpy().astype(np.complex64)).cuda()
d = torch.from_numpy(z["data"]).cuda()
u = torch.empty((n, n, n), dtype=torch.complex64, device="cuda")
r = m.reconstruct_device(f"n1={n}\nn0={n}\nn2={n}\nn_theta={n}\nh={n}\nw={n}\nn_outer={k}\n", d, u, reference=ph)
print(r.csv)
