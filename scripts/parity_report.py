"""rel-L2(u) of the device solve against every golden reconstruction (and the
audit match), for A/B experiments with numerics switches set in the env."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2511_01893_b200 as m  # noqa: E402

for case, memo in [("recon_c16_memo_grid", "local"), ("recon_c32_memo_grid", "local"), ("recon_c32_off_grid", "off"),
                   ("recon_c64_off_grid", "off"), ("recon_cfg1_memo_direct", "local")]:
    z = np.load(os.path.join(ROOT, "tests", "golden", case + ".npz"))
    n, nt = z["phantom"].shape[0], z["data"].shape[0]
    cfg = f"n1={n}\nn0={n}\nn2={n}\nn_theta={nt}\nh={n}\nw={n}\nn_outer=10\nmemoization={memo}\nnudft_path=gridding\n"
    u = torch.empty((n, n, n), dtype=torch.complex64, device="cuda")
    r = m.reconstruct_device(cfg, torch.from_numpy(z["data"]).cuda(), u, reference=torch.from_numpy(z["phantom"]).cuda())
    err = np.linalg.norm(u.cpu().numpy() - z["u"]) / np.linalg.norm(z["u"])
    audit = "" if memo == "off" else f" audit={'ok' if np.array_equal(r.audit()[0], z['audit_int']) else 'DIFF'}"
    print(f"{case:28s} rel-L2(u) {err:.3e}{audit}")
