"""Parity at scale against the C oracle (bit-identical to the reference on
every golden vector): 2^20 Bessel elements of the configs[1] distribution
(all of them) and the full ba20-shaped Jacobian (all 678,718 observations,
the bench's synthetic problem).  Writes profiles/r01/parity_at_scale.json."""
import json
import os
import sys
import time

import numpy as np
import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "oracle"))
import oracle as O  # noqa: E402

import bench  # noqa: E402
import paper_2003_04617_b200 as rg  # noqa: E402

out = {}
rng = np.random.default_rng(11)
z = rng.uniform(0.1, 10.0, 1 << 20)
t0 = time.perf_counter()
Jo, dzo, fo, trips = O.besselj_grad(2, z)
t_or = time.perf_counter() - t0
r = rg.besselj_grad(torch.as_tensor(z, device="cuda"), 2)
torch.cuda.synchronize()
J, dz, f = r.J.cpu().numpy(), r.dJdz.cpu().numpy(), r.fail.cpu().numpy()
ok = fo == 0
scale = np.abs(Jo[ok]) + 1e-300
out["bessel"] = {
    "elements": int(z.size), "fail_codes_equal": bool(np.array_equal(f, fo)),
    "sum_trips_equal": int(r.sum_trips) == int(trips),
    "J_bit_exact_frac": float(np.mean(J[ok] == Jo[ok])),
    "dJdz_bit_exact_frac": float(np.mean(dz[ok] == dzo[ok])),
    "J_max_abs_err": float(np.max(np.abs(J[ok] - Jo[ok]))),
    "dJdz_max_abs_err": float(np.max(np.abs(dz[ok] - dzo[ok]))),
    "J_max_rel_err_where_|J|>1e-3": float(np.max((np.abs(J[ok] - Jo[ok]) / scale)[np.abs(Jo[ok]) > 1e-3])),
    "oracle_seconds": round(t_or, 2)}
cams, X, w, feats, obs = bench.ba_synthetic(bench.BA_N, bench.BA_M, bench.BA_P)
t0 = time.perf_counter()
Jb_o, err_o, fb_o = O.ba_jac(cams, X, w, feats, obs)
t_or = time.perf_counter() - t0
t = lambda a: torch.as_tensor(a, device="cuda")  # noqa: E731
b = rg.ba_jacobian(t(cams), t(X), t(w), t(feats), t(obs))
torch.cuda.synchronize()
Jb = b.J.cpu().numpy()
rowmax = np.abs(Jb_o).max(1, keepdims=True)
out["ba"] = {
    "observations": int(w.size), "fail_codes_equal": bool(np.array_equal(b.fail.cpu().numpy(), fb_o)),
    "entries_bit_exact_frac": float(np.mean(Jb == Jb_o)),
    "zero_entries_exactly_zero": bool(np.all(Jb[Jb_o == 0] == 0)),
    "max_err_over_row_max": float(np.max(np.abs(Jb - Jb_o) / np.maximum(rowmax, 1e-300))),
    "oracle_seconds": round(t_or, 2)}
json.dump(out, open(os.path.join(REPO, "profiles", "r01", "parity_at_scale.json"), "w"), indent=1)
print(json.dumps(out, indent=1))
