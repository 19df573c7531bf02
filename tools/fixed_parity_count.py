"""Parity count of the Fixed (Q31.32) codegen path against codegen_fixed.npz (GPU tool)."""
import sys, numpy as np
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import paper_2003_04617_b200 as rg
from test_codegen_fixed_gpu import src, case_args, f64, call
g = dict(np.load("tests/golden/codegen_fixed.npz"))
d = {"run_acc": [], "g_b": [], "y": [], "fd": []}
for r in range(len(g["k"])):
    out, err = call(lambda: rg.run(src(), "fxmix", case_args(g, r)))
    if not err:
        d["run_acc"].append(out[0].raw - g["run"][r][0]); d["y"].append(out[1] - f64(g["run"][r][1]))
    for tag, seeds in (("gacc", None), ("gy", [("y!", (), 1.0)])):
        res, err = call(lambda: rg.gradient(src(), rg.GradRequest("fxmix", case_args(g, r), seeds=seeds)))
        if not err:
            d["g_b"].append(res[1]["b"].raw - g[tag][r][5])
    fd, err = call(lambda: rg.finite_difference(src(), "fxmix", case_args(g, r), 1e-6))
    if not err:
        d["fd"].append(max(abs(a - b) for a, b in zip((fd["acc!"], fd["y!"], fd["b"]), g["fd"][r])))
for k, v in d.items():
    v = np.array(v, dtype=float)
    print(k, len(v), "exact", int((v == 0).sum()), "maxabs", float(np.abs(v).max()))
