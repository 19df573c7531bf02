"""Golden-vector generator: runs the REFERENCE revlang interpreter.

Test infrastructure only (never imported by the product package).  It
imports the read-only reference package in place from
/root/reference/pkg/src, executes `revlang.gradient` (autodiff.py:136-180)
over the three benchmark programs shipped in
paper_2003_04617_b200/programs/*.rnl, and writes seeded inputs plus the
reference outputs to tests/golden/*.npz.  Those fixtures pin both the C
oracle (oracle/revoracle.c) and the CUDA kernels; the GPU box has no
/root/reference, so only the .npz files travel.

    PYTHONDONTWRITEBYTECODE=1 python oracle/gen_golden.py [bessel|ba|gmm ...]
"""

import math
import os
import sys
import time

import numpy as np

REF_SRC = "/root/reference/pkg/src"
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROG_DIR = os.path.join(REPO, "paper_2003_04617_b200", "programs")
OUT_DIR = os.path.join(REPO, "tests", "golden")

sys.dont_write_bytecode = True
sys.path.insert(0, REF_SRC)
from revlang import ExecOptions, GradRequest, gradient, parse_program, run, uncall  # noqa: E402
from revlang.errors import RevLangError  # noqa: E402
from revlang.values import Array, deep_copy  # noqa: E402


def _prog(name):
    with open(os.path.join(PROG_DIR, name)) as fh:
        return parse_program(fh.read(), name)


def _err_name(fn):
    try:
        return fn(), ""
    except RevLangError as err:
        return None, type(err).__name__


# --------------------------------------------------------------------------
# Bessel J_nu: C1 (1,000 z ~ U(0.1, 10), seed 0, nu = 2) plus other orders,
# edge arguments and the domain errors of z <= 0.
# --------------------------------------------------------------------------

def gen_bessel():
    p = _prog("besselj.rnl")
    cases = []
    z_c1 = np.random.default_rng(0).uniform(0.1, 10.0, 1000)
    cases += [(2, float(z)) for z in z_c1]
    rng = np.random.default_rng(10)
    for nu in (0, 1, 3, 5):
        cases += [(nu, float(z)) for z in rng.uniform(0.05, 12.0, 64)]
    edge = [1e-300, 1e-12, 1e-3, 0.1, 1.0, 2.404825557695773, 5.135622301840683,
            10.0, 15.0, 20.0, 30.0, 0.0, -1.0, -1e-300]
    for nu in (0, 2, 7):
        cases += [(nu, z) for z in edge]
    nus = np.array([c[0] for c in cases], np.int32)
    zs = np.array([c[1] for c in cases], np.float64)
    J = np.full(len(cases), np.nan)
    dz = np.full(len(cases), np.nan)
    errs = []
    t0 = time.perf_counter()
    for i, (nu, z) in enumerate(cases):
        res, en = _err_name(lambda: gradient(p, GradRequest("besselj", [0.0, nu, z])))
        if res is not None:
            primal, g = res
            J[i], dz[i] = primal[0], g["z"]
        errs.append(en)
    dt = time.perf_counter() - t0
    np.savez_compressed(os.path.join(OUT_DIR, "bessel.npz"), nu=nus, z=zs, J=J,
                        dJdz=dz, err=np.array(errs), thr=1e-16, tol=1e-9)
    print(f"bessel: {len(cases)} cases in {dt:.1f}s, errors={sum(1 for e in errs if e)}")


# --------------------------------------------------------------------------
# Bundle adjustment: per-observation 2 x 15 Jacobian block and the weight
# derivative, two seeded gradient passes per observation.
# --------------------------------------------------------------------------

def ba_inputs(rng, n_obs):
    cams = np.empty((n_obs, 11))
    cams[:, 0:3] = rng.normal(0.0, 0.3, (n_obs, 3))
    cams[:, 3:6] = rng.normal(0.0, 1.0, (n_obs, 3))
    cams[:, 6] = rng.uniform(500.0, 600.0, n_obs)
    cams[:, 7:9] = rng.uniform(0.0, 1.0, (n_obs, 2))
    cams[:, 9:11] = rng.normal(0.0, 0.01, (n_obs, 2))
    X = rng.normal(0.0, 1.0, (n_obs, 3))
    X[:, 2] += 10.0
    w = rng.uniform(0.0, 1.0, n_obs)
    feat = rng.uniform(0.0, 100.0, (n_obs, 2))
    return cams, X, w, feat


def gen_ba():
    p = _prog("ba.rnl")
    n_obs = 48
    cams, X, w, feat = ba_inputs(np.random.default_rng(3), n_obs)
    cams[5, 0:3] = 0.0          # zero rotation: the else branch (no rodrigues)
    cams[17, 0:3] = [0.0, 0.0, 1e-3]
    J = np.full((n_obs, 2, 15), np.nan)
    e = np.full((n_obs, 2), np.nan)
    wj = np.full(n_obs, np.nan)
    errs = []
    opts = ExecOptions()
    t0 = time.perf_counter()
    for o in range(n_obs):
        args = [0.0, 0.0, Array.vector(cams[o].tolist()), Array.vector(X[o].tolist()),
                float(w[o]), float(feat[o, 0]), float(feat[o, 1])]
        en = ""
        for r, seed in enumerate(("e1!", "e2!")):
            res, en = _err_name(lambda: gradient(p, GradRequest(
                "ba_proj", args, seeds=[(seed, (), 1.0)], wrt=["cam", "X", "w"]), opts))
            if res is None:
                break
            primal, g = res
            e[o] = primal[0], primal[1]
            J[o, r] = g["cam"].data + g["X"].data + [g["w"]]
        res, en2 = _err_name(lambda: gradient(p, GradRequest("ba_weight", [0.0, float(w[o])]), opts))
        if res is not None:
            wj[o] = res[1]["w"]
        errs.append(en or en2)
    dt = time.perf_counter() - t0
    np.savez_compressed(os.path.join(OUT_DIR, "ba.npz"), cams=cams, X=X, w=w, feat=feat,
                        J=J, e=e, wjac=wj, err=np.array(errs))
    print(f"ba: {n_obs} observations in {dt:.1f}s")


# --------------------------------------------------------------------------
# GMM: small (d, K, N) cases through the full reversible objective.
# --------------------------------------------------------------------------

def gmm_constants(d, K, N, gamma, m):
    n = d + m + 1
    lgd = 0.25 * d * (d - 1) * math.log(math.pi) + sum(
        math.lgamma(0.5 * n + 0.5 * (1 - j)) for j in range(1, d + 1))
    C = n * d * (math.log(gamma) - 0.5 * math.log(2.0)) - lgd
    return -N * d * 0.5 * math.log(2.0 * math.pi) - K * C


def gmm_inputs(rng, d, K, N):
    alphas = rng.normal(0.0, 1.0, K)
    means = rng.uniform(0.0, 1.0, (K, d))
    icf = rng.normal(0.0, 1.0, (K, d * (d + 1) // 2)) * 0.5
    x = rng.uniform(0.0, 1.0, (N, d))
    return alphas, means, icf, x


def gen_gmm():
    p = _prog("gmm.rnl")
    out = {}
    cases = [(3, 2, 4, 1.0, 0), (5, 4, 20, 1.0, 0), (8, 5, 10, 1.3, 2),
             (4, 3, 64, 1.0, 0), (16, 6, 6, 0.7, 1), (2, 1, 5, 1.0, 0), (4, 3, 23, 1.0, 0),
             (6, 8, 40, 1.0, 0)]
    t0 = time.perf_counter()
    for ci, (d, K, N, gamma, m) in enumerate(cases):
        alphas, means, icf, x = gmm_inputs(np.random.default_rng(100 + ci), d, K, N)
        cst = gmm_constants(d, K, N, gamma, m)
        A = lambda a: Array.matrix(a.tolist()) if a.ndim == 2 else Array.vector(a.tolist())
        Z = lambda *s: A(np.zeros(s))
        ZI = lambda n: Array.vector([0] * n)   # Int scratch (argmax record)
        args = [0.0, A(alphas), A(means), A(icf), A(x), Z(K, d), Z(K), Z(d), Z(d), Z(K), ZI(K),
                float(gamma), int(m), float(cst)]
        res, en = _err_name(lambda: gradient(p, GradRequest(
            "gmm", args, wrt=["alphas", "means", "icf"])))
        assert res is not None, en
        primal, g = res
        pre = f"c{ci}_"
        out.update({pre + "dims": np.array([d, K, N, m]), pre + "gamma": gamma, pre + "cst": cst,
                    pre + "alphas": alphas, pre + "means": means, pre + "icf": icf, pre + "x": x,
                    pre + "err": primal[0],
                    pre + "g_alphas": np.array(g["alphas"].data),
                    pre + "g_means": np.array(g["means"].data).reshape(K, d),
                    pre + "g_icf": np.array(g["icf"].data).reshape(K, -1)})
    out["ncases"] = len(cases)
    np.savez_compressed(os.path.join(OUT_DIR, "gmm.npz"), **out)
    print(f"gmm: {len(cases)} cases in {time.perf_counter() - t0:.1f}s")


# --------------------------------------------------------------------------
# run / uncall (reference interpreter.py:1021-1028) with non-zero outputs
# --------------------------------------------------------------------------

def gen_run():
    pb = _prog("besselj.rnl")
    rng = np.random.default_rng(20)
    z = rng.uniform(0.1, 10.0, 200)
    out0 = rng.normal(0.0, 1.0, 200)
    r_run, r_unc, errs = np.full(200, np.nan), np.full(200, np.nan), []
    z[7], z[8] = -2.0, 25.0              # RevDomainError, DirtyAncilla
    for i in range(200):
        a, en = _err_name(lambda: run(pb, "besselj", [float(out0[i]), 2, float(z[i])]))
        b, en2 = _err_name(lambda: uncall(pb, "besselj", [float(out0[i]), 2, float(z[i])]))
        if a is not None:
            r_run[i] = a[0]
        if b is not None:
            r_unc[i] = b[0]
        errs.append(en or en2)
    pa = _prog("ba.rnl")
    cams, X, w, feat = ba_inputs(np.random.default_rng(21), 16)
    e_in = np.random.default_rng(22).normal(0.0, 1.0, (16, 2))
    ba_run = np.full((16, 2), np.nan)
    ba_unc = np.full((16, 2), np.nan)
    for o in range(16):
        args = [float(e_in[o, 0]), float(e_in[o, 1]), Array.vector(cams[o].tolist()),
                Array.vector(X[o].tolist()), float(w[o]), float(feat[o, 0]), float(feat[o, 1])]
        a = run(pa, "ba_proj", args)
        b = uncall(pa, "ba_proj", args)
        ba_run[o], ba_unc[o] = a[:2], b[:2]
    np.savez_compressed(os.path.join(OUT_DIR, "run.npz"), bj_z=z, bj_out0=out0, bj_run=r_run,
                        bj_uncall=r_unc, bj_err=np.array(errs), ba_cams=cams, ba_X=X, ba_w=w,
                        ba_feat=feat, ba_e_in=e_in, ba_run=ba_run, ba_uncall=ba_unc)
    print("run/uncall goldens written")


def gen_hess():
    """reference autodiff.hessian (forward-over-reverse over Duals) of besselj:
    configs[0]'s 1,000 z (seed 0) at nu = 2, 40 z at nu = 0, 1, 5, and error
    cases; the full matrix over the Float leaves (out!, z)."""
    from revlang.autodiff import hessian
    pb = _prog("besselj.rnl")
    rng = np.random.default_rng(0)
    zs = [rng.uniform(0.1, 10.0, 1000)]
    nus = [np.full(1000, 2)]
    r2 = np.random.default_rng(31)
    for nu in (0, 1, 5):
        zs.append(np.concatenate([r2.uniform(0.1, 10.0, 37), [1e-3, 25.0, -1.0]]))
        nus.append(np.full(40, nu))
    z, nu = np.concatenate(zs), np.concatenate(nus)
    H = np.full((z.size, 2, 2), np.nan)
    errs = []
    t0 = time.time()
    for i in range(z.size):
        r, en = _err_name(lambda: hessian(pb, "besselj", [0.0, int(nu[i]), float(z[i])]))
        if r is not None:
            H[i] = r.matrix
        errs.append(en)
    np.savez_compressed(os.path.join(OUT_DIR, "hess.npz"), z=z, nu=nu, H=H, err=np.array(errs))
    print(f"hessian goldens written ({z.size} cases, {time.time() - t0:.1f} s)")


def gen_codegen():
    """reference gradient() of the codegen test programs (tests/golden/codegen/*.rnl):
    per row the primal outputs, the cotangents of the Float parameters and the
    error class (default seed: the first parameter)."""
    cases = {
        "mul_acc": (["y!", "a", "b"], {}, 64),
        "sink": (["out!", "x", "y"], {"n": 3}, 64),
        "wloop": (["acc!", "x"], {"n": 5}, 48),
        "prims": (["a!", "b!", "c!", "th"], {"n!": 3}, 40),
        "loose": (["y!", "x"], {}, 24),
        "xorfold": (["y!", "x"], {"n": 5, "m!": 6}, 16),
    }
    out = {}
    for fn, (floats, ints, n) in cases.items():
        prog = parse_program(open(os.path.join(OUT_DIR, "codegen", fn + ".rnl")).read())
        rng = np.random.default_rng(sum(map(ord, fn)))
        X = rng.uniform(0.05, 1.8, (n, len(floats)))
        X[:, 0] = rng.normal(size=n)
        if fn == "sink":
            X[3, 2], X[7, 1] = -0.5, -0.3          # RevDomainError rows (log y, log x)
        names = floats + list(ints)
        from revlang.autodiff import hessian
        P, G = np.full((n, len(floats)), np.nan), np.full((n, len(floats)), np.nan)
        H = np.full((n, len(floats), len(floats)), np.nan)
        errs, herrs = [], []
        for i in range(n):
            args = [float(v) for v in X[i]]
            call = []
            pn = prog.get(fn).param_names()
            for nm in pn:
                call.append(ints[nm] if nm in ints else args[floats.index(nm)])
            r, en = _err_name(lambda: gradient(prog, GradRequest(fn, call)))
            errs.append(en)
            h, hn = _err_name(lambda: hessian(prog, fn, call))
            herrs.append(hn)
            if h is not None:
                H[i] = h.matrix
            if r is not None:
                prim, grads = r
                for j, nm in enumerate(floats):
                    P[i, j] = prim[pn.index(nm)]
                    G[i, j] = grads[nm]
        out[fn + "_x"], out[fn + "_primal"], out[fn + "_grad"] = X, P, G
        out[fn + "_err"] = np.array(errs)
        out[fn + "_hess"], out[fn + "_hess_err"] = H, np.array(herrs)
    np.savez_compressed(os.path.join(OUT_DIR, "codegen.npz"), **out)
    print("codegen goldens written")


def _leaves_of(value, shape):
    """Flatten a scalar / Array value (or its cotangent structure) in leaf order."""
    if not shape:
        return [np.nan if value is None else float(value)]
    return [np.nan if v is None else float(v) for v in value.data]


def gen_codegen_arrays():
    """reference gradient() / hessian() of the array test programs
    (tests/golden/codegen/{quad,mix}.rnl).  Rows hold the Float leaves in
    codegen's column order (parameters in order, array cells row-major)."""
    from revlang.autodiff import hessian
    from revlang.values import Array
    cases = {
        # name: (file, fn, [(param, shape or None)], ints, seeds, rows, hessian?)
        "quad": ("quad", "quad", [("q!", ()), ("r!", (3,)), ("A", (3, 3)), ("u", (3,))],
                 {}, None, 40, True),
        "quad_bad": ("quad", "quad", [("q!", ()), ("r!", (2,)), ("A", (3, 2)), ("u", (2,))],
                     {}, None, 4, False),
    }
    xseed = [("x", (("idx", (1,)),), 1.0), ("x", (("idx", (3,)),), -0.5)]
    for k, m in ((1, 2), (3, 3), (5, 1), (2, 4)):
        cases[f"mix_fwd_{k}{m}"] = ("mix", "mix_fwd", [("x", (4,))], {"k": k, "m": m}, xseed,
                                    6, False)
    for k, m in ((1, 2), (3, 3), (0, 1)):
        cases[f"mix_grad_{k}{m}"] = ("mix", "mix_grad", [("y!", ()), ("x", (4,))],
                                     {"k": k, "m": m}, None, 6, True)
    cases["mix_arity"] = ("mix", "mix_arity", [("y!", ()), ("x", (4,))], {"k": 1}, None, 4,
                          False)
    out = {}
    for case, (file, fn, fparams, ints, seeds, n, with_h) in cases.items():
        prog = parse_program(open(os.path.join(OUT_DIR, "codegen", file + ".rnl")).read())
        pn = prog.get(fn).param_names()
        sizes = [int(np.prod(shp)) if shp else 1 for _, shp in fparams]
        NL = sum(sizes)
        rng = np.random.default_rng(sum(map(ord, case)))
        X = rng.uniform(-1.5, 1.5, (n, NL))
        P, G = np.full((n, NL), np.nan), np.full((n, NL), np.nan)
        H = np.full((n, NL, NL), np.nan)
        errs, herrs = [], []
        for i in range(n):
            vals, b = {}, 0
            for (nm, shp), sz in zip(fparams, sizes):
                row = [float(v) for v in X[i, b:b + sz]]
                b += sz
                if not shp:
                    vals[nm] = row[0]
                elif len(shp) == 1:
                    vals[nm] = Array.vector(row)
                else:
                    vals[nm] = Array.matrix([row[r * shp[1]:(r + 1) * shp[1]]
                                             for r in range(shp[0])])
            call = [ints[nm] if nm in ints else vals[nm] for nm in pn]
            r, en = _err_name(lambda: gradient(prog, GradRequest(fn, call, seeds=seeds)))
            errs.append(en)
            if r is not None:
                prim, grads = r
                pl, gl = [], []
                for nm, shp in fparams:
                    pl += _leaves_of(prim[pn.index(nm)], shp)
                    gl += _leaves_of(grads[nm], shp)
                P[i], G[i] = pl, gl
            if with_h:
                h, hn = _err_name(lambda: hessian(prog, fn, call))
                herrs.append(hn)
                if h is not None:
                    H[i] = h.matrix
        out[case + "_x"], out[case + "_primal"], out[case + "_grad"] = X, P, G
        out[case + "_err"] = np.array(errs)
        if with_h:
            out[case + "_hess"], out[case + "_hess_err"] = H, np.array(herrs)
    np.savez_compressed(os.path.join(OUT_DIR, "codegen_arrays.npz"), **out)
    print("codegen array goldens written:",
          {c: sorted(set(out[c + "_err"])) for c in cases})


def gen_codegen_programs():
    """reference hessian() of the paper programs themselves (programs/gmm.rnl
    case c5 of gmm.npz, programs/ba.rnl observations 0-3 of ba.npz), for the
    generic compiler's Dual-number kernels (gradient parity uses gmm.npz /
    ba.npz directly)."""
    from revlang.autodiff import hessian
    out = {}
    G = np.load(os.path.join(OUT_DIR, "gmm.npz"))
    pre = "c5_"
    d, K, N, m = (int(v) for v in G[pre + "dims"])
    A = lambda a: Array.matrix(a.tolist()) if a.ndim == 2 else Array.vector(a.tolist())  # noqa
    Z = lambda *s: A(np.zeros(s))  # noqa: E731
    args = [0.0, A(G[pre + "alphas"]), A(G[pre + "means"]), A(G[pre + "icf"]), A(G[pre + "x"]),
            Z(K, d), Z(K), Z(d), Z(d), Z(K), Array.vector([0] * K), float(G[pre + "gamma"]), m,
            float(G[pre + "cst"])]
    out["gmm_c5_hess"] = hessian(_prog("gmm.rnl"), "gmm", args).matrix
    B = np.load(os.path.join(OUT_DIR, "ba.npz"))
    Hs = []
    for o in range(4):
        args = [0.0, 0.0, Array.vector(B["cams"][o].tolist()), Array.vector(B["X"][o].tolist()),
                float(B["w"][o]), float(B["feat"][o, 0]), float(B["feat"][o, 1])]
        Hs.append(hessian(_prog("ba.rnl"), "ba_proj", args).matrix)
    out["ba_hess"] = np.array(Hs)
    np.savez_compressed(os.path.join(OUT_DIR, "codegen_programs.npz"), **out)
    print("codegen program hessians:", {k: v.shape for k, v in out.items()})


def gen_codegen_dropin():
    """reference run / uncall / check_reversibility / jacobian of the codegen
    test programs through the public API, for the drop-in generic path
    (autodiff / interp -> generic.py -> codegen.py)."""
    from revlang.autodiff import jacobian
    from revlang.interpreter import check_reversibility, run, uncall
    from revlang.values import Array
    out = {}
    g = np.load(os.path.join(OUT_DIR, "codegen.npz"))
    prog = parse_program(open(os.path.join(OUT_DIR, "codegen", "prims.rnl")).read())
    X = g["prims_x"][:6]
    runs, uncs, devs = [], [], []
    for row in X:
        args = [float(v) for v in row] + [3]
        runs.append(run(prog, "prims", list(args))[:4] + [0.0])
        uncs.append(uncall(prog, "prims", list(args))[:4] + [0.0])
        devs.append(check_reversibility(prog, "prims", list(args)).max_deviation)
    out["prims_x"], out["prims_run"], out["prims_uncall"] = X, np.array(runs)[:, :4], \
        np.array(uncs)[:, :4]
    out["prims_dev"] = np.array(devs)
    out["prims_jac"] = jacobian(prog, "prims", [float(v) for v in X[0]] + [3])
    q = parse_program(open(os.path.join(OUT_DIR, "codegen", "quad.rnl")).read())
    ga = np.load(os.path.join(OUT_DIR, "codegen_arrays.npz"))
    row = ga["quad_x"][0]
    args = [float(row[0]), Array.vector(row[1:4].tolist()),
            Array.matrix(row[4:13].reshape(3, 3).tolist()), Array.vector(row[13:16].tolist())]
    r = run(q, "quad", args)
    out["quad_run"] = np.array([r[0]] + list(r[1].data) + list(r[2].data) + list(r[3].data))
    np.savez_compressed(os.path.join(OUT_DIR, "codegen_dropin.npz"), **out)
    print("codegen drop-in goldens:", {k: np.shape(v) for k, v in out.items()})


def gen_codegen_nbody():
    """reference gradient() / run / uncall of tests/golden/codegen/nbody.rnl
    (nested calls whose view arguments are indexed by a loop variable that is
    itself an argument; 2-d arrays; routines in the callee): 4 bodies, 3
    steps, 12 random systems, seeds on pos![1, 1] and vel![2, 3]."""
    from revlang.interpreter import run, uncall
    from revlang.values import Array
    prog = parse_program(open(os.path.join(OUT_DIR, "codegen", "nbody.rnl")).read())
    rng = np.random.default_rng(11)
    nb, n = 4, 12
    X = np.concatenate([rng.uniform(-1, 1, (n, nb * 3)), rng.uniform(-0.2, 0.2, (n, nb * 3)),
                        rng.uniform(0.5, 1.5, (n, nb)), np.full((n, 1), 0.01)], 1)
    seeds = [("pos!", (("idx", (1, 1)),), 1.0), ("vel!", (("idx", (2, 3)),), 0.5)]
    P, G, R, U = [], [], [], []
    for row in X:
        pos, vel = row[:12].reshape(nb, 3), row[12:24].reshape(nb, 3)
        mass, h = row[24:28], float(row[28])
        args = lambda: [Array.matrix(pos.tolist()), Array.matrix(vel.tolist()),  # noqa: E731
                        Array.vector(mass.tolist()), h, 3]
        prim, g = gradient(prog, GradRequest("nbody", args(), seeds=seeds))
        P.append(list(prim[0].data) + list(prim[1].data))
        G.append(list(g["pos!"].data) + list(g["vel!"].data) + list(g["mass"].data) + [g["h"]])
        r = run(prog, "nbody", args())
        R.append(list(r[0].data) + list(r[1].data))
        u = uncall(prog, "nbody", args())
        U.append(list(u[0].data) + list(u[1].data))
    np.savez_compressed(os.path.join(OUT_DIR, "codegen_nbody.npz"), x=X, primal=np.array(P),
                        grad=np.array(G), run=np.array(R), uncall=np.array(U))
    print("nbody goldens:", np.array(G).shape)


def random_program(rng, name):
    """A random reversible function over Float cells y!, a, b, c and an Int n
    (this repository's generator, for differential testing of codegen.py):
    instructions with distinct operands, counted loops, branches whose
    condition the branch does not touch, ancilla blocks, SWAP / ROT."""
    cells = ["y!", "a", "b", "c"]
    fns1 = ["identity", "neg", "abs2", "sin", "cos", "sqrt", "exp"]
    fns2 = ["+", "-", "*", "/"]
    lines = []

    def instr(ind, avoid=()):
        tgt = rng.choice([x for x in cells if x not in avoid])
        op = rng.choice(["+=", "-="])
        others = [x for x in cells if x != tgt]
        if rng.random() < 0.5:
            f = rng.choice(fns1)
            x = rng.choice(others)
            return f"{ind}{tgt} {op} {x}" if f == "identity" else (
                f"{ind}{tgt} {op} -{x}" if f == "neg" else f"{ind}{tgt} {op} {f}({x})")
        f = rng.choice(fns2)
        x, z = rng.choice(others, 2, replace=False)
        if rng.random() < 0.3:
            z = repr(float(np.round(rng.uniform(0.5, 2.0), 3)))
        return f"{ind}{tgt} {op} {x} {f} {z}"

    for k in range(int(rng.integers(3, 7))):
        r = rng.random()
        if r < 0.45:
            lines.append(instr("    "))
        elif r < 0.6:
            lines += ["    for i = 1:1:n", instr("        "), "    end"]
        elif r < 0.72:
            x, z = rng.choice(cells, 2, replace=False)
            lines += [f"    if ({x} > {z}, ~)", instr("        ", (x, z)), "    else",
                      instr("        ", (x, z)), "    end"]
        elif r < 0.86:
            x = rng.choice(cells)
            t = f"t{k}"
            f = rng.choice(["sin", "cos", "abs2"])
            lines += [f"    {t} <- 0.0", f"    {t} += {f}({x})",
                      f"    {rng.choice([c for c in cells if c != x])} += {t}",
                      f"    {t} -= {f}({x})", f"    {t} -> 0.0"]
        elif r < 0.93:
            x, z = rng.choice(cells, 2, replace=False)
            lines.append(f"    SWAP({x}, {z})")
        else:
            x, z, w = rng.choice(cells, 3, replace=False)
            lines.append(f"    ROT({x}, {z}, {w})")
    return f"fn {name}(y!, a, b, c, n)\n" + "\n".join(lines) + "\nend\n"


def random_program_ulog(rng, name):
    """random_program's constructs plus log-domain ancilla blocks (ulog,
    *= / /= convert, += convert) and counted while loops over an Int ancilla."""
    base = random_program(rng, name).splitlines()[1:-1]
    cells = ["y!", "a", "b", "c"]
    extra = []
    for k in range(int(rng.integers(1, 3))):
        x, z = rng.choice(cells, 2, replace=False)
        l = f"l{k}"
        if rng.random() < 0.5:
            extra += [f"    {l} <- ulog(1.0)", f"    {l} *= convert({x})",
                      f"    {z} += convert({l})", f"    {l} /= convert({x})",
                      f"    {l} -> ulog(1.0)"]
        else:
            j = f"j{k}"
            w = rng.choice([c for c in cells if c != z])
            extra += [f"    {j} <- 0", f"    while ({j} < n, {j} > 0)", f"        {j} += 1",
                      f"        {z} += {w} * 0.5", "    end", f"    {j} -> n"]
    cut = int(rng.integers(0, len(base) + 1))
    body = base[:cut] + extra + base[cut:]
    return f"fn {name}(y!, a, b, c, n)\n" + "\n".join(body) + "\nend\n"


def gen_codegen_random():
    """reference gradient() of 80 random programs (40 random_program, 40
    random_program_ulog) on 6 random inputs each: primal outputs,
    cotangents and error classes."""
    rng = np.random.default_rng(2024)
    texts, X, P, G, E = [], [], [], [], []
    for q in range(80):
        name = f"r{q}"
        text = random_program(rng, name) if q < 40 else random_program_ulog(rng, name)
        prog = parse_program(text)
        xs = rng.uniform(-2.0, 2.0, (6, 4))
        ns = rng.integers(1, 4, 6)
        for row, n in zip(xs, ns):
            args = [float(v) for v in row] + [int(n)]
            r, en = _err_name(lambda: gradient(prog, GradRequest(name, args)))
            p = g = [np.nan] * 4
            if r is not None:
                prim, grads = r
                p = [float(v) for v in prim[:4]]
                g = [float(grads[c]) for c in ("y!", "a", "b", "c")]
            P.append(p)
            G.append(g)
            E.append(en)
            X.append(list(row) + [int(n)])
        texts.append(text)
    np.savez_compressed(os.path.join(OUT_DIR, "codegen_random.npz"), texts=np.array(texts),
                        x=np.array(X), primal=np.array(P), grad=np.array(G), err=np.array(E))
    from collections import Counter
    print("random programs:", len(texts), Counter(E))


def gen_codegen_complex():
    """reference gradient() (seeds y!.re, then y!.im) and hessian() of
    tests/golden/codegen/polar.rnl (Complex parameters, field views, abs2 /
    angle of a Complex operand, ROT by a field) on 12 random inputs."""
    from revlang.autodiff import hessian
    from revlang.values import Complex
    prog = parse_program(open(os.path.join(OUT_DIR, "codegen", "polar.rnl")).read())
    rng = np.random.default_rng(77)
    X = np.concatenate([rng.uniform(-1, 1, (12, 2)), rng.uniform(-2, 2, (12, 2)) *
                        rng.choice([-1, 1], (12, 2)), rng.uniform(-1, 1, (12, 2))], 1)
    X[3, 2:4] = 0.0                                 # x = 0: log(0) -> RevDomainError
    out = {"x": X}
    for tag, path in (("re", (("field", "re"),)), ("im", (("field", "im"),))):
        P, G, E = [], [], []
        for row in X:
            args = [Complex(row[0], row[1]), Complex(row[2], row[3]), row[4], row[5]]
            r, en = _err_name(lambda: gradient(prog, GradRequest("polar", args,
                                                                 seeds=[("y!", path, 1.0)])))
            p = g = [np.nan] * 6
            if r is not None:
                prim, gr = r
                p = [prim[0].re, prim[0].im, prim[1].re, prim[1].im, prim[2], prim[3]]
                g = [gr["y!"].re, gr["y!"].im, gr["x"].re, gr["x"].im, gr["p!"], gr["q!"]]
            P.append([float(v) for v in p])
            G.append([float(v) for v in g])
            E.append(en)
        out[f"primal_{tag}"], out[f"grad_{tag}"], out[f"err_{tag}"] = \
            np.array(P), np.array(G), np.array(E)
    H, HE = [], []
    for row in X:
        args = [Complex(row[0], row[1]), Complex(row[2], row[3]), row[4], row[5]]
        try:                  # the reference's Dual sqrt at 0 raises ZeroDivisionError
            h, hn = _err_name(lambda: hessian(prog, "polar", args))
        except ZeroDivisionError:
            h, hn = None, "ZeroDivisionError"
        H.append(h.matrix if h is not None else np.full((6, 6), np.nan))
        HE.append(hn)
    out["hess"], out["hess_err"] = np.array(H), np.array(HE)
    np.savez_compressed(os.path.join(OUT_DIR, "codegen_complex.npz"), **out)
    from collections import Counter
    print("complex goldens:", Counter(out["err_re"]), Counter(HE))


def gen_bessel_fuel():
    """FuelExhausted boundaries of besselj (ExecOptions.max_steps counts
    statement executions per interpreter, interpreter.py:461-466): for each
    (nu, z) the reference's step count S of one run (read from the
    interpreter's stats), then the outcomes of gradient(), run() and
    hessian() at max_steps = S (fits) and S - 1 (FuelExhausted)."""
    from revlang.autodiff import hessian
    from revlang.interpreter import Interpreter
    p = parse_program(open(os.path.join(PROG_DIR, "besselj.rnl")).read())
    cases = [(nu, z) for nu in (0, 1, 2, 5) for z in (0.05, 0.7, 3.0, 8.0, 13.0)]
    NU, Z, S, T = [], [], [], []
    out = {}
    for nu, z in cases:
        it = Interpreter(p, ExecOptions())
        it.run_function("besselj", [0.0, nu, z])
        steps = it.stats.steps
        NU.append(nu)
        Z.append(z)
        S.append(steps)
        T.append((steps - 31 - 6 * nu) // 22)
        for tag, fn in (("grad", lambda o: gradient(p, GradRequest("besselj", [0.0, nu, z]), o)),
                        ("run", lambda o: run(p, "besselj", [0.0, nu, z], o)),
                        ("hess", lambda o: hessian(p, "besselj", [0.0, nu, z], o))):
            for off in (0, -1):
                _, en = _err_name(lambda: fn(ExecOptions(max_steps=steps + off)))
                out.setdefault(f"{tag}_{-off}", []).append(en)
    np.savez_compressed(os.path.join(OUT_DIR, "bessel_fuel.npz"), nu=np.array(NU), z=np.array(Z),
                        steps=np.array(S), trips=np.array(T),
                        **{k: np.array(v) for k, v in out.items()})
    print("fuel goldens:", list(zip(NU, Z, S)), {k: sorted(set(v)) for k, v in out.items()})


def gen_gmm_fuel():
    """Statement counts of programs/gmm.rnl in the reference (the fuel unit of
    ExecOptions.max_steps) over small (d, K, N), from the run's interpreter
    stats, and the gradient's outcome at max_steps = S and S - 1."""
    from revlang.interpreter import Interpreter
    p = parse_program(open(os.path.join(PROG_DIR, "gmm.rnl")).read())
    A = lambda a: Array.matrix(a.tolist()) if a.ndim == 2 else Array.vector(a.tolist())  # noqa
    out = {k: [] for k in ("dims", "alphas", "means", "icf", "x", "steps", "grad_0", "grad_1")}
    for ci, (d, K, N) in enumerate(((2, 3, 4), (3, 4, 6), (5, 2, 3), (4, 6, 5))):
        rng = np.random.default_rng(500 + ci)
        al, me = rng.normal(0, 1, K), rng.uniform(0, 1, (K, d))
        ic, x = rng.normal(0, 1, (K, d * (d + 1) // 2)), rng.uniform(0, 1, (N, d))
        Z = lambda *s: A(np.zeros(s))  # noqa: E731
        args = [0.0, A(al), A(me), A(ic), A(x), Z(K, d), Z(K), Z(d), Z(d), Z(K),
                Array.vector([0] * K), 1.0, 0, 0.5]
        it = Interpreter(p, ExecOptions())
        it.run_function("gmm", [deep_copy(a) for a in args])
        steps = it.stats.steps
        for off in (0, 1):
            _, en = _err_name(lambda: gradient(p, GradRequest("gmm", [deep_copy(a) for a in args]),
                                               ExecOptions(max_steps=steps - off,
                                                           float_tolerance=1e-6)))
            out[f"grad_{off}"].append(en)
        for k, v in (("dims", [d, K, N]), ("alphas", al), ("means", me.ravel()),
                     ("icf", ic.ravel()), ("x", x.ravel()), ("steps", steps)):
            out[k].append(np.asarray(v))
    flat = {"ncases": np.array(len(out["steps"])), "steps": np.array(out["steps"]),
            "grad_0": np.array(out["grad_0"]), "grad_1": np.array(out["grad_1"])}
    for ci in range(len(out["steps"])):
        for k in ("dims", "alphas", "means", "icf", "x"):
            flat[f"c{ci}_{k}"] = np.asarray(out[k][ci])
    np.savez_compressed(os.path.join(OUT_DIR, "gmm_fuel.npz"), **flat)
    print("gmm fuel goldens:", out["steps"], out["grad_0"], out["grad_1"])


def gen_ba_fuel():
    """The reference's statement counts of ba_proj (with / without rotation)
    and ba_weight, and the gradient's outcome at max_steps = S and S - 1."""
    from revlang.interpreter import Interpreter
    p = parse_program(open(os.path.join(PROG_DIR, "ba.rnl")).read())
    out = {"rot": [], "steps": [], "grad_0": [], "grad_1": []}
    for rot in ([0.1, -0.2, 0.3], [0.0, 0.0, 0.0]):
        cam = Array.vector(rot + [0.1, 0.2, 0.3, 550.0, 0.5, 0.5, 0.001, -0.002])
        X = Array.vector([0.3, -0.4, 10.0])
        for fn, args in (("ba_proj", [0.0, 0.0, cam, X, 0.7, 3.0, 4.0]), ("ba_weight", [0.0, 0.7])):
            it = Interpreter(p, ExecOptions())
            it.run_function(fn, [deep_copy(a) for a in args])
            steps = it.stats.steps
            out["rot"].append(list(rot) + [1.0 if fn == "ba_proj" else 0.0])
            out["steps"].append(steps)
            for off in (0, 1):
                _, en = _err_name(lambda: gradient(p, GradRequest(fn, [deep_copy(a) for a in args]),
                                                   ExecOptions(max_steps=steps - off)))
                out[f"grad_{off}"].append(en)
    np.savez_compressed(os.path.join(OUT_DIR, "ba_fuel.npz"), **{k: np.array(v) for k, v in out.items()})
    print("ba fuel goldens:", out)


def gen_codegen_complex_fd():
    """reference finite_difference() of polar.rnl (Complex arguments: re/im
    leaves, default seed y!.re and an explicit y!.im seed), h = 1e-6."""
    from revlang.autodiff import finite_difference
    from revlang.values import Complex
    prog = parse_program(open(os.path.join(OUT_DIR, "codegen", "polar.rnl")).read())
    g = np.load(os.path.join(OUT_DIR, "codegen_complex.npz"))
    X = g["x"]
    rows = [i for i in range(X.shape[0]) if g["err_re"][i] == ""][:6]
    out = {"rows": np.array(rows), "h": np.array(1e-6)}
    for tag, seeds in (("re", None), ("im", [("y!", (("field", "im"),), 1.0)])):
        G = []
        for i in rows:
            row = X[i]
            args = [Complex(row[0], row[1]), Complex(row[2], row[3]), row[4], row[5]]
            fd = finite_difference(prog, "polar", args, 1e-6, seeds=seeds)
            G.append([fd["y!"].re, fd["y!"].im, fd["x"].re, fd["x"].im, fd["p!"], fd["q!"]])
        out["fd_" + tag] = np.array(G, dtype=np.float64)
    np.savez_compressed(os.path.join(OUT_DIR, "codegen_complex_fd.npz"), **out)
    print("complex fd goldens:", len(rows), "rows")


def gen_codegen_fixed():
    """fxmix.rnl (Fixed / Q31.32 cells) through the reference: run, uncall,
    gradient with the default seed (acc!, a Fixed leaf: Fixed cotangents,
    each accumulation quantized to 2^-32) and with a y! seed, and
    finite_difference (the measured Fixed step).  Fixed values are stored as
    their raw int64; errors as the exception class name."""
    from revlang import GradRequest, gradient, run, uncall
    from revlang.autodiff import finite_difference
    from revlang.values import Fixed
    prog = parse_program(open(os.path.join(OUT_DIR, "codegen", "fxmix.rnl")).read())
    rng = np.random.default_rng(61)
    cases = [(0.0, 0.0, 1.3, 5), (0.75, -2.0, 1.9, 7), (0.0, 0.0, 0.3, 5), (-1.5, 0.5, 0.5, 3),
             (0.0, 0.0, 1.9, 45), (0.0, 0.0, 1.9, 2000), (2.0, 1.0, 1.05, 0), (0.0, 0.0, -3.0, 4)]
    cases += [(float(rng.uniform(-2, 2)), float(rng.uniform(-2, 2)), float(rng.uniform(0.2, 2.2)),
               int(rng.integers(0, 12))) for _ in range(24)]
    out = {"cases": np.array([c[:3] for c in cases]), "k": np.array([c[3] for c in cases])}

    def rawv(v):
        return v.raw if isinstance(v, Fixed) else v

    for tag, fn in (("run", run), ("uncall", uncall)):
        R, E = [], []
        for a0, y0, b, k in cases:
            try:
                o = fn(prog, "fxmix", [Fixed.from_real(a0), y0, Fixed.from_real(b), k])
                R.append([o[0].raw, np.float64(o[1]).view(np.int64), o[2].raw])
                E.append("")
            except Exception as err:  # noqa: BLE001
                R.append([0, 0, 0])
                E.append(type(err).__name__)
        out[tag] = np.array(R, dtype=np.int64)
        out[tag + "_err"] = np.array(E)
    for tag, seeds in (("gacc", None), ("gy", [("y!", (), 1.0)])):
        R, E = [], []
        for a0, y0, b, k in cases:
            try:
                prim, g = gradient(prog, GradRequest("fxmix", [Fixed.from_real(a0), y0,
                                                               Fixed.from_real(b), k],
                                                     seeds=seeds))
                R.append([prim[0].raw, np.float64(prim[1]).view(np.int64), prim[2].raw,
                          g["acc!"].raw, np.float64(g["y!"]).view(np.int64), g["b"].raw])
                E.append("")
            except Exception as err:  # noqa: BLE001
                R.append([0] * 6)
                E.append(type(err).__name__)
        out[tag] = np.array(R, dtype=np.int64)
        out[tag + "_err"] = np.array(E)
    F, E = [], []
    for a0, y0, b, k in cases:
        try:
            fd = finite_difference(prog, "fxmix", [Fixed.from_real(a0), y0, Fixed.from_real(b), k],
                                   1e-6)
            F.append([fd["acc!"], fd["y!"], fd["b"]])
            E.append("")
        except Exception as err:  # noqa: BLE001
            F.append([0.0] * 3)
            E.append(type(err).__name__)
    out["fd"] = np.array(F, dtype=np.float64)
    out["fd_err"] = np.array(E)
    np.savez_compressed(os.path.join(OUT_DIR, "codegen_fixed.npz"), **out)
    print("fixed goldens:", len(cases), "cases; errors:", sorted(set(out["run_err"]) - {""}),
          sorted(set(out["gacc_err"]) - {""}))


def gen_codegen_recursion():
    """countdown.rnl (recursion through bijector-view arguments, Int cells)
    through the reference: run and uncall of chain for n = 0..12 and of tri
    for k = 0..20."""
    from revlang import run, uncall
    prog = parse_program(open(os.path.join(OUT_DIR, "codegen", "countdown.rnl")).read())
    ns = np.arange(13)
    out = {"n": ns, "k": np.arange(21)}
    out["chain_run"] = np.array([run(prog, "chain", [0, int(n)]) for n in ns], dtype=np.int64)
    out["chain_uncall"] = np.array([uncall(prog, "chain", [100, int(n)]) for n in ns],
                                   dtype=np.int64)
    out["tri_run"] = np.array([run(prog, "tri", [7, int(k)]) for k in out["k"]], dtype=np.int64)
    np.savez_compressed(os.path.join(OUT_DIR, "codegen_recursion.npz"), **out)
    print("recursion goldens:", len(ns), "chain cases")


if __name__ == "__main__":
    os.makedirs(OUT_DIR, exist_ok=True)
    which = sys.argv[1:] or ["bessel", "ba", "gmm", "run", "hess", "codegen",
                              "codegen_arrays", "codegen_programs",
                              "codegen_dropin", "codegen_nbody",
                              "codegen_random",
                              "codegen_complex", "codegen_complex_fd", "codegen_fixed",
                              "codegen_recursion", "bessel_fuel",
                              "gmm_fuel", "ba_fuel"]
    for w in which:
        globals()["gen_" + w]()
