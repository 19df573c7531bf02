"""ADBench on-disk formats either side of the BA / GMM paths (SURVEY.md §8(f)
rank 2): the instance files the paper's §5 benchmarks read and the Jacobian
files they write, so a real ADBench data directory can be fed straight to
the kernels.

Restated from ADBench (github.com/microsoft/ADBench, src/cpp/shared/utils.cpp
`read_gmm_instance` / `read_ba_instance` / `write_J` / `write_J_sparse`);
ADBench is not part of /root/reference and none of its data files are
available in this image, so the formats are pinned by round-trip tests and
hand-written instances only.  Host-side text I/O (numpy); not on the hot
path.

GMM instance (whitespace separated):
    d k n
    alphas            k values
    means             k rows of d
    icf               k rows of d(d+1)/2
    x                 n rows of d   (one row when replicate_point: ADBench's
                                     gmm_d*_K* inputs store one point)
    gamma m           the Wishart prior
BA instance:
    n m p
    one camera (11 values), one point (3), one weight, one feature (2);
    ADBench replicates them to n cameras, m points, p observations and sets
    obs[i] = (i mod n, i mod m).  `write_ba_instance(..., full=True)` writes
    our own explicit variant (all cameras, points, weights, features and the
    obs pairs) which read_ba_instance recognises by its header word.
"""

from dataclasses import dataclass

import numpy as np

BA_NCAMPARAMS = 11
_FULL_MAGIC = "revgpu-ba-full"


@dataclass
class GMMInstance:
    alphas: np.ndarray     # (K,)
    means: np.ndarray      # (K, d)
    icf: np.ndarray        # (K, d(d+1)/2)
    x: np.ndarray          # (N, d)
    gamma: float
    m: int

    @property
    def dims(self):
        K, d = self.means.shape
        return d, K, self.x.shape[0]


@dataclass
class BAInstance:
    cams: np.ndarray       # (n, 11)
    X: np.ndarray          # (m, 3)
    w: np.ndarray          # (p,)
    feats: np.ndarray      # (p, 2)
    obs: np.ndarray        # (p, 2) int32 (camera, point), 0-based

    @property
    def dims(self):
        return self.cams.shape[0], self.X.shape[0], self.w.shape[0]


class _Tokens:
    def __init__(self, path):
        with open(path) as f:
            self.t = f.read().split()
        self.i = 0

    def take(self, n, conv=float):
        if self.i + n > len(self.t):
            raise ValueError(f"truncated ADBench file: wanted {n} more values at token {self.i}")
        v = self.t[self.i:self.i + n]
        self.i += n
        return [conv(s) for s in v]

    def floats(self, n):
        return np.array(self.take(n), dtype=np.float64)


def read_gmm_instance(path, replicate_point=False):
    """ADBench read_gmm_instance: returns a GMMInstance (x expanded to n rows)."""
    t = _Tokens(path)
    d, K, n = t.take(3, int)
    P = d * (d + 1) // 2
    alphas = t.floats(K)
    means = t.floats(K * d).reshape(K, d)
    icf = t.floats(K * P).reshape(K, P)
    if replicate_point:
        x = np.tile(t.floats(d), (n, 1))
    else:
        x = t.floats(n * d).reshape(n, d)
    gamma = float(t.take(1)[0])
    m = int(t.take(1, lambda s: int(float(s)))[0])
    return GMMInstance(alphas, means, icf, x, gamma, m)


def write_gmm_instance(path, inst, replicate_point=False):
    d, K, n = inst.dims
    with open(path, "w") as f:
        f.write(f"{d} {K} {n}\n")
        for a in inst.alphas:
            f.write(f"{float(a)!r}\n")
        for rows in (inst.means, inst.icf):
            for r in rows:
                f.write(" ".join(repr(float(v)) for v in r) + "\n")
        xs = inst.x[:1] if replicate_point else inst.x
        for r in xs:
            f.write(" ".join(repr(float(v)) for v in r) + "\n")
        f.write(f"{float(inst.gamma)!r} {int(inst.m)}\n")


def read_ba_instance(path):
    """ADBench read_ba_instance (replicated) or our explicit full variant."""
    t = _Tokens(path)
    if t.t and t.t[0] == _FULL_MAGIC:
        t.i = 1
        n, m, p = t.take(3, int)
        cams = t.floats(n * BA_NCAMPARAMS).reshape(n, BA_NCAMPARAMS)
        X = t.floats(m * 3).reshape(m, 3)
        w = t.floats(p)
        feats = t.floats(p * 2).reshape(p, 2)
        obs = np.array(t.take(2 * p, int), dtype=np.int32).reshape(p, 2)
        return BAInstance(cams, X, w, feats, obs)
    n, m, p = t.take(3, int)
    cams = np.tile(t.floats(BA_NCAMPARAMS), (n, 1))
    X = np.tile(t.floats(3), (m, 1))
    w = np.full(p, t.floats(1)[0])
    feats = np.tile(t.floats(2), (p, 1))
    i = np.arange(p, dtype=np.int64)
    obs = np.stack([i % n, i % m], 1).astype(np.int32)
    return BAInstance(cams, X, w, feats, obs)


def write_ba_instance(path, inst, full=False):
    """ADBench layout (one camera/point/weight/feature, replicated on read)
    unless `full`, which keeps every value and the obs pairs."""
    n, m, p = inst.dims
    fl = lambda a: " ".join(repr(float(v)) for v in np.ravel(a))  # noqa: E731
    with open(path, "w") as f:
        if full:
            f.write(f"{_FULL_MAGIC}\n{n} {m} {p}\n")
            for blk in (inst.cams, inst.X, inst.w, inst.feats):
                for r in np.atleast_2d(blk) if blk.ndim > 1 else [blk]:
                    f.write(fl(r) + "\n")
            f.write(" ".join(str(int(v)) for v in np.ravel(inst.obs)) + "\n")
            return
        f.write(f"{n} {m} {p}\n{fl(inst.cams[0])}\n{fl(inst.X[0])}\n{fl(inst.w[:1])}\n"
                f"{fl(inst.feats[0])}\n")


def write_J(path, J):
    """ADBench write_J (dense): 'rows cols' then the values row by row —
    the GMM gradient is 1 x (K + K d + K d(d+1)/2), ordered alphas, means,
    icf (our packed vector without its leading objective)."""
    J = np.atleast_2d(np.asarray(J, dtype=np.float64))
    with open(path, "w") as f:
        f.write(f"{J.shape[0]} {J.shape[1]}\n")
        for r in J:
            f.write(" ".join(repr(float(v)) for v in r) + "\n")


def read_J(path):
    t = _Tokens(path)
    r, c = t.take(2, int)
    return t.floats(r * c).reshape(r, c)


def write_J_sparse(path, csr):
    """ADBench write_J_sparse: 'nrows ncols', then len(rows) and the row
    pointers, len(cols) and the column indices, then the values.  `csr` is
    a whole-problem BACsr (host or device arrays)."""
    f64 = lambda a: a.cpu().numpy() if hasattr(a, "cpu") else np.asarray(a)  # noqa: E731
    rows, cols, vals = f64(csr.rows), f64(csr.cols), f64(csr.vals)
    with open(path, "w") as f:
        f.write(f"{csr.shape[0]} {csr.shape[1]}\n")
        f.write(f"{rows.size}\n" + " ".join(str(int(v)) for v in rows) + "\n")
        f.write(f"{cols.size}\n" + " ".join(str(int(v)) for v in cols) + "\n")
        f.write(" ".join(repr(float(v)) for v in vals) + "\n")


def read_J_sparse(path):
    """-> (rows int32, cols int32, vals float64, (nrows, ncols))."""
    t = _Tokens(path)
    nr, nc = t.take(2, int)
    rows = np.array(t.take(t.take(1, int)[0], int), dtype=np.int32)
    cols = np.array(t.take(t.take(1, int)[0], int), dtype=np.int32)
    vals = t.floats(cols.size)
    return rows, cols, vals, (nr, nc)
