"""ADBench formats: instance/Jacobian file round trips,
and the oracle's BASparseMat restatement against an independent dense
assembly of the Jacobian (CPU only)."""

import numpy as np
import pytest

from paper_2003_04617_b200 import adbench
from oracle import ba_sparse


def test_gmm_instance_round_trip(tmp_path):
    rng = np.random.default_rng(0)
    d, K, n = 3, 4, 7
    inst = adbench.GMMInstance(rng.normal(size=K), rng.random((K, d)),
                               rng.normal(size=(K, d * (d + 1) // 2)), rng.random((n, d)), 1.0, 0)
    p = tmp_path / "gmm.txt"
    adbench.write_gmm_instance(p, inst)
    r = adbench.read_gmm_instance(p)
    for a in ("alphas", "means", "icf", "x"):
        assert np.array_equal(getattr(r, a), getattr(inst, a))     # repr() round-trips exactly
    assert (r.gamma, r.m, r.dims) == (1.0, 0, (d, K, n))
    adbench.write_gmm_instance(p, inst, replicate_point=True)
    r = adbench.read_gmm_instance(p, replicate_point=True)
    assert r.x.shape == (n, d) and (r.x == inst.x[0]).all()


def test_gmm_hand_written_instance(tmp_path):
    p = tmp_path / "gmm_d2_K1.txt"
    p.write_text("2 1 3\n0.5\n1 2\n0.1 0.2 0.3\n1 1\n2 2\n3 3\n1.0 0\n")
    r = adbench.read_gmm_instance(p)
    assert r.dims == (2, 1, 3) and r.icf.tolist() == [[0.1, 0.2, 0.3]]
    assert r.x.tolist() == [[1, 1], [2, 2], [3, 3]]
    with pytest.raises(ValueError):
        p.write_text("2 1 3\n0.5\n1 2\n")
        adbench.read_gmm_instance(p)


def test_ba_instance_adbench_replication(tmp_path):
    p = tmp_path / "ba1.txt"
    p.write_text("3 5 8\n" + " ".join(str(v) for v in range(11)) + "\n1 2 3\n0.75\n10 20\n")
    r = adbench.read_ba_instance(p)
    assert r.dims == (3, 5, 8)
    assert (r.cams == np.arange(11.0)).all() and (r.X == [1, 2, 3]).all()
    assert (r.w == 0.75).all() and (r.feats == [10, 20]).all()
    assert r.obs.dtype == np.int32
    assert r.obs.tolist() == [[i % 3, i % 5] for i in range(8)]
    adbench.write_ba_instance(p, r)
    r2 = adbench.read_ba_instance(p)
    assert all(np.array_equal(getattr(r, a), getattr(r2, a)) for a in ("cams", "X", "w", "feats",
                                                                         "obs"))


def test_ba_instance_full_round_trip(tmp_path):
    rng = np.random.default_rng(1)
    n, m, p_ = 4, 6, 9
    inst = adbench.BAInstance(rng.normal(size=(n, 11)), rng.normal(size=(m, 3)), rng.random(p_),
                              rng.random((p_, 2)) * 100,
                              np.stack([rng.integers(0, n, p_), rng.integers(0, m, p_)],
                                       1).astype(np.int32))
    path = tmp_path / "full.txt"
    adbench.write_ba_instance(path, inst, full=True)
    r = adbench.read_ba_instance(path)
    for a in ("cams", "X", "w", "feats", "obs"):
        assert np.array_equal(getattr(r, a), getattr(inst, a))


def dense_jacobian(n, m, obs, J31):
    """Direct statement of the BA Jacobian's structure: d[r_i]/d[params]."""
    p = obs.shape[0]
    D = np.zeros((3 * p, 11 * n + 3 * m + p))
    for i in range(p):
        c, q = obs[i]
        for r in range(2):
            row = J31[i, 15 * r:15 * r + 15]
            D[2 * i + r, 11 * c:11 * c + 11] = row[:11]
            D[2 * i + r, 11 * n + 3 * q:11 * n + 3 * q + 3] = row[11:14]
            D[2 * i + r, 11 * n + 3 * m + i] = row[14]
        D[2 * p + i, 11 * n + 3 * m + i] = J31[i, 30]
    return D


def test_oracle_ba_sparse_structure(golden):
    import scipy.sparse as sp
    rng = np.random.default_rng(2)
    n, m, p = 3, 4, 10
    obs = np.stack([rng.integers(0, n, p), rng.integers(0, m, p)], 1).astype(np.int32)
    J31 = rng.normal(size=(p, 31))
    rows, cols, vals, shape = ba_sparse(n, m, obs, J31)
    assert shape == (3 * p, 11 * n + 3 * m + p)
    assert rows.size == 3 * p + 1 and rows[-1] == 31 * p == cols.size == vals.size
    assert (np.diff(rows[:2 * p + 1]) == 15).all() and (np.diff(rows[2 * p:]) == 1).all()
    A = sp.csr_matrix((vals, cols, rows), shape=shape).toarray()
    assert np.array_equal(A, dense_jacobian(n, m, obs, J31))
    # the reference goldens' gradients through the same layout
    b = golden("ba")
    q = b["w"].size
    J = np.concatenate([b["J"].reshape(q, 30), b["wjac"][:, None]], 1)
    o = np.stack([np.arange(q), np.arange(q)], 1)
    rows, cols, vals, shape = ba_sparse(q, q, o, J)
    A = sp.csr_matrix((vals, cols, rows), shape=shape)
    assert np.array_equal(A.toarray(), dense_jacobian(q, q, o, J))


def test_J_files_round_trip(tmp_path):
    rng = np.random.default_rng(3)
    obs = np.array([[0, 1], [1, 0], [0, 0]], np.int32)
    rows, cols, vals, shape = ba_sparse(2, 2, obs, rng.normal(size=(3, 31)))

    class C:
        pass
    c = C()
    c.rows, c.cols, c.vals, c.shape = rows, cols, vals, shape
    adbench.write_J_sparse(tmp_path / "J.txt", c)
    r = adbench.read_J_sparse(tmp_path / "J.txt")
    assert np.array_equal(r[0], rows) and np.array_equal(r[1], cols)
    assert np.array_equal(r[2], vals) and r[3] == shape
    G = rng.normal(size=(1, 17))
    adbench.write_J(tmp_path / "g.txt", G)
    assert np.array_equal(adbench.read_J(tmp_path / "g.txt"), G)
