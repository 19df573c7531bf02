"""BA Jacobian in ADBench's BASparseMat CSR (rl_ba_jac_csr_f64, SURVEY §8(f)
rank 2).  Row pointers and column indices are integer work: bit-exact
against the oracle's restatement of BASparseMat.  Values: bit-identical to
the dense kernel (same arithmetic, re-strided), and within the dense
kernel's tolerance of the oracle."""

import numpy as np
import pytest
import torch

import paper_2003_04617_b200 as rg
from oracle import ba_jac, ba_sparse
from test_ba_gpu import ba_inputs, row_close, to_dev

pytestmark = pytest.mark.gpu


def dense_as_csr_vals(J):
    p = J.shape[0]
    return np.concatenate([J[:, :30].reshape(-1), J[:, 30]]) if p else np.empty(0)


@pytest.mark.parametrize("n_cams,n_pts,n_obs", [(7, 13, 1), (5, 11, 127), (17, 29, 1000),
                                                (40, 300, 20011)])
def test_csr_vs_oracle_and_dense(cuda, n_cams, n_pts, n_obs):
    rng = np.random.default_rng(n_obs)
    cams, X, w, feats, obs = ba_inputs(rng, n_cams, n_pts, n_obs)
    d = to_dev(cuda, cams, X, w, feats, obs)
    r = rg.ba_jacobian_csr(*d, want_err=True)
    dense = rg.ba_jacobian(*d)
    torch.cuda.synchronize()
    Jd = dense.J.cpu().numpy()
    assert np.array_equal(r.vals.cpu().numpy(), dense_as_csr_vals(Jd))     # bit-identical
    assert torch.equal(r.err, dense.err) and torch.equal(r.fail, dense.fail)
    Jo, _, fo = ba_jac(cams, X, w, feats, obs)
    rows, cols, vals, shape = ba_sparse(n_cams, n_pts, obs, Jo)
    assert r.shape == shape
    assert np.array_equal(r.rows.cpu().numpy(), rows)                       # integer: exact
    assert np.array_equal(r.cols.cpu().numpy(), cols)
    assert np.array_equal(r.fail.cpu().numpy(), fo)
    ok = row_close(Jd, Jo).all()
    assert ok
    # the scipy matrix of the device result equals the oracle's
    A = r.to_scipy()
    assert A.shape == shape and A.nnz == 31 * n_obs


def test_csr_values_only(cuda):
    rng = np.random.default_rng(5)
    d = to_dev(cuda, *ba_inputs(rng, 9, 20, 3000))
    a = rg.ba_jacobian_csr(*d)
    b = rg.ba_jacobian_csr(*d, pattern=False)
    torch.cuda.synchronize()
    assert b.rows is None and b.cols is None and torch.equal(a.vals, b.vals)


def test_csr_shards_concatenate(cuda):
    """Two shards (obs_offset, n_obs_total) reassemble into the whole matrix."""
    rng = np.random.default_rng(6)
    n_cams, n_pts, P = 11, 23, 5001
    cams, X, w, feats, obs = ba_inputs(rng, n_cams, n_pts, P)
    whole = rg.ba_jacobian_csr(*to_dev(cuda, cams, X, w, feats, obs))
    cut = 2222
    parts = [rg.ba_jacobian_csr(*to_dev(cuda, cams, X, w[a:b], feats[a:b], obs[a:b]),
                                obs_offset=a, n_obs_total=P) for a, b in ((0, cut), (cut, P))]
    torch.cuda.synchronize()
    for name, k in (("vals", 30), ("cols", 30)):
        rp = [getattr(p_, name).cpu().numpy() for p_ in parts]
        m = [cut, P - cut]
        cat = np.concatenate([rp[0][:k * m[0]], rp[1][:k * m[1]], rp[0][k * m[0]:],
                              rp[1][k * m[1]:]])
        assert np.array_equal(cat, getattr(whole, name).cpu().numpy()), name
    rp = [p_.rows.cpu().numpy() for p_ in parts]
    cat = np.concatenate([rp[0][:2 * cut], rp[1][:2 * (P - cut)], rp[0][2 * cut:-1],
                          rp[1][2 * (P - cut):]])
    assert np.array_equal(cat, whole.rows.cpu().numpy())
    assert parts[0].shape == parts[1].shape == whole.shape


def test_csr_host_entry(cuda):
    rng = np.random.default_rng(7)
    cams, X, w, feats, obs = ba_inputs(rng, 30, 400, (1 << 18) + 4097)   # > 1 pipeline chunk
    h = rg.ba_jacobian_csr_host(cams, X, w, feats, obs)
    d = rg.ba_jacobian_csr(*to_dev(cuda, cams, X, w, feats, obs))
    torch.cuda.synchronize()
    assert np.array_equal(h.rows, d.rows.cpu().numpy())
    assert np.array_equal(h.cols, d.cols.cpu().numpy())
    assert np.array_equal(h.vals, d.vals.cpu().numpy())
    assert h.counters == 0


def test_csr_bad_index_and_limits(cuda):
    rng = np.random.default_rng(8)
    cams, X, w, feats, obs = ba_inputs(rng, 4, 6, 50)
    obs[3] = (9, 0)                                        # camera out of range
    r = rg.ba_jacobian_csr(*to_dev(cuda, cams, X, w, feats, obs))
    torch.cuda.synchronize()
    fail = r.fail.cpu().numpy()
    assert fail[3] == 8 and (np.delete(fail, 3) == 0).all()   # IndexOutOfBounds
    cols = r.cols.cpu().numpy()
    assert (cols[90:90 + 14] == -1).all() and (cols[105:105 + 14] == -1).all()
    with pytest.raises(rg.NativeLibraryError):
        rg.ba_jacobian_csr(*to_dev(cuda, cams, X, w, feats, obs), obs_offset=0,
                           n_obs_total=(1 << 31) // 31 + 1)


def test_adbench_file_to_jacobian_file(cuda, tmp_path):
    from paper_2003_04617_b200 import adbench
    p = tmp_path / "ba_small.txt"
    p.write_text("3 5 40\n0.1 -0.2 0.05 0.3 0.1 -0.4 550 0.5 0.5 0.001 -0.002\n"
                 "0.2 -0.1 10.5\n0.8\n40.5 60.25\n")
    inst = adbench.read_ba_instance(p)
    r = rg.ba_jacobian_csr_host(inst.cams, inst.X, inst.w, inst.feats, inst.obs)
    adbench.write_J_sparse(tmp_path / "J.txt", r)
    rows, cols, vals, shape = adbench.read_J_sparse(tmp_path / "J.txt")
    Jo, _, _ = ba_jac(inst.cams, inst.X, inst.w, inst.feats, inst.obs)
    ro, co, vo, so = ba_sparse(3, 5, inst.obs, Jo)
    assert shape == so and np.array_equal(rows, ro) and np.array_equal(cols, co)
    assert np.allclose(vals, vo, rtol=1e-10, atol=1e-13 * np.abs(vo).max())
