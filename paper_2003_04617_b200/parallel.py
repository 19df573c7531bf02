"""Data-parallel execution over one process per GPU (torchrun, NCCL).

The reference is single-process; here the batch is sharded:

* Bessel / BA: every element / observation is independent — each rank takes a
  contiguous slice and no collective touches the data path.
* GMM: each rank evaluates the per-point terms of its points into the packed
  vector [err, g_alphas, g_means, g_icf]; rank 0 also adds the
  parameter-only terms with the GLOBAL point count; ONE all_reduce(sum,
  float64) over NVLink combines them.
"""

import torch

from . import kernels


def shard_range(n, rank, world):
    """Contiguous [lo, hi) slice of n units for `rank` of `world` (sizes differ by <= 1)."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    return n * rank // world, n * (rank + 1) // world


def _dist():
    import torch.distributed as dist
    return dist if dist.is_available() and dist.is_initialized() else None


def gmm_grad_distributed(alphas, means, icf, x_local, gamma, m, cst, N_total, *, group=None,
                         local_fn=None, **kw):
    """GMM objective + gradient over points sharded across the process group.

    `x_local` is this rank's slice of the N_total points.  `local_fn` computes
    the rank's packed partial (default: the CUDA kernel, kernels.gmm_grad);
    the only collective is one all_reduce of that vector."""
    dist = _dist()
    rank = dist.get_rank(group) if dist else 0
    fn = local_fn or kernels.gmm_grad
    res = fn(alphas, means, icf, x_local, gamma, m, cst, N_total=N_total,
             add_param_terms=(rank == 0), **kw)
    packed = res.packed
    if dist is not None and dist.get_world_size(group) > 1:
        dist.all_reduce(packed, op=dist.ReduceOp.SUM, group=group)
    K, d = means.shape
    return kernels.unpack_gmm(packed, d, K, res.fail, res.counters)


def besselj_grad_sharded(z, nu=2, *, group=None, **kw):
    """Each rank differentiates its own slice; no collective."""
    return kernels.besselj_grad(z, nu, **kw)


def ba_jacobian_sharded(cams, X, w, feats, obs, *, group=None, **kw):
    """Cameras and points replicated, observations sharded; no collective."""
    return kernels.ba_jacobian(cams, X, w, feats, obs, **kw)


def allreduce_max(value, device=None):
    """max over ranks of a host scalar (timing: the slowest rank defines the step)."""
    dist = _dist()
    if dist is None or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
