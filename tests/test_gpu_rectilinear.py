"""Rectilinear-mesh sampler and decode (NEXT-4; R36) through the
C ABI vs the oracle: one-step gradients, node-lattice grid decode, mesh-mapped
queries, cache snapshots keep the mesh."""
import numpy as np
import pytest
import torch

import synth
from oracle import decode as o_decode, fit as o_fit, sampler
from oracle.model import InrModel
from paper_2304_10516_b200 import inr

from gpu_util import gpu_volume, get_grads, get_params, make_gpu_model, normwise, oracle_config, per_tensor_rel, \
    stream, whole_view
from test_gpu_parity import linear_regime

pytestmark = pytest.mark.gpu

NET = dict(levels=8, features=2, log2_table_size=14, mlp_hidden_layers=2)
DIMS = (33, 25, 17)


def stretched(n, seed):
    w = np.random.default_rng(seed).uniform(0.5, 2.0, n - 1)
    return np.concatenate([[0.0], np.cumsum(w)]) + 10.0


MESH = tuple(stretched(d, s) for d, s in zip(DIMS, (11, 12, 13)))


def volume():
    Z, Y, X = np.meshgrid(MESH[2], MESH[1], MESH[0], indexing="ij")
    return (np.sin(0.2 * X) * np.cos(0.15 * Y) + 0.1 * Z).astype(np.float32).astype(np.float64)


@pytest.mark.parametrize("bid", [0, 5])
def test_one_step_gradients_rectilinear_fp32(bid):
    vol = volume()
    blk = sampler.decompose(DIMS, (16, 16, 16), MESH)[bid]
    cfg = oracle_config(**NET)
    p0, lo, hi, om = linear_regime(cfg, blk, vol, 9, 1000, 200, np.random.default_rng(3))
    m = make_gpu_model(blk, 9, reduction=1, **NET)
    inr.inr_set_mesh(m, MESH)
    inr.inr_set_params(m, p0)
    go = inr.inr_fit_opts_default()
    go.vmin, go.vmax, go.boundary_batch = lo, hi, 200
    vt = gpu_volume(vol)
    rep = inr.inr_fit(m, whole_view(vt), 1, 1000, go, stream())
    l1u, l1b, _ = o_fit.train_step(om, vol, o_fit.FitOpts(vmin=lo, vmax=hi, boundary_batch=200), 1000)
    assert abs(rep.loss_uniform - l1u) <= 1e-5 * l1u
    err = per_tensor_rel(cfg, get_grads(m), om.g)
    print("rectilinear block", bid, "per-tensor grad rel err", err)
    assert err <= 1e-5
    inr.inr_destroy(m)


@pytest.mark.parametrize("prec,tol", [(0, 1e-5), (1, 2e-3)])
def test_rectilinear_decode_grid_and_queries(prec, tol):
    vol = volume()
    blocks = sampler.decompose(DIMS, (16, 16, 16), MESH)
    cfg = oracle_config(**NET)
    vt = gpu_volume(vol)
    go = inr.inr_fit_opts_default()
    go.vmin, go.vmax = float(vol.min()), float(vol.max())
    gms, oms = [], {}
    for b in blocks:
        m = make_gpu_model(b, 5, precision=prec, **NET)
        inr.inr_set_mesh(m, MESH)
        inr.inr_fit(m, whole_view(vt), 30, 512, go, stream())
        om = InrModel(cfg, b, 5, params=get_params(m))
        om.vmin, om.vmax = go.vmin, go.vmax
        gms.append(m)
        oms[b.block_id] = om
    # node lattice of every block, assembled into the global grid
    full = torch.full(DIMS[::-1], float("nan"), device="cuda")
    for m, b in zip(gms, blocks):
        o = b.origin
        cnt = tuple(min(16, DIMS[d] - o[d]) for d in range(3))
        inr.inr_decode_grid(m, (16, 16, 16), full[o[2]:, o[1]:, o[0]:].data_ptr(), (1, DIMS[0], DIMS[0] * DIMS[1]),
                            None, None, stream(), count=cnt)
    z, y, x = np.meshgrid(*[np.arange(d) for d in DIMS[::-1]], indexing="ij")
    nodes = np.stack([x.ravel(), y.ravel(), z.ravel()], 1).astype(np.float32)
    ref = o_decode.decode_query(oms, nodes).reshape(DIMS[::-1])
    torch.cuda.synchronize()
    assert not torch.isnan(full).any()
    assert normwise(full.cpu().numpy(), ref) <= tol
    # random (fractional) queries through the mesh map
    pts = synth.random_points(20000, DIMS)
    pd = torch.from_numpy(pts).cuda()
    q = torch.empty(pts.shape[0], device="cuda")
    inr.inr_decode_group(gms, pd.data_ptr(), pts.shape[0], q.data_ptr(), 1, stream())
    torch.cuda.synchronize()
    assert normwise(q.cpu().numpy(), o_decode.decode_query(oms, pts)) <= tol
    # grid decode at nodes == query decode at the same nodes, bitwise
    qn = torch.empty(nodes.shape[0], device="cuda")
    nd = torch.from_numpy(nodes).cuda()
    inr.inr_decode_group(gms, nd.data_ptr(), nodes.shape[0], qn.data_ptr(), 1, stream())
    torch.cuda.synchronize()
    assert torch.equal(qn.reshape(DIMS[::-1]), full)
    # a cache snapshot keeps the mesh
    c = inr.cache_create(2)
    inr.cache_insert(c, 0, gms, stream())
    _, snap = inr.cache_get(c, 0)
    q2 = torch.empty_like(q)
    inr.inr_decode_group(snap, pd.data_ptr(), pts.shape[0], q2.data_ptr(), 1, stream())
    torch.cuda.synchronize()
    assert torch.equal(q, q2)
    with pytest.raises(inr.InrError):
        inr.inr_decode_grid(gms[0], (32, 32, 32), full.data_ptr(), None, None, None, stream())
    inr.cache_destroy(c)
    for m in gms:
        inr.inr_destroy(m)
