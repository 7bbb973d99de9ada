"""Vector fields (D = 3; NEXT-2) through the C ABI vs the oracle:
forward, one-step gradients, decode grid / query, per-channel value range.
Same tolerances as the scalar path; R28."""
import numpy as np
import pytest
import torch

import synth
from oracle import decode as o_decode, fit as o_fit, sampler
from oracle.model import InrModel, init_params
from paper_2304_10516_b200 import inr

from gpu_util import gpu_volume, get_grads, get_params, make_gpu_model, normwise, oracle_config, per_tensor_rel, \
    stream, whole_view
from test_gpu_parity import _perturbed_params, componentwise_ratio, gradient_abs_bound, linear_regime

pytestmark = pytest.mark.gpu

V1 = dict(levels=8, features=2, log2_table_size=14, mlp_hidden_layers=2, out_dim=3)
V2 = dict(levels=16, features=2, log2_table_size=16, mlp_hidden_layers=3, out_dim=3)
V3 = dict(levels=16, features=4, log2_table_size=14, mlp_hidden_layers=4, out_dim=3)   # the paper's net, D = 3


def tgv(n=32, t=0.0):
    return synth.taylor_green_volume(n, t, amp=2.0).double().numpy()


@pytest.mark.parametrize("prec,tol", [(0, 1e-5), (1, 2e-3)])
@pytest.mark.parametrize("kw", [V1, V2, V3])
def test_forward_vector(kw, prec, tol):
    blk = sampler.decompose((64, 64, 64), (64, 64, 64))[0]
    cfg = oracle_config(**kw)
    m = make_gpu_model(blk, 4, precision=prec, **kw)
    p = _perturbed_params(cfg, blk, 4, np.random.default_rng(3))
    inr.inr_set_params(m, p)
    x = np.random.default_rng(2).random((3001, 3)).astype(np.float32)
    xd = torch.from_numpy(x).cuda()
    y = torch.full((3001, 3), float("nan"), device="cuda")
    inr.inr_debug_forward(m, xd.data_ptr(), 3001, y.data_ptr(), stream())
    torch.cuda.synchronize()
    yo, _ = o_fit.forward(InrModel(cfg, blk, 4, params=p), x)
    err = normwise(y.cpu().numpy(), yo)
    print(kw, prec, "forward err", err)
    assert err <= tol
    inr.inr_destroy(m)


@pytest.mark.parametrize("prec", [0, 1])
@pytest.mark.parametrize("kw", [V1, V3])
def test_one_step_gradients_vector(kw, prec):
    """Branch-free regime per channel (R27): fp32 per tensor <= 1e-5 (det);
    fp16 componentwise within 2(H+2) u g_abs."""
    vol = tgv()
    blk = sampler.decompose((32, 32, 32), (16, 16, 16))[6]
    cfg = oracle_config(**kw)
    p0, lo, hi, om = linear_regime(cfg, blk, vol, 9, 1000, 200, np.random.default_rng(17))
    opts = o_fit.FitOpts(vmin=lo, vmax=hi, boundary_batch=200)
    m = make_gpu_model(blk, 9, reduction=1, precision=prec, **kw)
    inr.inr_set_params(m, p0)
    vt = gpu_volume(vol)
    go = inr.inr_fit_opts_default()
    go.set_range(lo, hi)
    go.boundary_batch = 200
    rep = inr.inr_fit(m, whole_view(vt), 1, 1000, go, stream())
    l1u, l1b, _ = o_fit.train_step(om, vol, opts, 1000)
    ltol = 1e-5 if prec == 0 else 2e-3
    assert abs(rep.loss_uniform - l1u) <= ltol * l1u and abs(rep.loss_boundary - l1b) <= ltol * l1b
    g = get_grads(m)
    if prec == 0:
        err = per_tensor_rel(cfg, g, om.g)
        print(kw, "fp32 vector per-tensor grad err", err)
        assert err <= 1e-5
    else:
        r = componentwise_ratio(cfg, g, om.g, gradient_abs_bound(cfg, blk, 9, p0, vol, opts, 1000)) / 2.0 ** -11
        print(kw, "fp16 vector componentwise err / (u g_abs)", r)
        assert r <= 2 * (cfg.mlp_hidden_layers + 2)
    inr.inr_destroy(m)


@pytest.mark.parametrize("prec,tol", [(0, 1e-5), (1, 2e-3)])
def test_decode_vector_grid_and_query(prec, tol):
    vol = tgv(33)
    blocks = sampler.decompose((33, 33, 33), (16, 16, 16))        # 27 blocks, ragged last layer
    cfg = oracle_config(**V1)
    lo, hi = sampler.value_range([vol])
    vt = gpu_volume(vol)
    go = inr.inr_fit_opts_default()
    go.set_range(lo, hi)
    gms, oms = [], {}
    for b in blocks:
        m = make_gpu_model(b, 5, precision=prec, **V1)
        inr.inr_fit(m, whole_view(vt), 20, 512, go, stream())
        p = np.empty(inr.inr_param_count(m), np.float32)
        inr.inr_get_params(m, p)
        om = InrModel(cfg, b, 5, params=p)
        om.vmin, om.vmax = lo, hi
        gms.append(m)
        oms[b.block_id] = om
    for res in ((16, 16, 16), (7, 16, 3)):
        out = torch.full(res[::-1] + (3,), float("nan"), device="cuda")
        inr.inr_decode_grid(gms[4], res, out.data_ptr(), None, None, None, stream())
        torch.cuda.synchronize()
        ref = o_decode.decode_grid(oms[blocks[4].block_id], res)
        assert normwise(out.cpu().numpy(), ref) <= tol
    pts = synth.random_points(20000, (33, 33, 33))
    pd = torch.from_numpy(pts).cuda()
    q = torch.full((pts.shape[0], 3), float("nan"), device="cuda")
    inr.inr_decode_group(gms, pd.data_ptr(), pts.shape[0], q.data_ptr(), 1, stream())
    torch.cuda.synchronize()
    assert normwise(q.cpu().numpy(), o_decode.decode_query(oms, pts)) <= tol
    # a group without block 0: its points get NaN in all three channels, the others are untouched
    q2 = torch.full((pts.shape[0], 3), 7.0, device="cuda")
    inr.inr_decode_group(gms[1:], pd.data_ptr(), pts.shape[0], q2.data_ptr(), 0, stream())
    torch.cuda.synchronize()
    in0 = np.all(np.minimum(np.floor(pts / 16), 1) == 0, axis=1)
    q2n = q2.cpu().numpy()
    assert in0.any() and np.isnan(q2n[in0]).all() and np.array_equal(q2n[~in0], q.cpu().numpy()[~in0])
    # SSE against the ground truth at the nodes, pooled over channels in normalized units
    full = torch.empty((32, 32, 32, 3), device="cuda")
    sse = torch.zeros(1, dtype=torch.float64, device="cuda")
    ref_t = vt[:32, :32, :32].contiguous()
    for m, b in zip(gms, blocks):
        o = b.origin
        if max(o) >= 32:
            continue
        inr.inr_decode_grid(m, (16, 16, 16), full[o[2]:, o[1]:, o[0]:].data_ptr(), (3, 96, 3 * 1024),
                            ref_t[o[2]:, o[1]:, o[0]:].data_ptr(), sse.data_ptr(), stream())
    torch.cuda.synchronize()
    ref_sse = o_decode.sse_normalized(full.cpu().numpy(), vol[:32, :32, :32], lo, hi)   # w = 0: a constant channel
    assert np.isfinite(ref_sse) and abs(float(sse.item()) - ref_sse) <= 1e-5 * ref_sse
    for m in gms:
        inr.inr_destroy(m)


def test_value_range_per_channel():
    vol = tgv(20).astype(np.float32)
    vol[..., 2] = np.arange(20 ** 3, dtype=np.float32).reshape(20, 20, 20)
    vt = gpu_volume(vol)
    mm = torch.tensor([float("inf"), float("-inf")] * 3, device="cuda")
    inr.inr_value_range(whole_view(vt), mm.data_ptr(), stream())
    torch.cuda.synchronize()
    lo, hi = sampler.value_range([vol])
    assert np.array_equal(mm.cpu().numpy()[0::2], lo.astype(np.float32))
    assert np.array_equal(mm.cpu().numpy()[1::2], hi.astype(np.float32))


def test_view_channels_must_match():
    blk = sampler.decompose((16, 16, 16), (16, 16, 16))[0]
    m = make_gpu_model(blk, 1, **V1)
    vt = gpu_volume(synth.g1_analytic(16).numpy())
    go = inr.inr_fit_opts_default()
    with pytest.raises(inr.InrError):
        inr.inr_fit(m, whole_view(vt), 1, 64, go, stream())
    inr.inr_destroy(m)


def test_replica_channels_match_scalar_model_bitwise():
    """A D = 3 model whose output rows all equal a D = 1 model's row decodes to
    three copies of the scalar model's values, bit for bit (same per-channel
    arithmetic), on both precisions."""
    blk = sampler.decompose((32, 32, 32), (32, 32, 32))[0]
    for prec in (0, 1):
        s_kw = dict(V2, out_dim=1)
        c1, c3 = oracle_config(**s_kw), oracle_config(**V2)
        p1 = _perturbed_params(c1, blk, 2, np.random.default_rng(8))
        om1, om3 = InrModel(c1, blk, 2, params=p1), InrModel(c3, blk, 2)
        p3 = om3.p.astype(np.float32)
        for name, shape, off in c3.tensor_layout():
            src = om1.view(p1, name)
            om3.view(p3, name)[...] = np.broadcast_to(src, shape) if name in ("W3", "b3") else src
        m1 = make_gpu_model(blk, 2, precision=prec, **s_kw)
        m3 = make_gpu_model(blk, 2, precision=prec, **V2)
        inr.inr_set_params(m1, p1)
        inr.inr_set_params(m3, p3)
        o1 = torch.empty((32, 32, 32), device="cuda")
        o3 = torch.empty((32, 32, 32, 3), device="cuda")
        inr.inr_decode_grid(m1, (32, 32, 32), o1.data_ptr(), None, None, None, stream())
        inr.inr_decode_grid(m3, (32, 32, 32), o3.data_ptr(), None, None, None, stream())
        torch.cuda.synchronize()
        for c in range(3):
            assert torch.equal(o3[..., c], o1), (prec, c)
        inr.inr_destroy(m1)
        inr.inr_destroy(m3)


@pytest.mark.parametrize("prec", [0, 1])
def test_vector_deterministic_and_grouping_independent(prec):
    """D = 3 in the deterministic mode: two runs are bitwise equal, and a block
    fitted in a group equals the same block fitted alone (65 tiles per block)."""
    vol = tgv(32)
    blocks = sampler.decompose((32, 32, 32), (16, 16, 16))
    lo, hi = sampler.value_range([vol])
    go = inr.inr_fit_opts_default()
    go.set_range(lo, hi)
    go.boundary_batch = 64
    vt = gpu_volume(vol)
    runs = []
    for _ in range(2):
        group = [make_gpu_model(b, 4, reduction=1, precision=prec, **V1) for b in blocks]
        inr.inr_fit_group(group, [whole_view(vt)] * len(group), 4, 8192, go, stream())
        runs.append([get_params(m) for m in group])
        for m in group:
            inr.inr_destroy(m)
    assert all(np.array_equal(a, b) for a, b in zip(*runs))
    single = make_gpu_model(blocks[3], 4, reduction=1, precision=prec, **V1)
    inr.inr_fit(single, whole_view(vt), 4, 8192, go, stream())
    assert np.array_equal(get_params(single), runs[0][3])
    inr.inr_destroy(single)
