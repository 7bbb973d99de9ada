"""CUDA path vs oracle, element by element on the same seeded inputs
(SURVEY.md §8(c) parity contract).  All calls go through the C ABI."""
import numpy as np
import pytest
import torch

import synth
from oracle import adam as o_adam, decode as o_decode, encoding as o_enc, fit as o_fit, sampler
from oracle.model import InrModel, init_params
from paper_2304_10516_b200 import inr

from gpu_util import (gpu_volume, get_grads, get_params, make_gpu_model, normwise, oracle_config, per_tensor_rel,
                      stream, whole_view)

pytestmark = pytest.mark.gpu

CFG1 = dict(levels=8, features=2, log2_table_size=14, mlp_hidden_layers=2)
CFG2 = dict(levels=16, features=2, log2_table_size=19, mlp_hidden_layers=3)


@pytest.mark.parametrize("kw", [CFG1, CFG2, dict(levels=4, features=4, log2_table_size=12, mlp_hidden_layers=1),
                                dict(levels=6, features=1, log2_table_size=10, mlp_hidden_layers=2, mlp_bias=0)])
def test_init_bitwise(kw):
    blk = sampler.decompose((64, 64, 64), (32, 32, 32))[5]
    m = make_gpu_model(blk, 77, **kw)
    try:
        assert np.array_equal(get_params(m), init_params(oracle_config(**kw), 77, blk.block_id))
    finally:
        inr.inr_destroy(m)


@pytest.mark.parametrize("kw", [CFG1, CFG2, dict(levels=8, features=8, log2_table_size=16, mlp_hidden_layers=1),
                                dict(levels=12, features=1, log2_table_size=12, mlp_hidden_layers=1),
                                dict(CFG2, log2_table_size=22)])                  # cfg5's table size
def test_encode_indices_bitexact_features_1e5(kw):
    blk = sampler.decompose((64, 64, 64), (64, 64, 64))[0]
    m = make_gpu_model(blk, 3, **kw)
    cfg = oracle_config(**kw)
    rng = np.random.default_rng(1)
    p = rng.normal(size=cfg.param_count()).astype(np.float32)
    inr.inr_set_params(m, p)
    lat = np.stack(np.meshgrid(*[np.arange(9) / 8.0] * 3, indexing="ij"), -1).reshape(-1, 3)
    x = np.concatenate([rng.random((5000, 3)), lat, [[1, 1, 1], [0, 0, 0], [1 - 2 ** -24] * 3]]).astype(np.float32)
    q = x.shape[0]
    xd = torch.from_numpy(x).cuda()
    idx = torch.zeros(q * cfg.levels * 8, dtype=torch.int32, device="cuda")
    feat = torch.zeros(q * cfg.levels * cfg.features, dtype=torch.float32, device="cuda")
    inr.inr_debug_encode(m, xd.data_ptr(), q, idx.data_ptr(), feat.data_ptr(), stream())
    torch.cuda.synchronize()
    om = InrModel(cfg, blk, 3, params=p)
    f_o, idx_o, _ = o_enc.encode_forward(om.tables(), x, cfg.resolutions(), cfg.table_size)
    assert np.array_equal(idx.cpu().numpy().view(np.uint32).reshape(q, cfg.levels, 8), idx_o)
    assert normwise(feat.cpu().numpy().reshape(q, -1), f_o) <= 1e-5
    inr.inr_destroy(m)


def test_forward_fp32_1e5():
    blk = sampler.decompose((64, 64, 64), (64, 64, 64))[0]
    for kw in (CFG1, CFG2):
        cfg = oracle_config(**kw)
        m = make_gpu_model(blk, 4, **kw)
        rng = np.random.default_rng(2)
        p = init_params(cfg, 4, 0)
        p[: sum(cfg.level_sizes()) * cfg.features] = rng.uniform(-1, 1, sum(cfg.level_sizes()) * cfg.features)
        inr.inr_set_params(m, p)
        x = rng.random((3000, 3)).astype(np.float32)
        xd = torch.from_numpy(x).cuda()
        y = torch.zeros(3000, device="cuda")
        inr.inr_debug_forward(m, xd.data_ptr(), 3000, y.data_ptr(), stream())
        torch.cuda.synchronize()
        yo, _ = o_fit.forward(InrModel(cfg, blk, 4, params=p), x)
        assert normwise(y.cpu().numpy(), yo[:, 0]) <= 1e-5
        inr.inr_destroy(m)


def _perturbed_params(cfg, blk, seed, rng):
    """Init parameters with O(0.1) tables and biases, so pre-activations sit
    well away from the ReLU kink (at init the tables are ~1e-4)."""
    p = init_params(cfg, seed, blk.block_id)
    for name, shape, off in cfg.tensor_layout():
        n = int(np.prod(shape))
        if name.startswith("table") or name.startswith("b"):
            p[off:off + n] = rng.uniform(-0.1, 0.1, n)
    return p


def _clean_seed(cfg, blk, vol, opts, batch, seeds, params, margin=1e-6):
    """First seed whose step-0 batch keeps every |y - t| and every hidden
    pre-activation at least `margin` away from the L1 / ReLU kinks, where GPU
    fp32 and oracle fp64 could legitimately branch differently."""
    for s in seeds:
        om = InrModel(cfg, blk, s, params=params)
        x_u, x_b, t_u, t_b, _ = o_fit.step_batch(om, vol, opts, batch)
        x = np.concatenate([x_u, x_b])
        y, cache = o_fit.forward(om, x)
        t = np.concatenate([t_u, t_b])
        zmin = min(float(np.min(np.abs(z))) for z in cache[3][:-1])
        if float(np.min(np.abs(y[:, 0] - t))) > margin and zmin > margin:
            return s, om
    pytest.skip("no clean seed found")


def _adam_reference(p0, g, lr=1e-2):
    """The oracle's Adam (PyTorch form, pinned in test_oracle_pins) applied to the
    GPU's own gradients: isolates the Adam kernel from gradient rounding, which
    Adam amplifies by lr/eps = 1e6 for |g| ~ eps."""
    p = p0.astype(np.float64).copy()
    m, v = np.zeros_like(p), np.zeros_like(p)
    o_adam.adam_update(p, g.astype(np.float64), m, v, 1, lr)
    return p, m, v


@pytest.mark.parametrize("det,tol", [(1, 1e-5), (0, 1e-5)])   # measured 4.4e-7 in both modes (north_star bound: 1e-4)
def test_one_step_gradients_and_adam_fp32(det, tol):
    """Gradients of one fit step in the fp32 mode: per tensor
    ||d||_inf/||ref||_inf <= 1e-4 with the deterministic reduction (north_star),
    1e-5 with fp32 atomics (measured 4.4e-7); the Adam update of those gradients to 1e-6."""
    dims = (32, 32, 32)
    vol = synth.g1_analytic(32).numpy()
    blk = sampler.decompose(dims, (16, 16, 16))[3]          # has interior faces -> boundary term
    lo, hi = sampler.value_range([vol])
    opts = o_fit.FitOpts(vmin=lo, vmax=hi, boundary_batch=128)
    cfg = oracle_config(**CFG1)
    p0 = _perturbed_params(cfg, blk, 1, np.random.default_rng(0))
    seed, om = _clean_seed(cfg, blk, vol, opts, 512, range(100, 200), p0)
    m = make_gpu_model(blk, seed, reduction=det, **CFG1)
    inr.inr_set_params(m, p0)
    vt = gpu_volume(vol)
    go = inr.inr_fit_opts_default()
    go.vmin, go.vmax, go.boundary_batch = lo, hi, 128
    rep = inr.inr_fit(m, whole_view(vt), 1, 512, go, stream())
    l1u, l1b, _ = o_fit.train_step(om, vol, opts, 512)
    g = get_grads(m)
    err = per_tensor_rel(cfg, g, om.g)
    print("per-tensor grad rel err", err)
    assert err <= tol
    assert abs(rep.loss_uniform - l1u) <= 1e-5 * l1u and abs(rep.loss_boundary - l1b) <= 1e-5 * l1b
    pe, me, ve = _adam_reference(p0, g)
    mg, vg = inr.inr_get_adam_state(m, np.empty_like(g), np.empty_like(g))
    assert np.max(np.abs(get_params(m) - pe)) <= 1e-6 * 1e-2 + 1e-7 * np.abs(pe).max()
    assert np.allclose(mg, me, rtol=1e-6, atol=0) and np.allclose(vg, ve, rtol=1e-5, atol=1e-30)
    inr.inr_destroy(m)


def linear_regime(cfg, blk, vol, seed, batch, boundary_batch, rng):
    """Parameters and a value range for which one fit step is branch-free on
    both sides (R27): O(0.1) tables; biases set layer by layer to
    max_batch |W_k h_{k-1}| + 1, so every hidden pre-activation of the step's
    batch is >= 1 (all ReLUs active, no kink within any rounding); and
    (vmin, vmax) placing every target at least 1 + 1% of max|y| below its
    output (sgn(y - t) = +1).  Bias-free nets get positive tables and weights
    instead.  Returns (params float32, vmin, vmax, oracle model)."""
    p = _perturbed_params(cfg, blk, 1, rng).astype(np.float32)
    om = InrModel(cfg, blk, seed, params=p)
    x_u, x_b, _, _, _ = o_fit.step_batch(om, vol, o_fit.FitOpts(boundary_batch=boundary_batch), batch)
    x = np.concatenate([x_u, x_b])
    H = cfg.mlp_hidden_layers
    if not cfg.mlp_bias:
        for name, shape, off in cfg.tensor_layout():
            n = int(np.prod(shape))
            p[off:off + n] = np.abs(p[off:off + n]) + (np.float32(0.01) if name.startswith("table") else 0)
    else:
        for k in range(H):
            _, cache = o_fit.forward(InrModel(cfg, blk, seed, params=p), x)
            b = om.view(p, f"b{k}")
            pre = cache[3][k] - b.astype(np.float64)[None, :]
            b[...] = (np.abs(pre).max(axis=0) + 1.0).astype(np.float32)
        om.view(p, f"b{H}")[...] = 0.0
    om = InrModel(cfg, blk, seed, params=p)
    y, cache = o_fit.forward(om, x)
    assert all(float(z.min()) >= 0.5 for z in cache[3][:-1]) or not cfg.mlp_bias
    assert all(float(z.min()) > 0 for z in cache[3][:-1])
    if vol.ndim == 4:    # vector field: per-channel ranges
        lo = vol.max(axis=(0, 1, 2)).astype(np.float64) - y.min(axis=0) + 1.0 + 0.01 * np.abs(y).max(axis=0)
        return p, lo, lo + 1.0, om
    lo = float(vol.max()) - float(y.min()) + 1.0 + 0.01 * float(np.abs(y).max())
    return p, lo, lo + 1.0, om


def gradient_abs_bound(cfg, blk, seed, p, vol, opts, batch):
    """The oracle's gradient of the same step with every parameter replaced by
    its absolute value (dy > 0 and all ReLUs active in the linear regime):
    the |W_k|...|dy| products that bound a rounded evaluation componentwise,
    |fl(g) - g| <= kappa * u * g_abs (the standard error bound of a chain of
    matrix products, e.g. Higham, Accuracy and Stability, Sec. 3.5)."""
    oa = InrModel(cfg, blk, seed, params=np.abs(p))
    oa.vmin, oa.vmax = opts.vmin, opts.vmax
    o_fit.train_step(oa, vol, opts, batch)
    return oa.g


def componentwise_ratio(cfg, g, g_ref, g_abs):
    """max |g - g_ref| / g_abs over entries some sample touched (untouched
    entries must be exactly zero on both sides)."""
    nz = g_abs > 0
    assert np.all(g[~nz] == 0) and np.all(g_ref[~nz] == 0)
    return float(np.max(np.abs(g[nz] - g_ref[nz]) / g_abs[nz]))


PAPER_NET = dict(levels=16, features=4, log2_table_size=14, mlp_hidden_layers=4)   # P:L217-218 (T scaled down)
ARCHS = [CFG1, PAPER_NET, dict(levels=4, features=8, log2_table_size=12, mlp_hidden_layers=1),
         dict(levels=16, features=1, log2_table_size=12, mlp_hidden_layers=3, mlp_bias=0)]


@pytest.mark.parametrize("arch", range(len(ARCHS)))
@pytest.mark.parametrize("prec", [0, 1])
def test_gradients_linear_regime_architectures(arch, prec):
    """Branch-free one-step gradient parity across encodings and MLP depths,
    including the paper's own 16 levels x 4 features, 4 x 64 MLP.
    fp32: per tensor <= 1e-5.  fp16 tensor-core MLP: componentwise within the
    first-order rounding bound 2(H+2) u g_abs, u = 2^-11 (fp16 features,
    weights, activations and dz, H+1 GEMMs each way) -- per-tensor norms are
    no bound here, since dfeat = W0^T dz0 cancels (R27)."""
    kw = ARCHS[arch]
    vol = synth.g2_energy(32).numpy()
    blk = sampler.decompose((32, 32, 32), (16, 16, 16))[6]
    cfg = oracle_config(**kw)
    p0, lo, hi, om = linear_regime(cfg, blk, vol, 9, 1000, 200, np.random.default_rng(7 + arch))
    opts = o_fit.FitOpts(vmin=lo, vmax=hi, boundary_batch=200)
    m = make_gpu_model(blk, 9, reduction=1, precision=prec, **kw)
    inr.inr_set_params(m, p0)
    vt = gpu_volume(vol)
    go = inr.inr_fit_opts_default()
    go.vmin, go.vmax, go.boundary_batch = lo, hi, 200
    inr.inr_fit(m, whole_view(vt), 1, 1000, go, stream())
    om.vmin, om.vmax = lo, hi
    o_fit.train_step(om, vol, opts, 1000)
    g = get_grads(m)
    if prec == 0:
        err = per_tensor_rel(cfg, g, om.g)
        print(kw, "fp32 per-tensor grad rel err", err)
        assert err <= 1e-5
    else:
        g_abs = gradient_abs_bound(cfg, blk, 9, p0, vol, opts, 1000)
        r = componentwise_ratio(cfg, g, om.g, g_abs) / 2.0 ** -11
        print(kw, "fp16 componentwise err / (u g_abs)", r, "bound", 2 * (cfg.mlp_hidden_layers + 2))
        assert r <= 2 * (cfg.mlp_hidden_layers + 2)
    inr.inr_destroy(m)


@pytest.mark.parametrize("prec", [0, 1])
def test_one_step_gradients_linear_regime(prec):
    """Flip-free gradient parity (targets far below the outputs: sgn(y-t) = +1
    everywhere; all ReLUs active).  Isolates the backward arithmetic of the fp16
    tensor-core MLP (fp16 operands, fp32 TMEM accumulation, 2^k loss scaling),
    whose realistic-batch comparison is dominated by legitimate L1/ReLU branch
    flips of samples within fp16 rounding of a kink (R27).  fp32: per
    tensor <= 1e-5; fp16: componentwise <= 2(H+2) u g_abs (R27)."""
    vol = synth.g1_analytic(32).numpy()
    blk = sampler.decompose((32, 32, 32), (16, 16, 16))[3]
    cfg = oracle_config(**CFG1)
    p0, lo, hi, om = linear_regime(cfg, blk, vol, 7, 1000, 128, np.random.default_rng(5))
    om.vmin, om.vmax = lo, hi
    opts = o_fit.FitOpts(vmin=lo, vmax=hi, boundary_batch=128)
    m = make_gpu_model(blk, 7, reduction=1, precision=prec, **CFG1)
    inr.inr_set_params(m, p0)
    vt = gpu_volume(vol)
    go = inr.inr_fit_opts_default()
    go.vmin, go.vmax, go.boundary_batch = lo, hi, 128
    inr.inr_fit(m, whole_view(vt), 1, 1000, go, stream())
    o_fit.train_step(om, vol, opts, 1000)
    g = get_grads(m)
    if prec == 0:
        err = per_tensor_rel(cfg, g, om.g)
        print("fp32 per-tensor grad rel err", err)
        assert err <= 1e-5
    else:
        g_abs = gradient_abs_bound(cfg, blk, 7, p0, vol, opts, 1000)
        r = componentwise_ratio(cfg, g, om.g, g_abs) / 2.0 ** -11
        print("fp16 componentwise err / (u g_abs)", r, "per-tensor", per_tensor_rel(cfg, g, om.g))
        assert r <= 2 * (cfg.mlp_hidden_layers + 2)
    inr.inr_destroy(m)


def test_forward_fp16_tensor_core_2e3():
    """The tcgen05 fp16 MLP (fp32 accumulate) within 2e-3 normwise (north_star)."""
    blk = sampler.decompose((64, 64, 64), (64, 64, 64))[0]
    for kw in (CFG1, CFG2, dict(levels=16, features=4, log2_table_size=14, mlp_hidden_layers=4),
               dict(levels=24, features=2, log2_table_size=12, mlp_hidden_layers=1, mlp_bias=0)):
        cfg = oracle_config(**kw)
        m = make_gpu_model(blk, 4, precision=1, **kw)
        p = _perturbed_params(cfg, blk, 4, np.random.default_rng(3))
        inr.inr_set_params(m, p)
        x = np.random.default_rng(2).random((3001, 3)).astype(np.float32)
        xd = torch.from_numpy(x).cuda()
        y = torch.full((3001,), float("nan"), device="cuda")
        inr.inr_debug_forward(m, xd.data_ptr(), 3001, y.data_ptr(), stream())
        torch.cuda.synchronize()
        yo, _ = o_fit.forward(InrModel(cfg, blk, 4, params=p), x)
        err = normwise(y.cpu().numpy(), yo[:, 0])
        print(kw, "fp16 forward normwise err", err)
        assert err <= 2e-3
        inr.inr_destroy(m)


@pytest.mark.parametrize("prec", [0, 1])
def test_deterministic_mode_bitwise_reproducible(prec):
    vol = synth.g1_analytic(32).numpy()
    blk = sampler.decompose((32, 32, 32), (16, 16, 16))[0]
    vt = gpu_volume(vol)
    go = inr.inr_fit_opts_default()
    go.vmin, go.vmax, go.boundary_batch = float(vol.min()), float(vol.max()), 256
    out = []
    for _ in range(2):
        m = make_gpu_model(blk, 5, reduction=1, precision=prec, **CFG1)
        inr.inr_fit(m, whole_view(vt), 5, 1024, go, stream())
        out.append((get_params(m), get_grads(m)))
        inr.inr_destroy(m)
    assert np.array_equal(out[0][0], out[1][0]) and np.array_equal(out[0][1], out[1][1])


@pytest.mark.parametrize("prec", [0, 1])
def test_adam_elementwise_across_lr_decays(prec):
    """Adam + the step schedule (R12, R13) element by element over 8
    steps that cross two learning-rate decays (lr_step = 3: lr = 1e-2 at
    s = 0-2, 8e-3 at s = 3-5, 6.4e-3 at s = 6-7) with the bias corrections of
    every t = 1..8.  Each step's GPU gradient is fed to the oracle's Adam
    (pinned against torch.optim.Adam in test_oracle_pins), which carries its
    own float64 (p, m, v); the GPU's fp32 state must track it to fp32 rounding.
    The same 8 steps as one call (the CUDA-graph path) end bitwise equal."""
    vol = synth.g1_analytic(32).numpy()
    blk = sampler.decompose((32, 32, 32), (16, 16, 16))[3]
    lo, hi = sampler.value_range([vol])
    go = inr.inr_fit_opts_default()
    go.vmin, go.vmax, go.boundary_batch, go.lr_step = lo, hi, 128, 3
    vt = gpu_volume(vol)
    m = make_gpu_model(blk, 8, reduction=1, precision=prec, **CFG1)
    p = get_params(m).astype(np.float64)
    mo, vo = np.zeros_like(p), np.zeros_like(p)
    gmax = np.zeros_like(p)
    worst = [0.0, 0.0, 0.0]
    for t in range(1, 9):
        inr.inr_fit(m, whole_view(vt), 1, 512, go, stream())
        g = get_grads(m).astype(np.float64)
        assert np.any(g != 0)
        gmax = np.maximum(gmax, np.abs(g))
        o_adam.adam_update(p, g, mo, vo, t, o_adam.lr_at(t - 1, 1e-2, 0.8, 3))
        pg = get_params(m)
        mg, vg = inr.inr_get_adam_state(m, np.empty_like(pg), np.empty_like(pg))
        # fp32 rounding of t fused updates: relative 2^-23 per operation, a few per step
        tol_p = t * (1e-6 * 1e-2 + 2.0 ** -21 * np.abs(p))
        tol_m = t * 2.0 ** -21 * gmax
        tol_v = t * 2.0 ** -21 * vo + 1e-37
        r = [float(np.max(np.abs(pg - p) / tol_p)), float(np.max(np.abs(mg - mo) / tol_m.clip(1e-30))),
             float(np.max(np.abs(vg - vo) / tol_v))]
        worst = [max(a, b) for a, b in zip(worst, r)]
        assert r[0] <= 1 and r[1] <= 1 and r[2] <= 1, (t, r)
    print("prec", prec, "worst |p|,|m|,|v| error / tolerance over t = 1..8:", worst)
    assert inr.inr_steps(m) == 8
    b = make_gpu_model(blk, 8, reduction=1, precision=prec, **CFG1)
    inr.inr_fit(b, whole_view(vt), 8, 512, go, stream())
    assert np.array_equal(get_params(b), get_params(m))
    inr.inr_destroy(m)
    inr.inr_destroy(b)


@pytest.mark.parametrize("prec", [0, 1])
def test_sparse_adam_elementwise(prec):
    """R37 (NEXT-4 touched-only Adam, opts.sparse_adam): each step's GPU
    gradient fed to the oracle's adam_update_sparse (pinned in test_oracle_pins)
    over 6 steps; table groups of 8 floats without a non-zero gradient keep p, m,
    v bitwise on the GPU, the rest track the oracle to fp32 rounding.  A small
    batch against T = 2^14 leaves most hashed-level groups untouched."""
    vol = synth.g1_analytic(32).numpy()
    blk = sampler.decompose((32, 32, 32), (16, 16, 16))[3]
    lo, hi = sampler.value_range([vol])
    go = inr.inr_fit_opts_default()
    go.vmin, go.vmax, go.boundary_batch, go.sparse_adam = lo, hi, 64, 1
    cfg = oracle_config(**CFG1)
    tables = [(off, int(np.prod(shape))) for name, shape, off in cfg.tensor_layout() if name.startswith("table")]
    vt = gpu_volume(vol)
    m = make_gpu_model(blk, 8, reduction=1, precision=prec, **CFG1)
    p = get_params(m).astype(np.float64)
    mo, vo = np.zeros_like(p), np.zeros_like(p)
    gmax = np.zeros_like(p)
    untouched_seen = 0
    for t in range(1, 7):
        prev = get_params(m)
        inr.inr_fit(m, whole_view(vt), 1, 256, go, stream())
        g = get_grads(m).astype(np.float64)
        gmax = np.maximum(gmax, np.abs(g))
        o_adam.adam_update_sparse(p, g, mo, vo, t, 1e-2, tables)
        pg = get_params(m)
        mg, vg = inr.inr_get_adam_state(m, np.empty_like(pg), np.empty_like(pg))
        keep = np.ones(p.shape, bool)
        for off, n in tables:
            keep[off:off + n] = ~o_adam.touched_groups(g[off:off + n])
        keep[tables[-1][0] + tables[-1][1]:] = False
        untouched_seen += int(keep.sum())
        assert np.array_equal(pg[keep], prev[keep])            # untouched groups: bitwise unchanged
        tol_p = t * (1e-6 * 1e-2 + 2.0 ** -21 * np.abs(p))
        assert np.all(np.abs(pg - p) <= tol_p)
        assert np.all(np.abs(mg - mo) <= t * 2.0 ** -21 * gmax + 1e-30)
        assert np.all(np.abs(vg - vo) <= t * 2.0 ** -21 * vo + 1e-37)
    print("prec", prec, "untouched parameter-steps", untouched_seen, "of", 6 * p.size)
    assert untouched_seen > p.size        # the variant skipped a substantial part of the table
    inr.inr_destroy(m)


@pytest.mark.parametrize("prec", [0, 1])
def test_probe_psnr_matches_oracle(prec):
    """The stop check's probe PSNR ("until the user-defined accuracy
    criterion (such as a PSNR target)"): the GPU's 32^3 probe SSE, as
    reported in inr_fit_report.probe_psnr, equals oracle.fit.probe_psnr of the
    same (GPU-trained) parameters to 1e-5 dB.  The probe evaluates the fp32
    parameters in fp32 in both precision modes."""
    vol = synth.g2_energy(32).numpy()
    blk = sampler.decompose((32, 32, 32), (16, 16, 16))[5]
    lo, hi = sampler.value_range([vol])
    go = inr.inr_fit_opts_default()
    go.vmin, go.vmax, go.boundary_batch = lo, hi, 256
    go.target_psnr, go.check_interval = 500.0, 5                # never reached: the check at step 10 reports
    m = make_gpu_model(blk, 4, precision=prec, **CFG1)
    vt = gpu_volume(vol)
    rep = inr.inr_fit(m, whole_view(vt), 10, 2048, go, stream())
    assert rep.steps_taken == 10 and rep.reached_target == 0
    om = InrModel(oracle_config(**CFG1), blk, 4, params=get_params(m))
    want = o_fit.probe_psnr(om, vol, o_fit.FitOpts(vmin=lo, vmax=hi))
    print("prec", prec, "probe psnr gpu", rep.probe_psnr, "oracle", want, "diff", rep.probe_psnr - want)
    assert 15.0 < want < 60.0
    assert abs(rep.probe_psnr - want) <= 1e-5          # measured 7e-7 dB
    inr.inr_destroy(m)


@pytest.mark.parametrize("lam", [0.0, 0.25, 1.0])
@pytest.mark.parametrize("prec", [0, 1])
def test_gradients_linear_regime_lambda(lam, prec):
    """Eq. 2 weighting away from lambda = 1/2 (P:L209 studies
    lambda): with boundary samples present, dL/dy = (1 - lambda)/|U| on uniform
    and lambda/|B| on boundary samples (pinned by central differences in
    test_oracle_pins), so a swap of the two weights -- invisible at 1/2 --
    changes every gradient here.  Branch-free regime (R27): fp32 per tensor
    <= 1e-5, fp16 componentwise <= 2(H+2) u g_abs."""
    vol = synth.g2_energy(32).numpy()
    blk = sampler.decompose((32, 32, 32), (16, 16, 16))[6]
    cfg = oracle_config(**CFG1)
    p0, lo, hi, om = linear_regime(cfg, blk, vol, 9, 1000, 200, np.random.default_rng(17))
    opts = o_fit.FitOpts(vmin=lo, vmax=hi, boundary_batch=200, lam=lam)
    m = make_gpu_model(blk, 9, reduction=1, precision=prec, **CFG1)
    inr.inr_set_params(m, p0)
    vt = gpu_volume(vol)
    go = inr.inr_fit_opts_default()
    go.vmin, go.vmax, go.boundary_batch, go.lambda_ = lo, hi, 200, lam
    rep = inr.inr_fit(m, whole_view(vt), 1, 1000, go, stream())
    om.vmin, om.vmax = lo, hi
    l1u, l1b, _ = o_fit.train_step(om, vol, opts, 1000)
    tl = 1e-5 if prec == 0 else 2e-3          # the L1 terms: fp32 forward 1e-5, fp16 MLP 2e-3 (north_star)
    assert abs(rep.loss_uniform - l1u) <= tl * l1u and abs(rep.loss_boundary - l1b) <= tl * l1b
    g = get_grads(m)
    if prec == 0:
        err = per_tensor_rel(cfg, g, om.g)
        print("lambda", lam, "fp32 per-tensor grad rel err", err)
        assert err <= 1e-5
    else:
        g_abs = gradient_abs_bound(cfg, blk, 9, p0, vol, opts, 1000)
        r = componentwise_ratio(cfg, g, om.g, g_abs) / 2.0 ** -11
        print("lambda", lam, "fp16 componentwise err / (u g_abs)", r)
        assert r <= 2 * (cfg.mlp_hidden_layers + 2)
    inr.inr_destroy(m)


@pytest.mark.parametrize("prec", [0, 1])
def test_cached_fit_graphs_replay_bitwise(prec):
    """inr_fit caches each call's one-step CUDA graph (keyed by its launch
    parameter bytes) and replays it in later identical calls: 1 + 2 + 3 steps in
    three calls, with another model's calls in between (another cache entry),
    end bitwise where one 6-step call ends (deterministic mode); a destroyed
    model's entries go, and a model created afterwards fits like a fresh one."""
    vol = synth.g2_energy(32).numpy()
    blk = sampler.decompose((32, 32, 32), (16, 16, 16))[2]
    vt = gpu_volume(vol)
    go = inr.inr_fit_opts_default()
    go.vmin, go.vmax, go.boundary_batch = float(vol.min()), float(vol.max()), 128
    a = make_gpu_model(blk, 3, reduction=1, precision=prec, **CFG1)
    b = make_gpu_model(blk, 4, reduction=1, precision=prec, **CFG1)
    for n in (1, 2, 3):
        inr.inr_fit(a, whole_view(vt), n, 1024, go, stream())
        inr.inr_fit(b, whole_view(vt), n, 1024, go, stream())
    ref = make_gpu_model(blk, 3, reduction=1, precision=prec, **CFG1)
    inr.inr_fit(ref, whole_view(vt), 6, 1024, go, stream())
    assert inr.inr_steps(a) == 6 and np.array_equal(get_params(a), get_params(ref))
    inr.inr_destroy(a)
    inr.inr_destroy(ref)
    c = make_gpu_model(blk, 3, reduction=1, precision=prec, **CFG1)
    d = make_gpu_model(blk, 3, reduction=1, precision=prec, **CFG1)
    inr.inr_fit(c, whole_view(vt), 2, 1024, go, stream())
    inr.inr_fit(c, whole_view(vt), 2, 1024, go, stream())
    inr.inr_fit(d, whole_view(vt), 4, 1024, go, stream())
    assert np.array_equal(get_params(c), get_params(d))
    for m in (b, c, d):
        inr.inr_destroy(m)


def test_decode_grid_and_query_vs_oracle():
    vol = synth.g1_analytic(32).numpy()
    blocks = sampler.decompose((32, 32, 32), (16, 16, 16))
    cfg = oracle_config(**CFG1)
    rng = np.random.default_rng(12)
    gms, oms = [], {}
    for b in blocks:
        p = init_params(cfg, 9, b.block_id)
        p[: sum(cfg.level_sizes()) * 2] = rng.uniform(-1, 1, sum(cfg.level_sizes()) * 2)
        m = make_gpu_model(b, 9, **CFG1)
        inr.inr_set_params(m, p)
        gms.append(m)
        om = InrModel(cfg, b, 9, params=p)
        oms[b.block_id] = om
    # decode grid of block 5 at 1x and a ragged resolution
    for res in ((16, 16, 16), (20, 7, 33)):
        out = torch.empty(res[::-1], device="cuda")
        inr.inr_decode_grid(gms[5], res, out.data_ptr(), None, None, None, stream())
        torch.cuda.synchronize()
        assert normwise(out.cpu().numpy(), o_decode.decode_grid(oms[5], res)) <= 1e-5
    # strided write of every block into one global volume; == query at nodes, bitwise
    full = torch.empty((32, 32, 32), device="cuda")
    for m, b in zip(gms, blocks):
        o = b.origin
        base = full[o[2]:, o[1]:, o[0]:]
        inr.inr_decode_grid(m, (16, 16, 16), base.data_ptr(), (1, 32, 1024), None, None, stream())
    z, y, x = np.meshgrid(np.arange(32), np.arange(32), np.arange(32), indexing="ij")
    pts = np.stack([x.ravel(), y.ravel(), z.ravel()], 1).astype(np.float32)
    pd = torch.from_numpy(pts).cuda()
    q = torch.empty(pts.shape[0], device="cuda")
    inr.inr_decode_group(gms, pd.data_ptr(), pts.shape[0], q.data_ptr(), 1, stream())
    torch.cuda.synchronize()
    assert torch.equal(q, full.reshape(-1))
    # random queries vs the oracle router
    rp = synth.random_points(4000, (32, 32, 32))
    rd = torch.from_numpy(rp).cuda()
    rq = torch.empty(4000, device="cuda")
    inr.inr_decode_group(gms, rd.data_ptr(), 4000, rq.data_ptr(), 1, stream())
    torch.cuda.synchronize()
    assert normwise(rq.cpu().numpy(), o_decode.decode_query(oms, rp)) <= 1e-5
    # strict domain error
    bad = torch.tensor([[-1.0, 0, 0]], device="cuda")
    with pytest.raises(inr.InrError) as e:
        inr.inr_decode_group(gms, bad.data_ptr(), 1, rq.data_ptr(), 1, stream())
    assert e.value.status == inr.INR_ERR_DOMAIN
    for m in gms:
        inr.inr_destroy(m)


def test_decode_grid_sse_matches_oracle():
    vol = synth.g1_analytic(32).numpy()
    blk = sampler.decompose((32, 32, 32), (32, 32, 32))[0]
    lo, hi = sampler.value_range([vol])
    m = make_gpu_model(blk, 2, **CFG1)
    vt = gpu_volume(vol)
    go = inr.inr_fit_opts_default()
    go.vmin, go.vmax = lo, hi
    inr.inr_fit(m, whole_view(vt), 20, 1024, go, stream())
    out = torch.empty((32, 32, 32), device="cuda")
    sse = torch.zeros(1, dtype=torch.float64, device="cuda")
    inr.inr_decode_grid(m, (32, 32, 32), out.data_ptr(), None, vt.data_ptr(), sse.data_ptr(), stream())
    torch.cuda.synchronize()
    want = o_decode.sse_normalized(out.cpu().numpy(), vol, lo, hi)
    assert abs(sse.item() - want) <= 1e-6 * want
    inr.inr_destroy(m)


def test_value_range_exact():
    vol = synth.g3_density(48).numpy()
    vt = gpu_volume(vol)
    mm = torch.tensor([float("inf"), float("-inf")], device="cuda")
    inr.inr_value_range(whole_view(vt), mm.data_ptr(), stream())
    sub = vt[8:40, 4:20, 0:48]
    v2 = inr.make_view(sub.data_ptr(), (0, 4, 8), (48, 16, 32), (1, 48, 48 * 48))
    mm2 = torch.tensor([float("inf"), float("-inf")], device="cuda")
    inr.inr_value_range(v2, mm2.data_ptr(), stream())
    torch.cuda.synchronize()
    assert mm.tolist() == [float(vol.min()), float(vol.max())]
    assert mm2.tolist() == [float(vol[8:40, 4:20].min()), float(vol[8:40, 4:20].max())]


@pytest.mark.parametrize("flags", [0, inr.CACHE_HOST_RESIDENT, inr.CACHE_FP16,
                                   inr.CACHE_HOST_RESIDENT | inr.CACHE_FP16])
def test_cache_fifo_and_decode_from_slot(flags):
    vol = synth.g1_analytic(16).numpy()
    blk = sampler.decompose((16, 16, 16), (16, 16, 16))[0]
    vt = gpu_volume(vol)
    go = inr.inr_fit_opts_default()
    go.vmin, go.vmax = float(vol.min()), float(vol.max())
    m = make_gpu_model(blk, 1, **CFG1)
    c = inr.cache_create(3, flags, 0)
    fp16 = bool(flags & inr.CACHE_FP16)
    snaps = {}
    for ts in (1, 2, 3, 4):
        inr.inr_reset(m, 100 + ts)
        inr.inr_fit(m, whole_view(vt), 3, 256, go, stream())
        ev = inr.cache_insert(c, ts, [m], stream())
        assert ev == (1 if ts == 4 else -1)
        p = get_params(m)
        snaps[ts] = p.astype(np.float16).astype(np.float32) if fp16 else p
    assert inr.cache_size(c) == 3
    assert inr.cache_bytes(c) == 3 * inr.inr_param_bytes(m) // (2 if fp16 else 1)
    with pytest.raises(inr.InrError):
        inr.cache_insert(c, 4, [m], stream())
    ts, blocks = inr.cache_get(c, 0)
    assert ts == 2
    assert np.array_equal(get_params(blocks[0]), snaps[2])
    out = torch.empty((16, 16, 16), device="cuda")
    inr.inr_decode_grid(blocks[0], (16, 16, 16), out.data_ptr(), None, None, None, stream())
    inr.inr_set_params(m, snaps[2])
    out2 = torch.empty((16, 16, 16), device="cuda")
    inr.inr_decode_grid(m, (16, 16, 16), out2.data_ptr(), None, None, None, stream())
    torch.cuda.synchronize()
    assert torch.equal(out, out2)
    with pytest.raises(inr.InrError) as e:
        inr.inr_fit(blocks[0], whole_view(vt), 1, 16, go, stream())
    assert e.value.status == inr.INR_ERR_STATE
    assert inr.cache_evict(c) == 2 and inr.cache_evict(c) == 3 and inr.cache_evict(c) == 4
    with pytest.raises(inr.InrError) as e:
        inr.cache_evict(c)
    assert e.value.status == inr.INR_ERR_STATE
    inr.cache_destroy(c)
    inr.inr_destroy(m)


@pytest.mark.parametrize("prec", [0, 1])
def test_group_fit_matches_single_fits(prec):
    """Blocks are independent: a grouped launch gives each model
    the same result as fitting it alone (deterministic mode, bitwise)."""
    vol = synth.g2_energy(32).numpy()
    blocks = sampler.decompose((32, 32, 32), (16, 16, 16))
    vt = gpu_volume(vol)
    go = inr.inr_fit_opts_default()
    go.vmin, go.vmax, go.boundary_batch = float(vol.min()), float(vol.max()), 64
    group = [make_gpu_model(b, 6, reduction=1, precision=prec, **CFG1) for b in blocks]
    # 8192 + 64 samples = 65 tiles per block: several tiles per MLP CTA, whose order of
    # fp32 accumulation must not depend on how many models share the launch
    reps = inr.inr_fit_group(group, [whole_view(vt)] * len(group), 6, 8192, go, stream())
    assert all(r.steps_taken == 6 for r in reps)
    single = make_gpu_model(blocks[6], 6, reduction=1, precision=prec, **CFG1)
    inr.inr_fit(single, whole_view(vt), 6, 8192, go, stream())
    assert np.array_equal(get_params(single), get_params(group[6]))
    for m in group + [single]:
        inr.inr_destroy(m)


def test_fit_errors():
    blk = sampler.decompose((16, 16, 16), (16, 16, 16))[0]
    m = make_gpu_model(blk, 1, **CFG1)
    vt = gpu_volume(synth.g1_analytic(16).numpy())
    go = inr.inr_fit_opts_default()
    for steps, batch in ((0, 16), (1, 0)):
        with pytest.raises(inr.InrError) as e:
            inr.inr_fit(m, whole_view(vt), steps, batch, go, stream())
        assert e.value.status == inr.INR_ERR_INVALID_ARG
    go.lambda_ = 1.5
    with pytest.raises(inr.InrError):
        inr.inr_fit(m, whole_view(vt), 1, 16, go, stream())
    go = inr.inr_fit_opts_default()
    small = inr.make_view(vt.data_ptr(), (0, 0, 0), (8, 16, 16), (1, 16, 256))
    with pytest.raises(inr.InrError):
        inr.inr_fit(m, small, 1, 16, go, stream())
    go.vmin = go.vmax = 0.5                                   # constant field: not an error
    rep = inr.inr_fit(m, whole_view(vt), 2, 16, go, stream())
    assert rep.constant_field == 1
    inr.inr_destroy(m)


def test_psnr_target_stopping():
    vol = synth.constant_field((16, 16, 16), 0.5)
    blk = sampler.decompose((16, 16, 16), (16, 16, 16))[0]
    m = make_gpu_model(blk, 5, **CFG1)
    vt = gpu_volume(vol)
    go = inr.inr_fit_opts_default()
    go.vmin, go.vmax, go.lr0, go.target_psnr, go.check_interval = 0.0, 1.0, 1e-3, 45.0, 10
    rep = inr.inr_fit(m, whole_view(vt), 400, 512, go, stream())
    assert rep.reached_target == 1 and rep.probe_psnr >= 45 and rep.steps_taken < 400
    inr.inr_destroy(m)


def test_decode_tensor_core_fp16_models():
    """fp16-MLP models decode on tensor cores: grid (R19 vertex elision) and
    bucket-sorted queries agree bitwise at the nodes, and both match the oracle
    within the fp16 tolerance (2e-3 normwise); a point whose block is not in the
    group decodes to NaN."""
    blocks = sampler.decompose((48, 48, 48), (16, 16, 16))   # 27 blocks
    cfg = oracle_config(**CFG1)
    rng = np.random.default_rng(21)
    gms, oms = [], {}
    for b in blocks[:-1]:                                     # the last block is left out
        p = _perturbed_params(cfg, b, 3, rng)
        m = make_gpu_model(b, 3, precision=1, **CFG1)
        inr.inr_set_params(m, p)
        gms.append(m)
        oms[b.block_id] = InrModel(cfg, b, 3, params=p)
    for res in ((16, 16, 16), (32, 32, 32), (13, 5, 21)):
        out = torch.empty(res[::-1], device="cuda")
        inr.inr_decode_grid(gms[7], res, out.data_ptr(), None, None, None, stream())
        torch.cuda.synchronize()
        assert normwise(out.cpu().numpy(), o_decode.decode_grid(oms[blocks[7].block_id], res)) <= 2e-3
    full = torch.empty((48, 48, 48), device="cuda")
    for m, b in zip(gms, blocks):
        o = b.origin
        inr.inr_decode_grid(m, (16, 16, 16), full[o[2]:, o[1]:, o[0]:].data_ptr(), (1, 48, 48 * 48), None, None,
                            stream())
    z, y, x = np.meshgrid(np.arange(48), np.arange(48), np.arange(48), indexing="ij")
    pts = np.stack([x.ravel(), y.ravel(), z.ravel()], 1).astype(np.float32)
    q = torch.empty(pts.shape[0], device="cuda")
    pd = torch.from_numpy(pts).cuda()
    inr.inr_decode_group(gms, pd.data_ptr(), pts.shape[0], q.data_ptr(), 0, stream())
    torch.cuda.synchronize()
    qn = q.cpu().numpy()
    last = blocks[-1]
    own = ((pts[:, 0] >= last.origin[0]) & (pts[:, 1] >= last.origin[1]) & (pts[:, 2] >= last.origin[2]))
    assert np.all(np.isnan(qn[own])) and not np.any(np.isnan(qn[~own]))
    assert np.array_equal(qn[~own], full.reshape(-1).cpu().numpy()[~own])
    rp = synth.random_points(20000, (48, 48, 48))
    rp = rp[~((rp[:, 0] >= 32) & (rp[:, 1] >= 32) & (rp[:, 2] >= 32))]
    rd = torch.from_numpy(rp).cuda()
    rq = torch.empty(rp.shape[0], device="cuda")
    inr.inr_decode_group(gms, rd.data_ptr(), rp.shape[0], rq.data_ptr(), 1, stream())
    torch.cuda.synchronize()
    assert normwise(rq.cpu().numpy(), o_decode.decode_query(oms, rp)) <= 2e-3
    for m in gms:
        inr.inr_destroy(m)


@pytest.mark.parametrize("prec", [0, 1])
def test_view_is_read_only_inside_its_contract(prec):
    """A block's view need only cover nodes [o, min(o+n, N-1)] (inr.h): embed the
    17^3 nodes of block 0 of a 32^3 volume in a NaN-filled buffer — samples on the
    block's far faces (x = 1, weight 0 on the next node) must not touch the NaNs,
    and the step equals the one on the full volume."""
    vol = synth.g1_analytic(32).numpy()
    blk = sampler.decompose((32, 32, 32), (16, 16, 16))[0]        # faces +x, +y, +z
    buf = torch.full((20, 20, 20), float("nan"), device="cuda")
    buf[:17, :17, :17] = torch.from_numpy(vol[:17, :17, :17]).cuda()
    view = inr.make_view(buf.data_ptr(), (0, 0, 0), (17, 17, 17), (1, 20, 400))
    go = inr.inr_fit_opts_default()
    go.vmin, go.vmax, go.boundary_batch = float(vol.min()), float(vol.max()), 512
    a = make_gpu_model(blk, 3, reduction=1, precision=prec, **CFG1)
    rep = inr.inr_fit(a, view, 2, 1024, go, stream())
    assert np.isfinite(rep.loss_uniform) and np.isfinite(rep.loss_boundary)
    b = make_gpu_model(blk, 3, reduction=1, precision=prec, **CFG1)
    vt = gpu_volume(vol)
    inr.inr_fit(b, whole_view(vt), 2, 1024, go, stream())
    assert np.array_equal(get_params(a), get_params(b))
    inr.inr_destroy(a)
    inr.inr_destroy(b)


def test_stream_ordered_loss_report_matches_fit_report():
    """inr_fit_losses (no synchronization) reports the same L1 terms as the
    synchronous inr_fit_report of the same step, per model of a group."""
    vol = synth.g1_analytic(32).numpy()
    blocks = sampler.decompose((32, 32, 32), (16, 16, 16))
    vt = gpu_volume(vol)
    go = inr.inr_fit_opts_default()
    go.vmin, go.vmax, go.boundary_batch = float(vol.min()), float(vol.max()), 64
    ms = [make_gpu_model(b, 3, precision=1, **CFG1) for b in blocks]
    reps = inr.inr_fit_group(ms, [whole_view(vt)] * len(ms), 3, 256, go, stream(), True)
    out = torch.full((3 * len(ms),), float("nan"), dtype=torch.float64, device="cuda")
    inr.inr_fit_losses(ms, out.data_ptr(), stream())
    torch.cuda.synchronize()
    o = out.cpu().numpy().reshape(-1, 3)
    for r, row in zip(reps, o):
        assert abs(row[0] - r.loss_uniform) <= 1e-15 * r.loss_uniform
        assert abs(row[1] - r.loss_boundary) <= 1e-15 * max(r.loss_boundary, 1e-300)
        assert row[2] == 0.0
    for m in ms:
        inr.inr_destroy(m)


def test_warm_start_keeps_parameters_and_restarts_adam():
    """inr_reset_optimizer (NEXT-4 warm start): parameters unchanged, Adam
    moments and the step counter zeroed, so the next step equals a fresh
    model loaded with those parameters (same seed streams) bitwise."""
    vol = synth.g1_analytic(32).numpy()
    blk = sampler.decompose((32, 32, 32), (32, 32, 32))[0]
    vt = gpu_volume(vol)
    go = inr.inr_fit_opts_default()
    go.vmin, go.vmax = float(vol.min()), float(vol.max())
    a = make_gpu_model(blk, 4, reduction=1, **CFG1)
    inr.inr_fit(a, whole_view(vt), 5, 256, go, stream())
    p5 = get_params(a)
    inr.inr_reset_optimizer(a)
    assert np.array_equal(get_params(a), p5) and inr.inr_steps(a) == 0
    m, v = inr.inr_get_adam_state(a, np.empty_like(p5), np.empty_like(p5))
    assert not m.any() and not v.any()
    b = make_gpu_model(blk, 4, reduction=1, **CFG1)
    inr.inr_set_params(b, p5)
    inr.inr_fit(a, whole_view(vt), 2, 256, go, stream())
    inr.inr_fit(b, whole_view(vt), 2, 256, go, stream())
    assert np.array_equal(get_params(a), get_params(b))
    inr.inr_destroy(a)
    inr.inr_destroy(b)


@pytest.mark.parametrize("prec", [0, 1])
def test_group_psnr_stopping_is_per_model(prec):
    """PSNR-target stopping inside a group: each block leaves the group at its own
    first check above the target (steps differ between blocks) and ends bitwise
    as if fitted alone with the same options (deterministic mode)."""
    vol = synth.g2_energy(32).numpy()
    blocks = sampler.decompose((32, 32, 32), (16, 16, 16))
    vt = gpu_volume(vol)
    go = inr.inr_fit_opts_default()
    go.vmin, go.vmax, go.boundary_batch = float(vol.min()), float(vol.max()), 64
    go.target_psnr, go.check_interval = 38.0, 10
    group = [make_gpu_model(b, 8, reduction=1, precision=prec, **CFG1) for b in blocks]
    reps = inr.inr_fit_group(group, [whole_view(vt)] * len(group), 300, 1024, go, stream())
    steps = [r.steps_taken for r in reps]
    print("steps per block", steps, [round(r.probe_psnr, 1) for r in reps])
    assert len(set(steps)) > 1 and all(r.reached_target for r in reps)
    for k in (int(np.argmin(steps)), int(np.argmax(steps))):
        single = make_gpu_model(blocks[k], 8, reduction=1, precision=prec, **CFG1)
        rep = inr.inr_fit(single, whole_view(vt), 300, 1024, go, stream())
        assert rep.steps_taken == steps[k] and inr.inr_steps(single) == steps[k]
        assert np.array_equal(get_params(single), get_params(group[k]))
        inr.inr_destroy(single)
    for m in group:
        inr.inr_destroy(m)
