"""Pins of the oracle's vector-field path (D = 3, "v can be a scalar
(D=1), 3-dimensional vector (D=3)"; R28):
symmetry against the scalar model, closed-form per-channel normalization,
central finite differences."""
import numpy as np

import synth
from oracle import decode, fit, sampler
from oracle.model import Config, InrModel

CFG = dict(levels=4, features=2, log2_table_size=10, mlp_width=64, mlp_hidden_layers=2)


def _replica(seed=3):
    """A D = 3 model whose output rows all equal the D = 1 model's single row."""
    blk = sampler.Block((0, 0, 0), (16, 16, 16), (16, 16, 16))
    m1 = InrModel(Config(**CFG), blk, seed)
    rng = np.random.default_rng(seed)
    m1.p[:] += rng.normal(size=m1.p.size) * 0.2
    c3 = Config(**CFG, out_dim=3)
    m3 = InrModel(c3, blk, seed)
    for name, shape, off in c3.tensor_layout():
        src = m1.view(m1.p, name)
        dst = m3.view(m3.p, name)
        dst[...] = np.broadcast_to(src, dst.shape) if name in ("W2", "b2") else src
    return m1, m3


def test_replica_outputs_equal_per_channel():
    m1, m3 = _replica()
    x = np.random.default_rng(0).random((500, 3)).astype(np.float32)
    y1, _ = fit.forward(m1, x)
    y3, _ = fit.forward(m3, x)
    assert y3.shape == (500, 3)
    assert np.allclose(y3, np.repeat(y1, 3, axis=1), rtol=1e-14, atol=0)     # BLAS order may differ


def test_replica_gradients_pool_over_channels():
    """Identical channels: L_3 = mean over n x 3 residuals = L_1, so every
    shared parameter's gradient equals the scalar model's and each output row
    gets a third of the scalar output-row gradient (R28)."""
    m1, m3 = _replica()
    f = synth.g1_analytic(17).double().numpy()
    vec = np.stack([f, f, f], axis=-1)
    lo, hi = sampler.value_range([f])
    o1 = fit.FitOpts(vmin=lo, vmax=hi)
    o3 = fit.FitOpts(vmin=np.array([lo] * 3), vmax=np.array([hi] * 3))
    l1 = fit.train_step(m1, f, o1, 400)
    l3 = fit.train_step(m3, vec, o3, 400)
    assert abs(l1[0] - l3[0]) < 1e-14
    for name, shape, off in m3.cfg.tensor_layout():
        g1, g3 = m1.view(m1.g, name), m3.view(m3.g, name)
        if name in ("W2", "b2"):
            assert np.allclose(g3, np.broadcast_to(g1 / 3.0, g3.shape), rtol=1e-12, atol=1e-15), name
        else:
            assert np.allclose(g3, g1, rtol=1e-11, atol=1e-15), name


def test_per_channel_normalization_closed_form():
    """Channels (f, 2f + 1, -f): per-channel ranges map them to t, t, 1 - t."""
    f = synth.g1_analytic(17).double().numpy()
    vec = np.stack([f, 2 * f + 1, -f], axis=-1)
    lo, hi = sampler.value_range([vec])
    assert np.allclose(lo, [f.min(), 2 * f.min() + 1, -f.max()]) and np.allclose(hi, [f.max(), 2 * f.max() + 1, -f.min()])
    blk = sampler.Block((0, 0, 0), (16, 16, 16), (17, 17, 17))
    x = np.random.default_rng(1).random((300, 3))
    t, const = sampler.targets(vec, blk, x, lo, hi)
    t0, _ = sampler.targets(f, blk, x, lo[0], hi[0])
    assert not const
    assert np.allclose(t[:, 0], t0, atol=1e-14) and np.allclose(t[:, 1], t0, atol=1e-14)
    assert np.allclose(t[:, 2], 1 - t0, atol=1e-14)
    # a constant channel normalizes to 0; the flag needs every channel constant
    vc = np.stack([f, np.full_like(f, 2.0), f], axis=-1)
    lo, hi = sampler.value_range([vc])
    t, const = sampler.targets(vc, blk, x, lo, hi)
    assert np.all(t[:, 1] == 0) and not const


def test_decode_denormalizes_per_channel():
    m1, m3 = _replica()
    m1.vmin, m1.vmax = 0.0, 1.0
    m3.vmin, m3.vmax = np.array([0.0, -2.0, 5.0]), np.array([1.0, 2.0, 6.0])
    g1 = decode.decode_grid(m1, (5, 4, 3))
    g3 = decode.decode_grid(m3, (5, 4, 3))
    assert g3.shape == (3, 4, 5, 3)
    assert np.allclose(g3[..., 0], g1, atol=1e-14)
    assert np.allclose(g3[..., 1], 4 * g1 - 2, atol=1e-13)
    assert np.allclose(g3[..., 2], g1 + 5, atol=1e-13)
    q = decode.decode_query({0: m3}, np.array([[1.0, 2.0, 3.0], [15.0, 0.5, 7.25]], np.float32))
    assert q.shape == (2, 3)


def test_vector_gradients_match_central_differences():
    """S:L229 finite differences (h = 1e-4, 1e-4 relative) on a tiny D = 3 net
    with a random per-channel upstream gradient."""
    cfg = Config(levels=2, features=2, log2_table_size=4, mlp_width=8, mlp_hidden_layers=2, out_dim=3)
    blk = sampler.Block((0, 0, 0), (8, 8, 8), (8, 8, 8))
    h, checked, seed = 1e-4, 0, 0
    while checked < 5:
        seed += 1
        m = InrModel(cfg, blk, seed)
        rng = np.random.default_rng(seed)
        m.p[:] = rng.uniform(-1, 1, m.p.size)
        x = rng.random((12, 3)).astype(np.float32)
        c = rng.normal(size=(12, 3))
        y, cache = fit.forward(m, x)
        if min(np.min(np.abs(z)) for z in cache[3][:-1]) < 50 * h:
            continue
        g = fit.gradients(m, x, c, cache)
        fd = np.empty_like(g)
        for j in range(m.p.size):
            old = m.p[j]
            m.p[j] = old + h
            fp = float(np.sum(c * fit.forward(m, x)[0]))
            m.p[j] = old - h
            fm = float(np.sum(c * fit.forward(m, x)[0]))
            m.p[j] = old
            fd[j] = (fp - fm) / (2 * h)
        assert np.max(np.abs(g - fd) / np.maximum(np.abs(fd), 1e-3)) < 1e-4
        checked += 1


def test_sse_constant_channel_contributes_zero():
    """a constant channel normalizes to 0 on both sides, so it adds
    nothing to the pooled SSE; the other channels add ((p - r) / range)^2."""
    pred = np.array([[1.0, 5.0, 2.0], [3.0, 5.0, 0.0]])
    ref = np.array([[0.0, 5.0, 1.0], [3.0, 5.0, 2.0]])
    s = decode.sse_normalized(pred, ref, np.array([0.0, 5.0, 0.0]), np.array([2.0, 5.0, 4.0]))
    assert s == (1 / 2) ** 2 + (1 / 4) ** 2 + (2 / 4) ** 2
