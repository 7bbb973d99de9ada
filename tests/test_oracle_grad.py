"""P9: the oracle's analytic gradients (MLP backward + table scatter) against
central finite differences of its forward pass (h = 1e-4,
1e-4 relative, tiny config L=2, T=16, F=2, MLP 2x8, >= 20 seeds), and against
torch autograd (library routine) on a larger case."""
import numpy as np
import torch

from oracle import fit, sampler
from oracle.model import Config, InrModel


def _tiny_model(seed):
    cfg = Config(levels=2, features=2, log2_table_size=4, mlp_width=8, mlp_hidden_layers=2)
    blk = sampler.Block((0, 0, 0), (8, 8, 8), (8, 8, 8))
    m = InrModel(cfg, blk, seed)
    rng = np.random.default_rng(seed)
    m.p[:] = rng.uniform(-1.0, 1.0, m.p.size)        # O(1) tables so every path carries gradient
    return m


def _surrogate(m, x, c):
    y, cache = fit.forward(m, x)
    return float(np.sum(c * y[:, 0])), y, cache


def test_gradients_match_central_differences():
    h = 1e-4
    checked = 0
    seed = 0
    while checked < 20:
        seed += 1
        m = _tiny_model(seed)
        rng = np.random.default_rng(1000 + seed)
        x = rng.random((16, 3)).astype(np.float32)
        c = rng.normal(size=16)
        _, y, cache = _surrogate(m, x, c)
        zs = cache[3]
        if min(np.min(np.abs(z)) for z in zs[:-1]) < 50 * h:   # too close to a ReLU kink: redraw
            continue
        g = fit.gradients(m, x, c[:, None], cache)
        fd = np.empty_like(g)
        for j in range(m.p.size):
            old = m.p[j]
            m.p[j] = old + h
            fp = _surrogate(m, x, c)[0]
            m.p[j] = old - h
            fm = _surrogate(m, x, c)[0]
            m.p[j] = old
            fd[j] = (fp - fm) / (2 * h)
        scale = np.maximum(np.abs(fd), 1e-3)
        assert np.max(np.abs(g - fd) / scale) < 1e-4, seed
        checked += 1


def test_untouched_entries_have_zero_gradient():
    cfg = Config(levels=4, features=2, log2_table_size=12, mlp_width=16, mlp_hidden_layers=2)
    blk = sampler.Block((0, 0, 0), (8, 8, 8), (8, 8, 8))
    m = InrModel(cfg, blk, 3)
    x = np.array([[0.1, 0.2, 0.3]], np.float32)
    y, cache = fit.forward(m, x)
    g = fit.gradients(m, x, np.ones((1, 1)), cache)
    idx = cache[1]
    for l in range(cfg.levels):
        gl = m.view(g, f"table{l}")
        touched = np.zeros(gl.shape[0], bool)
        touched[idx[0, l]] = True
        assert np.all(gl[~touched] == 0.0)


def test_gradients_match_torch_autograd():
    """Same forward written with torch ops (gather + linear + relu) and
    differentiated by autograd; the corner indices/weights are taken from the
    oracle's encoder (pinned separately in test_oracle_pins)."""
    cfg = Config(levels=8, features=2, log2_table_size=10, mlp_width=64, mlp_hidden_layers=3)
    blk = sampler.Block((0, 0, 0), (16, 16, 16), (16, 16, 16))
    m = InrModel(cfg, blk, 11)
    rng = np.random.default_rng(11)
    m.p[:] += rng.normal(size=m.p.size) * 0.1
    x = rng.random((300, 3)).astype(np.float32)
    dy = rng.normal(size=(300, 1))
    y, cache = fit.forward(m, x)
    g = fit.gradients(m, x, dy, cache)
    _, idx, wt, _, _ = cache
    P = torch.tensor(m.p, requires_grad=True)
    feats = []
    for l in range(cfg.levels):
        name, shape, off = cfg.tensor_layout()[l]
        tab = P[off:off + shape[0] * shape[1]].reshape(shape)
        feats.append((torch.tensor(wt[:, l, :, None]) * tab[torch.tensor(idx[:, l, :].astype(np.int64))]).sum(1))
    h = torch.cat(feats, 1)
    K = cfg.mlp_hidden_layers + 1
    lay = {n: (s, o) for n, s, o in cfg.tensor_layout()}
    for k in range(K):
        (so, oo), (sb, ob) = lay[f"W{k}"], lay[f"b{k}"]
        W = P[oo:oo + so[0] * so[1]].reshape(so)
        b = P[ob:ob + sb[0]]
        h = torch.nn.functional.linear(h, W, b)
        if k < K - 1:
            h = torch.relu(h)
    assert np.allclose(h.detach().numpy(), y, rtol=1e-12, atol=1e-13)
    (h * torch.tensor(dy)).sum().backward()
    assert np.allclose(P.grad.numpy(), g, rtol=1e-10, atol=1e-13)
