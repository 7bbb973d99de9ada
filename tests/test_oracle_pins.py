"""Pins of the oracle against what the paper and mathematics fix (SURVEY.md
§8(c) P1-P15, P18).  CPU only.  Each test names the passage it follows."""
import math

import numpy as np
import pytest
import torch

from oracle import adam, encoding, loss, mlp, philox, sampler
from oracle.model import Config, init_params


# ---------------------------------------------------------------- P15 Philox
def test_philox_known_answers(golden):
    for row in golden("philox_kat.txt"):
        v = [int(t, 16) for t in row]
        out = philox.philox4x32_10([[v[0]], [v[1]], [v[2]], [v[3]]], (v[4], v[5]))[:, 0]
        assert [int(o) for o in out] == v[6:10]


def test_philox_u01_range():
    u = np.array([0, 0xFF, 0x100, 0xFFFFFFFF], dtype=np.uint32)
    x = philox.u01(u)
    assert x.dtype == np.float32
    assert x[0] == 0.0 and x[1] == 0.0 and x[2] == np.float32(2.0 ** -24)
    assert x[3] == np.float32(1.0 - 2.0 ** -24)          # never reaches 1


# ---------------------------------------------------- P1 level resolution
def test_level_resolution_paper_values(golden):
    for l, n in golden("level_resolution.txt"):
        assert encoding.level_resolution(4, 2.0, int(l)) == int(n)


# ------------------------------------------------------- P2 table sizes
def test_table_sizes(golden):
    for row in golden("table_sizes.txt"):
        L, t, total = int(row[0]), int(row[1]), int(row[2])
        cfg = Config(levels=L, features=2, log2_table_size=t)
        sizes = cfg.level_sizes()
        assert sizes == [int(s) for s in row[3:3 + L]]
        assert sum(sizes) == total


def test_mlp_param_counts(golden):
    for fin, H, W, D, P in (map(int, r) for r in golden("mlp_params.txt")):
        cfg = Config(levels=fin, features=1, log2_table_size=4, mlp_width=W, mlp_hidden_layers=H, out_dim=D)
        n_mlp = cfg.param_count() - sum(cfg.level_sizes())
        assert n_mlp == P


# --------------------------------------------------------- P3 spatial hash
def test_hash_examples(golden):
    for t, x, y, z, h in (map(int, r) for r in golden("hash_examples.txt")):
        assert int(encoding.hash_index(x, y, z, 1 << t)) == h


def test_hash_identity_on_x_axis():
    x = np.arange(0, 70000, 37, dtype=np.uint32)
    for t in (14, 19, 22):
        assert np.array_equal(encoding.hash_index(x, 0, 0, 1 << t), x % (1 << t))


# --------------------------------------------------------- P4 dense index
def test_dense_index_bijection_and_examples():
    assert int(encoding.dense_index(1, 2, 3, 4)) == 86
    assert int(encoding.dense_index(4, 4, 4, 4)) == 124
    for n in (1, 2, 4, 7, 16):
        v = np.arange(n + 1)
        z, y, x = np.meshgrid(v, v, v, indexing="ij")
        idx = encoding.dense_index(x.ravel(), y.ravel(), z.ravel(), n)
        assert sorted(idx.tolist()) == list(range((n + 1) ** 3))


# ------------------------------------------------ P5 / P6 / P7 encoding
def _tables(cfg, rng, scale=1.0):
    return [rng.uniform(-scale, scale, (s, cfg.features)) for s in cfg.level_sizes()]


def test_vertex_identity_dense_and_hashed():
    """x on a level vertex => that level's slice equals the stored entry
    (S:L162).  The entries are located with the golden indices, not the
    oracle's index function."""
    cfg = Config(levels=8, features=2, log2_table_size=14)
    rng = np.random.default_rng(1)
    tabs = _tables(cfg, rng)
    res = cfg.resolutions()
    # dense level 0 (N=4): vertex (1,2,3) has index 86 (P4)
    f, _, _ = encoding.encode_forward(tabs, np.array([[0.25, 0.5, 0.75]], np.float32), res, cfg.table_size)
    assert np.array_equal(f[0, 0:2], tabs[0][86])
    # hashed level 3 (N=32, T=2^14): vertex (1,1,1) has hash 11813 (P3)
    x = np.array([[1 / 32, 1 / 32, 1 / 32]], np.float32)
    f, _, _ = encoding.encode_forward(tabs, x, res, cfg.table_size)
    assert np.array_equal(f[0, 6:8], tabs[3][11813])
    # x = 1 is the vertex N_l (R4): level 0 -> dense index of (4,4,4) = 124
    f, _, _ = encoding.encode_forward(tabs, np.ones((1, 3), np.float32), res, cfg.table_size)
    assert np.array_equal(f[0, 0:2], tabs[0][124])


def test_linear_reproduction_on_dense_level():
    """theta[v] = a.v + d on a dense level => feature = a.pos + d (trilinear
    interpolation reproduces affine functions)."""
    cfg = Config(levels=3, features=1, log2_table_size=14)
    res = cfg.resolutions()
    a = np.array([0.3, -1.7, 2.2])
    d = 0.4
    tabs = []
    for l, n in enumerate(res):
        t = np.empty((cfg.level_sizes()[l], 1))
        for vz in range(n + 1):
            for vy in range(n + 1):
                for vx in range(n + 1):
                    t[vx + (n + 1) * (vy + (n + 1) * vz), 0] = a @ [vx, vy, vz] + d
        tabs.append(t)
    x = np.random.default_rng(2).random((500, 3)).astype(np.float32)
    f, _, _ = encoding.encode_forward(tabs, x, res, cfg.table_size)
    for l, n in enumerate(res):
        pos = (x * np.float32(n)).astype(np.float64)
        assert np.allclose(f[:, l], pos @ a + d, rtol=0, atol=1e-12)


def test_partition_of_unity_and_zero_table():
    cfg = Config(levels=8, features=2, log2_table_size=14)
    x = np.random.default_rng(3).random((300, 3)).astype(np.float32)
    ones = [np.ones((s, 2)) for s in cfg.level_sizes()]
    f, _, wt = encoding.encode_forward(ones, x, cfg.resolutions(), cfg.table_size)
    assert np.allclose(f, 1.0, atol=1e-14)
    assert np.allclose(wt.sum(-1), 1.0, atol=1e-14)
    zeros = [np.zeros((s, 2)) for s in cfg.level_sizes()]
    f0, _, _ = encoding.encode_forward(zeros, x, cfg.resolutions(), cfg.table_size)
    assert np.all(f0 == 0.0)


def test_feature_length_paper_default():
    cfg = Config()                               # 16 levels x 4 features
    cfg.features = 4
    assert cfg.levels * cfg.features == 64


def test_brute_force_encode_tiny():
    """Brute-force re-derivation on a tiny grid: find the enclosing cell by
    scanning all cells (no floor), weights from the tent function."""
    cfg = Config(levels=2, features=1, log2_table_size=4)   # N = 4, 8; both hashed at T = 16
    rng = np.random.default_rng(4)
    tabs = _tables(cfg, rng)
    x = rng.random((40, 3)).astype(np.float32)
    f, _, _ = encoding.encode_forward(tabs, x, cfg.resolutions(), cfg.table_size)
    for l, n in enumerate(cfg.resolutions()):
        for i in range(x.shape[0]):
            pos = [float(np.float32(x[i, d]) * np.float32(n)) for d in range(3)]
            acc = 0.0
            for vz in range(n + 1):
                for vy in range(n + 1):
                    for vx in range(n + 1):
                        w = 1.0
                        for p, v in zip(pos, (vx, vy, vz)):
                            w *= max(0.0, 1.0 - abs(p - v))
                        if w > 0:
                            h = ((vx * 1) ^ (vy * 2654435761) ^ (vz * 805459861)) % 16
                            acc += w * tabs[l][h, 0]
            assert abs(acc - f[i, l]) < 1e-12


# ------------------------------------------------------------------ P8 MLP
def test_mlp_zero_weights_bias():
    Ws = [np.zeros((8, 4)), np.zeros((8, 8)), np.zeros((1, 8))]
    bs = [np.zeros(8), np.zeros(8), np.array([0.37])]
    y, _, _ = mlp.forward(Ws, bs, np.random.default_rng(0).random((5, 4)))
    assert np.all(y == 0.37)


def test_mlp_hand_example():
    """Pencil-and-paper 2->2->1.  x = (1, 1): z = [1+2+0.5, 3+4-1] =
    [3.5, 6], h = z, y = 0.5*3.5 - 6 + 0.25 = -4.0.  x = (1, -1): z = [-0.5, -2],
    both ReLU'd to 0, so y = the output bias 0.25."""
    Ws = [np.array([[1.0, 2.0], [3.0, 4.0]]), np.array([[0.5, -1.0]])]
    bs = [np.array([0.5, -1.0]), np.array([0.25])]
    y, zs, _ = mlp.forward(Ws, bs, np.array([[1.0, 1.0], [1.0, -1.0]]))
    assert y[0, 0] == -4.0
    assert np.array_equal(zs[0][1], [-0.5, -2.0]) and y[1, 0] == 0.25   # both ReLU'd to 0


def test_mlp_vs_torch_library():
    rng = np.random.default_rng(5)
    shapes = [(64, 32), (64, 64), (64, 64), (1, 64)]
    Ws = [rng.normal(size=s) / 8 for s in shapes]
    bs = [rng.normal(size=s[0]) for s in shapes]
    x = rng.normal(size=(257, 32))
    y, _, _ = mlp.forward(Ws, bs, x)
    h = torch.tensor(x)
    for k, (W, b) in enumerate(zip(Ws, bs)):
        h = torch.nn.functional.linear(h, torch.tensor(W), torch.tensor(b))
        if k < len(Ws) - 1:
            h = torch.relu(h)
    assert np.allclose(y, h.numpy(), rtol=1e-13, atol=1e-13)


# --------------------------------------------------------------- P10 loss
def test_loss_examples():
    # lambda = 0.5, L1_u = 0.2, L1_b = 0.4 -> 0.3
    tot, lu, lb, _, _ = loss.loss_and_grad([0.2, -0.2], [0, 0], [0.4], [0.0], 0.5)
    assert math.isclose(lu, 0.2) and math.isclose(lb, 0.4) and math.isclose(tot, 0.3)
    tot, lu, _, _, _ = loss.loss_and_grad([0.2, -0.2], [0, 0], [0.4], [0.0], 0.0)
    assert tot == lu
    tot, lu, _, dyu, dyb = loss.loss_and_grad([0.2, -0.2], [0, 0], [], [], 0.5)   # empty boundary
    assert tot == lu and dyb.size == 0 and np.array_equal(dyu, [0.5, -0.5])
    _, _, _, dyu, _ = loss.loss_and_grad([0.0, 1.0], [0.0, 0.0], [], [], 0.5)      # sgn(0) = 0
    assert dyu[0] == 0.0


def test_loss_linear_in_lambda():
    rng = np.random.default_rng(6)
    yu, tu, yb, tb = rng.random(10), rng.random(10), rng.random(7), rng.random(7)
    t0 = loss.loss_and_grad(yu, tu, yb, tb, 0.0)[0]
    t1 = loss.loss_and_grad(yu, tu, yb, tb, 1.0)[0]
    th = loss.loss_and_grad(yu, tu, yb, tb, 0.3)[0]
    assert math.isclose(th, 0.7 * t0 + 0.3 * t1, rel_tol=1e-14)


@pytest.mark.parametrize("lam", [0.0, 0.3, 0.8, 1.0])
def test_loss_dy_matches_central_differences(lam):
    """dL/dy of Eq. 2 against central differences of the pinned
    total: L is piecewise linear in each y_i, so with every |y_i - t_i| > h the
    difference quotient is exact up to rounding.  lam != 1/2 separates the
    (1 - lam)/|U| uniform weight from the lam/|B| boundary weight (a swap of the
    two, invisible at lam = 0.5, fails here); |U| != |B| separates the counts."""
    rng = np.random.default_rng(31)
    yu, tu = rng.random(9), rng.random(9)
    yb, tb = rng.random(4), rng.random(4)
    h = 1e-7
    assert min(np.abs(yu - tu).min(), np.abs(yb - tb).min()) > 10 * h
    _, _, _, dyu, dyb = loss.loss_and_grad(yu, tu, yb, tb, lam)

    def total(a, b):
        return loss.loss_and_grad(a, tu, b, tb, lam)[0]
    for i in range(9):
        e = np.zeros(9)
        e[i] = h
        fd = (total(yu + e, yb) - total(yu - e, yb)) / (2 * h)
        assert math.isclose(dyu[i], fd, rel_tol=1e-6, abs_tol=1e-9)
    for j in range(4):
        e = np.zeros(4)
        e[j] = h
        fd = (total(yu, yb + e) - total(yu, yb - e)) / (2 * h)
        assert math.isclose(dyb[j], fd, rel_tol=1e-6, abs_tol=1e-9)


# ---------------------------------------------------------- P11 lr, P12 Adam
def test_lr_schedule_examples():
    assert adam.lr_at(0) == 1e-2
    assert math.isclose(adam.lr_at(500), 8e-3)
    assert math.isclose(adam.lr_at(1250), 6.4e-3)
    assert adam.lr_at(499) == 1e-2


def test_adam_closed_forms():
    p = np.array([1.0, -2.0, 3.0])
    m, v = np.zeros(3), np.zeros(3)
    adam.adam_update(p, np.zeros(3), m, v, 1, 1e-2)
    assert np.array_equal(p, [1.0, -2.0, 3.0])               # zero grad, fresh state
    g = np.array([0.5, -3.0, 1e-3])
    p = np.zeros(3)
    adam.adam_update(p, g, np.zeros(3), np.zeros(3), 1, 1e-2)
    assert np.allclose(p, -1e-2 * g / (np.abs(g) + 1e-8), rtol=1e-12)


def test_adam_vs_torch_optim():
    rng = np.random.default_rng(7)
    p0 = rng.normal(size=50)
    p = p0.copy()
    m, v = np.zeros(50), np.zeros(50)
    tp = torch.tensor(p0.copy(), requires_grad=True)
    opt = torch.optim.Adam([tp], lr=1e-2, betas=(0.9, 0.999), eps=1e-8, foreach=False)
    for t in range(1, 31):
        g = rng.normal(size=50) * (t % 3)
        adam.adam_update(p, g, m, v, t, 1e-2)
        tp.grad = torch.tensor(g)
        opt.step()
    assert np.allclose(p, tp.detach().numpy(), rtol=1e-14, atol=1e-15)


def test_sparse_adam_groups():
    """R37 (NEXT-4 touched-only Adam): a table group of 8 floats with no
    non-zero gradient keeps p, m, v bitwise; a group with any non-zero entry,
    and every MLP parameter, takes exactly the dense R12 update (pinned above
    against torch.optim.Adam), zero-gradient members included; a ragged last
    group counts as a group."""
    rng = np.random.default_rng(12)
    n_tab, n_mlp = 21, 5                      # groups [0,8), [8,16), [16,21)
    p0, m0, v0 = rng.normal(size=26), rng.random(26) * 0.1, rng.random(26) * 0.01
    g = np.zeros(26)
    g[3] = 0.7                                # touches group 0 only
    g[n_tab:] = 0.0                           # MLP gradients zero: still updated (m, v decay)
    p, m, v = p0.copy(), m0.copy(), v0.copy()
    adam.adam_update_sparse(p, g, m, v, 3, 1e-2, [(0, n_tab)])
    pd, md, vd = p0.copy(), m0.copy(), v0.copy()
    adam.adam_update(pd, g, md, vd, 3, 1e-2)
    touched = np.r_[np.arange(0, 8), np.arange(n_tab, 26)]
    untouched = np.arange(8, n_tab)
    for a, b in ((p, pd), (m, md), (v, vd)):
        assert np.array_equal(a[touched], b[touched])
    for a, b in ((p, p0), (m, m0), (v, v0)):
        assert np.array_equal(a[untouched], b[untouched])
    assert not np.array_equal(m[n_tab:], m0[n_tab:])          # the MLP part moved with g = 0
    g2 = rng.normal(size=26)                                     # every group touched: dense
    p, m, v, pd, md, vd = p0.copy(), m0.copy(), v0.copy(), p0.copy(), m0.copy(), v0.copy()
    adam.adam_update_sparse(p, g2, m, v, 1, 1e-2, [(0, n_tab)])
    adam.adam_update(pd, g2, md, vd, 1, 1e-2)
    assert np.array_equal(p, pd) and np.array_equal(m, md) and np.array_equal(v, vd)
    assert list(np.nonzero(adam.touched_groups(np.r_[np.zeros(17), 1.0, np.zeros(3)]))[0]) == [16, 17, 18, 19, 20]


# ---------------------------------------------------- P13/P14/P18 sampler
def test_trilinear_identity_midpoint_linear():
    vol = np.random.default_rng(8).random((2, 2, 2)).astype(np.float32)
    for z in range(2):
        for y in range(2):
            for x in range(2):
                assert sampler.trilinear(vol, np.array([[x, y, z]], float))[0] == np.float64(vol[z, y, x])
    edge = np.zeros((2, 2, 2), np.float32)
    edge[0, 0, 1] = 1.0
    assert sampler.trilinear(edge, np.array([[0.5, 0, 0]]))[0] == 0.5
    lin = np.zeros((9, 7, 5), np.float32)
    z, y, x = np.meshgrid(np.arange(9), np.arange(7), np.arange(5), indexing="ij")
    lin[...] = x + 2 * y + 3 * z
    r = np.random.default_rng(9).random((100, 3)) * [4, 6, 8]
    assert np.allclose(sampler.trilinear(lin, r), r @ [1, 2, 3], atol=1e-12)


def test_normalization_and_psnr():
    t, c = sampler.normalize_values([5.0, 0.0, 10.0], 0.0, 10.0)
    assert np.array_equal(t, [0.5, 0.0, 1.0]) and not c
    t, c = sampler.normalize_values([3.0, 3.0], 3.0, 3.0)
    assert np.all(t == 0) and c
    a = np.random.default_rng(10).random(1000)
    assert sampler.psnr(a, a) == 200.0
    assert math.isclose(sampler.psnr(a + 0.1, a), 20.0, rel_tol=1e-9)


def test_probe_lattice_brute_force():
    """The 32^3 cell-centred probe lattice:
    enumerated by three plain loops, x fastest, every coordinate (j + 1/2)/32,
    exact in fp32 (a dyadic rational)."""
    xp = sampler.probe_lattice(32)
    assert xp.shape == (32768, 3) and xp.dtype == np.float32
    want = [((i + 0.5) / 32, (j + 0.5) / 32, (k + 0.5) / 32) for k in range(32) for j in range(32) for i in range(32)]
    assert np.array_equal(xp, np.array(want, np.float32))
    assert np.array_equal(sampler.probe_lattice(2), np.array([[.25, .25, .25], [.75, .25, .25], [.25, .75, .25],
                                                              [.75, .75, .25], [.25, .25, .75], [.75, .25, .75],
                                                              [.25, .75, .75], [.75, .75, .75]], np.float32))


def test_sse_normalized_closed_forms():
    """SSE in normalized units (R18): a uniform offset c (value units)
    over n voxels gives n (c / (vmax - vmin))^2; a constant channel adds 0
    (S:L70); per-channel spans divide per channel."""
    from oracle import decode
    ref = np.random.default_rng(11).random((5, 6, 7))
    assert math.isclose(decode.sse_normalized(ref + 0.3, ref, 2.0, 4.0), 210 * 0.15 ** 2, rel_tol=1e-12)
    assert decode.sse_normalized(ref, ref, 0.0, 1.0) == 0.0
    r3 = np.zeros((4, 3))
    p3 = r3 + [1.0, 2.0, 5.0]
    assert math.isclose(decode.sse_normalized(p3, r3, [0, 0, 0], [2.0, 4.0, 0.0]), 4 * (0.25 + 0.25), rel_tol=1e-12)


def test_value_range_permutation_invariant():
    parts = [np.array([0.0, 1.0]), np.array([-2.0, 0.5])]
    assert sampler.value_range(parts) == (-2.0, 1.0)
    assert sampler.value_range(parts[::-1]) == (-2.0, 1.0)


def test_decomposition_and_faces():
    blocks = sampler.decompose((256, 256, 256), (128, 128, 128))
    assert len(blocks) == 8 and [b.block_id for b in blocks] == list(range(8))
    assert all(len(b.interior_faces()) == 3 for b in blocks)        # 2x2x2: every block has 3
    single = sampler.decompose((64, 64, 64), (64, 64, 64))
    assert len(single) == 1 and single[0].interior_faces() == []
    b221 = sampler.decompose((64, 64, 32), (32, 32, 32))
    assert all(len(b.interior_faces()) == 2 for b in b221)          # S: (2,2,1) -> 2 faces each


def test_boundary_samples_lie_on_interior_faces():
    blk = sampler.decompose((64, 64, 64), (32, 32, 32))[0]          # faces +x, +y, +z
    x = sampler.boundary_samples(123, 0, blk, 3000)
    on = (x == 1.0)
    assert np.all(on.sum(1) >= 1)
    assert np.all(x >= 0) and np.all(x <= 1)
    counts = on.sum(0)
    assert np.all(counts > 800)                                      # ~uniform over 3 faces
    assert sampler.boundary_samples(1, 0, sampler.decompose((8, 8, 8), (8, 8, 8))[0], 10).shape == (0, 3)


def test_uniform_samples_half_open():
    x = sampler.uniform_samples(99, 3, 5, 20000)
    assert x.dtype == np.float32 and x.min() >= 0 and x.max() < 1
    assert abs(float(x.mean()) - 0.5) < 0.01


# ----------------------------------------------------------- init (R14)
def test_init_ranges_and_determinism():
    cfg = Config(levels=8, features=2, log2_table_size=14, mlp_hidden_layers=2)
    p = init_params(cfg, 42, 0)
    q = init_params(cfg, 42, 0)
    assert np.array_equal(p, q) and p.dtype == np.float32
    assert not np.array_equal(p, init_params(cfg, 42, 1))
    for name, shape, off in cfg.tensor_layout():
        v = p[off:off + int(np.prod(shape))]
        if name.startswith("table"):
            assert np.abs(v).max() <= 1e-4 and np.abs(v).max() > 0.9e-4
        elif name.startswith("W"):
            a = math.sqrt(6.0 / shape[1])
            assert np.abs(v).max() <= a and np.abs(v).max() > 0.9 * a
        else:
            assert np.all(v == 0)
