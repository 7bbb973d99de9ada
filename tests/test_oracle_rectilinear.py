"""Pins of the oracle's rectilinear-mesh sampler and decode (NEXT-4; P:L249
"For uniform and rectilinear meshes, we provide a native data sampler";
S:L26-27; R36)."""
import numpy as np

from oracle import decode, fit, sampler
from oracle.model import Config, InrModel


def stretched(n, seed):
    """Strictly increasing node coordinates with cell widths in [0.5, 2]."""
    w = np.random.default_rng(seed).uniform(0.5, 2.0, n - 1)
    return np.concatenate([[0.0], np.cumsum(w)]) - 3.0


def test_unit_mesh_reduces_to_the_uniform_sampler():
    dims = (33, 20, 17)
    mesh = tuple(np.arange(d, dtype=np.float64) for d in dims)
    vol = np.random.default_rng(0).random(dims[::-1])
    x = sampler.uniform_samples(5, 3, 2, 500)
    for b_u, b_r in zip(sampler.decompose(dims, (16, 8, 8)), sampler.decompose(dims, (16, 8, 8), mesh)):
        interior = all(b_u.origin[d] + b_u.n[d] <= dims[d] - 1 for d in range(3))
        if not interior:
            continue   # ragged upper blocks normalize by their actual extent on a rectilinear mesh (R36)
        assert np.allclose(sampler.sample_positions(b_r, x), sampler.sample_positions(b_u, x), rtol=0, atol=1e-12)
        t_u, _ = sampler.targets(vol, b_u, x, 0.0, 1.0)
        t_r, _ = sampler.targets(vol, b_r, x, 0.0, 1.0)
        assert np.allclose(t_u, t_r, atol=1e-12)


def test_physically_linear_field_is_reproduced_exactly():
    """Trilinear interpolation on a rectilinear cell reproduces any function that is
    linear in the physical coordinates (S:L47 on a stretched mesh)."""
    dims = (21, 17, 13)
    mesh = tuple(stretched(d, s) for d, s in zip(dims, (1, 2, 3)))
    Z, Y, X = np.meshgrid(mesh[2], mesh[1], mesh[0], indexing="ij")
    vol = 0.7 * X - 1.3 * Y + 2.1 * Z + 5.0
    x = sampler.uniform_samples(9, 0, 0, 2000)
    for b in sampler.decompose(dims, (8, 8, 8), mesh):
        lo, hi = b.physical_box()
        P = lo[None, :] + x.astype(np.float64) * (hi - lo)[None, :]
        t, _ = sampler.targets(vol, b, x, 0.0, 1.0)
        assert np.allclose(t, 0.7 * P[:, 0] - 1.3 * P[:, 1] + 2.1 * P[:, 2] + 5.0, rtol=0, atol=1e-11)


def test_index_physical_maps_are_inverse_and_hit_nodes():
    X = stretched(40, 4)
    r = np.random.default_rng(1).random(1000) * 39
    assert np.allclose(sampler.physical_to_index(X, sampler.index_to_physical(X, r)), r, atol=1e-12)
    assert np.array_equal(sampler.physical_to_index(X, X), np.arange(40.0))


def test_boundary_faces_are_shared_physical_planes():
    dims = (33, 9, 9)
    mesh = (stretched(33, 5), np.arange(9.0), np.arange(9.0))
    a, b = sampler.decompose(dims, (16, 8, 8), mesh)[:2]
    x1 = np.array([[1.0, 0.3, 0.6]])
    x0 = np.array([[0.0, 0.3, 0.6]])
    assert np.allclose(sampler.sample_positions(a, x1), sampler.sample_positions(b, x0), atol=1e-12)


def test_rectilinear_grid_decode_is_the_node_query():
    dims = (17, 9, 9)
    mesh = (stretched(17, 7), stretched(9, 8), stretched(9, 9))
    cfg = Config(levels=4, features=2, log2_table_size=10, mlp_width=16, mlp_hidden_layers=1)
    blocks = sampler.decompose(dims, (8, 8, 8), mesh)
    models = {}
    for b in blocks:
        m = InrModel(cfg, b, 3)
        m.p[:] += np.random.default_rng(b.block_id).normal(size=m.p.size) * 0.3
        models[b.block_id] = m
    b = blocks[0]
    g = decode.decode_grid(models[b.block_id], (8, 8, 8))
    z, y, x = np.meshgrid(np.arange(8), np.arange(8), np.arange(8), indexing="ij")
    pts = np.stack([x.ravel(), y.ravel(), z.ravel()], 1).astype(np.float32)
    q = decode.decode_query(models, pts).reshape(8, 8, 8)
    assert np.allclose(g, q, rtol=0, atol=1e-12)
    assert decode.mesh_grid_coords(b, (9, 1, 1))[-1, 0] == 1.0          # node o + n is x = 1


def test_one_node_thick_block_maps_to_x_zero():
    """N = 17, n = 8: the upper layer o = 16 holds one node; its span is 0 and the
    axis maps to x = 0 (R36), for grid and query decode alike."""
    dims = (17, 9, 9)
    mesh = (stretched(17, 1), stretched(9, 2), stretched(9, 3))
    b = sampler.decompose(dims, (8, 8, 8), mesh)[2]
    assert b.origin[0] == 16
    xs = decode.mesh_grid_coords(b, (1, 2, 2))
    assert np.all(xs[:, 0] == 0.0) and np.all(np.isfinite(xs))
