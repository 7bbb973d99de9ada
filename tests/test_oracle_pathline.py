"""Pins of oracle/pathline.py (NEXT-2) against closed forms and the
mathematics of RK4, never against itself."""
import math

import numpy as np
import torch

import synth
from oracle import pathline as pl

N = 17
DIMS = (N, N, N)


def const_grid(v):
    g = np.zeros((N, N, N, 3))
    g[...] = v
    return g


def linear_x_grid(a=1.0):
    """V = (a x, 0, 0): trilinear reproduces it exactly."""
    g = np.zeros((N, N, N, 3))
    g[..., 0] = a * np.arange(N)[None, None, :]
    return g


def test_constant_field_is_exact():
    # constant V = (1, 0, 0), dt = 0.1, p = (0, 0, 0) -> (0.1, 0, 0) per step
    g = const_grid((1.0, 0.0, 0.0))
    seeds = np.array([[0.0, 0.0, 0.0], [3.0, 4.0, 5.0]])
    v, c, r = pl.trace([g, g], [0.0, 1.0], seeds, 0.1, 100)
    assert list(c) == [11, 11] and list(r) == [pl.WINDOW_EXHAUSTED] * 2
    assert abs(v[0, 1, 0] - 0.1) < 1e-15
    assert np.allclose(v[:, -1 - (100 - 10), :3], seeds + [1.0, 0, 0], atol=1e-12, rtol=0)
    assert np.allclose(v[0, :11, 3], np.arange(11) * 0.1, atol=1e-15)
    assert np.allclose(v[0, :11, 4], 1.0)


def test_zero_field_leaves_seeds_in_place():
    g = const_grid((0.0, 0.0, 0.0))
    seeds = np.random.default_rng(0).random((20, 3)) * (N - 1)
    v, c, r = pl.trace([g, g, g], [0.0, 0.5, 1.5], seeds, 0.25, 100)
    assert np.all(c == 7) and np.all(v[:, 6, :3] == seeds)


def test_linear_field_rk4_polynomial_and_exponential():
    # V = (x, 0, 0) from x = 1, one step h: RK4 gives the degree-4 Taylor
    # polynomial of e^h exactly, and e^h to O(h^5)
    g = linear_x_grid()
    for h in (0.1, 0.05):
        v, c, _ = pl.trace([g, g], [0.0, h], np.array([[1.0, 2.0, 2.0]]), h, 10)
        x1 = v[0, 1, 0]
        assert abs(x1 - (1 + h + h * h / 2 + h ** 3 / 6 + h ** 4 / 24)) < 1e-15
        assert abs(x1 - math.exp(h)) < h ** 5 / 100
    # global convergence: error at t = 1 shrinks ~16x when dt halves
    errs = []
    for dt in (0.1, 0.05):
        v, c, _ = pl.trace([g, g], [0.0, 1.0], np.array([[1.0, 2.0, 2.0]]), dt, 100)
        errs.append(abs(v[0, c[0] - 1, 0] - math.e))
    assert 12 < errs[0] / errs[1] < 20


def test_time_interpolation_is_linear():
    # V_0 = 0, V_1 = (1, 0, 0) at t = 0, 1: dx/dt = t -> x(1) = x0 + 1/2 exactly
    # (RK4 is exact for polynomials in t of degree <= 4)
    v, c, _ = pl.trace([const_grid(0.0), const_grid((1.0, 0.0, 0.0))], [0.0, 1.0],
                       np.array([[2.0, 2.0, 2.0]]), 0.3, 100)
    assert c[0] == 5
    assert abs(v[0, 4, 0] - 2.5) < 1e-14 and abs(v[0, 4, 3] - 1.0) < 1e-15


def test_out_of_domain_terminates_before_leaving():
    g = const_grid((1.0, 0.0, 0.0))
    v, c, r = pl.trace([g, g], [0.0, 10.0], np.array([[14.5, 3.0, 3.0], [-1.0, 0.0, 0.0]]), 1.0, 100)
    assert r[0] == pl.OUT_OF_DOMAIN and c[0] == 2 and v[0, 1, 0] == 15.5
    assert r[1] == pl.OUT_OF_DOMAIN and c[1] == 0


def test_max_steps():
    g = const_grid((0.1, 0.0, 0.0))
    v, c, r = pl.trace([g, g], [0.0, 10.0], np.array([[1.0, 1.0, 1.0]]), 0.5, 7)
    assert r[0] == pl.MAX_STEPS and c[0] == 8


def test_reverse_negate_is_backward_integration():
    # a steady field duplicated across the window: forward tracing over
    # negate(reverse(W)) equals RK4 with a negative step on the original field
    gv = synth.taylor_green_volume(N, 0.0, amp=2.0).double().numpy()
    W, times = [gv, gv, gv], [0.0, 0.7, 2.0]
    rg, rt, sgn = pl.reverse_negate(W, times, reverse=True, negate=True)
    assert rt == [0.0, 1.3, 2.0] and sgn == -1.0
    seeds = np.random.default_rng(3).random((16, 3)) * 8 + 4
    v, c, r = pl.trace(rg, rt, seeds, 0.1, 1000, sgn)
    # independent backward integration: explicit RK4 with h < 0 over the same substeps
    p = seeds.copy()
    f = lambda q: pl.velocity(gv, gv, 0.0, q, 1.0)
    for (ta, tb) in ((2.0, 0.7), (0.7, 0.0)):
        k = math.ceil((ta - tb) / 0.1 - 1e-12)
        h = -(ta - tb) / k
        for _ in range(k):
            k1 = f(p); k2 = f(p + 0.5 * h * k1); k3 = f(p + 0.5 * h * k2); k4 = f(p + h * k3)
            p = p + h / 6 * (k1 + 2 * k2 + 2 * k3 + k4)
    ok = r == pl.WINDOW_EXHAUSTED
    assert ok.sum() >= 8
    end = v[np.arange(16), c - 1, :3]
    assert np.max(np.abs(end[ok] - p[ok])) < 1e-10


def test_taylor_green_round_trip():
    # P:L434 "both forward and backward tracing methods can yield nearly identical
    # results": backward over negate(reverse(W)), then forward from the end points
    n = 33
    times = [0.0, 0.5, 1.0, 1.5, 2.0]
    lat = synth.lattice((n, n, n))
    W = [synth.taylor_green(lat, (n, n, n), t, amp=3.0).numpy() for t in times]
    seeds = np.random.default_rng(5).random((32, 3)) * 16 + 8
    rg, rt, sgn = pl.reverse_negate(W, times, reverse=True, negate=True)
    vb, cb, rb = pl.trace(rg, rt, seeds, 0.05, 10000, sgn)
    ok = rb == pl.WINDOW_EXHAUSTED
    ends = vb[np.arange(32), cb - 1, :3][ok]
    vf, cf, rf = pl.trace(W, times, ends, 0.05, 10000)
    back = vf[np.arange(ends.shape[0]), cf - 1, :3]
    assert ok.sum() >= 16 and np.all(rf == pl.WINDOW_EXHAUSTED)
    assert np.max(np.abs(back - seeds[ok])) < 0.05


def test_reverse_is_an_involution():
    W, t = ["a", "b", "c"], [0.0, 1.0, 3.0]
    g1, t1, _ = pl.reverse_negate(W, t, reverse=True)
    assert g1 == ["c", "b", "a"] and t1 == [0.0, 2.0, 3.0]
    g2, t2, _ = pl.reverse_negate(g1, t1, reverse=True)
    assert g2 == W and t2 == t
