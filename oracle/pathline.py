"""Pathlines over a temporal window of decoded vector fields (NEXT-2).

P:L411 "Pathlines, which are integral curves of a time-varying vector field
V(x) beginning from a seed spatial coordinate x0 at time t0 ... Numerical
integration algorithms, such as the Euler or Runge-Kutta methods";
P:L416 "P=pathline(negate(reverse(W)),...)"; "the velocity field was
decoded back to the original mesh grid ... on an on-demand basis, allowing for
the retention of only two additional copies of the mesh grid at any given
time.  The operation of negate ... multiplied all field values ... by -1 ...
reverse ... the alteration of the index of the i-th element to N-i-1";
S:L391-408 (reverse / negate), S:L495-512 (rk4_step, trace_pathlines).

Readings (R29-R31): positions in global node units, velocity values
in node units per unit time, trilinear in space per channel and
linear in time between adjacent window elements; classical RK4 with
a fixed step: each window interval [t_i, t_{i+1}] is split into
k_i = ceil((t_{i+1} - t_i) / dt) equal substeps so no stage straddles a
window element; a seed terminates before the first step any of whose four
stage positions (or the result) leaves [0, N-1]^3.  The reversed window's
time axis is tau_i = t_{N-1} - t_{N-1-i}, so forward tracing in tau over
negate(reverse(W)) is backward tracing in t.

Test infrastructure only: numpy float64, no GPU code.
"""
import math

import numpy as np

from . import sampler

WINDOW_EXHAUSTED, OUT_OF_DOMAIN, MAX_STEPS = 0, 1, 2


def reverse_negate(grids, times, reverse=False, negate=False):
    """The window view negate(reverse(W)): element i of the
    reversed window is element N-1-i of W at tau_i = t_{N-1} - t_{N-1-i};
    negation is a sign on every value.  Returns (grids, times, sign)."""
    grids, times = list(grids), [float(t) for t in times]
    if reverse:
        last = times[-1]
        grids = grids[::-1]
        times = [last - t for t in times[::-1]]
    return grids, times, (-1.0 if negate else 1.0)


def in_domain(p, dims):
    hi = np.asarray(dims, np.float64) - 1.0
    return np.all((p >= 0.0) & (p <= hi[None, :]), axis=1)


def velocity(g0, g1, alpha, p, sign):
    """sign * ((1 - alpha) V_0(p) + alpha V_1(p)), V_i trilinear on grid i."""
    v0 = sampler.trilinear(g0, p)
    v1 = sampler.trilinear(g1, p)
    return sign * ((1.0 - alpha) * v0 + alpha * v1)


def rk4_step(f, p, t, h):
    """Classical fourth-order Runge-Kutta.  f(p, t) -> dp/dt.
    Returns (p', stage positions)."""
    k1 = f(p, t)
    p2 = p + 0.5 * h * k1
    k2 = f(p2, t + 0.5 * h)
    p3 = p + 0.5 * h * k2
    k3 = f(p3, t + 0.5 * h)
    p4 = p + h * k3
    k4 = f(p4, t + h)
    return p + (h / 6.0) * (k1 + 2.0 * k2 + 2.0 * k3 + k4), (p2, p3, p4)


def trace(grids, times, seeds, dt, max_steps, sign=1.0):
    """Trace every seed forward in time across the window.

    grids: list of (Nz, Ny, Nx, 3) velocity arrays at strictly increasing
    `times`; seeds (M, 3) node units.  Returns (vertices (M, max_steps + 1, 5)
    float64 rows (x, y, z, t, |V|) padded with NaN, counts (M,), reasons (M,)).
    """
    grids = [np.asarray(g, np.float64) for g in grids]
    dims = (grids[0].shape[2], grids[0].shape[1], grids[0].shape[0])
    seeds = np.asarray(seeds, np.float64)
    M = seeds.shape[0]
    out = np.full((M, max_steps + 1, 5), np.nan)
    counts = np.zeros(M, np.int64)
    reasons = np.full(M, WINDOW_EXHAUSTED, np.int64)
    p = seeds.copy()
    alive = in_domain(p, dims)
    reasons[~alive] = OUT_OF_DOMAIN
    if len(grids) < 2:
        raise ValueError("a pathline window needs at least two elements")
    t0 = times[0]

    def record(idx, pos, t, vel):
        out[idx, counts[idx], :3] = pos
        out[idx, counts[idx], 3] = t
        out[idx, counts[idx], 4] = np.linalg.norm(vel, axis=1)
        counts[idx] += 1

    a = np.flatnonzero(alive)
    record(a, p[a], t0, velocity(grids[0], grids[1], 0.0, p[a], sign))
    steps = np.zeros(M, np.int64)
    for i in range(len(grids) - 1):
        ta, tb = times[i], times[i + 1]
        k = max(1, int(math.ceil((tb - ta) / dt - 1e-12)))
        h = (tb - ta) / k
        g0, g1 = grids[i], grids[i + 1]

        def f(q, t):
            return velocity(g0, g1, (t - ta) / (tb - ta), q, sign)

        for j in range(k):
            a = np.flatnonzero(alive)
            if a.size == 0:
                break
            full = steps[a] >= max_steps
            reasons[a[full]] = MAX_STEPS
            alive[a[full]] = False
            a = a[~full]
            if a.size == 0:
                break
            t = ta + j * h
            pn, stages = rk4_step(f, p[a], t, h)
            ok = in_domain(pn, dims)
            for q in stages:
                ok &= in_domain(q, dims)
            reasons[a[~ok]] = OUT_OF_DOMAIN
            alive[a[~ok]] = False
            a = a[ok]
            p[a] = pn[ok]
            steps[a] += 1
            tn = ta + (j + 1) * h
            record(a, p[a], tn, velocity(g0, g1, (tn - ta) / (tb - ta), p[a], sign))
    return out, counts, reasons
