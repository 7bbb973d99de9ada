"""Sort-last direct-query volume rendering of a DNR (NEXT-3).

P:L268 "our volume renderer utilizes the sample-streaming algorithm and the
macro-cell acceleration structure proposed by Wu et al."; "a base
renderer using their sample-streaming algorithm ... macro-cell acceleration
structure for adaptive sampling ... a sort-last parallel rendering system ...
does not require decoding the neural representation back to a grid";
S:L446-494 (Camera, TransferFunction, MacroCellGrid, Image, ray_march,
build_macrocells, render_dnr).

This is the plain definition (R32-R35): every sample of every ray
is evaluated (no macro-cell skipping, no early-exit scheduling beyond the
rule itself), one ray at a time, in float64.

* camera: pinhole at `eye` looking at `look`, vertical field of view `fovy`
  degrees; the ray of pixel (px, py) (py = 0 the top row) has direction
  normalize(f + a u_x r + b u_y u') with a = (2 (px + 0.5) / W - 1) tan(fovy/2) W/H,
  b = (1 - 2 (py + 0.5) / H) tan(fovy/2), f = normalize(look - eye),
  r = normalize(f x up), u' = r x f;
* samples at t_k = (k + 0.5) step along the ray from the eye (k >= 0, global,
  so bricks split a ray without moving its samples); a brick [lo, hi] takes the
  k with t_enter <= t_k < t_exit;
* transfer function: s = clamp((v - vmin) / (vmax - vmin), 0, 1) -> RGBA by
  piecewise-linear interpolation of sorted control points (constant beyond the
  ends); opacity correction a = 1 - (1 - a_tf)^(step / base_step);
  front to back C += (1 - A) a c, A += (1 - A) a; stop once A >= stop_alpha;
* sort-last: fragments (C, A, t_enter) per pixel per brick, composited front to
  back in t_enter order, then the background: C + (1 - A) bg.

Test infrastructure only.
"""
import math

import numpy as np


def camera_rays(eye, look, up, fovy, width, height):
    """(H*W, 3) unit directions, row-major from the top-left pixel."""
    eye, look, up = (np.asarray(v, np.float64) for v in (eye, look, up))
    f = look - eye
    f = f / np.linalg.norm(f)
    r = np.cross(f, up)
    r = r / np.linalg.norm(r)
    u = np.cross(r, f)
    th = math.tan(math.radians(fovy) / 2.0)
    px, py = np.meshgrid(np.arange(width), np.arange(height))
    a = (2.0 * (px.reshape(-1) + 0.5) / width - 1.0) * th * (width / height)
    b = (1.0 - 2.0 * (py.reshape(-1) + 0.5) / height) * th
    d = f[None, :] + a[:, None] * r[None, :] + b[:, None] * u[None, :]
    return d / np.linalg.norm(d, axis=1, keepdims=True)


def box_interval(eye, d, lo, hi):
    """Slab test: (t_enter, t_exit) of the ray eye + t d with the box [lo, hi],
    t_enter clamped at 0; t_exit <= t_enter means no intersection."""
    t0, t1 = 0.0, math.inf
    for a in range(3):
        if d[a] != 0.0:
            ta = (lo[a] - eye[a]) / d[a]
            tb = (hi[a] - eye[a]) / d[a]
            t0 = max(t0, min(ta, tb))
            t1 = min(t1, max(ta, tb))
        elif not (lo[a] <= eye[a] <= hi[a]):
            return 0.0, 0.0
    return t0, t1


def tf_lookup(s, points, rgba):
    """Piecewise-linear RGBA at normalized s."""
    points = np.asarray(points, np.float64)
    rgba = np.asarray(rgba, np.float64)
    return np.array([np.interp(s, points, rgba[:, c]) for c in range(4)])


def sample_ts(t_enter, t_exit, step):
    """The global sample parameters t_k = (k + 0.5) step in [t_enter, t_exit)."""
    if not t_exit > t_enter:
        return np.zeros(0)
    k = max(0, math.ceil(t_enter / step - 0.5) - 1)   # one early: the t >= t_enter test decides
    ts = []
    while True:
        t = (k + 0.5) * step
        if t >= t_exit:
            break
        if t >= t_enter:
            ts.append(t)
        k += 1
    return np.array(ts)


def march(values, step, tf, stop_alpha=0.99):
    """Front-to-back emission-absorption over the sample values in ray order
    (S:L468-476).  Returns (C (3,), A)."""
    C = np.zeros(3)
    A = 0.0
    for v in values:
        s = min(max((v - tf["vmin"]) / (tf["vmax"] - tf["vmin"]), 0.0), 1.0)
        r, g, b, a_tf = tf_lookup(s, tf["points"], tf["rgba"])
        a = 1.0 - (1.0 - a_tf) ** (step / tf["base_step"])
        w = (1.0 - A) * a
        C = C + w * np.array([r, g, b])
        A = A + w
        if A >= stop_alpha:
            break
    return C, A


def ray_segment(field, eye, d, t_enter, t_exit, step, tf, stop_alpha=0.99):
    """One ray through one brick; field(p (3,)) -> value.  Returns (C, A)."""
    ts = sample_ts(t_enter, t_exit, step)
    return march([field(eye + t * d) for t in ts], step, tf, stop_alpha)


def render_brick(field, cam, lo, hi, step, tf, stop_alpha=0.99, batch_field=None):
    """Fragments of one brick: (H*W, 5) rows (C_r, C_g, C_b, A, t_enter);
    t_enter = +inf where the ray misses the brick.  batch_field(P (n, 3))
    evaluates all sample positions at once instead of field (same values: the
    samples after an early stop are computed but not composited)."""
    eye = np.asarray(cam["eye"], np.float64)
    dirs = camera_rays(cam["eye"], cam["look"], cam["up"], cam["fovy"], cam["width"], cam["height"])
    out = np.zeros((dirs.shape[0], 5))
    segs = []
    for i, d in enumerate(dirs):
        t0, t1 = box_interval(eye, d, lo, hi)
        segs.append((t0, t1, sample_ts(t0, t1, step)))
    if batch_field is not None:
        pts = [eye[None, :] + ts[:, None] * d[None, :] for (_, _, ts), d in zip(segs, dirs)]
        allv = batch_field(np.concatenate(pts)) if sum(p.shape[0] for p in pts) else np.zeros(0)
        offs = np.cumsum([0] + [p.shape[0] for p in pts])
    for i, d in enumerate(dirs):
        t0, t1, ts = segs[i]
        if not t1 > t0:
            out[i, 4] = math.inf
            continue
        if batch_field is not None:
            vals = allv[offs[i]:offs[i + 1]]
        else:
            vals = [field(eye + t * d) for t in ts]
        C, A = march(vals, step, tf, stop_alpha)
        out[i, :3], out[i, 3], out[i, 4] = C, A, t0
    return out


def composite(fragments, background=(0.0, 0.0, 0.0)):
    """Sort-last: fragments (nfrag, H*W, 5) -> image (H*W, 4) RGBA, front to back
    by t_enter, background last."""
    frags = np.asarray(fragments, np.float64)
    n = frags.shape[1]
    img = np.zeros((n, 4))
    bg = np.asarray(background, np.float64)
    for i in range(n):
        order = np.argsort(frags[:, i, 4], kind="stable")
        C = np.zeros(3)
        A = 0.0
        for j in order:
            if not np.isfinite(frags[j, i, 4]):
                continue
            C = C + (1.0 - A) * frags[j, i, :3]
            A = A + (1.0 - A) * frags[j, i, 3]
        img[i, :3] = C + (1.0 - A) * bg
        img[i, 3] = A
    return img
