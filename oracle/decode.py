"""Inference: direct coordinate queries and decode-to-grid (P:L175-176:
"the neural network can output v on-demand for any arbitrary coordinate ...
it may be necessary to decode the neural representation back to its original
grid-based representation"), plus the PSNR metric
(R18).

Coordinate math is float32 and mirrors DESIGN.md R5/R19:
  query: block b_d = min(floor(p_d / n_d), B_d - 1), x = fl32(fl32(p - o) / n)
  grid:  x_j = fl32(j / R), j < R per axis, x-fastest output.
"""
import numpy as np

from . import fit, sampler


def denormalize(y, vmin, vmax):
    """v = y (vmax - vmin) + vmin (inverse of P:L173 value normalization), per
    channel when vmin, vmax are (D,) arrays."""
    lo = np.asarray(vmin, np.float64)
    return np.asarray(y, np.float64) * (np.asarray(vmax, np.float64) - lo) + lo


def _channels(y):
    """(n, 1) -> (n,) for scalar fields; (n, D) unchanged."""
    return y[:, 0] if y.shape[1] == 1 else y


def grid_coords(res):
    """Block-normalized lattice x_j = fl32(j / R_d), x fastest -> (Rz*Ry*Rx, 3) float32."""
    ax = [np.arange(r, dtype=np.float32) / np.float32(r) for r in res]
    z, y, x = np.meshgrid(ax[2], ax[1], ax[0], indexing="ij")
    return np.stack([x.reshape(-1), y.reshape(-1), z.reshape(-1)], axis=1)


def mesh_grid_coords(block, count):
    """Rectilinear block: the block-normalized coordinates of its first count_d
    nodes, x_j = fl32((X_{o+j} - P_lo) / (P_hi - P_lo)) (R36), x fastest."""
    lo, hi = block.physical_box()
    span = hi - lo
    # a block one node thick on an axis (span 0) maps that axis to x = 0
    ax = [(((block.mesh[d][block.origin[d]:block.origin[d] + count[d]] - lo[d]) / span[d]) if span[d] > 0 else
           np.zeros(count[d])).astype(np.float32) for d in range(3)]
    z, y, x = np.meshgrid(ax[2], ax[1], ax[0], indexing="ij")
    return np.stack([x.reshape(-1), y.reshape(-1), z.reshape(-1)], axis=1)


def decode_grid(model, res, chunk=1 << 16):
    """Decoded values (R_z, R_y, R_x) float64 in data units, or (R_z, R_y, R_x, D).
    A rectilinear model decodes its nodes (res = the node counts, R36)."""
    xs = grid_coords(res) if model.block.mesh is None else mesh_grid_coords(model.block, res)
    D = model.cfg.out_dim
    out = np.empty((xs.shape[0], D), dtype=np.float64)
    for a in range(0, xs.shape[0], chunk):
        y, _ = fit.forward(model, xs[a:a + chunk])
        out[a:a + chunk] = denormalize(y, model.vmin, model.vmax)
    return out.reshape(res[2], res[1], res[0]) if D == 1 else out.reshape(res[2], res[1], res[0], D)


def route(p, n, global_dims):
    """Owner block coordinate per axis: min(max(floor(p/n), 0), B - 1) (R5)."""
    p = np.asarray(p, np.float32)
    n = np.asarray(n, np.int64)
    g = (np.asarray(global_dims, np.int64) + n - 1) // n
    b = np.floor(p / n.astype(np.float32)).astype(np.int64)
    return np.clip(b, 0, g - 1)


def decode_query(models, p, strict=False):
    """models: dict block_id -> InrModel (all same n, global_dims).  p: (q,3)
    float32 global node coordinates.  Returns float64 values; in strict mode
    coordinates outside [0, N-1] raise ValueError."""
    p = np.asarray(p, np.float32)
    any_m = next(iter(models.values()))
    n = any_m.block.n
    gd = any_m.block.global_dims
    if strict and (np.any(p < 0) or np.any(p > (gd - 1).astype(np.float32))):
        raise ValueError("query outside the global domain")
    bc = route(p, n, gd)
    g = (gd + n - 1) // n
    bid = (bc[:, 2] * g[1] + bc[:, 1]) * g[0] + bc[:, 0]
    D = any_m.cfg.out_dim
    out = np.full((p.shape[0], D), np.nan)
    for b in np.unique(bid):
        m = models[int(b)]
        sel = bid == b
        if m.block.mesh is None:
            o = m.block.origin.astype(np.float32)
            x = (p[sel] - o[None, :]) / m.block.n.astype(np.float32)[None, :]
        else:   # R36: node index -> physical coordinate -> the block's normalized box
            lo, hi = m.block.physical_box()
            P = np.stack([sampler.index_to_physical(m.block.mesh[d], p[sel][:, d].astype(np.float64))
                          for d in range(3)], axis=1)
            span = hi - lo
            x = np.where(span[None, :] > 0, (P - lo[None, :]) / np.where(span > 0, span, 1.0)[None, :], 0.0)
        y, _ = fit.forward(m, x.astype(np.float32))
        out[sel] = denormalize(y, m.vmin, m.vmax)
    return _channels(out)


def sse_normalized(pred, ref, vmin, vmax):
    """Sum of squared errors in normalized units, sum ((pred - ref)/(vmax - vmin))^2
    (over voxels and channels)."""
    span = np.asarray(vmax, np.float64) - np.asarray(vmin, np.float64)
    # a constant channel is 0 in normalized units on both sides
    d = np.where(span > 0, (np.asarray(pred, np.float64) - np.asarray(ref, np.float64)) / np.where(span > 0, span, 1.0),
                 0.0)
    return float(np.sum(d * d))


psnr = sampler.psnr
psnr_from_mse = sampler.psnr_from_mse
