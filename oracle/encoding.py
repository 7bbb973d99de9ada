"""Multiresolution hash-grid encoding ("multi-resolution hash encoding
layer", "16-level hash-grid encoding layer with 4 features per level.
Each level uses a hash table of 2^19 entries and the base level resolution is
4 with a scaling factor of 2"), made concrete by SPEC S:L147-164
and DESIGN.md readings R1-R4, R20.

Index math is float32 / uint32 (R4, R20): pos = fl32(x * N_l) with no fused
multiply-add, i = min(floor(pos), N_l - 1), w = pos - i (exact in float32).
Feature blending is float64.
"""
import numpy as np

PRIME_Y = np.uint32(2654435761)   # S:L236 spatial-hash primes (1, 2654435761, 805459861)
PRIME_Z = np.uint32(805459861)


def level_resolution(base_resolution, per_level_scale, l):
    """N_l = floor(N_min * b^l), evaluated in float64 then truncated (R3)."""
    return int(np.floor(np.float64(base_resolution) * np.float64(per_level_scale) ** l))


def level_table_size(n_l, table_size):
    """S_l = (N_l+1)^3 if that fits in T (dense level) else T (hashed) (R2)."""
    dense = (n_l + 1) ** 3
    return (dense, True) if dense <= table_size else (table_size, False)


def hash_index(vx, vy, vz, table_size):
    """((v_x * 1) xor (v_y * 2654435761) xor (v_z * 805459861)) mod T in uint32
    arithmetic (R1).  T | 2^32, so uint32 wrap-around before the mask
    equals the exact big-integer result."""
    vx = np.asarray(vx, dtype=np.uint32)
    vy = np.asarray(vy, dtype=np.uint32)
    vz = np.asarray(vz, dtype=np.uint32)
    with np.errstate(over="ignore"):
        h = vx ^ (vy * PRIME_Y) ^ (vz * PRIME_Z)
    return h & np.uint32(table_size - 1)


def dense_index(vx, vy, vz, n_l):
    """x-fastest dense index v_x + (N+1)(v_y + (N+1) v_z) (R2)."""
    s = np.int64(n_l + 1)
    return (np.asarray(vx, np.int64) + s * (np.asarray(vy, np.int64) + s * np.asarray(vz, np.int64))).astype(np.uint32)


def level_lookup(x, n_l):
    """x: (n,3) float32 in [0,1] (clamped here; R4) ->
    cell (n,3) int64 and fractional weights (n,3) float32.

    pos_d = fl32(x_d * N_l); i_d = min(floor(pos_d), N_l - 1); w_d = pos_d - i_d.
    """
    x = np.clip(np.asarray(x, dtype=np.float32), np.float32(0.0), np.float32(1.0))
    pos = x * np.float32(n_l)                      # one IEEE float32 multiply
    cell = np.minimum(np.floor(pos).astype(np.int64), n_l - 1)
    w = pos - cell.astype(np.float32)              # exact (Sterbenz)
    return cell, w


def corner_indices_and_weights(x, n_l, table_size):
    """For the 8 corners c = 0..7 (bit0 -> x, bit1 -> y, bit2 -> z) of the
    level-l cell containing x: uint32 table index and float64 trilinear weight
    Pi_d (bit ? w_d : 1 - w_d)."""
    cell, w = level_lookup(x, n_l)
    size, dense = level_table_size(n_l, table_size)
    w64 = w.astype(np.float64)
    n = cell.shape[0]
    idx = np.empty((n, 8), dtype=np.uint32)
    wt = np.empty((n, 8), dtype=np.float64)
    for c in range(8):
        b = [(c >> d) & 1 for d in range(3)]
        v = [cell[:, d] + b[d] for d in range(3)]
        if dense:
            idx[:, c] = dense_index(v[0], v[1], v[2], n_l)
        else:
            idx[:, c] = hash_index(v[0], v[1], v[2], table_size)
        wc = np.ones(n, dtype=np.float64)
        for d in range(3):
            wc = wc * (w64[:, d] if b[d] else (1.0 - w64[:, d]))
        wt[:, c] = wc
    return idx, wt


def encode_forward(tables, x, resolutions, table_size):
    """feat[:, l*F + f] = sum_{c=0..7} w_c * theta_l[idx_c, f], summed in c order,
    levels concatenated.

    tables: list of (S_l, F) float64 arrays.  Returns (feat (n, L*F) float64,
    idx (n, L, 8) uint32, wt (n, L, 8) float64)."""
    n = np.asarray(x).shape[0]
    L = len(tables)
    F = tables[0].shape[1]
    feat = np.zeros((n, L * F), dtype=np.float64)
    idx_all = np.empty((n, L, 8), dtype=np.uint32)
    wt_all = np.empty((n, L, 8), dtype=np.float64)
    for l in range(L):
        idx, wt = corner_indices_and_weights(x, resolutions[l], table_size)
        acc = np.zeros((n, F), dtype=np.float64)
        for c in range(8):
            acc = acc + wt[:, c:c + 1] * tables[l][idx[:, c]]
        feat[:, l * F:(l + 1) * F] = acc
        idx_all[:, l] = idx
        wt_all[:, l] = wt
    return feat, idx_all, wt_all


def encode_backward(dfeat, idx, wt, table_shapes):
    """d theta_l[idx_c][f] += w_c * dfeat[l*F + f], accumulated in sample order
    then corner order (R21).  np.add.at applies the updates
    sequentially in the order given (unbuffered)."""
    n, L, _ = idx.shape
    grads = [np.zeros(s, dtype=np.float64) for s in table_shapes]
    for l in range(L):
        F = table_shapes[l][1]
        contrib = wt[:, l, :, None] * dfeat[:, None, l * F:(l + 1) * F]   # (n, 8, F)
        np.add.at(grads[l], idx[:, l, :].reshape(-1), contrib.reshape(-1, F))
    return grads
