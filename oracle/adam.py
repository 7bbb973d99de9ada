"""Adam and the step learning-rate schedule ("Adam optimizer ...
beta1=0.9 and beta2=0.999 ... learning rate schedule that starts at 1e-2 and
decays by a factor of 0.8 every 500 steps").

R12: PyTorch torch.optim.Adam semantics (the paper trained in PyTorch,
P:L215): eps = 1e-8, dense update of every entry, no weight decay.
R13: lr at 0-based step s is lr0 * 0.8^floor(s/500).

R37 (NEXT-4, a flagged semantics change versus R12, off by default): the
touched-only ("sparse") variant updates a hash-table parameter only if its
aligned group of 8 consecutive table entries' floats (one 32-byte sector,
table-relative indices [8k, 8k + 8)) holds a non-zero gradient this step; the
group is then updated exactly as R12 (members with g = 0 included), every
other group keeps p, m and v unchanged.  MLP parameters always take R12.
"""
import math
import numpy as np


def lr_at(s, lr0=1e-2, decay=0.8, every=500):
    return lr0 * decay ** (s // every)


def adam_update(p, g, m, v, t, lr, beta1=0.9, beta2=0.999, eps=1e-8):
    """One in-place update at 1-based step t (PyTorch form):
    m <- b1 m + (1-b1) g;  v <- b2 v + (1-b2) g^2;
    p <- p - (lr / (1 - b1^t)) * m / (sqrt(v) / sqrt(1 - b2^t) + eps)."""
    m *= beta1
    m += (1.0 - beta1) * g
    v *= beta2
    v += (1.0 - beta2) * g * g
    bc1 = 1.0 - beta1 ** t
    bc2 = 1.0 - beta2 ** t
    denom = np.sqrt(v) / math.sqrt(bc2) + eps
    p -= (lr / bc1) * m / denom


def touched_groups(g_table, group=8):
    """Boolean mask over the elements of one table tensor (flat): True where the
    element's aligned group of `group` floats holds a non-zero gradient (R37)."""
    g = np.asarray(g_table).reshape(-1)
    n = g.size
    pad = (-n) % group
    nz = np.concatenate([g != 0, np.zeros(pad, bool)]).reshape(-1, group).any(axis=1)
    return np.repeat(nz, group)[:n]


def adam_update_sparse(p, g, m, v, t, lr, table_slices, beta1=0.9, beta2=0.999, eps=1e-8):
    """R37: adam_update on the MLP parameters and on the touched groups of every
    table tensor (table_slices: (offset, length) of each table in the flat
    vectors); untouched groups keep p, m, v.  In place."""
    sel = np.ones(p.shape, bool)
    for off, n in table_slices:
        sel[off:off + n] = touched_groups(g[off:off + n])
    ps, ms, vs = p[sel], m[sel], v[sel]
    adam_update(ps, g[sel], ms, vs, t, lr, beta1, beta2, eps)
    p[sel], m[sel], v[sel] = ps, ms, vs
