"""One block's INR Phi: R^3 -> R^D (Eq. 1): hash-grid tables +
MLP weights + Adam state, laid out as one flat parameter vector in the
declared order ("encoding tables by level, MLP layer by layer"):

    theta_0 (S_0 x F, entry-major) ... theta_{L-1}, W_0 (out x in, row-major),
    b_0, W_1, b_1, ..., W_H, b_H          (b_k present iff mlp_bias)

Initialization (P silent; R14): tables U[-1e-4, 1e-4], weights
U[-sqrt(6/fan_in), +sqrt(6/fan_in)], biases 0.  Parameter j of block b draws
U = u01(Philox4x32-10(key(seed, 0), ctr = (j, b, 0, 0)).x) and takes
fl32(lo + (hi - lo) U) evaluated in float64 (one multiply, two adds, each
rounded), so any independent implementation of the formula starts from the
same float32 values.
"""
import dataclasses
import math

import numpy as np

from . import encoding, philox


@dataclasses.dataclass
class Config:
    levels: int = 16
    features: int = 2
    log2_table_size: int = 19
    base_resolution: int = 4
    per_level_scale: float = 2.0
    mlp_width: int = 64
    mlp_hidden_layers: int = 3
    out_dim: int = 1
    mlp_bias: int = 1

    @property
    def table_size(self):
        return 1 << self.log2_table_size

    def resolutions(self):
        return [encoding.level_resolution(self.base_resolution, self.per_level_scale, l) for l in range(self.levels)]

    def level_sizes(self):
        return [encoding.level_table_size(n, self.table_size)[0] for n in self.resolutions()]

    def layer_shapes(self):
        """[(out, in)] for the H+1 weight matrices (R16)."""
        W, H = self.mlp_width, self.mlp_hidden_layers
        ins = [self.levels * self.features] + [W] * H
        outs = [W] * H + [self.out_dim]
        return list(zip(outs, ins))

    def tensor_layout(self):
        """[(name, shape, offset)] in declared order."""
        out, off = [], 0
        for l, s in enumerate(self.level_sizes()):
            out.append((f"table{l}", (s, self.features), off))
            off += s * self.features
        for k, (o, i) in enumerate(self.layer_shapes()):
            out.append((f"W{k}", (o, i), off))
            off += o * i
            if self.mlp_bias:
                out.append((f"b{k}", (o,), off))
                off += o
        return out

    def param_count(self):
        name, shape, off = self.tensor_layout()[-1]
        return off + int(np.prod(shape))


def init_params(cfg, seed, block_id):
    """float32 flat parameter vector (see module docstring)."""
    P = cfg.param_count()
    vals = np.zeros(P, dtype=np.float32)
    key = philox.stream_key(seed, 0)
    for name, shape, off in cfg.tensor_layout():
        n = int(np.prod(shape))
        if name.startswith("b"):
            continue                       # biases start at 0
        if name.startswith("table"):
            a = 1e-4
        else:
            a = math.sqrt(6.0 / shape[1])  # He-uniform on fan_in (R14)
        lo, hi = -a, a
        j = np.arange(off, off + n, dtype=np.uint64)
        u = philox.philox4x32_10((j, np.full_like(j, block_id), np.zeros_like(j), np.zeros_like(j)), key)[0]
        U = philox.u01(u).astype(np.float64)
        vals[off:off + n] = (lo + (hi - lo) * U).astype(np.float32)
    return vals


class InrModel:
    """Oracle model: float64 parameters + Adam state + its block and range."""

    def __init__(self, cfg, block, seed, params=None):
        self.cfg = cfg
        self.block = block
        self.seed = int(seed)
        p0 = init_params(cfg, seed, block.block_id) if params is None else np.asarray(params, np.float32)
        self.p = p0.astype(np.float64)
        self.m = np.zeros_like(self.p)
        self.v = np.zeros_like(self.p)
        self.g = np.zeros_like(self.p)
        self.step = 0
        self.vmin, self.vmax = 0.0, 1.0

    def view(self, flat, name):
        for nm, shape, off in self.cfg.tensor_layout():
            if nm == name:
                return flat[off:off + int(np.prod(shape))].reshape(shape)
        raise KeyError(name)

    def tables(self, flat=None):
        flat = self.p if flat is None else flat
        return [self.view(flat, f"table{l}") for l in range(self.cfg.levels)]

    def mlp(self, flat=None):
        flat = self.p if flat is None else flat
        K = self.cfg.mlp_hidden_layers + 1
        Ws = [self.view(flat, f"W{k}") for k in range(K)]
        bs = [self.view(flat, f"b{k}") if self.cfg.mlp_bias else None for k in range(K)]
        return Ws, bs
