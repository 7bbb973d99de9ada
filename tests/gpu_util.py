"""Helpers shared by the -m gpu tests: build matching (GPU model, oracle
model) pairs on the same seeded inputs.  Nothing here computes the method."""
import numpy as np
import torch

from oracle import sampler
from oracle.model import Config, InrModel
from paper_2304_10516_b200 import inr


def stream():
    return torch.cuda.current_stream().cuda_stream


def oracle_config(**kw):
    keys = ("levels", "features", "log2_table_size", "base_resolution", "per_level_scale", "mlp_width",
            "mlp_hidden_layers", "out_dim", "mlp_bias")
    return Config(**{k: v for k, v in kw.items() if k in keys})


def gpu_volume(vol_np):
    return torch.from_numpy(np.ascontiguousarray(vol_np, dtype=np.float32)).cuda()


def whole_view(vol_t):
    """View of a whole [z, y, x] scalar or [z, y, x, c] vector volume."""
    nz, ny, nx = vol_t.shape[:3]
    D = vol_t.shape[3] if vol_t.dim() == 4 else 1
    return inr.make_view(vol_t.data_ptr(), (0, 0, 0), (nx, ny, nz), (D, D * nx, D * nx * ny), D)


def make_gpu_model(blk, seed, **kw):
    cfg = inr.make_config(seed=seed, **kw)
    b = inr.make_block(tuple(int(v) for v in blk.origin), tuple(int(v) for v in blk.n),
                       tuple(int(v) for v in blk.global_dims))
    return inr.inr_create(cfg, b, 0)


def get_params(m):
    return inr.inr_get_params(m, np.empty(inr.inr_param_count(m), np.float32))


def get_grads(m):
    return inr.inr_get_grads(m, np.empty(inr.inr_param_count(m), np.float32))


def per_tensor_rel(cfg, a, b):
    """max over tensors of ||a - b||_inf / ||b||_inf (SURVEY §8(c) gradient metric)."""
    worst = 0.0
    for name, shape, off in cfg.tensor_layout():
        n = int(np.prod(shape))
        ref = np.abs(b[off:off + n]).max()
        if ref == 0:
            assert np.abs(a[off:off + n]).max() == 0, name
            continue
        worst = max(worst, float(np.abs(a[off:off + n] - b[off:off + n]).max() / ref))
    return worst


def normwise(a, b):
    return float(np.max(np.abs(np.asarray(a, np.float64) - b)) / max(np.max(np.abs(b)), 1e-300))
