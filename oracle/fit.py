"""The training loop of one block's INR (P:L172 uniform sampling; P:L198-202
Eq. 2 boundary-weighted loss; P:L220 Adam + step schedule; "training
... continues until the user-defined accuracy criterion (such as a PSNR
target) is reached"), in the order of SURVEY.md §8(c) step 3:

  lr_s -> uniform samples -> boundary samples -> targets -> encode -> MLP
  -> Eq. 2 loss and dL/dy -> backward (MLP, then table scatter) -> Adam.

Everything float64 except the pinned float32 index math.
"""
import dataclasses

import numpy as np

from . import adam, encoding, loss, mlp, sampler


@dataclasses.dataclass
class FitOpts:
    lam: float = 0.5              # P:L209 "sweet spot for lambda is 0.5"
    boundary_batch: int = 0
    lr0: float = 1e-2
    lr_decay: float = 0.8
    lr_step: int = 500
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8             # S:L239 (paper silent)
    vmin: float = 0.0
    vmax: float = 1.0
    target_psnr: float = 0.0      # <= 0: fixed step count
    check_interval: int = 0
    sparse_adam: int = 0          # R37 (NEXT-4 variant): touched-only table updates


@dataclasses.dataclass
class FitReport:
    steps_taken: int = 0
    reached_target: int = 0
    constant_field: int = 0
    loss_uniform: float = 0.0
    loss_boundary: float = 0.0
    probe_psnr: float = 0.0


def forward(model, x):
    """Phi(x) in normalized value units for block-normalized x (Eq. 1)."""
    cfg = model.cfg
    feat, idx, wt = encoding.encode_forward(model.tables(), x, cfg.resolutions(), cfg.table_size)
    Ws, bs = model.mlp()
    y, zs, hs = mlp.forward(Ws, bs, feat)
    return y, (feat, idx, wt, zs, hs)


def gradients(model, x, dy, cache):
    """Flat gradient vector (declared order) for upstream dL/dy."""
    cfg = model.cfg
    feat, idx, wt, zs, hs = cache
    Ws, bs = model.mlp()
    dW, db, dfeat = mlp.backward(Ws, bs, zs, hs, dy)
    shapes = [(s, cfg.features) for s in cfg.level_sizes()]
    gt = encoding.encode_backward(dfeat, idx, wt, shapes)
    g = np.zeros_like(model.p)
    for l in range(cfg.levels):
        model.view(g, f"table{l}")[...] = gt[l]
    for k in range(len(Ws)):
        model.view(g, f"W{k}")[...] = dW[k]
        if bs[k] is not None:
            model.view(g, f"b{k}")[...] = db[k]
    return g


def step_batch(model, volume, opts, batch):
    """The samples, targets and constant flag of the model's current step."""
    s = model.step
    blk = model.block
    x_u = sampler.uniform_samples(model.seed, s, blk.block_id, batch)
    x_b = sampler.boundary_samples(model.seed, s, blk, opts.boundary_batch)
    t_u, const = sampler.targets(volume, blk, x_u, opts.vmin, opts.vmax)
    t_b, _ = sampler.targets(volume, blk, x_b, opts.vmin, opts.vmax)
    return x_u, x_b, t_u, t_b, const


def train_step(model, volume, opts, batch):
    """One step.  Leaves this step's gradient in model.g.
    Returns (l1_uniform, l1_boundary, constant_flag)."""
    s = model.step
    lr = adam.lr_at(s, opts.lr0, opts.lr_decay, opts.lr_step)
    x_u, x_b, t_u, t_b, const = step_batch(model, volume, opts, batch)
    x = np.concatenate([x_u, x_b], axis=0)
    y, cache = forward(model, x)
    nu = x_u.shape[0]
    D = y.shape[1]
    yu, yb = (y[:nu, 0], y[nu:, 0]) if D == 1 else (y[:nu], y[nu:])
    _, l1u, l1b, dy_u, dy_b = loss.loss_and_grad(yu, t_u, yb, t_b, opts.lam)
    dy = np.concatenate([dy_u, dy_b]).reshape(-1, D)
    model.g = gradients(model, x, dy, cache)
    if opts.sparse_adam:
        tables = [(off, int(np.prod(shape))) for name, shape, off in model.cfg.tensor_layout() if name.startswith("table")]
        adam.adam_update_sparse(model.p, model.g, model.m, model.v, s + 1, lr, tables, opts.beta1, opts.beta2, opts.eps)
    else:
        adam.adam_update(model.p, model.g, model.m, model.v, s + 1, lr, opts.beta1, opts.beta2, opts.eps)
    model.step += 1
    return l1u, l1b, const


def probe_psnr(model, volume, opts):
    """PSNR on the 32^3 cell-centred probe lattice against sampler targets."""
    xp = sampler.probe_lattice(32)
    t, _ = sampler.targets(volume, model.block, xp, opts.vmin, opts.vmax)
    y, _ = forward(model, xp)
    return sampler.psnr(y[:, 0] if y.shape[1] == 1 else y, t)


def fit(model, volume, steps, batch, opts):
    """inr_fit semantics: `steps` >= 1 steps, stopping early when the
    probe PSNR reaches opts.target_psnr at a check interval."""
    if steps < 1 or batch < 1:
        raise ValueError("steps and batch must be >= 1")
    model.vmin, model.vmax = opts.vmin, opts.vmax
    rep = FitReport()
    for i in range(steps):
        l1u, l1b, const = train_step(model, volume, opts, batch)
        rep.steps_taken = i + 1
        rep.loss_uniform, rep.loss_boundary = l1u, l1b
        rep.constant_field = int(const)
        if opts.target_psnr > 0 and opts.check_interval > 0 and (i + 1) % opts.check_interval == 0:
            rep.probe_psnr = probe_psnr(model, volume, opts)
            if rep.probe_psnr >= opts.target_psnr:
                rep.reached_target = 1
                break
    return rep
