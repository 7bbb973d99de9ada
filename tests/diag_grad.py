"""Diagnostic (not collected by pytest): per-tensor gradient / Adam errors."""
import sys
import numpy as np
import torch
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import synth
from oracle import fit as o_fit, sampler
from oracle.model import InrModel
from paper_2304_10516_b200 import inr
from gpu_util import gpu_volume, get_grads, get_params, make_gpu_model, oracle_config, stream, whole_view
from test_gpu_parity import CFG1, _perturbed_params, _clean_seed

vol = synth.g1_analytic(32).numpy()
blk = sampler.decompose((32, 32, 32), (16, 16, 16))[3]
lo, hi = sampler.value_range([vol])
opts = o_fit.FitOpts(vmin=lo, vmax=hi, boundary_batch=128)
cfg = oracle_config(**CFG1)
p0 = _perturbed_params(cfg, blk, 1, np.random.default_rng(0))
for det, prec in ((1, 0), (0, 0), (1, 1)):
    seed, om = _clean_seed(cfg, blk, vol, opts, 512, range(100, 200), p0)
    m = make_gpu_model(blk, seed, reduction=det, precision=prec, **CFG1)
    inr.inr_set_params(m, p0)
    vt = gpu_volume(vol)
    go = inr.inr_fit_opts_default()
    go.vmin, go.vmax, go.boundary_batch = lo, hi, 128
    rep = inr.inr_fit(m, whole_view(vt), 1, 512, go, stream())
    l1u, l1b, _ = o_fit.train_step(om, vol, opts, 512)
    g = get_grads(m)
    p = get_params(m)
    print(f"== det={det} prec={prec} seed={seed} loss gpu {rep.loss_uniform:.6g} {rep.loss_boundary:.6g} oracle {l1u:.6g} {l1b:.6g}")
    for name, shape, off in cfg.tensor_layout():
        n = int(np.prod(shape))
        a, b = g[off:off + n], om.g[off:off + n]
        ref = np.abs(b).max()
        dp = np.abs(p[off:off + n] - om.p[off:off + n])
        k = int(np.argmax(dp))
        print(f"{name:8s} grad rel {np.abs(a-b).max()/max(ref,1e-30):.3e}  |ref|inf {ref:.3e}  "
              f"max dp {dp.max():.3e} at {k} g_gpu {a[k]:.4e} g_or {b[k]:.4e}")
    inr.inr_destroy(m)
