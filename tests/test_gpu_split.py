"""The split fit step (inr_fit_opts.split_step): a group's two halves
run the level-major pipeline in turn and each half's Adam runs beside the other
half's tensor-core MLP, half B's last Adam deferred to the end of the call.
Per model the operations and their order are the unsplit step's (blocks are
independent), so

  * in the deterministic reduction mode the parameters and Adam moments of a
    multi-step split fit are bitwise those of the unsplit fit (any misrouted
    workspace, skipped or doubled Adam shows up here), and
  * the TMA-fed Adam kernel that runs beside the MLP (plain fp32 gradients)
    is the PyTorch-form Adam of R12: each step's GPU gradient fed to the
    oracle's adam_update reproduces p, m, v to fp32 rounding (as
    test_gpu_parity.test_adam_elementwise_across_lr_decays)."""
import numpy as np
import pytest

import synth
from oracle import adam as o_adam, sampler
from paper_2304_10516_b200 import inr

from gpu_util import gpu_volume, get_grads, get_params, make_gpu_model, stream, whole_view

pytestmark = pytest.mark.gpu

CFG1 = dict(levels=8, features=2, log2_table_size=14, mlp_hidden_layers=2)


def _setup(n_models, reduction, seed0=11, vector=False, sparse=0):
    side = 32 if n_models <= 8 else 64
    if vector:   # D = 3: the Taylor-Green velocity field, per-channel ranges (R28)
        vol = synth.taylor_green_volume(side, 0.0, amp=2.0).numpy()
    else:
        vol = synth.g1_analytic(side).numpy()
    blocks = sampler.decompose((side,) * 3, (16, 16, 16))[:n_models]
    vt = gpu_volume(vol)
    kw = dict(CFG1, out_dim=3) if vector else CFG1
    models = [make_gpu_model(b, seed0 + i, reduction=reduction, precision=inr.INR_PREC_FP16_MLP, **kw)
              for i, b in enumerate(blocks)]
    go = inr.inr_fit_opts_default()
    if vector:
        for c in range(3):
            go.vmin_c[c], go.vmax_c[c] = float(vol[..., c].min()), float(vol[..., c].max())
    else:
        go.vmin, go.vmax = sampler.value_range([vol])
    go.boundary_batch, go.lr_step, go.sparse_adam = 256, 3, sparse
    return vt, models, go


def _state(m):
    p = get_params(m)
    mm, vv = inr.inr_get_adam_state(m, np.empty_like(p), np.empty_like(p))
    return p, mm, vv


@pytest.mark.parametrize("n_models,vector,sparse", [(2, False, 0), (5, False, 0), (4, True, 0), (4, False, 1),
                                                    (64, False, 0)],
                         ids=["2", "5", "4-vector", "4-sparse-adam", "64"])
def test_split_step_bitwise_equals_unsplit_deterministic(n_models, vector, sparse):
    """5 models: halves of 2 and 3.  Two calls (7 + 4 steps: the first-step and
    steady-step graphs, the final flush of half B's Adam, LR decays at s = 3, 6, 9);
    also D = 3 vector-field models (R28) and the R37 touched-only Adam beside the MLP."""
    out = []
    for split in (1, 0):
        vt, models, go = _setup(n_models, reduction=1, vector=vector, sparse=sparse)
        go.split_step = split
        views = [whole_view(vt)] * n_models
        for steps in (7, 4):
            inr.inr_fit_group(models, views, steps, 1024, go, stream())
        out.append([_state(m) for m in models] + [[inr.inr_steps(m) for m in models]])
        for m in models:
            inr.inr_destroy(m)
    a, b = out
    assert a[-1] == b[-1] == [11] * n_models   # (64 models: the largest group of one launch, 2 CTAs per model)
    for i in range(n_models):
        for x, y in zip(a[i], b[i]):
            assert np.array_equal(x, y), i


def test_split_step_tma_adam_elementwise():
    """Two models, plain fp32 gradients: in a one-step split call model 0's Adam
    is the TMA-fed kernel beside model 1's MLP, model 1's the final flush (the
    standalone kernel); both checked element by element against the oracle's
    Adam over 6 steps crossing two LR decays."""
    vt, models, go = _setup(2, reduction=0)
    views = [whole_view(vt)] * 2
    ref = []
    for m in models:
        p = get_params(m).astype(np.float64)
        ref.append([p, np.zeros_like(p), np.zeros_like(p), np.zeros_like(p)])
    worst = 0.0
    for t in range(1, 7):
        inr.inr_fit_group(models, views, 1, 1024, go, stream())
        for m, (p, mo, vo, gmax) in zip(models, ref):
            g = get_grads(m).astype(np.float64)
            assert np.any(g != 0)
            np.maximum(gmax, np.abs(g), out=gmax)
            o_adam.adam_update(p, g, mo, vo, t, o_adam.lr_at(t - 1, 1e-2, 0.8, 3))
            pg, mg, vg = _state(m)
            tol_p = t * (1e-6 * 1e-2 + 2.0 ** -21 * np.abs(p))
            tol_m = t * 2.0 ** -21 * gmax
            tol_v = t * 2.0 ** -21 * vo + 1e-37
            r = [float(np.max(np.abs(pg - p) / tol_p)), float(np.max(np.abs(mg - mo) / tol_m.clip(1e-30))),
                 float(np.max(np.abs(vg - vo) / tol_v))]
            worst = max(worst, max(r))
            assert max(r) <= 1, (t, r)
    print("split step, TMA Adam: worst error / tolerance", worst)
    for m in models:
        inr.inr_destroy(m)


def test_split_step_multistep_matches_unsplit_statistically():
    """Plain fp32 gradients (atomic reduction order varies run to run): a 40-step
    split fit of 4 models ends at the unsplit fit's loss to within the run-to-run
    spread (the TMA Adam of the steady graph included; elementwise agreement is
    the deterministic test's job)."""
    res = []
    for split in (1, 0):
        vt, models, go = _setup(4, reduction=0)
        go.split_step = split
        reps = inr.inr_fit_group(models, [whole_view(vt)] * 4, 40, 1024, go, stream())
        res.append(([r.loss_uniform for r in reps], [get_params(m) for m in models]))
        for m in models:
            inr.inr_destroy(m)
    (la, pa), (lb, pb) = res
    for x, y in zip(la, lb):
        assert abs(x - y) <= 0.05 * max(x, y), (la, lb)
    assert all(np.isfinite(x).all() for x in pa)


def test_live_split_with_psnr_target_stopping_bitwise():
    """Without CUDA graphs (PSNR-target stopping probes the models every
    check_interval steps) the split step is enqueued live and half B's deferred
    Adam is flushed before each probe; models leave the group as they converge
    (the halves are re-formed).  Deterministic mode: every model's parameters and
    step count equal the unsplit fit's bitwise."""
    out = []
    for split in (1, 0):
        vt, models, go = _setup(6, reduction=1, seed0=21)
        go.split_step = split
        go.target_psnr, go.check_interval = 38.0, 20
        reps = inr.inr_fit_group(models, [whole_view(vt)] * 6, 200, 1024, go, stream())
        out.append(([(r.steps_taken, r.reached_target) for r in reps], [_state(m) for m in models]))
        for m in models:
            inr.inr_destroy(m)
    (ra, sa), (rb, sb) = out
    print("live split, steps / reached:", ra)
    assert ra == rb and len({s for s, _ in ra}) > 1   # models stop at different checks
    for x, y in zip(sa, sb):
        for u, v in zip(x, y):
            assert np.array_equal(u, v)
