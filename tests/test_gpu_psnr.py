"""End-to-end PSNR parity after cfg1's seeded 200 steps.

L1 + Adam at lr 1e-2 is chaotic: rounding the oracle's OWN parameters to fp32
after every step moves a single seed's 200-step PSNR by up to +-1.2 dB
(measured, R26), so one seed cannot resolve a 0.3 dB bar.  The bar
is applied to the mean PSNR over 48 seeds (GPU group fit of 48 models vs 48
oracle runs on the box's CPU cores), whose sampling noise is ~0.15 dB."""
import multiprocessing as mp
import os

import numpy as np
import pytest
import torch

import synth
from oracle import sampler
from paper_2304_10516_b200 import inr

from gpu_util import gpu_volume, stream, whole_view
from oracle_runs import CFG1, cfg1_psnr

pytestmark = [pytest.mark.gpu]
SEEDS = list(range(1000, 1048))


@pytest.fixture(scope="module")
def oracle_psnrs():
    procs = max(1, min(len(SEEDS), (os.cpu_count() or 2) - 1))
    with mp.get_context("spawn").Pool(procs) as pool:
        return np.array(pool.map(cfg1_psnr, SEEDS))


def gpu_psnrs(precision):
    n = 64
    vol = synth.g1_analytic(n).numpy()
    lo, hi = sampler.value_range([vol])
    vt = gpu_volume(vol)
    blk = inr.make_block((0, 0, 0), (n, n, n), (n, n, n))
    models = [inr.inr_create(inr.make_config(seed=s, precision=precision, **CFG1), blk, 0) for s in SEEDS]
    go = inr.inr_fit_opts_default()
    go.vmin, go.vmax = lo, hi
    inr.inr_fit_group(models, [whole_view(vt)] * len(models), 200, 4096, go, stream())
    ref = (torch.from_numpy(vol).cuda().double() - lo) / (hi - lo)
    out = torch.empty((n, n, n), device="cuda")
    ps = []
    for m in models:
        inr.inr_decode_grid(m, (n, n, n), out.data_ptr(), None, None, None, stream())
        mse = float((((out.double() - lo) / (hi - lo) - ref) ** 2).mean())
        ps.append(-10 * np.log10(mse))
        inr.inr_destroy(m)
    return np.array(ps)


@pytest.mark.parametrize("precision", [0, 1])
def test_mean_psnr_within_0p3db(oracle_psnrs, precision):
    g = gpu_psnrs(precision)
    print("gpu", np.round(g, 2).tolist()); print("oracle", np.round(oracle_psnrs, 2).tolist())
    print(f"precision {precision}: gpu mean {g.mean():.3f} (sd {g.std():.2f}), "
          f"oracle mean {oracle_psnrs.mean():.3f} (sd {oracle_psnrs.std():.2f})")
    assert abs(g.mean() - oracle_psnrs.mean()) <= 0.3
