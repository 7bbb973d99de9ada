"""End-to-end PSNR parity after cfg1's seeded 200 steps.

L1 + Adam at lr 1e-2 is chaotic: rounding the oracle's OWN parameters to fp32
after every step moves a single seed's 200-step PSNR by up to +-1.2 dB
(measured, R26), and the seed-to-seed spread is 1.5 dB, so one seed
cannot resolve a 0.3 dB bar.  The bar is applied to the mean PSNR over 384
seeds: the GPU fits them here (8 group fits of 48 models), the oracle values
come from tests/golden/oracle_cfg1_psnr.txt (written by
tests/make_oracle_psnr_fixture.py, which calls only oracle/).  The standard
error of the difference of the two means is ~0.11 dB."""
import numpy as np
import pytest
import torch

import synth
from oracle import sampler
from paper_2304_10516_b200 import inr

from conftest import read_golden
from gpu_util import gpu_volume, stream, whole_view
from oracle_runs import CFG1

pytestmark = [pytest.mark.gpu]


def oracle_psnrs():
    rows = read_golden("oracle_cfg1_psnr.txt")
    return [int(r[0]) for r in rows], np.array([float(r[1]) for r in rows])


def gpu_psnrs(precision, seeds):
    n = 64
    vol = synth.g1_analytic(n).numpy()
    lo, hi = sampler.value_range([vol])
    vt = gpu_volume(vol)
    blk = inr.make_block((0, 0, 0), (n, n, n), (n, n, n))
    go = inr.inr_fit_opts_default()
    go.vmin, go.vmax = lo, hi
    ref = (torch.from_numpy(vol).cuda().double() - lo) / (hi - lo)
    out = torch.empty((n, n, n), device="cuda")
    ps = []
    for c in range(0, len(seeds), 48):
        models = [inr.inr_create(inr.make_config(seed=s, precision=precision, **CFG1), blk, 0)
                  for s in seeds[c:c + 48]]
        inr.inr_fit_group(models, [whole_view(vt)] * len(models), 200, 4096, go, stream())
        for m in models:
            inr.inr_decode_grid(m, (n, n, n), out.data_ptr(), None, None, None, stream())
            mse = float((((out.double() - lo) / (hi - lo) - ref) ** 2).mean())
            ps.append(-10 * np.log10(mse))
            inr.inr_destroy(m)
    return np.array(ps)


@pytest.mark.parametrize("precision", [0, 1])
def test_mean_psnr_within_0p3db(precision):
    seeds, o = oracle_psnrs()
    g = gpu_psnrs(precision, seeds)
    print(f"precision {precision}: gpu mean {g.mean():.3f} (sd {g.std():.2f}), "
          f"oracle mean {o.mean():.3f} (sd {o.std():.2f}), n {len(seeds)}")
    assert abs(g.mean() - o.mean()) <= 0.3
