"""Oracle training runs used by the statistical PSNR parity test (top-level
functions so multiprocessing can pickle them).  Test infrastructure only."""
import os

os.environ.setdefault("OMP_NUM_THREADS", "1")
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")

import numpy as np  # noqa: E402

import synth  # noqa: E402
from oracle import decode, fit, sampler  # noqa: E402
from oracle.model import Config, InrModel  # noqa: E402

CFG1 = dict(levels=8, features=2, log2_table_size=14, mlp_hidden_layers=2)


def cfg1_psnr(seed, steps=200, batch=4096, n=64):
    """cfg1: G1 64^3, one block, 200 steps of 4096 samples,
    then PSNR of the 64^3 decode against the data (normalized units)."""
    vol = synth.g1_analytic(n).numpy()
    lo, hi = sampler.value_range([vol])
    blk = sampler.decompose((n, n, n), (n, n, n))[0]
    m = InrModel(Config(**CFG1), blk, seed)
    fit.fit(m, vol, steps, batch, fit.FitOpts(vmin=lo, vmax=hi))
    ref = (vol.astype(np.float64) - lo) / (hi - lo)
    return sampler.psnr((decode.decode_grid(m, (n, n, n)) - lo) / (hi - lo), ref)
