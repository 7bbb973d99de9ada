"""NEXT-1: the boundary-continuity study of the paper on synthetic data.

PAPER.md L164-166 (Fig. 3): "the impact of the weighting factor lambda on
boundary connectivity and overall reconstruction quality ... average image PSNR
of two boundary slices relative to the ground truth slice ... average volume
PSNR of two partitions"; L184-186 (Fig. 4): both networks trained 10,000 steps,
lambda = 0.5 vs 0; L209: "the existence of the boundary connectivity loss can
significantly increase the data accuracy across the partition boundary ... as
the weight increases, we see a diminishing effect and a negative impact on the
overall reconstruction quality ... the sweet spot for lambda is 0.5".

A 2x1x1 split (S3D data unavailable: synthetic G2 field): both blocks are fitted
with Eq. 2 at each lambda; each network is evaluated on the shared face plane
(block 0 at x = 1, block 1 at x = 0, R5) and over its core.

    python -m studies.lambda_sweep [--steps 2000] [--out profiles/r1_lambda_sweep.json]
"""
import argparse
import json
import math
import os

import numpy as np
import torch

import synth
from paper_2304_10516_b200 import inr

LAMBDAS = (0.0, 0.25, 0.5, 0.75, 1.0)


def psnr(mse):
    return 200.0 if mse <= 0 else min(200.0, -10.0 * math.log10(mse))


def run(steps=2000, n=64, lambdas=LAMBDAS, precision=inr.INR_PREC_FP16_MLP, seed=11, batch=4096, boundary=1024):
    dev = torch.device("cuda")
    gd = (2 * n, n, n)
    vol = synth.evaluate("g2", synth.lattice(gd, dev), gd).to(torch.float32).contiguous()
    lo, hi = float(vol.min()), float(vol.max())
    view = inr.make_view(vol.data_ptr(), (0, 0, 0), gd, (1, gd[0], gd[0] * gd[1]))
    st = torch.cuda.current_stream().cuda_stream
    # the shared face x = n: node lattice (y, z) in 0..n-1, block-normalized coordinates
    ys, zs = torch.meshgrid(torch.arange(n, device=dev), torch.arange(n, device=dev), indexing="xy")
    face = torch.stack([torch.zeros(n * n, device=dev), ys.reshape(-1).float() / n, zs.reshape(-1).float() / n], 1)
    face0 = face.clone()
    face0[:, 0] = 1.0
    truth = (vol[:, :, n].reshape(-1).double() - lo) / (hi - lo)          # [z][y] at x = n
    out = []
    for lam in lambdas:
        cfg = inr.make_config(levels=8, features=2, log2_table_size=14, mlp_hidden_layers=2, precision=precision,
                              seed=seed)
        ms = [inr.inr_create(cfg, inr.make_block((b * n, 0, 0), (n, n, n), gd), 0) for b in range(2)]
        go = inr.inr_fit_opts_default()
        go.vmin, go.vmax, go.lambda_, go.boundary_batch = lo, hi, lam, boundary
        inr.inr_fit_group(ms, [view, view], steps, batch, go, st)
        y0 = torch.empty(n * n, device=dev)
        y1 = torch.empty(n * n, device=dev)
        inr.inr_debug_forward(ms[0], face0.contiguous().data_ptr(), n * n, y0.data_ptr(), st)
        inr.inr_debug_forward(ms[1], face.contiguous().data_ptr(), n * n, y1.data_ptr(), st)
        grid = torch.empty((n, n, 2 * n), device=dev)
        sse = torch.zeros(1, dtype=torch.float64, device=dev)
        for b in range(2):
            inr.inr_decode_grid(ms[b], (n, n, n), grid[:, :, b * n:].data_ptr(), (1, 2 * n, 2 * n * n),
                                vol[:, :, b * n:].data_ptr(), sse.data_ptr(), st)
        torch.cuda.synchronize()
        # y0/y1 are in [z][y] order matching `truth` (face rows: x fastest -> y, then z)
        r = {"lambda": lam,
             "volume_psnr_db": psnr(float(sse.item()) / vol.numel()),
             "slice_psnr_block0_db": psnr(float(((y0.double() - truth) ** 2).mean())),
             "slice_psnr_block1_db": psnr(float(((y1.double() - truth) ** 2).mean())),
             "slice_mismatch_rms": float(((y0.double() - y1.double()) ** 2).mean().sqrt())}
        r["slice_psnr_mean_db"] = 0.5 * (r["slice_psnr_block0_db"] + r["slice_psnr_block1_db"])
        diff = (y0 - y1).abs().cpu().numpy()
        r["mismatch_hist"] = np.histogram(diff, bins=8, range=(0, max(float(diff.max()), 1e-6)))[0].tolist()
        out.append(r)
        for m in ms:
            inr.inr_destroy(m)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--out", default=os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                                  "profiles", "r1_lambda_sweep.json"))
    a = ap.parse_args()
    res = run(a.steps)
    for r in res:
        print(json.dumps(r))
    with open(a.out, "w") as f:
        json.dump({"study": "NEXT-1 lambda sweep (P:L164-166, L184-186, L209), G2 2x1x1 split of 128x64x64",
                   "steps": a.steps, "results": res}, f, indent=1)


if __name__ == "__main__":
    main()
