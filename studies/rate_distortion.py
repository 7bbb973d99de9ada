"""PSNR @ compression ratio across hash-table sizes (BASELINE.json's "PSNR @ ratio"
on the cfg2 workload): G2 256^3, 8 blocks of 128^3, L = 16, F = 2, 3 x 64 MLP,
fp16 tensor-core fit of 2000 steps per table size T = 2^12 .. 2^19.  Reports the
global and worst-block PSNR (1x decode on the nodes), the ratio of raw fp32 core
bytes to stored parameters (fp32 and fp16 storage) and the fit rate.

    python studies/rate_distortion.py [--steps 2000] [--out profiles/r1_rate_distortion.json]"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
from paper_2304_10516_b200 import dnr, inr  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r1_rate_distortion.json"))
    a = ap.parse_args()
    torch.cuda.set_stream(torch.cuda.Stream())
    st = torch.cuda.current_stream().cuda_stream
    n = 256
    gd = (n, n, n)
    vol = torch.empty((n, n, n), device="cuda")
    for z0 in range(0, n, 16):
        vol[z0:z0 + 16] = synth.evaluate("g2", synth.lattice(gd, "cuda", (z0, z0 + 16)), gd).float()
    rows = []
    for log2t in (12, 14, 16, 17, 18, 19):
        cfg = inr.make_config(precision=inr.INR_PREC_FP16_MLP, levels=16, features=2, log2_table_size=log2t,
                              mlp_hidden_layers=3, seed=0x230410516)
        d = dnr.DNR(gd, (128, 128, 128), cfg)
        d.value_range(vol, st)
        o = inr.inr_fit_opts_default()
        o.boundary_batch = 16384
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        d.fit(vol, a.steps, 65536, o, st, report=True)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        out = torch.empty_like(vol)
        sse = torch.zeros(1, dtype=torch.float64, device="cuda")
        d.decode_grid_local(out, 1, vol, sse, st)
        torch.cuda.synchronize()
        bp = d.block_psnrs(vol, st)
        row = {"log2_table_size": log2t, "params_per_block": inr.inr_param_count(d.models[0]),
               "psnr_db": d.psnr(float(sse.item()), n ** 3), "psnr_block_min_db": min(bp.values()),
               "compression_ratio": 4.0 * n ** 3 / d.param_bytes(),
               "compression_ratio_fp16_stored": 8.0 * n ** 3 / d.param_bytes(),
               "fit_coords_per_s": 8 * (65536 + 16384) * a.steps / (ms / 1e3), "steps": a.steps}
        print(json.dumps(row), flush=True)
        rows.append(row)
        d.close()
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    with open(a.out, "w") as f:
        json.dump({"gpu": torch.cuda.get_device_name(0), "workload": "cfg2 G2 256^3, 8 x 128^3 blocks, L16 F2 3x64",
                   "rows": rows}, f, indent=1)


if __name__ == "__main__":
    main()
