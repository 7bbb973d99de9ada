"""Quickstart: fit a distributed neural representation of a volume on one GPU,
decode it, keep it in a temporal window, query it, render it.

    python examples/quickstart.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import synth  # noqa: E402
from paper_2304_10516_b200 import dnr, inr  # noqa: E402

torch.cuda.set_stream(torch.cuda.Stream())          # libinr captures CUDA graphs on the current stream
stream = torch.cuda.current_stream().cuda_stream

# a 256^3 scalar volume (the CloverLeaf3D-shaped blast field), resident on the GPU
n = 256
dims = (n, n, n)
vol = torch.empty((n, n, n), device="cuda")
for z0 in range(0, n, 16):
    vol[z0:z0 + 16] = synth.evaluate("g2", synth.lattice(dims, "cuda", (z0, z0 + 16)), dims).float()

# 2 x 2 x 2 blocks of 128^3, one hash-grid + MLP network each (fp16 tensor-core MLP).  The paper's
# T = 2^19 tables are larger than a 128^3 block; T = 2^16 compresses it (profiles/r1_rate_distortion.json)
cfg = inr.make_config(precision=inr.INR_PREC_FP16_MLP, levels=16, features=2, log2_table_size=16,
                      mlp_hidden_layers=3)
d = dnr.DNR(dims, (128, 128, 128), cfg)
d.value_range(vol, stream)                            # the global range every block normalizes with

opts = inr.inr_fit_opts_default()                     # lambda 0.5, Adam 1e-2 x 0.8 / 500 steps
opts.boundary_batch = 16384
rows = d.fit(vol, 1000, 65536, opts, stream)          # [block, steps, L1_uniform, L1_boundary, probe PSNR]
print("fit: last L1 per block", [round(r[2], 5) for r in rows])

# decode to the grid and measure the PSNR per block and overall
print("PSNR per block (dB)", {b: round(p, 2) for b, p in d.block_psnrs(vol, stream).items()})

# keep the trained networks as one timestep of a FIFO window (fp16 storage: 2x the compression)
cache = inr.cache_create(40, inr.CACHE_FP16)
inr.cache_insert(cache, 0, d.models, stream)
print("cached bytes", inr.cache_bytes(cache), "for", vol.numel() * 4, "bytes of raw data")

# random point queries against the cached timestep
ts, blocks = inr.cache_get(cache, 0)
pts = torch.rand((1 << 20, 3), device="cuda") * (n - 1)
vals = torch.empty(pts.shape[0], device="cuda")
inr.inr_decode_group(blocks, pts.data_ptr(), pts.shape[0], vals.data_ptr(), 1, stream)
torch.cuda.synchronize()
print("queried", vals.numel(), "points; mean value", float(vals.mean()))

# direct-query volume rendering (no decode to a grid)
cam = inr.make_camera((-180.0, 330.0, -260.0), (128.0, 110.0, 128.0), (0.0, 1.0, 0.0), 34.0, 512, 512)
tf = inr.make_tf([0.0, 0.3, 0.45, 0.7, 1.0], [[0, 0, 0, 0], [0, 0, 0, 0], [0.1, 0.4, 1.0, 0.02], [1.0, 0.8, 0.1, 0.15],
                                             [1.0, 0.1, 0.0, 0.6]], d.vmin, d.vmax)
img = d.render(cam, tf, 0.5, stream=stream)
print("rendered", tuple(img.shape), "mean opacity", float(img[:, 3].mean()))

inr.cache_destroy(cache)
d.close()
