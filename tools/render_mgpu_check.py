"""Sort-last rendering across ranks (NEXT-3): every rank fits its blocks of
a G2 volume, renders its brick, the fragments are gathered over NCCL to rank 0 and
depth-composited; rank 0 compares with a single-process render of the same models
(rank 0 re-creates and re-fits every block with the same seeds: fits are
deterministic per block in INR_REDUCE_DETERMINISTIC mode).
    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tools/render_mgpu_check.py"""
import json
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist
import synth
from paper_2304_10516_b200 import dnr, inr

world = int(os.environ.get("WORLD_SIZE", "1"))
rank = int(os.environ.get("RANK", "0"))
torch.cuda.set_device(rank)
if world > 1:
    dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
torch.cuda.set_stream(torch.cuda.Stream())
st = torch.cuda.current_stream().cuda_stream
N = 128
gd = (N, N, N * world)
cfg = inr.make_config(precision=1, reduction=1, levels=16, features=2, log2_table_size=16, mlp_hidden_layers=2)


def fitted(r, w):
    d = dnr.DNR(gd, (64, 64, 64), cfg, r, w, rank)
    vol = torch.empty((d.hi[2] - d.lo[2] + 1, d.hi[1] - d.lo[1] + 1, d.hi[0] - d.lo[0] + 1), device="cuda")
    pos = synth.lattice(gd, "cuda", (d.lo[2], d.hi[2] + 1))[:, d.lo[1]:d.hi[1] + 1, d.lo[0]:d.hi[0] + 1]
    vol[:] = synth.evaluate("g2", pos, gd).float()
    d.vmin, d.vmax = 0.0, 3.0                      # a fixed range: identical on every rank without the all-reduce
    o = inr.inr_fit_opts_default(); o.boundary_batch = 4096
    d.fit(vol, 200, 16384, o, st, report=False)
    return d


cam = inr.make_camera((-90.0, 160.0, -120.0), (64.0, 64.0, 64.0 * world), (0.0, 1.0, 0.0), 40.0, 256, 256)
tf = inr.make_tf([0.0, 0.35, 0.6, 1.0], [[0, 0, 0, 0], [0, 0, 0, 0], [0.1, 0.5, 1.0, 0.05], [1.0, 0.3, 0.0, 0.4]],
                 0.0, 3.0, 1.0)
d = fitted(rank, world)
img = d.render(cam, tf, 0.5, stop_alpha=2.0, stream=st)
if rank == 0:
    # reference: one renderer over every block (no process-group collectives here)
    ref_d = fitted(0, 1) if world > 1 else d
    r = inr.inr_renderer_create(ref_d.models, 16, 3e-3, st)
    frag = torch.empty((256 * 256, 5), device="cuda")
    inr.inr_render(r, cam, tf, [float(v) for v in ref_d.lo], [float(v) for v in ref_d.hi], 0.5, frag.data_ptr(), 2.0,
                   1, st)
    inr.inr_renderer_destroy(r)
    ref = torch.empty((256 * 256, 4), device="cuda")
    inr.inr_composite(frag.data_ptr(), 1, 256 * 256, (0.0, 0.0, 0.0), ref.data_ptr(), st)
    torch.cuda.synchronize()
    diff = float((img - ref).abs().max())
    import numpy as np
    pa = np.empty(inr.inr_param_count(d.models[0]), np.float32)
    pb = np.empty_like(pa)
    inr.inr_get_params(d.models[0], pa)
    inr.inr_get_params(ref_d.models[0], pb)
    # rank 0's own brick rendered from the reference models
    r0 = inr.inr_renderer_create(ref_d.models[:len(d.models)], 16, 3e-3, st)
    f0 = torch.empty((256 * 256, 5), device="cuda")
    inr.inr_render(r0, cam, tf, [float(v) for v in d.lo], [float(v) for v in d.hi], 0.5, f0.data_ptr(), 2.0, 1, st)
    inr.inr_renderer_destroy(r0)
    r1 = inr.inr_renderer_create(d.models, 16, 3e-3, st)
    f1 = torch.empty((256 * 256, 5), device="cuda")
    inr.inr_render(r1, cam, tf, [float(v) for v in d.lo], [float(v) for v in d.hi], 0.5, f1.data_ptr(), 2.0, 1, st)
    inr.inr_renderer_destroy(r1)
    torch.cuda.synchronize()
    fin = torch.isfinite(f0[:, 4])
    print("block0 params max diff", float(np.abs(pa - pb).max()), "rank0 brick frag diff",
          float((f0[fin] - f1[fin]).abs().max()), "lo/hi", d.lo, d.hi, ref_d.lo, ref_d.hi)
    print(json.dumps({"world": world, "image": [256, 256], "max_abs_diff_vs_single_rank": diff,
                      "mean_alpha": float(img[:, 3].mean())}))
if world > 1:
    dist.barrier()
    dist.destroy_process_group()
