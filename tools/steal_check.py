"""NEXT-4 cross-GPU block stealing for PSNR-target fits (DNR.fit_to_target).
Rank r owns 8 blocks of 128^3 (cfg2 network) of a 256 x 256 x (256 N) volume; rank 0's half is
a high-frequency periodic field, equally hard in every block (slow to reach the
target), the other ranks' halves are smooth G1 blobs (fast).  Runs the target fit with and without stealing on fresh
models and reports the max-over-ranks time and whether every block's final
parameters agree bitwise (deterministic mode).
    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tools/steal_check.py"""
import json
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import torch.distributed as dist
import synth
from paper_2304_10516_b200 import dnr, inr

world = int(os.environ.get("WORLD_SIZE", "1"))
rank = int(os.environ.get("RANK", "0"))
torch.cuda.set_device(rank)
dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
torch.cuda.set_stream(torch.cuda.Stream())
st = torch.cuda.current_stream().cuda_stream
gd = (256, 256, 256 * world)
TARGET = float(os.environ.get("TARGET", "45"))
cfg = inr.make_config(precision=1, reduction=1, levels=16, features=2, log2_table_size=19, mlp_hidden_layers=3)
# NCCL point-to-point connections are set up on first use (~1 s): do it before timing
for a in range(world):
    for b in range(world):
        if a != b and rank in (a, b):
            t = torch.zeros(1 << 20, device="cuda")
            dist.send(t, b) if rank == a else dist.recv(t, a)
torch.cuda.synchronize()


def run(steal):
    d = dnr.DNR(gd, (128, 128, 128), cfg, rank, world, rank)
    pos = synth.lattice(gd, "cuda", (d.lo[2], d.hi[2] + 1))[:, d.lo[1]:d.hi[1] + 1, d.lo[0]:d.hi[0] + 1]
    vol = torch.empty(pos.shape[:3], device="cuda")
    for z0 in range(0, pos.shape[0], 16):
        p = pos[z0:z0 + 16]
        if rank == 0:   # the same high-frequency pattern in every block: uniformly hard
            w = 2 * np.pi / 128.0
            f = (torch.sin(7 * w * p[..., 0]) * torch.sin(5 * w * p[..., 1]) * torch.sin(6 * w * p[..., 2])
                 + 0.5 * torch.sin(13 * w * (p[..., 0] + p[..., 2])))
        else:           # smooth blobs: easy
            f = synth.evaluate("g1", p, gd)
        vol[z0:z0 + 16] = f.float()
    del pos
    d.value_range(vol, st)
    o = inr.inr_fit_opts_default()
    o.boundary_batch = 16384
    dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = d.fit_to_target(vol, TARGET, 4000, 65536, o, check_interval=50, round_steps=200, steal=steal, stream=st)
    torch.cuda.synchronize()
    t = dnr.allreduce_max(time.perf_counter() - t0)
    params = [np.empty(inr.inr_param_count(m), np.float32) for m in d.models]
    for m, p in zip(d.models, params):
        inr.inr_get_params(m, p)
    return t, res, params, d


t0, r0, p0, d0 = run(False)
t1, r1, p1, d1 = run(True)
same = all(np.array_equal(a, b) for a, b in zip(p0, p1)) and r0 == r1
same_all = dnr.allreduce_sum([0.0 if same else 1.0])[0] == 0.0
allres = [None] * world
dist.all_gather_object(allres, {str(k): v for k, v in r0.items()})
if rank == 0:
    print(json.dumps({"world": world, "time_s_no_steal": t0, "time_s_steal": t1, "speedup": t0 / t1,
                      "target_psnr": TARGET, "blocks_steps_reached_by_rank": allres,
                      "identical_params_and_steps_all_ranks": bool(same_all)}))
dist.barrier()
dist.destroy_process_group()
