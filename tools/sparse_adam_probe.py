"""NEXT-4 touched-only Adam (R37, opts.sparse_adam) vs the dense PyTorch-form
Adam (R12): fit step time and PSNR after the same steps, on one GPU's share of
cfg5 (64 of the 512 blocks of 1024^3, T = 2^22: Adam-bound) and on cfg2
(8 blocks of 256^3, T = 2^19).  Writes JSON to stdout.

  python tools/sparse_adam_probe.py [cfg5_steps] [cfg2_steps]
"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import configs
from paper_2304_10516_b200 import dnr, inr

S5 = int(sys.argv[1]) if len(sys.argv) > 1 else 200
S2 = int(sys.argv[2]) if len(sys.argv) > 2 else 2000
torch.cuda.set_stream(torch.cuda.Stream())
st = torch.cuda.current_stream().cuda_stream
dev = torch.device("cuda")


def run(gdims, kind, net, world, steps, sparse):
    d = dnr.DNR(gdims, (128, 128, 128), inr.make_config(precision=1, seed=0x230410516, **net), rank=0, world=world)
    vol = configs.gen_local(kind, gdims, d.lo, d.hi, dev)
    d.value_range(vol, st)
    opts = inr.inr_fit_opts_default()
    opts.boundary_batch = 16384
    opts.sparse_adam = sparse
    d.fit(vol, 10, 65536, opts, st, report=True)
    torch.cuda.synchronize()
    e0, e1 = configs.ev(), configs.ev()
    e0.record()
    d.fit(vol, steps - 10, 65536, opts, st, report=True)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / (steps - 10)
    psnr, _, _ = configs.psnr_1x(d, vol, st)
    r = {"sparse_adam": sparse, "blocks": len(d.models), "steps": steps, "ms_per_step": ms,
         "fit_coords_per_s": len(d.models) * 81920 / (ms / 1e3), "psnr_db": psnr,
         "params_per_gpu": sum(inr.inr_param_count(m) for m in d.models)}
    d.close()
    del vol
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    return r


out = {"what": "R37 touched-only Adam vs dense Adam (fp16 MLP fit, 65536+16384 coords/block/step)"}
net5 = dict(configs.NET2, log2_table_size=22)
out["cfg5_share"] = [run((1024, 1024, 1024), "g3", net5, 8, S5, s) for s in (0, 1)]
out["cfg2"] = [run((256, 256, 256), "g2", configs.NET2, 1, S2, s) for s in (0, 1)]
print(json.dumps(out))
