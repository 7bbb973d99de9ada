"""cfg2 PSNR-target fit (probes every 50 steps, no CUDA graphs): ms per step with the
split step on / off / on.  python tools/target_probe.py"""
import sys, os, json
sys.path.insert(0, os.getcwd())
import torch, synth
from paper_2304_10516_b200 import dnr, inr
torch.cuda.set_stream(torch.cuda.Stream())
st = torch.cuda.current_stream().cuda_stream
cfg = inr.make_config(precision=1, seed=0x230410516, levels=16, features=2, log2_table_size=19, mlp_hidden_layers=3)
d = dnr.DNR((256,) * 3, (128,) * 3, cfg)
vol = synth.g2_energy(256, device="cuda").float().contiguous()
d.value_range(vol, st)
res = {}
for split in (1, 0, 1):
    o = inr.inr_fit_opts_default()
    o.boundary_batch = 16384
    o.split_step = split
    o.set_range(d.vmin, d.vmax)
    o.target_psnr, o.check_interval = 99.0, 50
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    inr.inr_fit_group(d.models, d.views(vol), 50, 65536, o, st, True)
    torch.cuda.synchronize()
    e0.record()
    inr.inr_fit_group(d.models, d.views(vol), 500, 65536, o, st, True)
    e1.record()
    torch.cuda.synchronize()
    res[f"split{split}"] = e0.elapsed_time(e1) / 500
print(json.dumps(res))
