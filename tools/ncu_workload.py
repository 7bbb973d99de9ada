"""One of each hot kernel on the bench workload (cfg2: 8 blocks of 128^3, fp16), for
`ncu --set full`: fit steps, a 128^3 grid decode, 2^22 random queries, a 512^2
render and a small pathline trace.  Not a benchmark (see bench.py / configs.py)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
from paper_2304_10516_b200 import dnr, inr
torch.cuda.set_stream(torch.cuda.Stream())
st = torch.cuda.current_stream().cuda_stream
gd = (256, 256, 256)
d = dnr.DNR(gd, (128,) * 3, inr.make_config(precision=1, levels=16, features=2, log2_table_size=19,
                                            mlp_hidden_layers=3))
vol = torch.empty((256, 256, 256), device="cuda")
for z0 in range(0, 256, 16):
    vol[z0:z0 + 16] = synth.evaluate("g2", synth.lattice(gd, "cuda", (z0, z0 + 16)), gd).float()
lo, hi = d.value_range(vol, st)
o = inr.inr_fit_opts_default(); o.boundary_batch = 16384
d.fit(vol, int(os.environ.get("FIT_STEPS", 2)), 65536, o, st, report=True)
out = torch.empty((128,) * 3, device="cuda")
inr.inr_decode_grid(d.models[0], (128,) * 3, out.data_ptr(), None, None, None, st)
g = torch.Generator(device="cuda"); g.manual_seed(7)
q = 1 << 22
pts = torch.rand((q, 3), device="cuda", generator=g) * 255.0
qo = torch.empty(q, device="cuda")
inr.inr_decode_group(d.models, pts.data_ptr(), q, qo.data_ptr(), 0, st)
cam = inr.make_camera((-180.0, 330.0, -260.0), (128.0, 110.0, 128.0), (0.0, 1.0, 0.0), 34.0, 512, 512)
tf = inr.make_tf([0.0, 0.3, 0.45, 0.7, 1.0], [[0, 0, 0, 0], [0, 0, 0, 0], [0.1, 0.4, 1.0, 0.02], [1.0, 0.8, 0.1, 0.15],
                                             [1.0, 0.1, 0.0, 0.6]], lo, hi, 1.0)
img = d.render(cam, tf, 0.5, stream=st)
vel = synth.taylor_green_volume(64, 0.0, device="cuda").contiguous()
seeds = (torch.rand((4096, 3), device="cuda", generator=g, dtype=torch.float64) * 40 + 10).contiguous()
vt = torch.empty((4096, 41, 5), dtype=torch.float64, device="cuda")
cn = torch.empty(4096, dtype=torch.int32, device="cuda")
rs = torch.empty(4096, dtype=torch.int32, device="cuda")
inr.inr_trace_grids([vel.data_ptr(), vel.data_ptr()], [0.0, 2.0], (64, 64, 64), 1.0, seeds.data_ptr(), 4096, 0.05, 40,
                    vt.data_ptr(), cn.data_ptr(), rs.data_ptr(), st)
torch.cuda.synchronize()
print("ok", float(out.mean()), float(qo.mean()), float(img[:, 3].mean()), int(cn.sum()))
