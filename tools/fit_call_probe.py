"""Host overhead of one inr_fit_group(steps=1, report) call on the cfg2 workload."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
from paper_2304_10516_b200 import dnr, inr
torch.cuda.set_stream(torch.cuda.Stream())
st = torch.cuda.current_stream().cuda_stream
d = dnr.DNR((256,) * 3, (128,) * 3, inr.make_config(precision=1, levels=16, features=2, log2_table_size=19, mlp_hidden_layers=3))
vol = torch.rand((257 if False else 256, 256, 256), device="cuda")
d.value_range(vol, st)
o = inr.inr_fit_opts_default(); o.boundary_batch = 16384
for rep in (True, False):
    for k in range(3): d.fit(vol, 1, 65536, o, st, report=rep)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for k in range(20): d.fit(vol, 1, 65536, o, st, report=rep)
    torch.cuda.synchronize()
    print("report" if rep else "async", "ms/call %.3f" % ((time.perf_counter() - t) / 20 * 1e3))
t = time.perf_counter(); d.fit(vol, 20, 65536, o, st, report=True); torch.cuda.synchronize()
print("graph 20 steps ms/step %.3f" % ((time.perf_counter() - t) / 20 * 1e3))
