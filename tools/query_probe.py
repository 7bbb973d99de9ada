"""Query-decode breakdown on the bench workload (cfg2, 8 blocks, fp16): 4 M uniform
random queries over the 256^3 volume, decoded with inr_decode_group."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2304_10516_b200 import dnr, inr
torch.cuda.set_stream(torch.cuda.Stream())
st = torch.cuda.current_stream().cuda_stream
d = dnr.DNR((256,) * 3, (128,) * 3, inr.make_config(precision=1, levels=16, features=2, log2_table_size=19,
                                                    mlp_hidden_layers=3))
vol = torch.rand((256, 256, 256), device="cuda")
d.value_range(vol, st)
o = inr.inr_fit_opts_default(); o.boundary_batch = 16384
d.fit(vol, 20, 65536, o, st, report=True)
q = int(os.environ.get("NQ", 1 << 22))
g = torch.Generator(device="cuda"); g.manual_seed(7)
pts = torch.rand((q, 3), device="cuda", generator=g) * 255.0
out = torch.empty(q, device="cuda")
for _ in range(3):
    inr.inr_decode_group(d.models, pts.data_ptr(), q, out.data_ptr(), 0, st)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    inr.inr_decode_group(d.models, pts.data_ptr(), q, out.data_ptr(), 0, st)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 5
print(f"queries {q}: {ms:.3f} ms, {q / ms / 1e6:.3f} G/s")
