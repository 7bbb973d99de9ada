"""cfg2 grid decode throughput (8 blocks of 128^3 at 1x, and 2x) after a short
fit, CUDA events, median of R repeats; checks grid == query at the nodes
bitwise on one block.

  python tools/decode_probe.py [R]
"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
from paper_2304_10516_b200 import dnr, inr

R = int(sys.argv[1]) if len(sys.argv) > 1 else 7


class SmClock:
    """Median SM clock (MHz) sampled by NVML every 5 ms while active."""
    def __init__(self):
        import threading
        import pynvml
        pynvml.nvmlInit()
        self.h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
        self.nv, self.samples, self.on = pynvml, [], True
        self.th = threading.Thread(target=self.run, daemon=True)
        self.th.start()

    def run(self):
        import time
        while self.on:
            self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
            time.sleep(0.005)

    def stop(self):
        self.on = False
        self.th.join()
        s = sorted(self.samples)
        return s[len(s) // 2] if s else None
torch.cuda.set_stream(torch.cuda.Stream())
st = torch.cuda.current_stream().cuda_stream
cfg = inr.make_config(precision=1, seed=0x230410516, levels=16, features=2, log2_table_size=19, mlp_hidden_layers=3)
d = dnr.DNR((256,) * 3, (128,) * 3, cfg)
vol = synth.g2_energy(256, device="cuda").float().contiguous()
d.value_range(vol, st)
o = inr.inr_fit_opts_default()
o.boundary_batch = 16384
d.fit(vol, 200, 65536, o, st, report=True)
out = torch.empty_like(vol)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
res = {}
for scale in (1, 2):
    if scale == 2:
        out = torch.empty((512, 512, 512), device="cuda")
    d.decode_grid_local(out, scale, None, None, st)
    torch.cuda.synchronize()
    ts = []
    clk = SmClock()
    for r in range(R):
        e0.record()
        for _ in range(5):
            d.decode_grid_local(out, scale, None, None, st)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / 5)
    mhz = clk.stop()
    ts.sort()
    vox = out.numel()
    res[f"{scale}x"] = {"ms_median": ts[len(ts) // 2], "voxels_per_s": vox / (ts[len(ts) // 2] / 1e3), "all_ms": ts,
                        "sm_mhz": mhz, "ms_at_1965": ts[len(ts) // 2] * mhz / 1965 if mhz else None}
# grid == query at the nodes of block 5 (bitwise)
out = torch.empty_like(vol)
d.decode_grid_local(out, 1, None, None, st)
z, y, x = torch.meshgrid(torch.arange(128, 256), torch.arange(0, 128), torch.arange(128, 256), indexing="ij")
pts = torch.stack([x.reshape(-1), y.reshape(-1), z.reshape(-1)], 1).float().cuda()
q = torch.empty(pts.shape[0], device="cuda")
inr.inr_decode_group(d.models, pts.data_ptr(), pts.shape[0], q.data_ptr(), 1, st)
torch.cuda.synchronize()
res["grid_equals_query_block5"] = bool(torch.equal(q, out[128:256, 0:128, 128:256].reshape(-1)))
print(json.dumps(res))
d.close()
