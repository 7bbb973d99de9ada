"""cfg2 fit-step time on the production path (no profiling: the cached one-step
CUDA graph replayed per step), CUDA events around K steps, median of R repeats;
then one profiled K-step run for per-kernel-class device time.  For A/B runs
of two builds in one gpurun call, point INR_LIB_PATH at each libinr.so.

  python tools/step_probe.py [K] [R] [NZ]

NZ (default 2): blocks along z, i.e. 4 NZ blocks of 128^3 (a 256 x 256 x 128 NZ volume,
the G2 field tiled along z): 8 = cfg2, 16 / 32 / 64 = cfg3's blocks per rank at 4 / 2 / 1 GPUs.
"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
from paper_2304_10516_b200 import dnr, inr

K = int(sys.argv[1]) if len(sys.argv) > 1 else 50
R = int(sys.argv[2]) if len(sys.argv) > 2 else 5
NZ = int(sys.argv[3]) if len(sys.argv) > 3 else 2
torch.cuda.set_stream(torch.cuda.Stream())
st = torch.cuda.current_stream().cuda_stream
cfg = inr.make_config(precision=1, seed=0x230410516, levels=16, features=2, log2_table_size=19, mlp_hidden_layers=3)
d = dnr.DNR((256, 256, 128 * NZ), (128,) * 3, cfg)
g2 = synth.g2_energy(256, device="cuda").float()
vol = torch.cat([g2[(z * 128) % 256:(z * 128) % 256 + 128] for z in range(NZ)], 0).contiguous() \
    if NZ != 2 else g2.contiguous()
d.value_range(vol, st)
o = inr.inr_fit_opts_default()
o.boundary_batch = 16384
d.fit(vol, 10, 65536, o, st, report=True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ts = []
for r in range(R):
    e0.record()
    d.fit(vol, K, 65536, o, st, report=False)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1) / K)
ts.sort()
inr.inr_profile_enable(1)
d.fit(vol, K, 65536, o, st, report=False)
torch.cuda.synchronize()
span = inr.inr_profile_span()
prof = {k: inr.inr_profile_read(k) for k in ("step_begin", "encode_fwd", "prep_image", "mlp_tc", "encode_bwd", "adam")}
inr.inr_profile_enable(0)
rep = d.fit(vol, 1, 65536, o, st, report=True)
print(json.dumps({"lib": inr.LIB_PATH, "ms_per_step_median": ts[len(ts) // 2], "ms_per_step_all": ts,
                  "coords_per_s": 4 * NZ * 81920 / (ts[len(ts) // 2] / 1e3),
                  "profiled_span_ms_per_step": span / K,
                  "per_step_ms": {k: v[0] / K for k, v in prof.items()},
                  "launches_per_step": {k: v[1] / K for k, v in prof.items()}}))
d.close()
