"""Diagnostic: mean cfg1 200-step PSNR over many seeds for one libinr build."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import synth
from oracle import sampler
from paper_2304_10516_b200 import inr
CFG1 = dict(levels=8, features=2, log2_table_size=14, mlp_hidden_layers=2)
prec = int(sys.argv[1]); seeds = range(int(sys.argv[2]), int(sys.argv[3]))
n = 64
vol = synth.g1_analytic(n).numpy(); lo, hi = sampler.value_range([vol])
vt = torch.from_numpy(vol).cuda()
view = inr.make_view(vt.data_ptr(), (0, 0, 0), (n, n, n), (1, n, n * n))
ref = (vt.double() - lo) / (hi - lo)
out = torch.empty((n, n, n), device="cuda")
blk = inr.make_block((0, 0, 0), (n, n, n), (n, n, n))
ps = []
seeds = list(seeds)
for c in range(0, len(seeds), 48):
    ms = [inr.inr_create(inr.make_config(seed=s, precision=prec, **CFG1), blk, 0) for s in seeds[c:c + 48]]
    go = inr.inr_fit_opts_default(); go.vmin, go.vmax = lo, hi
    inr.inr_fit_group(ms, [view] * len(ms), 200, 4096, go, 0)
    for m in ms:
        inr.inr_decode_grid(m, (n, n, n), out.data_ptr(), None, None, None, 0)
        ps.append(-10 * np.log10(float((((out.double() - lo) / (hi - lo) - ref) ** 2).mean())))
        inr.inr_destroy(m)
ps = np.array(ps)
print(os.environ.get("INR_LIB_PATH", "current"), "prec", prec, "n", len(ps), "mean %.3f sd %.2f se %.2f" % (ps.mean(), ps.std(), ps.std() / len(ps) ** .5), "min %.2f" % ps.min())
