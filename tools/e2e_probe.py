"""Where the cfg2 end-to-end step (bench.py's e2e: 64 MB volume H2D from pinned
memory on a copy stream, double-buffered, one inr_fit_group step per call, losses
D2H) spends its time: per-step copy and fit durations from CUDA events, the
wall-clock period, and the same loop with the copies removed / the fits removed.
  python tools/e2e_probe.py [steps]"""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import synth
from paper_2304_10516_b200 import dnr, inr

S = int(sys.argv[1]) if len(sys.argv) > 1 else 40
torch.cuda.set_stream(torch.cuda.Stream())
st = torch.cuda.current_stream().cuda_stream
cfg = inr.make_config(precision=1, seed=0x230410516, levels=16, features=2, log2_table_size=19, mlp_hidden_layers=3)
d = dnr.DNR((256,) * 3, (128,) * 3, cfg)
vol = synth.g2_energy(256, device="cuda").float().contiguous()
d.value_range(vol, st)
o = inr.inr_fit_opts_default()
o.boundary_batch = 16384
d.fit(vol, 10, 65536, o, st, report=True)
nb = len(d.models)
host = torch.empty(vol.shape, dtype=torch.float32, pin_memory=True)
host.copy_(vol)
bufs = [torch.empty_like(vol), torch.empty_like(vol)]
rep_dev = [torch.empty(3 * nb, dtype=torch.float64, device="cuda") for _ in range(2)]
rep_host = [torch.empty(3 * nb, dtype=torch.float64, pin_memory=True) for _ in range(2)]
cs = torch.cuda.Stream()
E = lambda: torch.cuda.Event(enable_timing=True)


def loop(do_copy=True, do_fit=True, do_report=True, do_sync=True):
    copied, freed, landed = [E(), E()], [E(), E()], [E(), E()]
    c0s, c1s, f0s, f1s = [E() for _ in range(S)], [E() for _ in range(S)], [E() for _ in range(S)], [E() for _ in range(S)]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    with torch.cuda.stream(cs):
        if do_copy:
            bufs[0].copy_(host, non_blocking=True)
        copied[0].record(cs)
    for i in range(S):
        cur, nxt = i % 2, (i + 1) % 2
        if i + 1 < S:
            with torch.cuda.stream(cs):
                if i >= 1:
                    cs.wait_event(freed[nxt])
                c0s[i].record(cs)
                if do_copy:
                    bufs[nxt].copy_(host, non_blocking=True)
                c1s[i].record(cs)
                copied[nxt].record(cs)
        torch.cuda.current_stream().wait_event(copied[cur])
        f0s[i].record()
        if do_fit:
            d.fit(bufs[cur], 1, 65536, o, st, report=False)
        f1s[i].record()
        freed[cur].record()
        if do_report:
            inr.inr_fit_losses(d.models, rep_dev[cur].data_ptr(), st)
            rep_host[cur].copy_(rep_dev[cur], non_blocking=True)
        landed[cur].record()
        if i >= 1 and do_sync:
            landed[(i - 1) % 2].synchronize()
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) / S * 1e3
    cp = sorted(c0s[i].elapsed_time(c1s[i]) for i in range(S - 1))
    ft = sorted(f0s[i].elapsed_time(f1s[i]) for i in range(S))
    per = sorted(f0s[i].elapsed_time(f0s[i + 1]) for i in range(S - 1))
    return {"wall_ms_per_step": wall, "copy_ms_median": cp[len(cp) // 2], "fit_ms_median": ft[len(ft) // 2],
            "period_ms_median": per[len(per) // 2], "coords_per_s_wall": nb * 81920 / (wall / 1e3)}


res = {"both": loop(), "fit_only": loop(do_copy=False), "copy_only": loop(do_fit=False), "both_again": loop()}
print(json.dumps(res))


def pure(alternate=True, k=10):
    ev = [E() for _ in range(2 * k)]
    torch.cuda.synchronize()
    for i in range(k):
        with torch.cuda.stream(cs):
            ev[2 * i].record(cs)
            bufs[i % 2 if alternate else 0].copy_(host, non_blocking=True)
            ev[2 * i + 1].record(cs)
    torch.cuda.synchronize()
    t = sorted(ev[2 * i].elapsed_time(ev[2 * i + 1]) for i in range(k))
    return t[len(t) // 2]


print(json.dumps({"copy_only_noreport": loop(do_fit=False, do_report=False),
                  "copy_only_nosync": loop(do_fit=False, do_sync=False),
                  "copy_only_neither": loop(do_fit=False, do_report=False, do_sync=False)}))
print(json.dumps({"pure_alternate_ms": pure(True), "pure_same_ms": pure(False),
                  "host_is_pinned": host.is_pinned(), "host_contig": host.is_contiguous()}))
