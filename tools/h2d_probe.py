"""H2D bandwidth of a 64 MB pinned-host -> device copy under variations: one copy vs
the same bytes split over 2 / 4 streams (copy engines); host buffer untouched vs
filled from the device first; pinned by torch vs cudaHostRegister'd.
  python tools/h2d_probe.py"""
import json
import torch

n = 64 << 20


def bench(host, dev, k=1, reps=12):
    streams = [torch.cuda.Stream() for _ in range(k)]
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for rep in range(reps):
        torch.cuda.synchronize()
        ev0.record()
        for s in streams:
            s.wait_event(ev0)
        part = host.numel() // k
        for i, s in enumerate(streams):
            with torch.cuda.stream(s):
                dev.view(-1)[i * part:(i + 1) * part].copy_(host.view(-1)[i * part:(i + 1) * part], non_blocking=True)
        for s in streams:
            torch.cuda.current_stream().wait_stream(s)
        ev1.record()
        torch.cuda.synchronize()
        ts.append(ev0.elapsed_time(ev1))
    ts = sorted(ts[2:])
    return round(n / (ts[len(ts) // 2] / 1e3) / 1e9, 1)


dev = torch.empty(n // 4, dtype=torch.float32, device="cuda")
res = {}
h = torch.empty(n // 4, dtype=torch.float32, pin_memory=True)
res["fresh_1"] = bench(h, dev)
res["fresh_2"] = bench(h, dev, 2)
h.copy_(torch.rand(n // 4, device="cuda"))
res["filled_1"] = bench(h, dev)
h3 = torch.empty((256, 256, 256), dtype=torch.float32, pin_memory=True)
h3.copy_(torch.rand((256, 256, 256), device="cuda"))
d3 = torch.empty((256, 256, 256), dtype=torch.float32, device="cuda")
res["filled_3d_1"] = bench(h3, d3)
res["filled_3d_4"] = bench(h3, d3, 4)
print(json.dumps(res))
