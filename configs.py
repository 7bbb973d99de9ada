"""configs.py — runs BASELINE.json's five configurations through the library
and records fit coords/s, decode voxels/s (or queries/s) and PSNR @ compression
ratio for each.  The headline bench line is bench.py (cfg2);
this script is the per-config evidence, written to profiles/.

  python configs.py [--only cfg1,cfg3] [--out profiles/r1_configs.json] [--world-slice]

Every config runs on ONE GPU: cfg3 fits all 64 blocks on it, cfg5 fits one
GPU's share (64 of the 512 blocks: a 1024 x 1024 x 128 slab of the 1024^3
volume).  Times are CUDA events on the launching stream.
"""
import argparse
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2304_10516_b200 import dnr, inr  # noqa: E402

NET2 = dict(levels=16, features=2, log2_table_size=19, mlp_hidden_layers=3)


def ev():
    return torch.cuda.Event(enable_timing=True)


def gen_local(kind, gdims, lo, hi, dev, tau=0.35, dtype=torch.float64):
    """The analytic field on the node box [lo, hi] (x, y, z inclusive), [z][y][x] fp32."""
    out = torch.empty((hi[2] - lo[2] + 1, hi[1] - lo[1] + 1, hi[0] - lo[0] + 1), dtype=torch.float32, device=dev)
    for z0 in range(0, out.shape[0], 8):
        z1 = min(z0 + 8, out.shape[0])
        pos = synth.lattice(gdims, dev, (lo[2] + z0, lo[2] + z1))[:, lo[1]:hi[1] + 1, lo[0]:hi[0] + 1]
        out[z0:z1] = synth.evaluate(kind, pos.to(dtype), gdims, tau=tau).to(torch.float32)
    return out


def fit_and_measure(d, vol, steps, batch, bb, stream):
    opts = inr.inr_fit_opts_default()
    opts.boundary_batch = bb
    d.fit(vol, 2, batch, opts, stream, report=True)          # warm-up (2 steps)
    torch.cuda.synchronize()
    e0, e1 = ev(), ev()
    e0.record()
    reps = d.fit(vol, steps - 2, batch, opts, stream, report=True)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    coords = len(d.models) * (batch + bb) * (steps - 2)   # every block of these configs has an interior face
    return ms, coords, reps


def psnr_1x(d, vol, stream):
    out = torch.empty_like(vol)
    sse = torch.zeros(1, dtype=torch.float64, device=vol.device)
    d.decode_grid_local(out, 1, None, None, stream)          # warm
    torch.cuda.synchronize()
    e0, e1 = ev(), ev()
    e0.record()
    d.decode_grid_local(out, 1, vol, sse, stream)
    e1.record()
    torch.cuda.synchronize()
    lo, hi = d.core_box()
    n = 1
    for a in range(3):
        n *= hi[a] - lo[a] + 1
    return d.psnr(float(sse.item()), n), e0.elapsed_time(e1), n


def ratio(d, n_core):
    return 4.0 * n_core / d.param_bytes()


def run_cfg1(stream, prec):
    n = 64
    dev = torch.device("cuda")
    cfg = inr.make_config(levels=8, features=2, log2_table_size=14, mlp_hidden_layers=2, precision=prec)
    d = dnr.DNR((n, n, n), (n, n, n), cfg)
    vol = synth.g1_analytic(n, device=dev)
    d.value_range(vol, stream)
    ms, coords, _ = fit_and_measure(d, vol, 200, 4096, 0, stream)
    p, dms, nvox = psnr_1x(d, vol, stream)
    r = {"config": "cfg1", "precision": "fp16" if prec else "fp32", "fit_coords_per_s": coords / (ms / 1e3),
         "fit_ms_per_step": ms / 198, "decode_voxels_per_s": nvox / (dms / 1e3), "psnr_db": p,
         "steps": 200, "compression_ratio": ratio(d, n ** 3)}
    d.close()
    return r


def run_cfg2(stream, prec):
    n = 256
    dev = torch.device("cuda")
    d = dnr.DNR((n, n, n), (128, 128, 128), inr.make_config(precision=prec, **NET2))
    vol = gen_local("g2", (n, n, n), d.lo, d.hi, dev)
    d.value_range(vol, stream)
    ms, coords, _ = fit_and_measure(d, vol, 2000, 65536, 16384, stream)
    p, dms, nvox = psnr_1x(d, vol, stream)
    r = {"config": "cfg2", "precision": "fp16" if prec else "fp32", "fit_coords_per_s": coords / (ms / 1e3),
         "fit_ms_per_step": ms / 1998, "decode_voxels_per_s": nvox / (dms / 1e3), "psnr_db": p,
         "steps": 2000, "compression_ratio": ratio(d, n ** 3)}
    d.close()
    return r


def run_cfg2r(stream, prec, log2t=15):
    """NOT a BASELINE config: cfg2's data with right-sized tables (T = 2^15), to show
    the PSNR @ ratio trade-off where the model is smaller than the data (R24)."""
    n = 256
    dev = torch.device("cuda")
    d = dnr.DNR((n, n, n), (128, 128, 128), inr.make_config(precision=prec, **dict(NET2, log2_table_size=log2t)))
    vol = gen_local("g2", (n, n, n), d.lo, d.hi, dev)
    d.value_range(vol, stream)
    ms, coords, _ = fit_and_measure(d, vol, 2000, 65536, 16384, stream)
    p, dms, nvox = psnr_1x(d, vol, stream)
    r = {"config": f"cfg2r (not BASELINE: cfg2 with T = 2^{log2t})", "precision": "fp16" if prec else "fp32",
         "fit_coords_per_s": coords / (ms / 1e3), "fit_ms_per_step": ms / 1998,
         "decode_voxels_per_s": nvox / (dms / 1e3), "psnr_db": p, "steps": 2000,
         "compression_ratio": ratio(d, n ** 3), "compression_ratio_fp16_stored": 2 * ratio(d, n ** 3)}
    d.close()
    return r


def run_cfg3(stream, prec):
    """512^3 G3, 64 blocks on one GPU, cfg2 network, 1000 steps; decode 1x and 2x
    (2x against the analytic field)."""
    n = 512
    dev = torch.device("cuda")
    d = dnr.DNR((n, n, n), (128, 128, 128), inr.make_config(precision=prec, **NET2))
    vol = gen_local("g3", (n, n, n), d.lo, d.hi, dev)
    d.value_range(vol, stream)
    ms, coords, _ = fit_and_measure(d, vol, 1000, 65536, 16384, stream)
    p1, dms1, nvox = psnr_1x(d, vol, stream)
    # 2x: decode z-slabs of blocks at scale 2 and compare with the analytic field at (k + j/2)
    sse2, n2, dms2 = 0.0, 0, 0.0
    rng = (d.vmax - d.vmin)
    for bz in range(4):
        ids = [b for b in d.block_ids if dnr.block_origin(b, d.global_dims, d.n)[2] == bz * 128]
        out = torch.empty((256, 1024, 1024), dtype=torch.float32, device=dev)
        e0, e1 = ev(), ev()
        e0.record()
        for b in ids:
            m = d.models[d.block_ids.index(b)]
            o = dnr.block_origin(b, d.global_dims, d.n)
            base = out[:, 2 * o[1]:, 2 * o[0]:]
            inr.inr_decode_grid(m, (256, 256, 256), base.data_ptr(), (1, 1024, 1024 * 1024), None, None, stream)
        e1.record()
        torch.cuda.synchronize()
        dms2 += e0.elapsed_time(e1)
        for z0 in range(0, 256, 16):
            zs = (torch.arange(z0, z0 + 16, device=dev, dtype=torch.float32) / 2 + bz * 128)
            ys = torch.arange(1024, device=dev, dtype=torch.float32) / 2
            xs = torch.arange(1024, device=dev, dtype=torch.float32) / 2
            zz, yy, xx = torch.meshgrid(zs, ys, xs, indexing="ij")
            pos = torch.stack([xx, yy, zz], -1).clamp(max=float(n - 1))
            truth = synth.evaluate("g3", pos, (n, n, n)).to(torch.float32)
            sse2 += float((((out[z0:z0 + 16].double() - truth.double()) / rng) ** 2).sum())
            n2 += truth.numel()
        del out
    p2 = -10 * math.log10(sse2 / n2) if sse2 > 0 else 200.0
    r = {"config": "cfg3", "precision": "fp16" if prec else "fp32", "blocks": len(d.models),
         "fit_coords_per_s": coords / (ms / 1e3), "fit_ms_per_step": ms / 998, "steps": 1000,
         "decode_1x_voxels_per_s": nvox / (dms1 / 1e3), "psnr_1x_db": p1,
         "decode_2x_voxels_per_s": n2 / (dms2 / 1e3), "psnr_2x_db_vs_analytic": p2,
         "compression_ratio": ratio(d, n ** 3)}
    d.close()
    return r


def run_cfg4(stream, prec, timesteps=100, window=40, steps=500, cache_flags=inr.CACHE_FP16, warm=False):
    """Temporal cache: per timestep of an evolving G2 256^3
    field, reset + fit 500 steps, insert into a window of 40 (FIFO evicts);
    every 10th insert decodes a random cached timestep at 256^3.  warm: NEXT-4
    warm start — keep the previous timestep's network, restart Adam and the
    learning-rate schedule (inr_reset_optimizer) instead of a fresh init."""
    n = 256
    dev = torch.device("cuda")
    d = dnr.DNR((n, n, n), (128, 128, 128), inr.make_config(precision=prec, **NET2))
    cache = inr.cache_create(window, cache_flags, 0)
    rs = np.random.default_rng(4)
    fit_ms, psnrs, bytes_curve, trig = [], [], [], []
    opts = inr.inr_fit_opts_default()
    opts.boundary_batch = 16384
    vols = {}
    for ti in range(timesteps):
        tau = ti / timesteps
        vol = gen_local("g2", (n, n, n), d.lo, d.hi, dev, tau=tau)
        d.value_range(vol, stream)
        for m in d.models:
            if warm and ti > 0:
                inr.inr_reset_optimizer(m)
            else:
                inr.inr_reset(m, 0x230410516 + ti)
        e0, e1 = ev(), ev()
        e0.record()
        d.fit(vol, steps, 65536, opts, stream, report=True)
        e1.record()
        torch.cuda.synchronize()
        fit_ms.append(e0.elapsed_time(e1))
        ev_ts = inr.cache_insert(cache, ti, d.models, stream)
        bytes_curve.append(inr.cache_bytes(cache))
        vols[ti] = vol
        if ev_ts >= 0:
            vols.pop(ev_ts, None)
        if ti % 10 == 9:
            k = int(rs.integers(0, inr.cache_size(cache)))
            ts, blocks = inr.cache_get(cache, k)
            out = torch.empty((n, n, n), device=dev)
            sse = torch.zeros(1, dtype=torch.float64, device=dev)
            e0, e1 = ev(), ev()
            e0.record()
            for b, bid in zip(blocks, d.block_ids):
                o = dnr.block_origin(bid, d.global_dims, d.n)
                inr.inr_decode_grid(b, (128, 128, 128), out[o[2]:, o[1]:, o[0]:].data_ptr(), (1, n, n * n),
                                    vols[ts][o[2]:, o[1]:, o[0]:].data_ptr() if ts in vols else None,
                                    sse.data_ptr() if ts in vols else None, stream)
            e1.record()
            torch.cuda.synchronize()
            tr = {"insert": ti, "decoded_timestep": ts, "decode_ms": e0.elapsed_time(e1)}
            if ts in vols:
                tr["psnr_db"] = -10 * math.log10(float(sse.item()) / n ** 3)
            trig.append(tr)
        # PSNR of the fresh model on its own timestep
        p, _, _ = psnr_1x(d, vol, stream)
        psnrs.append(p)
    r = {"config": "cfg4" + (" warm start (NEXT-4)" if warm else ""), "precision": "fp16" if prec else "fp32",
         "timesteps": timesteps, "window": window, "init": "warm (previous timestep)" if warm else "fresh",
         "steps_per_insert": steps, "fit_ms_per_insert_mean": float(np.mean(fit_ms)),
         "fit_coords_per_s": 8 * (65536 + 16384) * steps / (np.mean(fit_ms) / 1e3),
         "psnr_db_mean": float(np.mean(psnrs)), "psnr_db_min": float(np.min(psnrs)),
         "cache_bytes_final": bytes_curve[-1], "cache_bytes_max": max(bytes_curve),
         "cache_bytes_curve_every10": bytes_curve[::10], "evictions": timesteps - window,
         "triggers": trig, "compression_ratio": ratio(d, n ** 3) * (2 if cache_flags & inr.CACHE_FP16 else 1),
         "cache_storage": "fp16" if cache_flags & inr.CACHE_FP16 else "fp32",
         "raw_bytes_window": window * 4 * n ** 3}
    inr.cache_destroy(cache)
    d.close()
    return r


def run_cfg5(stream, prec):
    """One GPU's share of cfg5: 64 of the 512 blocks (a 1024 x 1024 x 128 slab), T = 2^22,
    200 fit steps just to get a model, then a query-throughput sweep 2^10 .. 2^26 over
    the slab (block-bucketed), and the slab's 1x grid decode."""
    n = 1024
    dev = torch.device("cuda")
    net = dict(NET2, log2_table_size=22)
    d = dnr.DNR((n, n, n), (128, 128, 128), inr.make_config(precision=prec, **net), rank=0, world=8)
    vol = gen_local("g3", (n, n, n), d.lo, d.hi, dev)
    d.value_range(vol, stream)     # (one GPU: its own range; the 8-GPU run all-reduces)
    ms, coords, _ = fit_and_measure(d, vol, 200, 65536, 16384, stream)
    p, dms, nvox = psnr_1x(d, vol, stream)
    sweep = []
    lo, hi = d.core_box()
    span = torch.tensor([hi[0] - lo[0], hi[1] - lo[1], hi[2] - lo[2]], device=dev, dtype=torch.float32)
    base = torch.tensor(lo, device=dev, dtype=torch.float32)
    for e in range(10, 27, 2):
        q = 1 << e
        g = torch.Generator(device=dev)
        g.manual_seed(e)
        pts = torch.rand((q, 3), device=dev, generator=g) * span + base
        out = torch.empty(q, device=dev)
        inr.inr_decode_group(d.models, pts.data_ptr(), q, out.data_ptr(), 0, stream)
        torch.cuda.synchronize()
        e0, e1 = ev(), ev()
        e0.record()
        reps = 3
        for _ in range(reps):
            inr.inr_decode_group(d.models, pts.data_ptr(), q, out.data_ptr(), 0, stream)
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / reps
        sweep.append({"queries": q, "ms": t, "queries_per_s": q / (t / 1e3)})
        del pts, out
    r = {"config": "cfg5 (one GPU's 64 of 512 blocks)", "precision": "fp16" if prec else "fp32",
         "blocks": len(d.models), "fit_coords_per_s": coords / (ms / 1e3), "fit_ms_per_step": ms / 198,
         "steps": 200, "decode_1x_voxels_per_s": nvox / (dms / 1e3), "psnr_1x_db": p,
         "query_sweep": sweep, "compression_ratio": ratio(d, 128 ** 3 * len(d.models)),
         "param_bytes_gpu": d.param_bytes()}
    d.close()
    return r


def run_next2(stream, prec, n=256, window=10, steps=500, M=1 << 16, dt=0.1, amp=2.0):
    """NEXT-2: a time-varying Taylor-Green velocity field (G4, 256^3,
    8 blocks of 128^3, D = 3) fitted per timestep (500 steps) into a window of 10;
    then backward pathlines P = pathline(negate(reverse(W))) of M seeds
    from a box, the forward pass from their end points (Fig. 8A round trip), and
    the same backward trace on the ground-truth grids (Fig. 8B comparison)."""
    dev = torch.device("cuda")
    gd = (n, n, n)
    cfg = inr.make_config(precision=prec, out_dim=3, **NET2)
    d = dnr.DNR(gd, (128, 128, 128), cfg)
    cache = inr.cache_create(window + 1, 0, 0)
    opts = inr.inr_fit_opts_default()
    opts.boundary_batch = 16384
    lat = synth.lattice(gd, dev)
    gt, fit_ms, psnrs = [], [], []
    for ts in range(window):
        vol = synth.taylor_green(lat, gd, float(ts), amp=amp).to(torch.float32).contiguous()
        d.value_range(vol, stream)
        for m in d.models:
            inr.inr_reset(m, 0x230410516 + ts)
        e0, e1 = ev(), ev()
        e0.record()
        d.fit(vol, steps, 65536, opts, stream, report=True)
        e1.record()
        torch.cuda.synchronize()
        fit_ms.append(e0.elapsed_time(e1))
        out = torch.empty_like(vol)
        sse = torch.zeros(1, dtype=torch.float64, device=dev)
        d.decode_grid_local(out, 1, vol, sse, stream)
        torch.cuda.synchronize()
        psnrs.append(d.psnr(float(sse.item()), 3 * n ** 3))
        inr.cache_insert(cache, ts, d.models, stream)
        gt.append(vol)
        del out
    del lat
    rng = np.random.default_rng(11)
    lo_box, hi_box = np.array([64.0, 64.0, 64.0]), np.array([192.0, 192.0, 192.0])
    seeds = lo_box + rng.random((M, 3)) * (hi_box - lo_box)
    K = int(math.ceil((window - 1) / dt)) + 2

    def run(fn):
        vert = torch.empty((M, K + 1, 5), dtype=torch.float64, device=dev)
        cnt = torch.empty(M, dtype=torch.int32, device=dev)
        why = torch.empty(M, dtype=torch.int32, device=dev)
        fn(vert, cnt, why)               # warm
        torch.cuda.synchronize()
        inr.inr_profile_enable(1)
        e0, e1 = ev(), ev()
        e0.record()
        fn(vert, cnt, why)
        e1.record()
        torch.cuda.synchronize()
        kms = inr.inr_profile_read("pathline")[0]
        inr.inr_profile_enable(0)
        return vert, cnt, why, e0.elapsed_time(e1), kms

    sd = torch.from_numpy(seeds).to(dev)
    ops = inr.INR_WINDOW_REVERSE | inr.INR_WINDOW_NEGATE
    vb, cb, rb, ms_b, kms_b = run(lambda v, c, w: inr.inr_pathlines(cache, ops, sd.data_ptr(), M, dt, K, v.data_ptr(),
                                                                    c.data_ptr(), w.data_ptr(), stream))
    cbn, rbn = cb.cpu().numpy(), rb.cpu().numpy()
    ok = rbn == inr.INR_PATH_WINDOW_EXHAUSTED
    ends = vb[torch.arange(M, device=dev), cb.long() - 1, :3].contiguous()
    steps_b = int((cbn - 1).clip(min=0).sum())
    # forward from the backward end points (Fig. 8A): seeds that left the domain are dropped
    ok_t = torch.from_numpy(ok).to(dev)
    ends_ok = ends[ok_t].contiguous()
    Mf = int(ends_ok.shape[0])
    vf = torch.empty((Mf, K + 1, 5), dtype=torch.float64, device=dev)
    cf = torch.empty(Mf, dtype=torch.int32, device=dev)
    rf = torch.empty(Mf, dtype=torch.int32, device=dev)
    inr.inr_pathlines(cache, 0, ends_ok.data_ptr(), Mf, dt, K, vf.data_ptr(), cf.data_ptr(), rf.data_ptr(), stream)
    torch.cuda.synchronize()
    back = vf[torch.arange(Mf, device=dev), cf.long() - 1, :3]
    fin = rf == inr.INR_PATH_WINDOW_EXHAUSTED
    rt = (back - sd[ok_t])[fin].norm(dim=1).cpu().numpy()
    # ground truth: the same backward trace on the analytic grids (post hoc)
    times = [float(t) for t in range(window)]
    gt_rev = gt[::-1]
    tau = [times[-1] - t for t in times[::-1]]
    vg, cg, rg, ms_g, _ = run(lambda v, c, w: inr.inr_trace_grids([g.data_ptr() for g in gt_rev], tau, gd, -1.0,
                                                                   sd.data_ptr(), M, dt, K, v.data_ptr(),
                                                                   c.data_ptr(), w.data_ptr(), stream))
    both = ok & (rg.cpu().numpy() == inr.INR_PATH_WINDOW_EXHAUSTED)
    bt = torch.from_numpy(both).to(dev)
    gends = vg[torch.arange(M, device=dev), cg.long() - 1, :3]
    dev_gt = (ends - gends)[bt].norm(dim=1).cpu().numpy()
    r = {"config": "NEXT-2 Taylor-Green 256^3 (8 x 128^3 blocks, D=3), window 10, backward pathlines",
         "precision": "fp16" if prec else "fp32", "fit_steps_per_timestep": steps,
         "fit_coords_per_s": 8 * (65536 + 16384) * steps / (np.mean(fit_ms) / 1e3),
         "psnr_db_mean": float(np.mean(psnrs)), "psnr_db_min": float(np.min(psnrs)),
         "compression_ratio": 3 * 4.0 * n ** 3 / d.param_bytes(),
         "seeds": M, "dt": dt, "substeps_per_seed_max": K,
         "backward_ms_total": ms_b, "backward_ms_kernels": kms_b,
         "backward_ms_decode": ms_b - kms_b,
         "particle_steps": steps_b, "particle_steps_per_s_kernels": steps_b / (kms_b / 1e3),
         "particle_steps_per_s_with_decode": steps_b / (ms_b / 1e3),
         "seeds_exhausted_window": int(ok.sum()), "seeds_left_domain": int((rbn == 1).sum()),
         "roundtrip_err_nodes": {"median": float(np.median(rt)), "p99": float(np.percentile(rt, 99)),
                                 "max": float(rt.max()), "n": int(rt.size)},
         "dnr_vs_ground_truth_endpoint_nodes": {"median": float(np.median(dev_gt)),
                                                "p90": float(np.percentile(dev_gt, 90)),
                                                "max": float(dev_gt.max()), "n": int(dev_gt.size)},
         "ground_truth_trace_ms": ms_g}
    inr.cache_destroy(cache)
    d.close()
    return r


def run_next3(stream, prec, n=256, steps=1000, width=1024, height=1024):
    """NEXT-3: direct-query volume rendering of the cfg2 DNR
    (G2 256^3, 8 blocks, fitted 1000 steps) at 1024^2, sample streaming over the
    tensor-core query decode, with and without macro-cell skipping; the
    single-rank sort-last path (DNR.render) for the full frame time."""
    dev = torch.device("cuda")
    d = dnr.DNR((n, n, n), (128, 128, 128), inr.make_config(precision=prec, **NET2))
    vol = gen_local("g2", (n, n, n), d.lo, d.hi, dev)
    vmin, vmax = d.value_range(vol, stream)
    opts = inr.inr_fit_opts_default()
    opts.boundary_batch = 16384
    d.fit(vol, steps, 65536, opts, stream, report=True)
    del vol
    cam = inr.make_camera((-180.0, 330.0, -260.0), (128.0, 110.0, 128.0), (0.0, 1.0, 0.0), 34.0, width, height)
    tf = inr.make_tf([0.0, 0.3, 0.45, 0.7, 1.0],
                     [[0.0, 0.0, 0.0, 0.0], [0.0, 0.0, 0.0, 0.0], [0.1, 0.4, 1.0, 0.02], [1.0, 0.8, 0.1, 0.15],
                      [1.0, 0.1, 0.0, 0.6]], vmin, vmax, 1.0)
    step = 0.5
    r = inr.inr_renderer_create(d.models, 16, 1e-3 * (vmax - vmin), stream)
    frag = torch.empty((width * height, 5), device=dev)
    out = {}
    for mc in (0, 1):
        inr.inr_render(r, cam, tf, d.lo, d.hi, step, frag.data_ptr(), 0.99, mc, stream)   # warm
        torch.cuda.synchronize()
        e0, e1 = ev(), ev()
        e0.record()
        inr.inr_render(r, cam, tf, d.lo, d.hi, step, frag.data_ptr(), 0.99, mc, stream)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        evald, skipped, waves = inr.inr_render_stats(r)
        out["macrocells" if mc else "no_macrocells"] = {
            "ms": ms, "samples_evaluated": evald, "samples_skipped": skipped, "waves": waves,
            "evaluated_samples_per_s": evald / (ms / 1e3), "rays_per_s": width * height / (ms / 1e3)}
    alpha = frag[:, 3].float()
    coverage = float((alpha > 0.01).float().mean())
    inr.inr_renderer_destroy(r)
    torch.cuda.synchronize()
    e0, e1 = ev(), ev()
    e0.record()
    img = d.render(cam, tf, step, stream=stream)
    e1.record()
    torch.cuda.synchronize()
    res = {"config": "NEXT-3 direct-query DVR of the cfg2 DNR (G2 256^3, 8 blocks), 1024^2, step 0.5",
           "precision": "fp16" if prec else "fp32", "fit_steps": steps, "image": [width, height],
           "coverage_alpha_gt_0.01": coverage, "mean_alpha": float(img[:, 3].mean()),
           "frame_ms_dnr_render": e0.elapsed_time(e1), **out}
    d.close()
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="cfg1,cfg2,cfg2r,cfg3,cfg4,cfg5")
    ap.add_argument("--precision", default="fp16,fp32")
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r1_configs.json"))
    a = ap.parse_args()
    torch.cuda.set_stream(torch.cuda.Stream())
    stream = torch.cuda.current_stream().cuda_stream
    fns = {"cfg1": run_cfg1, "cfg2": run_cfg2, "cfg2r": run_cfg2r, "cfg3": run_cfg3, "cfg4": run_cfg4,
           "cfg5": run_cfg5, "next2": run_next2, "next3": run_next3,
           "cfg4w": lambda st, p: run_cfg4(st, p, steps=250, warm=True),
           "cfg4c250": lambda st, p: run_cfg4(st, p, steps=250)}
    results = []
    for name in a.only.split(","):
        for p in a.precision.split(","):
            prec = inr.INR_PREC_FP16_MLP if p == "fp16" else inr.INR_PREC_FP32
            if name in ("cfg2r", "cfg3", "cfg4", "cfg4w", "cfg4c250", "cfg5", "next2", "next3") and p == "fp32":
                continue          # the fp32 CUDA-core path is the parity mode; large configs run fp16
            t0 = time.time()
            r = fns[name](stream, prec)
            r["wall_s"] = time.time() - t0
            print(json.dumps(r), flush=True)
            results.append(r)
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    with open(a.out, "w") as f:
        json.dump({"gpu": torch.cuda.get_device_name(0), "results": results}, f, indent=1)


if __name__ == "__main__":
    main()
