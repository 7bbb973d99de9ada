"""bench.py — fit coords/s (and decode voxels/s, PSNR @ ratio) of the hash-grid
INR hot path on B200, per the BASELINE.json metric on configs[1]:

  cfg2: a 256^3 CloverLeaf3D-shaped energy field (G2, tau =
  0.35), 2x2x2 blocks of 128^3 on one GPU, L=16 T=2^19 F=2, 3x64 MLP,
  B_u = 65536 uniform + B_b = 16384 boundary samples per block per step.

A "step" is one fit iteration over all local blocks (sampling, targets,
encode, MLP fwd, Eq. 2, MLP bwd, table scatter, Adam: §8(a) a2-a12).  Under
torchrun each rank fits its own 8 blocks of a 256 x 256 x 256N volume (weak
scaling; no collective inside the step).  `value` = coordinates fitted per
second over all ranks (max-over-ranks device time).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""
import argparse
import json
import math
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

BLOCK = 128
SIDE = 256
CFG = dict(levels=16, features=2, log2_table_size=19, mlp_hidden_layers=3)
B_U, B_B = 65536, 16384
PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=200)
    p.add_argument("--warmup", type=int, default=10)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--precision", default="fp16", choices=["fp16", "fp32"])
    p.add_argument("--psnr-steps", type=int, default=2000, help="total fit steps before the PSNR report (0: skip)")
    p.add_argument("--no-cpu-baseline", action="store_true")
    return p.parse_args()


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return d, "measured (MEASURED_PEAKS.json)"
    except OSError:
        return PEAKS_FALLBACK, "fallback (B200_PROFILING.md)"


# ------------------------------------------------------------------- CPU legs
def oracle_step_sample(steps, warmup, frac=0.25):
    """The oracle (test infrastructure) as it stands, on a bounded sample: each
    step is one fit step of ONE cfg2 block at `frac` of its batch.  Returns
    (coords/s, cores, description)."""
    import numpy as np
    from threadpoolctl import threadpool_limits

    import synth
    from oracle import fit as o_fit, sampler
    from oracle.model import Config, InrModel
    n = SIDE
    vol = synth.g2_energy(n).numpy()
    lo, hi = float(vol.min()), float(vol.max())
    blk = sampler.decompose((n, n, n), (BLOCK,) * 3)[0]
    bu, bb = int(B_U * frac), int(B_B * frac)
    with threadpool_limits(1):
        m = InrModel(Config(**CFG), blk, 1)
        opts = o_fit.FitOpts(vmin=lo, vmax=hi, boundary_batch=bb)
        for _ in range(warmup):
            o_fit.train_step(m, vol, opts, bu)
        t0 = time.perf_counter()
        for _ in range(steps):
            o_fit.train_step(m, vol, opts, bu)
        dt = time.perf_counter() - t0
    coords = steps * (bu + bb)
    desc = (f"{steps} oracle fit steps (after {warmup} warm-up) of one 128^3 cfg2 block at {bu}+{bb} "
            f"coords/step ({frac / 8:.4f} of a cfg2 step), numpy fp64, 1 thread")
    return coords / dt, 1, desc


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    steps, warm = max(1, args.steps), max(0, args.warmup)
    # each step a bounded sample of one cfg2 block-step, sized so that the whole
    # K + W run stays within ~2 minutes (the oracle does ~15 K coords/s on one core)
    frac = max(1.0 / 64, min(0.25, 15000.0 * 120.0 / (steps + warm) / (B_U + B_B)))
    v, cores, desc = oracle_step_sample(steps, warm, frac)
    line = {
        "metric": "fit_coords_per_s", "value": v, "unit": "coords/s", "impl": "reference",
        "n_gpus": args.gpus, "steps": steps, "warmup": warm, "higher_is_better": True,
        "dtype": "f64", "data": "synthetic", "config": workload_config(1, args),
        "cpu_baseline": {"value": v, "unit": "coords/s", "cores": cores, "kind": "oracle", "sample": desc},
        "e2e": {"value": v, "unit": "coords/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "vs_baseline": None,
    }
    print(json.dumps(line), flush=True)


def workload_config(world, args):
    return {"workload": "cfg2: G2 256^3 CloverLeaf3D-shaped energy, 2x2x2 blocks of 128^3 per GPU, "
                        "L16 T2^19 F2, 3x64 MLP, 65536+16384 coords/block/step",
            "global_dims": [SIDE, SIDE, SIDE * world], "blocks_per_gpu": 8, "block": BLOCK,
            "batch_uniform": B_U, "batch_boundary": B_B, "precision": args.precision,
            "parallelism": f"blocks{world}" if world > 1 else "single",
            "l2": "no flush: per-GPU working set (params+grads+Adam state 1.56 GB, volume 64 MB) >> 126 MB L2"}


# ------------------------------------------------------------------- clocks
class Clocks:
    """nvidia-smi sampled every 20 ms; only samples stamped inside the timed region count."""
    FIELDS = ("timestamp,clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "20"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None

    def stop(self, t0=None, t1=None):
        """Median SM clock and active throttle reasons over samples with t0 <= stamp <= t1 (host time)."""
        import datetime
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        sm, smax, reasons, n_all = [], None, set(), 0
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in out.strip().splitlines():
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 8:
                continue
            n_all += 1
            try:
                ts = datetime.datetime.strptime(f[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
                if t0 is not None and not (t0 - 0.02 <= ts <= t1 + 0.02):
                    continue
                sm.append(float(f[1]))
                smax = float(f[2])
            except ValueError:
                continue
            for nm, val in zip(names, f[4:8]):
                if val.lower() == "active":
                    reasons.add(nm)
        sm.sort()
        med = sm[len(sm) // 2] if sm else None
        return {"sm_mhz": med, "sm_max_mhz": smax, "reasons": sorted(reasons), "samples": len(sm),
                "samples_total": n_all}


def ncu_traffic(kernel):
    """dram__bytes_read.sum + dram__bytes_write.sum of one launch of `kernel` from the
    committed ncu --set full capture (profiles/), in bytes, or None."""
    name = {"adam": "adam_kernel", "mlp_tc": "mlp_fit_kernel", "encode_bwd": "encode_bwd_kernel",
            "encode_fwd": "encode_fwd_kernel"}.get(kernel, kernel)
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "r1_final_ncu_full.txt")
    try:
        blk = None
        for line in open(path):
            if line.startswith("["):
                blk = line.strip()
            elif blk and name in blk and line.strip().startswith("traffic (read+write)"):
                val, unit = float(line.split()[-2]), line.split()[-1]
                scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}[unit]
                return val * scale, os.path.relpath(path, os.path.dirname(path) + "/..") + \
                    " (ncu --set full, one launch)"
    except OSError:
        pass
    return None


# ------------------------------------------------------------------- our arm
def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    import synth
    from paper_2304_10516_b200 import dnr, inr

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    torch.cuda.set_stream(torch.cuda.Stream(dev))     # a capturable stream: libinr replays CUDA graphs on it
    stream = torch.cuda.current_stream().cuda_stream
    gdims = (SIDE, SIDE, SIDE * world)
    prec = inr.INR_PREC_FP16_MLP if args.precision == "fp16" else inr.INR_PREC_FP32
    cfg = inr.make_config(precision=prec, seed=0x230410516, **CFG)
    d = dnr.DNR(gdims, (BLOCK,) * 3, cfg, rank, world, local)
    lo, hi = d.lo, d.hi
    # the rank's sub-volume (cores + 1-node high ghost layer), generated on the GPU
    zs = torch.arange(lo[2], hi[2] + 1, dtype=torch.float64, device=dev)
    vol = torch.empty((hi[2] - lo[2] + 1, hi[1] - lo[1] + 1, hi[0] - lo[0] + 1), dtype=torch.float32, device=dev)
    for z0 in range(0, vol.shape[0], 16):
        z1 = min(z0 + 16, vol.shape[0])
        pos = synth.lattice(gdims, dev, (lo[2] + z0, lo[2] + z1))[:, lo[1]:hi[1] + 1, lo[0]:hi[0] + 1]
        vol[z0:z1] = synth.evaluate("g2", pos, gdims).to(torch.float32)
    del zs
    vmin, vmax = d.value_range(vol, stream)                    # a1 + all-reduce MIN/MAX
    opts = inr.inr_fit_opts_default()
    opts.boundary_batch = B_B
    nb = len(d.models)
    coords_per_step = nb * (B_U + B_B)

    # warm-up (untimed)
    d.fit(vol, max(args.warmup, 1), B_U, opts, stream, report=True)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()

    # ---- timed region: K fit steps, every kernel bracketed by CUDA events
    launches0 = inr.inr_kernel_launches()
    inr.inr_profile_enable(1)
    clocks = Clocks(local)
    clocks.start()
    time.sleep(0.5)   # nvidia-smi start-up: its first samples land before the timed region
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev0.record()
    t_host0 = time.time()
    d.fit(vol, args.steps, B_U, opts, stream, report=False)
    ev1.record()
    torch.cuda.synchronize()
    t_host1 = time.time()
    if world > 1:
        dist.barrier()
    ms_outer = ev0.elapsed_time(ev1)            # includes the host-side graph capture of the K steps
    ms = inr.inr_profile_span()                 # device time: first kernel start -> last kernel end
    clk = clocks.stop(t_host0, t_host1)
    launches = inr.inr_kernel_launches() - launches0
    prof = {k: inr.inr_profile_read(k)
            for k in ("step_begin", "encode_fwd", "prep_image", "mlp_tc", "encode_bwd", "fit_fp32", "adam")}
    inr.inr_profile_enable(0)
    ms_max = dnr.allreduce_max(ms)
    value = coords_per_step * world * args.steps / (ms_max / 1e3)

    # ---- roofline of the dominant kernel (device time share)
    P = inr.inr_param_count(d.models[0])
    pk, pv = peaks()
    kern = {k: v for k, v in prof.items() if v[1] > 0}
    dom = max(kern, key=lambda k: kern[k][0])
    dom_ms, dom_n = kern[dom]
    avg_s = dom_ms / dom_n / 1e3
    if dom == "adam":
        # algorithmic bytes: read p, g, m, v + write p, m, v (fp32) for every parameter of every block
        alg = 28.0 * P * nb
        roof = {"kernel": "adam", "bound": "hbm", "achieved": alg / avg_s / 1e9, "peak": pk["hbm_gbs"],
                "unit": "GB/s", "traffic": None, "algorithmic_bytes_per_launch": alg}
    else:
        # the fused fit kernel: the dense contraction part on the tensor roofline
        # (6 (LF W + (H-1) W^2 + W) FLOP per coordinate), plus its
        # algorithmic L2 gather/scatter bytes (2 x 8 L F 4 B per coordinate)
        LF, W, H = 32, 64, 3
        flop = 6.0 * (LF * W + (H - 1) * W * W + W) * coords_per_step
        peak = pk.get("bf16_tflops_sustained", pk["bf16_tflops"])  # fp16 dense rate == bf16 on B200
        roof = {"kernel": dom, "bound": "tensor", "achieved": flop / avg_s / 1e12, "peak": peak,
                "unit": "TFLOP/s", "traffic": None, "algorithmic_flop_per_launch": flop,
                "l2_gather_scatter_bytes_per_launch": 2 * 8 * 16 * 2 * 4.0 * coords_per_step}
    roof["frac"] = roof["achieved"] / roof["peak"]
    tr = ncu_traffic(roof["kernel"])
    if tr is not None:
        roof["traffic"], roof["traffic_source"] = tr
    roof["peak_source"] = pv
    roof["avg_launch_ms"] = avg_s * 1e3
    roof["share_of_step"] = dom_ms / ms
    kernels = {k: {"total_ms": v[0], "launches": v[1], "avg_ms": v[0] / max(v[1], 1)} for k, v in kern.items()}
    # the gather / scatter kernels against the measured random-access peaks (tools/l2_peaks.py)
    try:
        with open(os.path.join(ROOT, "profiles", "r1_l2_peaks.json")) as f:
            lp = {(r["op"], r["buffer_MB"]): r["per_s"] for r in json.load(f)["results"]}
        corners = 8.0 * CFG["levels"] * coords_per_step
        for k, op in (("encode_fwd", "gather_16B"), ("encode_bwd", "red_v4_f32")):
            if k in kernels:
                rate = corners / (kernels[k]["avg_ms"] / 1e3)
                kernels[k].update({"corner_accesses_per_s": rate, "random_access_peak_per_s": lp[(op, 4)],
                                   "peak_note": f"{op}, 4 MB L2-resident buffer, measured; x-neighbour corner "
                                                "pairs share one access, so corners/s can exceed the access peak"})
    except (OSError, KeyError, ValueError):
        pass

    # ---- end to end through the public API with host buffers: every step the
    # volume is copied H2D from pinned memory, one fit step runs through
    # inr_fit_group, and its losses come back to the host (inr_fit_losses -> D2H)
    host = torch.empty(vol.shape, dtype=torch.float32, pin_memory=True)
    host.copy_(vol)
    bufs = [torch.empty_like(vol), torch.empty_like(vol)]
    rep_dev = [torch.empty(3 * nb, dtype=torch.float64, device=dev) for _ in range(2)]
    rep_host = [torch.empty(3 * nb, dtype=torch.float64, pin_memory=True) for _ in range(2)]
    copy_stream = torch.cuda.Stream(dev)
    copied = [torch.cuda.Event(), torch.cuda.Event()]
    freed = [torch.cuda.Event(), torch.cuda.Event()]
    landed = [torch.cuda.Event(), torch.cuda.Event()]
    e_steps = max(3, min(args.steps, 50))
    losses = []

    def read_report(j):
        landed[j % 2].synchronize()
        r = rep_host[j % 2].numpy().reshape(nb, 3)
        if r[:, 2].any() or not np.isfinite(r[:, :2]).all():
            raise RuntimeError(f"non-finite loss at e2e step {j}")
        losses.append(float(r[:, 0].mean()))

    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    # step i's input volume is copied H2D from pinned memory on a copy stream while
    # step i-1 computes (double buffering); step i's losses are copied D2H behind it
    # and read on the host while step i+1 runs (one step in flight, no per-step stall)
    with torch.cuda.stream(copy_stream):
        bufs[0].copy_(host, non_blocking=True)
        copied[0].record(copy_stream)
    for i in range(e_steps):
        cur, nxt = i % 2, (i + 1) % 2
        if i + 1 < e_steps:
            with torch.cuda.stream(copy_stream):
                if i >= 1:
                    copy_stream.wait_event(freed[nxt])
                bufs[nxt].copy_(host, non_blocking=True)
                copied[nxt].record(copy_stream)
        torch.cuda.current_stream().wait_event(copied[cur])
        d.fit(bufs[cur], 1, B_U, opts, stream, report=False)
        freed[cur].record()
        inr.inr_fit_losses(d.models, rep_dev[cur].data_ptr(), stream)
        rep_host[cur].copy_(rep_dev[cur], non_blocking=True)
        landed[cur].record()
        if i >= 1:
            read_report(i - 1)
    read_report(e_steps - 1)
    torch.cuda.synchronize()
    e_s = dnr.allreduce_max(time.perf_counter() - t0)
    e2e = {"value": coords_per_step * world * e_steps / e_s, "unit": "coords/s",
           "h2d_bytes_per_step": int(vol.numel() * 4), "d2h_bytes_per_step": int(3 * nb * 8),
           "steps": e_steps, "clock": "host wall clock around the whole loop (first copy to last loss read), "
                                      "max over ranks",
           "pipeline": "each step's 64 MB input copied H2D from pinned memory on a copy stream during the "
                       "previous step (double-buffered); one inr_fit_group step; its losses (inr_fit_losses) "
                       "copied D2H and read on the host while the next step runs",
           "last_loss_uniform_mean": losses[-1]}

    # ---- decode throughput (1x grid of the local cores) and PSNR @ ratio
    out = torch.empty_like(vol)
    sse = torch.zeros(1, dtype=torch.float64, device=dev)
    d.decode_grid_local(out, 1, None, None, stream)                      # warm
    torch.cuda.synchronize()
    inr.inr_profile_enable(1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    d.decode_grid_local(out, 1, None, None, stream)
    e1.record()
    torch.cuda.synchronize()
    dec_ms = dnr.allreduce_max(e0.elapsed_time(e1))
    inr.inr_profile_enable(0)
    vox_local = BLOCK ** 3 * len(d.models)
    # random queries over the rank's blocks (bucketed by block, tensor-core MLP for fp16 models)
    nq = 1 << 22
    g = torch.Generator(device=dev)
    g.manual_seed(7)
    pts = torch.rand((nq, 3), device=dev, generator=g, dtype=torch.float32)
    span = torch.tensor([d.hi[0] - d.lo[0], d.hi[1] - d.lo[1], d.hi[2] - d.lo[2]], device=dev, dtype=torch.float32)
    pts = pts * span + torch.tensor(d.lo, device=dev, dtype=torch.float32)
    qout = torch.empty(nq, device=dev)
    inr.inr_decode_group(d.models, pts.data_ptr(), nq, qout.data_ptr(), 0, stream)   # warm
    torch.cuda.synchronize()
    e0.record()
    inr.inr_decode_group(d.models, pts.data_ptr(), nq, qout.data_ptr(), 0, stream)
    e1.record()
    torch.cuda.synchronize()
    q_ms = dnr.allreduce_max(e0.elapsed_time(e1))
    decode = {"voxels_per_s": vox_local * world / (dec_ms / 1e3), "ms": dec_ms, "voxels": vox_local * world,
              "kernel": "decode_grid: " + ("tcgen05 fp16 MLP, R19 vertex elision" if prec else "fp32 CUDA-core MLP"),
              "queries_per_s": nq * world / (q_ms / 1e3), "queries": nq * world, "query_ms": q_ms}
    if world > 1:   # a18: decoded slabs -> rank 0 (NCCL gather over NVLink), reported separately
        full = d.gather(out, 0)              # warm (NCCL communicator set-up)
        del full
        torch.cuda.synchronize()
        dist.barrier()
        t0 = time.perf_counter()
        full = d.gather(out, 0)
        torch.cuda.synchronize()
        decode["gather_ms"] = dnr.allreduce_max((time.perf_counter() - t0) * 1e3)
        decode["gather_bytes"] = int(4 * SIDE ** 3 * world)
        # the same gather fused into the decode: every rank's decode kernels store their
        # slab into rank 0's volume through NVLink peer memory (CUDA IPC)
        target = d.peer_volume(0)                # rank 0's volume, mapped once on every rank (CUDA IPC)
        d.decode_to_rank(target, stream)         # warm
        torch.cuda.synchronize()
        dist.barrier()
        t0 = time.perf_counter()
        p2p = d.decode_to_rank(target, stream)
        torch.cuda.synchronize()
        decode["decode_and_gather_p2p_ms"] = dnr.allreduce_max((time.perf_counter() - t0) * 1e3)
        decode["decode_then_nccl_gather_ms"] = dec_ms + decode["gather_ms"]
        if rank == 0:
            decode["p2p_equals_nccl_gather"] = bool(torch.equal(p2p, full))
        del full, p2p, target
    done = args.warmup + args.steps + e_steps
    if args.psnr_steps > done:
        d.fit(vol, args.psnr_steps - done, B_U, opts, stream, report=True)
        done = args.psnr_steps
    sse.zero_()
    d.decode_grid_local(out, 1, vol, sse, stream)
    torch.cuda.synchronize()
    # core nodes only (the high ghost layer belongs to the next rank)
    ncore = 1
    for dd in range(3):
        ncore *= (d.hi[dd] - d.lo[dd] + 1) if d.hi[dd] == gdims[dd] - 1 else (d.hi[dd] - d.lo[dd])
    psnr = d.psnr(float(sse.item()), ncore)
    bp = d.block_psnrs(vol, stream)
    psnr_block_min = dnr.allreduce_max(-min(bp.values())) * -1.0
    raw_bytes = 4.0 * SIDE ** 3
    ratio = raw_bytes / d.param_bytes()

    # ---- NEXT-3: sort-last direct-query volume rendering of the trained DNR (1024^2)
    W = H = 1024
    cam = inr.make_camera((-180.0, 330.0, -260.0 * world), (128.0, 110.0, 128.0 * world), (0.0, 1.0, 0.0), 34.0, W, H)
    tf = inr.make_tf([0.0, 0.3, 0.45, 0.7, 1.0], [[0.0, 0.0, 0.0, 0.0], [0.0, 0.0, 0.0, 0.0], [0.1, 0.4, 1.0, 0.02],
                                                 [1.0, 0.8, 0.1, 0.15], [1.0, 0.1, 0.0, 0.6]], vmin, vmax, 1.0)
    d.render(cam, tf, 0.5, stream=stream)                       # warm
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    nframes = 3                                                  # mean over a few frames (one frame is noisy)
    t0 = time.perf_counter()
    for _ in range(nframes):
        img = d.render(cam, tf, 0.5, stream=stream)
    torch.cuda.synchronize()
    r_ms = dnr.allreduce_max((time.perf_counter() - t0) * 1e3 / nframes)
    ev_s, sk_s, waves = d.last_render_stats
    tot = dnr.allreduce_sum([float(ev_s), float(sk_s)])
    render = {"image": [W, H], "frame_ms": r_ms, "frames_timed": nframes, "samples_evaluated": int(tot[0]),
              "samples_skipped": int(tot[1]),
              "evaluated_samples_per_s": tot[0] / (r_ms / 1e3), "waves_rank0": waves, "step": 0.5,
              "path": "per-rank sample-streaming ray march (tensor-core queries, macro-cells), fragments stored "
                      "into rank 0's stack through NVLink peer memory, depth-composited there"}
    if img is not None:
        render["mean_alpha"] = float(img[:, 3].mean())
    del img

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, cores, desc = oracle_step_sample(2, 0)
        cpu = {"value": v, "unit": "coords/s", "cores": cores, "kind": "oracle", "sample": desc,
               "cpu": _cpu_model()}
    if rank == 0:
        line = {
            "metric": "fit_coords_per_s", "value": value, "unit": "coords/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
            "timing": "CUDA events on the launching stream around every library kernel of the K steps "
                      "(one captured CUDA graph); ms = first kernel start -> last kernel end, max over ranks",
            "host_capture_ms": ms_outer - ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f16-mlp/f32" if prec else "f32", "data": "synthetic",
            "config": workload_config(world, args),
            "roofline": roof, "kernels": kernels, "cpu_baseline": cpu, "e2e": e2e,
            "decode": decode, "render": render, "psnr_db": psnr, "psnr_block_min_db": psnr_block_min,
            "psnr_after_steps": done,
            "compression_ratio": ratio,
            "clocks": clk, "gpu_launches": launches,
        }
        print(json.dumps(line), flush=True)
    d.close()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def _cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip() + f" x{os.cpu_count()}"
    except OSError:
        pass
    return None


if __name__ == "__main__":
    a = parse()
    if a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)
