"""Multi-GPU correctness of the distributed shell: two
ranks, one process each, fit their own blocks with no communication inside the
fit loop ("reduces the need for data communication ... during the
network training") and together decode exactly what one process fitting every
block decodes.  NCCL over two GPUs when the box has them; otherwise both
ranks share cuda:0 and their (few) collectives go over gloo -- the decode
comparison and the collective count do not depend on the backend."""
import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

GDIMS, BLOCK, STEPS, BATCH = (64, 64, 64), (32, 32, 32), 12, 2048
NET = dict(levels=8, features=2, log2_table_size=14, mlp_hidden_layers=2)
COLLECTIVES = ("all_reduce", "all_gather", "all_gather_object", "all_gather_into_tensor", "reduce_scatter",
               "reduce_scatter_tensor", "broadcast", "broadcast_object_list", "gather", "gather_object", "scatter",
               "reduce", "send", "recv", "isend", "irecv", "barrier", "all_to_all", "all_to_all_single")


def _volume():
    import synth
    return synth.g2_energy(64).numpy()


def _fit_and_decode(rank, world, vol_np):
    """This rank's blocks: value range (all-reduce), fit, 1x decode of the local
    cores.  Returns (local decode [z, y, x] on the CPU, lo corner, collectives
    counted while the unreported K-step DNR.fit ran)."""
    import torch.distributed as dist

    from paper_2304_10516_b200 import dnr, inr
    cfg = inr.make_config(seed=5, precision=inr.INR_PREC_FP16_MLP, reduction=inr.INR_REDUCE_DETERMINISTIC, **NET)
    d = dnr.DNR(GDIMS, BLOCK, cfg, rank, world, torch.cuda.current_device())
    lo, hi = d.lo, d.hi
    vol = torch.from_numpy(np.ascontiguousarray(vol_np[lo[2]:hi[2] + 1, lo[1]:hi[1] + 1, lo[0]:hi[0] + 1])).cuda()
    st = torch.cuda.current_stream().cuda_stream
    d.value_range(vol, st)
    opts = inr.inr_fit_opts_default()
    opts.boundary_batch = 512
    # count every torch.distributed call made while the fit runs
    counts = {"n": 0}
    saved = {}
    for name in COLLECTIVES:
        f = getattr(dist, name, None)
        if f is None:
            continue

        def wrap(*a, _f=f, **k):
            counts["n"] += 1
            return _f(*a, **k)
        saved[name] = f
        setattr(dist, name, wrap)
    try:
        # the whole K-step fit of the rank's blocks (report=False: no metadata all-gather
        # after the loop either, which is the only exchange DNR.fit can make)
        d.fit(vol, STEPS, BATCH, opts, st, report=False)
        torch.cuda.synchronize()
        n_fit = counts["n"]
        # the counter sees collectives: a reported fit ends with exactly one metadata
        # all-gather at N > 1, however many steps it takes
        rep = d.fit(vol, 2, BATCH, opts, st, report=True)
        torch.cuda.synchronize()
        n_report = counts["n"] - n_fit
        assert len(rep) == 8 and n_report == (1 if world > 1 else 0), n_report
    finally:
        for name, f in saved.items():
            setattr(dist, name, f)
    out = torch.empty_like(vol)
    d.decode_grid_local(out, 1, None, None, st)
    torch.cuda.synchronize()
    clo, chi = d.core_box()
    core = out[: chi[2] - clo[2] + 1, : chi[1] - clo[1] + 1, : chi[0] - clo[0] + 1].cpu().numpy()
    d.close()
    return core, clo, n_fit


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank_main(rank, world, port, backend, tmp):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dev = rank if backend == "nccl" else 0
    torch.cuda.set_device(dev)
    if backend == "nccl":
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", dev))
    else:
        dist.init_process_group("gloo", rank=rank, world_size=world)
    core, lo, n = _fit_and_decode(rank, world, _volume())
    np.save(os.path.join(tmp, f"core{rank}.npy"), core)
    np.save(os.path.join(tmp, f"meta{rank}.npy"), np.array(list(lo) + [n], np.int64))
    dist.barrier()
    dist.destroy_process_group()


def test_two_ranks_decode_equals_one_rank_and_fit_has_no_collectives():
    vol = _volume()
    ref, lo1, n1 = _fit_and_decode(0, 1, vol)           # one process, every block
    assert ref.shape == (64, 64, 64) and tuple(lo1) == (0, 0, 0) and n1 == 0
    backend = "nccl" if torch.cuda.device_count() >= 2 else "gloo"
    with tempfile.TemporaryDirectory() as tmp:
        ctx = mp.get_context("spawn")
        port = _free_port()
        ps = [ctx.Process(target=_rank_main, args=(r, 2, port, backend, tmp)) for r in range(2)]
        for p in ps:
            p.start()
        for p in ps:
            p.join(600)
        assert all(p.exitcode == 0 for p in ps), [p.exitcode for p in ps]
        full = np.full((64, 64, 64), np.nan, np.float32)
        for r in range(2):
            core = np.load(os.path.join(tmp, f"core{r}.npy"))
            meta = np.load(os.path.join(tmp, f"meta{r}.npy"))
            x, y, z, ncoll = (int(v) for v in meta)
            assert ncoll == 0, f"rank {r}: {ncoll} torch.distributed calls inside DNR.fit"
            full[z:z + core.shape[0], y:y + core.shape[1], x:x + core.shape[2]] = core
    print("backend", backend, "max |2-rank - 1-rank|", float(np.nanmax(np.abs(full - ref))))
    assert not np.isnan(full).any()
    assert np.array_equal(full, ref)                     # bitwise (deterministic reduction)
