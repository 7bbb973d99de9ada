"""Host-side logic of the multi-GPU shell (dnr.py) on CPU: block
partitioning, and the only collectives the method needs (P:L193-205:
range MIN/MAX before fitting, SSE SUM and metadata all-gather after), run
with world_size 2 over gloo."""
import os
import socket

import pytest
import torch.multiprocessing as mp

from paper_2304_10516_b200 import dnr


def test_partition_is_contiguous_and_covers():
    for nb, w in ((8, 1), (64, 8), (64, 3), (7, 4), (512, 8)):
        parts = [dnr.partition_blocks(nb, w, r) for r in range(w)]
        flat = [b for p in parts for b in p]
        assert flat == list(range(nb))
        assert max(map(len, parts)) - min(map(len, parts)) <= 1


def test_block_geometry_and_local_box():
    g = (256, 256, 512)
    assert dnr.block_grid(g, (128, 128, 128)) == (2, 2, 4)
    assert dnr.block_origin(5, g, (128,) * 3) == (128, 0, 128)
    ids = dnr.partition_blocks(16, 2, 0)                    # z rows 0..1
    assert dnr.local_node_box(ids, g, (128,) * 3) == ((0, 0, 0), (255, 255, 256))
    ids = dnr.partition_blocks(16, 2, 1)
    assert dnr.local_node_box(ids, g, (128,) * 3) == ((0, 0, 256), (255, 255, 511))


def test_block_box_check():
    """A rank's blocks must form an axis-aligned box (its sub-volume, slab and
    render brick are their bounding box): cfg3's 64 blocks split in 1/2/4/8
    and cfg2's weak-scaling slabs do; 64 blocks on 3 ranks do not."""
    g3, n = (512, 512, 512), (128,) * 3
    for w in (1, 2, 4, 8, 16):
        assert all(dnr.is_block_box(dnr.partition_blocks(64, w, r), g3, n) for r in range(w)), w
    assert not all(dnr.is_block_box(dnr.partition_blocks(64, 3, r), g3, n) for r in range(3))
    assert not dnr.is_block_box([0, 1, 2, 3, 4], g3, n)          # a row and a stray block
    assert dnr.is_block_box([5], g3, n) and not dnr.is_block_box([], g3, n)
    g2 = (256, 256, 256 * 4)
    assert all(dnr.is_block_box(dnr.partition_blocks(32, 4, r), g2, n) for r in range(4))


def test_psnr_from_sse():
    assert dnr.psnr_from_sse(0.0, 10) == 200.0
    assert abs(dnr.psnr_from_sse(0.01 * 10, 10) - 20.0) < 1e-12


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = [(0.0, 1.0), (-2.0, 0.5)][rank]
    rng = dnr.allreduce_range(lo, hi)
    sse = dnr.allreduce_sum([0.5 * (rank + 1), 100.0])
    meta = dnr.allgather_metadata([[float(rank), 10.0 + rank]])
    mx = dnr.allreduce_max(3.0 * rank)
    import torch
    # rank r owns z-slab r of a (4, 3, 2r+2)-shaped volume: slabs of different shapes
    slab = torch.full((2 + rank, 3, 4), float(rank + 1))
    vol = dnr.gather_slabs(slab, (0, 0, 2 * rank), (4, 3, 5))
    ok = None
    if rank == 0:
        ok = bool((vol[0:2] == 1).all() and (vol[2:5] == 2).all())
    # sort-last fragments (NEXT-3): every rank's [npix][5] image stacked in rank order on rank 0
    frag = torch.full((6, 5), float(rank)) + torch.arange(6.0)[:, None]
    fr = dnr.gather_fragments(frag)
    fok = None if fr is None else bool(fr.shape == (2, 6, 5) and (fr[1] - fr[0] == 1).all())
    vrng = dnr.allreduce_range([lo, 2.0 * lo], [hi, 3.0 * hi])     # per-channel ranges (vector fields)
    q.put((rank, rng, sse, meta, mx, (ok, fok), vrng))
    dist.destroy_process_group()


def test_collectives_world2_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(2))
    for p in ps:
        p.join(60)
    assert res[0][5] == (True, True) and res[1][5] == (None, None)     # slab / fragment gathers to rank 0
    for rank, rng, sse, meta, mx, _, vrng in res:
        assert vrng == ([-2.0, -4.0], [1.0, 3.0])
        assert rng == (-2.0, 1.0)                         # S:L275-277 example
        assert sse == [1.5, 200.0]
        assert meta == [[0.0, 10.0], [1.0, 11.0]]
        assert mx == 3.0


def test_steal_plan():
    # ranks 1 and 2 idle: rank 0's six unfinished blocks end up two per rank
    plan = dnr.steal_plan([(0, [0, 1, 2, 3, 4, 5]), (1, []), (2, [])])
    assert plan == [(0, 1, 5), (0, 1, 4), (0, 2, 3), (0, 2, 2)]
    # eight blocks, three idle ranks: 2 + 2 + 2 + 2
    plan = dnr.steal_plan([(0, list(range(8))), (1, []), (2, []), (3, [])])
    assert [sum(1 for p in plan if p[1] == r) for r in (1, 2, 3)] == [2, 2, 2]
    assert dnr.steal_plan([(0, [7]), (1, [])]) == []                  # never the last block
    assert dnr.steal_plan([(0, [1, 2]), (1, [])], already_moved={1, 2}) == []   # a block moves once
    assert dnr.steal_plan([(0, [1, 2]), (1, [3])]) == []              # nobody idle
