"""Degenerate and boundary cases through the C ABI (SURVEY §8(c) "edge cases"):
empty inputs, single-point lattices, a 1-node-thick upper block, the domain
corners, NaN routing of absent blocks, zero-seed traces, 1x1 renders."""
import numpy as np
import pytest
import torch

import synth
from oracle import decode as o_decode, sampler
from oracle.model import InrModel
from paper_2304_10516_b200 import inr

from gpu_util import gpu_volume, make_gpu_model, normwise, oracle_config, stream, whole_view

pytestmark = pytest.mark.gpu

NET = dict(levels=8, features=2, log2_table_size=12, mlp_hidden_layers=2)


@pytest.fixture(scope="module", params=[0, 1], ids=["fp32", "fp16"])
def models(request):
    vol = synth.g1_analytic(33).numpy()                    # 33^3 with 16^3 blocks: the upper layer is 1 node
    blocks = sampler.decompose((33, 33, 33), (16, 16, 16))
    vt = gpu_volume(vol)
    go = inr.inr_fit_opts_default()
    go.vmin, go.vmax, go.boundary_batch = float(vol.min()), float(vol.max()), 32
    cfg = oracle_config(**NET)
    gms, oms = [], {}
    for b in blocks:
        m = make_gpu_model(b, 2, precision=request.param, **NET)
        inr.inr_fit(m, whole_view(vt), 5, 128, go, stream())
        p = np.empty(inr.inr_param_count(m), np.float32)
        inr.inr_get_params(m, p)
        om = InrModel(cfg, b, 2, params=p)
        om.vmin, om.vmax = go.vmin, go.vmax
        gms.append(m)
        oms[b.block_id] = om
    yield dict(gms=gms, oms=oms, blocks=blocks, tol=1e-5 if request.param == 0 else 2e-3)
    for m in gms:
        inr.inr_destroy(m)


def test_zero_queries_is_a_no_op(models):
    out = torch.full((4,), 7.0, device="cuda")
    pts = torch.zeros((4, 3), device="cuda")
    inr.inr_decode_group(models["gms"], pts.data_ptr(), 0, out.data_ptr(), 0, stream())
    torch.cuda.synchronize()
    assert torch.all(out == 7.0)


def test_single_point_lattice_and_domain_corners(models):
    gms, oms, blocks = models["gms"], models["oms"], models["blocks"]
    out = torch.full((1,), float("nan"), device="cuda")
    inr.inr_decode_grid(gms[0], (1, 1, 1), out.data_ptr(), None, None, None, stream())
    corners = np.array([[0, 0, 0], [32, 32, 32], [32, 0, 0], [0, 32, 32], [16, 16, 16], [15.999, 31.5, 32]],
                       np.float32)
    pd = torch.from_numpy(corners).cuda()
    q = torch.full((corners.shape[0],), float("nan"), device="cuda")
    inr.inr_decode_group(gms, pd.data_ptr(), corners.shape[0], q.data_ptr(), 1, stream())
    torch.cuda.synchronize()
    ref = o_decode.decode_query(oms, corners)
    assert normwise(q.cpu().numpy(), ref) <= models["tol"]
    g0 = o_decode.decode_grid(oms[blocks[0].block_id], (1, 1, 1))
    assert normwise(out.cpu().numpy(), g0.reshape(-1)) <= models["tol"]


def test_one_node_upper_block_decodes_its_node(models):
    gms, oms, blocks = models["gms"], models["oms"], models["blocks"]
    b = blocks[-1]
    assert tuple(b.origin) == (32, 32, 32)
    out = torch.full((1,), float("nan"), device="cuda")
    inr.inr_decode_grid(gms[-1], (16, 16, 16), out.data_ptr(), (1, 1, 1), None, None, stream(), count=(1, 1, 1))
    torch.cuda.synchronize()
    ref = o_decode.decode_query(oms, np.array([[32, 32, 32]], np.float32))
    assert normwise(out.cpu().numpy(), ref) <= models["tol"]


def test_strict_queries_outside_the_domain(models):
    pts = torch.tensor([[1.0, 2.0, 3.0], [-0.5, 0.0, 0.0]], device="cuda")
    out = torch.empty(2, device="cuda")
    with pytest.raises(inr.InrError) as e:
        inr.inr_decode_group(models["gms"], pts.data_ptr(), 2, out.data_ptr(), 1, stream())
    assert e.value.status == inr.INR_ERR_DOMAIN
    torch.cuda.synchronize()
    assert torch.isfinite(out).all()          # values are still written (clamped routing)


def test_zero_seed_trace_and_all_seeds_outside():
    g = torch.zeros((5, 5, 5, 3), device="cuda")
    s = torch.tensor([[-1.0, 0.0, 0.0], [0.0, 9.0, 0.0]], dtype=torch.float64, device="cuda")
    v = torch.zeros((2, 4, 5), dtype=torch.float64, device="cuda")
    c = torch.full((2,), 9, dtype=torch.int32, device="cuda")
    w = torch.full((2,), 9, dtype=torch.int32, device="cuda")
    inr.inr_trace_grids([g.data_ptr(), g.data_ptr()], [0.0, 1.0], (5, 5, 5), 1.0, s.data_ptr(), 0, 0.1, 3,
                        v.data_ptr(), c.data_ptr(), w.data_ptr(), stream())
    torch.cuda.synchronize()
    assert torch.all(c == 9)                  # nseeds = 0: untouched
    inr.inr_trace_grids([g.data_ptr(), g.data_ptr()], [0.0, 1.0], (5, 5, 5), 1.0, s.data_ptr(), 2, 0.1, 3,
                        v.data_ptr(), c.data_ptr(), w.data_ptr(), stream())
    torch.cuda.synchronize()
    assert torch.all(c == 0) and torch.all(w == inr.INR_PATH_OUT_OF_DOMAIN)


def test_one_pixel_render_and_miss(models):
    r = inr.inr_renderer_create(models["gms"], 4)
    tf = inr.make_tf([0.0, 1.0], [[0, 0, 1, 0.1], [1, 0, 0, 0.5]], 0.0, 1.0)
    frag = torch.full((1, 5), float("nan"), device="cuda")
    cam = inr.make_camera((16.0, 16.0, -40.0), (16.0, 16.0, 16.0), (0.0, 1.0, 0.0), 10.0, 1, 1)
    inr.inr_render(r, cam, tf, (0, 0, 0), (32, 32, 32), 0.5, frag.data_ptr(), stream=stream())
    torch.cuda.synchronize()
    f = frag.cpu().numpy()[0]
    assert 0 < f[3] <= 1 and abs(f[4] - 40.0) < 1e-4            # enters the box at z = 0
    away = inr.make_camera((16.0, 16.0, -40.0), (16.0, 16.0, -80.0), (0.0, 1.0, 0.0), 10.0, 1, 1)
    inr.inr_render(r, away, tf, (0, 0, 0), (32, 32, 32), 0.5, frag.data_ptr(), stream=stream())
    torch.cuda.synchronize()
    f = frag.cpu().numpy()[0]
    assert np.all(f[:4] == 0) and np.isinf(f[4])
    inr.inr_renderer_destroy(r)


def test_decode_to_rank_single_process_matches_local_decode():
    """DNR.decode_to_rank without a process group: the global volume equals the
    local decode (the peer-memory path is exercised by bench.py at N > 1)."""
    from paper_2304_10516_b200 import dnr
    vol = torch.from_numpy(synth.g1_analytic(32).numpy()).cuda()
    d = dnr.DNR((32, 32, 32), (16, 16, 16), inr.make_config(precision=1, **NET))
    d.value_range(vol, stream())
    go = inr.inr_fit_opts_default()
    d.fit(vol, 10, 256, go, stream(), report=False)
    a = torch.empty_like(vol)
    d.decode_grid_local(a, 1, None, None, stream())
    b = d.decode_to_rank(d.peer_volume(0), stream())
    torch.cuda.synchronize()
    assert torch.equal(a, b)
    h, off = inr.inr_ipc_handle(b[3:].data_ptr())
    assert len(h) == 64 and off >= 3 * 32 * 32 * 4
    d.close()


@pytest.mark.parametrize("prec", [0, 1])
def test_nonfinite_loss_and_parameters_are_reported(prec):
    """a non-finite loss or parameter after a step is an error
    (INR_ERR_NONFINITE) of the synchronous report and flag 1 of inr_fit_losses."""
    blk = sampler.decompose((16, 16, 16), (16, 16, 16))[0]
    vol = synth.g1_analytic(16).numpy().copy()
    vol[5:11, 5:11, 5:11] = np.inf                        # targets become non-finite
    vt = gpu_volume(vol)
    go = inr.inr_fit_opts_default()
    go.vmin, go.vmax = 0.0, 1.0
    m = make_gpu_model(blk, 1, precision=prec, **NET)
    with pytest.raises(inr.InrError) as e:
        inr.inr_fit(m, whole_view(vt), 2, 512, go, stream())
    assert e.value.status == inr.INR_ERR_NONFINITE
    out = torch.zeros(3, dtype=torch.float64, device="cuda")
    inr.inr_fit_losses([m], out.data_ptr(), stream())
    torch.cuda.synchronize()
    assert out[2].item() == 1.0
    # a NaN parameter, finite data
    m2 = make_gpu_model(blk, 1, precision=prec, **NET)
    p = np.empty(inr.inr_param_count(m2), np.float32)
    inr.inr_get_params(m2, p)
    p[-70] = np.nan                                        # a weight of the last layer
    inr.inr_set_params(m2, p)
    vt2 = gpu_volume(synth.g1_analytic(16).numpy())
    with pytest.raises(inr.InrError) as e:
        inr.inr_fit(m2, whole_view(vt2), 1, 512, go, stream())
    assert e.value.status == inr.INR_ERR_NONFINITE
    inr.inr_destroy(m)
    inr.inr_destroy(m2)


def test_single_model_decode_equals_group_decode(models):
    """inr_decode (one model) is the group query with that model alone."""
    gms, blocks = models["gms"], models["blocks"]
    pts = synth.random_points(5000, (33, 33, 33))
    pts = pts[(pts < 16).all(axis=1)]                       # block 0's points
    pd = torch.from_numpy(np.ascontiguousarray(pts)).cuda()
    a = torch.empty(pts.shape[0], device="cuda")
    b = torch.empty(pts.shape[0], device="cuda")
    inr.inr_decode(gms[0], pd.data_ptr(), pts.shape[0], a.data_ptr(), 1, stream())
    inr.inr_decode_group([gms[0]], pd.data_ptr(), pts.shape[0], b.data_ptr(), 1, stream())
    torch.cuda.synchronize()
    assert torch.equal(a, b) and torch.isfinite(a).all()


@pytest.mark.parametrize("prec", [0, 1])
def test_state_export_import_continues_bitwise(prec):
    """inr_export_state / inr_import_state (block stealing): a fresh model that
    imports another's state after 4 steps continues exactly like it."""
    blk = sampler.decompose((32, 32, 32), (16, 16, 16))[5]
    vt = gpu_volume(synth.g1_analytic(32).numpy())
    go = inr.inr_fit_opts_default()
    go.vmin, go.vmax, go.boundary_batch = 0.0, 1.0, 64
    a = make_gpu_model(blk, 3, reduction=1, precision=prec, **NET)
    inr.inr_fit(a, whole_view(vt), 4, 1024, go, stream())
    buf = torch.empty(inr.inr_state_bytes(a), dtype=torch.uint8, device="cuda")
    inr.inr_export_state(a, buf.data_ptr(), stream())
    b = make_gpu_model(blk, 3, reduction=1, precision=prec, **NET)
    inr.inr_import_state(b, buf.data_ptr(), stream())
    assert inr.inr_steps(b) == 4
    inr.inr_fit(a, whole_view(vt), 3, 1024, go, stream())
    inr.inr_fit(b, whole_view(vt), 3, 1024, go, stream())
    pa = np.empty(inr.inr_param_count(a), np.float32)
    pb = np.empty_like(pa)
    inr.inr_get_params(a, pa)
    inr.inr_get_params(b, pb)
    assert np.array_equal(pa, pb)
    other = make_gpu_model(sampler.decompose((32, 32, 32), (16, 16, 16))[6], 3, reduction=1, precision=prec, **NET)
    with pytest.raises(inr.InrError):                       # another block's state is refused
        inr.inr_import_state(other, buf.data_ptr(), stream())
    for m in (a, b, other):
        inr.inr_destroy(m)


def test_fp16_fit_too_deep_for_tmem_is_unsupported_but_decodes():
    blk = sampler.decompose((16, 16, 16), (16, 16, 16))[0]
    kw = dict(levels=16, features=2, log2_table_size=10, mlp_hidden_layers=8)   # 64 + 40 + 7 x 72 > 512
    m = make_gpu_model(blk, 1, precision=1, **kw)
    vt = gpu_volume(synth.g1_analytic(16).numpy())
    go = inr.inr_fit_opts_default()
    with pytest.raises(inr.InrError) as e:
        inr.inr_fit(m, whole_view(vt), 1, 256, go, stream())
    assert e.value.status == inr.INR_ERR_UNSUPPORTED
    out = torch.full((16, 16, 16), float("nan"), device="cuda")
    inr.inr_decode_grid(m, (16, 16, 16), out.data_ptr(), None, None, None, stream())
    torch.cuda.synchronize()
    assert torch.isfinite(out).all()
    inr.inr_destroy(m)


def test_block_psnrs_pool_to_the_global_psnr():
    """DNR.block_psnrs: per-block SSE on each block's core nodes; the blocks tile
    the volume, so their pooled MSE is the global one."""
    from paper_2304_10516_b200 import dnr
    vol = torch.from_numpy(synth.g1_analytic(40).numpy()).cuda()      # ragged: 40 = 16 + 16 + 8
    d = dnr.DNR((40, 40, 40), (16, 16, 16), inr.make_config(precision=1, **NET))
    lo, hi = d.value_range(vol, stream())
    d.fit(vol, 30, 512, inr.inr_fit_opts_default(), stream(), report=False)
    bp = d.block_psnrs(vol, stream())
    out = torch.empty_like(vol)
    sse = torch.zeros(1, dtype=torch.float64, device="cuda")
    d.decode_grid_local(out, 1, vol, sse, stream())
    torch.cuda.synchronize()
    counts = {}
    for b in d.block_ids:
        o = dnr.block_origin(b, d.global_dims, d.n)
        c = [min(16, 40 - o[k]) for k in range(3)]
        counts[b] = c[0] * c[1] * c[2]
    pooled = sum(10 ** (-bp[b] / 10) * counts[b] for b in bp) / 40 ** 3
    assert abs(-10 * np.log10(pooled) - d.psnr(float(sse.item()), 40 ** 3)) < 1e-6
    assert len(bp) == 27 and min(bp.values()) <= -10 * np.log10(pooled) + 1e-9
    d.close()


@pytest.mark.parametrize("prec", [0, 1])
def test_groups_larger_than_one_launch(prec):
    """72 blocks (6 x 6 x 2 of 8^3) exceed one fused launch's 64 models: the fit
    runs as two chunks and the query decode routes over all 72.  Each block ends
    bitwise as if fitted alone (deterministic mode), chunk boundary included, and
    the group query decode equals every block's own grid decode at the nodes."""
    vol = synth.g2_energy(48).numpy()[:16]                  # 48 x 48 x 16 nodes (z, y, x)
    dims = (48, 48, 16)
    blocks = sampler.decompose(dims, (8, 8, 8))
    assert len(blocks) == 72
    net = dict(levels=8, features=2, log2_table_size=10, mlp_hidden_layers=1)
    vt = gpu_volume(vol)
    go = inr.inr_fit_opts_default()
    go.vmin, go.vmax, go.boundary_batch = float(vol.min()), float(vol.max()), 32
    ms = [make_gpu_model(b, 4, precision=prec, reduction=1, **net) for b in blocks]
    reps = inr.inr_fit_group(ms, [whole_view(vt)] * 72, 3, 256, go, stream())
    assert all(r.steps_taken == 3 for r in reps)
    from gpu_util import get_params
    for k in (0, 63, 64, 71):
        single = make_gpu_model(blocks[k], 4, precision=prec, reduction=1, **net)
        inr.inr_fit(single, whole_view(vt), 3, 256, go, stream())
        assert np.array_equal(get_params(single), get_params(ms[k])), k
        inr.inr_destroy(single)
    full = torch.empty((16, 48, 48), device="cuda")
    for m, b in zip(ms, blocks):
        o = b.origin
        cnt = tuple(min(8, dims[d] - o[d]) for d in range(3))
        inr.inr_decode_grid(m, (8, 8, 8), full[o[2]:, o[1]:, o[0]:].data_ptr(), (1, 48, 48 * 48), None, None,
                            stream(), count=cnt)
    z, y, x = np.meshgrid(np.arange(16), np.arange(48), np.arange(48), indexing="ij")
    pts = np.stack([x.ravel(), y.ravel(), z.ravel()], 1).astype(np.float32)
    pd = torch.from_numpy(pts).cuda()
    q = torch.empty(pts.shape[0], device="cuda")
    inr.inr_decode_group(ms, pd.data_ptr(), pts.shape[0], q.data_ptr(), 1, stream())
    torch.cuda.synchronize()
    assert torch.equal(q, full.reshape(-1))
    for m in ms:
        inr.inr_destroy(m)


def test_concurrent_fits_from_two_host_threads():
    """Distinct models are independent (inr.h): two host threads fitting their
    own models on their own streams at the same time (ctypes releases the GIL;
    both go through the fit-graph cache) end bitwise where sequential fits end
    (deterministic mode)."""
    import threading
    vol = synth.g2_energy(32).numpy()
    blocks = sampler.decompose((32, 32, 32), (16, 16, 16))
    vt = gpu_volume(vol)
    go = inr.inr_fit_opts_default()
    go.vmin, go.vmax, go.boundary_batch = float(vol.min()), float(vol.max()), 64
    net = dict(levels=8, features=2, log2_table_size=12, mlp_hidden_layers=2)
    from gpu_util import get_params

    def fit(ms, st, reps):
        for _ in range(reps):
            inr.inr_fit_group(ms, [whole_view(vt)] * len(ms), 3, 2048, go, st.cuda_stream, False)
        st.synchronize()

    a = [make_gpu_model(b, 9, precision=1, reduction=1, **net) for b in blocks[:4]]
    b = [make_gpu_model(b, 9, precision=1, reduction=1, **net) for b in blocks[4:]]
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    th = [threading.Thread(target=fit, args=(a, s1, 5)), threading.Thread(target=fit, args=(b, s2, 5))]
    for t_ in th:
        t_.start()
    for t_ in th:
        t_.join()
    ref = [make_gpu_model(bl, 9, precision=1, reduction=1, **net) for bl in blocks]
    fit(ref[:4], s1, 5)
    fit(ref[4:], s1, 5)
    for m, r in zip(a + b, ref):
        assert np.array_equal(get_params(m), get_params(r))
    for m in a + b + ref:
        inr.inr_destroy(m)


def test_legacy_default_stream_fit_and_snapshot_staging_on_two_streams():
    """inr_fit on the legacy default stream (NULL: no CUDA graph) ends bitwise
    where the same fit on a created stream (cached graph) ends; a host-resident
    fp16 cache snapshot decoded first on one stream and at once on another gets
    the same values on both (its staging completes before either decode reads it)."""
    vol = synth.g1_analytic(32).numpy()
    blk = sampler.decompose((32, 32, 32), (32, 32, 32))[0]
    vt = gpu_volume(vol)
    go = inr.inr_fit_opts_default()
    go.vmin, go.vmax = float(vol.min()), float(vol.max())
    from gpu_util import get_params
    a = make_gpu_model(blk, 3, precision=1, reduction=1, **NET)
    b = make_gpu_model(blk, 3, precision=1, reduction=1, **NET)
    inr.inr_fit(a, whole_view(vt), 4, 1024, go, 0)
    inr.inr_fit(b, whole_view(vt), 4, 1024, go, stream())
    assert np.array_equal(get_params(a), get_params(b))
    c = inr.cache_create(2, inr.CACHE_HOST_RESIDENT | inr.CACHE_FP16, 0)
    inr.cache_insert(c, 1, [a], stream())
    torch.cuda.synchronize()
    _, snap = inr.cache_get(c, 0)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    o1 = torch.empty((32, 32, 32), device="cuda")
    o2 = torch.empty((32, 32, 32), device="cuda")
    inr.inr_decode_grid(snap[0], (32, 32, 32), o1.data_ptr(), None, None, None, s1.cuda_stream)
    inr.inr_decode_grid(snap[0], (32, 32, 32), o2.data_ptr(), None, None, None, s2.cuda_stream)
    torch.cuda.synchronize()
    assert torch.equal(o1, o2) and torch.isfinite(o1).all()
    inr.cache_destroy(c)
    inr.inr_destroy(a)
    inr.inr_destroy(b)
