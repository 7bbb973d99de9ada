"""Pathlines over the temporal window (NEXT-2) through the C ABI vs
oracle/pathline.py (R29-R31).

* inr_trace_grids on the same fp32 grids as the oracle: the kernel follows the
  oracle's float64 operation order with no FMA contraction, so positions,
  times, counts and reasons are bit-exact (speeds to 1e-15);
* inr_pathlines over a cache of fitted D = 3 models equals decode + trace on
  the GPU bitwise, and the oracle's trace over its own fp64 decode of the same
  parameters within 1e-3 node units (fp32 vs fp64 decode, RK4 propagation);
* partial-lattice decode of a ragged upper block (inr_decode_grid_part)."""
import numpy as np
import pytest
import torch

import synth
from oracle import decode as o_decode, pathline as o_pl, sampler
from oracle.model import InrModel
from paper_2304_10516_b200 import inr

from gpu_util import gpu_volume, make_gpu_model, normwise, oracle_config, stream, whole_view

pytestmark = pytest.mark.gpu

V = dict(levels=8, features=2, log2_table_size=14, mlp_hidden_layers=2, out_dim=3)


def _gpu_trace(grids, times, dims, sign, seeds, dt, max_steps):
    gd = [torch.from_numpy(np.ascontiguousarray(g, np.float32)).cuda() for g in grids]
    sd = torch.from_numpy(np.ascontiguousarray(seeds, np.float64)).cuda()
    M = seeds.shape[0]
    vert = torch.full((M, max_steps + 1, 5), float("nan"), dtype=torch.float64, device="cuda")
    cnt = torch.zeros(M, dtype=torch.int32, device="cuda")
    why = torch.zeros(M, dtype=torch.int32, device="cuda")
    inr.inr_trace_grids([g.data_ptr() for g in gd], times, dims, sign, sd.data_ptr(), M, dt, max_steps,
                        vert.data_ptr(), cnt.data_ptr(), why.data_ptr(), stream())
    torch.cuda.synchronize()
    return vert.cpu().numpy(), cnt.cpu().numpy(), why.cpu().numpy()


def _assert_same(gpu, ora, exact=True, tol=0.0):
    (vg, cg, rg), (vo, co, ro) = gpu, ora
    assert np.array_equal(cg, co) and np.array_equal(rg, ro)
    for s in range(cg.shape[0]):
        a, b = vg[s, :cg[s]], vo[s, :co[s]]
        if exact:
            assert np.array_equal(a[:, :4], b[:, :4]), (s, np.max(np.abs(a[:, :4] - b[:, :4])))
            assert np.allclose(a[:, 4], b[:, 4], rtol=1e-15, atol=0)
        else:
            assert np.max(np.abs(a[:, :3] - b[:, :3])) <= tol, (s, np.max(np.abs(a[:, :3] - b[:, :3])))


def _tgv_window(n, times, amp=3.0):
    lat = synth.lattice((n, n, n))
    return [synth.taylor_green(lat, (n, n, n), t, amp=amp).to(torch.float32).numpy() for t in times]


def _seeds(n, m, rng):
    s = rng.random((m, 3)) * (n - 1)
    s[0] = [-0.5, 3.0, 3.0]                  # outside at t_0: no vertex
    s[1] = [n - 1.01, n / 2, n / 2]          # leaves the domain soon
    s[2] = [0.0, 0.0, 0.0]                   # a corner node
    return s


@pytest.mark.parametrize("backward", [False, True])
def test_trace_grids_bitexact_vs_oracle(backward):
    n = 33
    times = [0.0, 0.5, 1.25, 2.0]
    W = _tgv_window(n, times)
    seeds = _seeds(n, 200, np.random.default_rng(1))
    grids, tt, sign = o_pl.reverse_negate(W, times, reverse=backward, negate=backward)
    ora = o_pl.trace([g.astype(np.float64) for g in grids], tt, seeds, 0.07, 500, sign)
    gpu = _gpu_trace(grids, tt, (n, n, n), sign, seeds, 0.07, 500)
    assert np.sum(gpu[2] == inr.INR_PATH_OUT_OF_DOMAIN) >= 2 and np.sum(gpu[2] == 0) >= 100
    _assert_same(gpu, ora)


def test_trace_grids_max_steps_and_single_interval():
    n = 17
    W = _tgv_window(n, [0.0, 3.0])
    seeds = np.random.default_rng(2).random((64, 3)) * (n - 1)
    ora = o_pl.trace([g.astype(np.float64) for g in W], [0.0, 3.0], seeds, 0.1, 12)
    gpu = _gpu_trace(W, [0.0, 3.0], (n, n, n), 1.0, seeds, 0.1, 12)
    assert np.sum(gpu[2] == inr.INR_PATH_MAX_STEPS) >= 32
    _assert_same(gpu, ora)


def test_trace_rejects_bad_arguments():
    g = torch.zeros((4, 4, 4, 3), device="cuda")
    s = torch.zeros((1, 3), dtype=torch.float64, device="cuda")
    out = torch.zeros(10, dtype=torch.float64, device="cuda")
    c = torch.zeros(1, dtype=torch.int32, device="cuda")
    for times, dt in (([0.0, 0.0], 0.1), ([0.0, 1.0], 0.0)):
        with pytest.raises(inr.InrError):
            inr.inr_trace_grids([g.data_ptr(), g.data_ptr()], times, (4, 4, 4), 1.0, s.data_ptr(), 1, dt, 1,
                                out.data_ptr(), c.data_ptr(), c.data_ptr(), stream())


def test_decode_grid_part_ragged_upper_block():
    """N = 40, n = 16: the upper block (o = 32) holds 8 nodes; res = 16,
    count = 8 decodes exactly nodes 32..39 at x = j / 16 (R5, R19)."""
    vol = synth.g1_analytic(40).numpy()
    blocks = sampler.decompose((40, 40, 40), (16, 16, 16))
    b = blocks[-1]
    assert tuple(b.origin) == (32, 32, 32)
    kw = dict(V, out_dim=1)
    m = make_gpu_model(b, 3, **kw)
    vt = gpu_volume(vol)
    go = inr.inr_fit_opts_default()
    go.vmin, go.vmax = float(vol.min()), float(vol.max())
    inr.inr_fit(m, whole_view(vt), 10, 256, go, stream())
    p = np.empty(inr.inr_param_count(m), np.float32)
    inr.inr_get_params(m, p)
    om = InrModel(oracle_config(**kw), b, 3, params=p)
    om.vmin, om.vmax = go.vmin, go.vmax
    out = torch.full((8, 8, 8), float("nan"), device="cuda")
    inr.inr_decode_grid(m, (16, 16, 16), out.data_ptr(), (1, 8, 64), None, None, stream(), count=(8, 8, 8))
    torch.cuda.synchronize()
    z, y, x = np.meshgrid(*[np.arange(32, 40)] * 3, indexing="ij")
    pts = np.stack([x.ravel(), y.ravel(), z.ravel()], 1).astype(np.float32)
    ref = o_decode.decode_query({b.block_id: om}, pts).reshape(8, 8, 8)
    assert normwise(out.cpu().numpy(), ref) <= 1e-5
    inr.inr_destroy(m)


@pytest.mark.parametrize("flags", [inr.CACHE_FP16 | inr.CACHE_HOST_RESIDENT, inr.CACHE_HOST_RESIDENT])
def test_pathlines_from_host_and_fp16_caches(flags):
    """inr_pathlines over a pinned-host / fp16 window equals decoding every
    element (staged the same way) and tracing on the GPU, bitwise."""
    n, nb = 33, 16
    steps = [3, 4, 5]
    W = _tgv_window(n, [0.25 * s for s in steps])
    blocks = sampler.decompose((n, n, n), (nb, nb, nb))
    cache = inr.cache_create(4, flags)
    for ts, vol in zip(steps, W):
        vt = gpu_volume(vol)
        lo, hi = sampler.value_range([vol])
        go = inr.inr_fit_opts_default()
        go.set_range(lo, hi)
        ms = []
        for b in blocks:
            m = make_gpu_model(b, 7, precision=1, **V)
            inr.inr_fit(m, whole_view(vt), 20, 1024, go, stream())
            ms.append(m)
        inr.cache_insert(cache, ts, ms, stream())
        for m in ms:
            inr.inr_destroy(m)
    seeds = _seeds(n, 64, np.random.default_rng(9))
    M, K = seeds.shape[0], 100
    sd = torch.from_numpy(seeds).cuda()
    vert = torch.full((M, K + 1, 5), float("nan"), dtype=torch.float64, device="cuda")
    cnt = torch.zeros(M, dtype=torch.int32, device="cuda")
    why = torch.zeros(M, dtype=torch.int32, device="cuda")
    inr.inr_pathlines(cache, inr.INR_WINDOW_REVERSE | inr.INR_WINDOW_NEGATE, sd.data_ptr(), M, 0.05, K,
                      vert.data_ptr(), cnt.data_ptr(), why.data_ptr(), stream())
    torch.cuda.synchronize()
    gpu = (vert.cpu().numpy(), cnt.cpu().numpy(), why.cpu().numpy())
    dec = []
    for i in range(len(steps)):
        _, ms = inr.cache_get(cache, i)
        g = torch.empty((n, n, n, 3), device="cuda")
        for m, b in zip(ms, blocks):
            o = b.origin
            c = tuple(min(nb, n - o[d]) for d in range(3))
            inr.inr_decode_grid(m, (nb, nb, nb), g[o[2]:, o[1]:, o[0]:].data_ptr(), (3, 3 * n, 3 * n * n), None,
                                None, stream(), count=c)
        torch.cuda.synchronize()
        dec.append(g.cpu().numpy())
    rg, rt, sgn = o_pl.reverse_negate(dec, [float(s) for s in steps], reverse=True, negate=True)
    _assert_same(gpu, _gpu_trace(rg, rt, (n, n, n), sgn, seeds, 0.05, K))
    inr.cache_destroy(cache)


def test_pathlines_over_cached_window():
    """Backward tracing P = pathline(negate(reverse(W))) over four
    cached timesteps of fitted D = 3 block models (27 blocks, ragged)."""
    n, nb = 33, 16
    steps = [10, 11, 12, 13]
    W = _tgv_window(n, [0.25 * s for s in steps])
    blocks = sampler.decompose((n, n, n), (nb, nb, nb))
    cfg = oracle_config(**V)
    cache = inr.cache_create(8)
    oracle_grids = []
    for ts, vol in zip(steps, W):
        vt = gpu_volume(vol)
        lo, hi = sampler.value_range([vol])
        go = inr.inr_fit_opts_default()
        go.set_range(lo, hi)
        ms, grid = [], np.zeros((n, n, n, 3))
        for b in blocks:
            m = make_gpu_model(b, 7, **V)
            inr.inr_fit(m, whole_view(vt), 30, 1024, go, stream())
            ms.append(m)
            p = np.empty(inr.inr_param_count(m), np.float32)
            inr.inr_get_params(m, p)
            om = InrModel(cfg, b, 7, params=p)
            om.vmin, om.vmax = lo, hi
            o = b.origin
            c = [min(nb, n - o[d]) for d in range(3)]
            g = o_decode.decode_grid(om, (nb, nb, nb))
            grid[o[2]:o[2] + c[2], o[1]:o[1] + c[1], o[0]:o[0] + c[0]] = g[:c[2], :c[1], :c[0]]
        inr.cache_insert(cache, ts, ms, stream())
        for m in ms:
            inr.inr_destroy(m)
        oracle_grids.append(grid)
    seeds = _seeds(n, 128, np.random.default_rng(4))
    M, K = seeds.shape[0], 400
    sd = torch.from_numpy(seeds).cuda()
    vert = torch.full((M, K + 1, 5), float("nan"), dtype=torch.float64, device="cuda")
    cnt = torch.zeros(M, dtype=torch.int32, device="cuda")
    why = torch.zeros(M, dtype=torch.int32, device="cuda")
    ops = inr.INR_WINDOW_REVERSE | inr.INR_WINDOW_NEGATE
    inr.inr_pathlines(cache, ops, sd.data_ptr(), M, 0.05, K, vert.data_ptr(), cnt.data_ptr(), why.data_ptr(),
                      stream())
    torch.cuda.synchronize()
    gpu = (vert.cpu().numpy(), cnt.cpu().numpy(), why.cpu().numpy())
    # (a) == GPU decode of every element, then inr_trace_grids over negate(reverse(.))
    dec = []
    for i in range(len(steps)):
        ts, ms = inr.cache_get(cache, i)
        g = torch.empty((n, n, n, 3), device="cuda")
        for m, b in zip(ms, blocks):
            o = b.origin
            c = tuple(min(nb, n - o[d]) for d in range(3))
            inr.inr_decode_grid(m, (nb, nb, nb), g[o[2]:, o[1]:, o[0]:].data_ptr(), (3, 3 * n, 3 * n * n), None,
                                None, stream(), count=c)
        torch.cuda.synchronize()
        dec.append(g.cpu().numpy())
    rg, rt, sgn = o_pl.reverse_negate(dec, [float(s) for s in steps], reverse=True, negate=True)
    _assert_same(gpu, _gpu_trace(rg, rt, (n, n, n), sgn, seeds, 0.05, K))
    # (b) the oracle over its own fp64 decode of the same parameters
    og, ot, osg = o_pl.reverse_negate(oracle_grids, [float(s) for s in steps], reverse=True, negate=True)
    ora = o_pl.trace(og, ot, seeds, 0.05, K, osg)
    ok = (gpu[2] == ora[2]) & (gpu[1] == ora[1])
    print("window trace: same counts/reasons for", ok.mean(), "of the seeds")
    assert ok.mean() >= 0.95
    for s in np.flatnonzero(ok & (gpu[1] > 0)):
        dev = np.max(np.abs(gpu[0][s, :gpu[1][s], :3] - ora[0][s, :ora[1][s], :3]))
        assert dev <= 1e-3, (s, dev)
    inr.cache_destroy(cache)
