"""Direct-query volume rendering (NEXT-3) through the C ABI vs oracle/render.py
(R32-R35): fragments of a brick, macro-cell skipping,
sort-last compositing."""
import numpy as np
import pytest
import torch

import synth
from oracle import decode as o_decode, render as o_r, sampler
from oracle.model import InrModel
from paper_2304_10516_b200 import inr

from gpu_util import gpu_volume, make_gpu_model, oracle_config, stream, whole_view

pytestmark = pytest.mark.gpu

NET = dict(levels=8, features=2, log2_table_size=14, mlp_hidden_layers=2)
N, NB = 40, 16
CAM = dict(eye=(-25.0, 52.0, -38.0), look=(20.0, 19.0, 21.0), up=(0.0, 1.0, 0.0), fovy=38.0, width=48, height=36)
TF = dict(points=[0.0, 0.35, 0.6, 1.0], rgba=[[0.0, 0.0, 1.0, 0.0], [0.0, 0.0, 1.0, 0.0], [0.2, 1.0, 0.3, 0.08],
                                             [1.0, 0.2, 0.0, 0.5]], base_step=1.0)


@pytest.fixture(scope="module", params=[0, 1], ids=["fp32", "fp16"])
def scene(request):
    prec = request.param
    vol = synth.g1_analytic(N).numpy()
    blocks = sampler.decompose((N, N, N), (NB, NB, NB))          # 27 blocks, ragged upper layer
    lo, hi = float(vol.min()), float(vol.max())
    vt = gpu_volume(vol)
    go = inr.inr_fit_opts_default()
    go.vmin, go.vmax = lo, hi
    cfg = oracle_config(**NET)
    gms, oms = [], {}
    for b in blocks:
        m = make_gpu_model(b, 5, precision=prec, **NET)
        inr.inr_fit(m, whole_view(vt), 40, 1024, go, stream())
        p = np.empty(inr.inr_param_count(m), np.float32)
        inr.inr_get_params(m, p)
        om = InrModel(cfg, b, 5, params=p)
        om.vmin, om.vmax = lo, hi
        gms.append(m)
        oms[b.block_id] = om
    tf = dict(TF, vmin=lo, vmax=hi)
    yield dict(prec=prec, gms=gms, oms=oms, blocks=blocks, tf=tf, vol=vol)
    for m in gms:
        inr.inr_destroy(m)


def _gpu_frag(r, tf, lo, hi, step, stop=0.99, mc=1, cam=CAM):
    c = inr.make_camera(cam["eye"], cam["look"], cam["up"], cam["fovy"], cam["width"], cam["height"])
    t = inr.make_tf(tf["points"], tf["rgba"], tf["vmin"], tf["vmax"], tf["base_step"])
    frag = torch.full((cam["width"] * cam["height"], 5), float("nan"), device="cuda")
    inr.inr_render(r, c, t, lo, hi, step, frag.data_ptr(), stop, mc, stream())
    torch.cuda.synchronize()
    return frag.cpu().numpy().astype(np.float64)


def _oracle_frag(scene, lo, hi, step, stop=0.99, cam=CAM):
    field = lambda P: o_decode.decode_query(scene["oms"], P.astype(np.float32))
    return o_r.render_brick(None, cam, lo, hi, step, scene["tf"], stop, batch_field=field)


def _compare(g, o, tol):
    miss = np.isinf(o[:, 4])
    assert np.array_equal(np.isinf(g[:, 4]), miss)
    assert np.allclose(g[~miss, 4], o[~miss, 4], rtol=1e-6, atol=1e-5)
    err = np.max(np.abs(g[:, :4] - o[:, :4]))
    print("render fragment max err", err, "max alpha", o[:, 3].max())
    assert err <= tol


def test_render_brick_matches_oracle(scene):
    r = inr.inr_renderer_create(scene["gms"], 8, 1e-3 * (scene["tf"]["vmax"] - scene["tf"]["vmin"]))
    lo, hi = (0.0, 0.0, 0.0), (N - 1.0,) * 3
    g = _gpu_frag(r, scene["tf"], lo, hi, 0.5, mc=0)
    o = _oracle_frag(scene, lo, hi, 0.5)
    assert o[:, 3].max() > 0.3 and (o[:, 3] > 0).mean() > 0.1     # a non-trivial image
    _compare(g, o, 2.5e-6 if scene["prec"] == 0 else 2e-3)   # ~10x the measured 2.5e-7 / 1.9e-4
    ev, sk, waves = inr.inr_render_stats(r)
    assert ev > 0 and sk == 0 and waves >= 1
    inr.inr_renderer_destroy(r)


def test_macrocell_skipping_is_exact_here(scene):
    """skipping cells whose TF opacity is 0 over their padded range
    leaves the image unchanged (here: bitwise, the skipped samples have a = 0
    exactly) while evaluating fewer samples."""
    r = inr.inr_renderer_create(scene["gms"], 8, 1e-3 * (scene["tf"]["vmax"] - scene["tf"]["vmin"]))
    lo, hi = (0.0, 0.0, 0.0), (N - 1.0,) * 3
    a = _gpu_frag(r, scene["tf"], lo, hi, 0.5, mc=0)
    ev0, _, _ = inr.inr_render_stats(r)
    b = _gpu_frag(r, scene["tf"], lo, hi, 0.5, mc=1)
    ev1, sk1, _ = inr.inr_render_stats(r)
    print("samples evaluated without / with macro-cells", ev0, ev1, "skipped", sk1)
    assert sk1 > 0 and ev1 < ev0 and ev1 + sk1 >= ev0 * 0.9
    assert np.array_equal(a[:, 4], b[:, 4]) and np.max(np.abs(a[:, :4] - b[:, :4])) <= 1e-6
    inr.inr_renderer_destroy(r)


def test_sort_last_two_bricks_equal_one(scene):
    """Two 'ranks' (the blocks with z-origin < 16 and the rest) render their
    bricks; depth-sorted compositing equals the single-brick image (no early
    termination, so the split changes nothing but rounding), in either
    fragment order."""
    blocks, gms = scene["blocks"], scene["gms"]
    front = [m for m, b in zip(gms, blocks) if b.origin[2] < 16]
    back = [m for m, b in zip(gms, blocks) if b.origin[2] >= 16]
    rf = inr.inr_renderer_create(front, 8)
    rb = inr.inr_renderer_create(back, 8)
    ra = inr.inr_renderer_create(gms, 8)
    tf = scene["tf"]
    fa = _gpu_frag(ra, tf, (0.0, 0.0, 0.0), (N - 1.0,) * 3, 0.5, stop=2.0)
    ff = _gpu_frag(rf, tf, (0.0, 0.0, 0.0), (N - 1.0, N - 1.0, 16.0), 0.5, stop=2.0)
    fb = _gpu_frag(rb, tf, (0.0, 0.0, 16.0), (N - 1.0,) * 3, 0.5, stop=2.0)
    npix = fa.shape[0]
    imgs = []
    for order in ([fa], [ff, fb], [fb, ff]):
        fr = torch.from_numpy(np.stack(order).astype(np.float32)).cuda().contiguous()
        img = torch.empty((npix, 4), device="cuda")
        inr.inr_composite(fr.data_ptr(), len(order), npix, (0.1, 0.1, 0.1), img.data_ptr(), stream())
        torch.cuda.synchronize()
        imgs.append(img.cpu().numpy())
    assert np.array_equal(imgs[1], imgs[2])
    assert np.max(np.abs(imgs[0] - imgs[1])) <= 2e-6
    ref = o_r.composite([fa], (0.1, 0.1, 0.1))
    assert np.max(np.abs(imgs[0] - ref)) <= 1e-6
    for r in (rf, rb, ra):
        inr.inr_renderer_destroy(r)


def test_render_rejects_vector_models_and_bad_tf():
    blk = sampler.decompose((16, 16, 16), (16, 16, 16))[0]
    m = make_gpu_model(blk, 1, out_dim=3, **NET)
    with pytest.raises(inr.InrError):
        inr.inr_renderer_create([m])
    inr.inr_destroy(m)
    m = make_gpu_model(blk, 1, **NET)
    r = inr.inr_renderer_create([m], 4)
    frag = torch.empty((4, 5), device="cuda")
    bad = inr.make_tf([0.5, 0.2], [[0, 0, 0, 0], [1, 1, 1, 1]], 0.0, 1.0)
    cam = inr.make_camera((8, 8, -20), (8, 8, 8), (0, 1, 0), 30, 2, 2)
    with pytest.raises(inr.InrError):
        inr.inr_render(r, cam, bad, (0, 0, 0), (15, 15, 15), 0.5, frag.data_ptr())
    inr.inr_renderer_destroy(r)
    inr.inr_destroy(m)
