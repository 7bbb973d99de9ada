"""C-ABI contract checks that need no GPU: the library loads, exports every
symbol include/inr.h declares, its struct layouts match the ctypes binding,
and argument validation fails with the documented status before touching the
device."""
import os
import re
import subprocess
import tempfile

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "inr.h")
LIB = os.path.join(ROOT, "paper_2304_10516_b200", "lib", "libinr.so")


def declared_symbols():
    src = open(HDR).read()
    return sorted(set(re.findall(r"^INR_API [^(]*?\b((?:inr|cache)_\w+)\(", src, re.M)))


def test_header_declares_the_north_star_calls():
    names = declared_symbols()
    for n in ("inr_create", "inr_fit", "inr_decode", "inr_decode_grid", "cache_insert", "cache_evict"):
        assert n in names


def test_library_exports_every_declared_symbol():
    assert os.path.exists(LIB), "build libinr.so first (__graft_entry__.build())"
    out = subprocess.run(["nm", "-D", "--defined-only", LIB], capture_output=True, text=True, check=True).stdout
    exported = {ln.split()[-1] for ln in out.splitlines() if " T " in ln}
    missing = [n for n in declared_symbols() if n not in exported]
    assert not missing, missing


def test_struct_layouts_match_binding():
    import ctypes
    from paper_2304_10516_b200 import inr
    prog = r'''
#include <stdio.h>
#include <stddef.h>
#include "inr.h"
int main(void) {
  printf("%zu %zu %zu %zu %zu\n", sizeof(inr_config), sizeof(inr_block), sizeof(inr_fit_opts),
         sizeof(inr_fit_report), sizeof(inr_view));
  printf("%zu %zu %zu\n", offsetof(inr_config, seed), offsetof(inr_view, stride), offsetof(inr_fit_report, probe_psnr));
  return 0;
}'''
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "t.c")
        open(c, "w").write(prog)
        exe = os.path.join(d, "t")
        subprocess.run(["gcc", "-I", os.path.dirname(HDR), c, "-o", exe], check=True)
        sizes = [int(v) for v in subprocess.run([exe], capture_output=True, text=True).stdout.split()]
    assert sizes[:5] == [ctypes.sizeof(t) for t in (inr.inr_config, inr.inr_block, inr.inr_fit_opts,
                                                     inr.inr_fit_report, inr.inr_view)]
    assert sizes[5] == inr.inr_config.seed.offset
    assert sizes[6] == inr.inr_view.stride.offset
    assert sizes[7] == inr.inr_fit_report.probe_psnr.offset


def test_argument_validation_without_device():
    import ctypes
    from paper_2304_10516_b200 import inr
    L = inr.lib
    h = ctypes.c_void_p()
    assert L.inr_create(None, None, 0, ctypes.byref(h)) == inr.INR_ERR_INVALID_ARG
    assert "NULL" in inr.inr_last_error()
    blk = inr.make_block((0, 0, 0), (8, 8, 8), (8, 8, 8))
    bad = [dict(levels=0), dict(log2_table_size=0), dict(per_level_scale=1.0), dict(mlp_hidden_layers=0),
           dict(levels=32, base_resolution=4, per_level_scale=2.0)]          # N_31 = 2^33 > 2^30
    for kw in bad:
        cfg = inr.make_config(**{**dict(levels=4, log2_table_size=10), **kw})
        assert L.inr_create(ctypes.byref(cfg), ctypes.byref(blk), 0, ctypes.byref(h)) == inr.INR_ERR_INVALID_ARG
    for kw in (dict(features=3), dict(mlp_width=32), dict(out_dim=2), dict(levels=16, features=8)):
        cfg = inr.make_config(**{**dict(levels=4, log2_table_size=10), **kw})
        assert L.inr_create(ctypes.byref(cfg), ctypes.byref(blk), 0, ctypes.byref(h)) == inr.INR_ERR_UNSUPPORTED
    cfg = inr.make_config(levels=4, log2_table_size=10)
    badblk = inr.make_block((3, 0, 0), (8, 8, 8), (16, 8, 8))
    assert L.inr_create(ctypes.byref(cfg), ctypes.byref(badblk), 0, ctypes.byref(h)) == inr.INR_ERR_INVALID_ARG
    assert L.cache_create(0, 0, 0, ctypes.byref(h)) == inr.INR_ERR_INVALID_ARG
    opts = inr.inr_fit_opts_default()
    assert abs(opts.lambda_ - 0.5) < 1e-7 and abs(opts.lr0 - 1e-2) < 1e-9 and opts.lr_step == 500
    assert L.inr_fit(None, None, 1, 1, ctypes.byref(opts), None, None) == inr.INR_ERR_INVALID_ARG
    assert L.inr_destroy(None) == inr.INR_OK
    assert L.cache_destroy(None) == inr.INR_OK
    assert L.cache_evict(None, None) == inr.INR_ERR_INVALID_ARG
