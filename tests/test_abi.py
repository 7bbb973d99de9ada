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


def test_missing_library_fails_loudly(tmp_path):
    """No CPU fallback: importing the binding without libinr.so raises ImportError."""
    import subprocess
    import sys
    code = ("import sys; sys.path.insert(0, %r)\n"
            "try:\n    from paper_2304_10516_b200 import inr\nexcept ImportError as e:\n"
            "    print('IMPORT_ERROR', e); sys.exit(0)\nsys.exit(3)\n") % ROOT
    env = dict(os.environ, INR_LIB_PATH=str(tmp_path / "absent" / "libinr.so"))
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and "no CPU fallback" in r.stdout, r.stdout + r.stderr


def test_compute_without_a_device_is_a_cuda_error():
    """Without a GPU a valid create fails with INR_ERR_CUDA (nothing runs on the host)."""
    import ctypes
    import torch
    if torch.cuda.is_available():
        pytest.skip("a device is present")
    from paper_2304_10516_b200 import inr
    h = ctypes.c_void_p()
    cfg = inr.make_config(levels=4, log2_table_size=10)
    blk = inr.make_block((0, 0, 0), (8, 8, 8), (9, 9, 9))
    assert inr.lib.inr_create(ctypes.byref(cfg), ctypes.byref(blk), 0, ctypes.byref(h)) == inr.INR_ERR_CUDA


def test_product_path_never_imports_the_oracle():
    """oracle/ is test infrastructure: no module of the package or its CUDA sources
    references it except in comments."""
    import re
    pkg = os.path.join(ROOT, "paper_2304_10516_b200")
    for name in ("inr.py", "dnr.py", "__init__.py"):
        src = open(os.path.join(pkg, name)).read()
        assert not re.search(r"^\s*(from|import)\s+oracle\b|import_module\(['\"]oracle", src, re.M), name
    for d, _, files in os.walk(os.path.join(pkg, "csrc")):
        for f in files:
            for line in open(os.path.join(d, f)):
                code = line.split("//")[0]
                assert "oracle" not in code, (f, line)
