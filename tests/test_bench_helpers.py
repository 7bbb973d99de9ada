"""bench.py's host-side helpers (CPU): the committed ncu capture parses into the
per-kernel DRAM bytes and L2 sector counts the bench line reports, the measured
peaks load, and the workload config names BASELINE.json's configs[1]."""
import json
import os

import bench

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_ncu_capture_parses_every_fit_kernel():
    cap = bench.ncu_capture()
    # the split fit step's kernels (no step_begin in the fp16 step), each captured per half of 4 blocks
    for k in ("encode_fwd", "prep_image", "mlp_tc", "encode_bwd", "adam"):
        assert k in cap and cap[k]["dram_bytes"] >= 0, k
    assert cap["encode_fwd"]["l2_read_sectors"] > 1e7 and cap["encode_bwd"]["l2_red_sectors"] > 1e7
    assert 1.0e9 < cap["adam"]["dram_bytes"] < 1.75e9          # ~28 B x 48.7 M params (one half)


def test_peaks_and_workload():
    pk, src = bench.peaks()
    assert pk["hbm_gbs"] > 1000 and pk["bf16_tflops"] > 100 and src
    cfg = bench.workload_config(1, type("A", (), {"precision": "fp16"})())
    base = json.load(open(os.path.join(ROOT, "BASELINE.json")))
    assert "256^3" in base["configs"][1] and "256^3" in cfg["workload"] and cfg["blocks_per_gpu"] == 8
    assert cfg["batch_uniform"] == 65536 and cfg["batch_boundary"] == 16384
