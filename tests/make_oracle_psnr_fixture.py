"""Writes tests/golden/oracle_cfg1_psnr.txt: the ORACLE's cfg1 PSNR after 200
seeded fit steps for seeds [1000, 1384) (calls only oracle/ and synth/; no
CUDA-path value is involved).  Used by tests/test_gpu_psnr.py (R26).

    python tests/make_oracle_psnr_fixture.py [procs]      (~30 s per seed per core)
"""
import multiprocessing as mp
import os
import sys

os.environ.setdefault("OMP_NUM_THREADS", "1")
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

SEEDS = range(1000, 1384)
OUT = os.path.join(ROOT, "tests", "golden", "oracle_cfg1_psnr.txt")


def main():
    from oracle_runs import cfg1_psnr
    procs = int(sys.argv[1]) if len(sys.argv) > 1 else os.cpu_count()
    with mp.get_context("spawn").Pool(procs) as pool:
        ps = pool.map(cfg1_psnr, list(SEEDS))
    with open(OUT, "w") as f:
        f.write("# Oracle (numpy fp64) PSNR in dB of cfg1 after 200 fit steps (G1 64^3, one block, L8 T2^14 F2,\n"
                "# 2x64 MLP, 4096 samples/step, paper Adam + schedule), decode 64^3 vs data, normalized units.\n"
                "# Written by tests/make_oracle_psnr_fixture.py.  Columns: seed psnr_db\n")
        for s, p in zip(SEEDS, ps):
            f.write(f"{s} {p:.6f}\n")


if __name__ == "__main__":
    main()
