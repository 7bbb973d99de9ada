"""Measure random-access gather / red throughput peaks on the GPU (the
denominators of the encode kernels' rooflines) -> profiles/r1_l2_peaks.json.

    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC tools/l2_peaks.cu -o tools/libl2peaks.so
    python tools/l2_peaks.py
"""
import ctypes
import json
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "libl2peaks.so")


def build():
    subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared", "-Xcompiler", "-fPIC",
                    os.path.join(HERE, "l2_peaks.cu"), "-o", LIB], check=True)


def measure():
    lib = ctypes.CDLL(LIB)
    lib.l2_peak.restype = ctypes.c_double
    lib.l2_peak.argtypes = [ctypes.c_int, ctypes.c_longlong, ctypes.c_longlong]
    res = []
    names = {0: "gather_8B", 1: "gather_16B", 2: "red_v2_f32", 3: "red_v4_f32"}
    for kind in range(4):
        for mb in (4, 32, 64, 1024):
            r = lib.l2_peak(kind, mb << 20, 1 << 30)
            res.append({"op": names[kind], "buffer_MB": mb, "per_s": r})
            print(names[kind], mb, "MB", f"{r / 1e9:.1f} G/s", flush=True)
    return res


if __name__ == "__main__":
    if not os.path.exists(LIB):
        build()
    out = {"method": "random uniform index per access (hash), 8 independent accesses per thread, 148x8 CTAs x 256",
           "results": measure()}
    with open(os.path.join(os.path.dirname(HERE), "profiles", "r1_l2_peaks.json"), "w") as f:
        json.dump(out, f, indent=1)
