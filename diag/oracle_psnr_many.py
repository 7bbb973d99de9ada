"""Diagnostic: oracle cfg1 200-step PSNR over many seeds (fp64, and with the
parameters rounded to fp32 after every step)."""
import os, sys, multiprocessing as mp
os.environ["OMP_NUM_THREADS"] = "1"; os.environ["OPENBLAS_NUM_THREADS"] = "1"
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np

def run(args):
    seed, r32 = args
    import synth
    from oracle import decode, fit, sampler
    from oracle.model import Config, InrModel
    n = 64
    vol = synth.g1_analytic(n).numpy(); lo, hi = sampler.value_range([vol])
    blk = sampler.decompose((n,) * 3, (n,) * 3)[0]
    m = InrModel(Config(levels=8, features=2, log2_table_size=14, mlp_hidden_layers=2), blk, seed)
    m.vmin, m.vmax = lo, hi
    opts = fit.FitOpts(vmin=lo, vmax=hi)
    for s in range(200):
        fit.train_step(m, vol, opts, 4096)
        if r32:
            m.p[:] = m.p.astype(np.float32); m.m[:] = m.m.astype(np.float32); m.v[:] = m.v.astype(np.float32)
    ref = (vol.astype(np.float64) - lo) / (hi - lo)
    return sampler.psnr((decode.decode_grid(m, (n,) * 3) - lo) / (hi - lo), ref)

if __name__ == "__main__":
    a, b, r32 = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
    with mp.get_context("spawn").Pool(int(sys.argv[4]) if len(sys.argv) > 4 else os.cpu_count()) as p:
        ps = np.array(p.map(run, [(s, r32) for s in range(a, b)]))
    np.save(f"diag/oracle_psnr_{a}_{b}_r{r32}.npy", ps)
    print("oracle r32", r32, "n", len(ps), "mean %.3f sd %.2f se %.2f min %.2f" % (ps.mean(), ps.std(), ps.std() / len(ps) ** .5, ps.min()))
