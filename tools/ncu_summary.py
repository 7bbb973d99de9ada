"""Summarize an ncu launch list (--metrics gpu__time_duration.sum --csv) and a
--set full report into profiles/ text files.

    python tools/ncu_summary.py launches.csv report.ncu-rep out_prefix "command line"
"""
import collections
import csv
import subprocess
import sys

WANT = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 'lts__t_sectors_srcunit_tex_op_read.sum',
        'lts__t_sectors_srcunit_tex_op_red.sum', 'lts__t_sector_hit_rate.pct',
        'lts__throughput.avg.pct_of_peak_sustained_elapsed', 'l1tex__throughput.avg.pct_of_peak_sustained_active',
        'sm__throughput.avg.pct_of_peak_sustained_elapsed', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'launch__registers_per_thread', 'sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active',
        'lts__d_atomic_input_cycles_active.avg.pct_of_peak_sustained_elapsed', 'launch__grid_size',
        'launch__block_size']
SCALE = {'ns': 1e-3, 'nsecond': 1e-3, 'us': 1.0, 'usecond': 1.0, 'ms': 1e3, 'msecond': 1e3}


def launches(path, out, cmd):
    rows = list(csv.reader(open(path)))
    hdr, agg = None, collections.OrderedDict()
    for r in rows:
        if r and r[0] == 'ID':
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d.get('Metric Name') != 'gpu__time_duration.sum':
            continue
        name = d['Kernel Name'].split('(')[0].replace('void ', '')
        v = float(d['Metric Value'].replace(',', '')) * SCALE[d['Metric Unit']]
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += v
    # (names may carry the inr:: namespace or not, depending on the ncu name base)
    ours = {k.replace('inr::', ''): v for k, v in agg.items()
            if k.startswith('inr::') or ('_kernel' in k and 'at::' not in k and 'elementwise' not in k)}
    # one launch of each per fp16 fit step; prep_image also serves the decodes, so the
    # share uses per-launch averages: avg(kernel) / sum of the step kernels' averages
    stepk = ('step_begin', 'sample_kernel', 'encode_fwd', 'prep_image', 'mlp_fit', 'encode_bwd', 'adam')   # (adam_tma too)
    step = sum(v[1] / v[0] for k, v in ours.items() if any(s in k for s in stepk))
    with open(out, 'w') as f:
        f.write("# ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised per launch)\n")
        f.write(f"# command: {cmd}\n# libinr kernels only; share = avg launch / sum of the fit-step kernels' "
                "avg launches\n")
        f.write(f"# {'kernel':45s} launches   total_us     avg_us   share_of_fit_step\n")
        for k, (n, v) in ours.items():
            share = (v / n) / step if any(s in k for s in stepk) else float('nan')
            f.write(f"{k:47s} {n:5d} {v:11.1f} {v / n:10.1f}   {share:6.3f}\n")


def full(rep, out, cmd):
    raw = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units = rows[0], rows[1]
    lines = [f"# ncu --set full --clock-control none --import-source on (per launch)", f"# command: {cmd}",
             "# traffic = dram__bytes_read.sum + dram__bytes_write.sum"]
    for r in rows[2:]:
        lines.append(f"\n[{r[hdr.index('Kernel Name')].split('(')[0]}]")
        for w in WANT:
            if w in hdr:
                i = hdr.index(w)
                lines.append(f"  {w:70s} {r[i]:>18s} {units[i]}")
        i_r, i_w = hdr.index('dram__bytes_read.sum'), hdr.index('dram__bytes_write.sum')
        lines.append(f"  {'traffic (read+write)':70s} {float(r[i_r]) + float(r[i_w]):18.4f} {units[i_r]}")
    open(out, 'w').write("\n".join(lines) + "\n")


if __name__ == '__main__':
    launches(sys.argv[1], sys.argv[3] + '_launches.txt', sys.argv[4])
    full(sys.argv[2], sys.argv[3] + '_ncu_full.txt', sys.argv[4])
