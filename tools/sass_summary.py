"""Counts of the Blackwell-native SASS instructions (tcgen05 MMA / TMEM loads /
TMA bulk copies / tcgen05 barriers) per kernel of libinr.so, from cuobjdump.

  python tools/sass_summary.py [paper_2304_10516_b200/lib/libinr.so] > profiles/r2_sass_summary.txt
"""
import collections, re, subprocess, sys

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_2304_10516_b200/lib/libinr.so"
sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
OPS = ("UTCHMMA", "UTCQMMA", "UTCBAR", "LDTM", "STTM", "UBLKCP", "UTMALDG", "UTMASTG", "HMMA", "REDG", "ATOMG",
       "CCTL")
per = collections.OrderedDict()
cur = None
for ln in sass.splitlines():
    m = re.search(r"Function : (\S+)", ln)
    if m:
        cur = m.group(1)
        per[cur] = collections.Counter()
        continue
    if cur is None:
        continue
    for op in OPS:
        if re.search(r"\b" + op + r"\b", ln):
            per[cur][op] += 1
arch = re.findall(r"arch = (sm_\w+)", subprocess.run(["cuobjdump", "-lelf", lib], capture_output=True, text=True).stdout)
print(f"# cuobjdump -sass {lib}: Blackwell-native instruction counts per kernel (static, in the SASS)")
print("# UTCHMMA = tcgen05.mma (fp16 kind), LDTM = tcgen05.ld, UTCBAR = tcgen05.commit, UBLKCP = cp.async.bulk (TMA),")
print("# HMMA = legacy mma.sync (none expected), REDG/ATOMG = global reductions / atomics")
tot = collections.Counter()
for k, c in per.items():
    if not c:
        continue
    tot.update(c)
    name = subprocess.run(["c++filt", k], capture_output=True, text=True).stdout.strip()
    print(f"{name[:110]:110s} " + " ".join(f"{op}={c[op]}" for op in OPS if c[op]))
print("TOTAL " + " ".join(f"{op}={tot[op]}" for op in OPS if tot[op]))
