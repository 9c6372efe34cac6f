"""Group the SASS of one kernel of an ncu report (``--set full --import-source
on``) into runs of equal execution count (loop bodies, per-step code, ...) and
print each run's instruction count, share of stall samples and of executed
instructions -- where a latency-bound kernel spends its time.

    python tools/ncu_sass_regions.py gpurun_out/x.ncu-rep [kernel-id] [--dump N]
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
kid = sys.argv[2] if len(sys.argv) > 2 and not sys.argv[2].startswith("--") else "0"
dump = int(sys.argv[sys.argv.index("--dump") + 1]) if "--dump" in sys.argv else 0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
starts = [i for i, r in enumerate(rows) if r and r[0] == "Kernel Name"] + [len(rows)]
sec = rows[starts[int(kid)]:starts[int(kid) + 1]]
print(sec[0][1][:120])
h = sec[1]
ix = {k: i for i, k in enumerate(h)}
data = [r for r in sec[2:] if len(r) == len(h)]
S = lambda r: float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
E = lambda r: float(r[ix["Instructions Executed"]] or 0)
tot = sum(S(r) for r in data) or 1.0
totI = sum(E(r) for r in data) or 1.0
agg = defaultdict(lambda: [0, 0.0, 0.0])
for r in data:
    e = E(r)
    agg[e][0] += 1
    agg[e][1] += S(r)
    agg[e][2] += e
print(f"{len(data)} SASS instructions, {totI:.0f} executed, {tot:.0f} samples")
for e, (n, s, ei) in sorted(agg.items(), key=lambda x: -x[1][1])[:14]:
    print(f"exec {e:10.0f}  ninstr {n:5d}  samples {100 * s / tot:5.1f}%  inst {100 * ei / totI:5.1f}%")
if dump:
    for e, _ in sorted(agg.items(), key=lambda x: -x[1][1])[:dump]:
        print(f"--- exec {e:.0f}")
        for r in data:
            if E(r) == e:
                print(f"  {100 * S(r) / tot:5.2f}%  {r[ix['Source']][:100]}")
