"""Per CUDA source line of one kernel of an ncu report (--set full --import-source on):
executed warp instructions and stall samples, top N lines.

    python tools/ncu_lines.py rep.ncu-rep [kernel-index] [N]
"""
import csv, io, subprocess, sys
rep = sys.argv[1]
kid = int(sys.argv[2]) if len(sys.argv) > 2 else 0
N = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
# sections start with a "File Path" row followed by "Function Name"
secs = []
for i, r in enumerate(rows):
    if r and r[0] == "Function Name":
        secs.append(i)
names = [rows[i][1] for i in secs]
uniq = []
for nm in names:
    if nm not in uniq:
        uniq.append(nm)
want = uniq[kid]
print(want[:110])
tot_i = tot_s = 0
lines = {}
for si, i in enumerate(secs):
    if rows[i][1] != want:
        continue
    end = secs[si + 1] - 1 if si + 1 < len(secs) else len(rows)
    fpath = rows[i - 1][1] if rows[i - 1][0] == "File Path" else "?"
    hdr = rows[i + 1]
    ix = {k: j for j, k in enumerate(hdr)}
    for r in rows[i + 2:end]:
        if len(r) != len(hdr) or not r[0]:
            continue
        try:
            e = float(r[ix["Instructions Executed"]]); s = float(r[ix["Warp Stall Sampling (All Samples)"]])
        except ValueError:
            continue
        key = (fpath.split("/")[-1], int(r[0]), r[1].strip()[:90])
        a = lines.setdefault(key, [0.0, 0.0])
        a[0] += e; a[1] += s
        tot_i += e; tot_s += s
print(f"total executed {tot_i:.0f}  samples {tot_s:.0f}")
for (f, ln, src), (e, s) in sorted(lines.items(), key=lambda kv: -kv[1][0])[:N]:
    print(f"{100*e/tot_i:5.1f}% inst {100*s/max(tot_s,1):5.1f}% smp  {f}:{ln:4d}  {src}")
