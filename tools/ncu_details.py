"""Print the details page of an ncu report as `section | metric | value unit`
lines (one kernel), optionally filtered by a regex.

    python tools/ncu_details.py gpurun_out/x.ncu-rep [regex]
"""
import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]
pat = re.compile(sys.argv[2]) if len(sys.argv) > 2 else None
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[0]
ix = {h: i for i, h in enumerate(hdr)}
for r in rows[1:]:
    line = f"{r[ix['ID']]} {r[ix['Section Name']][:28]:28s} | {r[ix['Metric Name']][:44]:44s} | " \
           f"{r[ix['Metric Value']]} {r[ix['Metric Unit']]}"
    if pat is None or pat.search(line):
        print(line)
