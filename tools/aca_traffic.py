"""profiles/rNN_aca_traffic.json from an `ncu --set full` capture of the four ACA class
launches of one config-3 build (tools/host_profile.py 64):

    python tools/aca_traffic.py gpurun_out/aca_r02.ncu-rep "source note" > profiles/r02_aca_traffic.json
"""
import csv, io, json, subprocess, sys

rep = sys.argv[1]
note = sys.argv[2] if len(sys.argv) > 2 else ""
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, u, data = rows[0], rows[1], rows[2:]
ix = {k: i for i, k in enumerate(h)}
SC = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3,
      "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3, "sector": 1, "": 1}


def val(r, k):
    i = ix[k]
    return float(r[i].replace(",", "")) * SC.get(u[i], 1)


per = []
for r in data:
    per.append({
        "kernel": r[ix["Kernel Name"]][:40],
        "time_ms": val(r, "gpu__time_duration.sum"),
        "dram_read": val(r, "dram__bytes_read.sum"),
        "dram_write": val(r, "dram__bytes_write.sum"),
        "l2_read_from_l1": val(r, "lts__t_sectors_srcunit_tex_op_read.sum") * 32,
        "l2_write_from_l1": val(r, "lts__t_sectors_srcunit_tex_op_write.sum") * 32,
        "local_store_instructions": val(r, "sass__inst_executed_local_stores"),
        "issue_slots_busy_pct": val(r, "sm__inst_issued.avg.pct_of_peak_sustained_active") if "sm__inst_issued.avg.pct_of_peak_sustained_active" in ix else None,
    })
print(json.dumps({
    "per_class": per,
    "source": note,
    "dram_bytes_per_build": sum(p["dram_read"] + p["dram_write"] for p in per),
    "l2_bytes_per_build": sum(p["l2_read_from_l1"] + p["l2_write_from_l1"] for p in per),
    "serialised_time_ms": sum(p["time_ms"] for p in per),
}, indent=1))
