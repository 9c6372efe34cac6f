"""Condense `ncu --set full` reports into a per-kernel table for profiles/.

    python tools/ncu_summary.py gpurun_out/r01_aca_full.ncu-rep [more.ncu-rep ...]

Per launch: duration, DRAM bytes and bandwidth, L2 bytes, issue-slot and
tensor-pipe utilisation, achieved occupancy, registers, and the two largest
warp-stall reasons (per issued instruction).
"""

import csv
import subprocess
import sys

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "usecond": 1e-6, "msecond": 1e-3,
         "nsecond": 1e-9, "second": 1.0, "ns": 1e-9, "us": 1e-6, "ms": 1e-3}


def rows(report):
    out = subprocess.run(["ncu", "-i", report, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    data = list(csv.reader(out.splitlines()))
    return data[0], data[1], data[2:]


def val(h, u, r, name):
    if name not in h:
        return None
    i = h.index(name)
    try:
        v = float(r[i].replace(",", ""))
    except ValueError:
        return None
    return v * SCALE.get(u[i], 1.0)


def main():
    print(f"{'kernel':44s} {'ms':>8s} {'DRAM MB':>9s} {'DRAM GB/s':>9s} {'L2 GB':>7s} "
          f"{'issue%':>6s} {'tensor%':>7s} {'occ%':>5s} {'regs':>4s}  top stalls")
    for rep in sys.argv[1:]:
        h, u, data = rows(rep)
        stalls = [k for k in h if k.startswith("smsp__average_warps_issue_stalled_")
                  and k.endswith("_per_issue_active.ratio")]
        for r in data:
            name = r[h.index("Kernel Name")].replace("(anonymous namespace)::", "")
            name = name.replace("<unnamed>::", "").split("(")[0][:44]
            t = val(h, u, r, "gpu__time_duration.sum") or 0.0
            rd = val(h, u, r, "dram__bytes_read.sum") or 0.0
            wr = val(h, u, r, "dram__bytes_write.sum") or 0.0
            l2 = (val(h, u, r, "lts__t_sectors.sum") or 0.0) * 32
            issue = val(h, u, r, "smsp__issue_active.avg.pct_of_peak_sustained_active") or 0.0
            tens = val(h, u, r, "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed")
            occ = val(h, u, r, "sm__warps_active.avg.pct_of_peak_sustained_active") or 0.0
            regs = val(h, u, r, "launch__registers_per_thread") or 0
            top = sorted(((val(h, u, r, k) or 0.0, k) for k in stalls), reverse=True)[:2]
            top_s = ", ".join(f"{k.split('stalled_')[1].split('_per_issue')[0]} {v:.2f}" for v, k in top)
            print(f"{name:44s} {t * 1e3:8.3f} {(rd + wr) / 1e6:9.1f} {(rd + wr) / max(t, 1e-12) / 1e9:9.1f} "
                  f"{l2 / 1e9:7.2f} {issue:6.1f} {tens if tens is not None else 0.0:7.1f} {occ:5.1f} "
                  f"{int(regs):4d}  {top_s}")


if __name__ == "__main__":
    main()
