"""Summarise an ncu launch list (``--metrics gpu__time_duration.sum --csv``).

    python tools/launch_summary.py gpurun_out/launches.csv [--ours] > profiles/rNN_launches_summary.txt

Groups launches by kernel name (template arguments kept, argument lists
dropped) and prints total time, share and count, largest first.  ``--ours``
restricts the table to kernels of libhodlr_b200.so (drops torch's fills and
front-generation kernels).  ncu serialises launches and runs them cold-cache,
so absolute times exceed the bench's; the shares are what matter.
"""

import csv
import re
import sys
from collections import defaultdict

OURS = ("aca_kernel", "aca_cluster_kernel", "gj_cl_kernel", "sgemv_kernel", "pdot_kernel",
        "gemv4_kernel", "solve_sweep_kernel", "h2d_stream_kernel", "arnoldi_batch_kernel",
        "norms_kernel", "gemm_kernel", "gj_", "matvec_kernel", "dot_kernel", "transpose_kernel",
        "copy_kernel", "fill_kernel", "skeleton_kernel", "cpiv_kernel", "lu_inv_kernel",
        "arnoldi_kernel", "combine_kernel", "gemv_rm_kernel", "norm_kernel", "scale_kernel",
        "axpby_kernel", "diag_scale_kernel")


def short(name: str) -> str:
    name = re.sub(r"^void ", "", name)
    name = re.sub(r"\(anonymous namespace\)::|<unnamed>::", "", name)
    depth, out = 0, []
    for ch in name:                     # drop the argument list, keep template args
        if ch == "(" and depth == 0:
            break
        depth += ch == "<"
        depth -= ch == ">"
        out.append(ch)
    return "".join(out).strip()


def main():
    path = sys.argv[1]
    ours = "--ours" in sys.argv
    tot = defaultdict(float)
    cnt = defaultdict(int)
    with open(path) as fh:
        lines = [ln for ln in fh if ln.startswith('"')]
    rows = [r for r in csv.DictReader(lines) if r.get("Metric Name") == "gpu__time_duration.sum"]
    # --from-first NAME / --before-first NAME: split the list at the first launch whose
    # kernel name contains NAME (e.g. transpose_kernel = the first HODLR build)
    for flag in ("--from-first", "--before-first"):
        if flag in sys.argv:
            name = sys.argv[sys.argv.index(flag) + 1]
            first = next((i for i, r in enumerate(rows) if name in r["Kernel Name"]), len(rows))
            rows = rows[first:] if flag == "--from-first" else rows[:first]
    for row in rows:
        k = short(row["Kernel Name"])
        if ours and not k.startswith(OURS):
            continue
        scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(
            row["Metric Unit"], 1e-3)
        tot[k] += float(row["Metric Value"].replace(",", "")) * scale
        cnt[k] += 1
    grand = sum(tot.values())
    for k in sorted(tot, key=tot.get, reverse=True):
        print(f"{tot[k]:10.1f} us  {100 * tot[k] / grand:5.1f}%  n={cnt[k]:4d}  {k}")
    print(f"total {grand:.1f} us over {sum(cnt.values())} launches")


if __name__ == "__main__":
    main()
