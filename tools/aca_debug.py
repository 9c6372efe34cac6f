"""Golden-block ACA check with a per-block report (first diverging pivot,
U/V differences): python tools/aca_debug.py"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import paper_1403_5337_b200 as hk
g = np.load(Path(__file__).resolve().parent.parent / "tests" / "golden" / "aca_blocks.npz")
bad = 0
for name in g["names"]:
    name = str(name)
    mr = int(g[f"{name}_maxrank"]) or None
    cfg = hk.CompressionConfig(scheme="aca", tol=float(g[f"{name}_tol"]), max_rank=mr)
    tr = {}
    A = g[f"{name}_A"]
    f = hk.compress_aca(hk.BlockAccessor(A), cfg, trace=tr)
    rows, cols = g[f"{name}_rows"], g[f"{name}_cols"]
    ok = (np.array_equal(tr["rows"], rows) and np.array_equal(tr["cols"], cols)
          and np.array_equal(f.u, g[f"{name}_U"]) and np.array_equal(f.v, g[f"{name}_V"]))
    if not ok:
        bad += 1
        k = min(len(rows), len(tr["rows"]))
        d = [i for i in range(k) if rows[i] != tr["rows"][i]]
        kc = min(len(cols), len(tr["cols"]))
        dc = [i for i in range(kc) if cols[i] != tr["cols"][i]]
        r0 = g[f"{name}_U"].shape[1]
        msg = f"{name}: A{A.shape} rank {f.rank} vs {r0}; rows {len(tr['rows'])} vs {len(rows)} first diff {d[:1]}; cols first diff {dc[:1]}"
        if f.rank and r0:
            rr = min(f.rank, r0)
            du = np.abs(f.u[:, :rr] - g[f"{name}_U"][:, :rr]).max(axis=0)
            msg += f"; first U col diff {int(np.argmax(du > 0)) if (du > 0).any() else -1}"
        print(msg)
print("bad", bad, "of", len(g["names"]))
