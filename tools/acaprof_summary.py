"""Summarise an HK_ACA_PROFILE dump: per size class, chain durations and start/end times."""
import sys, numpy as np
for fn in sys.argv[1:]:
    d = np.loadtxt(fn)
    m, n, r, blk, t0, t1, sm = d.T
    T0 = t0.min()
    print(fn, "tasks", len(d), "span %.3f ms" % ((t1.max() - T0) * 1e-6))
    for L in sorted(set(np.maximum(m, n)), reverse=True):
        s = np.maximum(m, n) == L
        dur = (t1 - t0)[s] * 1e-3
        steps = r[s] + 1
        print("  L=%4d tasks %5d  rank %.0f  chain us mean %.0f p10 %.0f p90 %.0f  us/step %.2f  start ms p10 %.2f p50 %.2f p90 %.2f  end max %.2f  thread-ms %.0f" % (
            L, s.sum(), r[s].mean(), dur.mean(), np.percentile(dur, 10), np.percentile(dur, 90),
            (dur / steps).mean(), *(np.percentile((t0[s] - T0) * 1e-6, [10, 50, 90])), (t1[s].max() - T0) * 1e-6,
            dur.sum() * 1e-3 * min(256, L / 2)))
