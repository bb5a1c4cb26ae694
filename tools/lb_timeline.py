"""Summarise a TERN_LB_TL dump (k_scan_lb per-CTA globaltimer marks, debug): per slice j,
median times (us from the launch's first mark) of: start, pass A done (gates + carry, which
runs tile by tile behind the gates), hop done, pass B carry done, CTA end.
python tools/lb_timeline.py FILE [--launch -1]"""
import sys

import numpy as np

path = sys.argv[1]
which = int(sys.argv[sys.argv.index("--launch") + 1]) if "--launch" in sys.argv else -1
launches, cur = [], None
for line in open(path):
    if line.startswith("launch"):
        cur = {"hdr": line.strip(), "rows": []}
        launches.append(cur)
    else:
        cur["rows"].append([int(v) for v in line.split()])
Lh = launches[which]
hdr = dict(kv.split("=") for kv in Lh["hdr"].split()[1:])
nch = int(hdr["nch"])
a = np.array(Lh["rows"], dtype=np.float64)
t0 = a[:, 0].min()
a = (a - t0) / 1e3
print(Lh["hdr"])
print("slice | start  passA-done  hop-done  passB-done  end   (median us over CTAs)")
for j in range(nch):
    s = a[j::nch]   # blockIdx = (sequence, channel group) * nch + slice
    print(f"{j:5d} | {np.median(s[:, 0]):6.2f} {np.median(s[:, 1]):10.2f} {np.median(s[:, 2]):9.2f} "
          f"{np.median(s[:, 3]):11.2f} {np.median(s[:, 5]):6.2f}")
if a.shape[1] > 6:
    print("CTA entry (first / median / last, us rel. to first post-sync mark):",
          round(a[:, 6].min(), 2), round(float(np.median(a[:, 6])), 2), round(a[:, 6].max(), 2))
print("kernel span (first mark to last end):", round(a[:, 5].max(), 2), "us")
