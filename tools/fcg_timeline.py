"""Parse a TERN_FS_TL dump (k_fcgscan CTA 0 phase clocks, debug) and print, per M-tile,
the MMA window, each quad's gate phases (A start/end, carry-wait end, C end, min over the
quad's 4 warps / max) and the carry's per-quad windows, in cycles from the first mark.
python tools/fcg_timeline.py FILE [--launch -1]"""
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
L = launches[which]
nt = int(L["hdr"].split("nt=")[1])
a = np.array(L["rows"], dtype=np.int64).reshape(20, nt, 8)
t0 = a[a > 0].min()
r = np.where(a > 0, a - t0, -1)
print(L["hdr"])
print("tile | mma start end | quad q: A0 A1 (tfull wait end, A end) Cw C1 (carry wait end, C end) | carry h0 q0..q3 start/end")
for i in range(nt):
    s = f"{i:3d} | {r[1, i, 0]:7d} {r[1, i, 1]:7d} |"
    for q in range(4):
        ws = [2 + q + 4 * c for c in range(4)]   # gate warps of quad q (warp & 3 == q)
        ws = [w for w in range(2, 18) if (w & 3) == q]
        g = r[ws, i]
        s += f" q{q}: {g[:, 1].max():7d} {g[:, 2].max():7d} {g[:, 3].max():7d} {g[:, 4].max():7d} |"
    c = r[18, i]
    s += " " + " ".join(f"{c[2 * q]}-{c[2 * q + 1]}" for q in range(4))
    print(s)
per = np.diff(r[1, :, 0])
print("mean tile period (MMA start to start):", per.mean() if len(per) else 0)
