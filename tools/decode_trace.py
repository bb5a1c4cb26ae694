"""Device timeline of one graph-replayed decode step (debug): per GEMV launch,
when its CTAs start relative to the previous launch's end, when
griddepcontrol.wait releases them, and how long the post-wait part takes.
python tools/decode_trace.py [--config c2] [--blocks 4]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2406_02528_b200 import _lib as L  # noqa: E402
from paper_2406_02528_b200 import model, synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--blocks", type=int, default=4)
ap.add_argument("--lean-marks", action="store_true",
                help="label the marks of the batch-1 kernel k_gemv1 (x, norm, q, dot0, sums0, dots)")
ap.add_argument("--per-block", action="store_true",
                help="trace the per-block launch chain instead of the persistent kernel")
args = ap.parse_args()
L.load()
cfg = synth.CONFIGS[args.config]
st = model.Stack.random(cfg, device="cuda", gen_device="cuda", n_blocks=args.blocks)
st.persistent_decode = not args.per_block
states = st.new_state(cfg.decode_B)
L.tern_trace_enable(True)
g, xin, yout = st.capture_decode(cfg.decode_B, states)
xin.copy_(synth.hidden((cfg.decode_B, cfg.d), synth.generator(5, "cuda"), cfg.dtype, device="cuda"))
for _ in range(5):
    g.replay()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    g.replay()
e1.record()
torch.cuda.synchronize()
print(f"path: {st.last_decode_path}")
print(f"graph replay: {e0.elapsed_time(e1) / 20 * 1e3:.1f} us per step, "
      f"{4 * args.blocks} launches -> {e0.elapsed_time(e1) / 20 * 1e3 / (4 * args.blocks):.2f} us/launch")
recs = L.tern_trace_collect()
# the captured launches are the last 4*blocks slots assigned (capture assigns slots)
recs = recs[-4 * args.blocks:]
names = ["fcg", "o", "gu", "down"]
prev_end = None
t0 = min(int(r[:, 0].min()) for _, r in recs)
print(f"{'launch':>8} {'ctas':>5} {'start_min':>9} {'start_max':>9} {'rel_min':>8} {'rel_max':>8} "
      f"{'end_max':>8} {'post_wait':>9} {'gap_after_prev':>14} | mean ns after release: "
      f"sq warpred bar r quant dot0 epi end  ('-': mark not recorded by this kernel)")
for i, (u, r) in enumerate(recs):
    u &= 0xFFFFF
    s0, s1 = int(r[:, 0].min()) - t0, int(r[:, 0].max()) - t0
    w0, w1 = int(r[:, 1].min()) - t0, int(r[:, 1].max()) - t0
    e = int(r[:, 2].max()) - t0
    gap = (w0 - prev_end) if prev_end is not None else 0
    # marks: slots 5..10 = GPROF(2..7), slot 12 = GPROF(9) (slot 11 is never written)
    ph = []
    for k in ((9, 10, 5, 6, 7, 8) if args.lean_marks else (5, 6, 7, 8, 9, 10, 12)):
        col = r[:, k]
        ph.append(int((col - r[:, 1]).mean()) if np.all(col > 0) else None)
    ph.append(int((r[:, 2] - r[:, 1]).mean()))
    ghz = float(np.median((r[:, 4] - r[:, 3]) / np.maximum(r[:, 2] - r[:, 0], 1)))
    print(f"{names[i % 4] + str(i // 4):>8} {u:5d} {s0:9d} {s1:9d} {w0:8d} {w1:8d} {e:8d} {e - w0:9d} {gap:14d} | "
          + " ".join(f"{v:5d}" if v is not None else "    -" for v in ph) + f"  clk {ghz:.2f} GHz")
    prev_end = e
