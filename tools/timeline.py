"""Device timeline of one graph-replayed decode step or one eager prefill
(debug): for every kernel launch of the library, when its CTAs started, when
their dependency wait released, when the last one ended, and the gap to the
previous launch (tern_trace_enable).
python tools/timeline.py [--config c4] [--B 128] [--blocks 2] [--prefill] [--T 128]"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
# the timeline marks exist only in the trace build (build.py --trace)
os.environ.setdefault("TERN_LIB", os.path.join(ROOT, "paper_2406_02528_b200", "libtern_trace.so"))
import torch  # noqa: E402

from paper_2406_02528_b200 import _lib as L  # noqa: E402
from paper_2406_02528_b200 import model, synth  # noqa: E402

NAMES = {0: "quant", 1: "gemv", 2: "gemm", 18: "splitk_epi", 34: "gemm_sab", 3: "scan", 4: "fcgscan",
         5: "stack", 6: "fin"}
ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c4")
ap.add_argument("--B", type=int, default=None)
ap.add_argument("--T", type=int, default=None)
ap.add_argument("--blocks", type=int, default=2)
ap.add_argument("--prefill", action="store_true")
ap.add_argument("--fin", action="store_true", help="batched decode with the row-wise finalize")
args = ap.parse_args()
L.load()
L.tern_set_batched_fin(args.fin)
cfg = synth.CONFIGS[args.config]
st = model.Stack.random(cfg, device="cuda", gen_device="cuda", n_blocks=args.blocks)
if args.prefill:
    B, T = args.B or cfg.prefill_B, args.T or cfg.prefill_T
else:
    B, T = args.B or cfg.decode_B, 1
x = synth.hidden((B, T, cfg.d), synth.generator(5, "cuda"), cfg.dtype, device="cuda")
states = st.new_state(B)
if args.prefill:
    for _ in range(2):
        st.prefill(x, states)
    torch.cuda.synchronize()
    L.tern_trace_enable(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    st.prefill(x, states)
    e1.record()
    torch.cuda.synchronize()
    total = e0.elapsed_time(e1) * 1e3
else:
    L.tern_trace_enable(True)
    g, xin, yout = st.capture_decode(B, states)
    xin.copy_(x[:, 0])
    for _ in range(5):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    total = e0.elapsed_time(e1) / 20 * 1e3
recs = L.tern_trace_collect(with_kind=True)
L.tern_trace_enable(False)
# the last step's launches: decode = the captured slots (all), prefill = all
mode = "prefill" if args.prefill else "decode (graph)"
print(f"{args.config} {mode} B={B} T={T} blocks={args.blocks}: {total:.1f} us per step, "
      f"{len(recs)} launches")
t0 = min(int(r[:, 0].min()) for _, _, r in recs)
prev = None
print(f"{'#':>3} {'kernel':>11} {'ctas':>5} {'start':>8} {'rel_min':>8} {'rel_max':>8} {'end':>8} "
      f"{'exec':>7} {'gap':>6}")
tot_exec = tot_gap = 0
for i, (k, u, r) in enumerate(recs):
    s0 = int(r[:, 0].min()) - t0
    w0, w1 = int(r[:, 1].min()) - t0, int(r[:, 1].max()) - t0
    e = int(r[:, 2].max()) - t0
    gap = w0 - prev if prev is not None else 0
    print(f"{i:3d} {NAMES.get(k, str(k)):>11} {u:5d} {s0:8d} {w0:8d} {w1:8d} {e:8d} {e - w0:7d} "
          f"{gap:6d}")
    tot_exec += e - w0
    tot_gap += gap
    prev = e
print(f"sum exec {tot_exec} ns, sum gaps {tot_gap} ns")
