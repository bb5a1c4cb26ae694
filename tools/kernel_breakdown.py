"""Per-launch device times (library events on the launching stream) of a few
decode or prefill steps, grouped by kernel / epilogue / shape (debug).
python tools/kernel_breakdown.py [--config c4] [--B 128] [--blocks 2] [--prefill] [--T 128]"""
import argparse
import collections
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2406_02528_b200 import _lib as L  # noqa: E402
from paper_2406_02528_b200 import model, synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c4")
ap.add_argument("--B", type=int, default=None)
ap.add_argument("--T", type=int, default=None)
ap.add_argument("--blocks", type=int, default=2)
ap.add_argument("--steps", type=int, default=5)
ap.add_argument("--prefill", action="store_true")
ap.add_argument("--unfused", action="store_true", help="GEMM + scan instead of the fused f|c|g+scan")
args = ap.parse_args()
L.load()
if args.unfused:
    L.tern_set_fused_scan(False)
cfg = synth.CONFIGS[args.config]
st = model.Stack.random(cfg, device="cuda", gen_device="cuda", n_blocks=args.blocks)
B = args.B or (cfg.prefill_B if args.prefill else cfg.decode_B)
T = (args.T or cfg.prefill_T) if args.prefill else 1
x = synth.hidden((B, T, cfg.d), synth.generator(3, "cuda"), cfg.dtype, device="cuda")
h = st.new_state(B)


def step():
    if args.prefill:
        st.prefill(x, h)
    else:
        st.decode(x[:, 0].contiguous(), h)


for _ in range(3):
    step()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(args.steps):
    step()
e1.record()
torch.cuda.synchronize()
print(f"{args.config} {'prefill' if args.prefill else 'decode'} B={B} T={T}: "
      f"{e0.elapsed_time(e1) / args.steps / args.blocks * 1e3:.1f} us per block (no profiling)")
L.tern_profile_enable(True)
for _ in range(args.steps):
    step()
torch.cuda.synchronize()
L.tern_profile_enable(False)
recs = L.tern_profile_collect()
epi = {0: "store", 1: "resid", 2: "fcg", 3: "mlgru", 4: "swiglu", 5: "acc", 6: "resid_red"}
agg = collections.OrderedDict()
for r in recs:
    key = f'{r["kernel"]}:{epi.get(r["epi"], r["epi"]) if r["kernel"] != "quant" else ""}:n{r["n"]}k{r["k"]}'
    a = agg.setdefault(key, [0, 0.0])
    a[0] += 1
    a[1] += r["ms"]
tot = sum(v[1] for v in agg.values())
print(f"{'launch':44s} {'us':>8s} {'share':>6s}")
for k, (n, ms) in agg.items():
    print(f"{k:44s} {ms / n * 1e3:8.2f} {ms / tot:6.3f}")
print(f"sum of launches: {tot / args.steps / args.blocks * 1e3:.1f} us per block (serialised by events)")
