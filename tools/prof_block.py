"""Profiling driver: one c2-shaped block prefill (8 x 2048 tokens) repeated a
few times, for ncu captures of the top kernels (B200_PROFILING.md)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2406_02528_b200 import _lib as L  # noqa: E402
from paper_2406_02528_b200 import model, synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--B", type=int, default=None)
ap.add_argument("--T", type=int, default=None)
ap.add_argument("--decode", action="store_true")
args = ap.parse_args()
L.load()
cfg = synth.CONFIGS[args.config]
st = model.Stack.random(cfg, device="cuda", gen_device="cuda", n_blocks=1)
B = args.B or cfg.prefill_B
T = args.T or cfg.prefill_T
if args.decode:
    T = 1
    B = args.B or cfg.decode_B
x = synth.hidden((B, T, cfg.d), synth.generator(1, "cuda"), cfg.dtype, device="cuda")
states = st.new_state(B)
for _ in range(args.reps):
    if args.decode:
        st.decode(x[:, 0].contiguous(), states)
    else:
        st.prefill(x, states)
torch.cuda.synchronize()
print("ok")
