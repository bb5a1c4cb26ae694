"""Per-launch time of the quant kernels in one block prefill of a config (library event records).
python tools/quant_time.py [--config c3]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2406_02528_b200 import _lib as L  # noqa: E402
from paper_2406_02528_b200 import model, synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3")
args = ap.parse_args()
L.load()
cfg = synth.CONFIGS[args.config]
st = model.Stack.random(cfg, device="cuda", gen_device="cuda", n_blocks=1)
x = synth.hidden((cfg.prefill_B, cfg.prefill_T, cfg.d), synth.generator(1, "cuda"), cfg.dtype, device="cuda")
h = st.new_state(cfg.prefill_B)
for _ in range(3):
    st.prefill(x, h)
torch.cuda.synchronize()
L.tern_profile_enable(True)
for _ in range(5):
    st.prefill(x, h)
torch.cuda.synchronize()
L.tern_profile_enable(False)
recs = [r for r in L.tern_profile_collect() if r["kernel"] == "quant"]
by = {}
for r in recs:
    by.setdefault(r["k"], []).append(r["ms"])
for k, v in sorted(by.items()):
    print(f"{args.config} quant K={k}: {1e3 * sum(v) / len(v):.1f} us per launch ({len(v)} launches)")
