"""Eager prefill vs the same prefill captured in a CUDA graph (host launch overhead test).
python tools/prefill_graph_test.py [--config c2]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2406_02528_b200 import _lib as L  # noqa: E402
from paper_2406_02528_b200 import model, synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--blocks", type=int, default=None)
args = ap.parse_args()
L.load()
cfg = synth.CONFIGS[args.config]
st = model.Stack.random(cfg, device="cuda", gen_device="cuda", n_blocks=args.blocks)
B, T = cfg.prefill_B, cfg.prefill_T
x = synth.hidden((B, T, cfg.d), synth.generator(1, "cuda"), cfg.dtype, device="cuda")
y = torch.empty_like(x)
bufs = (torch.empty_like(x), torch.empty_like(x))
h = st.new_state(B)
for _ in range(3):
    st.prefill(x, h, out=y, bufs=bufs)
torch.cuda.synchronize()


def timeit(fn, n=5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


eager = timeit(lambda: st.prefill(x, h, out=y, bufs=bufs))
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
g = torch.cuda.CUDAGraph()
with torch.cuda.stream(s):
    st.prefill(x, h, out=y, bufs=bufs)
torch.cuda.current_stream().wait_stream(s)
with torch.cuda.graph(g):
    st.prefill(x, h, out=y, bufs=bufs)
graph = timeit(lambda: g.replay())
n = len(st.blocks)
print(f"{args.config} {n} blocks: eager {eager:.3f} ms ({eager * 1e3 / n:.1f} us/block), "
      f"graph {graph:.3f} ms ({graph * 1e3 / n:.1f} us/block)")
