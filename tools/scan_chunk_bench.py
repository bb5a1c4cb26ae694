"""Time the prefill scan at few sequences with the sequential (num_chunks = 1) and the chunked
(num_chunks = 4, 8) scan: per-launch scan time from the library's event records, and one block's
prefill.  python tools/scan_chunk_bench.py [--config c2] [--B 1] [--T 2048]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2406_02528_b200 import _lib as L  # noqa: E402
from paper_2406_02528_b200 import model, synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--B", type=int, default=1)
ap.add_argument("--T", type=int, default=None)
args = ap.parse_args()
L.load()
cfg = synth.CONFIGS[args.config]
T = args.T or cfg.prefill_T
x = synth.hidden((args.B, T, cfg.d), synth.generator(3, "cuda"), cfg.dtype, device="cuda")
for nc in (1, 4, 8):
    st = model.Stack.random(cfg, device="cuda", gen_device="cuda", n_blocks=1, num_chunks=nc)
    hs = st.new_state(args.B)
    for _ in range(3):
        st.prefill(x, hs)
    torch.cuda.synchronize()
    L.tern_profile_enable(True)
    for _ in range(5):
        st.prefill(x, hs)
    torch.cuda.synchronize()
    L.tern_profile_enable(False)
    recs = [r for r in L.tern_profile_collect() if r["kernel"] == "scan"]
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        st.prefill(x, hs)
    e1.record()
    torch.cuda.synchronize()
    scan_us = 1e3 * sum(r["ms"] for r in recs) / max(len(recs), 1)
    byts = args.B * T * cfg.d * 4 * (2 if cfg.dtype == "bf16" else 4)   # 3 in + 1 out
    print(f"{args.config} B={args.B} T={T} num_chunks={nc} (resolved {st.blocks[0].scan_chunks(args.B, T)}): "
          f"scan {scan_us:.1f} us ({byts / scan_us / 1e3:.0f} GB/s), block prefill "
          f"{e0.elapsed_time(e1) * 100:.1f} us")
