"""Device time of bitlinear_bwd (Alg. 1 BackwardPass, f4(iii)) at c2-sized BitLinears,
tensor-core path vs the fp32 CUDA-core path (CUDA events, L2 flushed between calls).
python tools/bwd_bench.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2406_02528_b200 import _lib as L  # noqa: E402
from paper_2406_02528_b200 import model, synth  # noqa: E402

L.load()
out = {}
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for (m, k, n) in [(16384, 1024, 1024), (16384, 2816, 1024), (16384, 1024, 2816)]:
    g = synth.generator(1)
    W = synth.latent_matrix(n, k, g).cuda()
    pw = model.PackedWeight([W])
    x = torch.randn(m, k, device="cuda")
    dO = torch.randn(m, n, device="cuda")
    dX = torch.empty_like(x)
    dW = torch.empty(n, k, device="cuda")
    db = torch.empty(n, device="cuda")
    ws = torch.empty(int(L.load().bitlinear_bwd_workspace(m, k, n)), dtype=torch.uint8,
                     device="cuda")
    for tc in (True, False):
        L.tern_set_bwd_tc(tc)
        for _ in range(2):
            L.bitlinear_bwd(x, pw.struct, dO, dX, dW, db, ws=ws)
        ts = []
        for _ in range(5):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            L.bitlinear_bwd(x, pw.struct, dO, dX, dW, db, ws=ws)
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        ms = sorted(ts)[len(ts) // 2]
        flops = 4.0 * m * n * k   # dY and dW, 2 m n k each (the dense products the method computes)
        out[f"m{m}_k{k}_n{n}_{'tc' if tc else 'cuda_core'}"] = {
            "ms": round(ms, 4), "TFLOP/s (fp32-equivalent, dY+dW)": round(flops / ms / 1e9, 1)}
L.tern_set_bwd_tc(True)
print(json.dumps(out, indent=1))
