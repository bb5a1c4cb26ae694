"""BASELINE.json configs[1] / SURVEY 8(d): the isolated BitLinear sweep.

bf16 activations x [M][K] -> bf16 y [M][N] through bitlinear_fwd (C ABI) for
M in {1, 16, 256, 4096, 16384} x (K, N) in {(1024,1024), (2048,5632), (5632,2048)}.
Each point cycles through enough distinct packed-weight and activation copies
that together exceed 4x the L2 (so weights and activations stream from HBM),
replays the calls from a CUDA graph and reports per call:
  * HBM roofline: algorithmic bytes (packed weights N*Kp/4 + x + y) / time
    against MEASURED_PEAKS.json hbm_gbs;
  * INT8 roofline: dense-equivalent 2*M*N*K ops / time against 2 x MEASURED_PEAKS.json
    bf16_tflops (the burst figure: each point is a short isolated run; bench.py's rule);
  * which path ran (decode GEMV for M <= 4, else quant + tcgen05 GEMM).
SURVEY's gates: GEMV >= 70 % of HBM at M = 1; GEMM >= 50 % of INT8 above the
ridge (M >= 4096 with (2048,5632) / (5632,2048)).
python tools/c1_sweep.py [--out profiles/r02_c1_sweep.json] [--reps 3]"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2406_02528_b200 import _lib as L  # noqa: E402
from paper_2406_02528_b200 import model, synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--out", default=None)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--ms", default="1,16,256,4096,16384")
args = ap.parse_args()
L.load()
dev = torch.device("cuda")
peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
mp = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
hbm = float(peaks["hbm_gbs"])
int8 = 2.0 * float(mp["bf16_tflops"])
l2 = torch.cuda.get_device_properties(0).L2_cache_size
cfg = synth.CONFIGS["c1"]
shapes, Ms = cfg.sweep
Ms = [int(m) for m in args.ms.split(",")]
g = synth.generator(cfg.seed, "cuda")
rows = []
for K, N in shapes:
    kp = (K + 127) // 128 * 128
    wbytes = N * kp // 4
    for M in Ms:
        xb, yb = M * K * 2, M * N * 2
        per = wbytes + xb + yb
        ncopy = max(2, min(256, -(-4 * l2 // per)))
        nw = ncopy
        # weights: distinct packed copies (the u8 copy only where M > 256 uses it)
        ws = []
        for _ in range(nw):
            lat = synth.latent_matrix(N, K, g, device="cuda")
            ws.append(model.PackedWeight([lat], expand=M > 256))
            del lat
        nx = max(2, min(ncopy, -(-4 * l2 // max(xb + yb, 1))))
        nx = min(nx, 64)
        xs = [synth.hidden((M, K), g, "bf16", device="cuda") for _ in range(nx)]
        ys = [torch.empty((M, N), dtype=torch.bfloat16, device=dev) for _ in range(nx)]
        wsb = torch.empty(int(L.load().tern_bitlinear_workspace(M, K)) + 16, dtype=torch.uint8,
                          device=dev)
        calls = max(nw, nx)

        def run():
            for i in range(calls):
                L.bitlinear_fwd(xs[i % nx], ws[i % nw].struct, ys[i % nx], ws=wsb)

        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            run()
        torch.cuda.current_stream().wait_stream(s)
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr):
            run()
        gr.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.reps):
            gr.replay()
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / (args.reps * calls)
        gbs = per / (us * 1e-6) / 1e9
        tops = 2.0 * M * N * K / (us * 1e-6) / 1e12
        path = "gemv" if M <= L.tern_get_gemv_max_m() else "quant+gemm_tc"
        rows.append({"M": M, "K": K, "N": N, "path": path, "us_per_call": round(us, 2),
                     "hbm_GBps": round(gbs, 1), "hbm_frac": round(gbs / hbm, 4),
                     "int8_TOPS": round(tops, 1), "int8_frac": round(tops / int8, 4),
                     "bytes_per_call": per, "weight_copies": nw, "act_copies": nx})
        print(json.dumps(rows[-1]), flush=True)
        del ws, xs, ys, gr
        torch.cuda.empty_cache()
out = {"config": "c1 (BASELINE.json configs[1]): isolated BitLinear, bf16 in/out",
       "hbm_peak_GBps": hbm, "int8_peak_TOPS": int8, "l2_bytes": l2,
       "method": "CUDA-graph replay of calls cycling through >= 4x L2 of distinct weights "
                 "and activations (HBM-resident), CUDA events, average per call",
       "points": rows}
if args.out:
    with open(args.out, "w") as f:
        json.dump(out, f, indent=1)
print(json.dumps({"summary": [(r["M"], r["K"], r["N"], r["us_per_call"], r["hbm_frac"],
                               r["int8_frac"]) for r in rows]}))
