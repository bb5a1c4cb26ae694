"""Experiment: does running the prefill as S independent sequence groups on S streams (an
HBM-bound quant of one group under a tensor-bound GEMM of another) beat one stream?
Rows are independent (P:409 block, P:446-456 scan per sequence), so results are identical.

    python tools/overlap_bench.py [--config c2] [--splits 1,2,4] [--stagger 0,1]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2406_02528_b200 import _lib as L  # noqa: E402
from paper_2406_02528_b200 import model, synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--splits", default="1,2,4")
    ap.add_argument("--steps", type=int, default=5)
    args = ap.parse_args()
    dev = torch.device("cuda:0")
    cfg = synth.CONFIGS[args.config]
    st = model.Stack.random(cfg, device=dev, gen_device=dev)
    B, T = cfg.prefill_B, cfg.prefill_T
    x = synth.hidden((B, T, cfg.d), synth.generator(cfg.seed + 7919, dev), cfg.dtype, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    ref = None
    res = {}
    for S in [int(s) for s in args.splits.split(",")]:
        if B % S:
            continue
        g = B // S
        xs = [x[i * g:(i + 1) * g].contiguous() for i in range(S)]
        ys = [torch.empty_like(t) for t in xs]
        bufs = [(torch.empty_like(t), torch.empty_like(t)) for t in xs]
        states = [st.new_state(g) for _ in range(S)]
        wsb = max(b.workspace_bytes(g, T, st.dtype) for b in st.blocks)
        wss = [torch.empty(wsb, dtype=torch.uint8, device=dev) for _ in range(S)]
        streams = [torch.cuda.Stream(dev) for _ in range(S)]
        main_s = torch.cuda.current_stream(dev)

        def run():
            for s in streams:
                s.wait_stream(main_s)
            # interleave launches block by block so the groups stay in step
            cur = list(xs)
            nb = len(st.blocks)
            for i, blk in enumerate(st.blocks):
                for k in range(S):
                    nxt = bufs[k][i % 2] if i < nb - 1 else ys[k]
                    L.block_prefill(blk.struct, cur[k], nxt, states[k][i], wss[k],
                                    stream=streams[k])
                    cur[k] = nxt
            for s in streams:
                main_s.wait_stream(s)

        for _ in range(3):
            run()
        torch.cuda.synchronize()
        ms = 0.0
        for i in range(args.steps):
            for hs in states:
                for h in hs:
                    h.zero_()
            flush.fill_(float(i))
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            run()
            b.record()
            torch.cuda.synchronize()
            ms += a.elapsed_time(b)
        ms /= args.steps
        y = torch.cat(ys, 0)
        if ref is None:
            ref = y.clone()
        res[S] = {"ms_per_step": round(ms, 3), "tok_s": round(B * T / ms * 1e3, 1),
                  "identical_to_1": bool(torch.equal(y, ref))}
        print(S, res[S], flush=True)
    print(json.dumps({"config": args.config, "splits": res}))


if __name__ == "__main__":
    main()
