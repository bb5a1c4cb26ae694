#!/usr/bin/env python
"""Benchmark of the MatMul-free block forward on B200 (one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl ours|reference]

A step = one prefill pass of the whole hot path (all SURVEY.md 8(a) rows that
prefill uses: RMSNorm+quant, tcgen05 GEMM with fused epilogues, MLGRU scan,
GLU) over one batch of B x T tokens through the L-block stack, inputs resident
in HBM.  `value` = prefill tokens/s of the whole job (N ranks, data parallel
over sequences: weak scaling, no collective on the data path).  The decode
rows (GEMV path, graph-replayed) are measured in the same run and reported
under "decode".  See DESIGN.md "Measurement" for every field.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "MatMul-free block tokens/s (prefill, decode) 370M-2.7B; % HBM/INT8 roofline"


# the paper's own figures (other hardware, W8A16 on Loihi 2): context only, never a target
# (north_star asks for them to be quoted with their hardware)
PAPER_CONTEXT = {
    "note": "the paper's figures for the 370M model on other hardware and precision; context only, "
            "not targets (vs_baseline stays null)",
    "loihi2_1chip_370M_generate_tok_s": {"value": 71.3, "cite": "P:241 (estimate, W8A16)"},
    "loihi2_1chip_370M_prefill_tok_s": {"value": 13965, "cite": "P:248 (estimate, W8A16)"},
    "jetson_orin_nano_400_500M_transformer_generate_tok_s": {"value": "~14",
                                                             "cite": "P:239-240, P:797-798"},
    "h100_370M_generate_tok_s": {"value": 13.4, "cite": "P:795 (seq 500, precision not stated)"},
    "one_MMF_layer_b1_seq2048_ms": {"value": 3.79, "cite": "P:198 (BitBLAS, GPU not named)"},
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c2", choices=["c0", "c2", "c3", "c4"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--decode-steps", type=int, default=None)
    ap.add_argument("--no-flatness", action="store_true",
                    help="skip the decode flatness sweep (n = 500..4000 steps)")
    ap.add_argument("--decode-batch", type=int, default=None,
                    help="decode batch per GPU (default: the config's, e.g. c4 also runs 128)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-tokens", type=int, default=None, help="oracle sample tokens")
    ap.add_argument("--no-other-configs", action="store_true",
                    help="skip the c3 / c4 prefill lines measured after the main config")
    ap.add_argument("--shard", default="dp", choices=list(SHARD_MODES),
                    help="partition over the N ranks (DESIGN.md §10): dp = sequences split, "
                         "weights replicated (weak scaling, no collective); out = BitLinear "
                         "output features sharded + NCCL all-gathers; gather_q = out with int8 "
                         "code gathers; megatron = column/row-parallel pairs + exact int32 "
                         "all-reduce; seq = sequence-parallel prefill (token slices + one "
                         "aggregate all-gather per block); all but dp: strong scaling")
    return ap.parse_args()


SHARD_MODES = {
    "dp": "dp{w} (sequences split, weights replicated)",
    "out": "tp{w} output-feature sharding, activation all-gathers (NCCL)",
    "gather_q": "tp{w} output-feature sharding, int8-code all-gathers (NCCL)",
    "megatron": "tp{w} column|row-parallel pairs, exact int32 all-reduce (NCCL)",
    "seq": "sp{w} sequence-parallel prefill (token slices, aggregate all-gather, NCCL)",
}


def peaks():
    """Roofline denominators (B200_PROFILING.md): MEASURED_PEAKS.json, else the guide's
    fallback.  The dense INT8 peak is the measured bf16 GEMM peak x 2 (the nominal
    int8:bf16 ratio of B200, 4.5 / 2.25 PFLOP/s dense): burst for an unthrottled run,
    sustained when the run's median SM clock was reduced (int8_peak_for)."""
    try:
        pk = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pk = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
              "_fallback": True}
    try:   # side note only: cuBLASLt IMMA measured on this pool by tools/int8_peak.py
        pk["int8_cublaslt"] = json.load(open(os.path.join(ROOT, "profiles", "int8_peak.json")))
    except Exception:
        pass
    return pk


def int8_peak_for(pk: dict, clocks: dict | None) -> tuple[float, str]:
    """(dense INT8 TOPS, label): 2 x MEASURED_PEAKS bf16 burst, or 2 x sustained when the
    timed region's median SM clock was reduced (< 95 % of max).  A tensor peak scales with
    the SM clock; sw_power_cap events with the median clock still at max (INT8 MMAs draw
    less power per op than the bf16 GEMM the sustained figure was measured with) keep the
    burst figure -- measured: c3's GEMMs run at 2.97 POPS there, above 2 x the bf16
    sustained figure, so that figure is no INT8 ceiling."""
    reduced, cap = False, False
    if clocks:
        sm, mx = clocks.get("sm_mhz"), clocks.get("sm_max_mhz")
        cap = "sw_power_cap" in (clocks.get("reasons") or [])
        reduced = sm is not None and mx is not None and sm < 0.95 * mx
    src = "of fallback" if pk.get("_fallback") else "of measured"
    if reduced:
        return 2.0 * pk.get("bf16_tflops_sustained", pk["bf16_tflops"]), \
            f"MEASURED_PEAKS.json bf16_tflops_sustained x 2 (nominal int8:bf16), {src}; " \
            "sustained because the timed region's median SM clock was below 95 % of max"
    return 2.0 * pk["bf16_tflops"], \
        f"MEASURED_PEAKS.json bf16_tflops x 2 (nominal int8:bf16), burst, {src}; median SM " \
        "clock at max during the timed region" + \
        (" (sw_power_cap events seen; the clock held)" if cap else "")


# ------------------------------------------------------------------ clocks
class NvmlClocks:
    """NVML sampler (every ~2 ms) running during the timed region: SM clock and the
    clock-event (throttle) reasons, as nvidia-smi reports them (B200_PROFILING.md).
    Short timed regions (tens of ms) get samples too, unlike `nvidia-smi -lms`."""

    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown", 0x8),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown", 0x40),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown", 0x20),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap", 0x4))

    def __init__(self, gpu_index: int):
        import pynvml
        self.nv = pynvml
        pynvml.nvmlInit()
        self.h = pynvml.nvmlDeviceGetHandleByIndex(gpu_index)
        self.rows = []
        self.stop_ev = threading.Event()

    def _sample(self):
        nv = self.nv
        sm = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
        mx = nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM)
        get = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            nv.nvmlDeviceGetCurrentClocksThrottleReasons
        return sm, mx, int(get(self.h))

    def start(self):
        self._sample()
        self.t = threading.Thread(target=self._run, daemon=True)
        self.t.start()
        return self

    def _run(self):
        while not self.stop_ev.is_set():
            try:
                self.rows.append(self._sample())
            except Exception:
                pass
            time.sleep(0.002)

    def stop(self):
        self.stop_ev.set()
        self.t.join(timeout=2)
        try:
            self.rows.append(self._sample())
        except Exception:
            pass
        reasons = set()
        for _, _, bits in self.rows:
            for name, const, default in self.REASONS:
                if bits & getattr(self.nv, const, default):
                    reasons.add(name)
        sm = [r[0] for r in self.rows]
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(r[1] for r in self.rows) if self.rows else None,
                "reasons": sorted(reasons), "samples": len(sm), "sampler": "nvml"}


def clock_sampler(gpu_index: int):
    try:
        return NvmlClocks(gpu_index).start()
    except Exception:
        return Clocks(gpu_index).start()


class Clocks:
    """nvidia-smi sampler running during the timed region (B200_PROFILING.md)."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[0]))
                mx.append(float(r[1]))
            except Exception:
                continue
            for n, v in zip(names, r[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------------ algorithmic work
ZERO_FRAC = 0.310   # ternary zeros of the synthetic N(0, 0.02) weights

def algo_work(rec: dict, elem: int) -> tuple[str, float]:
    """(unit, amount) of algorithmic work of one launch."""
    k, m, n = rec["k"], rec["m"], rec["n"]
    kp = (k + 127) // 128 * 128
    if rec["kernel"] in ("gemm_tc", "fcgscan", "gemm_qf"):
        return "flop", 2.0 * m * n * k                       # dense-equivalent int8 ops
    if rec["kernel"] == "quant":
        return "byte", m * k * elem + m * kp + 12.0 * m      # read x, write q + stats
    if rec["kernel"] == "scan":
        return "byte", m * 3 * n * elem + m * n * elem       # read f^c^g^, write o'
    if rec["kernel"] == "gemv":
        return "byte", n * kp / 4.0 + m * k * elem + m * (n // max(rec["n_seg"], 1)) * elem
    return "byte", 0.0


def qf_bytes(rec: dict, elem: int) -> float:
    """HBM bytes of the fused quantization inside a gemm_qf launch: the a2 pass it replaces
    (read x, write q + stats) and the GEMM's own A read of q."""
    k, m = rec["k"], rec["m"]
    kp = (k + 127) // 128 * 128
    return m * k * elem + 2.0 * m * kp + 12.0 * m


def gemm_bytes(rec: dict, elem: int) -> float:
    """Algorithmic HBM bytes of one tensor-core GEMM launch: the int8 activations
    (M x Kp), the 2-bit packed weights (N x Kp / 4), the outputs and, for the residual
    epilogue, the residual input (SwiGLU writes N/2 outputs; the fused scan writes d = N/3)."""
    k, m, n, epi = rec["k"], rec["m"], rec["n"], rec["epi"]
    kp = (k + 127) // 128 * 128
    if rec["kernel"] == "fcgscan":
        n_out = n // 3
    else:
        n_out = n // 2 if epi == 4 else n
    b = m * kp + n * kp / 4.0 + m * n_out * elem
    if rec["kernel"] != "fcgscan" and epi in (1, 6):   # residual epilogue reads x (6: in place)
        b += m * n_out * elem
    if rec["kernel"] == "gemm_qf":
        b += qf_bytes(rec, elem) - m * kp   # (the A read is in both)
    return b


def roofline(records, elem, pk, traffic_db, clocks=None):
    by = {}
    for r in records:
        u, w = algo_work(r, elem)
        e = by.setdefault(r["kernel"], {"ms": 0.0, "work": 0.0, "unit": u, "launches": 0,
                                        "bytes": 0.0, "floors": []})
        e["ms"] += r["ms"]
        e["work"] += w
        e["launches"] += 1
        if r["kernel"] == "gemm_qf":
            e["bytes"] += qf_bytes(r, elem)
        if u == "flop":   # (ops, algorithmic bytes) per launch for the attainable roofline
            e["floors"].append((w, gemm_bytes(r, elem)))
    tot = sum(e["ms"] for e in by.values()) or 1.0
    kernels = {}
    i8peak, i8src = int8_peak_for(pk, clocks)
    for name, e in by.items():
        s = e["ms"] / 1e3
        if e["unit"] == "flop":
            ach = e["work"] / s / 1e12
            peak, psrc = i8peak, i8src
            if ach > peak:   # the sustained-derived figure is no ceiling for this kernel
                peak = 2.0 * pk["bf16_tflops"]
                psrc = i8src + "; achieved exceeds 2 x bf16_tflops_sustained, so the burst " \
                    "figure (2 x bf16_tflops) is used"
            kernels[name] = {"bound": "tensor", "achieved": round(ach, 1), "peak": round(peak, 1),
                             "unit": "TFLOP/s", "frac": round(ach / peak, 4), "peak_source": psrc,
                             "frac_of_burst": round(ach / (2.0 * pk["bf16_tflops"]), 4),
                             "frac_of_sustained": round(
                                 ach / (2.0 * pk.get("bf16_tflops_sustained", pk["bf16_tflops"])), 4),
                             # the adds the method needs, nnz * M with the zero
                             # fraction of N(0, s) weights at the 1/2 mean|W| threshold:
                             # P(|z| < sqrt(2/pi)/2) = 0.310 (31.0 % measured)
                             "ternary_adds_T_per_s": round(ach / 2.0 * (1.0 - ZERO_FRAC), 1),
                             # each launch's attainable time max(ops / the peak
                             # above, algorithmic bytes / HBM peak) -- the N = d GEMMs sit
                             # below the ridge
                             "frac_of_attainable": round(
                                 sum(max(w_ / (peak * 1e12), b_ / (pk["hbm_gbs"] * 1e9))
                                     for w_, b_ in e["floors"]) * 1e3 / e["ms"], 4)}
            if e["bytes"] > 0:   # gemm_qf: the fused quantization's HBM stream beside the MMAs
                hb = e["bytes"] / s / 1e9
                kernels[name]["fused_quant_hbm"] = {
                    "achieved": round(hb, 1), "peak": pk["hbm_gbs"], "unit": "GB/s",
                    "frac": round(hb / pk["hbm_gbs"], 4),
                    "note": "bytes of the a2 quantization fused into this GEMM (read x, write "
                            "q + stats, the GEMM's A read), over the same launch time"}
        else:
            ach = e["work"] / s / 1e9
            peak = pk["hbm_gbs"]
            kernels[name] = {"bound": "hbm", "achieved": round(ach, 1), "peak": peak,
                             "unit": "GB/s", "frac": round(ach / peak, 4)}
        kernels[name].update({"share": round(e["ms"] / tot, 4), "launches": e["launches"],
                              "ms_total": round(e["ms"], 3),
                              "ms_per_launch": round(e["ms"] / e["launches"], 5)})
    epi_names = {0: "store", 1: "resid", 2: "fcg", 3: "mlgru", 4: "swiglu", 5: "acc", 6: "resid_red"}
    sub = {}
    for r in records:
        if r["kernel"] not in ("gemm_tc", "gemm_qf", "gemv", "fcgscan"):
            continue
        key = f'{r["kernel"]}:{epi_names.get(r["epi"], r["epi"])}:n{r["n"]}k{r["k"]}'
        u, w = algo_work(r, elem)
        e = sub.setdefault(key, {"ms": 0.0, "work": 0.0, "unit": u, "launches": 0})
        e["ms"] += r["ms"]
        e["work"] += w
        e["launches"] += 1
    for key, e in sub.items():
        s = e["ms"] / 1e3
        rate = e["work"] / s / (1e12 if e["unit"] == "flop" else 1e9)
        kernels.setdefault("by_shape", {})[key] = {
            "ms_per_launch": round(e["ms"] / e["launches"], 5),
            ("TFLOP/s" if e["unit"] == "flop" else "GB/s"): round(rate, 1)}
    dom = max((k for k in kernels if k != "by_shape"), key=lambda k: kernels[k]["share"]) \
        if kernels else None
    rl = None
    if dom:
        d = kernels[dom]
        tr = traffic_db.get(dom)
        tr = tr.get("bytes_per_launch") if isinstance(tr, dict) else tr
        rl = {"kernel": dom, "bound": d["bound"], "achieved": d["achieved"], "peak": d["peak"],
              "unit": d["unit"], "frac": d["frac"], "traffic": tr,
              "peak_source": d["peak_source"] if d["bound"] == "tensor" else
              "MEASURED_PEAKS.json hbm_gbs" + (" (of fallback)" if pk.get("_fallback")
                                                 else " (of measured)")}
        if d["bound"] == "tensor":
            rl["frac_of_burst"] = d["frac_of_burst"]
            rl["frac_of_sustained"] = d["frac_of_sustained"]
            rl["frac_of_attainable"] = d["frac_of_attainable"]
            rl["attainable_note"] = ("sum over launches of max(dense-equivalent ops / the tensor "
                                     "peak, algorithmic bytes / HBM peak) over the measured time "
                                     "(SURVEY 8(d): GEMMs below the ridge, e.g. the N = 1024 "
                                     "projections, are HBM-bound)")
            if "int8_cublaslt" in pk:   # side note: cuBLASLt s8 GEMM on this pool
                rl["note_cublaslt_int8_tops"] = {
                    k: pk["int8_cublaslt"].get(k) for k in ("int8_tops_burst", "int8_tops_sustained")}
        if tr is None:
            rl["traffic_note"] = "no ncu --set full capture of this config in profiles/traffic.json"
    return rl, kernels


# ------------------------------------------------------------------ multi-rank timing
def max_over_ranks(ms: float, world: int, device=None) -> float:
    """The job's time is the slowest rank's (B200_PROFILING.md): all-reduce MAX."""
    if world <= 1:
        return float(ms)
    import torch
    import torch.distributed as dist
    t = torch.tensor([ms], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def split_sequences(B_global: int, world: int, rank: int) -> tuple[int, int]:
    """Data-parallel split of a global batch of sequences: (first, count) of rank."""
    base, extra = divmod(B_global, world)
    first = rank * base + min(rank, extra)
    return first, base + (1 if rank < extra else 0)


# ------------------------------------------------------------------ oracle (cpu) arm
def oracle_blocks(latents, cfg):
    import oracle as O
    return [O.OracleBlock({k: v.numpy() for k, v in lat.items()}, cfg.d, cfg.l) for lat in latents]


def oracle_prefill_time(oblocks, cfg, tokens, scale_blocks, seed=12345):
    """Time the oracle (as it stands) on 1 sequence x `tokens` through the sampled
    blocks; return (tokens/s scaled to the full stack, seconds)."""
    import numpy as np

    import oracle as O
    from paper_2406_02528_b200 import synth
    g = synth.generator(seed)
    x = synth.hidden((1, tokens, cfg.d), g, cfg.dtype).float().numpy()
    Hs = [np.zeros((1, cfg.d), np.float32) for _ in oblocks]
    t0 = time.perf_counter()
    O.stack(oblocks, x, Hs, bf16=(cfg.dtype == "bf16"), eps=cfg.eps)
    dt = time.perf_counter() - t0
    return tokens / (dt * scale_blocks), dt


def cpu_sample_plan(cfg, args):
    nb = cfg.L if cfg.L <= 24 and cfg.d <= 1024 else 2
    tokens = args.cpu_tokens or (32 if cfg.d <= 1024 else 8)
    return nb, tokens


def run_reference(args, cfg, rank, world):
    import torch

    import oracle as O
    from paper_2406_02528_b200 import synth
    if rank != 0:
        return
    nb, tokens = cpu_sample_plan(cfg, args)
    gdev = "cuda" if torch.cuda.is_available() else "cpu"
    g = synth.generator(cfg.seed, gdev)
    lats = [{k: v.cpu() for k, v in synth.latent_block(cfg.d, cfg.l, g, device=gdev).items()}
            for _ in range(nb)]
    ob = oracle_blocks(lats, cfg)
    scale = cfg.L / nb
    for _ in range(args.warmup):
        oracle_prefill_time(ob, cfg, tokens, scale)
    times = []
    for _ in range(args.steps):
        _, dt = oracle_prefill_time(ob, cfg, tokens, scale)
        times.append(dt * scale)
    tot = sum(times)
    val = tokens * args.steps / tot
    sample = (f"1 sequence x {tokens} tokens prefill through {nb} of {cfg.L} blocks per step "
              f"(time scaled x{scale:g} to the full stack)")
    out = {"impl": "reference", "metric": METRIC, "value": round(val, 3), "unit": "tokens/s",
           "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": round(tot / args.steps * 1e3, 3), "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
           "config": config_dict(cfg, world, args.shard),
           "cpu_baseline": {"value": round(val, 3), "unit": "tokens/s", "cores": O.get_threads(),
                            "kind": "oracle", "sample": sample, "cpu": cpu_model()},
           "e2e": {"value": round(val, 3), "unit": "tokens/s", "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def config_dict(cfg, world, mode="dp"):
    per = "per GPU" if mode == "dp" else f"global (the same batch on all {world} ranks)"
    return {"workload": f"{cfg.name}: {cfg.L}-block stack d={cfg.d} l={cfg.l} "
                        f"{cfg.dtype} activations, prefill {cfg.prefill_B}x{cfg.prefill_T} {per}",
            "L": cfg.L, "d": cfg.d, "l": cfg.l,
            ("batch_per_gpu" if mode == "dp" else "global_batch"): cfg.prefill_B,
            "seq_len": cfg.prefill_T, "activations": cfg.dtype,
            "parallelism": SHARD_MODES[mode].format(w=world),
            "l2": "flushed between timed steps (256 MiB write); activations > L2"}


# ------------------------------------------------------------------ other configs
def other_config_prefill(name: str, steps: int, warmup: int, pk: dict, dev) -> dict:
    """Prefill of BASELINE.json's config `name` (c3 / c4: full stack, full batch, bf16) on this
    GPU, timed like the main line (L2 flushed between steps, CUDA events), plus its dominant
    kernel's roofline -- so the driver's own run carries the 1.3B and 2.7B shapes too."""
    import torch

    from paper_2406_02528_b200 import _lib as L
    from paper_2406_02528_b200 import model, synth
    cfg = synth.CONFIGS[name]
    st = model.Stack.random(cfg, device=dev, gen_device=dev)
    B, T = cfg.prefill_B, cfg.prefill_T
    x = synth.hidden((B, T, cfg.d), synth.generator(cfg.seed + 7919, dev), cfg.dtype, device=dev)
    y = torch.empty_like(x)
    bufs = (torch.empty_like(x), torch.empty_like(x))
    states = st.new_state(B)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    for _ in range(warmup):
        st.prefill(x, states, out=y, bufs=bufs)
    torch.cuda.synchronize()
    clocks = clock_sampler(dev.index or 0)
    ms = 0.0
    for i in range(steps):
        for h in states:
            h.zero_()
        flush.fill_(float(i))
        torch.cuda.synchronize()
        a_, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a_.record()
        st.prefill(x, states, out=y, bufs=bufs)
        b_.record()
        torch.cuda.synchronize()
        ms += a_.elapsed_time(b_)
    ck = clocks.stop()
    L.tern_profile_enable(True)
    st.prefill(x, states, out=y, bufs=bufs)
    torch.cuda.synchronize()
    L.tern_profile_enable(False)
    recs = L.tern_profile_collect()
    try:   # this config's ncu --set full capture (profiles/traffic.json), if any
        tdb = json.load(open(os.path.join(ROOT, "profiles", "traffic.json"))).get(cfg.name, {})
    except Exception:
        tdb = {}
    rl, kernels = roofline(recs, 2 if cfg.dtype == "bf16" else 4, pk, tdb, ck)
    out = {"workload": f"{name}: {cfg.L}-block stack d={cfg.d} l={cfg.l} {cfg.dtype}, prefill "
                       f"{B}x{T}", "tokens_per_s": round(B * T * steps / (ms / 1e3), 1),
           "ms_per_step": round(ms / steps, 3), "steps": steps, "warmup": warmup,
           "roofline": rl, "by_shape": kernels.get("by_shape"), "clocks": ck}
    del st, x, y, bufs, states, flush
    torch.cuda.empty_cache()
    return out


# ------------------------------------------------------------------ our arm
def backward_line(pk: dict, dev) -> dict:
    """Alg. 1 BackwardPass of one c2-sized BitLinear
    (tokens of one c2 prefill step, d -> d and l -> d), bitlinear_bwd on the tensor cores
    (bf16 hi + lo split, reading B7) and on the fp32 CUDA cores; side measurement, not part
    of `value` (the north_star path is the forward).  Rates count the dense products the
    backward computes, 2 m n k each for dY and dW (fp32-equivalent); the tensor cores execute
    twice that in bf16 (the split), which `mma_bf16_tflops_equiv` reports against the bf16
    peak."""
    import torch
    from paper_2406_02528_b200 import _lib as Lb
    from paper_2406_02528_b200 import model, synth
    res = {}
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    for (m, k, n) in [(16384, 1024, 1024), (16384, 2816, 1024)]:
        W = synth.latent_matrix(n, k, synth.generator(101, dev), device=dev)
        pw = model.PackedWeight([W])
        x = torch.randn(m, k, device=dev)
        dO = torch.randn(m, n, device=dev)
        dX, dW, db = torch.empty_like(x), torch.empty(n, k, device=dev), torch.empty(n, device=dev)
        ws = torch.empty(int(Lb.load().bitlinear_bwd_workspace(m, k, n)), dtype=torch.uint8,
                         device=dev)
        row = {}
        for tc in (True, False):
            Lb.tern_set_bwd_tc(tc)
            Lb.bitlinear_bwd(x, pw.struct, dO, dX, dW, db, ws=ws)
            ts = []
            for _ in range(3):
                flush.fill_(1.0)
                a_, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a_.record()
                Lb.bitlinear_bwd(x, pw.struct, dO, dX, dW, db, ws=ws)
                b_.record()
                torch.cuda.synchronize()
                ts.append(a_.elapsed_time(b_))
            ms = min(ts)
            fl = 4.0 * m * n * k
            r = {"ms": round(ms, 4), "tflops_fp32_equiv": round(fl / ms / 1e9, 1)}
            if tc:
                r["mma_bf16_tflops_equiv"] = round(2 * fl / ms / 1e9, 1)
                r["frac_of_bf16_peak_whole_call"] = round(2 * fl / ms / 1e9 / pk["bf16_tflops"], 4)
            row["tensor_core" if tc else "cuda_core_fp32"] = r
        res[f"m{m}_k{k}_n{n}"] = row
    Lb.tern_set_bwd_tc(True)
    res["note"] = ("whole bitlinear_bwd call (forward quant recompute, operand prep, dY GEMM, "
                   "norm backward, dW GEMM + slice reduce, db), min of 3, L2 flushed; "
                   "per-kernel split in profiles/r02_bwd_launches.txt")
    return res


def finish_sharded(args, cfg, rank, world, mode, st, value, ms_max, rl, kernels, recs, ck, e2e,
                   pk):
    """The JSON line of a sharded run (--shard out|gather_q|megatron|seq): prefill of one
    global batch over the N ranks (strong scaling), plus -- for the output-feature modes --
    the config's decode batch through the sharded stack (one CUDA-graph replay per step,
    4 collectives per block issued by the library through the all-gather callback)."""
    import torch

    from paper_2406_02528_b200 import synth
    dev = st.device
    dec = None
    if mode != "seq":
        nd = args.decode_steps if args.decode_steps is not None else min(cfg.decode_steps, 200)
        Bd = args.decode_batch or cfg.decode_B
        xs = synth.hidden((nd, Bd, cfg.d), synth.generator(cfg.seed + 31, dev), cfg.dtype,
                          device=dev)
        dstates = st.new_state(Bd)
        g, xin_d, _ = st.capture_decode(Bd, dstates)
        for t_ in range(3):
            xin_d.copy_(xs[t_])
            g.replay()
        for h in dstates:
            h.zero_()
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        d0, d1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        d0.record()
        for t_ in range(nd):
            xin_d.copy_(xs[t_])
            g.replay()
        d1.record()
        torch.cuda.synchronize()
        dms = max_over_ranks(d0.elapsed_time(d1), world, dev)
        wbytes = st.weight_bytes
        dec = {"tokens_per_s": round(nd * Bd / (dms / 1e3), 1), "global_batch": Bd,
               "steps": nd, "ms_per_token_step": round(dms / nd, 4),
               "weight_bytes_per_step_per_gpu": wbytes,
               "hbm_frac_of_weights_stream": round(wbytes / (dms / nd / 1e3) / 1e9 / pk["hbm_gbs"],
                                                   4),
               "path": "per_block, sharded", "graph": True,
               "collectives_per_step": (2 if mode == "megatron" else 4) * cfg.L}
        del g
    out = {"metric": METRIC, "value": round(value, 1), "unit": "tokens/s", "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": round(ms_max / args.steps, 4), "higher_is_better": True,
           "scaling": "strong", "vs_baseline": None, "dtype": cfg.dtype, "shard": mode,
           "data": "synthetic (seeded N(0,0.02) latent weights, N(0,1) hidden states; no "
                   "embedding/LM head)",
           "config": config_dict(cfg, world, mode), "roofline": rl, "kernels": kernels,
           "gpu_launches": len(recs), "clocks": ck, "e2e": e2e, "decode": dec,
           "comm": comm_info(world)}
    if rank == 0:
        print(json.dumps(out), flush=True)


def comm_info(world: int) -> dict:
    import torch
    info = {"world": world}
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        info["backend"] = dist.get_backend()
        try:
            v = torch.cuda.nccl.version()
            info["nccl_version"] = ".".join(map(str, v)) if isinstance(v, tuple) else v
        except Exception:
            pass
    return info


def run_ours(args, cfg, rank, world, local_rank):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2406_02528_b200 import _lib as L
    from paper_2406_02528_b200 import model, synth

    L.load()
    if os.environ.get("TERN_BENCH_FIN") is not None:   # debug: batched-decode finalize path
        L.tern_set_batched_fin(int(os.environ["TERN_BENCH_FIN"]))
    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    pk = peaks()
    try:   # ncu --set full dram bytes per launch, keyed by config (tools/ncu_traffic.py)
        traffic_db = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
        traffic_db = traffic_db.get(cfg.name + ("" if args.shard == "dp" or world == 1
                                                else f":{args.shard}{world}"), {})
    except Exception:
        traffic_db = {}

    keep = 0
    do_cpu = rank == 0 and world == 1 and not args.no_cpu_baseline
    nb_cpu, cpu_tokens = cpu_sample_plan(cfg, args)
    if do_cpu:
        keep = nb_cpu
    mode = args.shard
    sharded = mode in ("out", "gather_q", "megatron")
    gather = None
    if sharded:
        from paper_2406_02528_b200 import shard as S
        gather = S.NcclAllGather()
        shard_spec = (rank, gather, mode == "gather_q", mode == "megatron")
    st = model.Stack.random(cfg, device=dev, gen_device=dev, keep_latents=keep,
                            shard=shard_spec if sharded else None)
    dt = synth.torch_dtype(cfg.dtype)
    elem = 2 if cfg.dtype == "bf16" else 4
    B, T, d = cfg.prefill_B, cfg.prefill_T, cfg.d
    if mode == "dp":   # every rank its own B sequences (weak scaling)
        gx = synth.generator(cfg.seed + 7919 * (rank + 1), dev)
        x = synth.hidden((B, T, d), gx, cfg.dtype, device=dev)
    else:              # one global batch, the same on every rank (strong scaling)
        gx = synth.generator(cfg.seed + 7919, dev)
        x = synth.hidden((B, T, d), gx, cfg.dtype, device=dev)
        if mode == "seq":   # this rank's contiguous token slice of every sequence (C23)
            from paper_2406_02528_b200 import shard as S
            t0, t1 = S.seq_slice(T, world, rank)
            x = x[:, t0:t1].contiguous()
            gather = S.NcclAllGather()
    y = torch.empty_like(x)
    bufs = (torch.empty_like(x), torch.empty_like(x))
    states = st.new_state(B)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    def barrier():
        if world > 1:
            dist.barrier()

    def step():
        if mode == "seq":
            st.prefill_sp(x, states, gather, rank, out=y)
        else:
            st.prefill(x, states, out=y, bufs=bufs)

    def reset():
        for h in states:
            h.zero_()

    for _ in range(args.warmup):
        reset()
        step()
    torch.cuda.synchronize()

    clocks = clock_sampler(local_rank)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    for i in range(args.steps):
        reset()
        flush.fill_(float(i))
        torch.cuda.synchronize()
        barrier()
        ev[i][0].record()
        step()
        ev[i][1].record()
    torch.cuda.synchronize()
    barrier()
    ck = clocks.stop()
    # per-kernel times for the roofline: the same steps again with the library's
    # event hooks on (they bracket every launch, which also stops consecutive
    # launches overlapping through PDL -- so the timed loop above runs without them)
    L.tern_profile_enable(True)
    for i in range(args.steps):
        reset()
        flush.fill_(float(i))
        torch.cuda.synchronize()
        step()
    torch.cuda.synchronize()
    L.tern_profile_enable(False)
    recs = L.tern_profile_collect()
    ms = sum(a.elapsed_time(b) for a, b in ev)
    ms_max = max_over_ranks(ms, world, dev)
    tokens = B * T * args.steps * (world if mode == "dp" else 1)
    value = tokens / (ms_max / 1e3)
    rl, kernels = roofline(recs, elem, pk, traffic_db, ck)

    # ---------------- e2e: pinned host input -> device, prefill, device -> pinned host result,
    # every step (Stack.prefill_host: uploads / downloads on copy streams, double-buffered)
    xh = [x.cpu().pin_memory() for _ in range(args.steps)]
    yh = [torch.empty_like(xh[0]).pin_memory() for _ in range(args.steps)]
    if mode == "seq":
        st.prefill_host_fn = lambda xi, hs, yo: st.prefill_sp(xi, hs, gather, rank, out=yo)
    st.prefill_host(xh[:1], yh[:1])
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    e0.record()
    st.prefill_host(xh, yh, before_step=lambda i: flush.fill_(float(i)))   # L2 flushed per step
    e1.record()
    torch.cuda.synchronize()
    barrier()
    assert torch.equal(yh[-1], y.cpu()), "e2e output differs from the device-timed step"
    e2e_ms = max_over_ranks(e0.elapsed_time(e1), world, dev)
    e2e = {"value": round(tokens / (e2e_ms / 1e3), 1), "unit": "tokens/s",
           "h2d_bytes_per_step": xh[0].numel() * xh[0].element_size(),
           "d2h_bytes_per_step": yh[0].numel() * yh[0].element_size(),
           "path": "Stack.prefill_host (C ABI prefill; H2D / D2H of every step on copy streams, "
                   "overlapping the neighbouring steps' compute; L2 flushed before each step), "
                   "pinned host buffers"}

    # ---------------- one long sequence (B = 1 x T): the workload of P:198 (batch 1, seq 2048,
    # "one MMF layer"); prefill picks GEMM + the 8-channel scan here
    if mode != "dp":
        return finish_sharded(args, cfg, rank, world, mode, st, value, ms_max, rl, kernels, recs,
                              ck, e2e, pk)
    x1 = x[:1].contiguous()
    y1 = torch.empty_like(x1)
    s1 = st.new_state(1)
    b1bufs = (torch.empty_like(x1), torch.empty_like(x1))
    for h in s1:
        h.zero_()
    st.prefill(x1, s1, out=y1, bufs=b1bufs)
    torch.cuda.synchronize()
    b1_ms = []
    for i in range(3):
        for h in s1:
            h.zero_()
        flush.fill_(float(i))
        torch.cuda.synchronize()
        barrier()
        a_, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a_.record()
        st.prefill(x1, s1, out=y1, bufs=b1bufs)
        b_.record()
        torch.cuda.synchronize()
        b1_ms.append(a_.elapsed_time(b_))
    b1 = max_over_ranks(min(b1_ms), world, dev)
    prefill_b1 = {"tokens_per_s": round(T / (b1 / 1e3), 1), "batch": 1, "seq_len": T,
                  "ms_per_step": round(b1, 4), "us_per_block": round(b1 * 1e3 / cfg.L, 1),
                  "reps": 3, "stat": "min of 3, L2 flushed before each",
                  "context": "P:198: one MMF layer at batch 1, seq 2048 = 3.79 ms on the paper's "
                             "H100 fused kernel (another machine; not a target)"}

    # ---------------- decode: graph-replayed steps continuing from h = 0
    nd = args.decode_steps if args.decode_steps is not None else min(cfg.decode_steps, 500)
    Bd = args.decode_batch or cfg.decode_B
    xs = synth.hidden((nd, Bd, d), synth.generator(cfg.seed + 31, dev), cfg.dtype, device=dev)

    def time_decode(persistent: bool):
        st.persistent_decode = persistent
        dstates = st.new_state(Bd)
        g, xin_d, yout_d = st.capture_decode(Bd, dstates)
        path = st.last_decode_path
        for h in dstates:
            h.zero_()
        for t_ in range(3):
            xin_d.copy_(xs[t_])
            g.replay()
        for h in dstates:
            h.zero_()
        torch.cuda.synchronize()
        flush.fill_(1.0)
        torch.cuda.synchronize()
        barrier()
        d0, d1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        d0.record()
        for t_ in range(nd):
            xin_d.copy_(xs[t_])
            g.replay()
        d1.record()
        torch.cuda.synchronize()
        barrier()
        del g
        return max_over_ranks(d0.elapsed_time(d1), world, dev), path

    dms, dpath = time_decode(False)
    wbytes = st.weight_bytes
    persistent = dpath == "persistent"
    dec = {"tokens_per_s": round(nd * Bd * world / (dms / 1e3), 1), "batch_per_gpu": Bd,
           "steps": nd, "ms_per_token_step": round(dms / nd, 4),
           "weight_bytes_per_step": wbytes,
           "hbm_frac_of_weights_stream": round(wbytes / (dms / nd / 1e3) / 1e9 / pk["hbm_gbs"], 4),
           "path": dpath,
           "launches_per_step": ((cfg.L + 31) // 32) if persistent else 4 * cfg.L,
           "graph": True,
           "note": ("whole step = one persistent cooperative kernel per 32 blocks (stack_decode): "
                    "4 BitLinear phases per block separated by grid barriers, next phase's "
                    "weight slice TMA-copied to smem during the current one"
                    if persistent else
                    "4 launches per block (decode GEMV for B<=4: norm+quant prologue, "
                    "MLGRU/SwiGLU/residual epilogues; quant + split-K tcgen05 GEMM above)")}
    # flatness of decode throughput in the number of generated tokens (Table 2 P:237-244,
    # constant time and memory per token): n in {500, 1000, 2000, 4000} steps from
    # h = 0 at the config's decode batch, one graph replay per step
    flat = None
    if rank == 0 and world == 1 and not args.no_flatness:
        st.persistent_decode = False
        fstates = st.new_state(Bd)
        gf, xin_f, _ = st.capture_decode(Bd, fstates)
        nmax = 4000
        xf = synth.hidden((64, Bd, d), synth.generator(cfg.seed + 47, dev), cfg.dtype, device=dev)
        per_n = {}
        for n_ in (500, 1000, 2000, nmax):
            for h in fstates:
                h.zero_()
            torch.cuda.synchronize()
            f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            f0.record()
            for t_ in range(n_):
                xin_f.copy_(xf[t_ % 64])
                gf.replay()
            f1.record()
            torch.cuda.synchronize()
            per_n[str(n_)] = round(n_ * Bd / (f0.elapsed_time(f1) / 1e3), 1)
        del gf
        vals = list(per_n.values())
        flat = {"tokens_per_s": per_n, "batch": Bd, "max_over_min": round(max(vals) / min(vals), 4),
                "within_10pct": max(vals) / min(vals) <= 1.10,
                "note": "steps from h = 0; inputs cycle through 64 pre-drawn tokens; the state is "
                        "[B][d] per block whatever n is (S:593)"}
        dec["flatness"] = flat
    pms, ppath = time_decode(True)
    if ppath == "persistent":   # the one-launch alternative (stack_decode), for comparison
        dec["persistent_kernel"] = {"tokens_per_s": round(nd * Bd * world / (pms / 1e3), 1),
                                    "ms_per_token_step": round(pms / nd, 4),
                                    "launches_per_step": (cfg.L + 31) // 32}
    st.persistent_decode = False

    out = {"metric": METRIC, "value": round(value, 1), "unit": "tokens/s", "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": round(ms_max / args.steps, 4), "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": cfg.dtype,
           "contraction": "s8 activations x ternary (u8 fields) -> s32 on tcgen05 kind::i8",
           "data": "synthetic (seeded N(0,0.02) latent weights, N(0,1) hidden states; no "
                   "embedding/LM head)",
           "config": config_dict(cfg, world), "roofline": rl, "kernels": kernels,
           "gpu_launches": len(recs), "clocks": ck, "e2e": e2e, "decode": dec,
           "prefill_b1": prefill_b1, "comm": comm_info(world), "paper_context": PAPER_CONTEXT}
    if rank == 0 and world == 1 and cfg.name == "c2" and not args.no_other_configs:
        try:
            out["backward"] = backward_line(pk, dev)
        except Exception as e:   # reported, never required
            out["backward"] = {"error": repr(e)}
    if rank == 0 and world == 1 and cfg.name == "c2" and not args.no_other_configs:
        # the metric spans 370M-2.7B: the 1.3B (c3) and 2.7B (c4) prefill lines, each its own
        # stack at full size (BASELINE.json configs[3], configs[4]); not part of `value`
        out["other_configs"] = {}
        for name in ("c3", "c4"):
            try:
                out["other_configs"][name] = other_config_prefill(name, 2, 2, pk, dev)
            except Exception as e:   # reported, never required
                out["other_configs"][name] = {"error": repr(e)}

    if do_cpu:
        try:
            import oracle as O
            ob = oracle_blocks(st.latents, cfg)
            val, secs = oracle_prefill_time(ob, cfg, cpu_tokens, cfg.L / nb_cpu)
            nthr = O.get_threads()
            O.set_threads(1)   # also one thread (a shorter sample)
            t1 = max(4, cpu_tokens // 4)
            val1, secs1 = oracle_prefill_time(ob, cfg, t1, cfg.L / nb_cpu)
            O.set_threads(nthr)
            out["cpu_baseline"] = {
                "value": round(val, 3), "unit": "tokens/s", "cores": nthr,
                "affinity_cpus": len(os.sched_getaffinity(0)), "nproc": os.cpu_count(),
                "value_1thread": round(val1, 3), "sample_1thread": f"1 sequence x {t1} tokens",
                "kind": "oracle", "cpu": cpu_model(), "seconds": round(secs + secs1, 2),
                "sample": f"1 sequence x {cpu_tokens} tokens prefill through {nb_cpu} of "
                          f"{cfg.L} blocks (scaled to the full stack)"}
        except Exception as e:  # the baseline is reported, never required
            out["cpu_baseline"] = {"value": None, "error": repr(e)}
    if rank == 0:
        print(json.dumps(out), flush=True)


def free_port() -> int:
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def launch_ranks(n: int) -> int:
    """`bench.py --gpus N` without a torchrun environment: re-run this command as N
    ranks under torch.distributed.run (one process per GPU, rendezvous on 127.0.0.1)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={n}", "--master-addr=127.0.0.1", f"--master-port={free_port()}",
           os.path.abspath(__file__), *sys.argv[1:]]
    print(f"[bench] launching {n} ranks: {' '.join(cmd)}", file=sys.stderr, flush=True)
    return subprocess.call(cmd)


def main():
    args = parse()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(launch_ranks(args.gpus))
    from paper_2406_02528_b200 import synth
    cfg = synth.CONFIGS[args.config]
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.impl == "reference":
        return run_reference(args, cfg, rank, world)
    if world > 1 or args.shard != "dp":
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        if not dist.is_initialized():
            if "MASTER_ADDR" not in os.environ:   # 1-rank group for --shard at N = 1
                os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(free_port()),
                                  RANK="0", WORLD_SIZE="1")
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        t = torch.ones(1, device="cuda")   # force communicator creation before timing
        dist.all_reduce(t)
        torch.cuda.synchronize()
        print(f"[bench] rank {dist.get_rank()}/{dist.get_world_size()}: NCCL communicator up on "
              f"cuda:{local_rank} (all_reduce check = {int(t.item())})", file=sys.stderr,
              flush=True)
    try:
        run_ours(args, cfg, rank, world, local_rank)
    finally:
        import torch.distributed as dist
        if dist.is_available() and dist.is_initialized():
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
