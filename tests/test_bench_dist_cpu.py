"""bench.py's multi-rank plumbing on CPU (world_size 2, gloo): the timed value is
the max over ranks, and the data-parallel split covers every sequence once
(BASELINE configs[4] "MLGRU scan batch-split")."""
import os
import socket
import sys

import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    import bench
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, bench.max_over_ranks(10.0 + rank * 5.0, world, "cpu")))
    finally:
        dist.destroy_process_group()


def test_max_over_ranks_gloo():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    got = dict(q.get(timeout=120) for _ in range(2))
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert got == {0: 15.0, 1: 15.0}


def test_split_sequences_covers_batch():
    sys.path.insert(0, ROOT)
    import bench
    for B, world in [(32, 8), (8, 3), (5, 8), (16, 1)]:
        seen = []
        for r in range(world):
            f, n = bench.split_sequences(B, world, r)
            seen += list(range(f, f + n))
        assert seen == list(range(B))


def _bench(args, env_extra=None, timeout=300):
    import json
    import subprocess
    env = {k: v for k, v in os.environ.items()
           if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    env.update(env_extra or {})
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT,
                       env=env, capture_output=True, text=True, timeout=timeout)
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    return r, lines


def test_bench_gpus_flag_spawns_ranks():
    """`bench.py --gpus 2` without torchrun re-launches itself as 2 ranks (ADVICE r1:
    --gpus was ignored); the reference arm prints one line, from rank 0, with n_gpus 2."""
    r, lines = _bench(["--impl", "reference", "--gpus", "2", "--config", "c0", "--steps", "1",
                       "--warmup", "0", "--cpu-tokens", "2"])
    assert r.returncode == 0, r.stderr[-2000:]
    assert len(lines) == 1 and lines[0]["n_gpus"] == 2 and lines[0]["impl"] == "reference"
    assert "launching 2 ranks" in r.stderr


def test_bench_gpus_mismatch_fails():
    r, lines = _bench(["--impl", "reference", "--gpus", "2", "--config", "c0"],
                      {"WORLD_SIZE": "1", "RANK": "0", "LOCAL_RANK": "0"})
    assert r.returncode != 0 and not lines and "WORLD_SIZE=1" in r.stderr


def test_bench_shard_modes_parse():
    sys.path.insert(0, ROOT)
    import bench
    assert set(bench.SHARD_MODES) == {"dp", "out", "gather_q", "megatron", "seq"}
    assert bench.config_dict(type("C", (), dict(name="c3", L=24, d=2048, l=5632, dtype="bf16",
                                                prefill_B=16, prefill_T=2048))(), 8,
                             "out")["parallelism"].startswith("tp8")


def test_int8_peak_from_measured_peaks():
    """The INT8 roofline peak is reproducible from MEASURED_PEAKS.json: 2 x bf16 burst for an
    unthrottled run, 2 x sustained under sw_power_cap."""
    sys.path.insert(0, ROOT)
    import json
    import bench
    mp = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    pk = bench.peaks()
    p, src = bench.int8_peak_for(pk, {"sm_mhz": 1965.0, "sm_max_mhz": 1965.0, "reasons": []})
    assert p == 2 * mp["bf16_tflops"] and "burst" in src
    p, src = bench.int8_peak_for(pk, {"sm_mhz": 1700.0, "sm_max_mhz": 1965.0,
                                      "reasons": ["sw_power_cap"]})
    assert p == 2 * mp["bf16_tflops_sustained"] and "sustained" in src
    # power-cap events with the clock held at max: the burst figure (a tensor peak follows
    # the clock)
    p, src = bench.int8_peak_for(pk, {"sm_mhz": 1965.0, "sm_max_mhz": 1965.0,
                                      "reasons": ["sw_power_cap"]})
    assert p == 2 * mp["bf16_tflops"] and "burst" in src and "held" in src
    # a GEMM above the sustained-derived figure under a reduced clock is measured against
    # the burst figure (no fraction > 1)
    m, n, k = 131072, 2560, 6912
    ach = 1.05 * 2 * mp["bf16_tflops_sustained"]
    rec = {"kernel": "gemm_tc", "ms": 2 * m * n * k / (ach * 1e12) * 1e3, "m": m, "n": n, "k": k,
           "n_seg": 1, "epi": "resid"}
    rl, _ = bench.roofline([rec], 2, pk, {}, {"sm_mhz": 1725.0, "sm_max_mhz": 1965.0,
                                              "reasons": ["sw_power_cap"]})
    assert rl["peak"] == round(2 * mp["bf16_tflops"], 1) and rl["frac"] < 1.0
