"""One-shot all-gather over torch symmetric memory (shard.SymmMemAllGather; SURVEY 8(f)
f1(iii)) on the one GPU a test gets: a 1-rank NCCL process group, so the signal-pad
barriers and peer-buffer pulls run for real (no kernel waits on another GPU).  Checks the
callback contract, CUDA-graph capture (the decode-graph use), the exact int32 all-reduce,
and the library's sequence-parallel prefill through it (equal to block_prefill at world 1).
Multi-rank behaviour needs more GPUs than this sandbox gives one call."""
import os
import socket

import pytest
import torch

from paper_2406_02528_b200 import synth

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.fixture(scope="module")
def gather():
    import torch.distributed as dist
    from paper_2406_02528_b200 import shard
    own = not dist.is_initialized()
    if own:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(_free_port())
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    g = shard.SymmMemAllGather(capacity=8 << 20)
    yield g
    if own:
        dist.destroy_process_group()


def test_gather_contract_and_graph(gather):
    n = 12345
    send = torch.randint(0, 255, (n,), dtype=torch.uint8, device="cuda")
    recv = torch.zeros(n, dtype=torch.uint8, device="cuda")
    gather.register(send, recv)
    s = torch.cuda.current_stream()
    assert gather._call(0, send.data_ptr(), recv.data_ptr(), n, s.cuda_stream) == 0
    torch.cuda.synchronize()
    assert torch.equal(recv, send)
    # captured in a CUDA graph and replayed with new contents
    cs = torch.cuda.Stream()
    cs.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=cs):
        gather.gather(0, send.data_ptr(), recv.data_ptr(), n, cs.cuda_stream)
    send.fill_(7)
    recv.zero_()
    g.replay()
    torch.cuda.synchronize()
    assert torch.all(recv == 7)


def test_all_reduce_exact(gather):
    a = torch.randint(-2 ** 30, 2 ** 30, (1000,), dtype=torch.int32, device="cuda")
    out = torch.zeros_like(a)
    gather.register(a, out)
    gather.all_reduce(0, a.data_ptr(), out.data_ptr(), a.numel(),
                      torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    assert torch.equal(out, a)


def test_seqpar_prefill_through_symmetric_memory(gather):
    from paper_2406_02528_b200 import model
    B, T = 2, 160
    cfg = synth.Config("sym", 2, 256, 688, "f32", 23, B, T, B, 0)
    st = model.Stack.random(cfg, device="cuda", gen_device="cpu")
    x = synth.hidden((B, T, cfg.d), synth.generator(29), "f32").cuda()
    h1 = st.new_state(B)
    y1 = st.prefill_sp(x, h1, gather, 0)
    h = st.new_state(B)
    y = st.prefill(x, h)
    torch.cuda.synchronize()
    assert torch.equal(y1, y) and all(torch.equal(a, b) for a, b in zip(h1, h))
