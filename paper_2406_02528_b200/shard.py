"""Output-feature sharding of the MatMul-free block over ranks (tern.h
`tern_shard`; BASELINE.json configs[3,4]).

Rank r owns channels [r*ds, (r+1)*ds) of f, c, g, o and down (ds = d/world)
and [r*ls, (r+1)*ls) of gate and up (ls = l/world).  Its weight rows are packed
with the FULL matrix's absmean scale (one scale per matrix), so every
output element is computed exactly as without sharding; the library gathers
the 4 per-block activations (o', x1, p, y) through the callback of an
`AllGather` object.  Three back-ends:
  * `NcclAllGather`: torch.distributed all_gather_into_tensor (NCCL over
    NVLink / NVSwitch, one process per GPU) on the library's stream;
  * `SymmMemAllGather`: a one-shot all-gather over torch symmetric memory
    (P2P loads, device-side barriers, graph-capturable).
  * `ThreadAllGather`: `world` virtual ranks as host threads on one GPU, each
    with its own stream, ordered by CUDA events (no kernel waits on another) --
    the single-GPU emulation used by the tests.
`plan()` is the pure host-side partition (tested on CPU with gloo against the
oracle in tests/test_shard_cpu.py).
"""
from __future__ import annotations

import ctypes as C
import threading
import weakref

import torch

from . import _lib as L


def plan(d: int, l: int, world: int, rank: int) -> dict:
    """Channel ranges of `rank` (pure host logic)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"rank {rank} of world {world}")
    if d % world or l % world:
        raise ValueError(f"d={d} and l={l} must divide by world={world}")
    ds, ls = d // world, l // world
    if world > 1 and (ds % 64 or ls % 16):
        raise ValueError(f"d/world={ds} must be a multiple of 64 and l/world={ls} of 16")
    return {"ds": ds, "ls": ls, "ch": (rank * ds, (rank + 1) * ds),
            "gl": (rank * ls, (rank + 1) * ls)}


def seq_slice(T: int, world: int, rank: int) -> tuple[int, int]:
    """Token range [t0, t1) of `rank` in the sequence-parallel prefill (reading C23:
    contiguous slices [r T / world, (r+1) T / world)); pure host logic."""
    if world < 1 or not 0 <= rank < world or T < 0:
        raise ValueError(f"rank {rank} of world {world}, T={T}")
    return rank * T // world, (rank + 1) * T // world


def shard_latents(latent: dict, d: int, l: int, world: int, rank: int,
                  megatron: bool = False) -> dict:
    """Slices of one block's latent matrices for `rank` (see plan()): output rows
    of every matrix, or with megatron the input COLUMNS of W_o
    and W_down (row-parallel: [r*ds, (r+1)*ds) of o's and [r*ls, (r+1)*ls) of
    down's inputs, all d outputs)."""
    p = plan(d, l, world, rank)
    c0, c1 = p["ch"]
    g0, g1 = p["gl"]
    out = {k: latent[k][c0:c1] for k in ("f", "c", "g", "o", "down")}
    out.update({k: latent[k][g0:g1] for k in ("gate", "up")})
    if megatron:
        out["o"] = latent["o"][:, c0:c1].contiguous()
        out["down"] = latent["down"][:, g0:g1].contiguous()
    return out


def full_scales(latent: dict, device) -> dict:
    """mean|W| of each full latent matrix, computed by tern_pack (binary64 sum, C4)."""
    from .model import PackedWeight
    return {k: PackedWeight([latent[k].to(device)], expand=False).scales[0:1].clone()
            for k in ("f", "c", "g", "o", "gate", "up", "down")}


class AllGather:
    """Base: owns the ctypes callback and resolves raw device pointers back to
    byte views of registered torch tensors (workspaces, activations)."""

    def __init__(self, world: int):
        self.world = world
        self._tensors = {}   # (data_ptr, nbytes) -> weakref to the tensor
        self._lock = threading.Lock()
        self.cb = L.ALLGATHER_FN(self._call)
        self.cb_ar = L.ALLREDUCE_FN(self._call_ar)
        self.error = None

    def register(self, *tensors):
        """Make the tensors' memory resolvable by view().  Only weak references are kept:
        a tensor the caller drops leaves the registry (no memory is held alive by it)."""
        with self._lock:
            for k in [k for k, r in self._tensors.items() if r() is None]:
                del self._tensors[k]
            for t in tensors:
                self._tensors[(t.data_ptr(), t.numel() * t.element_size())] = weakref.ref(t)

    def view(self, p: int, nbytes: int) -> torch.Tensor:
        with self._lock:
            live = [r() for r in self._tensors.values()]
        for t in live:
            if t is None:
                continue
            base = t.data_ptr()
            size = t.numel() * t.element_size()
            if base <= p and p + nbytes <= base + size:
                flat = t.view(torch.uint8).reshape(-1) if t.dtype != torch.uint8 else t.reshape(-1)
                return flat[p - base:p - base + nbytes]
        raise KeyError(f"pointer {p:#x} (+{nbytes}) is in no registered tensor")

    def _call(self, ctx, send, recv, nbytes, stream):
        try:
            self.gather(int(ctx or 0), int(send), int(recv), int(nbytes), int(stream or 0))
            return 0
        except Exception as e:  # surfaces as TERN_ERR_CUDA in the C call
            self.error = e
            return 1

    def gather(self, rank, send, recv, nbytes, stream):
        raise NotImplementedError

    def _call_ar(self, ctx, send, recv, count, stream):
        try:
            self.all_reduce(int(ctx or 0), int(send), int(recv), int(count), int(stream or 0))
            return 0
        except Exception as e:
            self.error = e
            return 1

    def all_reduce(self, rank, send, recv, count, stream):
        raise NotImplementedError


class NcclAllGather(AllGather):
    """torch.distributed all-gather (NCCL) on the library's stream."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        super().__init__(dist.get_world_size(group))

    def gather(self, rank, send, recv, nbytes, stream):
        s = torch.cuda.ExternalStream(stream) if stream else torch.cuda.current_stream()
        with torch.cuda.stream(s):
            self.dist.all_gather_into_tensor(self.view(recv, nbytes * self.world),
                                             self.view(send, nbytes), group=self.group)

    def all_reduce(self, rank, send, recv, count, stream):
        s = torch.cuda.ExternalStream(stream) if stream else torch.cuda.current_stream()
        with torch.cuda.stream(s):
            r = self.view(recv, count * 4).view(torch.int32)
            if send != recv:
                r.copy_(self.view(send, count * 4).view(torch.int32))
            self.dist.all_reduce(r, group=self.group)


class SymmMemAllGather(AllGather):
    """One-shot all-gather over torch symmetric memory: every rank
    copies its chunk into its slot of a symmetric buffer, a device-side barrier on the
    signal pads orders the ranks, and each rank pulls every peer's chunk straight out of the
    peer's memory (P2P loads over NVLink) into `recv`; a second barrier keeps a slot from
    being overwritten before all peers have read it.  No NCCL kernel, no host sync, and
    CUDA-graph capturable (the decode graph), so its latency is a few copy kernels and two
    signal exchanges.  The buffer is allocated and rendezvoused once, at construction
    (`capacity` bytes per rank: the largest per-rank chunk any call will move).  Needs an
    initialised torch.distributed process group with CUDA devices; multicast (NVLS) is used
    by torch when the fabric offers it."""

    def __init__(self, capacity: int, group=None):
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm_mem
        self.dist = dist
        self.group = group or dist.group.WORLD
        super().__init__(dist.get_world_size(self.group))
        self.rank_ = dist.get_rank(self.group)
        self.capacity = int(capacity)
        self.buf = symm_mem.empty(self.capacity, dtype=torch.uint8, device="cuda")
        self.hdl = symm_mem.rendezvous(self.buf, self.group.group_name)
        self.peers = [self.hdl.get_buffer(r, (self.capacity,), torch.uint8, 0)
                      for r in range(self.world)]

    def gather(self, rank, send, recv, nbytes, stream):
        if nbytes > self.capacity:
            raise ValueError(f"chunk of {nbytes} B exceeds the symmetric buffer ({self.capacity})")
        s = torch.cuda.ExternalStream(stream) if stream else torch.cuda.current_stream()
        with torch.cuda.stream(s):
            self.buf[:nbytes].copy_(self.view(send, nbytes))
            self.hdl.barrier(channel=0)
            for r in range(self.world):
                self.view(recv + r * nbytes, nbytes).copy_(self.peers[r][:nbytes])
            self.hdl.barrier(channel=1)

    def all_reduce(self, rank, send, recv, count, stream):
        """Exact int32 sum in rank order from the peers' slots (as gather, then a sum)."""
        nbytes = count * 4
        if nbytes > self.capacity:
            raise ValueError(f"{nbytes} B exceeds the symmetric buffer ({self.capacity})")
        s = torch.cuda.ExternalStream(stream) if stream else torch.cuda.current_stream()
        with torch.cuda.stream(s):
            self.buf[:nbytes].copy_(self.view(send, nbytes))
            self.hdl.barrier(channel=0)
            acc = self.peers[0][:nbytes].view(torch.int32).clone()
            for r in range(1, self.world):
                acc += self.peers[r][:nbytes].view(torch.int32)
            self.hdl.barrier(channel=1)
            self.view(recv, nbytes).view(torch.int32).copy_(acc)


class ThreadAllGather(AllGather):
    """`world` virtual ranks as host threads on one GPU (one stream each).  At a
    gather every rank records an event, meets the others at a host barrier,
    then copies all ranks' chunks on its own stream after their events; a
    second round of events keeps a rank from overwriting its send buffer before
    every peer has copied it."""

    def __init__(self, world: int):
        super().__init__(world)
        self.barrier = threading.Barrier(world)
        self.sends = [None] * world
        self.ev = [None] * world
        self.ev2 = [None] * world
        self.streams = {}
        self.lock = threading.Lock()
        self.slots = None   # all-reduce staging: [world][n] int32

    def gather(self, rank, send, recv, nbytes, stream):
        s = torch.cuda.ExternalStream(stream)
        e = torch.cuda.Event()
        e.record(s)
        self.sends[rank], self.ev[rank] = send, e
        self.barrier.wait()
        with torch.cuda.stream(s):
            for r in range(self.world):
                s.wait_event(self.ev[r])
                self.view(recv + r * nbytes, nbytes).copy_(self.view(self.sends[r], nbytes))
        e2 = torch.cuda.Event()
        e2.record(s)
        self.ev2[rank] = e2
        self.barrier.wait()
        for r in range(self.world):
            s.wait_event(self.ev2[r])
        self.barrier.wait()   # all waits enqueued before the slots are reused

    def all_reduce(self, rank, send, recv, count, stream):
        """Each rank stages its int32 vector, then every rank sums all of them
        (in rank order; integer sums are exact anyway) into its recv."""
        s = torch.cuda.ExternalStream(stream)
        with self.lock:
            if self.slots is None or self.slots.shape[1] < count:
                self.slots = torch.empty((self.world, count), dtype=torch.int32,
                                         device=torch.device("cuda"))
        self.barrier.wait()   # slots allocated before anyone stages
        slots = self.slots
        with torch.cuda.stream(s):
            slots[rank, :count].copy_(self.view(send, count * 4).view(torch.int32))
        e = torch.cuda.Event()
        e.record(s)
        self.ev[rank] = e
        self.barrier.wait()
        with torch.cuda.stream(s):
            for r in range(self.world):
                s.wait_event(self.ev[r])
            acc = slots[0, :count].clone()
            for r in range(1, self.world):
                acc += slots[r, :count]
            self.view(recv, count * 4).view(torch.int32).copy_(acc)
        e2 = torch.cuda.Event()
        e2.record(s)
        self.ev2[rank] = e2
        self.barrier.wait()
        for r in range(self.world):
            s.wait_event(self.ev2[r])
        self.barrier.wait()


def make_shard(gather: AllGather, rank: int, gather_q: bool = False,
               megatron: bool = False) -> "L.tern_shard":
    """gather_q: move o', x1 and p between ranks as int8 codes + row-moment
    partials instead of activations (tern.h tern_shard.gather_q).
    megatron: row-parallel o and down with exact int32 all-reduces (f1(ii))."""
    return L.tern_shard(rank, gather.world, gather.cb, C.c_void_p(rank), int(bool(gather_q)),
                        int(bool(megatron)), gather.cb_ar)
