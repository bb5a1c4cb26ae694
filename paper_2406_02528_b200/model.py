"""Python driver over the C ABI: packed weights, blocks and the L-block stack.

Everything numeric runs inside libtern.so; this module owns device buffers
(torch tensors), streams and CUDA graphs.  (P:409 block = token mixer +
channel mixer; P:698 prefill = pipelined mode, decode = fall-through mode.)
"""
from __future__ import annotations

import ctypes as C
import os

import torch

from . import _lib as L
from . import synth


class PackedWeight:
    """A fused group of n_seg ternary matrices packed 16 trits per word (a1).

    latents: list of fp32 [n_out][k] device tensors (one per segment)."""

    def __init__(self, latents, scales_in=None, expand=True):
        n_seg = len(latents)
        n_out, k = latents[0].shape
        dev = latents[0].device
        self.n_out, self.k, self.n_seg = int(n_out), int(k), n_seg
        self.n_rows = L.tern_packed_rows(self.n_out, n_seg)
        self.ldw = L.tern_packed_ldw(self.k)
        # K-block-major packed layout [Kp/128][n_rows][8] (include/tern.h)
        self.codes = torch.empty((self.ldw // 8, self.n_rows, 8), dtype=torch.int32, device=dev)
        self.scales = torch.empty(n_seg, dtype=torch.float32, device=dev)
        L.tern_codes_init(self.codes)
        for s, W in enumerate(latents):
            W = W.to(device=dev, dtype=torch.float32).contiguous()
            sin = None if scales_in is None else scales_in[s]
            L.tern_pack(W, self.codes, self.scales[s:s + 1], n_seg=n_seg, seg_idx=s, scale_in=sin)
        self.struct = L.tern_weight(self.codes.data_ptr(), self.scales.data_ptr(), self.n_out,
                                    self.k, self.ldw, self.n_seg, self.n_rows, None)
        self.e8 = None
        if expand:
            # u8 copy of the fields for the prefill GEMM's TMA path (4x the codes' bytes)
            self.e8 = torch.empty((self.n_rows, self.ldw * 16), dtype=torch.uint8, device=dev)
            L.tern_expand(self.struct, self.e8)
            self.struct.e8 = self.e8.data_ptr()

    @property
    def nbytes(self) -> int:
        return self.codes.numel() * 4


class Block:
    """One MatMul-free block: MLGRU token mixer + GLU channel mixer."""

    def __init__(self, latent: dict, d: int, l: int, gate=L.TERN_GATE_SIGMOID_H, eps=1e-6,
                 gains: dict | None = None, biases: dict | None = None, device="cuda",
                 shard=None, norm=L.TERN_NORM_RMS, num_chunks: int = 0):
        """shard = (rank, AllGather[, gather_q[, megatron]]) for a sharded block (shard.py);
        latent holds the FULL matrices, gains/biases this rank's slices.  norm: the
        norm in front of every BitLinear (TERN_NORM_RMS, or TERN_NORM_CENTERED =
        Alg. 1's centred form).  num_chunks: the prefill scan over time (tern.h
        tern_mlgru.num_chunks: 0 auto, 1 exact sequential, 4 or 8 chunked, reading C23)."""
        self.d, self.l = d, l
        dev = torch.device(device)
        lat = {k: v.to(dev) for k, v in latent.items()}
        sc = {k: None for k in lat}
        if shard is not None:
            from . import shard as S
            rank, gather = shard[0], shard[1]
            mega = len(shard) > 3 and bool(shard[3])
            sc = S.full_scales(lat, dev)
            lat = S.shard_latents(lat, d, l, gather.world, rank, megatron=mega)
        # which groups keep only the 2-bit codes (the prefill GEMM then unpacks B
        # tiles in shared memory instead of loading the u8 copy): debug knob
        packed_only = set(os.environ.get("TERN_PACKED_B", "").split(","))
        self.fcg = PackedWeight([lat["f"], lat["c"], lat["g"]],
                                None if sc["f"] is None else [sc["f"], sc["c"], sc["g"]],
                                expand="fcg" not in packed_only)
        self.o = PackedWeight([lat["o"]], None if sc["o"] is None else [sc["o"]],
                              expand="o" not in packed_only)
        self.gu = PackedWeight([lat["gate"], lat["up"]],
                               None if sc["gate"] is None else [sc["gate"], sc["up"]],
                               expand="gu" not in packed_only)
        self.down = PackedWeight([lat["down"]], None if sc["down"] is None else [sc["down"]],
                                 expand="down" not in packed_only)
        gains = gains or {}
        biases = biases or {}
        self._keep = []

        def dp(t):
            if t is None:
                return None
            t = t.to(device=dev, dtype=torch.float32).contiguous()
            self._keep.append(t)
            return t.data_ptr()

        bias_fcg = None
        if any(biases.get(k) is not None for k in ("f", "c", "g")):
            z = torch.zeros(self.fcg.n_out)
            bias_fcg = torch.cat([biases.get(k, z).float().cpu() for k in ("f", "c", "g")])
        self.mix = L.tern_mlgru(self.fcg.struct, self.o.struct, dp(gains.get("x")),
                                dp(gains.get("o")), dp(bias_fcg), dp(biases.get("o")), int(gate),
                                float(eps), int(norm), int(num_chunks))
        self.ch = L.tern_glu(self.gu.struct, self.down.struct, dp(gains.get("x1")),
                             dp(gains.get("p")), float(eps), int(norm))
        self.struct = L.tern_block(self.mix, self.ch, d, l)
        if shard is not None:
            from . import shard as S
            self.struct.shard = S.make_shard(shard[1], shard[0], *shard[2:4])

    @property
    def weight_bytes(self) -> int:
        return sum(w.nbytes for w in (self.fcg, self.o, self.gu, self.down))

    def scan_chunks(self, B: int, T: int) -> int:
        """The prefill scan's chunk count for B x T (1 = exact sequential; tern_mlgru_chunks)."""
        return int(L.load().tern_mlgru_chunks(C.byref(self.mix), B, T, self.d))

    def workspace_bytes(self, B: int, T: int, dtype: torch.dtype) -> int:
        return int(L.load().tern_block_workspace(C.byref(self.struct), B, T, L.dtype_code(dtype)))

    def ws_layout(self, B: int, T: int, dtype: torch.dtype) -> dict:
        t = L.tern_block_taps()
        L._check(L.load().tern_block_ws_layout(C.byref(self.struct), B, T, L.dtype_code(dtype),
                                               C.byref(t)), "tern_block_ws_layout")
        return {"fcg": t.fcg, "oprime": t.oprime, "x1": t.x1, "p": t.p}


class Stack:
    """L blocks; prefill over [B][T][d] and graph-captured decode steps."""

    def __init__(self, blocks, d: int, l: int, dtype: torch.dtype, device="cuda"):
        self.blocks = list(blocks)
        self.d, self.l, self.dtype = d, l, dtype
        self.device = torch.device(device)
        self._ws = None
        self._ws_bytes = 0
        self._graph = None
        self.gather = None   # shard.AllGather of a sharded stack

    def link_blocks(self):
        """Point each block's next_block hint at its successor (decode L2 prefetch)."""
        for a, b in zip(self.blocks, self.blocks[1:]):
            a.struct.next_block = C.addressof(b.struct)

    def _reg(self, *ts):
        if self.gather is not None:
            self.gather.register(*[t for t in ts if t is not None])

    @classmethod
    def random(cls, cfg: synth.Config, device="cuda", gate=L.TERN_GATE_SIGMOID_H, n_blocks=None,
               gen_device=None, keep_latents=0, shard=None, norm=L.TERN_NORM_RMS, num_chunks=0):
        """Build cfg's stack from seeded N(0, 0.02) latents (drawn per block on
        gen_device, packed on the GPU and dropped).  keep_latents=n keeps the
        first n blocks' latents on the host (for oracle parity)."""
        gen_device = gen_device or device
        g = synth.generator(cfg.seed, gen_device)
        blocks, kept = [], []
        for i in range(n_blocks if n_blocks is not None else cfg.L):
            lat = synth.latent_block(cfg.d, cfg.l, g, device=gen_device)
            if i < keep_latents:
                kept.append({k: v.cpu() for k, v in lat.items()})
            blocks.append(Block(lat, cfg.d, cfg.l, gate=gate, eps=cfg.eps, device=device,
                                shard=shard, norm=norm, num_chunks=num_chunks))
            del lat
        st = cls(blocks, cfg.d, cfg.l, synth.torch_dtype(cfg.dtype), device)
        st.gather = None if shard is None else shard[1]
        st.link_blocks()
        st.latents = kept
        st.generator = g
        return st

    @property
    def weight_bytes(self) -> int:
        return sum(b.weight_bytes for b in self.blocks)

    def workspace(self, B: int, T: int) -> torch.Tensor:
        need = max(b.workspace_bytes(B, T, self.dtype) for b in self.blocks)
        if self._ws is None or self._ws_bytes < need:
            self._ws = torch.empty(need, dtype=torch.uint8, device=self.device)
            self._ws_bytes = need
            self._reg(self._ws)
        return self._ws

    def new_state(self, B: int) -> list:
        """One fp32 state per block: [B][d], or [B][d/world] for a sharded stack."""
        w = self.gather.world if self.gather is not None else 1
        return [torch.zeros((B, self.d // w), dtype=torch.float32, device=self.device)
                for _ in self.blocks]

    def prefill(self, x: torch.Tensor, states: list, out: torch.Tensor | None = None,
                bufs=None) -> torch.Tensor:
        """x [B][T][d] -> y [B][T][d]; states (one fp32 [B][d] per block) updated."""
        B, T, d = x.shape
        ws = self.workspace(B, T)
        if bufs is None:
            bufs = (torch.empty_like(x), torch.empty_like(x))
        self._reg(x, out, *bufs)
        cur = x
        for i, blk in enumerate(self.blocks):
            nxt = bufs[i % 2] if (i < len(self.blocks) - 1 or out is None) else out
            L.block_prefill(blk.struct, cur, nxt, states[i], ws)
            cur = nxt
        return cur

    def prefill_sp(self, x: torch.Tensor, states: list, gather, rank: int,
                   out: torch.Tensor | None = None) -> torch.Tensor:
        """Sequence-parallel prefill (tern.h block_prefill_sp, reading C23): x is
        this rank's token slice [B][T_local][d] (shard.seq_slice); states start as the state
        of the whole sequence's start on every rank and end as the state after the whole
        sequence (identical on all ranks).  One all-gather of 2 B d floats per block."""
        B, T, d = x.shape
        world = gather.world
        dt = L.dtype_code(self.dtype)
        # workspace + ping-pong buffers, kept per (shape, rank): virtual ranks (threads)
        # may share one Stack, so each rank owns its own set
        key = (B, T, world, rank, x.dtype)
        cache = self.__dict__.setdefault("_sp_cache", {})
        if key not in cache:
            need = max(int(L.load().tern_block_prefill_sp_workspace(C.byref(b.struct), B, T, dt,
                                                                      world))
                       for b in self.blocks)
            cache[key] = (torch.empty(need, dtype=torch.uint8, device=x.device),
                          (torch.empty_like(x), torch.empty_like(x)))
        ws, bufs = cache[key]
        gather.register(ws, x, *bufs, *([out] if out is not None else []))
        sp = L.tern_seqpar(rank, world, gather.cb, C.c_void_p(rank))
        cur = x
        for i, blk in enumerate(self.blocks):
            nxt = bufs[i % 2] if (i < len(self.blocks) - 1 or out is None) else out
            L.block_prefill_sp(blk.struct, cur, nxt, states[i], sp, ws, B, T, self.dtype)
            cur = nxt
        return cur

    def _stack_struct(self):
        if getattr(self, "_blk_arr", None) is None:
            self._blk_arr = (L.tern_block * len(self.blocks))(*[b.struct for b in self.blocks])
        return self._blk_arr

    def prefill_host(self, xs_host: list, ys_host: list, before_step=None) -> None:
        """Serve a sequence of independent prefill requests host to host: each
        pinned [B][T][d] input in xs_host is copied to the device, run through
        the stack from h = 0, and its output copied into the pinned ys_host
        entry.  Copies run on their own streams, double-buffered, so request
        i+1's upload and request i-1's download overlap request i's compute.
        before_step(i), if given, is called before request i's compute is
        enqueued (bench.py flushes L2 there).  Returns when every output has
        landed on the host."""
        if not xs_host:
            return
        B, T, d = xs_host[0].shape
        main = torch.cuda.current_stream(self.device)
        up, down = torch.cuda.Stream(self.device), torch.cuda.Stream(self.device)
        xin = [torch.empty((B, T, d), dtype=self.dtype, device=self.device) for _ in range(2)]
        yout = [torch.empty_like(xin[0]) for _ in range(2)]
        bufs = (torch.empty_like(xin[0]), torch.empty_like(xin[0]))
        states = self.new_state(B)
        ev_in = [torch.cuda.Event() for _ in range(2)]
        ev_free = [torch.cuda.Event() for _ in range(2)]    # xin[k] consumed
        ev_out = [torch.cuda.Event() for _ in range(2)]
        ev_drained = [torch.cuda.Event() for _ in range(2)]  # yout[k] copied out
        for k in range(2):
            ev_free[k].record(main)
            ev_drained[k].record(main)
        for i, (xh, yh) in enumerate(zip(xs_host, ys_host)):
            k = i % 2
            with torch.cuda.stream(up):
                up.wait_event(ev_free[k])
                xin[k].copy_(xh, non_blocking=True)
                ev_in[k].record(up)
            main.wait_event(ev_in[k])
            main.wait_event(ev_drained[k])
            for h in states:
                h.zero_()
            if before_step is not None:
                before_step(i)
            fn = getattr(self, "prefill_host_fn", None)   # e.g. the sequence-parallel prefill
            if fn is not None:
                fn(xin[k], states, yout[k])
            else:
                self.prefill(xin[k], states, out=yout[k], bufs=bufs)
            ev_free[k].record(main)
            ev_out[k].record(main)
            with torch.cuda.stream(down):
                down.wait_event(ev_out[k])
                yh.copy_(yout[k], non_blocking=True)
                ev_drained[k].record(down)
        main.wait_stream(down)

    def decode(self, x: torch.Tensor, states: list, out: torch.Tensor | None = None,
               bufs=None, persistent: bool | None = None) -> torch.Tensor:
        """One decode step: x [B][d] -> y [B][d] through all blocks.

        persistent (default: self.persistent_decode, False): the whole step in
        one persistent launch (tern.h stack_decode) when the library supports
        the shape; otherwise (or False) one block_decode call per block.  The
        results are identical.  The per-block PDL launch chain is the default
        because it measured faster on B200."""
        B, d = x.shape
        if persistent is None:
            persistent = getattr(self, "persistent_decode", False)
        if persistent and self.gather is None and B > 0:
            arr = self._stack_struct()
            need = L.tern_stack_decode_workspace(arr, B, self.dtype)
            if getattr(self, "_sws", None) is None or self._sws.numel() < need:
                self._sws = torch.empty(need, dtype=torch.uint8, device=self.device)
            y = out if out is not None else torch.empty_like(x)
            st = L.stack_decode(arr, x, y, states, self._sws, allow_unsupported=True)
            if st == L.TERN_OK:
                self.last_decode_path = "persistent"
                return y
        self.last_decode_path = "per_block"
        ws = self.workspace(B, 1)
        if bufs is None:
            bufs = (torch.empty_like(x), torch.empty_like(x))
        self._reg(x, out, *bufs)
        cur = x
        for i, blk in enumerate(self.blocks):
            nxt = bufs[i % 2] if (i < len(self.blocks) - 1 or out is None) else out
            L.block_decode(blk.struct, cur, nxt, states[i], ws)
            cur = nxt
        return cur

    def capture_decode(self, B: int, states: list):
        """Capture one whole-stack decode step in a CUDA graph.  Returns
        (graph, x_in, y_out): copy the step input into x_in, replay, read y_out."""
        x_in = torch.zeros((B, self.d), dtype=self.dtype, device=self.device)
        y_out = torch.empty_like(x_in)
        bufs = (torch.empty_like(x_in), torch.empty_like(x_in))
        self.workspace(B, 1)
        s = torch.cuda.Stream(device=self.device)
        s.wait_stream(torch.cuda.current_stream())
        saved = [h.clone() for h in states]
        with torch.cuda.stream(s):
            self.decode(x_in, states, out=y_out, bufs=bufs)   # warm-up (sets attributes)
        torch.cuda.current_stream().wait_stream(s)
        for h, h0 in zip(states, saved):
            h.copy_(h0)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self.decode(x_in, states, out=y_out, bufs=bufs)
        self._graph_bufs = bufs
        return g, x_in, y_out
