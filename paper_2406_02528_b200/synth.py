"""Seeded synthetic inputs shared by the CUDA path's tests/bench and the oracle.

This module draws random numbers and nothing else: it holds none of the
method's arithmetic (no quantization, normalization, packing or recurrence),
so both sides may consume its buffers without sharing method code.

Recipe (BASELINE.json configs):
  * latent weights  W ~ N(0, 0.02) fp32, shape [out][in], drawn per block in
    the order f, c, g, o, gate, up, down (d->d x4, d->l x2, l->d);
  * hidden states   x ~ N(0, 1) fp32 [B][T][d] (cast to bf16 where the config
    says bf16 activations -- the cast is the R0 storage rounding);
  * one torch.Generator per config seeded with the config's seed; weights are
    drawn first, then the prefill input, then the decode inputs.
The paper's trained weights and datasets are not available (and not needed:
kernel cost does not depend on values); these stand in with the paper's shapes
 and BASELINE.json's distributions.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import torch

WEIGHT_STD = 0.02
WEIGHT_ORDER = ("f", "c", "g", "o", "gate", "up", "down")


@dataclass(frozen=True)
class Config:
    name: str
    L: int
    d: int
    l: int
    dtype: str            # "f32" or "bf16" activations
    seed: int
    prefill_B: int
    prefill_T: int
    decode_B: int
    decode_steps: int
    eps: float = 1e-6
    sweep: tuple = field(default_factory=tuple)   # c1 only: ((K, N), ...) and Ms


CONFIGS = {
    # BASELINE.json configs[0]: one block, fp32, d=256, l=688, batch 2 x 128, 16 decode steps
    "c0": Config("c0", 1, 256, 688, "f32", 0, 2, 128, 2, 16),
    # configs[1]: isolated BitLinear sweep, bf16 activations, seed 1
    "c1": Config("c1", 0, 0, 0, "bf16", 1, 0, 0, 0, 0,
                 sweep=(((1024, 1024), (2048, 5632), (5632, 2048)), (1, 16, 256, 4096, 16384))),
    # configs[2]: 370M shape, 24 blocks, d=1024, l=2816 (fp32, reading C18)
    "c2": Config("c2", 24, 1024, 2816, "f32", 2, 8, 2048, 1, 500),
    # configs[3]: 1.3B shape, bf16
    "c3": Config("c3", 24, 2048, 5632, "bf16", 3, 16, 2048, 64, 1000),
    # configs[4]: 2.7B shape, bf16
    "c4": Config("c4", 32, 2560, 6912, "bf16", 4, 32, 4096, 1, 100),
}


def generator(seed: int, device="cpu") -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed(int(seed))
    return g


def weight_shapes(d: int, l: int) -> dict:
    """[out][in] shapes of one block's seven latent matrices."""
    return {"f": (d, d), "c": (d, d), "g": (d, d), "o": (d, d),
            "gate": (l, d), "up": (l, d), "down": (d, l)}


def latent_block(d: int, l: int, gen: torch.Generator, device="cpu") -> dict:
    """Draw one block's latent fp32 weights N(0, 0.02) in WEIGHT_ORDER."""
    shapes = weight_shapes(d, l)
    return {k: torch.randn(shapes[k], generator=gen, device=device, dtype=torch.float32) * WEIGHT_STD
            for k in WEIGHT_ORDER}


def latent_matrix(n: int, k: int, gen: torch.Generator, device="cpu") -> torch.Tensor:
    return torch.randn((n, k), generator=gen, device=device, dtype=torch.float32) * WEIGHT_STD


def hidden(shape, gen: torch.Generator, dtype: str = "f32", device="cpu") -> torch.Tensor:
    """N(0,1) hidden states; bf16 configs store them as bf16 (R0)."""
    x = torch.randn(tuple(shape), generator=gen, device=device, dtype=torch.float32)
    return x.to(torch.bfloat16) if dtype == "bf16" else x


def torch_dtype(dtype: str):
    return torch.bfloat16 if dtype == "bf16" else torch.float32
