"""Seeded synthetic inputs for the CATS hot path -- shared by tests, bench.py and smoke().

This module holds NONE of the method's arithmetic (no SiLU, no threshold, no GEMV, no
quantile): it only draws random tensors with the shapes and value distributions of the
paper's workloads (DESIGN.md §4 "Input recipe"). Both the CUDA path and the oracle consume
the identical bytes it produces; neither side imports the other.

Recipe:
  * tokens x ~ N(0, 1)                        (heavy: Student-t_3 / sqrt(3))
  * W_gate rows ~ N(0, sigma_u^2 / d), sigma_u = 0.30, so the gate pre-activation of a
    Gaussian token is ~ N(0, 0.30^2) -- reproduces the paper's "70% <-> t ~ 0.15"
    (heavy: each row scaled by a per-neuron gain g_j ~ LogNormal(0, 0.5), RMS-normalised to 1,
    which makes masks correlated across tokens: "hot neurons")
  * W_up, W_down rows ~ N(0, 1/d)
  * all weights NEURON-MAJOR [m][d] (HF gate_proj.weight, up_proj.weight, down_proj.weight.T)
  * calibration activations: i.i.d. N(0, sigma^2) (heavy: sigma * t_3/sqrt(3)), rounded to
    the requested dtype; the quantile only depends on the multiset of bit patterns.
  * App. B projections: W input-major [d_in][d_out] ~ N(0, 1/d_in); attention inputs are tokens x
Seeds: 0 calibration, 1 decode tokens, 2/3/4 W_gate/W_up/W_down, 5 App. B W, +1000*layer per layer.
"""
from __future__ import annotations

import math

import torch

SIGMA_U = 0.30

MODELS = {
    # name: (d, m)  -- P:526-527 (Mistral-7B, Llama2-7B), BASELINE.json configs
    "toy": (64, 176),
    "mistral-7b": (4096, 14336),
    "llama2-7b": (4096, 11008),
    "llama2-13b": (5120, 13824),
}


def _gen(seed: int) -> torch.Generator:
    g = torch.Generator(device="cpu")
    g.manual_seed(int(seed))
    return g


def _student_t3(shape, g: torch.Generator) -> torch.Tensor:
    # t_3 = Z / sqrt(chi2_3 / 3); divided by sqrt(3) for unit variance
    z = torch.randn(shape, generator=g, dtype=torch.float32)
    chi = (torch.randn((3,) + tuple(shape), generator=g, dtype=torch.float32) ** 2).sum(0)
    return z / torch.sqrt(chi / 3.0) / math.sqrt(3.0)


def tokens(b: int, d: int, dtype=torch.bfloat16, seed: int = 1, heavy: bool = False) -> torch.Tensor:
    """Decode-step hidden states x [b][d]."""
    g = _gen(seed)
    x = _student_t3((b, d), g) if heavy else torch.randn((b, d), generator=g, dtype=torch.float32)
    return x.to(dtype).contiguous()


def mlp_weights(d: int, m: int, dtype=torch.bfloat16, layer: int = 0, heavy: bool = False,
                sigma_u: float = SIGMA_U):
    """(W_gate, W_up, W_down_nm), each neuron-major [m][d]."""
    base = 1000 * layer
    gg, gu, gd = _gen(2 + base), _gen(3 + base), _gen(4 + base)
    wg = torch.randn((m, d), generator=gg, dtype=torch.float32) * (sigma_u / math.sqrt(d))
    if heavy:
        gain = torch.exp(0.5 * torch.randn((m, 1), generator=gg, dtype=torch.float32))
        gain = gain / torch.sqrt((gain ** 2).mean())
        wg = wg * gain
    wu = torch.randn((m, d), generator=gu, dtype=torch.float32) / math.sqrt(d)
    wd = torch.randn((m, d), generator=gd, dtype=torch.float32) / math.sqrt(d)
    return wg.to(dtype).contiguous(), wu.to(dtype).contiguous(), wd.to(dtype).contiguous()


def attn_weights(d_in: int, d_out: int, dtype=torch.bfloat16, layer: int = 0):
    """App. B projection weights, INPUT-major [d_in][d_out] (q/k/v_proj.weight.T concatenated along
    d_out), rows ~ N(0, 1/d_in). Seed 5 + 1000*layer."""
    g = _gen(5 + 1000 * layer)
    w = torch.randn((d_in, d_out), generator=g, dtype=torch.float32) / math.sqrt(d_in)
    return w.to(dtype).contiguous()


def calib_acts(n: int, dtype=torch.bfloat16, seed: int = 0, sigma: float = SIGMA_U, heavy: bool = False,
               device="cpu", chunk: int = 1 << 28) -> torch.Tensor:
    """n calibration activation values (1-D), generated in chunks so n may be ~1e10 on a GPU."""
    out = torch.empty(n, dtype=dtype, device=device)
    g = torch.Generator(device=device)
    g.manual_seed(int(seed))
    for s in range(0, n, chunk):
        e = min(n, s + chunk)
        if heavy:
            z = torch.randn(e - s, generator=g, device=device, dtype=torch.float32)
            chi = torch.zeros_like(z)
            for _ in range(3):
                chi += torch.randn(e - s, generator=g, device=device, dtype=torch.float32) ** 2
            v = z / torch.sqrt(chi / 3.0) / math.sqrt(3.0)
        else:
            v = torch.randn(e - s, generator=g, device=device, dtype=torch.float32)
        out[s:e] = (v * sigma).to(dtype)
    return out


def bf16_bits(t: torch.Tensor):
    """numpy uint16 view of a CPU bfloat16 tensor (what the oracle takes)."""
    assert t.dtype == torch.bfloat16
    return t.detach().cpu().contiguous().view(torch.int16).numpy().view("uint16")


def to_oracle(t: torch.Tensor):
    """numpy array in the oracle's input convention (float32, or uint16 bf16 bits)."""
    if t.dtype == torch.bfloat16:
        return bf16_bits(t)
    return t.detach().cpu().contiguous().to(torch.float32).numpy()
