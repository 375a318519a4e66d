"""Seeded synthetic inputs for the MoE layer step (shared by the oracle tests, the GPU
parity tests and bench.py).

This module holds NONE of the method's arithmetic: it only draws random numbers and
rounds them to the storage precision of the inputs.  Both the oracle (oracle/) and the
CUDA path (paper_2404_19429_b200/) consume its arrays; neither imports the other.

Recipe (SURVEY.md §8(d) "Configs as concrete synthetic inputs"):
  * numpy PCG64, seed = base + 1000*rank + tensor_id for per-rank tensors (x, dy),
    seed = base + tensor_id (>= 100) for replicated / global tensors (u, Wg, W1, W2).
  * tokens       x  = bf16(z + u),   z ~ N(0, I_d),  u a fixed unit vector
                    (LayerNorm-output-like scale; "B x S" tokens of width d).
  * gate         Wg = G0/sqrt(d) + u (x) b,  G0 ~ N(0,1),  b_e = linspace(-beta, beta, E)
                    (beta = routing skew; 0 balanced, 0.25 throughput default,
                     0.5 parity default, which makes capacity bind and drop tokens).
  * experts      W1[e] ~ N(0, 0.02^2) of shape [f, d],  W2[e] ~ N(0, 0.02^2) of shape [d, f]
                    (GPT-2 init scale; expert e's weights depend only on (base, e), so the
                     same global experts can be placed on any number of ranks).
  * upstream grad dy ~ N(0, 1).
All floating arrays are returned as numpy float32; in bf16 mode their values are exactly
representable in bfloat16 (round-to-nearest-even), so the GPU side converts them losslessly.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

__all__ = [
    "LayerShape", "round_to_bf16", "gen_u", "gen_tokens", "gen_gate", "gen_experts",
    "gen_dy", "gen_rank_inputs", "TINY", "CFG2", "BlockShape", "CFG4", "TINY_BLOCK",
    "gen_block_params", "gen_block_rank_inputs",
]

_TID_X, _TID_DY = 1, 2
_TID_U, _TID_WG, _TID_W1, _TID_W2 = 100, 101, 102, 103
_TID_LN1G, _TID_LN1B, _TID_LN2G, _TID_LN2B, _TID_WQKV, _TID_WO = 104, 105, 106, 107, 108, 109


@dataclass(frozen=True)
class LayerShape:
    """Per-rank shape of one MoE layer (SURVEY.md §8 notation)."""
    T: int            # tokens per rank
    d: int            # d_model
    f: int            # ffn width
    E: int            # experts in total
    G: int            # ranks
    k: int            # top-k
    cf: float         # capacity factor
    n_chunks: int     # batch chunks

    @property
    def E_l(self) -> int:
        return self.E // self.G


@dataclass(frozen=True)
class BlockShape:
    """Per-rank shape of one GPT-MoE block (BASELINE.json configs[3]): T = n_seq * seq_len
    tokens per rank, causal self-attention with n_heads heads, then the MoE layer."""
    n_seq: int        # sequences per rank (the batch dimension B)
    seq_len: int      # S
    d: int            # d_model
    n_heads: int
    f: int            # expert ffn width
    E: int            # experts in total
    G: int            # ranks
    k: int            # top-k (1: Switch)
    cf: float
    n_chunks: int     # batch chunks (whole sequences; n_chunks divides n_seq)

    @property
    def T(self) -> int:
        return self.n_seq * self.seq_len

    @property
    def E_l(self) -> int:
        return self.E // self.G

    @property
    def head_dim(self) -> int:
        return self.d // self.n_heads

    def layer(self) -> LayerShape:
        return LayerShape(T=self.T, d=self.d, f=self.f, E=self.E, G=self.G, k=self.k, cf=self.cf,
                          n_chunks=self.n_chunks)


# BASELINE.json configs[0] (64 tokens over 2 ranks) and configs[1] (GPT-MoE layer).
TINY = LayerShape(T=32, d=16, f=32, E=4, G=2, k=2, cf=1.25, n_chunks=2)
CFG2 = LayerShape(T=16384, d=1024, f=4096, E=8, G=8, k=2, cf=1.25, n_chunks=4)
# configs[3]: full GPT-MoE block, d = 2048, 16 heads, 32 experts (4 per GPU), Switch top-1,
# seq 1024 x 8 sequences per GPU; f = 4 d (SURVEY.md §8(d) "Config 4")
CFG4 = BlockShape(n_seq=8, seq_len=1024, d=2048, n_heads=16, f=8192, E=32, G=8, k=1, cf=1.25, n_chunks=4)
# a small block for the CPU oracle tests (head_dim 128 as on the GPU path)
TINY_BLOCK = BlockShape(n_seq=4, seq_len=32, d=256, n_heads=2, f=256, E=4, G=2, k=1, cf=1.25, n_chunks=2)


def round_to_bf16(a: np.ndarray) -> np.ndarray:
    """Round float32 values to the nearest bfloat16 (ties to even); returns float32.

    Storage-precision conversion of generated inputs only (NaN/Inf are never generated)."""
    a = np.ascontiguousarray(a, dtype=np.float32)
    b = a.view(np.uint32).astype(np.uint64)
    lsb = (b >> 16) & 1
    b = (b + 0x7FFF + lsb) & 0xFFFF0000
    return b.astype(np.uint32).view(np.float32)


def _rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed))


def _store(a: np.ndarray, dtype: str) -> np.ndarray:
    a = a.astype(np.float32)
    if dtype == "bf16":
        return round_to_bf16(a)
    if dtype == "fp32":
        return a
    raise ValueError(f"dtype must be 'bf16' or 'fp32', got {dtype!r}")


def gen_u(base: int, d: int) -> np.ndarray:
    """The fixed unit vector u (float64, shape [d])."""
    v = _rng(base + _TID_U).standard_normal(d)
    return v / np.linalg.norm(v)


def gen_tokens(base: int, rank: int, T: int, d: int, dtype: str = "bf16") -> np.ndarray:
    """x = z + u for rank `rank`; shape [T, d]."""
    z = _rng(base + 1000 * rank + _TID_X).standard_normal((T, d), dtype=np.float32)
    return _store(z + gen_u(base, d)[None, :].astype(np.float32), dtype)


def gen_gate(base: int, d: int, E: int, beta: float) -> np.ndarray:
    """Wg = G0/sqrt(d) + u (x) b, float32 [d, E] (the router is kept in fp32, R1)."""
    g0 = _rng(base + _TID_WG).standard_normal((d, E))
    b = np.linspace(-beta, beta, E) if E > 1 else np.zeros(1)
    return (g0 / math.sqrt(d) + np.outer(gen_u(base, d), b)).astype(np.float32)


def gen_experts(base: int, E: int, d: int, f: int, dtype: str = "bf16",
                experts: range | None = None, std: float = 0.02):
    """Global expert weights W1 [E', f, d], W2 [E', d, f] for experts in `experts`."""
    experts = range(E) if experts is None else experts
    w1 = np.empty((len(experts), f, d), dtype=np.float32)
    w2 = np.empty((len(experts), d, f), dtype=np.float32)
    for i, e in enumerate(experts):
        w1[i] = _rng(base + _TID_W1 + 7919 * (e + 1)).standard_normal((f, d), dtype=np.float32) * std
        w2[i] = _rng(base + _TID_W2 + 7919 * (e + 1)).standard_normal((d, f), dtype=np.float32) * std
    return _store(w1, dtype), _store(w2, dtype)


def gen_dy(base: int, rank: int, T: int, d: int, dtype: str = "bf16") -> np.ndarray:
    return _store(_rng(base + 1000 * rank + _TID_DY).standard_normal((T, d), dtype=np.float32), dtype)


def gen_rank_inputs(base: int, rank: int, shape: LayerShape, beta: float = 0.5,
                    dtype: str = "bf16", with_dy: bool = True) -> dict:
    """All inputs rank `rank` passes to lancet_moe_forward/backward, as numpy arrays."""
    E_l = shape.E_l
    w1, w2 = gen_experts(base, shape.E, shape.d, shape.f, dtype,
                         experts=range(rank * E_l, (rank + 1) * E_l))
    out = dict(x=gen_tokens(base, rank, shape.T, shape.d, dtype),
               wg=gen_gate(base, shape.d, shape.E, beta), w1=w1, w2=w2)
    if with_dy:
        out["dy"] = gen_dy(base, rank, shape.T, shape.d, dtype)
    return out


def gen_block_params(base: int, d: int, dtype: str = "bf16", std: float = 0.02) -> dict:
    """Non-MoE parameters of a GPT-MoE block: LayerNorm gains / biases (fp32; gain 1 + 0.1 z,
    bias 0.1 z), the fused QKV projection W_qkv [3d, d] (rows: q | k | v, head h at rows
    h*hd .. h*hd+hd-1 of each) and the output projection W_o [d, d], both N(0, std^2)
    (GPT-2 init scale), stored in `dtype`."""
    def ln(tid):
        return (1.0 + 0.1 * _rng(base + tid).standard_normal(d)).astype(np.float32)

    def bias(tid):
        return (0.1 * _rng(base + tid).standard_normal(d)).astype(np.float32)
    w_qkv = _rng(base + _TID_WQKV).standard_normal((3 * d, d), dtype=np.float32) * std
    w_o = _rng(base + _TID_WO).standard_normal((d, d), dtype=np.float32) * std
    return dict(ln1_g=ln(_TID_LN1G), ln1_b=bias(_TID_LN1B), ln2_g=ln(_TID_LN2G), ln2_b=bias(_TID_LN2B),
                w_qkv=_store(w_qkv, dtype), w_o=_store(w_o, dtype))


def gen_block_rank_inputs(base: int, rank: int, shape: BlockShape, beta: float = 0.5,
                          dtype: str = "bf16", with_dy: bool = True) -> dict:
    """Everything rank `rank` passes to lancet_block_forward / backward (numpy arrays)."""
    out = gen_rank_inputs(base, rank, shape.layer(), beta, dtype, with_dy)
    out.update(gen_block_params(base, shape.d, dtype))
    return out
