"""oracle/ -- plain, slow, obviously-correct CPU implementation of the MoE layer step.

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py (its
cpu_baseline leg and `--impl reference`) may import, call, link or execute anything here.
The product path (paper_2404_19429_b200/) never imports it and shares no code with it.

Contents
  moe.py           routing, expert FFN, layer forward/backward over G simulated ranks (fp64)
  gate_logits.c    the fp32 fma-chain gate logits of DESIGN.md R1 (bit-exact routing)
  _native.py       gcc build + ctypes loader for gate_logits.c
  block.py         GPT-MoE block (LN, causal attention, MoE) and its pre-MoE partitioned form
Each function cites the PAPER.md passage it follows; DESIGN.md lists the readings (R1-R14)
taken where the paper is silent, and the CPU tests that pin every function.
"""
from . import moe  # noqa: F401
from . import block  # noqa: F401
from ._native import build  # noqa: F401
