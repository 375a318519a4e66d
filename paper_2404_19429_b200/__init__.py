"""paper_2404_19429_b200 -- a B200-native (sm_100a) implementation of the hot path of Lancet
(arXiv 2404.19429): the expert-parallel MoE layer step whose all-to-all is pipelined over
batch chunks and overlapped with expert computation and weight-gradient GEMMs.

The product is the C-ABI library liblancet_moe.so (include/lancet_moe.h); `lancet` is its
thin ctypes binding.  Build with `python -m paper_2404_19429_b200.build`.
"""
from .lancet import (Context, LayerConfig, LocalGroup, LancetError, load_library,  # noqa: F401
                     exposed_comm_us, FLAG_RENORMALIZE, FLAG_TIMELINE, FLAG_SERIAL,
                     FLAG_SIMT_GEMM, FLAG_NO_DW_OVERLAP, FLAG_NO_SIDE_STREAM, FLAG_GEMM_MULTICAST,
                     FLAG_UNFUSED_GATE_BWD, FLAG_NO_PDL, FLAG_FORCE_EP, FLAG_GATE_BPR, FLAG_DEFER_DW, FLAG_GATE_RANDOM, FLAG_PEER_PUSH,
                     FLAG_NO_COMM, FLAG_CHUNK_LAUNCHES,
                     dw_schedule, stack_dw_plan,
                     EXPORTS, LIB_PATH)
