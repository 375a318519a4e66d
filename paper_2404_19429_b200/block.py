"""Thin Python binding of the GPT-MoE block (include/lancet_block.h).

Argument marshalling only: LN, the projections, attention and the MoE layer all run in
liblancet_moe.so's kernels.  The block's MoE layer is a peer-transport push context
(`Block.moe`, a borrowed lancet.Context: counts, timeline, flags, and the MoE backward)."""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import torch

from . import lancet as L

_BLOCK_SIG = {
    "lancet_block_create_peer": None,
    "lancet_block_moe": None,
    "lancet_block_destroy": None,
    "lancet_block_forward": None,
    "lancet_block_debug_copy": None,
    "lancet_block_backward": None,
    "lancet_block_forward_stack": None,
}
EXPORTS = list(_BLOCK_SIG)


class _BlockConfig(ctypes.Structure):
    _fields_ = [("moe", L._Config), ("n_heads", ctypes.c_int32), ("seq_len", ctypes.c_int32),
                ("max_capacity_factor", ctypes.c_double)]


_loaded = False


def _lib():
    global _loaded
    lib = L.load_library()
    if not _loaded:
        P, I32 = ctypes.c_void_p, ctypes.c_int32
        lib.lancet_block_create_peer.argtypes = [ctypes.POINTER(P), I32, I32, I32, ctypes.POINTER(_BlockConfig)]
        lib.lancet_block_create_peer.restype = I32
        lib.lancet_block_moe.argtypes = [P]
        lib.lancet_block_moe.restype = P
        lib.lancet_block_destroy.argtypes = [P]
        lib.lancet_block_destroy.restype = I32
        lib.lancet_block_forward.argtypes = [P] + [P] * 10 + [I32, I32, ctypes.c_double, I32, P, P]
        lib.lancet_block_forward.restype = I32
        lib.lancet_block_forward_stack.argtypes = [P, I32, P, P, I32, I32, ctypes.c_double, I32, P, P]
        lib.lancet_block_forward_stack.restype = I32
        lib.lancet_block_backward.argtypes = [P] * 13
        lib.lancet_block_backward.restype = I32
        lib.lancet_block_debug_copy.argtypes = [P, I32, P, ctypes.c_size_t]
        lib.lancet_block_debug_copy.restype = I32
        _loaded = True
    return lib


@dataclass
class BlockConfig:
    moe: L.LayerConfig
    n_heads: int
    seq_len: int
    max_capacity_factor: float = 2.0

    def _c(self) -> _BlockConfig:
        return _BlockConfig(self.moe._c(), self.n_heads, self.seq_len, float(self.max_capacity_factor))


PARAMS = ("ln1_g", "ln1_b", "w_qkv", "w_o", "ln2_g", "ln2_b", "wg", "w1", "w2")


class Block:
    """One rank's lancet_block (world 1: a one-rank peer group; world > 1: the blobs are
    all-gathered over the torch process group `pg`)."""

    def __init__(self, cfg: BlockConfig, world: int = 1, rank: int = 0, device: int | None = None, pg=None):
        import torch.distributed as dist
        lib = _lib()
        self.cfg = cfg
        self.world, self.rank = world, rank
        self.device = torch.cuda.current_device() if device is None else device
        self._p = ctypes.c_void_p()
        ok = lib.lancet_block_create_peer(ctypes.byref(self._p), world, rank, self.device, ctypes.byref(cfg._c())) == 0
        if world > 1:
            flags = [None] * world
            dist.all_gather_object(flags, bool(ok), group=pg)
            ok = all(flags)
        if not ok:
            msg = lib.lancet_last_error(None)
            self.close()
            raise L.LancetError(6, f"block creation failed on some rank: {msg.decode() if msg else ''}")
        moe = L.Context.__new__(L.Context)
        moe.cfg, moe.world, moe.rank, moe.device = cfg.moe, world, rank, self.device
        moe._p = ctypes.c_void_p(lib.lancet_block_moe(self._p))
        moe._borrowed = True
        moe.E_l = cfg.moe.n_experts // world
        moe._last = None
        self.moe = moe
        nb = lib.lancet_peer_blob_bytes()
        blob = ctypes.create_string_buffer(nb)
        L._check(lib.lancet_peer_export(moe._p, blob), moe._p)
        blobs = [bytes(blob.raw)]
        if world > 1:
            blobs = [None] * world
            dist.all_gather_object(blobs, bytes(blob.raw), group=pg)
        L._check(lib.lancet_peer_import(moe._p, ctypes.create_string_buffer(b"".join(blobs), nb * world)), moe._p)
        self._last = None

    def close(self):
        if self._p:
            _lib().lancet_block_destroy(self._p)
            self._p = ctypes.c_void_p()
            if hasattr(self, "moe"):
                self.moe._p = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def forward(self, x, p: dict, k: int, capacity_factor: float, n_chunks: int, out=None, stream=None):
        """out = h + MoE(LN2(h)), h = x + Attn(LN1(x)).  p: the PARAMS tensors (ln* fp32 [d],
        w_qkv [3d][d], w_o [d][d] bf16, wg [d][E] fp32, w1 [E_l][f][d], w2 [E_l][d][f] bf16)."""
        T = x.shape[0]
        out = torch.empty_like(x) if out is None else out
        st = _lib().lancet_block_forward(self._p, L._ptr(x), *[L._ptr(p[n]) for n in PARAMS], T, k,
                                         float(capacity_factor), n_chunks, L._ptr(out), L._stream(stream))
        L._check(st, self.moe._p)
        self._last = (x, p)
        self._k = k
        self.moe._last = (None, p["wg"], p["w1"], p["w2"])     # the MoE layer's backward
        self.moe._last_n = n_chunks
        return out

    def backward(self, dout, stream=None):
        """Gradients of <dout, out> of the last forward: dict(dx, dln1_g, dln1_b, dw_qkv, dw_o,
        dln2_g, dln2_b, dwg, dw1, dw2)."""
        x, p = self._last
        dev = dout.device
        f32 = torch.float32
        g = dict(dx=torch.empty_like(dout), dln1_g=torch.empty(p["ln1_g"].shape, dtype=f32, device=dev),
                 dln1_b=torch.empty(p["ln1_b"].shape, dtype=f32, device=dev),
                 dw_qkv=torch.empty(p["w_qkv"].shape, dtype=f32, device=dev),
                 dw_o=torch.empty(p["w_o"].shape, dtype=f32, device=dev),
                 dln2_g=torch.empty(p["ln2_g"].shape, dtype=f32, device=dev),
                 dln2_b=torch.empty(p["ln2_b"].shape, dtype=f32, device=dev),
                 dwg=torch.empty(p["wg"].shape, dtype=f32, device=dev),
                 dw1=torch.empty(p["w1"].shape, dtype=f32, device=dev),
                 dw2=torch.empty(p["w2"].shape, dtype=f32, device=dev))
        order = ("dx", "dln1_g", "dln1_b", "dw_qkv", "dw_o", "dln2_g", "dln2_b", "dwg", "dw1", "dw2")
        st = _lib().lancet_block_backward(self._p, L._ptr(dout), *[L._ptr(g[n]) for n in order], L._stream(stream))
        L._check(st, self.moe._p)
        return g

    def debug(self, which: str, T: int):
        """An intermediate of the last forward as a torch CPU tensor: h, u, att, qkv, a1 (bf16),
        lse (fp32 [H][T], log2 domain), idx / slot (int32 [T][k], the MoE layer's routing)."""
        d = self.cfg.moe.d_model
        k = self._k
        shapes = {"h": (0, (T, d)), "u": (1, (T, d)), "att": (2, (T, d)), "qkv": (3, (T, 3 * d)),
                  "a1": (4, (T, d)), "lse": (5, (self.cfg.n_heads, T)), "idx": (6, (T, k)), "slot": (7, (T, k)),
                  "dqkv": (8, (T, 3 * d)), "dh": (9, (T, d)), "datt": (10, (T, d))}
        w, shape = shapes[which]
        dt = {"lse": torch.float32, "idx": torch.int32, "slot": torch.int32}.get(which, torch.bfloat16)
        t = torch.empty(shape, dtype=dt)
        L._check(_lib().lancet_block_debug_copy(self._p, w, ctypes.c_void_p(t.data_ptr()),
                                                t.numel() * t.element_size()), self.moe._p)
        return t


def forward_stack(blocks, x, params, k: int, capacity_factor: float, n_chunks: int, outs=None, stream=None):
    """lancet_block_forward_stack: blocks[l] with params[l] (PARAMS dicts); returns the list of
    every block's output (outs[l] = block l's out, block l+1's input)."""
    nl = len(blocks)
    T = x.shape[0]
    outs = [torch.empty_like(x) for _ in range(nl)] if outs is None else outs
    bp = (ctypes.c_void_p * nl)(*[b._p.value for b in blocks])
    pp = (ctypes.c_void_p * (9 * nl))(*[params[l][n].data_ptr() for l in range(nl) for n in PARAMS])
    op = (ctypes.c_void_p * nl)(*[o.data_ptr() for o in outs])
    st = _lib().lancet_block_forward_stack(bp, nl, ctypes.c_void_p(x.data_ptr()), pp, T, k,
                                           float(capacity_factor), n_chunks, op, L._stream(stream))
    L._check(st, blocks[0].moe._p)
    for l, b in enumerate(blocks):
        b._last = (x if l == 0 else outs[l - 1], params[l])
        b._k = k
        b.moe._last = (None, params[l]["wg"], params[l]["w1"], params[l]["w2"])
        b.moe._last_n = n_chunks
    return outs
