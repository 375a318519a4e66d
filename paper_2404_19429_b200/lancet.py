"""Thin Python binding of liblancet_moe.so (include/lancet_moe.h).

Argument marshalling only: every step of the MoE layer runs in the library's CUDA kernels.
torch provides device memory, streams and (for world > 1) the process group used to
broadcast the NCCL unique id.  There is no fallback: if the shared library is missing or the
device is not a B200 the calls raise.
"""
from __future__ import annotations

import ctypes
import os
import threading
from dataclasses import dataclass

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
# LANCET_LIB: alternative build of the same library (A/B experiments); default the in-tree build
LIB_PATH = os.environ.get("LANCET_LIB") or os.path.join(_HERE, "liblancet_moe.so")

STATUS = {0: "OK", 1: "ERR_ARG", 2: "ERR_CUDA", 3: "ERR_NCCL", 4: "ERR_NOMEM", 5: "ERR_STATE",
          6: "ERR_UNSUPPORTED"}
DTYPES = {"bf16": 0, "fp32": 1}
ACTS = {"gelu_tanh": 0, "relu": 1, "identity_expert": 2}
FLAG_RENORMALIZE, FLAG_TIMELINE, FLAG_SERIAL, FLAG_SIMT_GEMM, FLAG_NO_DW_OVERLAP = 1, 2, 4, 8, 16
FLAG_NO_SIDE_STREAM = 32
FLAG_GEMM_MULTICAST = 64
FLAG_UNFUSED_GATE_BWD = 128
FLAG_NO_PDL = 256
FLAG_FORCE_EP = 512
FLAG_TIMELINE_GEMM_ONLY = 1024
FLAG_GATE_BPR = 2048
FLAG_DEFER_DW = 4096
FLAG_GATE_RANDOM = 8192
FLAG_PEER_PUSH = 16384
FLAG_NO_COMM = 32768          # timing only: the data exchanges are skipped (results are wrong)
FLAG_CHUNK_LAUNCHES = 65536   # push mode: one GEMM launch per chunk (A/B of the device-side pipeline)
# LANCET_EXTRA_FLAGS: OR'ed into every context's flags (e.g. run the test suite under PDL)
EXTRA_FLAGS = int(os.environ.get("LANCET_EXTRA_FLAGS", "0"), 0)

EXPORTS = ["lancet_abi_version", "lancet_last_error", "lancet_nccl_unique_id", "lancet_create",
           "lancet_local_group_create", "lancet_local_group_destroy", "lancet_create_local",
           "lancet_destroy", "lancet_set_flags", "lancet_moe_forward", "lancet_moe_backward",
           "lancet_get_counts", "lancet_timeline_begin", "lancet_last_timeline", "lancet_debug_copy",
           "lancet_workspace_bytes", "lancet_launch_counts", "lancet_plan_exchange",
           "lancet_create_peer", "lancet_peer_blob_bytes", "lancet_peer_export", "lancet_peer_import",
           "lancet_moe_backward_dw", "lancet_set_dw_fillers", "lancet_dw_schedule", "lancet_stack_dw_plan",
           "lancet_set_gate_seed", "lancet_set_peer_timeout_ms", "lancet_peer_abort", "lancet_peer_status",
           "lancet_tune_chunks", "lancet_moe_forward_partitioned", "lancet_nccl_registered"]


class LancetError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class _Config(ctypes.Structure):
    _fields_ = [("d_model", ctypes.c_int32), ("d_ffn", ctypes.c_int32),
                ("n_experts", ctypes.c_int32), ("max_tokens", ctypes.c_int32),
                ("max_k", ctypes.c_int32), ("max_chunks", ctypes.c_int32),
                ("dtype", ctypes.c_int32), ("act", ctypes.c_int32), ("flags", ctypes.c_uint32),
                ("gemm_sms", ctypes.c_int32)]


class _OpRecord(ctypes.Structure):
    _fields_ = [("name", ctypes.c_char * 24), ("lane", ctypes.c_int32), ("chunk", ctypes.c_int32),
                ("start_us", ctypes.c_float), ("end_us", ctypes.c_float)]


_lib = None
_lib_lock = threading.Lock()


def load_library(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load liblancet_moe.so (build it with `python -m paper_2404_19429_b200.build`)."""
    global _lib
    with _lib_lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise RuntimeError(f"{path} is missing: run `python -m paper_2404_19429_b200.build` "
                               "(there is no CPU fallback)")
        lib = ctypes.CDLL(path)
        P, I32, U32, F32 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_uint32, ctypes.c_float
        sig = {
            "lancet_abi_version": ([], I32),
            "lancet_last_error": ([P], ctypes.c_char_p),
            "lancet_nccl_unique_id": ([P], I32),
            "lancet_create": ([ctypes.POINTER(P), I32, I32, I32, P, ctypes.POINTER(_Config)], I32),
            "lancet_local_group_create": ([ctypes.POINTER(P), I32], I32),
            "lancet_local_group_destroy": ([P], I32),
            "lancet_create_local": ([ctypes.POINTER(P), P, I32, I32, ctypes.POINTER(_Config)], I32),
            "lancet_create_peer": ([ctypes.POINTER(P), I32, I32, I32, ctypes.POINTER(_Config)], I32),
            "lancet_peer_blob_bytes": ([], ctypes.c_size_t),
            "lancet_peer_export": ([P, P], I32),
            "lancet_peer_import": ([P, P], I32),
            "lancet_destroy": ([P], I32),
            "lancet_set_flags": ([P, U32], I32),
            "lancet_moe_forward": ([P, P, P, P, P, I32, I32, ctypes.c_double, I32, P, P, P, P, P], I32),
            "lancet_moe_backward": ([P, P, P, P, P, P, P], I32),
            "lancet_moe_forward_partitioned": ([P, P, P, P, P, I32, I32, ctypes.c_double, I32, P, P, P, P, P, P],
                                               I32),
            "lancet_get_counts": ([P, P, P, P], I32),
            "lancet_timeline_begin": ([P, P], I32),
            "lancet_last_timeline": ([P, ctypes.POINTER(_OpRecord), I32, ctypes.POINTER(I32)], I32),
            "lancet_debug_copy": ([P, I32, P, ctypes.c_size_t], I32),
            "lancet_workspace_bytes": ([P, ctypes.POINTER(ctypes.c_size_t)], I32),
            "lancet_nccl_registered": ([P, ctypes.POINTER(I32)], I32),
            "lancet_launch_counts": ([P, ctypes.POINTER(I32), ctypes.POINTER(I32)], I32),
            "lancet_plan_exchange": ([I32, I32, I32, P, P, P, P, P, P, P, ctypes.POINTER(I32)], I32),
            "lancet_moe_backward_dw": ([P, I32, P], I32),
            "lancet_set_gate_seed": ([P, ctypes.c_uint64], I32),
            "lancet_set_dw_fillers": ([P, I32, P, P, P], I32),
            "lancet_dw_schedule": ([I32, P, P, I32, P, P], I32),
            "lancet_stack_dw_plan": ([I32, I32, P, P, P, P], I32),
            "lancet_set_peer_timeout_ms": ([P, ctypes.c_int64], I32),
            "lancet_peer_abort": ([P], I32),
            "lancet_peer_status": ([P], I32),
        }
        for name, (args, res) in sig.items():
            f = getattr(lib, name)
            f.argtypes, f.restype = args, res
        _lib = lib
        return lib


def _check(st: int, ctx_ptr=None):
    if st != 0:
        msg = load_library().lancet_last_error(ctx_ptr)
        raise LancetError(st, msg.decode() if msg else "")


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(stream) -> ctypes.c_void_p:
    s = torch.cuda.current_stream() if stream is None else stream
    return ctypes.c_void_p(s.cuda_stream)


@dataclass
class LayerConfig:
    d_model: int
    d_ffn: int
    n_experts: int
    max_tokens: int
    max_k: int = 2
    max_chunks: int = 8
    dtype: str = "bf16"
    act: str = "gelu_tanh"
    flags: int = 0
    gemm_sms: int = 0

    def _c(self) -> _Config:
        return _Config(self.d_model, self.d_ffn, self.n_experts, self.max_tokens, self.max_k,
                       self.max_chunks, DTYPES[self.dtype], ACTS[self.act],
                       self.flags | EXTRA_FLAGS, self.gemm_sms)

    @property
    def torch_dtype(self):
        return torch.bfloat16 if self.dtype == "bf16" else torch.float32


class LocalGroup:
    """G simulated ranks in one process on one device (lancet_local_group)."""

    def __init__(self, world: int):
        lib = load_library()
        self.world = world
        self._p = ctypes.c_void_p()
        _check(lib.lancet_local_group_create(ctypes.byref(self._p), world))

    def close(self):
        if self._p:
            load_library().lancet_local_group_destroy(self._p)
            self._p = ctypes.c_void_p()


def plan_exchange(G: int, E_l: int, n: int, send_counts, recv_counts) -> dict:
    """Host-side exchange plan (lancet_plan_exchange) as numpy arrays."""
    import numpy as np
    E = G * E_l
    send = np.ascontiguousarray(send_counts, dtype=np.int32).reshape(E, n)
    recv = np.ascontiguousarray(recv_counts, dtype=np.int32).reshape(G, E_l, n)
    out = dict(send_off=np.zeros(E, np.int32), S=np.zeros((E, n + 1), np.int32),
               grp_rows=np.zeros((n, E_l), np.int32), grp_off=np.zeros((n, E_l), np.int32),
               src_off=np.zeros((G, E_l, n), np.int32))
    tot = ctypes.c_int32()
    p = lambda a: a.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
    _check(load_library().lancet_plan_exchange(G, E_l, n, p(send), p(recv), p(out["send_off"]), p(out["S"]),
                                               p(out["grp_rows"]), p(out["grp_off"]), p(out["src_off"]),
                                               ctypes.byref(tot)))
    out["total_rows"] = tot.value
    return out


def dw_schedule(kinds, costs, edges):
    """Alg. 1 (lancet_dw_schedule) on an instruction DAG; returns assign[i] (a2a index or -1)."""
    import numpy as np
    kinds = np.ascontiguousarray(kinds, dtype=np.int32)
    costs = np.ascontiguousarray(costs, dtype=np.float64)
    ed = np.ascontiguousarray(np.asarray(edges, dtype=np.int32).reshape(-1, 2))
    out = np.full(len(kinds), -1, dtype=np.int32)
    p = lambda a: a.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
    _check(load_library().lancet_dw_schedule(len(kinds), p(kinds), p(costs), len(ed), p(ed), p(out)))
    return out


def stack_dw_plan(t_a2a, t_dw):
    """Alg. 1 on the backward of an L-layer stack (lancet_stack_dw_plan).  t_a2a [L][2n] (each
    layer's all-to-alls in issue order), t_dw [L][2] (dW2, dW1).  Returns (host_layer,
    host_a2a), each [L][2] int32, -1 = unassigned."""
    import numpy as np
    t_a2a = np.ascontiguousarray(t_a2a, dtype=np.float64)
    t_dw = np.ascontiguousarray(t_dw, dtype=np.float64)
    L, n2 = t_a2a.shape
    hl = np.full((L, 2), -1, dtype=np.int32)
    ha = np.full((L, 2), -1, dtype=np.int32)
    p = lambda a: a.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
    _check(load_library().lancet_stack_dw_plan(L, n2 // 2, p(t_a2a), p(t_dw), p(hl), p(ha)))
    return hl, ha


def share_nccl_id(pg=None, rank: int = 0) -> bytes:
    """Rank 0 creates the NCCL unique id; it is broadcast over the torch process group."""
    import torch.distributed as dist
    obj = [nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=pg)
    return obj[0]


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(load_library().lancet_nccl_unique_id(buf))
    return buf.raw


class Context:
    """One rank's lancet_ctx.

    world == 1: no communication.  world > 1 with `pg` (a torch.distributed group): NCCL,
    rank 0 creates the unique id and it is broadcast over `pg`.  `local_group`: a
    LocalGroup of simulated ranks on one device (each rank must call from its own thread).
    """

    def __init__(self, cfg: LayerConfig, world: int = 1, rank: int = 0, device: int | None = None,
                 pg=None, local_group: LocalGroup | None = None, transport: str = "nccl"):
        """transport: "nccl" (world > 1: NCCL grouped send/recv) or "peer" (copy engines over
        CUDA IPC; the blobs are all-gathered over the torch process group `pg`)."""
        lib = load_library()
        self.cfg = cfg
        self.world, self.rank = world, rank
        self.device = torch.cuda.current_device() if device is None else device
        self._p = ctypes.c_void_p()
        c = cfg._c()
        if transport == "peer":
            self._create_peer(lib, c, world, rank, pg)
        elif local_group is not None:
            _check(lib.lancet_create_local(ctypes.byref(self._p), local_group._p, rank, self.device,
                                           ctypes.byref(c)))
        else:
            nid = None
            if world > 1:
                nid = ctypes.create_string_buffer(share_nccl_id(pg, rank), 128)
            elif (cfg.flags | EXTRA_FLAGS) & FLAG_FORCE_EP:          # one-rank NCCL communicator
                nid = ctypes.create_string_buffer(nccl_unique_id(), 128)
            _check(lib.lancet_create(ctypes.byref(self._p), world, rank, self.device, nid,
                                     ctypes.byref(c)))
        self.E_l = cfg.n_experts // world
        self._last = None

    def _create_peer(self, lib, c, world, rank, pg):
        """Copy-engine peer transport: create, export the IPC blob, all-gather the blobs over
        `pg`, import.  Every rank takes part in both gathers even if its own step failed, so a
        failure anywhere raises on every rank (no rank is left waiting in a collective)."""
        import torch.distributed as dist

        def agree(ok: bool, what: str):
            if world > 1:
                flags = [None] * world
                dist.all_gather_object(flags, bool(ok), group=pg)
                ok = all(flags)
            if not ok:
                self.close()
                raise LancetError(6, f"peer transport: {what} failed on some rank")

        nb = lib.lancet_peer_blob_bytes()
        blob = ctypes.create_string_buffer(nb)
        ok = lib.lancet_create_peer(ctypes.byref(self._p), world, rank, self.device, ctypes.byref(c)) == 0
        ok = ok and lib.lancet_peer_export(self._p, blob) == 0
        agree(ok, "create / export")
        blobs = [bytes(blob.raw)]
        if world > 1:
            blobs = [None] * world
            dist.all_gather_object(blobs, bytes(blob.raw), group=pg)
        allb = ctypes.create_string_buffer(b"".join(blobs), nb * world)
        agree(lib.lancet_peer_import(self._p, allb) == 0, "import")

    # -- lifecycle --------------------------------------------------------------------------
    def close(self):
        if self._p and not getattr(self, "_borrowed", False):
            load_library().lancet_destroy(self._p)
        self._p = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_flags(self, flags: int):
        flags |= EXTRA_FLAGS
        _check(load_library().lancet_set_flags(self._p, flags), self._p)
        self.cfg.flags = flags

    # -- the layer ----------------------------------------------------------------------------
    def forward(self, x, wg, w1, w2, k: int, capacity_factor: float, n_chunks: int,
                y=None, stream=None, routing: bool = True):
        T = x.shape[0]
        dev = x.device
        y = torch.empty_like(x) if y is None else y
        idx = slot = w = None
        if routing:
            idx = torch.empty((T, k), dtype=torch.int32, device=dev)
            slot = torch.empty((T, k), dtype=torch.int32, device=dev)
            w = torch.empty((T, k), dtype=torch.float32, device=dev)
        st = load_library().lancet_moe_forward(
            self._p, _ptr(x), _ptr(wg), _ptr(w1), _ptr(w2), T, k, float(capacity_factor),
            n_chunks, _ptr(y), _ptr(idx), _ptr(slot), _ptr(w), _stream(stream))
        _check(st, self._p)
        self._last = (x, wg, w1, w2)       # the library keeps pointers until backward
        self._last_n = n_chunks
        return y, idx, slot, w

    def forward_partitioned(self, x, wg, w1, w2, k: int, capacity_factor: float, n_chunks: int,
                            resid=None, y=None, stream=None, routing: bool = True):
        """lancet_moe_forward_partitioned: every chunk gated on its own with the carried capacity
        state (the block's pre-MoE partition); y = resid + MoE(x)."""
        T = x.shape[0]
        dev = x.device
        y = torch.empty_like(x) if y is None else y
        idx = slot = w = None
        if routing:
            idx = torch.empty((T, k), dtype=torch.int32, device=dev)
            slot = torch.empty((T, k), dtype=torch.int32, device=dev)
            w = torch.empty((T, k), dtype=torch.float32, device=dev)
        st = load_library().lancet_moe_forward_partitioned(
            self._p, _ptr(x), _ptr(wg), _ptr(w1), _ptr(w2), T, k, float(capacity_factor), n_chunks,
            _ptr(resid), _ptr(y), _ptr(idx), _ptr(slot), _ptr(w), _stream(stream))
        _check(st, self._p)
        self._last = (x, wg, w1, w2)
        self._last_n = n_chunks
        return y, idx, slot, w

    def backward(self, dy, dx=None, dwg=None, dw1=None, dw2=None, stream=None):
        x, wg, w1, w2 = self._last
        dx = torch.empty_like(dy) if dx is None else dx
        dwg = torch.empty(wg.shape, dtype=torch.float32, device=dy.device) if dwg is None else dwg
        if self.cfg.act != "identity_expert":
            dw1 = torch.empty(w1.shape, dtype=torch.float32, device=dy.device) if dw1 is None else dw1
            dw2 = torch.empty(w2.shape, dtype=torch.float32, device=dy.device) if dw2 is None else dw2
        st = load_library().lancet_moe_backward(self._p, _ptr(dy), _ptr(dx), _ptr(dwg), _ptr(dw1),
                                                _ptr(dw2), _stream(stream))
        _check(st, self._p)
        return dx, dwg, dw1, dw2

    # -- peer transport failure handling (include/lancet_moe.h) ---------------------------------
    def set_peer_timeout_ms(self, ms: int):
        _check(load_library().lancet_set_peer_timeout_ms(self._p, int(ms)), self._p)

    def peer_abort(self):
        _check(load_library().lancet_peer_abort(self._p), self._p)

    def status(self):
        """Raise LancetError if an asynchronous failure (a timed-out peer wait) poisoned the
        context; never blocks."""
        _check(load_library().lancet_peer_status(self._p), self._p)

    def set_gate_seed(self, seed: int):
        """Seed of the Random gate (FLAG_GATE_RANDOM) for the following forwards."""
        _check(load_library().lancet_set_gate_seed(self._p, seed & ((1 << 64) - 1)), self._p)

    # -- cross-layer dW scheduling (R17) ---------------------------------------------
    def backward_dw(self, which: int = 3, stream=None):
        """Enqueue this context's pending dW GEMMs (after a backward under FLAG_DEFER_DW)."""
        _check(load_library().lancet_moe_backward_dw(self._p, which, _stream(stream)), self._p)

    def set_dw_fillers(self, fillers):
        """fillers: [(other Context, which (1 dW1 | 2 dW2), a2a index)] for the next backward."""
        n = len(fillers)
        others = (ctypes.c_void_p * max(n, 1))(*[f[0]._p.value for f in fillers])
        which = (ctypes.c_int32 * max(n, 1))(*[f[1] for f in fillers])
        idx = (ctypes.c_int32 * max(n, 1))(*[f[2] for f in fillers])
        _check(load_library().lancet_set_dw_fillers(self._p, n, others, which, idx), self._p)

    # -- introspection ------------------------------------------------------------------------
    def counts(self, n_chunks: int | None = None):
        """(send [E][n], recv [G][E_l][n], C) of the last forward; n is that forward's chunk
        count (the host arrays are sized by it)."""
        import numpy as np
        last = getattr(self, "_last_n", None)
        if last is None:
            raise LancetError(5, "no forward yet")
        if n_chunks is not None and n_chunks != last:
            raise LancetError(1, f"counts({n_chunks}): the last forward ran {last} chunks")
        n_chunks = last
        E, G = self.cfg.n_experts, self.world
        send = np.zeros((E, n_chunks), dtype=np.int32)
        recv = np.zeros((G, self.E_l, n_chunks), dtype=np.int32)
        C = ctypes.c_int32()
        _check(load_library().lancet_get_counts(self._p, send.ctypes.data_as(ctypes.c_void_p),
                                                recv.ctypes.data_as(ctypes.c_void_p),
                                                ctypes.byref(C)), self._p)
        return send, recv, C.value

    def logits(self, T: int):
        import numpy as np
        out = np.empty((T, self.cfg.n_experts), dtype=np.float32)
        _check(load_library().lancet_debug_copy(self._p, 0, out.ctypes.data_as(ctypes.c_void_p),
                                                out.nbytes), self._p)
        return out

    def timeline_begin(self, stream=None):
        _check(load_library().lancet_timeline_begin(self._p, _stream(stream)), self._p)

    def timeline(self, cap: int = 1024):
        recs = (_OpRecord * cap)()
        n = ctypes.c_int32()
        _check(load_library().lancet_last_timeline(self._p, recs, cap, ctypes.byref(n)), self._p)
        return [dict(name=r.name.decode(), lane=r.lane, chunk=r.chunk, start_us=r.start_us,
                     end_us=r.end_us) for r in recs[:n.value]]

    def workspace_bytes(self) -> int:
        b = ctypes.c_size_t()
        _check(load_library().lancet_workspace_bytes(self._p, ctypes.byref(b)), self._p)
        return b.value

    def nccl_registered(self) -> int:
        """Buffers registered with the NCCL communicator (lancet_nccl_registered)."""
        n = ctypes.c_int32()
        _check(load_library().lancet_nccl_registered(self._p, ctypes.byref(n)), self._p)
        return n.value

    def launch_counts(self):
        f, b = ctypes.c_int32(), ctypes.c_int32()
        _check(load_library().lancet_launch_counts(self._p, ctypes.byref(f), ctypes.byref(b)), self._p)
        return f.value, b.value


def exposed_comm_us(timeline) -> dict:
    """SPEC-style decomposition of one timeline: comm time not covered by any
    compute op ('exposed'), total comm busy time, compute busy time."""
    def union(iv):
        iv = sorted(iv)
        out = []
        for a, b in iv:
            if out and a <= out[-1][1]:
                out[-1][1] = max(out[-1][1], b)
            else:
                out.append([a, b])
        return out
    def exposed(iv, cover):
        tot = sum(b - a for a, b in iv)
        ov = 0.0
        for a, b in iv:
            for c, d in cover:
                lo, hi = max(a, c), min(b, d)
                if hi > lo:
                    ov += hi - lo
        return tot, tot - ov

    comm = union([(r["start_us"], r["end_us"]) for r in timeline if r["lane"] == 1])
    comp = union([(r["start_us"], r["end_us"]) for r in timeline if r["lane"] != 1])
    tot_comm, exp = exposed(comm, comp)
    # split: the size exchange (C1) and the data exchanges (C2)
    cnt = union([(r["start_us"], r["end_us"]) for r in timeline if r["lane"] == 1 and r["name"].startswith("a2a_counts")])
    dat = union([(r["start_us"], r["end_us"]) for r in timeline if r["lane"] == 1 and not r["name"].startswith("a2a_counts")])
    return dict(exposed_us=exp, comm_us=tot_comm, compute_us=sum(b - a for a, b in comp),
                exposed_counts_us=exposed(cnt, comp)[1], exposed_data_us=exposed(dat, comp)[1])
