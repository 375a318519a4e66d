"""CPU-only checks of the C-ABI boundary: the library loads, exports every entry point that
include/lancet_moe.h declares, rejects bad arguments before touching a device, and the product
package never imports the oracle."""
import ast
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "lancet_moe.h")
BLOCK_HEADER = os.path.join(ROOT, "include", "lancet_block.h")
PKG = os.path.join(ROOT, "paper_2404_19429_b200")


@pytest.fixture(scope="module")
def lib():
    from paper_2404_19429_b200 import build
    build.build()
    from paper_2404_19429_b200 import lancet
    return lancet.load_library()


def declared_functions(path=HEADER):
    src = open(path).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(lancet_[a-z_0-9]+)\s*\(", src)))


def test_header_declares_the_north_star_entry_points():
    names = declared_functions()
    assert "lancet_moe_forward" in names and "lancet_moe_backward" in names
    assert len(names) >= 14


def test_every_declared_symbol_is_exported(lib):
    from paper_2404_19429_b200 import block, lancet
    for name in declared_functions():
        assert hasattr(lib, name), name
    assert set(declared_functions()) == set(lancet.EXPORTS)
    # the GPT-MoE block (include/lancet_block.h)
    for name in declared_functions(BLOCK_HEADER):
        assert hasattr(lib, name), name
    assert set(declared_functions(BLOCK_HEADER)) == set(block.EXPORTS)


def test_block_create_rejects_bad_config_without_a_device(lib):
    from paper_2404_19429_b200 import block, lancet
    b = ctypes.c_void_p()
    good = dict(d_model=256, d_ffn=512, n_experts=4, max_tokens=512)
    for moe_kw, heads, seq in [(dict(good), 3, 128),                          # head_dim != 128
                               (dict(good), 2, 100),                          # seq % 128
                               (dict(good, max_tokens=500), 2, 128),          # max_tokens % seq
                               (dict(good, act="identity_expert"), 2, 128),
                               (dict(good, dtype="fp32"), 2, 128)]:
        cfg = block.BlockConfig(lancet.LayerConfig(**moe_kw), n_heads=heads, seq_len=seq)
        st = block._lib().lancet_block_create_peer(ctypes.byref(b), 1, 0, 0, ctypes.byref(cfg._c()))
        assert st in (1, 6), (moe_kw, heads, seq, st)
        assert not b.value


def test_abi_version(lib):
    assert lib.lancet_abi_version() == 2


def test_create_rejects_bad_config_without_a_device(lib):
    from paper_2404_19429_b200 import lancet
    ctx = ctypes.c_void_p()
    bad = [
        lancet.LayerConfig(d_model=12, d_ffn=64, n_experts=8, max_tokens=16),      # d % 8
        lancet.LayerConfig(d_model=64, d_ffn=64, n_experts=5, max_tokens=16),      # E % world (2)
        lancet.LayerConfig(d_model=64, d_ffn=64, n_experts=8, max_tokens=16, max_k=9),
        lancet.LayerConfig(d_model=64, d_ffn=64, n_experts=8, max_tokens=16, max_chunks=65),
        lancet.LayerConfig(d_model=64, d_ffn=64, n_experts=300, max_tokens=16, max_k=2),
    ]
    for cfg in bad:
        c = cfg._c()
        st = lib.lancet_create(ctypes.byref(ctx), 2 if cfg.n_experts == 5 else 1, 0, 0,
                               b"\0" * 128, ctypes.byref(c))
        assert st == 1, cfg                                          # LANCET_ERR_ARG
        assert lib.lancet_last_error(None)
    assert lib.lancet_create(None, 1, 0, 0, None, None) == 1


def test_null_context_calls_fail_cleanly(lib):
    assert lib.lancet_moe_forward(None, None, None, None, None, 1, 1, 1.0, 1, None, None, None,
                                  None, None) == 1
    assert lib.lancet_moe_backward(None, None, None, None, None, None, None) == 1
    assert lib.lancet_destroy(None) == 0


def test_product_never_imports_the_oracle():
    for dirpath, _, files in os.walk(PKG):
        for f in files:
            if f.endswith(".py"):
                tree = ast.parse(open(os.path.join(dirpath, f)).read())
                for node in ast.walk(tree):
                    if isinstance(node, ast.Import):
                        assert not any(a.name.split(".")[0] == "oracle" for a in node.names), f
                    if isinstance(node, ast.ImportFrom):
                        assert (node.module or "").split(".")[0] != "oracle", f
            if f.endswith((".cu", ".cpp", ".h", ".cuh")):
                assert "oracle" not in open(os.path.join(dirpath, f)).read().lower().replace(
                    "no oracle", ""), f


def test_local_group_lifecycle_without_device(lib):
    g = ctypes.c_void_p()
    assert lib.lancet_local_group_create(ctypes.byref(g), 2) == 0
    assert lib.lancet_local_group_destroy(g) == 0


def test_binding_flag_values_match_the_header():
    # every LANCET_FLAG_* of the header has the same value in the Python binding
    from paper_2404_19429_b200 import lancet
    src = re.sub(r"/\*.*?\*/", "", open(HEADER).read(), flags=re.S)
    flags = dict((name, 1 << int(bit)) for name, bit in
                 re.findall(r"LANCET_FLAG_([A-Z_0-9]+)\s*=\s*1u\s*<<\s*(\d+)", src))
    assert len(flags) >= 10
    for name, val in flags.items():
        assert getattr(lancet, "FLAG_" + name) == val, name
    assert len(set(flags.values())) == len(flags), "flag bits collide"
    comm = re.search(r"#define\s+LANCET_COMM_SMS\s+(\d+)", src)
    assert comm and int(comm.group(1)) > 0
