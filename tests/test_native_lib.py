"""CPU-side checks of the drop-in boundary: libmgb.so builds for sm_100a, loads, and exports every
entry point include/mgb.h declares; SASS proves tcgen05/TMA are used; the product path fails
loudly without the library (no CPU fallback)."""

import os
import re
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_symbols():
    with open(os.path.join(ROOT, "include", "mgb.h")) as f:
        txt = f.read()
    return sorted(set(re.findall(r"\b(mgb_[a-z0-9_]+)\s*\(", txt)))


@pytest.fixture(scope="module")
def lib():
    from paper_2503_09716_b200 import _native, build

    build.build(verbose=False)
    return _native.LIB.load()


def test_library_exports_every_declared_symbol(lib):
    syms = _header_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(lib, s), f"{s} declared in include/mgb.h but not exported"


def test_python_binding_covers_header():
    from paper_2503_09716_b200 import _native

    declared = set(_header_symbols())
    bound = set(_native.exported_symbols())
    assert declared == bound, (declared - bound, bound - declared)


def test_value_entry_points_without_gpu(lib):
    from paper_2503_09716_b200 import _native

    assert _native.value("mgb_abi_version") == 2
    assert _native.value("mgb_kv_page_size") == 64
    assert _native.value("mgb_router_num_blocks", 827) == 104


def test_sass_uses_tcgen05_and_tma():
    from paper_2503_09716_b200 import build

    build.build(verbose=False)
    obj = os.path.join(ROOT, "paper_2503_09716_b200", "_lib", "moe_gemm_cu.o")
    sass = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
    assert "UTCHMMA" in sass and "UTMALDG" in sass and "LDTM" in sass
    attn = subprocess.run(["cuobjdump", "-sass", os.path.join(ROOT, "paper_2503_09716_b200", "_lib", "attn_gqa_cu.o")],
                          capture_output=True, text=True).stdout
    assert "UBLKCP" in attn and "HMMA" in attn
    mla = subprocess.run(["cuobjdump", "-sass", os.path.join(ROOT, "paper_2503_09716_b200", "_lib", "attn_mla_cu.o")],
                         capture_output=True, text=True).stdout
    assert "UTCHMMA" in mla and "UBLKCP" in mla and "LDTM" in mla


def test_missing_library_fails_loudly(tmp_path):
    code = ("import os, sys; sys.path.insert(0, %r)\n"
            "from paper_2503_09716_b200 import _native\n"
            "try:\n    _native.LIB.load()\nexcept _native.NativeError as e:\n    print('LOUD', e)\n") % ROOT
    env = dict(os.environ, MGB_LIB=str(tmp_path / "nope.so"), MGB_NO_BUILD="1")
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env)
    assert "LOUD" in out.stdout


def test_engine_refuses_without_cuda():
    import torch

    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    from paper_2503_09716_b200.engine import Engine

    with pytest.raises(RuntimeError, match="no CPU fallback"):
        Engine("tiny-mixtral", None, prompt_len=4, decode_len=4)
