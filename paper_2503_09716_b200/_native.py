"""ctypes binding of libmgb.so — the C-ABI declared in include/mgb.h.

This is the only bridge between Python and the sm_100a kernels.  There is deliberately no CPU
or PyTorch fallback: if the library is missing or a call fails, we raise.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

from . import build as _build

P = ctypes.c_void_p
I = ctypes.c_int
F = ctypes.c_float
L = ctypes.c_int64

# name -> argument types (every entry point returns int status, 0 = ok)
SIGNATURES: dict[str, list] = {
    # introspection
    "mgb_abi_version": [],
    "mgb_num_sms": [],
    "mgb_moe_check_capacity": [P, I, I, P, P],
    "mgb_moe_route_chunks": [I],
    "mgb_moe_route_stamps": [P],
    "mgb_moe_route_supported": [I, I, I],
    "mgb_moe_route": [P, P, P, F, I, I, P, P, P, I, I, I, F, I, I, P, P, P, P, P, P, P, P, P, P, P, P],
    "mgb_capacity_status": [P, I],
    "mgb_kv_page_size": [],
    "mgb_router_num_blocks": [I],
    "mgb_router_tokens_per_block": [],
    # router / permutation / combine (routing.cu)
    "mgb_router_topk": [P, P, P, I, I, I, I, I, F, I, I, P, P, P, P, P, P, P, P, P],
    "mgb_permute": [P, P, P, P, P, I, I, I, I, P, P, P, P],
    "mgb_unpermute_combine": [P, P, P, P, P, I, I, I, P, P, F, P, P],
    # grouped expert FFN (moe_gemm.cu)
    "mgb_moe_gemm_gate_up": [P, P, P, I, I, I, I, P, P],
    "mgb_moe_gemm_down": [P, P, P, I, I, I, I, P, P],
    "mgb_moe_ffn": [P, P, P, P, I, I, I, I, P, P, P, P],
    "mgb_grouped_ffn": [P, P, P, P, I, I, I, I, P, P, P],
    "mgb_moe_gemm_down_ep": [P, P, P, I, I, I, I, P, P],
    "mgb_ep_permute_dispatch": [P, P, P, P, P, I, I, I, I, I, P, P, I, P, P, P],
    "mgb_ep_row_ptrs": [P, P, P, I, I, P, I, I, P, P],
    # attention (attn_gqa.cu)
    "mgb_decode_attn_gqa": [P, P, P, P, I, P, I, I, I, I, F, P, P],
    "mgb_decode_attn_gqa_sched": [P, P, P, P, I, P, I, I, I, I, F, P, P, P],
    "mgb_decode_attn_gqa_rope": [P, P, P, P, P, P, P, I, P, I, I, I, I, F, P, P, P],
    # elementwise.cu
    "mgb_add_rmsnorm": [P, P, P, F, I, I, P, P, P],
    "mgb_rope_append_gqa": [P, I, I, P, P, P, I, I, I, P, I, P, P, P, P, P],
    "mgb_rope_append_gqa_prefill": [P, I, I, I, P, P, I, I, I, P, I, P, P, P, P, P, P],
    "mgb_embed": [P, P, I, I, P, P],
    "mgb_silu_mul": [P, I, I, P, P],
    "mgb_argmax": [P, I, I, P, P],
    "mgb_decode_advance": [P, I, P, I, P, P, P],
    "mgb_fill_uniform_bf16": [P, L, ctypes.c_uint64, ctypes.c_uint64, F, F, I, P],
    "mgb_fill_uniform_bf16_range": [P, L, L, ctypes.c_uint64, ctypes.c_uint64, F, P],
    # attn_mla.cu
    "mgb_mla_page_size": [],
    "mgb_mla_page_elems": [I, I],
    "mgb_decode_attn_mla": [P, P, P, P, I, P, I, I, I, I, F, P, P],
    "mgb_mla_append": [P, P, P, F, I, I, I, I, I, P, P, P, P, I, P, P, P, P, P],
    "mgb_mla_append_prefill": [P, P, P, F, I, I, I, I, I, I, I, P, P, P, I, P, P, P, P],
    # attn_prefill.cu
    "mgb_prefill_attn_supported": [I, I],
    "mgb_prefill_attn": [P, I, I, P, I, I, P, I, I, P, I, I, I, I, I, I, I, I, I, F, P, I, P],
    # kv_stream.cu
    "mgb_kv_token_copy": [P, P, I, P, P, I, P, I, I, L, I, I, L, P],
    "mgb_copy_bytes": [P, P, L, P],
    # cpu_attn.cpp (host code: ATTN_MECH_CPU)
    "mgb_cpu_attn_gqa": [P],
    "mgb_cpu_attn_gqa_enqueue": [P, P],
    "mgb_cpu_threads": [I],
    "mgb_cpu_attn_simd": [],
}


class CpuAttnGqa(ctypes.Structure):
    """struct MgbCpuAttnGqa (include/mgb.h): one layer's CPU-attention job description."""

    _fields_ = [("k_pages", P), ("v_pages", P), ("q", P), ("seq_lens", P), ("out", P), ("first_page", L),
                ("pps", ctypes.c_int32), ("B", ctypes.c_int32), ("Hq", ctypes.c_int32), ("Hkv", ctypes.c_int32),
                ("hd", ctypes.c_int32), ("page_tokens", ctypes.c_int32), ("scale", F), ("status", ctypes.c_int32)]

# entry points that return a value rather than a status
VALUE_FNS = {"mgb_moe_route_chunks", "mgb_moe_route_supported", "mgb_prefill_attn_supported", "mgb_cpu_threads", "mgb_cpu_attn_simd", "mgb_abi_version", "mgb_num_sms", "mgb_kv_page_size", "mgb_mla_page_size", "mgb_mla_page_elems",
             "mgb_router_num_blocks", "mgb_router_tokens_per_block"}

STATUS = {0: "ok", -1: "invalid argument", -2: "capacity exceeded", -3: "CUDA error"}


class NativeError(RuntimeError):
    pass


class _Lib:
    def __init__(self) -> None:
        self._lib = None
        self.calls = 0  # libmgb entry-point calls (each launches exactly one kernel)

    def load(self) -> ctypes.CDLL:
        if self._lib is not None:
            return self._lib
        path = Path(os.environ.get("MGB_LIB", str(_build.LIB_PATH)))
        if not path.exists():
            if os.environ.get("MGB_NO_BUILD"):
                raise NativeError(f"libmgb.so not found at {path}; run __graft_entry__.build()")
            _build.build(verbose=False)
        lib = ctypes.CDLL(str(path), mode=ctypes.RTLD_GLOBAL)
        for name, args in SIGNATURES.items():
            if "MGB_LIB" in os.environ and not hasattr(lib, name):
                continue  # an A/B variant build (tools/build_variant.py) of an older tree
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = ctypes.c_int
        lib.mgb_last_error.restype = ctypes.c_char_p
        lib.mgb_last_error.argtypes = []
        self._lib = lib
        return lib

    def value(self, name: str, *args) -> int:
        assert name in VALUE_FNS
        return int(getattr(self.load(), name)(*args))

    def raw(self, name: str, *args) -> int:
        """Call an entry point and return its status (for callers that handle MGB_ECAPACITY)."""
        return int(getattr(self.load(), name)(*args))

    def call(self, name: str, *args) -> None:
        lib = self.load()
        self.calls += 1
        rc = getattr(lib, name)(*args)
        if rc != 0:
            err = lib.mgb_last_error().decode()
            raise NativeError(f"{name} failed: {STATUS.get(rc, rc)} (cuda: {err})")

    @property
    def path(self) -> str:
        return str(_build.LIB_PATH)


LIB = _Lib()


def call(name: str, *args) -> None:
    LIB.call(name, *args)


def raw(name: str, *args) -> int:
    return LIB.raw(name, *args)


def value(name: str, *args) -> int:
    return LIB.value(name, *args)


def exported_symbols() -> list[str]:
    return list(SIGNATURES) + ["mgb_last_error"]
