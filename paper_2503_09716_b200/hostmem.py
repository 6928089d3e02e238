"""Exact-size pinned host memory for the offloaded weight and KV stores.

torch's pinned allocator rounds every block up to a power of two, which on a host with 196 GB of
RAM would waste up to half of it on 100 GB-class stores.  Here an anonymous mapping of exactly the
requested size is page-locked in place with cudaHostRegister (portable + mapped), so the copy
engines DMA from it and kernels can store into it through its UVA address (KV_COPY_OUT,
kv_stream.cu).  The registration is dropped when the last tensor viewing the mapping dies."""

from __future__ import annotations

import ctypes
import mmap
import weakref

import torch

_PORTABLE_MAPPED = 0x01 | 0x02  # cudaHostRegisterPortable | cudaHostRegisterMapped


def _unregister(addr: int) -> None:
    try:
        torch.cuda.cudart().cudaHostUnregister(addr)
    except Exception:  # interpreter shutdown
        pass


def pinned_empty(n: int, dtype: torch.dtype = torch.bfloat16) -> torch.Tensor:
    nbytes = n * torch.empty((), dtype=dtype).element_size()
    if nbytes == 0:
        return torch.empty(0, dtype=dtype)
    m = mmap.mmap(-1, nbytes)
    c = ctypes.c_char.from_buffer(m)
    addr = ctypes.addressof(c)
    del c
    rc = torch.cuda.cudart().cudaHostRegister(addr, nbytes, _PORTABLE_MAPPED)
    if int(rc) != 0:
        raise RuntimeError(f"cudaHostRegister of {nbytes} bytes failed ({rc})")
    weakref.finalize(m, _unregister, addr)  # runs when the last view releases the mapping
    return torch.frombuffer(m, dtype=dtype, count=n)
