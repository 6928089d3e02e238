"""ORACLE / TEST INFRASTRUCTURE ONLY — never imported by the product path.

numpy mirror of the counter-based weight generator in
paper_2503_09716_b200/csrc/elementwise.cu (fill_uniform_kernel), bit-exact:
    x = (seed * K1 + tensor_id) * K2 + i          (mod 2^64)
    z = splitmix64_mix(x)
    u = int(z >> 40) - 2^23                        uniform over [-2^23, 2^23)
    value = bf16_rne(fp32(u) * fp32(std * sqrt(3) / 2^23))
so identical random-init weights exist on host and device without shipping files
(SURVEY.md §7 step 1c).
"""

from __future__ import annotations

import numpy as np
import torch

_K1 = np.uint64(0x9E3779B97F4A7C15)
_K2 = np.uint64(0xD1B54A32D192ED03)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def _mix(z: np.ndarray) -> np.ndarray:
    z = (z ^ (z >> np.uint64(30))) * _M1
    z = (z ^ (z >> np.uint64(27))) * _M2
    return z ^ (z >> np.uint64(31))


def uniform_bf16(shape, seed: int, tensor_id: int, std: float) -> torch.Tensor:
    n = int(np.prod(shape))
    with np.errstate(over="ignore"):
        base = (np.uint64(seed) * _K1 + np.uint64(tensor_id)) * _K2
        z = _mix(base + np.arange(n, dtype=np.uint64))
    u = (z >> np.uint64(40)).astype(np.int64) - (1 << 23)
    # the C-ABI takes std as fp32, then widens to double for the scale
    scale = np.float32(float(np.float32(std)) * 1.7320508075688772 / 8388608.0)
    f = u.astype(np.float32) * scale  # exact int -> fp32, one IEEE RN multiply
    return torch.from_numpy(f.reshape(shape)).to(torch.bfloat16)  # RNE, like __float2bfloat16_rn
