"""ATTN_MECH_CPU (csrc/cpu_attn.cpp): GQA decode attention on the host cores over the host KV page
store, the MoE-Gen CPU attention split (omega > 0).  Runs without a GPU:
it is host code behind the C-ABI.  Checked against a plain fp32 torch reference of the same op
(scores fp32, softmax fp32, probabilities rounded to bf16, fp32 PV, one bf16 rounding) on the AVX-512
BF16 path and the scalar path, across page boundaries, ragged lengths and GQA group sizes."""

import ctypes
import os
import subprocess
import sys

import pytest
import torch

from paper_2503_09716_b200 import _native as nat

BF16 = torch.bfloat16


def _pages(dense, P, pps):
    """dense [B, L, Hkv, hd] -> chunk-major pages [B*pps][Hkv][hd/8][P][8] (attn_gqa.cu layout)."""
    B, L, H, hd = dense.shape
    full = torch.zeros(B, pps * P, H, hd, dtype=dense.dtype)
    full[:, :L] = dense
    x = full.view(B, pps, P, H, hd // 8, 8).permute(0, 1, 3, 4, 2, 5)  # [B, pps, H, c, P, 8]
    return x.contiguous().reshape(-1)


def _reference(q, k, v, lens, scale):
    B, Hq, hd = q.shape
    Hkv = k.shape[2]
    G = Hq // Hkv
    out = torch.zeros(B, Hq, hd)
    for b in range(B):
        L = int(lens[b])
        kk = k[b, :L].float().repeat_interleave(G, dim=1)  # [L, Hq, hd]
        vv = v[b, :L].float().repeat_interleave(G, dim=1)
        s = torch.einsum("hd,lhd->hl", q[b].float(), kk) * scale
        p = torch.softmax(s, -1).to(BF16).float()
        out[b] = torch.einsum("hl,lhd->hd", p, vv)
    return out.to(BF16)


def _run(B, Hq, Hkv, hd, lens, P=64, seed=0):
    g = torch.Generator().manual_seed(seed)
    pps = (max(lens) + P - 1) // P + 1
    L = max(lens)
    q = (torch.randn(B, Hq, hd, generator=g)).to(BF16)
    k = (torch.randn(B, L, Hkv, hd, generator=g)).to(BF16)
    v = (torch.randn(B, L, Hkv, hd, generator=g)).to(BF16)
    kp, vp = _pages(k, P, pps), _pages(v, P, pps)
    sl = torch.tensor(lens, dtype=torch.int32)
    out = torch.zeros(B, Hq * hd, dtype=BF16)
    d = nat.CpuAttnGqa(kp.data_ptr(), vp.data_ptr(), q.data_ptr(), sl.data_ptr(), out.data_ptr(), 0, pps, B, Hq, Hkv,
                       hd, P, hd ** -0.5, 99)
    nat.call("mgb_cpu_attn_gqa", ctypes.byref(d))
    assert d.status == 0
    ref = _reference(q, k, v, sl, hd ** -0.5)
    err = (out.view(B, Hq, hd).float() - ref.float()).abs().max().item() / ref.float().abs().max().item()
    return err


@pytest.mark.parametrize("B,Hq,Hkv,hd,lens", [
    (3, 32, 8, 128, [1, 64, 130]),          # Mixtral heads, page boundaries, single key
    (4, 8, 2, 32, [7, 63, 65, 200]),        # tiny config, odd lengths
    (2, 16, 16, 64, [33, 96]),              # MHA (G = 1)
    (5, 48, 8, 128, [768, 513, 640, 700, 767]),  # Mixtral-8x22B heads at decode contexts
])
def test_cpu_attention_matches_fp32_reference(B, Hq, Hkv, hd, lens):
    assert _run(B, Hq, Hkv, hd, lens) <= 1e-2


def test_cpu_attention_scalar_path_and_threads():
    """The scalar path (hosts without AVX-512 BF16) gives the same answer within tolerance; the
    thread pool can be resized."""
    here = os.path.dirname(os.path.abspath(__file__))
    code = ("import sys; sys.path[:0] = [%r, %r]; from test_cpu_attn import _run; "
            "from paper_2503_09716_b200 import _native as nat; "
            "assert nat.value('mgb_cpu_attn_simd') == 0; print(_run(3, 32, 8, 128, [5, 70, 300]))"
            % (here, os.path.dirname(here)))
    env = dict(os.environ, MGB_CPU_SCALAR="1")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    assert float(r.stdout.strip().splitlines()[-1]) <= 1e-2
    n = nat.value("mgb_cpu_threads", 0)
    assert nat.value("mgb_cpu_threads", 3) == 3
    assert _run(4, 8, 2, 32, [7, 63, 65, 200]) <= 1e-2
    nat.value("mgb_cpu_threads", n)


def test_cpu_attention_rejects_bad_lengths():
    B, Hq, Hkv, hd, P, pps = 1, 8, 2, 32, 64, 1
    kp = torch.zeros(pps * Hkv * hd * P, dtype=BF16)
    q = torch.zeros(B, Hq, hd, dtype=BF16)
    out = torch.zeros(B, Hq * hd, dtype=BF16)
    sl = torch.tensor([P + 1], dtype=torch.int32)  # more keys than the sequence's pages hold
    d = nat.CpuAttnGqa(kp.data_ptr(), kp.data_ptr(), q.data_ptr(), sl.data_ptr(), out.data_ptr(), 0, pps, B, Hq,
                       Hkv, hd, P, 1.0, 0)
    with pytest.raises(nat.NativeError):
        nat.call("mgb_cpu_attn_gqa", ctypes.byref(d))
