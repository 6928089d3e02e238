"""mgb_prefill_attn (attn_prefill.cu, tcgen05 causal prefill attention) vs a plain fp32 PyTorch
reference of the same op (HF sdpa semantics: fp32 scores / softmax / P.V, causal), for the GQA head
layout of Mixtral and the MLA layout of DeepSeek-V2 (K = [k_nope_h | shared k_pe], V inside the
up-projected rows), including prompts that are not a multiple of the 128-query tile."""

import pytest
import torch

pytestmark = pytest.mark.gpu
BF16 = torch.bfloat16


def _ref(q, k, v, n_seq, P, scale):
    """q [T, Hq, dq], k [T, Hkv, dq], v [T, Hkv, dv] -> [T, Hq * dv] fp32, causal per prompt."""
    Hq, Hkv = q.shape[1], k.shape[1]
    out = []
    for s in range(n_seq):
        sl = slice(s * P, (s + 1) * P)
        qs, ks, vs = (t[sl].float().transpose(0, 1) for t in (q, k, v))       # [H, P, d]
        ks, vs = ks.repeat_interleave(Hq // Hkv, 0), vs.repeat_interleave(Hq // Hkv, 0)
        sc = qs @ ks.transpose(1, 2) * scale
        sc = sc.masked_fill(torch.triu(torch.ones(P, P, dtype=torch.bool), 1), float("-inf"))
        out.append((torch.softmax(sc, -1) @ vs).transpose(0, 1).reshape(P, -1))
    return torch.cat(out)


def _err(a, b):
    return ((a.float() - b).abs().max() / b.abs().max()).item()


@pytest.mark.parametrize("n_seq,P,Hq,Hkv,hd", [(2, 512, 32, 8, 128), (3, 200, 8, 2, 128), (2, 1, 8, 8, 128),
                                               (1, 130, 4, 4, 64), (5, 128, 8, 1, 128), (1, 700, 48, 8, 128)])
def test_prefill_attn_gqa(n_seq, P, Hq, Hkv, hd):
    from paper_2503_09716_b200 import ops

    T = n_seq * P
    g = torch.Generator().manual_seed(P + Hq)
    q = torch.randn(T, Hq * hd, generator=g).to(BF16)
    k = torch.randn(T, Hkv * hd, generator=g).to(BF16)
    v = torch.randn(T, Hkv * hd, generator=g).to(BF16)
    out = torch.full((T, Hq * hd), float("nan"), dtype=BF16, device="cuda")
    qd, kd, vd = q.cuda(), k.cuda(), v.cuda()
    ops.prefill_attn(qd, kd, vd, out, n_seq, P, Hq, Hkv, hd, hd, hd ** -0.5, hd, hd, hd)
    ref = _ref(q.view(T, Hq, hd), k.view(T, Hkv, hd), v.view(T, Hkv, hd), n_seq, P, hd ** -0.5)
    assert not out.isnan().any()
    assert _err(out.cpu(), ref) <= 1e-2


@pytest.mark.parametrize("n_seq,P,H", [(2, 300, 16), (1, 512, 16), (2, 64, 128)])
def test_prefill_attn_mla(n_seq, P, H):
    from paper_2503_09716_b200 import ops

    nope, r, vd = 128, 64, 128
    T = n_seq * P
    g = torch.Generator().manual_seed(P + H)
    q = torch.randn(T, H * (nope + r), generator=g).to(BF16)
    kv = torch.randn(T, H * (nope + vd), generator=g).to(BF16)
    kpe = torch.randn(T, r, generator=g).to(BF16)
    out = torch.zeros(T, H * vd, dtype=BF16, device="cuda")
    scale = (nope + r) ** -0.5
    qd, kvd, kped = q.cuda(), kv.cuda(), kpe.cuda()
    ops.prefill_attn(qd, kvd, kvd, out, n_seq, P, H, H, nope + r, vd, scale, nope + r, nope + vd, nope + vd,
                     v_col0=nope, kr=kped)
    kv3 = kv.view(T, H, nope + vd)
    key = torch.cat([kv3[..., :nope], kpe[:, None, :].expand(T, H, r)], -1)
    ref = _ref(q.view(T, H, nope + r), key, kv3[..., nope:], n_seq, P, scale)
    assert _err(out.cpu(), ref) <= 1e-2


def test_prefill_attn_rejects_unsupported():
    from paper_2503_09716_b200 import _native as nat
    from paper_2503_09716_b200 import ops

    assert ops.prefill_attn_supported(128, 128) and not ops.prefill_attn_supported(32, 32)
    x = torch.zeros(64, 256, dtype=BF16, device="cuda")
    with pytest.raises(nat.NativeError):
        ops.prefill_attn(x, x, x, x, 1, 64, 8, 2, 32, 32, 1.0, 32, 32, 32)
