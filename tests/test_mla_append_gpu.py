"""The decode-step latent append (mgb_mla_append): the warp-per-token kernel writes the same page
bytes, q_pe and q_nope as the per-token-CTA kernel it replaces (the RoPE'd parts, the q re-layout
and the zero padding bit-exact; the normalised latent within one bf16 rounding, from the order the
variance is summed in)."""

import math
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import sys, torch
sys.path.insert(0, %r)
from paper_2503_09716_b200 import _native as nat
from oracle.rng import uniform_bf16
B, H, R, RP, NOPE = %d, %d, %d, %d, %d
page = nat.value("mgb_mla_page_size")
pps = 3
DP = (R + RP + 63) // 64 * 64
cache = torch.full((B * pps * DP * page,), float("nan"), dtype=torch.bfloat16, device="cuda")
q = uniform_bf16((B, H, NOPE + RP), 3, 1, 1.0).cuda()
ckv = uniform_bf16((B, R + RP), 3, 2, 2.0).cuda()
nw = (1 + uniform_bf16((R,), 3, 3, 0.2).float()).bfloat16().cuda()
pos = torch.randint(0, pps * page, (B,), generator=torch.Generator().manual_seed(4)).int().cuda()
bt = torch.arange(B * pps, dtype=torch.int32).view(B, pps).cuda()
freqs = torch.outer(torch.arange(pps * page).float(), 1.0 / (10000 ** (torch.arange(0, RP, 2).float() / RP)))
cos_t, sin_t = freqs.cos().contiguous().cuda(), freqs.sin().contiguous().cuda()
qn = torch.zeros(H, B, NOPE, dtype=torch.bfloat16, device="cuda")
qp = torch.zeros(B, H, RP, dtype=torch.bfloat16, device="cuda")
lens = torch.zeros(B + 4, dtype=torch.int32, device="cuda")
nat.call("mgb_mla_append", q.data_ptr(), ckv.data_ptr(), nw.data_ptr(), 1e-6, B, H, R, RP, NOPE, pos.data_ptr(),
         cos_t.data_ptr(), sin_t.data_ptr(), bt.data_ptr(), pps, cache.data_ptr(), qn.data_ptr(), qp.data_ptr(),
         lens.data_ptr(), torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
torch.save({"cache": cache.cpu(), "qn": qn.cpu(), "qp": qp.cpu(), "lens": lens.cpu()}, sys.argv[1])
"""


@pytest.mark.parametrize("B,H,R,RP,NOPE", [(37, 16, 512, 64, 128), (9, 128, 512, 64, 128), (5, 4, 128, 32, 64)])
def test_warp_append_matches_block_append(tmp_path, B, H, R, RP, NOPE):
    outs = []
    for blk in ("0", "1"):
        path = tmp_path / f"out{blk}.pt"
        env = dict(os.environ, MGB_MLA_APPEND_BLOCK=blk)
        subprocess.run([sys.executable, "-c", SCRIPT % (ROOT, B, H, R, RP, NOPE), str(path)], check=True, env=env,
                       cwd=ROOT, timeout=300)
        outs.append(torch.load(path))
    new, old = outs
    assert torch.equal(new["qn"], old["qn"]) and torch.equal(new["qp"], old["qp"])
    assert torch.equal(new["lens"], old["lens"])
    a, b = new["cache"].float(), old["cache"].float()
    written = ~torch.isnan(b)
    assert torch.equal(~torch.isnan(a), written)  # the same bytes of every page were written
    d = (a[written] - b[written]).abs()
    assert float((d > 0).float().mean()) < 2e-3
    assert float(d.max()) <= float(b[written].abs().max()) * 2 ** -7
