"""The fused decode routing front end (route.cu, mgb_moe_route) against the unfused kernels and a
torch fp32 reference: residual add bit-exact; RMSNorm within one bf16 rounding; router logits
within fp32 accumulation-order error of an fp32 GEMM; and -- given the logits the fused kernel
produced -- top-k indices / weights, counts, offsets, dst_pos, src_token and the permuted rows
bit-exact with mgb_router_topk + mgb_permute (the pinned-order contract of BASELINE north_star)."""

import pytest
import torch

from oracle.rng import uniform_bf16

pytestmark = pytest.mark.gpu

BF16 = torch.bfloat16


@pytest.mark.parametrize("T,d,E,k,mode,ng,tg", [
    (1, 256, 8, 2, 0, 1, 1), (33, 256, 8, 2, 0, 1, 1), (827, 4096, 8, 2, 0, 1, 1),
    (6058, 2048, 64, 6, 1, 1, 1), (257, 5120, 160, 6, 2, 8, 3), (300, 2048, 64, 6, 1, 1, 1),
    (1000, 6144, 8, 2, 0, 1, 1),
    (2000, 4096, 8, 2, 0, 1, 1), (3001, 1024, 8, 2, 0, 1, 1)])  # > 1 chunk per CTA (rows via h_out)
def test_moe_route_matches_unfused(T, d, E, k, mode, ng, tg):
    from paper_2503_09716_b200 import ops

    if not ops.moe_route_supported(T, d, E):
        pytest.skip("beyond one co-resident grid")
    dev = "cuda"
    x = uniform_bf16((T, d), 0, 1 + T, 2.0).to(dev)
    delta = uniform_bf16((T, d), 0, 2 + T, 1.0).to(dev)
    ln_w = (1.0 + uniform_bf16((d,), 0, 3, 0.2).float()).to(BF16).to(dev)
    wr = uniform_bf16((E, d), 0, 4 + E, 0.05).to(dev)
    eps = 1e-5
    ws = ops.RouterWorkspace(T, E, k)
    h = torch.empty(T, d, dtype=BF16, device=dev)
    x_out = torch.empty(T, d, dtype=BF16, device=dev)
    xp = torch.empty(T * k, d, dtype=BF16, device=dev)
    lg = torch.empty(T, E, dtype=torch.float32, device=dev)
    for _ in range(2):  # the grid barrier's workspace is reused by the second launch
        ops.moe_route(x, delta, ln_w, eps, h, wr, ws, xp, mode, 2.5, ng, tg, x_out=x_out, logits_out=lg)
    torch.cuda.synchronize()

    # residual add: bit-exact; norm: within one bf16 rounding of the unfused kernel
    x_ref = torch.empty_like(x_out)
    h_ref = torch.empty_like(h)
    ops.add_rmsnorm(x, ln_w, eps, h_ref, delta=delta, x_out=x_ref)
    assert torch.equal(x_out, x_ref)
    dh = (h.float() - h_ref.float()).abs()
    assert float(dh.max()) <= float(h_ref.float().abs().max()) * 2 ** -7
    assert float((dh > 0).float().mean()) < 1e-3

    # logits vs an fp32 GEMM of the kernel's own h
    ref = h.float() @ wr.float().t()
    if mode == 0:
        ref = ref.to(BF16).float()
    torch.testing.assert_close(lg, ref, rtol=1e-2 if mode == 0 else 1e-4, atol=1e-3 if mode == 0 else 1e-4)

    # routing + permutation given the fused kernel's logits: bit-exact with the unfused kernels
    ws2 = ops.RouterWorkspace(T, E, k)
    ops.router_topk(None, None, ws2, k, mode, 2.5, ng, tg, logits_in=lg)
    xp2 = torch.empty_like(xp)
    ops.permute(h, ws2, xp2)
    torch.cuda.synchronize()
    assert torch.equal(ws.topk_idx, ws2.topk_idx)
    assert torch.equal(ws.topk_w, ws2.topk_w)
    assert torch.equal(ws.counts, ws2.counts)
    assert torch.equal(ws.offsets, ws2.offsets)
    assert torch.equal(ws.dst_pos, ws2.dst_pos)
    assert torch.equal(ws.src_token, ws2.src_token)
    assert torch.equal(xp, xp2)
    assert torch.equal(xp, h[ws.src_token.long()])


def test_moe_route_graph_replay():
    """Captured once, replayed: the grid barrier's counters return to zero every launch."""
    from paper_2503_09716_b200 import ops

    T, d, E, k = 200, 1024, 8, 2
    x = uniform_bf16((T, d), 0, 5, 1.0).cuda()
    ln_w = torch.ones(d, dtype=BF16, device="cuda")
    wr = uniform_bf16((E, d), 0, 6, 0.1).cuda()
    ws = ops.RouterWorkspace(T, E, k)
    h = torch.empty(T, d, dtype=BF16, device="cuda")
    xp = torch.empty(T * k, d, dtype=BF16, device="cuda")
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        ops.moe_route(x, None, ln_w, 1e-6, h, wr, ws, xp, 0)
    torch.cuda.synchronize()
    first = (ws.topk_idx.clone(), ws.dst_pos.clone(), xp.clone())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        ops.moe_route(x, None, ln_w, 1e-6, h, wr, ws, xp, 0)
    for _ in range(5):
        ws.dst_pos.zero_()
        g.replay()
    torch.cuda.synchronize()
    assert int(ws.sync[0]) & 0x7FFFFFFF == 0  # the barrier word's low bits return to zero every launch
    assert torch.equal(ws.topk_idx, first[0]) and torch.equal(ws.dst_pos, first[1]) and torch.equal(xp, first[2])


@pytest.mark.parametrize("T,d", [(827, 4096), (909, 4096), (64, 256)])
def test_moe_route_without_h_out(T, d):
    """One chunk per CTA (the engine's decode batches): h_out=None leaves the normalised rows only in
    x_perm, bit-identical to a launch that also writes h_out; both permutation store paths."""
    import os
    import subprocess
    import sys

    from paper_2503_09716_b200 import ops

    if not ops.moe_route_single_pass(T, d, 8):
        pytest.skip("not a one-pass batch on this device")
    for bulk in ("0", "1"):
        code = f"""
import torch
from oracle.rng import uniform_bf16
from paper_2503_09716_b200 import ops
T, d, E, k = {T}, {d}, 8, 2
x = uniform_bf16((T, d), 0, 11, 2.0).cuda(); o = uniform_bf16((T, d), 0, 12, 1.0).cuda()
ln = torch.ones(d, dtype=torch.bfloat16, device="cuda"); wr = uniform_bf16((E, d), 0, 13, 0.05).cuda()
res = []
for h in (torch.empty(T, d, dtype=torch.bfloat16, device="cuda"), None):
    ws = ops.RouterWorkspace(T, E, k); xp = torch.empty(T * k, d, dtype=torch.bfloat16, device="cuda")
    xo = torch.empty(T, d, dtype=torch.bfloat16, device="cuda")
    ops.moe_route(x, o, ln, 1e-5, h, wr, ws, xp, 0, x_out=xo)
    torch.cuda.synchronize()
    res.append((xp, ws.dst_pos.clone(), ws.src_token.clone(), xo, h))
(xa, pa, sa, oa, ha), (xb, pb, sb, ob, _) = res
assert torch.equal(xa, xb) and torch.equal(pa, pb) and torch.equal(sa, sb) and torch.equal(oa, ob)
assert torch.equal(xa, ha[sa.long()])
"""
        env = dict(os.environ, MGB_ROUTE_BULK=bulk)
        root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
        r = subprocess.run([sys.executable, "-c", code], env=env, cwd=root, capture_output=True, text=True)
        assert r.returncode == 0, f"MGB_ROUTE_BULK={bulk}: {r.stderr[-2000:]}"
