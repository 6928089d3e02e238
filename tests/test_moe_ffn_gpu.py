"""The fused expert FFN launch (mgb_moe_ffn: gate/up + SiLU*up + down in one persistent CTA-pair
kernel whose down units wait on per-expert completion counters) is bit-identical to the two grouped
GEMM launches it replaces (same unit tiling, same K order per output element), leaves its counters
zero for the next launch (graph replay), honours the capacity contract, and matches an fp32 torch
reference within bf16 tolerance."""

import pytest
import torch

from oracle.rng import uniform_bf16

pytestmark = pytest.mark.gpu

BF16 = torch.bfloat16


def _case(E, d, f, counts, seed=0):
    T = sum(counts)
    x = uniform_bf16((max(T, 1), d), seed, 1, 1.0).cuda()
    wgu = uniform_bf16((E, 2 * f, d), seed, 2, 0.05).cuda()
    wd = uniform_bf16((E, d, f), seed, 3, 0.05).cuda()
    offs = torch.tensor([0] + list(torch.tensor(counts).cumsum(0)), dtype=torch.int32).cuda()
    return x, wgu, wd, offs


@pytest.mark.parametrize("E,d,f,counts", [
    (8, 4096, 14336, [207, 190, 221, 0, 240, 198, 215, 383]),   # Mixtral dims, one empty expert
    (64, 2048, 1408, [95 + (i * 37) % 40 for i in range(64)]),  # DeepSeek-V2-Lite routed dims
    (1, 2048, 2816, [600]),                                     # DSV2-Lite shared experts (E = 1 segment)
    (8, 256, 512, [3, 0, 1, 17, 0, 0, 9, 2]),                   # tiny, ragged
    (4, 512, 384, [40, 30, 20, 10]),                            # f % 128 != 0: two-launch fallback
])
def test_moe_ffn_equals_two_launches(E, d, f, counts):
    from paper_2503_09716_b200 import ops

    x, wgu, wd, offs = _case(E, d, f, counts)
    R = x.shape[0]
    h1, y1 = torch.zeros(R, f, dtype=BF16, device="cuda"), torch.zeros(R, d, dtype=BF16, device="cuda")
    ops.moe_gemm_gate_up(wgu, x, offs, h1)
    ops.moe_gemm_down(wd, h1, offs, y1)
    sync = torch.zeros(257, dtype=torch.int32, device="cuda")
    h2, y2 = torch.zeros_like(h1), torch.zeros_like(y1)
    for _ in range(2):  # the counters are reset by each launch
        ops.moe_ffn(wgu, wd, x, offs, h2, y2, sync)
    torch.cuda.synchronize()
    assert int(sync.abs().sum()) == 0
    n = int(offs[-1])
    assert torch.equal(h1[:n], h2[:n])
    assert torch.equal(y1[:n], y2[:n])
    # fp32 reference (HF MixtralExperts rounding points) on a few rows of every non-empty expert
    for e in range(E):
        a, b = int(offs[e]), int(offs[e + 1])
        if b == a:
            continue
        r = slice(a, min(b, a + 4))
        xe = x[r].float()
        g = (xe @ wgu[e, :f].float().T).to(BF16).float()
        u = (xe @ wgu[e, f:].float().T).to(BF16).float()
        hh = (torch.nn.functional.silu(g).to(BF16).float() * u).to(BF16)
        yy = (hh.float() @ wd[e].float().T)
        err = (y2[r].float() - yy).abs().max() / yy.abs().max().clamp_min(1e-6)
        assert float(err) <= 2e-2, (e, float(err))


def test_moe_ffn_graph_replay_and_capacity():
    from paper_2503_09716_b200 import ops

    E, d, f = 8, 1024, 2048
    counts = [50, 61, 0, 33, 70, 12, 90, 41]
    x, wgu, wd, offs = _case(E, d, f, counts, seed=1)
    R = x.shape[0]
    sync = torch.zeros(257, dtype=torch.int32, device="cuda")
    h, y = torch.zeros(R, f, dtype=BF16, device="cuda"), torch.zeros(R, d, dtype=BF16, device="cuda")
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        ops.moe_ffn(wgu, wd, x, offs, h, y, sync)
    torch.cuda.synchronize()
    ref = y.clone()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        ops.moe_ffn(wgu, wd, x, offs, h, y, sync)
    for _ in range(4):
        y.zero_()
        g.replay()
    torch.cuda.synchronize()
    assert torch.equal(y, ref) and int(sync.abs().sum()) == 0
    # capacity: buffers smaller than offsets[E] -> no rows written, status recorded
    ops.capacity_status(reset=True)
    cap = R - 10
    yc = torch.full((R, d), 5.0, dtype=BF16, device="cuda")
    hc = torch.full((R, f), 5.0, dtype=BF16, device="cuda")
    ops.moe_ffn(wgu, wd, x[:cap], offs, hc[:cap], yc[:cap], sync)
    with pytest.raises(ops.CapacityError):
        ops.capacity_status(reset=True)
    assert bool((yc == 5.0).all()) and bool((hc == 5.0).all())
    assert int(sync.abs().sum()) == 0
