"""mgb_add_rmsnorm's warp-per-token path (T >= 1024, d <= 2048) against its CTA-per-token path (the
same rows issued in batches under 1024): the residual add bit-exact, the normalised rows within one
bf16 rounding (the variance is summed in a different order)."""

import pytest
import torch

from oracle.rng import uniform_bf16

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("T,d,with_delta", [(6058, 2048, True), (1500, 1024, True), (1024, 2048, False)])
def test_warp_norm_matches_block_norm(T, d, with_delta):
    from paper_2503_09716_b200 import ops

    x = uniform_bf16((T, d), 5, 1, 2.0).cuda()
    delta = uniform_bf16((T, d), 5, 2, 1.0).cuda() if with_delta else None
    w = (1 + uniform_bf16((d,), 5, 3, 0.2).float()).bfloat16().cuda()
    xo, y = torch.empty_like(x), torch.empty_like(x)
    ops.add_rmsnorm(x, w, 1e-6, y, delta=delta, x_out=xo)  # warp path
    xo2, y2 = torch.empty_like(x), torch.empty_like(x)
    for s0 in range(0, T, 1000):  # CTA-per-token path (T < 1024 per launch)
        s1 = min(T, s0 + 1000)
        ops.add_rmsnorm(x[s0:s1], w, 1e-6, y2[s0:s1], delta=None if delta is None else delta[s0:s1], x_out=xo2[s0:s1])
    torch.cuda.synchronize()
    assert torch.equal(xo, xo2)
    dy = (y.float() - y2.float()).abs()
    assert float((dy > 0).float().mean()) < 2e-3
    assert float(dy.max()) <= float(y2.float().abs().max()) * 2 ** -7
