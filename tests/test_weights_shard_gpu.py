"""Expert-parallel weight shards generated in place (weights.routed_experts_, mgb_fill_uniform_bf16_range):
a rank's experts [lo, lo + n) equal the same slice of the whole-model tensors, bit for bit, so EP ranks
never materialise the other ranks' experts (DeepSeek-V2 236B EP8: 20 of 160 experts per layer)."""

import pytest
import torch

from paper_2503_09716_b200.configs import get_arch

pytestmark = pytest.mark.gpu


def test_fill_range_equals_slice():
    from paper_2503_09716_b200.weights import fill_uniform_

    n = 10_000_019
    full = fill_uniform_(torch.empty(n, dtype=torch.bfloat16, device="cuda"), 3, 1234, 0.02)
    for first, m in [(0, 1000), (1, 7), (4_999_999, 3_000_001), (n - 5, 5)]:
        part = fill_uniform_(torch.empty(m, dtype=torch.bfloat16, device="cuda"), 3, 1234, 0.02, first=first)
        assert torch.equal(part, full[first:first + m]), (first, m)


@pytest.mark.parametrize("cfg,shard", [("tiny-mixtral", (2, 3)), ("deepseek-v2-lite", (48, 16))])
def test_layer_shard_equals_slice(cfg, shard):
    from paper_2503_09716_b200 import weights as Wt

    a = get_arch(cfg)
    build = Wt.deepseek_layer if a.is_mla else Wt.mixtral_layer
    l = a.first_k_dense if a.is_mla else 1
    full = build(a, l, 0, "cuda")
    part = build(a, l, 0, "cuda", None, shard)
    lo, n = shard
    for k in full:
        if k in ("w_gate_up", "w_down"):
            assert part[k].shape[0] == n
            assert torch.equal(part[k], full[k][lo:lo + n]), k
        elif k not in Wt.DERIVED:
            assert torch.equal(part[k], full[k]), k
