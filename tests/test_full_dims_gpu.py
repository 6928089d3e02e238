"""Parity at the BASELINE configs' real layer dimensions (not the tiny stand-ins): the engine's decode
step for Mixtral-8x7B (d 4096, f 14336, 32/8 heads, V 32000), DeepSeek-V2-Lite (d 2048, 64+2
experts top-6, MLA 512+64, V 102400), Mixtral-8x22B (d 6144, f 16384, 48/8 heads) and DeepSeek-V2
236B (d 5120, 160+2 experts, group-limited top-6, q_lora 1536, 128 heads), truncated in depth so the CPU oracle finishes in seconds,
vs oracle/moe_ref.py on the very same weights (copied from the engine, which generates them with
the counter-based generator the oracle mirrors).

Checks per teacher-forced step: routing (top-k expert sets) equal on >= 99 % of tokens given the
same inputs to the first MoE layer, logits within the north_star bf16 tolerance (median row
max-abs error / row max <= 2e-2, median row cosine >= 0.999), and the greedy argmax identical on every row
whose oracle top1-top2 margin exceeds 4x the largest |delta logit| of the step.
"""

import dataclasses

import pytest
import torch

from oracle import moe_ref as R

pytestmark = pytest.mark.gpu


def _oracle_weights(eng):
    """The engine's weights in the oracle's layout (CPU copies)."""
    a, w = eng.arch, eng.w
    layers = []
    for L in w.layers:
        c = {k: v.cpu() for k, v in L.items() if k not in ("w_uk", "w_uv_t") and v is not None}
        if a.family == "mixtral":
            hd = a.head_dim
            qd, kvd = a.n_heads * hd, a.n_kv_heads * hd
            wqkv = c.pop("wqkv")
            c.update(wq=wqkv[:qd], wk=wqkv[qd:qd + kvd], wv=wqkv[qd + kvd:])
        else:
            for k in ("sh_gate_up", "sh_down", "dense_gate_up", "dense_down"):
                if k in c:
                    c[k] = c[k][0]
        layers.append(c)
    return R.MixtralWeights(embed=w.embed.cpu(), final_norm=w.final_norm.cpu(), lm_head=w.lm_head.cpu(),
                            layers=layers)


@pytest.mark.parametrize("name,layers", [("mixtral-8x7b", 2), ("deepseek-v2-lite", 2), ("mixtral-8x22b", 1),
                                         ("deepseek-v2-236b", 2)])
def test_full_dims_decode_vs_oracle(name, layers):
    from paper_2503_09716_b200.configs import get_arch
    from paper_2503_09716_b200.engine import Engine
    from paper_2503_09716_b200.planner import BatchingPlan, ModelSpec

    A = dataclasses.replace(get_arch(name), layers=layers)
    B, steps = 48, 3
    mb = ModelSpec.from_document(A.model_spec_document()).model_bytes
    eng = Engine(A, BatchingPlan(B, B, 4096, 0.0, 0, mb), prompt_len=steps, decode_len=1, use_graph=False)
    W = _oracle_weights(eng)
    orc = (R.DeepseekV2Oracle if A.family == "deepseek_v2" else R.MixtralOracle)(A, W)
    toks = torch.randint(0, A.vocab, (B, steps), generator=torch.Generator().manual_seed(5))
    for pos in range(steps):
        eng.debug_taps = {}
        le = eng.debug_forward(toks[:, pos], pos)["logits"].cpu().float()
        traces = [dict() for _ in range(A.layers)]
        lo = orc.step(toks[:, pos], pos, traces=traces).float()
        # routing given the engine's own router input: the oracle's top-k on the same hidden state
        h2 = eng.debug_taps["h2"].cpu()
        idx_e = eng.debug_taps["topk_idx"].cpu().long()
        wr = W.layers[A.layers - 1]["router"]
        if A.family == "deepseek_v2":  # fp32 gate (modeling_deepseek_v2.py:125)
            logits_r = torch.nn.functional.linear(h2.float(), wr.float())
        else:                          # bf16 gate (modeling_mixtral.py:111)
            logits_r = torch.nn.functional.linear(h2, wr)
        idx_o, _ = R.route(logits_r, A.top_k, A.router_mode, A.routed_scaling, A.n_group, A.topk_group)
        same = (idx_e.sort(-1).values == idx_o.long().sort(-1).values).all(-1).float().mean().item()
        assert same >= 0.99, f"{name} pos {pos}: routing agreement {same}"
        rows = [((le[i] - lo[i]).abs().max() / lo[i].abs().max()).item() for i in range(B)]
        rows.sort()
        # a near-tied bf16 router logit may send one token to another expert, so
        # the bar is on the median row; routing above is checked given identical router inputs
        cos = torch.nn.functional.cosine_similarity(le, lo, dim=-1).median().item()
        assert rows[B // 2] <= 2e-2 and cos >= 0.999, f"{name} pos {pos}: median {rows[B // 2]:.3e} cos {cos:.5f}"
        delta = (le - lo).abs().max().item()
        top2 = lo.topk(2, dim=-1).values
        safe = (top2[:, 0] - top2[:, 1]) > 4 * delta
        assert torch.equal(le.argmax(-1)[safe], lo.argmax(-1)[safe])
