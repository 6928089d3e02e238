"""Pins the CPU oracle (oracle/moe_ref.py) against HF transformers 5.5.0 run on the same
counter-based weights (tests/golden/hf_tiny_mixtral.pt, produced by tests/golden/make_golden.py),
and checks the oracle's pinned orders (routing tie rule, stable permutation) as properties."""

import os

import pytest
import torch
from hypothesis import given, settings
from hypothesis import strategies as st

from oracle import moe_ref as R
from oracle.rng import uniform_bf16
from paper_2503_09716_b200.configs import TINY

GOLD = torch.load(os.path.join(os.path.dirname(__file__), "golden", "hf_tiny_mixtral.pt"), weights_only=False)


@pytest.fixture(scope="module")
def weights():
    return R.make_mixtral_weights(TINY, seed=0)


def _prefill(orc, ids):
    B, P = ids.shape
    hs = None
    logits = None
    for p in range(P):
        tr = [] if p == P - 1 else None
        logits = orc.step(ids[:, p], p, traces=tr)
        if tr is not None:
            hs = tr
    return logits, hs


def test_oracle_matches_hf_forward(weights):
    """Per-layer hidden state at the last prompt position and the logits, HF (sdpa attention,
    grouped_mm experts) vs the oracle: rel err <= 2e-2, cosine >= 0.999."""
    orc = R.MixtralOracle(TINY, weights)
    ids = GOLD["input_ids"]
    logits, traces = _prefill(orc, ids)
    hf_h = GOLD["hidden_states"]  # [embeddings, layer1, ..., final-normed]
    k = TINY.top_k
    routed_same = torch.ones(ids.shape[0], dtype=torch.bool)
    for l in range(TINY.layers):
        hf_lg = GOLD["router_logits"][l].float()
        hf_sets = torch.topk(hf_lg, k, -1).indices.sort(-1).values
        same = (traces[l]["topk_idx"].sort(-1).values == hf_sets).all(-1)
        # a routing difference is only legitimate on a bf16 near-tie of HF's k-th/(k+1)-th logit
        gap = torch.topk(hf_lg, k + 1, -1).values
        gap = gap[:, k - 1] - gap[:, k]
        assert bool((same | (gap < 0.02)).all())
        routed_same &= same
        if l < TINY.layers - 1:  # HF's last hidden state is post final-norm
            for i in range(ids.shape[0]):
                if routed_same[i]:
                    assert R.rel_err(traces[l]["x_out"][i], hf_h[l + 1][i]) <= 2e-2
    assert routed_same.float().mean() >= 0.5
    for i in range(ids.shape[0]):
        if routed_same[i]:
            assert R.rel_err(logits[i], GOLD["last_logits"][i]) <= 2e-2
    assert R.cosine(logits, GOLD["last_logits"]) >= 0.99


def test_oracle_routing_matches_hf_router(weights):
    """Given HF's own router logits, the oracle's expert sets equal HF's top-k sets."""
    for lg in GOLD["router_logits"]:
        idx, w = R.route(lg.float(), TINY.top_k, 0)
        hf = torch.topk(torch.softmax(lg.float(), -1), TINY.top_k, dim=-1)
        assert torch.equal(idx.sort(-1).values, hf.indices.sort(-1).values)
        torch.testing.assert_close(w.sort(-1).values, (hf.values / hf.values.sum(-1, keepdim=True)).sort(-1).values)


def test_oracle_greedy_vs_hf_margin_filtered(weights):
    """Greedy tokens: identical on every teacher-forced step whose HF top1-top2 margin exceeds
    4x the max observed |delta logit|; reports the unfiltered identical prefix."""
    orc = R.MixtralOracle(TINY, weights)
    gen = GOLD["generated"]
    P, N = GOLD["meta"]["P"], GOLD["meta"]["N"]
    top_v, top_i = GOLD["tf_top16_values"], GOLD["tf_top16_indices"]
    steps = []
    for p in range(P + N - 1):
        lg = orc.step(gen[:, p], p)
        if p >= P - 1:
            steps.append(lg)
    maxdelta = 0.0
    for n, lg in enumerate(steps):
        ref_v = top_v[:, n]
        mine = torch.gather(lg.float(), 1, top_i[:, n])
        maxdelta = max(maxdelta, (mine - ref_v).abs().max().item())
    for n, lg in enumerate(steps):
        margin = top_v[:, n, 0] - top_v[:, n, 1]
        agree = torch.argmax(lg.float(), -1) == top_i[:, n, 0]
        assert bool((agree | (margin <= 4 * maxdelta)).all())


def test_rng_deterministic_and_distribution():
    a = uniform_bf16((1000, 100), 3, 9, 0.02)
    b = uniform_bf16((1000, 100), 3, 9, 0.02)
    assert torch.equal(a, b)
    assert not torch.equal(a, uniform_bf16((1000, 100), 3, 10, 0.02))
    assert abs(a.float().std().item() - 0.02) < 1e-3 and abs(a.float().mean().item()) < 1e-3
    # counter-based: a prefix of a larger tensor is the smaller tensor
    assert torch.equal(uniform_bf16((50,), 3, 9, 0.02), a.view(-1)[:50])


@settings(max_examples=60, deadline=None)
@given(T=st.integers(1, 40), E=st.sampled_from([4, 8, 16, 64]), k=st.integers(1, 4), seed=st.integers(0, 10**6))
def test_route_tie_rule_and_permutation_properties(T, E, k, seed):
    k = min(k, E)
    g = torch.Generator().manual_seed(seed)
    lg = torch.randint(-3, 3, (T, E), generator=g).float()  # many exact ties
    idx, w = R.route(lg, k, 0)
    for t in range(T):
        row = lg[t]
        sel = idx[t].tolist()
        # value descending, index ascending on ties
        keyed = sorted(range(E), key=lambda e: (-row[e].item(), e))[:k]
        assert sel == keyed
    order, dst, counts, offsets = R.permutation(idx, E)
    flat = idx.reshape(-1)
    assert torch.equal(flat[order], flat[order].sort(stable=True).values)  # expert-major
    for e in range(E):
        rows = order[offsets[e]:offsets[e + 1]]
        assert torch.equal(rows, rows.sort().values)  # token order kept within an expert
    assert torch.equal(order[dst], torch.arange(T * k))
    assert int(offsets[-1]) == T * k
    torch.testing.assert_close(w.sum(-1), torch.ones(T))


def test_group_limited_routing_respects_groups():
    g = torch.Generator().manual_seed(0)
    lg = torch.randn(64, 160, generator=g)
    idx, w = R.route(lg, 6, 2, scaling=16.0, n_group=8, topk_group=3)
    groups = idx // 20
    assert all(len(set(r.tolist())) <= 3 for r in groups)
    gmax = lg.view(64, 8, 20).max(-1).values
    best3 = torch.sort(-gmax, dim=-1, stable=True).indices[:, :3].sort(-1).values
    for t in range(64):
        assert set(groups[t].tolist()) <= set(best3[t].tolist())
    probs = torch.softmax(lg, -1)
    torch.testing.assert_close(w, torch.gather(probs, 1, idx) * 16.0)


def test_dsv2_oracle_matches_hf():
    """DeepSeek-V2 family (MLA, fp32 group-limited router, shared experts, dense layer 0): the
    oracle vs HF DeepseekV2ForCausalLM on the same counter-based weights."""
    from paper_2503_09716_b200.configs import TINY_DSV2 as A

    G = torch.load(os.path.join(os.path.dirname(__file__), "golden", "hf_tiny_dsv2.pt"), weights_only=False)
    w = R.make_dsv2_weights(A, seed=0)
    orc = R.DeepseekV2Oracle(A, w)
    ids = G["input_ids"]
    for p in range(ids.shape[1]):
        tr = []
        lg = orc.step(ids[:, p], p, traces=tr)
    for l in range(A.layers - 1):
        assert R.rel_err(tr[l]["x_out"], G["hidden_states"][l + 1]) <= 2e-2
    assert R.rel_err(lg, G["last_logits"]) <= 2e-2
    gen = R.DeepseekV2Oracle(A, w).generate(ids, G["meta"]["N"])
    assert (gen == G["generated"]).all(1).float().mean() >= 0.75
