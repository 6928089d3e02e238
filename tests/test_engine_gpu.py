"""End-to-end parity of the B200 engine vs the CPU oracle on the tiny Mixtral config (cfg0 shape,
scaled down in B/prompt so the pure-CPU oracle finishes in seconds).

Criteria (BASELINE.json north_star):
  - per-layer hidden states (test_per_layer_hidden_states): max|a-b|/max|b| <= 2e-2 per layer;
  - per-step logits under teacher forcing (no per-layer re-synchronisation, so a near-tied bf16 router
    logit may route one token differently): median row error <= 2e-2 and cosine >= 0.99;
  - greedy argmax identical on every step whose oracle top1-top2 margin exceeds 4x the max
    |delta logit| observed on that run;
  - CUDA-graph replay == eager issue, bit for bit.
"""

import pytest
import torch

from oracle import moe_ref as R

pytestmark = pytest.mark.gpu

TOL = 2e-2


def _engine(B=8, prompt=6, decode=10, use_graph=False):
    from paper_2503_09716_b200.configs import TINY
    from paper_2503_09716_b200.engine import Engine
    from paper_2503_09716_b200.planner import BatchingPlan

    spec_bytes = None
    plan = BatchingPlan(B=B, b_a=max(1, B // 2), b_e=16, omega=0.0, s_expert=0,
                        s_params=_model_bytes(TINY))
    return Engine(TINY, plan, prompt_len=prompt, decode_len=decode, seed=0, use_graph=use_graph)


def _model_bytes(arch):
    from paper_2503_09716_b200.planner import ModelSpec

    return ModelSpec.from_document(arch.model_spec_document()).model_bytes


@pytest.fixture(scope="module")
def oracle_weights():
    from paper_2503_09716_b200.configs import TINY

    return R.make_mixtral_weights(TINY, seed=0)


def test_weights_bit_identical(oracle_weights):
    eng = _engine()
    w = oracle_weights
    assert torch.equal(eng.w.embed.cpu(), w.embed)
    assert torch.equal(eng.w.lm_head.cpu(), w.lm_head)
    L0 = eng.w.layers[0]
    a = eng.arch
    qd, kvd = a.n_heads * a.head_dim, a.n_kv_heads * a.head_dim
    assert torch.equal(L0["wqkv"][:qd].cpu(), w.layers[0]["wq"])
    assert torch.equal(L0["wqkv"][qd + kvd:].cpu(), w.layers[0]["wv"])
    assert torch.equal(L0["w_gate_up"].cpu(), w.layers[0]["w_gate_up"])
    assert torch.equal(eng.w.layers[-1]["w_down"].cpu(), w.layers[-1]["w_down"])


def test_teacher_forced_logits(oracle_weights):
    from paper_2503_09716_b200.configs import TINY

    B, P, N = 8, 6, 10
    eng = _engine(B, P, N)
    orc = R.MixtralOracle(TINY, oracle_weights)
    g = torch.Generator().manual_seed(1)
    toks = torch.randint(0, TINY.vocab, (B, P + N), generator=g)
    row_errs, cos_min, maxdelta = [], 1.0, 0.0
    margins, flips = [], []
    for pos in range(P + N):
        lo = orc.step(toks[:, pos], pos)
        le = eng.debug_forward(toks[:, pos], pos)["logits"].cpu()
        row_errs += [R.rel_err(le[i], lo[i]) for i in range(B)]
        cos_min = min(cos_min, R.cosine(le, lo))
        maxdelta = max(maxdelta, (le.float() - lo.float()).abs().max().item())
        margins.append(R.softmax_margin(lo))
        flips.append(torch.argmax(le.float(), -1) != torch.argmax(lo.float(), -1))
    # without re-synchronisation a near-tied bf16 router logit may legitimately pick another
    # expert for one token; the per-layer bar is test_per_layer_hidden_states.
    row_errs.sort()
    print(f"teacher-forced logits: median row rel err {row_errs[len(row_errs) // 2]:.2e}, "
          f"p90 {row_errs[int(0.9 * len(row_errs))]:.2e}, min cosine {cos_min:.5f}, max|dlogit| {maxdelta:.3e}")
    assert row_errs[len(row_errs) // 2] <= TOL
    assert cos_min >= 0.99
    for m, f in zip(margins, flips):
        assert not bool((f & (m > 4 * maxdelta)).any())


def test_graph_replay_equals_eager():
    B, P, N = 8, 4, 6
    e1 = _engine(B, P, N, use_graph=False)
    e2 = _engine(B, P, N, use_graph=True)
    ids = torch.randint(0, 32000, (B, P), generator=torch.Generator().manual_seed(3))
    o1 = e1.generate(ids, N)
    o2 = e2.generate(ids, N)
    assert torch.equal(o1, o2)
    assert torch.equal(e1.buf.logits.cpu(), e2.buf.logits.cpu())


def test_generate_matches_oracle_prefix(oracle_weights):
    from paper_2503_09716_b200.configs import TINY

    B, P, N = 8, 6, 8
    eng = _engine(B, P, N, use_graph=True)
    ids = torch.randint(0, TINY.vocab, (B, P), generator=torch.Generator().manual_seed(5))
    out = eng.generate(ids, N)
    orc = R.MixtralOracle(TINY, oracle_weights)
    ref, _ = orc.generate(ids, N)
    assert out.shape == ref.shape
    assert torch.equal(out[:, :P], ids)
    # report-only: rows whose whole greedy continuation matches (bf16 ties can legitimately flip)
    same = (out == ref).all(dim=1).float().mean().item()
    print(f"identical greedy rows: {same:.2f}")
    assert same >= 0.5


def test_per_layer_hidden_states(oracle_weights):
    """Layer-by-layer (residual stream re-synchronised to the oracle after every layer):
    hidden state, attention output and routing per layer."""
    from paper_2503_09716_b200 import ops
    from paper_2503_09716_b200.configs import TINY

    B, P, N = 8, 6, 10
    eng = _engine(B, P, N)
    orc = R.MixtralOracle(TINY, oracle_weights)
    toks = torch.randint(0, TINY.vocab, (B, P + N), generator=torch.Generator().manual_seed(1))
    route_equal = 0
    total = 0
    for pos in range(5):
        eng.buf.positions.fill_(pos)
        eng.buf.next_ids.copy_(toks[:, pos].to(torch.int32))
        ops.embed(eng.buf.next_ids, eng.w.embed, eng.buf.x)
        x = orc.w.embed[toks[:, pos]]
        assert torch.equal(eng.buf.x.cpu(), x)
        for l in range(TINY.layers):
            tr = {}
            x = orc.layer_forward(l, x, pos, tr)
            eng.debug_taps = {}
            eng._issue_layer(l)
            torch.cuda.synchronize()
            b, taps = eng.buf, eng.debug_taps
            eng.debug_taps = None
            assert R.rel_err(taps["attn"].cpu(), tr["attn"]) <= TOL
            assert R.rel_err(taps["h2"].cpu(), tr["h2"]) <= TOL
            assert R.rel_err(b.x.cpu(), x) <= TOL
            total += 1
            eng_idx = taps["topk_idx"].cpu().long()
            route_equal += int(torch.equal(eng_idx, tr["topk_idx"]))
            # bit-exact routing given identical logits: re-route the engine's own logits on the CPU
            lg = torch.zeros(B, TINY.n_experts, device="cuda")
            ws2 = ops.RouterWorkspace(B, TINY.n_experts, TINY.top_k)
            ops.router_topk(taps["h2"], eng.w.layers[l]["router"], ws2, TINY.top_k, 0, logits_out=lg)
            assert torch.equal(ws2.topk_idx.cpu().long(), eng_idx)
            assert torch.equal(R.route(lg.cpu(), TINY.top_k, 0)[0], eng_idx)
            b.x.copy_(x)  # re-synchronise the residual stream (and the fused next-layer norm)
            nxt = eng.w.layers[l + 1]["ln1"] if l + 1 < TINY.layers else eng.w.final_norm
            ops.add_rmsnorm(b.x, nxt, TINY.rms_eps, b.h)
    # end-to-end (not re-synchronised) routing may flip on bf16 near-ties
    assert route_equal >= 0.9 * total


def test_offloaded_weights_match_resident_bit_exact():
    """Module-based batching with weights partly in pinned host memory (prefetch subsystem):
    uncached dense layers / experts (reference cache_placement) are streamed on the H2D copy
    stream into the dense buffer / expert slots; outputs must equal the fully resident engine bit
    for bit, eagerly and under CUDA-graph replay, and the trace's H2D bytes = uncached bytes."""
    from paper_2503_09716_b200.configs import TINY
    from paper_2503_09716_b200.engine import Engine
    from paper_2503_09716_b200.planner import BatchingPlan, ModelSpec, placement

    spec = ModelSpec.from_document(TINY.model_spec_document())
    dense, ex = spec.dense_bytes_per_layer, spec.expert_bytes
    B, P, N = 8, 4, 5
    res_plan = BatchingPlan(B, 4, 16, 0.0, 0, spec.model_bytes)
    ids = torch.randint(0, TINY.vocab, (B, P), generator=torch.Generator().manual_seed(11))
    ref = Engine(TINY, res_plan, prompt_len=P, decode_len=N, use_graph=False).generate(ids, N, prefill=False)
    for s_params, slots in ((2 * dense + dense // 2, 2), (4 * dense + 10 * ex, 3)):
        off_plan = BatchingPlan(B, 4, 16, 0.0, slots * ex, s_params)
        pl = placement(spec, s_params)  # reference cache_placement (memory_model.py:147-164)
        assert pl.uncached_expert_count > 0
        for graph in (False, True):
            eng = Engine(TINY, off_plan, prompt_len=P, decode_len=N, use_graph=graph)
            assert eng.offload and eng.w.n_slots == slots
            assert torch.equal(eng.generate(ids, N), ref)
        recs, rep = eng.trace_step()
        uncached = (TINY.layers - pl.dense_layers) * dense + pl.uncached_expert_count * ex
        assert rep["bytes_htod"] == uncached
        assert {r["kind"] for r in recs} >= {"weight_copy", "expert_compute", "router"}


@pytest.mark.parametrize("P,chunk", [(6, 32768), (70, 140)])  # one chunk; several chunks across a page
def test_batched_prefill_matches_tokenwise(oracle_weights, P, chunk):
    """Engine.prefill (the prefill phase: all P prompt tokens per forward, causal attention, paged KV
    written for every position) vs consuming the prompt through the decode step one position at a
    time: logits at the last prompt position within the bf16 tolerance, the paged KV close, and
    the oracle agrees on the margin-filtered first token."""
    from paper_2503_09716_b200.configs import TINY

    B, N = 8, 4
    ids = torch.randint(0, TINY.vocab, (B, P), generator=torch.Generator().manual_seed(21))
    e_pf, e_tw = _engine(B, P, N), _engine(B, P, N)
    first = e_pf.prefill(ids, chunk_tokens=chunk)
    lg_pf = e_pf.buf.logits.cpu().float()
    e_tw.reset(0)
    for p in range(P):
        e_tw.buf.next_ids.copy_(ids[:, p].cuda().int())
        e_tw.run_step()
    lg_tw = e_tw.buf.logits.cpu().float()
    rows = sorted(((lg_pf[i] - lg_tw[i]).abs().max() / lg_tw[i].abs().max()).item() for i in range(B))
    assert rows[B // 2] <= 2e-2, rows
    kc_pf, kc_tw = e_pf.k_cache[0].float(), e_tw.k_cache[0].float()
    assert (kc_pf - kc_tw).abs().max().item() <= 2e-2 * kc_tw.abs().max().item()  # layer 0 K: same inputs
    assert int(e_pf.buf.positions[0]) == P and e_pf.host_pos == P
    orc = R.MixtralOracle(TINY, oracle_weights)
    for p in range(P):
        lo = orc.step(ids[:, p], p).float()
    delta = (lg_pf - lo).abs().max().item()
    top2 = lo.topk(2, dim=-1).values
    safe = (top2[:, 0] - top2[:, 1]) > 4 * delta
    assert torch.equal(first[safe], lo.argmax(-1)[safe])
    out = e_pf.generate(ids, N)  # prefill + graph-replayed decode through the public API
    assert out.shape == (B, P + N) and torch.equal(out[:, P], first)
