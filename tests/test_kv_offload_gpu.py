"""kv_policy="offload": the reference's full-KV-offload mode (memory_model.py:182-205).

Every sequence's KV pages live in pinned host memory; per layer and attention micro-batch the
engine streams the slice into an HBM ring slot (KV_COPY_IN), appends the new token into staging
pages (PRE_ATTENTION), writes it back to the host store (KV_COPY_OUT, offload_dag.py:372-392) and
attends over the slot.  Same kernels, same data => outputs must equal the HBM-resident engine bit
for bit, eagerly and under CUDA-graph replay, across page boundaries and ring-slot reuse.
"""

import pytest
import torch

pytestmark = pytest.mark.gpu


def _plan(arch, B, b_a):
    from paper_2503_09716_b200.planner import BatchingPlan, ModelSpec

    mb = ModelSpec.from_document(arch.model_spec_document()).model_bytes
    return BatchingPlan(B, b_a, 16, 0.0, 0, mb)


@pytest.mark.parametrize("unit,n_units,page", [(16, 16, 64), (128, 9, 56)])
@pytest.mark.parametrize("host_dst", [False, True])
def test_kv_token_copy(unit, n_units, page, host_dst):
    """mgb_kv_token_copy moves exactly the new token's runs (device->device and device->mapped host)."""
    from paper_2503_09716_b200 import _native as nat

    B, pps = 5, 3
    page_bytes = n_units * unit * page
    src = torch.randint(0, 255, (B * pps * page_bytes,), dtype=torch.uint8, device="cuda")
    dst = torch.zeros(B * pps * page_bytes, dtype=torch.uint8)
    if host_dst:  # registered in place, as the engine's host stores are (hostmem.py)
        from paper_2503_09716_b200.hostmem import pinned_empty

        dst = pinned_empty(dst.numel(), torch.uint8).zero_()
    else:
        dst = dst.cuda()
    src_table = torch.randperm(B * pps, dtype=torch.int32).view(B, pps).cuda()
    dst_table = torch.randperm(B * pps, dtype=torch.int32).view(B, pps).cuda()
    pos = torch.tensor([0, page - 1, page, 2 * page + 7, 3 * page - 1], dtype=torch.int32, device="cuda")
    nat.call("mgb_kv_token_copy", src.data_ptr(), src_table.data_ptr(), pps, dst.data_ptr(), dst_table.data_ptr(),
             pps, pos.data_ptr(), B, page, page_bytes, unit, n_units, unit * page,
             torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    exp = torch.zeros(B * pps * page_bytes, dtype=torch.uint8)
    s, st, dt, p = src.cpu(), src_table.cpu(), dst_table.cpu(), pos.cpu()
    for b in range(B):
        pg, slot = int(p[b]) // page, int(p[b]) % page
        for u in range(n_units):
            o = u * unit * page + slot * unit
            exp[int(dt[b, pg]) * page_bytes + o:int(dt[b, pg]) * page_bytes + o + unit] = \
                s[int(st[b, pg]) * page_bytes + o:int(st[b, pg]) * page_bytes + o + unit]
    assert torch.equal(dst.cpu(), exp)


@pytest.mark.parametrize("family", ["mixtral", "deepseek_v2"])
def test_kv_offload_generate_equals_resident(family):
    from paper_2503_09716_b200.configs import TINY, TINY_DSV2
    from paper_2503_09716_b200.engine import Engine

    A = TINY if family == "mixtral" else TINY_DSV2
    B, P, N = 8, 5, 6
    plan = _plan(A, B, 3)  # micro-batches of 3, 3, 2 sequences
    ids = torch.randint(0, A.vocab, (B, P), generator=torch.Generator().manual_seed(21))
    res = Engine(A, plan, prompt_len=P, decode_len=N, use_graph=False)
    ref = res.generate(ids, N, prefill=False)
    ref_pf = res.generate(ids, N)  # batched prefill (KV written to the host store through staging)
    for graph in (False, True):
        eng = Engine(A, plan, prompt_len=P, decode_len=N, use_graph=graph, kv_policy="offload", kv_ring_slots=2)
        assert not eng.kv[0][0].is_cuda and eng.kv_ring_n == 2
        # host pages start as garbage: every row a step reads past a sequence's length must be
        # ignored (0 * NaN would poison P.V), so fill the whole host store with NaN first
        eng.kv_host.fill_(float("nan"))
        assert torch.equal(eng.generate(ids, N, prefill=False), ref)
        eng.kv_host.fill_(float("nan"))
        assert torch.equal(eng.generate(ids, N), ref_pf)


@pytest.mark.parametrize("family", ["mixtral", "deepseek_v2"])
def test_kv_offload_decode_across_pages(family):
    """Synthetic prefill into the host store, then decode across a page boundary (GQA pages hold
    64 tokens, MLA pages 56): tokens equal the resident engine's; the trace's H2D/D2H bytes are the
    schedule's KV_COPY_IN / KV_COPY_OUT bytes."""
    from paper_2503_09716_b200.configs import TINY, TINY_DSV2
    from paper_2503_09716_b200.engine import Engine

    A = TINY if family == "mixtral" else TINY_DSV2
    B, P, N = 6, 52, 14
    plan = _plan(A, B, 4)
    first = torch.randint(0, A.vocab, (B,), generator=torch.Generator().manual_seed(3))
    outs = []
    for policy in ("resident", "offload"):
        eng = Engine(A, plan, prompt_len=P, decode_len=N, use_graph=True, kv_policy=policy)
        eng.synthetic_prefill(seed=5, std=1.0)
        outs.append(eng.decode(first, N))
    assert torch.equal(outs[0], outs[1])
    recs, rep = eng.trace_step()
    kv = A.kv_bytes_per_token_layer
    assert rep["bytes_htod"] == A.layers * B * (P + N) * kv
    assert rep["bytes_dtoh"] == A.layers * B * kv
    assert {r["kind"] for r in recs} >= {"kv_copy_in", "kv_copy_out", "attn_mech_gpu"}


def test_dsv2_offloaded_weights_and_kv_match_resident():
    """DeepSeek-V2 module-based batching with weights partly in pinned host memory (dense modules =
    MLA projections + shared experts through the single dense buffer; routed experts through the
    slots) and, on top, the KV store offloaded: bit-identical to the resident engine; the trace's
    H2D bytes are the uncached weight bytes plus the KV_COPY_IN bytes."""
    from paper_2503_09716_b200.configs import TINY_DSV2 as A
    from paper_2503_09716_b200.engine import Engine
    from paper_2503_09716_b200.planner import BatchingPlan, ModelSpec, placement

    spec = ModelSpec.from_document(A.model_spec_document())
    dense, ex = spec.dense_bytes_per_layer, spec.expert_bytes
    B, P, N = 8, 4, 5
    ids = torch.randint(0, A.vocab, (B, P), generator=torch.Generator().manual_seed(13))
    ref = Engine(A, BatchingPlan(B, 4, 16, 0.0, 0, spec.model_bytes), prompt_len=P, decode_len=N,
                 use_graph=False).generate(ids, N, prefill=False)
    two_layers = 2 * dense + ((dense - 1) // ex) * ex  # 2 dense layers cached + a few experts
    for s_params, slots, policy in ((dense + dense // 2, 2, "resident"), (two_layers, 3, "offload")):
        plan = BatchingPlan(B, 4, 16, 0.0, slots * ex, s_params)
        pl = placement(spec, s_params)
        assert pl.uncached_expert_count > 0 and pl.dense_layers < A.layers
        for graph in (False, True):
            eng = Engine(A, plan, prompt_len=P, decode_len=N, use_graph=graph, kv_policy=policy)
            assert eng.offload
            assert torch.equal(eng.generate(ids, N, prefill=False), ref), (s_params, policy, graph)
        recs, rep = eng.trace_step()
        uncached = (A.layers - pl.dense_layers) * dense + pl.uncached_expert_count * ex
        # the reference's all-MoE model charges experts to the dense first layer too: none move
        phantom = sum(A.n_experts - pl.experts_per_layer[l] for l in range(A.first_k_dense)) * ex
        kv_in = A.layers * B * (P + N) * A.kv_bytes_per_token_layer if policy == "offload" else 0
        assert rep["bytes_htod"] == uncached - phantom + kv_in


def test_cpu_attention_share_matches_gpu_engine():
    """omega > 0 (MoE-Gen(H)): the first round(omega*B) sequences attend on the host cores over the
    host page store (ATTN_MECH_CPU as a host node of the step graph), the rest on the GPU.
    1. On a one-layer model (identical inputs, identical KV history) the attention outputs of the CPU
       share match the all-GPU engine's within bf16 tolerance at every position, across a page.
    2. End to end (4 layers, teacher forced) the logits keep the per-layer bar (median row error
       <= 2e-2; a near-tied bf16 router logit may flip an expert).
    3. Greedy decode runs eagerly and as a CUDA graph with identical results."""
    import dataclasses

    from paper_2503_09716_b200.configs import TINY as A
    from paper_2503_09716_b200.engine import Engine
    from paper_2503_09716_b200.planner import BatchingPlan, ModelSpec

    def engines(arch, P, N):
        mb = ModelSpec.from_document(arch.model_spec_document()).model_bytes
        ref = Engine(arch, BatchingPlan(8, 4, 16, 0.0, 0, mb), prompt_len=P, decode_len=N, use_graph=False)
        cpu = Engine(arch, BatchingPlan(8, 2, 16, 0.5, 0, mb), prompt_len=P, decode_len=N, use_graph=False,
                     kv_policy="offload")
        return ref, cpu

    B, P, N = 8, 6, 70  # crosses a 64-token page
    toks = torch.randint(0, A.vocab, (B, P + N), generator=torch.Generator().manual_seed(17))
    ref, cpu = engines(dataclasses.replace(A, layers=1), P, N)
    assert cpu.n_cpu == 4 and cpu.cpu_stream is not None
    worst = 0.0
    for pos in range(P + N):
        outs = []
        for e in (ref, cpu):
            e.debug_taps = {}
            e.debug_forward(toks[:, pos], pos)
            outs.append(e.debug_taps["attn"][:4].float())
        worst = max(worst, ((outs[0] - outs[1]).abs().max() / outs[0].abs().max()).item())
    assert worst <= 1e-2, worst
    ref, cpu = engines(A, P, N)
    errs = []
    for pos in range(P + N):
        lr = ref.debug_forward(toks[:, pos], pos)["logits"].float()
        lc = cpu.debug_forward(toks[:, pos], pos)["logits"].float()
        errs += [((lr[i] - lc[i]).abs().max() / lr[i].abs().max()).item() for i in range(B)]
    errs.sort()
    assert errs[len(errs) // 2] <= 2e-2, errs[len(errs) // 2]
    mb = ModelSpec.from_document(A.model_spec_document()).model_bytes
    outs = [Engine(A, BatchingPlan(B, 2, 16, 0.5, 0, mb), prompt_len=P, decode_len=N, use_graph=g,
                   kv_policy="offload").generate(toks[:, :P], 8) for g in (False, True)]
    assert torch.equal(outs[0], outs[1])
    cpu.reset(P)
    recs, rep = cpu.trace_step()
    assert rep["busy"].get("cpu_compute", 0.0) > 0 and {r["kind"] for r in recs} >= {"attn_mech_cpu", "kv_copy_out"}


@pytest.mark.parametrize("family", ["mixtral", "deepseek_v2"])
def test_streamed_prefill_with_offloaded_weights(family):
    """Prefill with offloaded weights runs layer-major (each streamed module crosses the link once
    per layer for all prompt tokens, experts double-buffered through two slots): the first tokens
    and the last-position logits match the resident engine's chunked prefill."""
    from paper_2503_09716_b200.configs import TINY, TINY_DSV2
    from paper_2503_09716_b200.engine import Engine
    from paper_2503_09716_b200.planner import BatchingPlan, ModelSpec

    A = TINY if family == "mixtral" else TINY_DSV2
    spec = ModelSpec.from_document(A.model_spec_document())
    dense, ex = spec.dense_bytes_per_layer, spec.expert_bytes
    B, P, N = 8, 40, 4
    ids = torch.randint(0, A.vocab, (B, P), generator=torch.Generator().manual_seed(41))
    res = Engine(A, BatchingPlan(B, 4, 16, 0.0, 0, spec.model_bytes), prompt_len=P, decode_len=N, use_graph=False)
    first_res = res.prefill(ids, chunk_tokens=3 * P)
    lg_res = res.buf.logits.cpu().float()
    for policy in ("resident", "offload"):
        s_params = dense + dense // 2 if family == "deepseek_v2" else 2 * dense + 3 * ex
        eng = Engine(A, BatchingPlan(B, 4, 16, 0.0, 3 * ex, s_params), prompt_len=P, decode_len=N,
                     use_graph=True, kv_policy=policy)
        assert eng.offload and eng.w.place.uncached_expert_count > 0
        first = eng.prefill(ids, chunk_tokens=3 * P)
        lg = eng.buf.logits.cpu().float()
        rows = sorted(((lg[i] - lg_res[i]).abs().max() / lg_res[i].abs().max()).item() for i in range(B))
        assert rows[B // 2] <= 2e-2, rows
        assert (first == first_res).float().mean() >= 0.75
        out = eng.generate(ids, N)  # streamed prefill + graph-replayed offloaded decode
        assert out.shape == (B, P + N) and torch.equal(out[:, P], first)
        # a second prefill over the same engine (its prefill staging reused): same tokens.  (This
        # once faulted for DeepSeek-V2 with the KV offloaded: latent-row padding left unwritten.)
        assert torch.equal(eng.generate(ids, N), out)
