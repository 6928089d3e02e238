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
    ref = Engine(A, plan, prompt_len=P, decode_len=N, use_graph=False).generate(ids, N)
    for graph in (False, True):
        eng = Engine(A, plan, prompt_len=P, decode_len=N, use_graph=graph, kv_policy="offload", kv_ring_slots=2)
        assert not eng.kv[0][0].is_cuda and eng.kv_ring_n == 2
        assert torch.equal(eng.generate(ids, N), ref)


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
                 use_graph=False).generate(ids, N)
    two_layers = 2 * dense + ((dense - 1) // ex) * ex  # 2 dense layers cached + a few experts
    for s_params, slots, policy in ((dense + dense // 2, 2, "resident"), (two_layers, 3, "offload")):
        plan = BatchingPlan(B, 4, 16, 0.0, slots * ex, s_params)
        pl = placement(spec, s_params)
        assert pl.uncached_expert_count > 0 and pl.dense_layers < A.layers
        for graph in (False, True):
            eng = Engine(A, plan, prompt_len=P, decode_len=N, use_graph=graph, kv_policy=policy)
            assert eng.offload
            assert torch.equal(eng.generate(ids, N), ref), (s_params, policy, graph)
        recs, rep = eng.trace_step()
        uncached = (A.layers - pl.dense_layers) * dense + pl.uncached_expert_count * ex
        # the reference's all-MoE model charges experts to the dense first layer too: none move
        phantom = sum(A.n_experts - pl.experts_per_layer[l] for l in range(A.first_k_dense)) * ex
        kv_in = A.layers * B * (P + N) * A.kv_bytes_per_token_layer if policy == "offload" else 0
        assert rep["bytes_htod"] == uncached - phantom + kv_in
