"""Capacity contract (reference exec_sim.py:170-175 "groups larger than b_e split
into extra micro-batches instead of failing", SPEC.md invariants "every byte scheduled ... is
either transferred or the run is marked"): a grouped launch whose row segments exceed the buffer
they land in writes nothing out of bounds and reports MGB_ECAPACITY with the rows it needed; the
host pre-flight returns the per-expert counts; the engine's streamed prefill re-splits expert
groups by b_e and stays bit-identical."""

import pytest
import torch

from oracle.rng import uniform_bf16

pytestmark = pytest.mark.gpu

BF16 = torch.bfloat16


def _route(T, E, k, d, seed=0):
    from paper_2503_09716_b200 import ops

    x = uniform_bf16((T, d), 0, 10 + seed, 1.0).cuda()
    wr = uniform_bf16((E, d), 0, 1, 0.3).cuda()
    ws = ops.RouterWorkspace(T, E, k)
    ops.router_topk(None, None, ws, k, 0, logits_in=torch.mm(x, wr.t(), out_dtype=torch.float32))
    return x, ws


def test_preflight_counts_and_overflow():
    from paper_2503_09716_b200 import ops

    T, E, k, d = 100, 8, 2, 256
    _, ws = _route(T, E, k, d)
    counts = ops.check_capacity(ws.offsets, T * k)
    assert counts == ws.counts.cpu().tolist() and sum(counts) == T * k
    with pytest.raises(ops.CapacityError) as ei:
        ops.check_capacity(ws.offsets, T * k - 1)
    assert ei.value.counts == counts and ei.value.needed == T * k


@pytest.mark.parametrize("which", ["gate_up", "down"])
def test_grouped_gemm_overflow_is_a_status_not_a_write(which):
    from paper_2503_09716_b200 import ops

    ops.capacity_status(reset=True)  # clean slate
    T, E, k, d, f = 64, 8, 2, 256, 512
    x, ws = _route(T, E, k, d)
    cap = T * k - 37  # smaller than offsets[E]
    guard = 5
    if which == "gate_up":
        w = uniform_bf16((E, 2 * f, d), 0, 2, 0.05).cuda()
        src = torch.zeros(cap, d, dtype=BF16, device="cuda")
        out = torch.full((cap + guard, f), 7.0, dtype=BF16, device="cuda")
        ops.moe_gemm_gate_up(w, src, ws.offsets, out[:cap])
        site = 1
    else:
        w = uniform_bf16((E, d, f), 0, 3, 0.05).cuda()
        src = torch.zeros(cap, f, dtype=BF16, device="cuda")
        out = torch.full((cap + guard, d), 7.0, dtype=BF16, device="cuda")
        ops.moe_gemm_down(w, src, ws.offsets, out[:cap])
        site = 2
    with pytest.raises(ops.CapacityError) as ei:
        ops.capacity_status(reset=True)
    assert (ei.value.needed, ei.value.rows_cap, ei.value.site) == (T * k, cap, site)
    assert bool((out == 7.0).all()), "an overflowing launch wrote rows"
    ops.capacity_status(reset=True)  # cleared: no raise
    # a fitting launch on the same buffers still runs and records nothing
    ok = torch.zeros(T * k, out.shape[1], dtype=BF16, device="cuda")
    srcf = torch.ones(T * k, src.shape[1], dtype=BF16, device="cuda")
    (ops.moe_gemm_gate_up if which == "gate_up" else ops.moe_gemm_down)(w, srcf, ws.offsets, ok)
    ops.capacity_status(reset=True)
    assert bool(ok.abs().sum() > 0)


def test_ep_dispatch_overflow_guard():
    """Peer-memory EP dispatch into fixed-capacity receive buffers smaller than the rows routed to
    an owner: nothing lands past the buffer (the guard rows after it keep their value), the overflow
    is reported with site 3."""
    from paper_2503_09716_b200 import ops
    from paper_2503_09716_b200.ep import PeerExpertParallel

    ops.capacity_status(reset=True)
    W, E, k, d, T = 2, 8, 2, 256, 48
    xs, wss = zip(*[_route(T, E, k, d, seed=r) for r in range(W)])
    cap, guard = 30, 8
    store = [torch.full((cap + guard, d), 3.0, dtype=BF16, device="cuda") for _ in range(W)]
    yperm = [torch.zeros(T * k, d, dtype=BF16, device="cuda") for _ in range(W)]
    peps = [PeerExpertParallel(E, W, r, [b.data_ptr() for b in store], [b.data_ptr() for b in yperm], recv_rows=cap)
            for r in range(W)]
    counts_all = torch.stack([ws.counts for ws in wss])
    assert int(counts_all.sum()) > W * cap  # some owner must overflow
    for r in range(W):
        peps[r].dispatch(xs[r], wss[r], peps[r].tables(counts_all))
    with pytest.raises(ops.CapacityError) as ei:
        ops.capacity_status(reset=True)
    assert ei.value.site == 3 and ei.value.rows_cap == cap and ei.value.needed > cap
    for b in store:
        assert bool((b[cap:] == 3.0).all()), "dispatch wrote past the receive buffer"


def test_streamed_prefill_resplit_by_be():
    """Offloaded-weight prefill with a b_e far below the per-expert group size: every group runs as
    several b_e-row launches and the result equals a run whose b_e covers the groups."""
    from paper_2503_09716_b200.configs import TINY
    from paper_2503_09716_b200.engine import Engine
    from paper_2503_09716_b200.planner import BatchingPlan, ModelSpec

    spec = ModelSpec.from_document(TINY.model_spec_document())
    B, P = 8, 40  # 320 tokens x top-2 over 8 experts: ~80 rows per expert group
    s_exp = spec.expert_bytes * 2
    ids = torch.randint(0, TINY.vocab, (B, P), generator=torch.Generator().manual_seed(3))
    outs = []
    for be in (1024, 16):  # groups of ~80 rows: one launch per expert vs 5-6 b_e-row launches
        plan = BatchingPlan(B, B, be, 0.0, spec.model_bytes // 2, s_exp)
        eng = Engine(TINY, plan, prompt_len=P, decode_len=2, use_graph=False)
        eng.prefill_min_be = 1
        first = eng.prefill(ids)
        torch.cuda.synchronize()
        outs.append((first.cpu(), eng.buf.logits.float().cpu()))
        del eng
    assert torch.equal(outs[0][0], outs[1][0])
    assert torch.equal(outs[0][1], outs[1][1])
