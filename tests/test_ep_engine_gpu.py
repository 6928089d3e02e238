"""Expert parallelism inside the engine: experts shard E/W per rank, sequences
data-parallel, one exchange per MoE layer on the router -> expert and expert -> combine edges
(offload_dag.py:418-472), fused into the kernels over peer memory (ep.PeerExpertParallel: dispatch
in the permutation, combine in the down GEMM's epilogue, only E counts exchanged, offsets on the
device).

1. W virtual ranks on one GPU (ep.VirtualPeerGroup: one engine per host thread and stream, event
   barriers): every rank's greedy tokens equal a plain single-GPU engine on the same sequences,
   bit for bit, and each rank holds only its expert shard.
2. The real multi-GPU wiring (NCCL count all-gather + torch symmetric memory barrier) at world 1 on
   this box: the EP decode step is captured as ONE CUDA graph and equals the plain engine.
   (world 2 is tests/test_ep_peer_gpu.py::test_symmetric_memory_two_ranks, on a multi-GPU box.)
"""

import threading

import pytest
import torch

pytestmark = pytest.mark.gpu


def _arch(family):
    from paper_2503_09716_b200.configs import TINY, TINY_DSV2

    return TINY if family == "mixtral" else TINY_DSV2


def _plan(A, B):
    from paper_2503_09716_b200.planner import BatchingPlan, ModelSpec

    return BatchingPlan(B, B, 16, 0.0, 0, ModelSpec.from_document(A.model_spec_document()).model_bytes)


@pytest.mark.parametrize("family,W", [("mixtral", 2), ("mixtral", 4), ("deepseek_v2", 2), ("deepseek_v2", 4)])
def test_peer_ep_engine_virtual_ranks(family, W):
    from paper_2503_09716_b200.engine import Engine
    from paper_2503_09716_b200.ep import PeerExpertParallel, VirtualPeerGroup

    A = _arch(family)
    B, P, N = 8, 4, 5
    ids = [torch.randint(0, A.vocab, (B, P), generator=torch.Generator().manual_seed(30 + r)) for r in range(W)]
    refs = [Engine(A, _plan(A, B), prompt_len=P, decode_len=N, use_graph=False).generate(x, N, prefill=False)
            for x in ids]
    group = VirtualPeerGroup(W, A.n_experts)
    cap = W * B * A.top_k
    recv = [torch.zeros(cap, A.hidden, dtype=torch.bfloat16, device="cuda") for _ in range(W)]
    yperm = [torch.zeros(B * A.top_k, A.hidden, dtype=torch.bfloat16, device="cuda") for _ in range(W)]
    engines = []
    for r in range(W):
        pep = PeerExpertParallel(A.n_experts, W, r, [t.data_ptr() for t in recv], [t.data_ptr() for t in yperm],
                                 recv=recv[r], yperm=yperm[r], comm=group.member(r))
        eng = Engine(A, _plan(A, B), prompt_len=P, decode_len=N, use_graph=True, ep=pep)
        assert not eng.use_graph  # virtual ranks: eager (their phases are different streams' work)
        L = A.n_experts // W
        moe = [w for w in eng.w.layers if w.get("w_gate_up") is not None]
        assert all(w["w_gate_up"].shape[0] == L for w in moe)  # only this rank's experts are resident
        engines.append(eng)
    torch.cuda.synchronize()
    outs, errs = [None] * W, []

    def run(r):
        try:
            with torch.cuda.stream(engines[r].stream):
                outs[r] = engines[r].generate(ids[r], N, prefill=False)
        except Exception as e:  # noqa: BLE001
            errs.append(e)
            group._tb.abort()

    th = [threading.Thread(target=run, args=(r,)) for r in range(W)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    assert not errs, errs
    for r in range(W):
        assert torch.equal(outs[r], refs[r]), f"rank {r}: tokens differ from the single-GPU engine"


def _symm_engine_worker(port, family, q):
    import os

    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        from paper_2503_09716_b200.engine import Engine
        from paper_2503_09716_b200.ep import PeerExpertParallel

        A = _arch(family)
        B, P, N = 8, 4, 6
        ids = torch.randint(0, A.vocab, (B, P), generator=torch.Generator().manual_seed(41))
        ref = Engine(A, _plan(A, B), prompt_len=P, decode_len=N, use_graph=False).generate(ids, N, prefill=False)
        pep = PeerExpertParallel.from_symmetric_memory(A.n_experts, dist.group.WORLD, B * A.top_k, B * A.top_k, A.hidden)
        eng = Engine(A, _plan(A, B), prompt_len=P, decode_len=N, use_graph=True, ep=pep)
        out = eng.generate(ids, N, prefill=False)
        q.put((eng.use_graph and eng.graph is not None, bool(torch.equal(out, ref))))
    except Exception as e:  # noqa: BLE001
        q.put(("error", repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("family", ["mixtral", "deepseek_v2"])
def test_peer_ep_engine_symmetric_memory_graph(family):
    import socket

    import torch.multiprocessing as mp

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_symm_engine_worker, args=(port, family, q))
    p.start()
    res = q.get(timeout=600)
    p.join(timeout=60)
    assert res == (True, True), res
