"""Expert parallelism fused with the data path over peer memory (ep.PeerExpertParallel):
dispatch inside the permutation kernel, combine inside the down GEMM's epilogue.  On one GPU the
W ranks are virtual (their buffers are device pointers of the same GPU, exactly what UVA peer
pointers are on an NVLink box), phases run in rank order (the barrier).  Every rank's y_perm and
combined MoE output must equal the single-rank computation bit for bit."""

import pytest
import torch

from oracle.rng import uniform_bf16

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("W,E,k,d,f,T", [(2, 8, 2, 256, 512, 40), (4, 16, 4, 256, 128, 33), (4, 8, 2, 512, 384, 7)])
def test_peer_ep_bit_exact(W, E, k, d, f, T):
    from paper_2503_09716_b200 import ops
    from paper_2503_09716_b200.ep import PeerExpertParallel

    dev = "cuda"
    wr = uniform_bf16((E, d), 0, 1, 0.3).to(dev)
    wgu = uniform_bf16((E, 2 * f, d), 0, 2, 0.05).to(dev)
    wd = uniform_bf16((E, d, f), 0, 3, 0.05).to(dev)
    xs = [uniform_bf16((T, d), 0, 10 + r, 1.0).to(dev) for r in range(W)]
    wss = [ops.RouterWorkspace(T, E, k) for _ in range(W)]
    for x, ws in zip(xs, wss):
        lg = torch.mm(x, wr.t(), out_dtype=torch.float32)
        ops.router_topk(None, None, ws, k, 0, logits_in=lg)
    # single-rank reference for every rank's tokens
    ref_y, ref_out = [], []
    for x, ws in zip(xs, wss):
        xp = torch.empty(T * k, d, dtype=torch.bfloat16, device=dev)
        ops.permute(x, ws, xp)
        h = torch.empty(T * k, f, dtype=torch.bfloat16, device=dev)
        y = torch.empty(T * k, d, dtype=torch.bfloat16, device=dev)
        ops.moe_gemm_gate_up(wgu, xp, ws.offsets, h)
        ops.moe_gemm_down(wd, h, ws.offsets, y)
        out = torch.empty(T, d, dtype=torch.bfloat16, device=dev)
        ops.unpermute_combine(y, ws, out, T)
        ref_y.append(y.clone())
        ref_out.append(out)
    # peer-memory EP over W virtual ranks
    cap = W * T * k
    recv = [torch.zeros(cap, d, dtype=torch.bfloat16, device=dev) for _ in range(W)]
    yperm = [torch.zeros(T * k, d, dtype=torch.bfloat16, device=dev) for _ in range(W)]
    counts_all = torch.stack([ws.counts for ws in wss])
    L = E // W
    peps = [PeerExpertParallel(E, W, r, [b.data_ptr() for b in recv], [b.data_ptr() for b in yperm], recv_rows=cap)
            for r in range(W)]
    tabs = [p.tables(counts_all) for p in peps]
    for r in range(W):  # phase 1: every source dispatches
        peps[r].dispatch(xs[r], wss[r], tabs[r])
    for r in range(W):  # phase 2: every owner runs its experts, rows go home from the epilogue
        h = torch.empty(cap, f, dtype=torch.bfloat16, device=dev)
        row_ptr = torch.empty(cap, dtype=torch.int64, device=dev)
        peps[r].experts(wgu[r * L:(r + 1) * L], wd[r * L:(r + 1) * L], recv[r], h, row_ptr, tabs[r])
    torch.cuda.synchronize()
    for r in range(W):  # phase 3: local weighted combine
        out = torch.empty(T, d, dtype=torch.bfloat16, device=dev)
        ops.unpermute_combine(yperm[r], wss[r], out, T)
        assert torch.equal(yperm[r], ref_y[r]), f"rank {r}: y_perm differs"
        assert torch.equal(out, ref_out[r]), f"rank {r}: MoE output differs"


def _symm_worker(rank, world, port, q):
    import os

    import torch.distributed as dist

    from paper_2503_09716_b200 import ops
    from paper_2503_09716_b200.ep import PeerExpertParallel

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world)
    E, k, d, f, T = 8, 2, 256, 512, 24
    dev = f"cuda:{rank}"
    wr, wgu, wd = (uniform_bf16((E, d), 0, 1, 0.3).to(dev), uniform_bf16((E, 2 * f, d), 0, 2, 0.05).to(dev),
                   uniform_bf16((E, d, f), 0, 3, 0.05).to(dev))
    x = uniform_bf16((T, d), 0, 10 + rank, 1.0).to(dev)
    ws = ops.RouterWorkspace(T, E, k, device=dev)
    ops.router_topk(None, None, ws, k, 0, logits_in=torch.mm(x, wr.t(), out_dtype=torch.float32))
    L = E // world
    pep = PeerExpertParallel.from_symmetric_memory(E, dist.group.WORLD, world * T * k, T * k, d, device=dev)
    y = pep.moe(x, ws, wgu[rank * L:(rank + 1) * L], wd[rank * L:(rank + 1) * L],
                torch.empty(world * T * k, f, dtype=torch.bfloat16, device=dev),
                torch.empty(world * T * k, dtype=torch.int64, device=dev))
    xp = torch.empty(T * k, d, dtype=torch.bfloat16, device=dev)
    ops.permute(x, ws, xp)
    h = torch.empty(T * k, f, dtype=torch.bfloat16, device=dev)
    ref = torch.empty(T * k, d, dtype=torch.bfloat16, device=dev)
    ops.moe_gemm_gate_up(wgu, xp, ws.offsets, h)
    ops.moe_gemm_down(wd, h, ws.offsets, ref)
    torch.cuda.synchronize()
    q.put((rank, bool(torch.equal(y, ref))))
    dist.destroy_process_group()


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs 2 GPUs with NVLink peer access")
def test_symmetric_memory_two_ranks():
    """The same fused dispatch/combine across two real GPUs through torch symmetric memory."""
    import socket

    import torch.multiprocessing as mp

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_symm_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=300) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    assert res == {0: True, 1: True}
