"""Expert-parallel dispatch/combine (paper_2503_09716_b200/ep.py) on CPU with gloo, world size 2
and 4: every rank routes its own tokens, rows travel to the experts' owner ranks and back, and
the combined MoE output equals the single-process computation bit for bit (the per-row expert
math and the j-ascending fp32 combine are unchanged)."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import moe_ref as R
from oracle.rng import uniform_bf16

E, K, D, F, T_PER_RANK = 8, 2, 64, 128, 24


def _weights():
    return (uniform_bf16((E, D), 0, 1, 0.2), uniform_bf16((E, 2 * F, D), 0, 2, 0.05),
            uniform_bf16((E, D, F), 0, 3, 0.05))


def _tokens(world):
    return uniform_bf16((T_PER_RANK * world, D), 0, 4, 1.0)


def _moe_ep(x, ep, wr, wgu, wd):
    """One MoE block with experts sharded over ranks (CPU torch stand-ins for the kernels)."""
    T = x.shape[0]
    idx, w = R.route(torch.nn.functional.linear(x, wr), K, 0)
    order, dst, counts, offsets = R.permutation(idx, E)
    x_perm = x[order // K]
    x_loc, loc_offs, st = ep.dispatch(x_perm, counts)
    y_loc = torch.empty_like(x_loc)
    for i, e in enumerate(ep.local_experts()):
        a, b = int(loc_offs[i]), int(loc_offs[i + 1])
        if b > a:
            y_loc[a:b] = R.expert_ffn(x_loc[a:b], wgu[e], wd[e])
    y_perm = ep.combine(y_loc, st)
    acc = torch.zeros(T, D)
    for j in range(K):
        acc += y_perm[dst.view(T, K)[:, j]].float() * w[:, j:j + 1]
    return acc.to(torch.bfloat16)


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2503_09716_b200.ep import ExpertParallel, shard_sequences

        ep = ExpertParallel(E)
        wr, wgu, wd = _weights()
        x = _tokens(world)
        s0, s1 = shard_sequences(x.shape[0], rank, world)
        out = _moe_ep(x[s0:s1], ep, wr, wgu, wd)
        gathered = [torch.empty_like(out) for _ in range(world)]
        dist.all_gather(gathered, out)
        if rank == 0:
            q.put(torch.cat(gathered))
    finally:
        dist.destroy_process_group()


def _run_world(target, world, attempts: int = 3):
    """Spawn `world` gloo ranks on a fresh port and return rank 0's result.  A rendezvous that fails
    (the free port taken between probe and bind, a slow spawn on a loaded host) is retried on a new
    port; a rank that runs and fails its checks fails the test on the last attempt."""
    import queue as _queue

    ctx = mp.get_context("spawn")
    err = None
    for _ in range(attempts):
        q = ctx.Queue()
        port = _free_port()
        procs = [ctx.Process(target=target, args=(r, world, port, q)) for r in range(world)]
        for p in procs:
            p.start()
        try:
            got = q.get(timeout=300)
        except _queue.Empty:
            got, err = None, "rank 0 returned nothing within 300 s"
        for p in procs:
            p.join(timeout=120)
            if p.exitcode is None:
                p.kill()
        codes = [p.exitcode for p in procs]
        if got is not None and all(c == 0 for c in codes):
            return got
        err = err or f"rank exit codes {codes}"
    raise AssertionError(f"gloo world {world} failed {attempts} times: {err}")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world", [2, 4])
def test_ep_dispatch_combine_matches_single_process(world):
    got = _run_world(_worker, world)
    wr, wgu, wd = _weights()
    x = _tokens(world)
    ref = R.moe_block(x, wr, wgu, wd, K, 0)
    assert torch.equal(got, ref)


def test_single_rank_is_identity():
    from paper_2503_09716_b200.ep import ExpertParallel, shard_sequences

    ep = ExpertParallel(E)
    wr, wgu, wd = _weights()
    x = _tokens(1)
    assert torch.equal(_moe_ep(x, ep, wr, wgu, wd), R.moe_block(x, wr, wgu, wd, K, 0))
    assert shard_sequences(10, 0, 3) == (0, 4) and shard_sequences(10, 2, 3) == (7, 10)


@pytest.mark.parametrize("W,E", [(2, 8), (4, 16), (8, 64)])
def test_peer_ep_tables_route_every_row_home(W, E):
    """PeerExpertParallel.tables (host-independent, computed on the counts alone): the dispatch rows
    of all sources tile each owner's receive buffer exactly (expert-major, source-major within an
    expert), and the owner's combine segments send every row back to the position it came from in
    its source's expert-major permutation."""
    from paper_2503_09716_b200.ep import PeerExpertParallel

    g = torch.Generator().manual_seed(W * E)
    C = torch.randint(0, 9, (W, E), generator=g)
    peps = [PeerExpertParallel(E, W, r, [0] * W, [0] * W, device="cpu") for r in range(W)]
    tabs = [p.tables(C) for p in peps]
    L = E // W
    src_off = torch.cumsum(C, 1) - C
    for r in range(W):
        owner = tabs[r]
        n = int(owner["n_recv"][0])
        filled = torch.zeros(n, dtype=torch.int64) - 1
        back = {}
        for s in range(W):
            for e in range(r * L, (r + 1) * L):
                for m in range(int(C[s, e])):
                    q = int(tabs[s]["disp_row"][e]) + m          # where source s's row lands
                    assert filled[q] == -1
                    filled[q] = s
                    back[q] = (s, int(src_off[s, e]) + m)         # where it must go home
        assert (filled >= 0).all()
        seg_start, seg_len, seg_delta = owner["seg_start"], owner["seg_len"], owner["seg_delta"]
        for q, (s, home) in back.items():
            j = int((seg_start <= q).nonzero().max())
            while int(seg_len[j]) == 0 or q >= int(seg_start[j]) + int(seg_len[j]):
                j -= 1
            assert j % W == s and q + int(seg_delta[j]) == home
        assert torch.equal(owner["loc_offsets"][1:].long() - owner["loc_offsets"][:-1].long(), C[:, r * L:(r + 1) * L].sum(0))
