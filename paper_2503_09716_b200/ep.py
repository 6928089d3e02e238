"""Expert parallelism across GPUs: experts shard E/G per rank, tokens stay
data-parallel, and each MoE layer has exactly one exchange step -- token dispatch before the
grouped expert GEMM and combine after it -- over torch.distributed (NCCL over NVLink 5 on the
8xB200 box; gloo in the CPU tests).

The single-GPU path (reference offload_dag.py:427-463) produces an expert-major, stable
permutation `x_perm` with `offsets[E+1]`; because experts are sharded in contiguous ranges the
same order is also destination-rank-major, so dispatch is one all_to_all of the counts and one
all_to_all_single of the rows with no extra packing.  On the receiving rank the rows arrive
source-major (src 0: e0..e_{L-1}, src 1: ...) and are regrouped expert-major (stable by source,
so the order is deterministic) for the local grouped GEMM; combine is the exact inverse.  The
weighted sum itself stays on the token's home rank (mgb_unpermute_combine), so results are
bit-identical to the single-GPU path.

Split sizes are read back to the host once per layer (a device->host sync); the fixed-capacity,
graph-capturable variant is a next step (SURVEY.md §7 hard part 5).
"""

from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist


@dataclass
class DispatchState:
    send_splits: list[int]       # rows sent to each rank (= rows of its expert range)
    recv_splits: list[int]       # rows received from each rank
    order: torch.Tensor          # received row -> local expert-major position
    local_counts: torch.Tensor   # [E_local] rows per local expert (all sources)


class ExpertParallel:
    def __init__(self, n_experts: int, group=None):
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        if n_experts % self.world:
            raise ValueError(f"{n_experts} experts do not shard over {self.world} ranks")
        self.E = n_experts
        self.E_local = n_experts // self.world
        self.first = self.rank * self.E_local

    def local_experts(self) -> range:
        return range(self.first, self.first + self.E_local)

    def dispatch(self, x_perm: torch.Tensor, counts: torch.Tensor) -> tuple[torch.Tensor, torch.Tensor, DispatchState]:
        """x_perm [sum(counts), d] expert-major rows of this rank's tokens, counts [E] int.
        Returns (x_local expert-major rows of the local experts from all ranks, local offsets
        [E_local + 1] int32, state for combine)."""
        W, L = self.world, self.E_local
        counts = counts.to(torch.int64).view(W, L)
        if W == 1:
            loc = counts.view(L)
            offs = torch.zeros(L + 1, dtype=torch.int32, device=x_perm.device)
            offs[1:] = torch.cumsum(loc, 0)
            n = int(loc.sum())
            return x_perm[:n], offs, DispatchState([n], [n], torch.arange(n, device=x_perm.device), loc)
        recv_counts = torch.empty_like(counts)  # [src, L]
        dist.all_to_all_single(recv_counts, counts.contiguous(), group=self.group)
        send_splits = counts.sum(1).tolist()
        recv_splits = recv_counts.sum(1).tolist()
        n_recv = sum(recv_splits)
        recv = x_perm.new_empty((n_recv, x_perm.shape[1]))
        dist.all_to_all_single(recv, x_perm[:sum(send_splits)].contiguous(), recv_splits, send_splits,
                               group=self.group)
        # regroup source-major -> expert-major (stable by source)
        rc = recv_counts.to(x_perm.device)                      # [src, L], received (src, e) blocks
        local_counts = rc.sum(0)
        flat = rc.reshape(-1)
        recv_start = torch.cumsum(flat, 0) - flat                 # block start in the received buffer
        exp_base = torch.cumsum(local_counts, 0) - local_counts    # expert segment start (local)
        within = torch.cumsum(rc, 0) - rc                         # earlier sources' rows of the expert
        dest_start = (exp_base[None, :] + within).reshape(-1)
        dest = torch.repeat_interleave(dest_start - recv_start, flat, output_size=n_recv) + \
            torch.arange(n_recv, device=x_perm.device)
        x_local = torch.empty_like(recv)
        x_local[dest] = recv
        offs = torch.zeros(L + 1, dtype=torch.int32, device=x_perm.device)
        offs[1:] = torch.cumsum(local_counts, 0).to(x_perm.device)
        return x_local, offs, DispatchState(send_splits, recv_splits, dest, local_counts.to(x_perm.device))

    def combine(self, y_local: torch.Tensor, st: DispatchState) -> torch.Tensor:
        """Inverse of dispatch: expert outputs back to their home ranks, in the home rank's
        expert-major row order (ready for mgb_unpermute_combine)."""
        if self.world == 1:
            return y_local
        back = y_local[st.order]  # local expert-major -> source-major
        out = y_local.new_empty((sum(st.send_splits), y_local.shape[1]))
        dist.all_to_all_single(out, back.contiguous(), st.send_splits, st.recv_splits, group=self.group)
        return out


def shard_sequences(B_total: int, rank: int, world: int) -> tuple[int, int]:
    """Data-parallel share [s0, s1) of B_total independent sequences for `rank`."""
    q, r = divmod(B_total, world)
    s0 = rank * q + min(rank, r)
    return s0, s0 + q + (rank < r)
