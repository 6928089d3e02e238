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


class PeerExpertParallel:
    """Expert parallelism with the exchange fused into the kernels over peer memory (NVLink 5 /
    NVSwitch, UVA peer pointers), the B200-native alternative to the all_to_all path above:

      dispatch  the permutation kernel writes each routed row straight into the receive buffer of
                the expert's owner rank (mgb_ep_permute_dispatch), at this source's slot of the
                expert's segment -- no x_perm round trip, no packing, no collective on the data;
      combine   the down-projection GEMM's epilogue stores each output row straight into the home
                rank's y_perm (mgb_moe_gemm_down_ep with mgb_ep_row_ptrs), where the usual weighted
                unpermute_combine runs -- so results stay bit-identical to the single-GPU path.

    Only the per-expert counts (E ints per rank) are exchanged as a collective.  Every offset is
    computed on the device from them (`tables`), so the layer has no host synchronisation.  The
    receive-buffer layout per owner rank is expert-major over its E/W local experts and
    source-rank-major within an expert.  `recv_ptrs[r]` / `yperm_ptrs[r]` are rank r's buffers as
    seen from this rank (torch symmetric memory buffer_ptrs on a multi-GPU box; plain device
    pointers when several virtual ranks share one GPU, as in tests/test_ep_peer_gpu.py).
    Cross-rank ordering (all writes into a buffer landed before it is read) is the caller's
    barrier between the three phases."""

    def __init__(self, n_experts: int, world: int, rank: int, recv_ptrs, yperm_ptrs, device="cuda",
                 recv: torch.Tensor | None = None, yperm: torch.Tensor | None = None, comm=None,
                 recv_rows: int | None = None):
        if n_experts % world:
            raise ValueError(f"{n_experts} experts do not shard over {world} ranks")
        self.E, self.W, self.rank = n_experts, world, rank
        self.world = world
        self.L = n_experts // world
        self.E_local = self.L
        self.first = rank * self.L
        self.peer_recv = torch.tensor([int(p) for p in recv_ptrs], dtype=torch.int64, device=device)
        self.peer_y = torch.tensor([int(p) for p in yperm_ptrs], dtype=torch.int64, device=device)
        # this rank's own buffers (the engine's EP path reads them) and the count exchange / barrier
        # (`comm`: _SymmComm over NCCL + symmetric memory, or VirtualPeerGroup.member for virtual ranks)
        self.recv, self.yperm, self.comm = recv, yperm, comm
        # rows of every rank's (equal-sized) receive buffer: the dispatch kernel never writes past it
        # and records an overflow for ops.capacity_status instead (SPEC.md invariants: no silent drop)
        self.recv_rows = int(recv_rows if recv_rows is not None else recv.shape[0] if recv is not None else 2 ** 31 - 1)

    def local_experts(self) -> range:
        return range(self.first, self.first + self.L)

    def tables(self, counts_all: torch.Tensor) -> dict:
        """counts_all [W, E]: rows source s routes to expert e.  Returns this rank's dispatch rows
        (as a source) and receive / combine tables (as an owner), all int32 on counts_all's device."""
        C = counts_all.to(torch.int64)
        W, L, r, E = self.W, self.L, self.rank, self.E
        tot = C.sum(0)                                    # [E] rows per expert over all sources
        tr = tot.view(W, L)
        loc_base = (tr.cumsum(1) - tr).reshape(E)         # expert e's block start in its owner's buffer
        pre_src = C.cumsum(0) - C                         # [W, E] rows of e from earlier sources
        src_off = C.cumsum(1) - C                         # [W, E] e's segment start in source s's x_perm
        e0 = r * L
        seg_start = loc_base[e0:e0 + L][:, None] + pre_src[:, e0:e0 + L].t()   # [L, W], i-major
        loc_offsets = torch.zeros(L + 1, dtype=torch.int64, device=C.device)
        loc_offsets[1:] = tot[e0:e0 + L].cumsum(0)
        i32 = torch.int32
        return dict(disp_row=(loc_base + pre_src[r]).to(i32), loc_offsets=loc_offsets.to(i32),
                    n_recv=loc_offsets[-1:].to(i32),
                    seg_start=seg_start.reshape(-1).to(i32), seg_len=C[:, e0:e0 + L].t().reshape(-1).to(i32),
                    seg_delta=(src_off[:, e0:e0 + L].t() - seg_start).reshape(-1).to(i32))

    # ---- the three phases (each rank issues its own; barriers between phases are the caller's) ----
    def dispatch(self, h: torch.Tensor, ws, tab: dict) -> None:
        """Route + permute + send: this rank's routed rows land in the owners' receive buffers."""
        from . import _native as nat

        T, d = h.shape
        nat.call("mgb_ep_permute_dispatch", h.data_ptr(), ws.topk_idx.data_ptr(), ws.local_rank.data_ptr(),
                 ws.block_hist.data_ptr(), ws.offsets.data_ptr(), T, d, ws.k, self.E, self.L,
                 self.peer_recv.data_ptr(), tab["disp_row"].data_ptr(), self.recv_rows, ws.src_token.data_ptr(),
                 ws.dst_pos.data_ptr(), torch.cuda.current_stream().cuda_stream)

    def experts(self, w_gate_up: torch.Tensor, w_down: torch.Tensor, recv: torch.Tensor, h_ffn: torch.Tensor,
                row_ptr: torch.Tensor, tab: dict) -> None:
        """The local experts' grouped GEMMs over the receive buffer; the down GEMM's epilogue sends
        every output row home.  w_gate_up / w_down are this rank's [E/W, ...] expert shards."""
        from . import _native as nat
        from . import ops

        st = torch.cuda.current_stream().cuda_stream
        L, d = self.L, recv.shape[1]
        f = w_down.shape[2]
        ops.moe_gemm_gate_up(w_gate_up, recv, tab["loc_offsets"], h_ffn)
        nat.call("mgb_ep_row_ptrs", tab["seg_start"].data_ptr(), tab["seg_len"].data_ptr(),
                 tab["seg_delta"].data_ptr(), L * self.W, self.W, self.peer_y.data_ptr(), d * 2, recv.shape[0],
                 row_ptr.data_ptr(), st)
        nat.call("mgb_moe_gemm_down_ep", w_down.data_ptr(), h_ffn.data_ptr(), tab["loc_offsets"].data_ptr(), L, d, f,
                 recv.shape[0], row_ptr.data_ptr(), st)

    # ---- multi-GPU wiring: torch symmetric memory (NVLink peer mappings + device-side barrier) ----
    @classmethod
    def from_symmetric_memory(cls, n_experts: int, group, recv_rows: int, yperm_rows: int, d: int,
                              device: str = "cuda") -> "PeerExpertParallel":
        """Allocate this rank's receive buffer and y_perm in symmetric memory and exchange their
        peer mappings (one rendezvous at setup).  `recv_rows` must cover the worst case (every
        source's T*k rows landing on this rank's experts)."""
        import torch.distributed._symmetric_memory as symm

        recv = symm.empty(recv_rows, d, dtype=torch.bfloat16, device=device)
        yperm = symm.empty(yperm_rows, d, dtype=torch.bfloat16, device=device)
        hr, hy = symm.rendezvous(recv, group), symm.rendezvous(yperm, group)
        comm = _SymmComm(group, hr, hr.world_size, n_experts, device)
        self = cls(n_experts, hr.world_size, hr.rank, hr.buffer_ptrs, hy.buffer_ptrs, device=device, recv=recv,
                   yperm=yperm, comm=comm)
        self.group, self._handle = group, hr
        return self

    def barrier(self) -> None:
        """Stream-ordered cross-rank barrier (all peer writes of the phase have landed)."""
        self.comm.barrier()

    def moe(self, h: torch.Tensor, ws, w_gate_up_local: torch.Tensor, w_down_local: torch.Tensor,
            h_ffn: torch.Tensor, row_ptr: torch.Tensor) -> torch.Tensor:
        """One routed-expert layer across the group after this rank's router: returns this rank's
        y_perm (home rows of its tokens' expert outputs) for mgb_unpermute_combine."""
        counts_all = self.comm.exchange_counts(ws.counts)
        tab = self.tables(counts_all)
        self.dispatch(h, ws, tab)
        self.barrier()
        self.experts(w_gate_up_local, w_down_local, self.recv, h_ffn, row_ptr, tab)
        self.barrier()
        return self.yperm


class _SymmComm:
    """Count exchange + barrier of PeerExpertParallel across real GPUs: NCCL all-gather of the E
    per-expert counts into a fixed device table (graph-capturable: fixed size, fixed address) and
    torch symmetric memory's stream-ordered signal-pad barrier."""

    graph_safe = True

    def __init__(self, group, handle, world: int, E: int, device):
        self.group, self.handle = group, handle
        self.counts_all = torch.zeros(world, E, dtype=torch.int32, device=device)

    def exchange_counts(self, counts: torch.Tensor) -> torch.Tensor:
        dist.all_gather_into_tensor(self.counts_all, counts, group=self.group)
        return self.counts_all

    # a peer that died must not leave the others spinning on the signal pad forever (a stuck GPU):
    # the barrier kernel traps after this long (ranks that are merely slower -- engine set-up of a
    # large model -- stay well inside it)
    BARRIER_TIMEOUT_MS = 300_000

    def barrier(self) -> None:
        self.handle.barrier(timeout_ms=self.BARRIER_TIMEOUT_MS)


class VirtualPeerGroup:
    """W virtual ranks sharing one GPU (tests and single-GPU validation of the EP data path): each
    rank is an Engine driven from its own host thread on its own CUDA stream; the barrier is a
    host-thread rendezvous plus cross-stream event waits (every rank's stream waits for every
    rank's work issued before the barrier), the count exchange a shared device table.  Eager only:
    the phases of different ranks are different streams' work, not one capturable graph."""

    def __init__(self, W: int, E: int, device="cuda"):
        import threading

        self.W = W
        self.counts_all = torch.zeros(W, E, dtype=torch.int32, device=device)
        self._tb = threading.Barrier(W)
        self._ev = [torch.cuda.Event() for _ in range(W)]

    def member(self, rank: int) -> "_VirtualComm":
        return _VirtualComm(self, rank)


class _VirtualComm:
    graph_safe = False

    def __init__(self, group: VirtualPeerGroup, rank: int):
        self.g, self.rank = group, rank

    def exchange_counts(self, counts: torch.Tensor) -> torch.Tensor:
        self.g.counts_all[self.rank].copy_(counts)
        self.barrier()
        return self.g.counts_all

    def barrier(self) -> None:
        g, st = self.g, torch.cuda.current_stream()
        g._ev[self.rank].record(st)
        g._tb.wait()
        for e in g._ev:
            st.wait_event(e)
        g._tb.wait()  # nobody re-records before every rank has queued its waits
