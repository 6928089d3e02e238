"""MoE-Gen engine on one B200: executes the module-based batching job list with the sm_100a
kernels of libmgb.so.

The scheduler side follows the reference: the engine takes the planner's decision vector
(`plan.json` / BatchingPlan, reference memory_model.py:66-89, cli.py:74-109), sizes its HBM
buffers from it, builds the per-layer job list with `schedule.build_schedule` (the reference's
`_build_graph`, offload_dag.py:240-492) and issues those jobs in submission order on CUDA
streams.  Per layer (decode):
    pre_attention(mb)  : RMSNorm -> fused QKV GEMM (cuBLAS) -> RoPE + paged-KV append   [b_a seqs]
    attn_mech_gpu(mb)  : paged GQA decode attention (mgb_decode_attn_gqa)               [b_a seqs]
    post_attention     : O GEMM (cuBLAS) -> residual add + RMSNorm                      [B seqs]
    router             : fused gate GEMV + softmax + top-k + counts (mgb_router_topk) + stable permute
    expert_compute     : tcgen05 grouped GEMM gate/up+SiLU, down (all experts' chunks in one
                         persistent launch each) -> weighted combine + residual add
The whole decode step (all layers + LM head + greedy argmax + bookkeeping) is captured once as a
CUDA graph and replayed per generated token, so the host issues one launch per token.
"""

from __future__ import annotations

import json
import os
import math
import time
from dataclasses import dataclass

import torch

from . import _native as nat
from . import ops
from .configs import ModelArch, get_arch
from .planner import BatchingPlan, Hardware, ModelSpec, WorkloadSpec, largest_batch, load_plan
from .schedule import Schedule, build_schedule
from .hostmem import pinned_empty
from .weights import DeepseekDeviceWeights, MixtralDeviceWeights

BF16 = torch.bfloat16


def b200_hardware(host_bytes: int = 2_000_000_000_000, hbm_bytes: int | None = None) -> Hardware:
    """B200 machine description for the planner (capacities; rates only seed the estimate)."""
    if hbm_bytes is None:
        hbm_bytes = torch.cuda.get_device_properties(0).total_memory if torch.cuda.is_available() else 183_359 << 20
    return Hardware(m_g=int(hbm_bytes), m_c=int(host_bytes), bw_htod=55e9, bw_dtoh=55e9, gpu_peak_flops=1.63e15,
                    gpu_mem_bw=6.54e12, gpu_launch_overhead=5e-6, cpu_attn_flops=0.0)


def _unit_latency(kind: str, tokens: int, ctx: int) -> float:
    return 1e-6 * tokens


def routed_expert_bytes(arch: ModelArch) -> int:
    """Bytes of all routed experts of all MoE layers (bf16 gate, up and down)."""
    return (arch.layers - arch.first_k_dense) * arch.n_experts * 3 * arch.hidden * arch.moe_ffn * 2


def resident_plan(arch: ModelArch, prompt_len: int, decode_len: int, B: int | None = None,
                  b_a: int | None = None, b_e: int = 4096, reserve_bytes: int = 12 << 30,
                  hbm_bytes: int | None = None, ep_world: int = 1) -> BatchingPlan:
    """Plan for an HBM-resident model (s_params = whole model, no expert slots): B is the largest
    batch whose paged KV fits next to the weights (reference max_feasible_B with the resident KV
    policy), capped by `B` if given.  ep_world > 1: one rank of an expert-parallel group, which
    holds 1/ep_world of the routed experts; the planner sees the whole model next to an HBM enlarged
    by the other ranks' expert bytes, so B is this rank's KV capacity."""
    spec = ModelSpec.from_document(arch.model_spec_document())
    hw = b200_hardware(hbm_bytes=hbm_bytes)
    others = routed_expert_bytes(arch) * (ep_world - 1) // ep_world
    hw = Hardware(**{**hw.__dict__, "m_g": hw.m_g - reserve_bytes + others})
    wl = WorkloadSpec(prompt_len, decode_len, 1, "decode")
    tmpl = BatchingPlan(1, 1, b_e, 0.0, 0, spec.model_bytes)
    from .planner import footprint

    bmax = largest_batch(spec, hw, wl, tmpl, kv_policy="resident")
    if b_a is None:  # one attention micro-batch: re-size B with b_a = B charged (Eq. 3)
        bmax = largest_batch(spec, hw, wl, BatchingPlan(1, bmax, b_e, 0.0, 0, spec.model_bytes), kv_policy="resident")
    B = bmax if B is None else min(B, bmax)
    b_a = B if b_a is None else min(b_a, B)
    # largest attention micro-batch the GPU constraint admits (Eq. 3 charges b_a's activations)
    while b_a > 1 and not footprint(spec, hw, wl, BatchingPlan(B, b_a, b_e, 0.0, 0, spec.model_bytes),
                                    "resident").feasible:
        b_a = (b_a + 1) // 2
    return BatchingPlan(B, b_a, b_e, 0.0, 0, spec.model_bytes)


@dataclass
class StepBuffers:
    x: torch.Tensor
    h: torch.Tensor
    qkv: torch.Tensor
    q: torch.Tensor
    attn: torch.Tensor
    o: torch.Tensor
    x_perm: torch.Tensor
    h_ffn: torch.Tensor
    y_perm: torch.Tensor
    logits: torch.Tensor
    next_ids: torch.Tensor
    positions: torch.Tensor
    seq_lens: torch.Tensor
    step: torch.Tensor


class Engine:
    """Greedy MoE decoding engine (Mixtral and DeepSeek-V2 families; HBM-resident or partly
    host-offloaded weights, paged KV in HBM, optional expert parallelism)."""

    def __init__(self, arch: ModelArch | str | None, plan=None, *, prompt_len: int, decode_len: int, seed: int = 0,
                 kv_policy: str = "resident", use_graph: bool = True, device: str = "cuda", ep=None,
                 kv_ring_slots: int = 3, lookahead: bool = True, checkpoint=None):
        """`checkpoint`: a HF safetensors checkpoint directory (checkpoint.py) to load the weights
        from instead of the counter-based random init; `arch` None takes the architecture from its
        config.json, an explicit arch may truncate the depth (layers <= the checkpoint's)."""
        if not torch.cuda.is_available():
            raise RuntimeError("the B200 engine needs a CUDA device (there is no CPU fallback)")
        self.source = None
        if checkpoint is not None:
            from .checkpoint import open_checkpoint

            self.source = open_checkpoint(checkpoint)
            ck = self.source.arch
            if arch is None:
                arch = ck
            else:
                arch = get_arch(arch) if isinstance(arch, str) else arch
                import dataclasses as _dc
                if _dc.replace(arch, name=ck.name, layers=ck.layers, init_std=ck.init_std) != ck or arch.layers > ck.layers:
                    raise ValueError(f"architecture {arch.name!r} does not match the checkpoint's config.json ({ck})")
        elif arch is None:
            raise ValueError("arch is required without a checkpoint")
        self.arch = get_arch(arch) if isinstance(arch, str) else arch
        if self.arch.family not in ("mixtral", "deepseek_v2"):
            raise NotImplementedError(f"unknown model family {self.arch.family!r}")
        if kv_policy not in ("resident", "offload"):
            raise ValueError(f"kv_policy must be 'resident' or 'offload', got {kv_policy!r}")
        a = self.arch
        self.mla = a.family == "deepseek_v2"
        self.kv_policy = kv_policy
        self.prompt_len, self.decode_len = prompt_len, decode_len
        self.max_ctx = prompt_len + decode_len
        self.plan = load_plan(plan) if plan is not None else resident_plan(a, prompt_len, decode_len)
        self.spec = ModelSpec.from_document(a.model_spec_document())
        self.workload = WorkloadSpec(prompt_len, decode_len, self.plan.B, "decode")
        self.B = B = self.plan.B
        self.device = device
        # expert parallelism (ep.ExpertParallel): experts of this rank's range run locally, token
        # rows are dispatched/combined over torch.distributed; the host-side split sizes make the
        # EP step eager (no CUDA graph) in this build
        from .ep import PeerExpertParallel

        # PeerExpertParallel: dispatch fused into the permutation, combine into the down GEMM's epilogue,
        # only the E counts exchanged, all offsets on the device -> the EP step is graph-capturable when
        # its comm is (NCCL + symmetric memory); kept even at world 1 (the same code path, one rank)
        self.peer_ep = isinstance(ep, PeerExpertParallel)
        self.ep = ep if (ep is not None and (self.peer_ep or ep.world > 1)) else None
        if ep is not None and self.plan.s_params < self.spec.model_bytes:
            # the EP path slices this rank's expert range out of the resident expert tensors; streamed
            # experts live in slots indexed by copy order, which the dispatch offsets do not describe
            raise ValueError("expert parallelism needs HBM-resident weights (plan.s_params = model bytes)")
        self.use_graph = use_graph and (self.ep is None or (self.peer_ep and getattr(ep.comm, "graph_safe", False)))
        # ---- job list (structure only; durations are measured, not modelled) ----
        # ---- CPU attention share (omega > 0): GQA over the host page store on the host cores ----
        self.n_cpu = self.plan.cpu_sequences()
        if self.n_cpu > 0 and (kv_policy != "offload" or self.mla_family() or ep is not None):
            raise ValueError("a CPU attention share (omega > 0) needs kv_policy='offload', a GQA model and no EP "
                             "(the paper runs DeepSeek with omega = 0, PAPER.md:509)")
        hw_sched = b200_hardware()
        if self.n_cpu > 0:  # the schedule only needs a nonzero CPU rate to admit CPU jobs
            hw_sched = Hardware(**{**hw_sched.__dict__, "cpu_attn_flops": 1e11})
        self.schedule: Schedule = build_schedule(self.spec, hw_sched, _unit_latency, self.workload, self.plan,
                                                 kv_policy=kv_policy)
        self.layer_jobs = [[] for _ in range(a.layers)]
        for j in self.schedule.jobs:
            if j.resource is not None and j.layer >= 0:
                self.layer_jobs[j.layer].append(j)
        self.offload = self.plan.s_params < self.spec.model_bytes
        self.kv_ring_cap = kv_ring_slots
        self.use_lookahead = lookahead
        # measurement only: False issues every job except the host<->device copies (compute-only
        # step time for the transfer/compute overlap figure; outputs are then meaningless)
        self.copies_enabled = True
        self.compute_enabled = True  # False: copies only (the link-bound time of the same step)
        self._plan_streams()
        # ---- weights ----
        if self.offload:
            from .offload import OffloadedWeights
            self.w = OffloadedWeights(a, self.spec, self.plan.s_params, self.plan.s_expert, seed=seed,
                                      extra_slots=self.lookahead_expert_slots, extra_dense=len(self.dense_buf_of),
                                      device=device, source=self.source)
        else:
            # an expert-parallel rank generates (or loads) only its expert range [first, first + E_local):
            # DeepSeek-V2 236B EP8 holds 20 of 160 experts per layer, never the 453 GB of all of them
            shard = (self.ep.first, self.ep.E_local) if self.ep is not None else None
            cls = DeepseekDeviceWeights if self.mla else MixtralDeviceWeights
            self.w = cls(a, seed=seed, device=device, source=self.source, experts=shard)
        d, k, f = a.hidden, a.top_k, a.moe_ffn
        bf = dict(dtype=BF16, device=device)
        i32 = dict(dtype=torch.int32, device=device)
        if self.peer_ep:  # local expert GEMM scratch over the whole receive buffer, per-row home pointers
            cap = self.ep.recv.shape[0]
            self.ep_h = torch.zeros(cap, f, **bf)
            self.ep_row_ptr = torch.zeros(cap, dtype=torch.int64, device=device)
        # ---- paged KV (identity block table: sequence b owns pages [b*pps, (b+1)*pps)) ----
        if self.mla:
            # latent pages: swizzled 64-dim blocks [ceil((R + r)/64)][page tok][64] (attn_mla.cu)
            self.page = nat.value("mgb_mla_page_size")
            self.page_elems = nat.value("mgb_mla_page_elems", a.kv_lora_rank, a.qk_rope_dim)
            self.kv_unit = (128, self.page_elems // (64 * self.page), 128 * self.page)  # bytes, runs, run stride
            n_stores = 1
            r = a.qk_rope_dim
            inv_freq = 1.0 / (a.rope_theta ** (torch.arange(0, r, 2, dtype=torch.int64).float() / r))
            freqs = torch.arange(self.max_ctx).float()[:, None] * inv_freq[None, :]
            cis = torch.polar(torch.ones_like(freqs), freqs)  # fp32, HF DeepseekV2RotaryEmbedding
            self.cos_t = cis.real.contiguous().to(device)
            self.sin_t = cis.imag.contiguous().to(device)
        else:
            # chunk-major K and V pages [Hkv][hd/8][page tok][8] (attn_gqa.cu)
            self.page = ops.kv_page_size()
            self.page_elems = a.n_kv_heads * a.head_dim * self.page
            self.kv_unit = (16, a.n_kv_heads * a.head_dim // 8, 16 * self.page)
            n_stores = 2
            # RoPE tables (HF MixtralRotaryEmbedding, bf16-rounded, modeling_mixtral.py:210-220)
            hd = a.head_dim
            inv_freq = 1.0 / (a.rope_theta ** (torch.arange(0, hd, 2, dtype=torch.int64).float() / hd))
            freqs = torch.arange(self.max_ctx).float()[:, None] * inv_freq[None, :]
            self.cos_t = freqs.cos().to(BF16).float().contiguous().to(device)
            self.sin_t = freqs.sin().to(BF16).float().contiguous().to(device)
        self.pps = math.ceil(self.max_ctx / self.page)
        n_pages = B * self.pps
        # kv[l][s] = the page store of layer l, store s (GQA: K, V; MLA: latent): HBM when resident,
        # pinned host memory when offloaded (then see _init_kv_stream for the HBM ring and staging)
        if kv_policy == "resident":
            self.kv = [[torch.zeros(n_pages * self.page_elems, **bf) for _ in range(n_stores)]
                       for _ in range(a.layers)]
        else:
            self._init_kv_stream(n_stores, n_pages)
        if self.mla:
            self.latent = [st[0] for st in self.kv]
        else:
            self.k_cache = [st[0] for st in self.kv]
            self.v_cache = [st[1] for st in self.kv]
        self.block_table = torch.arange(n_pages, dtype=torch.int32, device=device).view(B, self.pps)
        # ---- step buffers ----
        rows = B * k
        if self.mla:
            H = a.n_heads
            qd = H * (a.qk_nope_dim + a.qk_rope_dim)
            self.mb = dict(q=torch.zeros(B, qd, **bf), ckv=torch.zeros(B, a.kv_lora_rank + a.qk_rope_dim, **bf),
                           q_nope=torch.zeros(H * B * a.qk_nope_dim, **bf),
                           q_pe=torch.zeros(B, H, a.qk_rope_dim, **bf),
                           q_lat=torch.zeros(H * B * a.kv_lora_rank, **bf),
                           o_lat=torch.zeros(H * B * a.kv_lora_rank, **bf),
                           o_cat=torch.zeros(B, H * a.v_head_dim, **bf),
                           offsets_all=torch.tensor([0, B], dtype=torch.int32, device=device))
            if a.q_lora_rank:
                self.mb.update(q_a=torch.zeros(B, a.q_lora_rank, **bf), q_an=torch.zeros(B, a.q_lora_rank, **bf))
            fs = a.moe_ffn * a.n_shared
            self.mb.update(sh_h=torch.zeros(B, fs, **bf), de_h=torch.zeros(B, max(a.dense_ffn, 8), **bf),
                           sh_out=torch.zeros(B, d, **bf),
                           logits_r=torch.zeros(B, a.n_experts, dtype=torch.float32, device=device))
            qkv_cols, attn_cols = 8, 8  # unused for MLA
        else:
            hd = a.head_dim
            qkv_cols, attn_cols = (a.n_heads + 2 * a.n_kv_heads) * hd, a.n_heads * hd
        self.buf = StepBuffers(
            x=torch.zeros(B, d, **bf), h=torch.zeros(B, d, **bf), qkv=torch.zeros(B, qkv_cols, **bf),
            q=torch.zeros(B, attn_cols, **bf), attn=torch.zeros(B, attn_cols, **bf), o=torch.zeros(B, d, **bf),
            x_perm=torch.zeros(rows, d, **bf), h_ffn=torch.zeros(rows, f, **bf), y_perm=torch.zeros(rows, d, **bf),
            logits=torch.zeros(B, a.vocab, **bf), next_ids=torch.zeros(B, **i32), positions=torch.zeros(B, **i32),
            seq_lens=torch.zeros(B + 4, **i32), step=torch.zeros(1, **i32))  # +4: 16-byte copies
        self.rws = ops.RouterWorkspace(B, a.n_experts, k, device=device)
        self.out_tokens = torch.zeros(B, max(1, self.max_ctx), dtype=torch.int64, device=device)
        self.graph: torch.cuda.CUDAGraph | None = None
        self.debug_taps: dict | None = None
        self.router_logits = os.environ.get("MGB_ROUTER_LOGITS", "cublas")  # or "fused": GEMV in mgb_router_topk
        self.logits_r = torch.zeros(B, a.n_experts, dtype=torch.float32, device=device)
        self.stream = torch.cuda.Stream(device=device)
        self.streaming = self.offload or kv_policy == "offload"
        self.h2d = torch.cuda.Stream(device=device) if self.streaming else None
        self.d2h = torch.cuda.Stream(device=device) if kv_policy == "offload" else None
        self._join2 = torch.cuda.Event()
        self.cpu_stream = torch.cuda.Stream(device=device) if self.n_cpu > 0 else None
        self._join3 = torch.cuda.Event()
        if self.n_cpu > 0:
            self._init_cpu_attention()
        self._fork, self._join = torch.cuda.Event(), torch.cuda.Event()
        # DeepSeek shared experts on a side stream (MGB_SHARED_STREAM=0: in line): they read only the
        # post-attention norm's rows, so they overlap the router chain (logits GEMM, top-k, scan,
        # permute) and the routed GEMMs' tails, and join before the combine that adds their output.
        # HBM-resident, non-EP engines only (offloaded shared experts live in the dense buffer, which is
        # handed to the next layer's copy right after them, offload_dag.py:308-321)
        self.shared_stream = (torch.cuda.Stream(device=device)
                              if (self.mla and a.n_shared > 0 and not self.offload and self.ep is None
                                  and os.environ.get("MGB_SHARED_STREAM", "1") != "0") else None)
        self._sh_fork, self._sh_join = torch.cuda.Event(), torch.cuda.Event()
        self._sh_pending = False
        self.serial_jobs = False  # measurement: every job in line on one stream (per-kernel breakdowns)
        self.events = {i: torch.cuda.Event() for i in self.need_event}
        self.trace_events: dict | None = None  # job id -> (start, end) timing events (eager trace mode)
        self._trace_counts: torch.Tensor | None = None  # [layers, E] routed rows per expert (trace mode)
        self._forced_logits: torch.Tensor | None = None  # [layers, B, E] router input (force_routing)
        self._segments: dict[int, torch.Tensor] = {}
        # completion counters of the fused expert FFN launch (mgb_moe_ffn); every launch of this engine
        # runs on its compute stream, one after another, and leaves them zero
        self.ffn_sync = torch.zeros(257, dtype=torch.int32, device=device)
        # dynamic work-item counter of the GQA decode attention launches (all on the compute stream)
        self.attn_sched = (torch.zeros(2, dtype=torch.int32, device=device)
                           if os.environ.get("MGB_ATTN_SCHED", "1") != "0" else None)
        ffn_env = os.environ.get("MGB_FFN_FUSED")
        self._ffn_fused = None if ffn_env is None else ffn_env != "0"
        self._dense_mlp_cublas = os.environ.get("MGB_DENSE_MLP", "gemm") == "cublas"
        # decode routing front end as ONE launch (route.cu: residual add + RMSNorm + router logits +
        # top-k + counts/offsets + permutation) for HBM-resident weights without EP; MGB_FUSED_ROUTE=0
        # restores add_rmsnorm + cuBLAS logits + router_topk + permute
        # (measured, tools/route_bench.py: faster for Mixtral's 8 experts; DeepSeek's 64-160-expert routing
        # stays on the unfused kernels, whose cuBLAS logits GEMM and wide top-k grid win there)
        self.fused_route = (os.environ.get("MGB_FUSED_ROUTE", "1") != "0" and not self.offload and self.ep is None
                            and a.n_experts <= 16 and ops.moe_route_supported(B, a.hidden, a.n_experts))
        # one chunk per CTA: the normalised rows need not be written to b.h (only x_perm reads them;
        # the debug taps still get them)
        self._route_1pass = self.fused_route and ops.moe_route_single_pass(B, a.hidden, a.n_experts)
        # GQA decode: the step's RoPE + KV append inside the attention launch (mgb_decode_attn_gqa_rope,
        # MGB_FUSED_ROPE=1) when the pages are the resident store and no CPU share reads the RoPE'd q.
        # Off by default: bit-identical and faster eagerly (12.47 vs 12.29 + 0.41 ms per Mixtral forward),
        # but the graph-replayed step measured 0.3-0.4 ms SLOWER in same-box A/Bs
        self.fused_rope = (os.environ.get("MGB_FUSED_ROPE", "0") == "1" and not self.mla
                           and kv_policy == "resident" and self.n_cpu == 0)
        self.kernel_launches_per_step = self._count_launches()
        self.host_pos = 0

    # ------------------------------------------------------------------------------------
    # job issue
    # ------------------------------------------------------------------------------------
    def mla_family(self) -> bool:
        return self.arch.family == "deepseek_v2"

    def _plan_streams(self) -> None:
        """Cross-resource edges of the serialized schedule become cudaEvent waits; same-resource
        chains are plain in-order stream semantics.  Barriers are expanded into their producers."""
        jobs = self.schedule.jobs
        preds = self.schedule.preds()
        eff: dict[int, list[int]] = {}

        def producers(i: int) -> list[int]:
            if jobs[i].resource is not None:
                return [i]
            if i not in eff:
                out: list[int] = []
                for p in preds[i]:
                    out += producers(p)
                eff[i] = sorted(set(out))
            return eff[i]

        self.xwait: dict[int, list[int]] = {}
        self.need_event: set[int] = set()
        for j in jobs:
            if j.resource is None:
                continue
            w = []
            for p in preds[j.id]:
                for q in producers(p):
                    if jobs[q].resource != j.resource:
                        w.append(q)
            self.xwait[j.id] = sorted(set(w))
            self.need_event.update(w)
        # expert slot of every uncached expert copy: copy k reuses slot k % slots
        # (the schedule's recycle edge, offload_dag.py:446-448)
        self.slot_of: dict[tuple[int, int], int] = {}
        slots = max(1, self.plan.s_expert // self.spec.expert_bytes) if self.spec.expert_bytes else 1
        k = 0
        for j in jobs:
            if j.kind == "weight_copy" and "/expert" in j.label:
                e = int(j.label.split("/expert")[1].split("_")[0])
                self.slot_of[(j.layer, e)] = k % slots
                k += 1
        # first / last expert_compute job of each layer (resident group launch / combine)
        self.first_expert_job, self.last_expert_job = {}, {}
        for j in jobs:
            if j.kind == "expert_compute":
                self.first_expert_job.setdefault(j.layer, j.id)
                self.last_expert_job[j.layer] = j.id
        # KV streaming (kv_policy="offload"): copy-in k lands in ring slot k % n; its slot is free once
        # the attention of copy k - n has run (the schedule's ring edge, offload_dag.py:383-386, when
        # n equals the planner's ring).  The new-token staging pages are double-buffered by layer
        # parity, so pre_attention(l, mb) also waits for kv_copy_out(l - 2, mb) to have read them.
        kins = [j for j in jobs if j.kind == "kv_copy_in"]
        self.kv_ring_n = min(len(kins), self.kv_ring_cap) if kins else 0
        self.kv_slot_of: dict[int, int] = {}
        mech_of_kin: dict[int, int] = {}
        succ = self.schedule.succs()
        for i, kj in enumerate(kins):
            self.kv_slot_of[kj.id] = i % self.kv_ring_n
            mech_of_kin[kj.id] = next(v for v in succ[kj.id] if jobs[v].kind == "attn_mech_gpu")
        self.kin_of_mech = {m: k for k, m in mech_of_kin.items()}
        for i, kj in enumerate(kins):
            if i >= self.kv_ring_n:
                m = mech_of_kin[kins[i - self.kv_ring_n].id]
                self.xwait[kj.id] = sorted(set(self.xwait[kj.id]) | {m})
                self.need_event.add(m)
        kv_out = {(j.layer, j.label.rsplit("/", 1)[1]): j.id for j in jobs if j.kind == "kv_copy_out"}
        for j in jobs:
            if j.kind == "attn_mech_cpu":  # reads the host pages the share's KV_COPY_OUT writes
                o = kv_out[(j.layer, "cpu")]
                self.xwait[j.id] = sorted(set(self.xwait[j.id]) | {o})
                self.need_event.add(o)
            if j.kind == "pre_attention" and (j.layer - 2, j.label.rsplit("/", 1)[1]) in kv_out:
                o = kv_out[(j.layer - 2, j.label.rsplit("/", 1)[1])]
                self.xwait[j.id] = sorted(set(self.xwait[j.id]) | {o})
                self.need_event.add(o)
        self._plan_lookahead(jobs, preds, mech_of_kin)
        if self.plan.B * self.arch.top_k < self.arch.n_experts:
            raise ValueError("B * top_k < experts: some experts would have no scheduled expert_compute job")

    def _plan_lookahead(self, jobs, preds, mech_of_kin) -> None:
        """Cross-step copy lookahead.  The leading H2D copies of a step that wait on no compute of
        their own step (the first dense copy, the first `slots` expert copies, the first KV slices)
        are issued at the END of the previous step, so the host link keeps streaming through the step
        boundary instead of idling while the GPU drains the last layer and starts the next.  Each
        lookahead copy lands in a buffer of its own (one extra dense buffer, expert slot or KV ring
        slot per copy, beyond the plan's s_expert), which only that copy's consumers in the step read:
        the next step's copy into it waits for those consumers alone (and, for a KV slice, for the
        step's KV_COPY_OUT of the same slice), not for the last layer.  The first step of a decode
        call gets them from an eager prologue."""
        copies = [j for j in jobs if j.resource == "htod_link"]
        self.lookahead: list = []
        for c in copies:  # leading copies with no recycle wait on this step's compute
            if self.xwait[c.id] or not self.use_lookahead:
                break
            self.lookahead.append(c)
        ids = {c.id for c in self.lookahead}
        succ = self.schedule.succs()
        kv_out = {(j.layer, j.label.rsplit("/", 1)[1]): j.id for j in jobs if j.kind == "kv_copy_out"}
        n_slots = max(1, self.plan.s_expert // self.spec.expert_bytes) if self.spec.expert_bytes else 1
        self.dense_buf_of: dict[int, int] = {}
        self.lookahead_waits: dict[int, list[int]] = {}
        n_e = n_kv = 0
        for c in self.lookahead:
            if c.label.endswith("dense_copy"):
                self.dense_buf_of[c.layer] = 1
                w = [next(j.id for j in jobs if j.kind == "post_attention" and j.layer == c.layer)]
            elif c.kind == "weight_copy":
                e = int(c.label.split("/expert")[1].split("_")[0])
                self.slot_of[(c.layer, e)] = n_slots + n_e
                n_e += 1
                w = [max(v for v in succ[c.id] if jobs[v].kind == "expert_compute")]
            else:
                self.kv_slot_of[c.id] = self.kv_ring_n + n_kv
                n_kv += 1
                w = [mech_of_kin[c.id], kv_out[(c.layer, c.label.rsplit("/", 1)[1])]]
            self.lookahead_waits[c.id] = w
            self.need_event.update(w)
        self.lookahead_expert_slots, self.lookahead_kv_slots = n_e, n_kv
        # consumers in the step no longer wait on the (previous-step) lookahead copies
        for jid, ws in self.xwait.items():
            self.xwait[jid] = [p for p in ws if p not in ids]
        self.need_event -= ids
        self._lookahead_ids = ids
        self._primed = False

    def _issue_lookahead(self, prologue: bool) -> None:
        """Issue the lookahead copies on the H2D stream: as the eager prologue of a decode call, or
        at the end of a step for the next one (after their buffers' last users in this step)."""
        if not self.lookahead:
            return
        for c in self.lookahead:
            if not prologue:
                for p in self.lookahead_waits[c.id]:
                    self.h2d.wait_event(self.events[p])
            te = None if prologue else self.trace_events
            with torch.cuda.stream(self.h2d):
                if te is not None:
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(self.h2d)
                self._kv_job(c.layer, c) or self._weight_copy_job(c.layer, c)
                if te is not None:
                    e1.record(self.h2d)
                    te[c.id] = (e0, e1)
        self._primed = True

    def prime(self) -> None:
        """Eager prologue: land the lookahead copies the first step of a decode call expects."""
        if self._primed or not self.streaming:
            return
        self.h2d.wait_stream(self.stream)
        self.h2d.wait_stream(torch.cuda.current_stream())
        self._issue_lookahead(prologue=True)
        self.stream.wait_stream(self.h2d)
        torch.cuda.current_stream().wait_stream(self.h2d)

    def _stream_of(self, j) -> torch.cuda.Stream:
        return {"htod_link": self.h2d, "dtoh_link": self.d2h, "cpu_compute": self.cpu_stream}.get(j.resource,
                                                                                                    self.stream)

    def _init_kv_stream(self, n_stores: int, n_pages: int) -> None:
        """Full KV offload (reference memory_model.py:182-205): every sequence's pages live in pinned
        host memory; HBM holds `kv_ring_n` micro-batch slices (the KV_COPY_IN ring) and one staging
        page per sequence and store for the new token, double-buffered by layer parity."""
        a, pe, bf = self.arch, self.page_elems, dict(dtype=BF16, device=self.device)
        per_layer = n_pages * pe
        host = pinned_empty(a.layers * n_stores * per_layer)
        self.kv_host = host
        self.kv = [[host[(l * n_stores + s) * per_layer:(l * n_stores + s + 1) * per_layer] for s in range(n_stores)]
                   for l in range(a.layers)]
        slice_pages = self.plan.b_a * self.pps
        self.kv_ring = [[torch.zeros(slice_pages * pe, **bf) for _ in range(n_stores)]
                        for _ in range(max(1, self.kv_ring_n) + self.lookahead_kv_slots)]
        self.kv_stage = [[torch.zeros(self.B * pe, **bf) for _ in range(n_stores)] for _ in range(2)]
        i32 = dict(dtype=torch.int32, device=self.device)
        # staging table: every page index of sequence b maps to staging page b
        self.stage_table = torch.arange(self.B, **i32)[:, None].expand(self.B, self.pps).contiguous()
        # ring-slot table: the micro-batch's sequence i owns slot pages [i*pps, (i+1)*pps)
        self.slot_table = torch.arange(slice_pages, **i32).view(self.plan.b_a, self.pps)

    def _kv_token_copy(self, src, src_table, dst, dst_table, s0: int, n: int) -> None:
        ub, nu, us = self.kv_unit
        nat.call("mgb_kv_token_copy", src.data_ptr(), src_table.data_ptr(), self.pps, dst.data_ptr(),
                 dst_table.data_ptr(), self.pps, self.buf.positions[s0:].data_ptr(), n, self.page,
                 self.page_elems * 2, ub, nu, us, torch.cuda.current_stream().cuda_stream)

    def _weight_copy_job(self, l: int, j) -> bool:
        """WEIGHT_COPY (offload_dag.py:308-321,438-448): one DMA of a layer's dense blob into the single
        dense buffer, or of one expert's [gate_up | down] blob into its slot."""
        if j.kind != "weight_copy":
            return False
        if not self.copies_enabled:
            return True
        if j.label.endswith("dense_copy"):
            self.w.dense_bufs[self.dense_buf_of.get(l, 0)].copy_(self.w.host_dense[l], non_blocking=True)
        elif self.w.host_experts[l] is not None:  # (DeepSeek-V2's dense first layers have no experts)
            e = int(j.label.split("/expert")[1].split("_")[0])
            n_c = self.w.place.experts_per_layer[l]
            self.w.slots[self.slot_of[(l, e)]].copy_(self.w.host_experts[l][e - n_c], non_blocking=True)
        return True

    def _init_cpu_attention(self) -> None:
        """Pinned staging for the CPU share (q out, output back) and one job description per layer
        for the host node (csrc/cpu_attn.cpp)."""
        a, n = self.arch, self.n_cpu
        width = a.n_heads * a.head_dim
        # the host kernel's limits (csrc/cpu_attn.cpp): refuse here, where the error is visible, instead
        # of a host node that only sets desc.status inside a replayed graph
        G = a.n_heads // a.n_kv_heads
        if a.n_heads % a.n_kv_heads or G > 16 or a.head_dim % 8 or a.head_dim // 8 > 16 or self.page % 4:
            raise ValueError(f"CPU attention share: unsupported shape (G={G}, head_dim={a.head_dim}, "
                             f"page={self.page})")
        self.cpu_q = torch.empty(n, width, dtype=BF16, pin_memory=True)
        self.cpu_lens_bytes = (4 * n + 15) // 16 * 16  # copied in whole 16-byte units
        self.cpu_lens = torch.empty(self.cpu_lens_bytes // 4, dtype=torch.int32, pin_memory=True)
        self.cpu_out = torch.empty(n, width, dtype=BF16, pin_memory=True)
        self.cpu_desc = [nat.CpuAttnGqa(self.kv[l][0].data_ptr(), self.kv[l][1].data_ptr(), self.cpu_q.data_ptr(),
                                        self.cpu_lens.data_ptr(), self.cpu_out.data_ptr(), 0, self.pps, n, a.n_heads,
                                        a.n_kv_heads, a.head_dim, self.page, a.head_dim ** -0.5, 0)
                         for l in range(a.layers)]

    def _cpu_attention_job(self, l: int) -> None:
        """ATTN_MECH_CPU (offload_dag.py:343-357): q and lengths of the CPU share go host-ward, the host
        cores attend over the host page store (a host node of the step's graph), the output comes back
        for post_attention.  All three on the CPU-attention stream, in order."""
        import ctypes

        b, n = self.buf, self.n_cpu
        st = torch.cuda.current_stream().cuda_stream
        # SM-driven copies through mapped pinned memory: these few MB must not queue on a copy
        # engine behind the GPU share's KV_COPY_IN slices
        nat.call("mgb_copy_bytes", self.cpu_q.data_ptr(), b.q.data_ptr(), self.cpu_q.nbytes, st)
        nat.call("mgb_copy_bytes", self.cpu_lens.data_ptr(), b.seq_lens.data_ptr(), self.cpu_lens_bytes, st)
        nat.call("mgb_cpu_attn_gqa_enqueue", ctypes.byref(self.cpu_desc[l]), st)
        nat.call("mgb_copy_bytes", b.attn.data_ptr(), self.cpu_out.data_ptr(), self.cpu_out.nbytes, st)

    def _moved_bytes(self, j) -> float:
        """Bytes a copy job really moves: the schedule's bytes, except the expert copies the
        reference's all-MoE model charges to DeepSeek-V2's dense first layers (no experts exist)."""
        if (j.kind == "weight_copy" and not j.label.endswith("dense_copy") and self.offload
                and self.w.host_experts[j.layer] is None):
            return 0.0
        return j.nbytes

    def _kv_job(self, l: int, j) -> bool:
        """KV_COPY_IN / KV_COPY_OUT jobs (offload_dag.py:372-392); returns False for other kinds."""
        if j.kind in ("kv_copy_in", "kv_copy_out") and not self.copies_enabled:
            return True
        if j.kind == "kv_copy_in":
            s0, s1 = self._mb_range(j)
            r, pe, pps = self.kv_slot_of[j.id], self.page_elems, self.pps
            for s, host in enumerate(self.kv[l]):
                self.kv_ring[r][s][:(s1 - s0) * pps * pe].copy_(host[s0 * pps * pe:s1 * pps * pe], non_blocking=True)
            return True
        if j.kind == "kv_copy_out":
            s0, s1 = self._mb_range(j)
            for s, host in enumerate(self.kv[l]):
                self._kv_token_copy(self.kv_stage[l % 2][s], self.stage_table[s0:], host, self.block_table[s0:],
                                    s0, s1 - s0)
            return True
        return False

    def _kv_views(self, l: int, j, s0: int, s1: int, phase: str):
        """(stores, block_table rows from s0) the pre_attention append / attention of micro-batch
        [s0, s1) of layer l work on.  Resident: the layer's page store.  Offloaded: the staging pages
        for the append; for the attention the ring slot its copy-in filled, after the new token is
        inserted into it."""
        if self.kv_policy == "resident":
            return self.kv[l], self.block_table[s0:]
        if phase == "append":
            return self.kv_stage[l % 2], self.stage_table[s0:]
        kin = self.kin_of_mech[j.id]
        slot = self.kv_ring[self.kv_slot_of[kin]]
        for s in range(len(slot)):
            self._kv_token_copy(self.kv_stage[l % 2][s], self.stage_table[s0:], slot[s], self.slot_table, s0, s1 - s0)
        return slot, self.slot_table

    def _issue_layer(self, l: int) -> None:
        skip = self._lookahead_ids
        for j in self.layer_jobs[l]:
            if j.id in skip:  # landed at the end of the previous step (or by the prologue)
                continue
            st = self._stream_of(j)
            for p in self.xwait.get(j.id, ()):
                st.wait_event(self.events[p])
            with torch.cuda.stream(st):
                te = self.trace_events
                if te is not None:
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(st)
                if self.compute_enabled or j.resource in ("htod_link", "dtoh_link"):
                    self._issue_job(l, j)
                if te is not None:
                    e1.record(st)
                    te[j.id] = (e0, e1)
                    if j.kind == "router" and self._trace_counts is not None:  # outside the timed span
                        self._trace_counts[l].copy_(self.rws.counts)
                if j.id in self.need_event:
                    self.events[j.id].record(st)

    def _layer_weights(self, l: int) -> dict:
        W = self.w.layers[l]
        if self.offload and l >= self.w.place.dense_layers:
            W = dict(W, **self.w.dense_views(self.dense_buf_of.get(l, 0)))
        return W

    # ---- DeepSeek-V2 (MLA) jobs ------------------------------------------------------------
    def _ds_views(self, s0: int, s1: int):
        """Per-micro-batch [H, Bmb, *] views of the head-major MLA scratch buffers."""
        a, m = self.arch, self.mb
        H, n = a.n_heads, s1 - s0
        R, nope, v = a.kv_lora_rank, a.qk_nope_dim, a.v_head_dim
        off = H * s0
        return (m["q_nope"][off * nope:(off + H * n) * nope].view(H, n, nope),
                m["q_lat"][off * R:(off + H * n) * R].view(H, n, R),
                m["o_lat"][off * R:(off + H * n) * R].view(H, n, R),
                # W_UV o_lat lands head-major straight in o_cat's rows (strided batched GEMM output)
                m["o_cat"][s0:s1].view(n, H, v).transpose(0, 1))

    def _ds_job(self, l: int, j, W: dict) -> None:
        """DeepseekV2DecoderLayer (modeling_deepseek_v2.py:399-430) as module jobs; attention in the
        absorbed latent form (q_lat = W_UK^T q_nope, o = W_UV o_lat, attn_mla.cu)."""
        a, b, m = self.arch, self.buf, self.mb
        H, R, r, nope = a.n_heads, a.kv_lora_rank, a.qk_rope_dim, a.qk_nope_dim
        if j.kind == "pre_attention":
            s0, s1 = self._mb_range(j)
            if l == 0:
                ops.add_rmsnorm(b.x[s0:s1], W["ln1"], a.rms_eps, b.h[s0:s1])
            h = b.h[s0:s1]
            if a.q_lora_rank:
                torch.mm(h, W["q_a"].t(), out=m["q_a"][s0:s1])
                ops.add_rmsnorm(m["q_a"][s0:s1], W["q_a_norm"], a.rms_eps, m["q_an"][s0:s1])
                torch.mm(m["q_an"][s0:s1], W["q_b"].t(), out=m["q"][s0:s1])
            else:
                torch.mm(h, W["q_proj"].t(), out=m["q"][s0:s1])
            torch.mm(h, W["kv_a"].t(), out=m["ckv"][s0:s1])
            q_nope, q_lat, _, _ = self._ds_views(s0, s1)
            (cache,), table = self._kv_views(l, j, s0, s1, "append")
            nat.call("mgb_mla_append", m["q"][s0:s1].data_ptr(), m["ckv"][s0:s1].data_ptr(),
                     W["kv_a_norm"].data_ptr(), a.rms_eps, s1 - s0, H, R, r, nope, b.positions[s0:].data_ptr(),
                     self.cos_t.data_ptr(), self.sin_t.data_ptr(), table.data_ptr(), self.pps,
                     cache.data_ptr(), q_nope.data_ptr(), m["q_pe"][s0:s1].data_ptr(),
                     b.seq_lens[s0:].data_ptr(), torch.cuda.current_stream().cuda_stream)
            torch.bmm(q_nope, W["w_uk"], out=q_lat)
        elif j.kind == "attn_mech_gpu":
            s0, s1 = self._mb_range(j)
            _, q_lat, o_lat, o_hb = self._ds_views(s0, s1)
            scale = (a.qk_nope_dim + a.qk_rope_dim) ** -0.5
            (cache,), table = self._kv_views(l, j, s0, s1, "attend")
            nat.call("mgb_decode_attn_mla", q_lat.data_ptr(), m["q_pe"][s0:s1].data_ptr(), cache.data_ptr(),
                     table.data_ptr(), self.pps, b.seq_lens[s0:].data_ptr(), s1 - s0, H, R, r, scale,
                     o_lat.data_ptr(), torch.cuda.current_stream().cuda_stream)
            torch.bmm(o_lat, W["w_uv_t"], out=o_hb)  # o_hb is a [H, n, v] view of o_cat[s0:s1]
        elif j.kind == "post_attention":
            torch.mm(m["o_cat"], W["wo"].t(), out=b.o)
            if self._route_fused(l):
                return  # residual add + norm, routing and the shared experts run in the router job
            ops.add_rmsnorm(b.x, W["ln2"], a.rms_eps, b.h, delta=b.o, x_out=b.x)
            if l >= a.first_k_dense:
                # shared experts on every token (DeepseekV2Moe.shared_experts) as one grouped-GEMM
                # segment.  They are part of the layer's dense modules (dense_bytes_per_layer), so with
                # offloaded weights they run before the single dense buffer is handed to the next
                # layer's copy (offload_dag.py:308-321); resident, they run on the side stream
                if self.shared_stream is not None and self.trace_events is None and not self.serial_jobs:
                    cur = torch.cuda.current_stream()
                    self._sh_fork.record(cur)
                    with torch.cuda.stream(self.shared_stream):
                        self.shared_stream.wait_event(self._sh_fork)
                        self._dense_mlp(W["sh_gate_up"], W["sh_down"], b.h, m["sh_h"], m["sh_out"],
                                        m["offsets_all"])
                        self._sh_join.record(self.shared_stream)
                    self._sh_pending = True
                else:
                    self._dense_mlp(W["sh_gate_up"], W["sh_down"], b.h, m["sh_h"], m["sh_out"], m["offsets_all"])
        elif j.kind == "router":
            if self._route_fused(l):
                ops.moe_route(b.x, b.o, W["ln2"], a.rms_eps, b.h, W["router"], self.rws, b.x_perm, a.router_mode,
                              a.routed_scaling, a.n_group, a.topk_group, x_out=b.x, logits_out=m["logits_r"])
                self._dense_mlp(W["sh_gate_up"], W["sh_down"], b.h, m["sh_h"], m["sh_out"], m["offsets_all"])
                if self.debug_taps is not None:
                    self.debug_taps.update(h2=b.h.clone(), topk_idx=self.rws.topk_idx.clone())
            elif l >= a.first_k_dense:
                # fp32 router logits (HF: F.linear(x.float(), W.float()), modeling_deepseek_v2.py:125) as a
                # bf16 tensor-core GEMM with fp32 output (exact products, fp32 accumulation)
                lg = m["logits_r"]
                if self._forced_logits is not None:
                    lg = self._forced_logits[l]
                else:
                    torch.mm(b.h, W["router"].t(), out_dtype=torch.float32, out=lg)
                ops.router_topk(None, None, self.rws, a.top_k, a.router_mode, a.routed_scaling, a.n_group,
                                a.topk_group, logits_in=lg)
                if not self.peer_ep:
                    ops.permute(b.h, self.rws, b.x_perm)
                if self.debug_taps is not None:
                    self.debug_taps.update(h2=b.h.clone(), topk_idx=self.rws.topk_idx.clone())
        elif j.kind == "expert_compute":
            if l < a.first_k_dense:
                # dense MLP of the first layers (DeepseekV2MLP): cuBLAS + fused SiLU*up
                if j.id == self.first_expert_job[l]:
                    nxt = self.w.layers[l + 1]["ln1"] if l + 1 < a.layers else self.w.final_norm
                    F = a.dense_ffn
                    self._dense_mlp(W["dense_gate_up"], W["dense_down"], b.h, m["de_h"][:, :F], b.o, m["offsets_all"])
                    ops.add_rmsnorm(b.x, nxt, a.rms_eps, b.h, delta=b.o, x_out=b.x)
                return
            self._expert_job(l, j, W, shared_out=m["sh_out"])
        else:
            raise RuntimeError(f"job kind {j.kind!r} is not executable under kv_policy={self.kv_policy!r}")

    def _dense_mlp(self, w_gate_up, w_down, x, h, y, seg) -> None:
        """A dense SwiGLU MLP (DeepSeek-V2's shared experts, DeepseekV2Moe.shared_experts, and the dense
        first layers' DeepseekV2MLP, modeling_deepseek_v2.py:134-146) as ONE segment of the grouped
        expert GEMMs: w_gate_up [1, 2F, d] (gate rows then up rows), w_down [1, d, F], all T rows of x
        in segment `seg` = [0, T]; SiLU*up is formed in the gate/up GEMM's epilogue (no separate
        activation pass).  MGB_DENSE_MLP=cublas restores cuBLAS + mgb_silu_mul (A/B measurement)."""
        if self._dense_mlp_cublas:
            gu = torch.mm(x, w_gate_up[0].t())
            ops.silu_mul(gu, h)
            torch.mm(h, w_down[0].t(), out=y)
            return
        self._ffn(w_gate_up, w_down, x, seg, h, y)

    def _ffn(self, w_gate_up, w_down, x, offsets, h, y) -> None:
        """Expert FFN over expert-major rows: the fused single launch (mgb_moe_ffn) for a few large
        experts (Mixtral: its gate/up and down waves share one tail, -3.5 % of the FFN time in the bench,
        same-box A/B), two grouped launches otherwise (DeepSeek's 64 routed experts: +3 % fused; a
        single expert segment: every down unit would wait for the last gate/up unit anyway).
        MGB_FFN_FUSED=0/1 forces either."""
        E = w_gate_up.shape[0]
        fused = self._ffn_fused if self._ffn_fused is not None else 2 <= E <= 16
        if fused:
            ops.moe_ffn(w_gate_up, w_down, x, offsets, h, y, self.ffn_sync)
        else:
            ops.moe_gemm_gate_up(w_gate_up, x, offsets, h)
            ops.moe_gemm_down(w_down, h, offsets, y)

    def _segment(self, T: int) -> torch.Tensor:
        """Device offsets [0, T] of a one-segment grouped GEMM (cached per T)."""
        seg = self._segments.get(T)
        if seg is None:
            seg = self._segments[T] = torch.tensor([0, T], dtype=torch.int32, device=self.device)
        return seg

    def _expert_job(self, l: int, j, W: dict, shared_out=None) -> None:
        """EXPERT_COMPUTE (offload_dag.py:449-463).  The b_e chunks of one expert run inside one
        persistent grouped launch (the kernel's token tiles are the chunks); all HBM-resident experts
        of the layer share one launch, each streamed expert runs from its slot once its copy has
        landed; the layer's last job combines back to token order (+ shared experts, + residual) and
        applies the next layer's input norm."""
        a, b = self.arch, self.buf
        e = int(j.label.split("/expert")[1].split("/")[0])
        first_chunk = j.label.endswith("/chunk0")
        n_c = self.w.place.experts_per_layer[l] if self.offload else a.n_experts
        if j.id == self.first_expert_job[l] and n_c > 0:
            self._routed_experts(W)
        elif first_chunk and e >= n_c:
            gu, dn = self.w.slot_views(self.slot_of[(l, e)])
            offs = self.rws.offsets[e:e + 2]
            self._ffn(gu, dn, b.x_perm, offs, b.h_ffn, b.y_perm)
        if j.id == self.last_expert_job[l]:
            nxt = self.w.layers[l + 1]["ln1"] if l + 1 < a.layers else self.w.final_norm
            y_perm = self.ep.yperm if self.peer_ep else b.y_perm
            if self._sh_pending:  # the shared experts' side stream joins before their output is added
                torch.cuda.current_stream().wait_event(self._sh_join)
                self._sh_pending = False
            ops.unpermute_combine(y_perm, self.rws, b.x, self.B, residual=b.x, shared_out=shared_out,
                                  norm_w=nxt, eps=a.rms_eps, norm_out=b.h)

    def _routed_experts(self, W: dict) -> None:
        """Grouped expert FFN over the permuted rows; with expert parallelism the rows go to the
        experts' owner ranks and back around the local grouped GEMMs (ep.py)."""
        b = self.buf
        if self.ep is None:
            self._ffn(W["w_gate_up"], W["w_down"], b.x_perm, self.rws.offsets, b.h_ffn, b.y_perm)
            return
        a, ep = self.arch, self.ep
        if self.peer_ep:
            # counts of every rank -> device tables; this rank's routed rows into the owners' receive
            # buffers; barrier; local experts, each output row stored at its home rank's y_perm by the
            # down GEMM's epilogue; barrier (offload_dag.py:418-472: the exchange sits on the
            # router -> expert and expert -> combine edges)
            counts_all = ep.comm.exchange_counts(self.rws.counts)
            tab = ep.tables(counts_all)
            ep.dispatch(b.h, self.rws, tab)
            ep.comm.barrier()
            ep.experts(W["w_gate_up"], W["w_down"], ep.recv, self.ep_h, self.ep_row_ptr, tab)
            ep.comm.barrier()
            return
        x_loc, offs, st = ep.dispatch(b.x_perm, self.rws.counts)
        n = x_loc.shape[0]
        y_loc = torch.empty(n, a.hidden, dtype=BF16, device=self.device)
        if n > 0:
            h = torch.empty(n, a.moe_ffn, dtype=BF16, device=self.device)
            self._ffn(W["w_gate_up"], W["w_down"], x_loc, offs, h, y_loc)
        y = ep.combine(y_loc, st)
        b.y_perm[:y.shape[0]].copy_(y)

    def _issue_job(self, l: int, j) -> None:
        a, b = self.arch, self.buf
        if self._kv_job(l, j) or self._weight_copy_job(l, j):
            return
        if j.kind == "attn_mech_cpu":
            return self._cpu_attention_job(l)
        W = self._layer_weights(l)
        if self.mla:
            return self._ds_job(l, j, W)
        hd, Hq, Hkv = a.head_dim, a.n_heads, a.n_kv_heads
        if j.kind == "pre_attention":
            s0, s1 = self._mb_range(j)
            if l == 0:  # later layers get h from the previous layer's fused combine+norm
                ops.add_rmsnorm(b.x[s0:s1], W["ln1"], a.rms_eps, b.h[s0:s1])
            torch.mm(b.h[s0:s1], W["wqkv"].t(), out=b.qkv[s0:s1])
            if not self.fused_rope:  # else the attention launch rotates and appends
                (kc, vc), table = self._kv_views(l, j, 0, s1, "append")
                ops.rope_append_gqa(b.qkv[s0:s1], s0, b.positions, self.cos_t, self.sin_t, Hq, Hkv, hd,
                                    table, kc, vc, b.q[s0:s1], b.seq_lens)
        elif j.kind == "attn_mech_gpu":
            s0, s1 = self._mb_range(j)
            (kc, vc), table = self._kv_views(l, j, s0, s1, "attend")
            if self.fused_rope:
                ops.decode_attn_gqa_rope(b.qkv[s0:s1], b.positions[s0:s1], self.cos_t, self.sin_t, kc, vc,
                                         table[:s1 - s0], b.seq_lens[s0:s1], Hq, Hkv, hd, b.attn[s0:s1],
                                         sched=self.attn_sched)
            else:
                ops.decode_attn_gqa(b.q[s0:s1], kc, vc, table[:s1 - s0], b.seq_lens[s0:s1], Hq, Hkv, hd,
                                    b.attn[s0:s1], sched=self.attn_sched)
        elif j.kind == "post_attention":
            torch.mm(b.attn, W["wo"].t(), out=b.o)
            if not self._route_fused(l):  # else the router job's fused kernel adds + normalises
                ops.add_rmsnorm(b.x, W["ln2"], a.rms_eps, b.h, delta=b.o, x_out=b.x)
        elif j.kind == "router":
            if self._route_fused(l):
                h_out = None if (self._route_1pass and self.debug_taps is None) else b.h
                ops.moe_route(b.x, b.o, W["ln2"], a.rms_eps, h_out, W["router"], self.rws, b.x_perm, a.router_mode,
                              a.routed_scaling, a.n_group, a.topk_group, x_out=b.x, logits_out=self.logits_r)
            elif self._forced_logits is not None:
                ops.router_topk(None, None, self.rws, a.top_k, a.router_mode, a.routed_scaling, a.n_group,
                                a.topk_group, logits_in=self._forced_logits[l])
            elif self.router_logits == "cublas":
                # gate GEMM on the tensor cores with fp32 output; the router kernel rounds it to
                # bf16 exactly as HF's bf16 F.linear does (modeling_mixtral.py:111)
                torch.mm(b.h, W["router"].t(), out_dtype=torch.float32, out=self.logits_r)
                ops.router_topk(None, None, self.rws, a.top_k, a.router_mode, a.routed_scaling, a.n_group,
                                a.topk_group, logits_in=self.logits_r)
            else:
                ops.router_topk(b.h, W["router"], self.rws, a.top_k, a.router_mode, a.routed_scaling,
                                a.n_group, a.topk_group)
            if not self.peer_ep and not self._route_fused(l):  # peer EP permutes inside its dispatch
                ops.permute(b.h, self.rws, b.x_perm)
            if self.debug_taps is not None:  # eager-only parity hook
                self.debug_taps.update(h2=b.h.clone(), topk_idx=self.rws.topk_idx.clone(), attn=b.attn.clone())
        elif j.kind == "expert_compute":
            self._expert_job(l, j, W)
        else:
            raise RuntimeError(f"job kind {j.kind!r} is not executable under kv_policy={self.kv_policy!r}")

    def _route_fused(self, l: int) -> bool:
        """Layer l's routing front end runs as the fused mgb_moe_route launch (MoE layers of a resident,
        non-EP engine without forced routing)."""
        return (self.fused_route and self._forced_logits is None
                and not (self.mla and l < self.arch.first_k_dense))

    def _mb_range(self, j) -> tuple[int, int]:
        """Sequences of a per-micro-batch job: the CPU share is [0, n_cpu), GPU micro-batch m is
        [n_cpu + m*b_a, ...) (the schedule issues the CPU share first, offload_dag.py:328-357)."""
        if j.label.endswith("/cpu"):
            return 0, self.n_cpu
        mb = int(j.label.rsplit("mb", 1)[1])
        s0 = self.n_cpu + mb * self.plan.b_a
        if j.kind in ("kv_copy_in", "kv_copy_out"):  # copy jobs carry bytes, not seqs
            return s0, min(s0 + self.plan.b_a, self.plan.B)
        return s0, s0 + j.seqs

    def _count_launches(self) -> int:
        n = 1  # embed (the final norm is fused into the last combine)
        for l in range(self.arch.layers):
            fused = self._route_fused(l)  # one mgb_moe_route instead of add_rmsnorm + router_topk + permute
            for j in self.layer_jobs[l]:
                pre = (1 if l == 0 else 0) + (0 if getattr(self, "fused_rope", False) else 1)
                n += {"pre_attention": pre, "attn_mech_gpu": 1, "post_attention": 0 if fused else 1,
                      "router": 1 if fused else 2}.get(j.kind, 0)
            n += 3  # gate_up, down, combine
        return n + 2  # argmax, advance  (cuBLAS GEMMs are library launches, not counted)

    def _step(self, record: bool = True) -> None:
        """One decode forward of all B sequences (one token each)."""
        a, b = self.arch, self.buf
        if self.streaming:  # fork the copy streams off the compute stream
            self._fork.record(self.stream)
            self.h2d.wait_event(self._fork)
            if self.d2h is not None:
                self.d2h.wait_event(self._fork)
            if self.cpu_stream is not None:
                self.cpu_stream.wait_event(self._fork)
            if not self._primed:  # eager first step: land this step's lookahead copies now
                self._issue_lookahead(prologue=True)
                self.stream.wait_stream(self.h2d)
        ops.embed(b.next_ids, self.w.embed, b.x)
        for l in range(a.layers):
            self._issue_layer(l)
        if self.streaming:  # next step's leading copies stream while the GPU finishes this one
            self._issue_lookahead(prologue=False)
        torch.mm(b.h, self.w.lm_head.t(), out=b.logits)
        ops.argmax(b.logits, b.next_ids)
        if self.streaming:  # join: every copy has landed -- and, before positions advance, every
            # KV_COPY_OUT / CPU-attention job (they read this step's positions) has run
            self._join.record(self.h2d)
            self.stream.wait_event(self._join)
            if self.d2h is not None:
                self._join2.record(self.d2h)
                self.stream.wait_event(self._join2)
            if self.cpu_stream is not None:
                self._join3.record(self.cpu_stream)
                self.stream.wait_event(self._join3)
        ops.decode_advance(b.next_ids, self.out_tokens if record else None, b.step, b.positions)

    # ------------------------------------------------------------------------------------
    # graph capture / replay
    # ------------------------------------------------------------------------------------
    def capture(self) -> None:
        if self.graph is not None or not self.use_graph:
            return
        # snapshot mutable state: the eager warm-up step must not advance it
        snap = [t.clone() for t in (self.buf.positions, self.buf.step, self.buf.next_ids, self.buf.seq_lens)]
        self.stream.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(self.stream):
            self._step()
        torch.cuda.current_stream().wait_stream(self.stream)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        n0 = nat.LIB.calls
        with torch.cuda.graph(g, stream=self.stream):
            self._step()
        self.kernel_launches_per_step = nat.LIB.calls - n0  # libmgb launches captured per step
        torch.cuda.synchronize()
        for t, s in zip((self.buf.positions, self.buf.step, self.buf.next_ids, self.buf.seq_lens), snap):
            t.copy_(s)
        torch.cuda.synchronize()
        self.graph = g

    def run_step(self) -> None:
        # every sequence appends one token at `host_pos`: past the paged context the block table has
        # no page for it, so refuse rather than let a kernel index outside the cache
        if not 0 <= self.host_pos < self.max_ctx:
            raise ValueError(f"decode position {self.host_pos} outside the planned context [0, {self.max_ctx})")
        self.host_pos += 1
        if self.use_graph:
            if self.graph is None:
                self.capture()
            self.prime()
            self.graph.replay()
        else:  # eager issue on the engine stream, ordered after the caller's stream both ways
            self.stream.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(self.stream):
                self._step()
            torch.cuda.current_stream().wait_stream(self.stream)

    # ------------------------------------------------------------------------------------
    # public API
    # ------------------------------------------------------------------------------------
    def reset(self, start_pos: int = 0) -> None:
        self._primed = False
        self.host_pos = start_pos  # host mirror of the (uniform) device positions
        self.buf.positions.fill_(start_pos)
        self.buf.seq_lens.fill_(start_pos)
        self.buf.step.zero_()
        self.out_tokens.zero_()

    def synthetic_prefill(self, seed: int = 1, std: float = 1.0) -> None:
        """Stand-in for the prefill phase (excluded from the decode metric): fill every KV page
        with counter-based values (std ~ real K/V scale) and position all sequences at
        prompt_len, so decode steps attend over prompt_len..prompt_len+decode_len keys."""
        from .weights import fill_uniform_
        for l in range(self.arch.layers):
            for s, store in enumerate(self.kv[l]):
                tid = 10_000_000 + 2 * l + s  # MLA: one latent store per layer; GQA: K then V
                if store.is_cuda:
                    fill_uniform_(store, seed, tid, std)
                else:  # host page store of the offloaded KV: generate on the device, then copy
                    store.copy_(fill_uniform_(torch.empty_like(store, device=self.device), seed, tid, std))
        torch.cuda.synchronize()
        self._primed = False
        self.reset(self.prompt_len)

    def force_routing(self, counts: list | None) -> None:
        """Route every decode step by prescribed per-expert token counts instead of the gate GEMM
        (counts[l][e] rows of layer l go to expert e, sum B * top_k) -- the reference simulator's
        routing stand-in (exec_sim.py:61-81, `simulate.sample_routing`), so a measured step and
        `simulate_plan` see the same expert groups.  The assignment lists expert e counts[l][e]
        times in expert order and hands entry i to token i % B as its (i // B)-th choice; a token
        never gets one expert twice because counts[l][e] <= B.  The router kernel then runs on
        logits that are 0 for a token's experts and -1e4 elsewhere.  None restores the gate."""
        if counts is None:
            self._forced_logits = None
            return
        a, B, k, E = self.arch, self.B, self.arch.top_k, self.arch.n_experts
        if a.router_mode == 2:
            raise NotImplementedError("forced routing under group-limited selection")
        if len(counts) != a.layers:
            raise ValueError(f"need counts for {a.layers} layers, got {len(counts)}")
        lg = torch.full((a.layers, B, E), -1e4, dtype=torch.float32)
        for l, row in enumerate(counts):
            row = [int(c) for c in row]
            if len(row) != E or sum(row) != B * k or min(row) < 0:
                raise ValueError(f"layer {l}: counts must be {E} non-negative ints summing to B*top_k={B * k}")
            if max(row) > B:
                raise ValueError(f"layer {l}: an expert cannot take {max(row)} of {B} tokens (each token picks it once)")
            flat = torch.repeat_interleave(torch.arange(E), torch.tensor(row))
            tok = torch.arange(B * k) % B
            lg[l, tok, flat] = 0.0
        self._forced_logits = lg.to(self.device)
        self.graph = None  # the captured step read the gate GEMM's output

    def check_cpu_attention(self) -> None:
        """Raise if a CPU-attention host node reported invalid input (desc.status != 0); call after
        the steps have completed (the status is written by the host node when it runs)."""
        if self.n_cpu > 0:
            bad = [l for l, dsc in enumerate(self.cpu_desc) if dsc.status != 0]
            if bad:
                raise RuntimeError(f"CPU attention failed (status != 0) in layers {bad}")

    def decode(self, first_tokens: torch.Tensor, n_steps: int) -> torch.Tensor:
        """Decode phase through the public API: host `first_tokens` [B] (pinned H2D), n_steps
        greedy forwards from the current positions; returns host int64 [B, n_steps]."""
        assert first_tokens.shape == (self.B,)
        self.buf.next_ids.copy_(first_tokens.to(torch.int32), non_blocking=True)
        self.buf.step.zero_()
        for _ in range(n_steps):
            self.run_step()
        out = self.out_tokens[:, :n_steps].to("cpu", non_blocking=False)
        self.check_cpu_attention()
        return out

    def can_prefill(self) -> bool:
        """Batched prefill: both families, weights resident (chunk-major) or offloaded (layer-major,
        `_prefill_streamed`), KV resident or in the host page store (incl. a CPU attention share);
        not under expert parallelism (the prompt then goes through the decode step)."""
        return self.ep is None

    def _prefill_kv_target(self, l: int, s0: int, n: int):
        """(stores, block table, seq0) the prefill KV write of sequences [s0, s0+n) goes to: the HBM
        page store, or -- with the KV offloaded -- a device staging copy of the chunk's pages that
        `_prefill_kv_flush` then moves to the host store in one contiguous copy per store."""
        if self.kv_policy == "resident":
            return self.kv[l], self.block_table, s0
        pe, pps = self.page_elems, self.pps
        if getattr(self, "_pf_stage_pages", 0) < n * pps:
            # zeros: the flush copies whole pages, so positions >= P of every staged page reach the host
            # store; decode reads those rows (as P = 0 columns) and they must never hold NaN / Inf bits
            self._pf_stage = [torch.zeros(n * pps * pe, dtype=BF16, device=self.device) for _ in self.kv[l]]
            self._pf_stage_table = torch.arange(n * pps, dtype=torch.int32, device=self.device).view(n, pps)
            self._pf_stage_pages = n * pps
        return self._pf_stage, self._pf_stage_table, 0

    def _prefill_kv_flush(self, l: int, s0: int, n: int) -> None:
        if self.kv_policy == "resident":
            return
        pe, pps = self.page_elems, self.pps
        for s, host in enumerate(self.kv[l]):
            host[s0 * pps * pe:(s0 + n) * pps * pe].copy_(self._pf_stage[s][:n * pps * pe], non_blocking=True)

    def _prefill_scratch(self, T: int) -> dict:
        """Activation buffers for one chunk of T prompt tokens (allocated once, grown on demand)."""
        if getattr(self, "_pf_T", 0) >= T:
            return self._pf
        a, k = self.arch, self.arch.top_k
        d = a.hidden
        bf = dict(dtype=BF16, device=self.device)
        S = dict(x=torch.empty(T, d, **bf), h=torch.empty(T, d, **bf), o=torch.empty(T, d, **bf),
                 xp=torch.empty(T * k, d, **bf), hf=torch.empty(T * k, a.moe_ffn, **bf), yp=torch.empty(T * k, d, **bf),
                 lg=torch.empty(T, a.n_experts, dtype=torch.float32, device=self.device),
                 ws=ops.RouterWorkspace(T, a.n_experts, k, device=self.device))
        if self.mla:
            H, qk = a.n_heads, a.qk_nope_dim + a.qk_rope_dim
            fs = a.moe_ffn * a.n_shared
            S.update(q=torch.empty(T, H * qk, **bf), ckv=torch.empty(T, a.kv_lora_rank + a.qk_rope_dim, **bf),
                     c=torch.empty(T, a.kv_lora_rank, **bf), kpe=torch.empty(T, a.qk_rope_dim, **bf),
                     kv=torch.empty(T, H * (a.qk_nope_dim + a.v_head_dim), **bf), k=torch.empty(T, H, qk, **bf),
                     attn=torch.empty(T, H * a.v_head_dim, **bf), sh_h=torch.empty(T, fs, **bf),
                     sh_out=torch.empty(T, d, **bf))
            if a.q_lora_rank:
                S.update(qa=torch.empty(T, a.q_lora_rank, **bf), qan=torch.empty(T, a.q_lora_rank, **bf))
            if a.first_k_dense:
                S.update(de_h=torch.empty(T, a.dense_ffn, **bf))
        else:
            hd, Hq, Hkv = a.head_dim, a.n_heads, a.n_kv_heads
            S.update(qkv=torch.empty(T, (Hq + 2 * Hkv) * hd, **bf), q=torch.empty(T, Hq * hd, **bf),
                     k=torch.empty(T, Hkv * hd, **bf), v=torch.empty(T, Hkv * hd, **bf),
                     attn=torch.empty(T, Hq * hd, **bf))
        self._pf, self._pf_T = S, T
        return S

    def _prefill_attention_gqa(self, l: int, W: dict, S: dict, s0: int, n: int, P: int,
                               h: torch.Tensor) -> torch.Tensor:
        a = self.arch
        t, hd, Hq, Hkv = n * P, a.head_dim, a.n_heads, a.n_kv_heads
        qkv, q, kk, vv = S["qkv"][:t], S["q"][:t], S["k"][:t], S["v"][:t]
        torch.mm(h, W["wqkv"].t(), out=qkv)
        (kc, vc), table, seq0 = self._prefill_kv_target(l, s0, n)
        nat.call("mgb_rope_append_gqa_prefill", qkv.data_ptr(), t, seq0, P, self.cos_t.data_ptr(),
                 self.sin_t.data_ptr(), Hq, Hkv, hd, table.data_ptr(), self.pps, kc.data_ptr(), vc.data_ptr(),
                 q.data_ptr(), kk.data_ptr(), vv.data_ptr(), torch.cuda.current_stream().cuda_stream)
        self._prefill_kv_flush(l, s0, n)
        if self._prefill_kernel(hd, hd):  # tcgen05 causal attention (attn_prefill.cu)
            att = S["attn"][:t]
            ops.prefill_attn(q, kk, vv, att, n, P, Hq, Hkv, hd, hd, hd ** -0.5, hd, hd, hd)
            return att
        # head dims the kernel is not instantiated for (the tiny test models): torch SDPA
        att = torch.nn.functional.scaled_dot_product_attention(
            q.view(n, P, Hq, hd).transpose(1, 2), kk.view(n, P, Hkv, hd).transpose(1, 2),
            vv.view(n, P, Hkv, hd).transpose(1, 2), is_causal=True, enable_gqa=True)
        return att.transpose(1, 2).reshape(t, Hq * hd)

    def _prefill_kernel(self, hd_qk: int, hd_v: int, rope: int = 0) -> bool:
        """Whether the prefill attention runs on mgb_prefill_attn (MGB_PREFILL_ATTN=sdpa: torch SDPA, A/B)."""
        if os.environ.get("MGB_PREFILL_ATTN", "mgb") == "sdpa":
            return False
        return ops.prefill_attn_supported(hd_qk, hd_v) and rope % 64 == 0 and (hd_qk - rope) % 64 == 0

    def _prefill_attention_mla(self, l: int, W: dict, S: dict, s0: int, n: int, P: int,
                               h: torch.Tensor) -> torch.Tensor:
        """HF DeepseekV2Attention on the prompt (modeling_deepseek_v2.py:337-396): the latent is
        up-projected per head (no absorption: every key is attended by P queries), causal SDPA."""
        a = self.arch
        t, H, R, r, nope, vd = n * P, a.n_heads, a.kv_lora_rank, a.qk_rope_dim, a.qk_nope_dim, a.v_head_dim
        q = S["q"][:t]
        if a.q_lora_rank:
            torch.mm(h, W["q_a"].t(), out=S["qa"][:t])
            ops.add_rmsnorm(S["qa"][:t], W["q_a_norm"], a.rms_eps, S["qan"][:t])
            torch.mm(S["qan"][:t], W["q_b"].t(), out=q)
        else:
            torch.mm(h, W["q_proj"].t(), out=q)
        torch.mm(h, W["kv_a"].t(), out=S["ckv"][:t])
        (cache,), table, seq0 = self._prefill_kv_target(l, s0, n)
        nat.call("mgb_mla_append_prefill", q.data_ptr(), S["ckv"].data_ptr(), W["kv_a_norm"].data_ptr(), a.rms_eps, t,
                 seq0, P, H, R, r, nope, self.cos_t.data_ptr(), self.sin_t.data_ptr(), table.data_ptr(),
                 self.pps, cache.data_ptr(), S["c"].data_ptr(), S["kpe"].data_ptr(),
                 torch.cuda.current_stream().cuda_stream)
        self._prefill_kv_flush(l, s0, n)
        kv = S["kv"][:t]
        torch.mm(S["c"][:t], W["kv_b"].t(), out=kv)
        if self._prefill_kernel(nope + r, vd, r):
            # K_h = [k_nope_h | k_pe] read straight from the up-projected rows and the shared rotated
            # k_pe rows; V_h = the v part of the same rows (no per-head K is materialised)
            att = S["attn"][:t]
            ops.prefill_attn(q, kv, kv, att, n, P, H, H, nope + r, vd, (nope + r) ** -0.5, nope + r, nope + vd,
                             nope + vd, v_col0=nope, kr=S["kpe"][:t])
            return att
        kv = kv.view(t, H, nope + vd)
        k = S["k"][:t]
        k[:, :, :nope].copy_(kv[:, :, :nope])
        k[:, :, nope:].copy_(S["kpe"][:t, None, :].expand(t, H, r))
        att = torch.nn.functional.scaled_dot_product_attention(
            q.view(n, P, H, nope + r).transpose(1, 2), k.view(n, P, H, nope + r).transpose(1, 2),
            kv[:, :, nope:].reshape(n, P, H, vd).transpose(1, 2), is_causal=True, scale=(nope + r) ** -0.5)
        return att.transpose(1, 2).reshape(t, H * vd)

    @torch.no_grad()
    def prefill(self, input_ids: torch.Tensor, chunk_tokens: int | None = None) -> torch.Tensor:
        """Batched prefill (the reference's prefill phase: every prompt token of a sequence in one
        forward, tokens_per_seq_in_flight = P, memory_model.py:53-60).  Sequences
        are processed `chunk_tokens // P` at a time: embed -> per layer the family's attention on the
        prompt (RoPE + paged KV / latent write by mgb_rope_append_gqa_prefill / mgb_mla_append_prefill,
        causal torch SDPA on contiguous K/V rows), O GEMM + residual/norm, then the same router /
        grouped expert GEMM / combine kernels as decode (DeepSeek: shared experts, dense first layers)
        -> LM head on each sequence's last position.  Leaves every sequence at position P with its
        first generated token in next_ids (and out_tokens[:, P-1]); returns it (host int64 [B])."""
        if not self.can_prefill():
            raise NotImplementedError("batched prefill is not available for this engine configuration (see can_prefill)")
        a, b = self.arch, self.buf
        B, P = input_ids.shape
        assert B == self.B and 1 <= P <= self.max_ctx
        if self.offload:
            return self._prefill_streamed(input_ids, chunk_tokens or 32768)
        if chunk_tokens is None:
            # at most ~4096 routed rows per expert per chunk: the grouped down GEMM keeps its token tiles
            # in L2 there (Mixtral-8x7B: 16 k-token chunks 41.9 k vs 40.6 k prompt tokens/s at 32 k; 8 k
            # rows per expert drop its down GEMM to 0.64 of peak), capped at 32 k tokens
            chunk_tokens = min(32768, max(P, 4096 * a.n_experts // a.top_k))
        Bp = max(1, min(B, chunk_tokens // P))
        S = self._prefill_scratch(Bp * P)
        d, k = a.hidden, a.top_k
        ids = input_ids.to(self.device, torch.int32)
        self.reset(0)
        self.stream.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(self.stream):
            for s0 in range(0, B, Bp):
                n = min(Bp, B - s0)
                t = n * P
                x, h, o = S["x"][:t], S["h"][:t], S["o"][:t]
                ops.embed(ids[s0:s0 + n].reshape(-1), self.w.embed, x)
                ws = S["ws"]
                for l in range(a.layers):
                    W = self.w.layers[l]
                    if l == 0:
                        ops.add_rmsnorm(x, W["ln1"], a.rms_eps, h)
                    if self.mla:
                        att = self._prefill_attention_mla(l, W, S, s0, n, P, h)
                    else:
                        att = self._prefill_attention_gqa(l, W, S, s0, n, P, h)
                    torch.mm(att, W["wo"].t(), out=o)
                    ops.add_rmsnorm(x, W["ln2"], a.rms_eps, h, delta=o, x_out=x)
                    nxt = self.w.layers[l + 1]["ln1"] if l + 1 < a.layers else self.w.final_norm
                    seg = self._segment(t)
                    if self.mla and l < a.first_k_dense:  # DeepseekV2MLP of the dense first layers
                        self._dense_mlp(W["dense_gate_up"], W["dense_down"], h, S["de_h"][:t], o, seg)
                        ops.add_rmsnorm(x, nxt, a.rms_eps, h, delta=o, x_out=x)
                        continue
                    shared = None
                    if self.mla:  # shared experts on every token
                        self._dense_mlp(W["sh_gate_up"], W["sh_down"], h, S["sh_h"][:t], S["sh_out"][:t], seg)
                        shared = S["sh_out"][:t]
                    torch.mm(h, W["router"].t(), out_dtype=torch.float32, out=S["lg"][:t])
                    ops.router_topk(None, None, ws, k, a.router_mode, a.routed_scaling, a.n_group, a.topk_group,
                                    logits_in=S["lg"][:t])
                    ops.permute(h, ws, S["xp"])
                    self._ffn(W["w_gate_up"], W["w_down"], S["xp"], ws.offsets, S["hf"], S["yp"])
                    ops.unpermute_combine(S["yp"], ws, x, t, residual=x, shared_out=shared, norm_w=nxt,
                                          eps=a.rms_eps, norm_out=h)
                last = h.view(n, P, d)[:, P - 1].contiguous()
                logits = torch.mm(last, self.w.lm_head.t())
                b.logits[s0:s0 + n].copy_(logits)
                ops.argmax(logits, b.next_ids[s0:s0 + n])
            b.positions.fill_(P)
            b.seq_lens.fill_(P)
            b.step.fill_(P)
            self.out_tokens[:, P - 1].copy_(b.next_ids)
        torch.cuda.current_stream().wait_stream(self.stream)
        self.host_pos = P
        return b.next_ids.to("cpu", torch.int64)

    prefill_min_be = 256  # floor of the streamed prefill's expert scratch (rows)

    @torch.no_grad()
    def _prefill_streamed(self, input_ids: torch.Tensor, chunk_tokens: int) -> torch.Tensor:
        """Prefill with offloaded weights, module-based batching style: layer by
        layer over ALL prompt tokens, so every streamed weight crosses the host link once per layer.
        The layer's dense blob is copied into the dense buffer; attention runs in sequence chunks;
        the MoE routes all tokens at once and runs expert by expert, each uncached expert streamed
        into one of two slots on the H2D stream while the previous expert computes."""
        a, b, w = self.arch, self.buf, self.w
        B, P = input_ids.shape
        T = B * P
        d, k, f, E = a.hidden, a.top_k, a.moe_ffn, a.n_experts
        bf = dict(dtype=BF16, device=self.device)
        Bp = max(1, min(B, chunk_tokens // P))
        S = self._prefill_scratch(Bp * P)
        x_all, h_all = torch.empty(T, d, **bf), torch.empty(T, d, **bf)
        sh_all = torch.empty(T, d, **bf) if self.mla else None
        xp, yp = torch.empty(T * k, d, **bf), torch.empty(T * k, d, **bf)
        lg = torch.empty(T, E, dtype=torch.float32, device=self.device)
        ws = ops.RouterWorkspace(T, E, k, device=self.device)
        # expert activation scratch of b_e rows (the planner's memory model, memory_model.py): an expert
        # group larger than b_e is re-split into b_e-row launches (exec_sim.py:170-175), never overrun
        be = max(self.prefill_min_be, int(self.plan.b_e))
        hf = torch.empty(be, f, **bf)
        ids = input_ids.to(self.device, torch.int32)
        self.reset(0)
        st, cp = self.stream, self.h2d
        st.wait_stream(torch.cuda.current_stream())
        cp.wait_stream(torch.cuda.current_stream())
        # every uncached expert of every layer, in compute order, streamed through the expert slots: the
        # copy of the i-th one is issued as soon as the compute that last read its slot (i - nsl) has
        # been issued, so the link runs up to nsl experts ahead of the GEMMs -- across layer
        # boundaries, through the next layer's attention and the per-layer routing sync
        nsl = max(2, int(w.slots.shape[0]))
        stream_order = [(l, e) for l in range(a.layers) if self._has_router(l)
                        for e in range(w.place.experts_per_layer[l], E)]
        slot_free = [torch.cuda.Event() for _ in range(nsl)]
        landed = [torch.cuda.Event() for _ in range(nsl)]
        dense_landed, dense_free = torch.cuda.Event(), torch.cuda.Event()
        for ev in slot_free:
            ev.record(st)
        issued = [0]

        def issue_copies(upto: int) -> None:
            while issued[0] < min(upto, len(stream_order)):
                i = issued[0]
                l2, e2 = stream_order[i]
                sl = i % nsl
                cp.wait_event(slot_free[sl])  # recorded by the compute of stream_order[i - nsl]
                with torch.cuda.stream(cp):
                    if copy:
                        w.slots[sl].copy_(w.host_experts[l2][e2 - w.place.experts_per_layer[l2]], non_blocking=True)
                    landed[sl].record(cp)
                issued[0] += 1
        # copies_enabled / compute_enabled = False: the same prefill with its host->device copies or its
        # kernels skipped (the copies-only / compute-only times of the overlap measurement)
        run, copy = self.compute_enabled, self.copies_enabled

        def dense_copy(l: int) -> None:
            """Layer l's dense blob (attention + router + shared experts) into the dense buffer on the
            H2D stream, after the previous layer's last reader of the buffer (its router)."""
            if l >= a.layers or l < w.place.dense_layers:
                return
            cp.wait_event(dense_free)
            with torch.cuda.stream(cp):
                if copy:
                    w.dense_bufs[0].copy_(w.host_dense[l], non_blocking=True)
                dense_landed.record(cp)

        dense_free.record(st)
        dense_copy(0)
        issue_copies(nsl)
        computed = 0  # uncached experts whose GEMMs are issued
        with torch.cuda.stream(st):
            if run:
                ops.embed(ids.reshape(-1), w.embed, x_all)
            for l in range(a.layers):
                L = w.layers[l]
                W = dict(L)
                if l >= w.place.dense_layers:  # the layer's attention (+ shared experts) blob
                    st.wait_event(dense_landed)
                    W.update(w.dense_views(0))
                if l == 0 and run:
                    ops.add_rmsnorm(x_all, W["ln1"], a.rms_eps, h_all)
                nxt = w.layers[l + 1]["ln1"] if l + 1 < a.layers else w.final_norm
                dense_mlp = self.mla and l < a.first_k_dense
                for s0 in range(0, B, Bp):
                    if not run:
                        break
                    n = min(Bp, B - s0)
                    t0, t1 = s0 * P, (s0 + n) * P
                    x, h, o = x_all[t0:t1], h_all[t0:t1], S["o"][:t1 - t0]
                    att = (self._prefill_attention_mla if self.mla else self._prefill_attention_gqa)(
                        l, W, S, s0, n, P, h)
                    torch.mm(att, W["wo"].t(), out=o)
                    ops.add_rmsnorm(x, W["ln2"], a.rms_eps, h, delta=o, x_out=x)
                    t = t1 - t0
                    seg = self._segment(t)
                    if dense_mlp:
                        self._dense_mlp(W["dense_gate_up"], W["dense_down"], h, S["de_h"][:t], o, seg)
                        ops.add_rmsnorm(x, nxt, a.rms_eps, h, delta=o, x_out=x)
                    elif self.mla:
                        self._dense_mlp(W["sh_gate_up"], W["sh_down"], h, S["sh_h"][:t], sh_all[t0:t1], seg)
                if dense_mlp:
                    dense_free.record(st)
                    dense_copy(l + 1)
                    continue
                if run:
                    torch.mm(h_all, W["router"].t(), out_dtype=torch.float32, out=lg)
                    ops.router_topk(None, None, ws, k, a.router_mode, a.routed_scaling, a.n_group, a.topk_group,
                                    logits_in=lg)
                    ops.permute(h_all, ws, xp)
                dense_free.record(st)  # the layer's last reader of the dense buffer was the router
                # host sync once per layer: per-expert row counts (the capacity pre-flight; x_perm holds
                # all T*k rows by construction, the b_e scratch is handled by the re-split below)
                cnt = ops.check_capacity(ws.offsets, T * k)
                offs = [0]
                for c in cnt:
                    offs.append(offs[-1] + c)
                n_c = w.place.experts_per_layer[l]
                dense_copy(l + 1)  # the dense buffer is free again (the router was its last reader)
                for e in range(E):
                    r0, r1 = offs[e], offs[e + 1]
                    if e < n_c:
                        gu, dn = L["w_gate_up"][e:e + 1], L["w_down"][e:e + 1]
                    else:  # streamed: wait for its copy (issued up to nsl experts earlier)
                        assert stream_order[computed] == (l, e)
                        sl = computed % nsl
                        st.wait_event(landed[sl])
                        gu, dn = w.slot_views(sl)
                    for c0 in range(r0, r1, be) if run else ():  # b_e-row pieces of the expert's group
                        c1 = min(r1, c0 + be)
                        lo = self._segment(c1 - c0)
                        self._ffn(gu, dn, xp[c0:c1], lo, hf[:c1 - c0], yp[c0:c1])
                    if e >= n_c:
                        slot_free[computed % nsl].record(st)
                        computed += 1
                        issue_copies(computed + nsl)
                if run:
                    ops.unpermute_combine(yp, ws, x_all, T, residual=x_all, shared_out=sh_all, norm_w=nxt,
                                          eps=a.rms_eps, norm_out=h_all)
            if run:
                last = h_all.view(B, P, d)[:, P - 1].contiguous()
                torch.mm(last, w.lm_head.t(), out=b.logits)
                ops.argmax(b.logits, b.next_ids)
            b.positions.fill_(P)
            b.seq_lens.fill_(P)
            b.step.fill_(P)
            self.out_tokens[:, P - 1].copy_(b.next_ids)
        torch.cuda.current_stream().wait_stream(st)
        self.host_pos = P
        return b.next_ids.to("cpu", torch.int64)

    @torch.no_grad()
    def generate(self, input_ids: torch.Tensor, max_new_tokens: int, prefill: bool = True) -> torch.Tensor:
        """Greedy generation (HF generate semantics: no EOS stop, equal-length prompts).  The
        prompt is consumed through the same decode step, one position per step."""
        B, P = input_ids.shape
        assert B == self.B, f"engine was planned for B={self.B}"
        assert P + max_new_tokens <= self.max_ctx
        if prefill and self.can_prefill():
            self.prefill(input_ids)
        else:  # the prompt through the decode step, one position per step
            self.reset(0)
            prompt = input_ids.to(self.device, torch.int32)
            for p in range(P):
                self.buf.next_ids.copy_(prompt[:, p])
                self.run_step()
        # step P-1 predicted the first new token; it is already in next_ids
        for _ in range(max_new_tokens - 1):
            self.run_step()
        gen = self.out_tokens[:, P - 1:P - 1 + max_new_tokens].cpu()
        self.check_cpu_attention()
        return torch.cat([input_ids.cpu().to(torch.int64), gen], dim=1)

    def debug_forward(self, tokens: torch.Tensor, pos: int) -> dict:
        """One eager step at absolute position `pos` (all sequences), returning intermediate
        tensors of layer 0 and the logits (parity tests)."""
        self.buf.positions.fill_(pos)
        self.host_pos = pos + 1
        self.buf.next_ids.copy_(tokens.to(torch.int32))
        self.stream.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(self.stream):
            self._step(record=False)
        torch.cuda.current_stream().wait_stream(self.stream)
        torch.cuda.synchronize()
        return dict(logits=self.buf.logits.clone(), next_ids=self.buf.next_ids.clone())

    def trace_step(self) -> tuple[list[dict], dict]:
        """One eager decode step with timing events around every job on its own stream.
        Returns (records, report): records use the reference simulator's JSONL trace schema
        {time, node, kind, resource, action} (exec_sim.py:113-136) with measured times, and the
        report carries SimReport-style busy / idle / bytes / makespan (exec_sim.py:84-110) plus the
        transfer/compute overlap 1 - (makespan - max(busy)) / min(busy)."""
        self.trace_events = {}
        self._trace_counts = torch.zeros(self.arch.layers, self.arch.n_experts, dtype=torch.int32, device=self.device)
        torch.cuda.synchronize()
        torch.cuda.reset_peak_memory_stats(self.device)
        t0 = torch.cuda.Event(enable_timing=True)
        saved = [t.clone() for t in (self.buf.positions, self.buf.step, self.buf.next_ids, self.buf.seq_lens)]
        self.stream.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(self.stream):
            torch.cuda._sleep(int(5e7))  # host enqueues the whole step before the GPU starts
            t0.record(self.stream)
            self._step(record=False)
            t1 = torch.cuda.Event(enable_timing=True)
            t1.record(self.stream)
        torch.cuda.synchronize()
        self.check_cpu_attention()
        for t, s in zip((self.buf.positions, self.buf.step, self.buf.next_ids, self.buf.seq_lens), saved):
            t.copy_(s)
        jobs = self.schedule.jobs
        recs, busy = [], {}
        nbytes = {"htod_link": 0.0, "dtoh_link": 0.0}
        for jid, (e0, e1) in self.trace_events.items():
            j = jobs[jid]
            s, e = t0.elapsed_time(e0) * 1e-3, t0.elapsed_time(e1) * 1e-3
            recs.append({"time": s, "node": jid, "kind": j.kind, "resource": j.resource, "action": "start"})
            recs.append({"time": e, "node": jid, "kind": j.kind, "resource": j.resource, "action": "finish"})
            busy[j.resource] = busy.get(j.resource, 0.0) + (e - s)
            if j.resource in nbytes:
                nbytes[j.resource] += self._moved_bytes(j)
        self.trace_events = None
        peak = float(torch.cuda.max_memory_allocated(self.device))
        routed = self._trace_counts.cpu().tolist()
        self._trace_counts = None
        # layers without a router launch (DeepSeek's dense first layers) keep the schedule's counts
        sched = self.schedule_counts()
        expert_tokens = [routed[l] if self._has_router(l) else sched[l] for l in range(self.arch.layers)]
        recs.sort(key=lambda r: (r["time"], r["node"], r["action"] != "start"))
        makespan = t0.elapsed_time(t1) * 1e-3
        g, h = busy.get("gpu_compute", 0.0), busy.get("htod_link", 0.0)
        overlap = 1.0 - (makespan - max(g, h)) / min(g, h) if min(g, h) > 0 else None
        report = {"makespan": makespan, "busy": busy,
                  "idle_fraction": {r: 1.0 - v / makespan for r, v in busy.items()},
                  "bytes_htod": nbytes["htod_link"], "bytes_dtoh": nbytes["dtoh_link"],
                  "htod_gbs": nbytes["htod_link"] / h / 1e9 if h > 0 else None,
                  "throughput": self.B / makespan, "overlap": overlap,
                  # SimReport fields (exec_sim.py:97-110): measured allocator peak of the step (every
                  # HBM buffer the engine holds plus the step's transients), the routed rows per
                  # expert and layer, and whether the peak exceeded the device
                  "peak_gpu_bytes": peak, "oom_flag": peak > torch.cuda.get_device_properties(self.device).total_memory,
                  "expert_tokens": expert_tokens,
                  "mean_tokens_per_expert": sum(map(sum, expert_tokens)) / (len(expert_tokens) * self.arch.n_experts)}
        return recs, report

    def _has_router(self, l: int) -> bool:
        return not (self.mla and l < self.arch.first_k_dense)

    def schedule_counts(self) -> list[list[int]]:
        """Per-layer expert token counts the job list was built with (even split: the schedule's
        default, offload_dag.py:173-185)."""
        from .schedule import even_split

        return [even_split(self.B * self.arch.top_k, self.arch.n_experts) for _ in range(self.arch.layers)]

    def job_trace(self) -> list[dict]:
        """The issued job list (kinds/labels/shapes), in submission order."""
        return [dict(id=j.id, kind=j.kind, resource=j.resource, label=j.label, layer=j.layer, tokens=j.tokens,
                     seqs=j.seqs, nbytes=j.nbytes) for j in self.schedule.jobs]

    def plan_document(self) -> str:
        return json.dumps({"plan": self.plan.to_document(), "phase": "decode", "kv_policy": self.kv_policy},
                          sort_keys=True)
