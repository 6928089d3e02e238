"""Measured B200 latency tables for the planner (the paper's profiling step).

The reference prices every schedule job from per-module latency tables `(tokens, context) ->
seconds` (hw_profile.py:52-149, LatencyTable) and otherwise synthesizes them from a roofline
(hw_profile.py:260-354).  `profile_engine` measures them instead, on this engine's own kernels:
each module kind is issued exactly as the engine issues that job, for a token count of the grid,
on one decoder layer of the model, and timed with CUDA events (median of `reps` after warm-up).

    pre_attention             QKV projection(s) + RoPE + KV append (+ MLA absorption bmm)
    attention_mechanism_gpu   paged decode attention over `context` keys (ctx grid)
    post_attention            O projection + residual add + RMSNorm (+ DeepSeek shared experts)
    router                    gate logits GEMM + fused top-k/softmax/counts + stable permutation
    expert                    grouped gate/up+SiLU and down GEMMs of ONE expert with `tokens` rows
    attention_mechanism_cpu   (GQA models, `cpu_token_grid`) the host-core attention of the CPU share

The result is a profile document in the reference's schema (hw_profile.py:156-249, ingestible by
its `ingest_profile`), with the machine's capacities and measured link/HBM rates.

Peak memory per module ("latency and peak memory usage for each module ...
measured using the torch memory stats related APIs") rides in the same document under
`memory_tables` (`ingest_profile` reads only `hardware` and `latency_tables`, so the document stays
ingestible): entries `[tokens, context, bytes]` = the engine's own activation buffers that module
reads or writes for `tokens` rows (sizes taken from the allocated tensors) plus the transient peak
the torch allocator records across the job (`max_memory_allocated` above the pre-call level).
`activation_coefficients` fits the reference's three per-token memory-model coefficients
(model_catalog.py:82-84, memory_model.py:201-213) from those tables, so the planner's memory
constraint can run on measured rather than assumed activation sizes.
"""

from __future__ import annotations

import dataclasses
import json
import os
import statistics
from typing import Sequence

import torch

from . import _native as nat
from . import ops
from .configs import ModelArch, get_arch
from .planner import BatchingPlan, Hardware, LatencyCurve, ModelSpec, profile_document

BF16 = torch.bfloat16
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _time(fn, reps: int) -> float:
    for _ in range(2):
        fn()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e-3)
    return statistics.median(ts)


def _transient_peak(fn) -> int:
    """Bytes the torch allocator holds above its pre-call level at the peak of one call of fn."""
    torch.cuda.synchronize()
    base = torch.cuda.memory_allocated()
    torch.cuda.reset_peak_memory_stats()
    fn()
    torch.cuda.synchronize()
    return max(0, torch.cuda.max_memory_allocated() - base)


def _per_row(t: torch.Tensor, rows: int) -> int:
    return t.numel() * t.element_size() // rows


def module_row_bytes(eng) -> dict[str, int]:
    """Activation bytes per token row of each module kind: the engine buffers the module's job reads
    or writes (engine.py _issue_job / _ds_job), sized from the tensors the engine allocated.  The
    resident hidden state x is excluded (the reference charges it separately as hidden residency,
    memory_model.py:207); `expert` is per routed row (x_perm in, h_ffn, y_perm out)."""
    b, B = eng.buf, eng.B
    rw = eng.rws
    router = [b.h, eng.logits_r]
    per_tok = lambda ts: sum(_per_row(t, B) for t in ts)  # noqa: E731
    out = {"router": per_tok(router + [rw.topk_idx, rw.topk_w, rw.local_rank, rw.src_token, rw.dst_pos])
           + _per_row(b.x_perm, B)}
    if eng.mla:
        m = eng.mb
        pre = [b.h, m["q"], m["ckv"], m["q_nope"], m["q_pe"], m["q_lat"]] + [m[n] for n in ("q_a", "q_an") if n in m]
        out["pre_attention"] = per_tok(pre)
        out["attention_mechanism_gpu"] = per_tok([m["q_lat"], m["q_pe"], m["o_lat"]])
        out["post_attention"] = per_tok([m["o_lat"], m["o_cat"], b.o, b.h, m["sh_h"], m["sh_out"]])
    else:
        out["pre_attention"] = per_tok([b.h, b.qkv, b.q])
        out["attention_mechanism_gpu"] = per_tok([b.q, b.attn])
        out["post_attention"] = per_tok([b.attn, b.o, b.h])
    rows = b.x_perm.shape[0]
    out["expert"] = sum(_per_row(t, rows) for t in (b.x_perm, b.h_ffn, b.y_perm))
    return out


def activation_coefficients(doc: dict) -> dict[str, float]:
    """The reference memory model's per-token activation coefficients (ModelSpec fields,
    model_catalog.py:82-84; used by memory_model.intermediate_bytes) fitted to a profile's
    `memory_tables`: the attention coefficient is the largest per-token slope of the three attention
    modules (the reference charges the peak per-kernel activation), the context coefficient the
    attention module's slope over context per sequence, the expert coefficient the expert module's
    slope per routed row.  Merge the result into a model-spec document to plan on measured sizes."""
    tabs = {t["module_kind"]: t["entries"] for t in doc["memory_tables"]}

    def slope(entries, ctx=None):
        es = sorted((e for e in entries if ctx is None or e[1] == ctx), key=lambda e: e[0])
        (t0, _, b0), (t1, _, b1) = es[0], es[-1]
        return (b1 - b0) / (t1 - t0) if t1 > t0 else b1 / max(t1, 1)

    attn = tabs["attention_mechanism_gpu"]
    ctxs = sorted({e[1] for e in attn})
    per_tok = max(slope(tabs["pre_attention"]), slope(tabs["post_attention"]), slope(attn, ctxs[0]))
    Tmax = max(e[0] for e in attn)
    at_t = sorted((e for e in attn if e[0] == Tmax), key=lambda e: e[1])
    per_ctx = 0.0
    if len(at_t) > 1 and at_t[-1][1] > at_t[0][1]:
        per_ctx = max(0.0, (at_t[-1][2] - at_t[0][2]) / ((at_t[-1][1] - at_t[0][1]) * Tmax))
    return {"attn_activation_bytes_per_token": float(per_tok), "attn_activation_bytes_per_ctx_token": per_ctx,
            "expert_activation_bytes_per_token": float(slope(tabs["expert"]))}


def measure_links(nbytes: int = 1 << 30, reps: int = 5) -> tuple[float, float]:
    """Pinned host<->device copy rates (bytes/s), the PAPER.md:701 procedure."""
    h = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    d = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    up = nbytes / _time(lambda: d.copy_(h, non_blocking=True), reps)
    down = nbytes / _time(lambda: h.copy_(d, non_blocking=True), reps)
    return up, down


def measured_hardware(host_bytes: int | None = None) -> Hardware:
    up, down = measure_links()
    peaks = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            peaks = json.load(f)
    except OSError:
        pass
    if host_bytes is None:
        host_bytes = os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_PHYS_PAGES")
    return Hardware(m_g=torch.cuda.get_device_properties(0).total_memory, m_c=int(host_bytes), bw_htod=up,
                    bw_dtoh=down, gpu_peak_flops=float(peaks.get("bf16_tflops_sustained", 1388.0)) * 1e12,
                    gpu_mem_bw=float(peaks.get("hbm_gbs", 6550.0)) * 1e9, gpu_launch_overhead=5e-6,
                    cpu_attn_flops=0.0)


def _profile_cpu_attention(arch: ModelArch, token_grid: Sequence[int], ctx_grid: Sequence[int],
                           under_copy_load: bool = True):
    """ATTN_MECH_CPU on the host cores (csrc/cpu_attn.cpp) for T sequences over `ctx` keys; also the
    achieved attention FLOP/s (the reference's cpu_attn_flops, hw_profile.py:52-149).

    With `under_copy_load` the timing runs while the copy engine streams pinned host memory to the
    GPU back to back, as the KV_COPY_IN slices of the GPU share do during a step: the CPU share and
    the host link read the same host DRAM, and a table measured on an idle host overestimates the
    CPU share's speed (a 29 % optimistic plan estimate in profiles/r1_plan_mixtral8x7b_cpu.json)."""
    import ctypes
    import threading
    import time

    stop = threading.Event()
    loader = None
    if under_copy_load and torch.cuda.is_available():
        src = torch.empty(1 << 30, dtype=torch.uint8).pin_memory()
        dst = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
        side = torch.cuda.Stream()

        def load():
            with torch.cuda.stream(side):
                while not stop.is_set():
                    for _ in range(4):
                        dst.copy_(src, non_blocking=True)
                    side.synchronize()

        loader = threading.Thread(target=load, daemon=True)
        loader.start()
        time.sleep(0.2)

    a, P = arch, ops.kv_page_size()
    Tm, cm = max(token_grid), max(ctx_grid)
    pps = (cm + P - 1) // P
    blk = a.n_kv_heads * a.head_dim * P
    k = torch.zeros(Tm * pps * blk, dtype=BF16)
    v = torch.zeros(Tm * pps * blk, dtype=BF16)
    q = torch.zeros(Tm, a.n_heads * a.head_dim, dtype=BF16)
    out = torch.empty_like(q)
    rows, rate = [], 0.0
    for T in token_grid:
        for ctx in ctx_grid:
            lens = torch.full((T,), ctx, dtype=torch.int32)
            d = nat.CpuAttnGqa(k.data_ptr(), v.data_ptr(), q.data_ptr(), lens.data_ptr(), out.data_ptr(), 0, pps, T,
                               a.n_heads, a.n_kv_heads, a.head_dim, P, 1.0, 0)
            nat.call("mgb_cpu_attn_gqa", ctypes.byref(d))
            ts = []
            for _ in range(3):
                t0 = time.perf_counter()
                nat.call("mgb_cpu_attn_gqa", ctypes.byref(d))
                ts.append(time.perf_counter() - t0)
            sec = statistics.median(ts)
            rows.append([T, ctx, sec])
            rate = max(rate, T * ctx * 4 * a.n_heads * a.head_dim / sec)
    stop.set()
    if loader is not None:
        loader.join()
    return rows, rate


def profile_engine(arch: ModelArch | str, token_grid: Sequence[int] | None = None,
                   ctx_grid: Sequence[int] = (128, 512, 768), reps: int = 5,
                   hardware: Hardware | None = None, cpu_token_grid: Sequence[int] = ()) -> dict:
    """Profile document with measured tables for every GPU module kind of `arch` (one decoder
    layer of it is instantiated; the latency of a job does not depend on the layer index)."""
    from .engine import Engine

    full = get_arch(arch) if isinstance(arch, str) else arch
    first_moe = full.first_k_dense if full.is_mla else 0
    one = dataclasses.replace(full, layers=first_moe + 1, name=f"{full.name}[profile]")
    token_grid = list(token_grid or [2 ** i for i in range(0, 14)])
    Tmax = max(token_grid)
    ctx_max = max(ctx_grid)
    spec = ModelSpec.from_document(one.model_spec_document())
    plan = BatchingPlan(Tmax, Tmax, 1 << 20, 0.0, 0, spec.model_bytes)
    eng = Engine(one, plan, prompt_len=max(1, ctx_max - 1), decode_len=1, use_graph=False)
    eng.fused_rope = False  # pre_attention's RoPE/append and the attention are timed as separate modules
    eng.synthetic_prefill()
    a, b, l = eng.arch, eng.buf, first_moe
    W = eng._layer_weights(l)
    d = a.hidden
    b.h.normal_(0.0, 1.0)
    b.positions.fill_(ctx_max - 1)
    g = torch.Generator(device="cuda").manual_seed(0)
    tables: dict[str, list] = {k: [] for k in ("pre_attention", "attention_mechanism_gpu", "post_attention",
                                               "router", "expert")}
    mem: dict[str, list] = {k: [] for k in tables}
    row_bytes = module_row_bytes(eng)
    from .schedule import Job

    def timed(kind: str, T: int, fn, ctx: int = 0) -> None:
        tables[kind].append([T, ctx, _time(fn, reps)])
        mem[kind].append([T, ctx, T * row_bytes[kind] + _transient_peak(fn)])

    def job(kind: str, T: int):
        return Job(0, kind, "gpu_compute", 0.0, f"L{l}/{kind}/mb0", layer=l, tokens=T, seqs=T)

    for T in token_grid:
        # pre-attention: exactly the engine's job on micro-batch [0, T)
        timed("pre_attention", T, lambda: eng._issue_job(l, job("pre_attention", T)))
        # post-attention on T tokens (O projection + residual/norm [+ shared experts])
        if eng.mla:
            m = eng.mb

            def post():
                torch.mm(m["o_cat"][:T], W["wo"].t(), out=b.o[:T])
                ops.add_rmsnorm(b.x[:T], W["ln2"], a.rms_eps, b.h[:T], delta=b.o[:T], x_out=b.x[:T])
                eng._dense_mlp(W["sh_gate_up"], W["sh_down"], b.h[:T], m["sh_h"][:T], m["sh_out"][:T], eng._segment(T))
        else:
            def post():
                torch.mm(b.attn[:T], W["wo"].t(), out=b.o[:T])
                ops.add_rmsnorm(b.x[:T], W["ln2"], a.rms_eps, b.h[:T], delta=b.o[:T], x_out=b.x[:T])
        timed("post_attention", T, post)
        # router on T tokens: logits GEMM + fused top-k + stable permutation
        ws = ops.RouterWorkspace(T, a.n_experts, a.top_k)
        logits = torch.empty(T, a.n_experts, dtype=torch.float32, device="cuda")
        xp = torch.empty(T * a.top_k, d, dtype=BF16, device="cuda")

        def route():
            logits.copy_(torch.mm(b.h[:T], W["router"].t(), out_dtype=torch.float32))
            ops.router_topk(None, None, ws, a.top_k, a.router_mode, a.routed_scaling, a.n_group, a.topk_group,
                            logits_in=logits)
            ops.permute(b.h[:T], ws, xp)
        timed("router", T, route)
        # one expert with T rows (the EXPERT_COMPUTE chunk): gate/up+SiLU then down
        rows = max(T, 1)
        x = torch.randn(rows, d, generator=g, device="cuda").to(BF16)
        h = torch.empty(rows, a.moe_ffn, dtype=BF16, device="cuda")
        y = torch.empty(rows, d, dtype=BF16, device="cuda")
        offs = torch.tensor([0, T], dtype=torch.int32, device="cuda")
        gu, dn = W["w_gate_up"][:1], W["w_down"][:1]

        def expert():
            ops.moe_gemm_gate_up(gu, x, offs, h)
            ops.moe_gemm_down(dn, h, offs, y)
        timed("expert", T, expert)
        # attention over `ctx` keys for T sequences
        for ctx in ctx_grid:
            b.seq_lens[:T].fill_(ctx)
            if eng.mla:
                _, q_lat, o_lat, _ = eng._ds_views(0, T)
                scale = (a.qk_nope_dim + a.qk_rope_dim) ** -0.5

                def attn():
                    nat.call("mgb_decode_attn_mla", q_lat.data_ptr(), eng.mb["q_pe"][:T].data_ptr(),
                             eng.latent[l].data_ptr(), eng.block_table.data_ptr(), eng.pps, b.seq_lens.data_ptr(),
                             T, a.n_heads, a.kv_lora_rank, a.qk_rope_dim, scale, o_lat.data_ptr(),
                             torch.cuda.current_stream().cuda_stream)
            else:
                def attn():
                    ops.decode_attn_gqa(b.q[:T], eng.k_cache[l], eng.v_cache[l], eng.block_table[:T],
                                        b.seq_lens[:T], a.n_heads, a.n_kv_heads, a.head_dim, b.attn[:T])
            timed("attention_mechanism_gpu", T, attn, ctx)
    del eng
    torch.cuda.empty_cache()
    cpu_rate = 0.0
    if not full.is_mla and cpu_token_grid:
        tables["attention_mechanism_cpu"], cpu_rate = _profile_cpu_attention(one, cpu_token_grid, ctx_grid)
    # the reference requires tables monotone in tokens (hw_profile.py:117-142): running max per context
    for k, v in tables.items():
        best: dict[int, float] = {}
        for e in sorted(v, key=lambda e: (e[1], e[0])):
            e[2] = best[e[1]] = max(e[2], best.get(e[1], 0.0))
    curves = [LatencyCurve(k, [tuple(e) for e in v]) for k, v in tables.items()]
    hw = hardware or measured_hardware()
    if cpu_rate > 0:
        hw = Hardware(**{**hw.__dict__, "cpu_attn_flops": cpu_rate})
    doc = profile_document(hw, curves)
    doc["memory_tables"] = [{"module_kind": k, "entries": v} for k, v in mem.items()]
    doc["activation_coefficients"] = activation_coefficients(doc)
    return doc
