#!/usr/bin/env python
"""Decode throughput of the B200 MoE-Gen engine (BASELINE.json metric: decode tokens/sec at
prompt 512 / gen 256; expert GEMM tensor-pipe utilisation) on the Mixtral-8x7B shape, 1 B200
resident (BASELINE.json configs[1]).

  python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference] [--batch B]

A step = one full decode phase of one batch: B sequences x 256 greedy decode forwards at
positions 512..767 (the reference's accounting: B tokens per decode forward,
plan_search.py:62-65), replayed as CUDA graphs.  Prefill is excluded from the metric; its KV state
is synthetic (counter-based values in every page).  Weights are random-init (counter-based, in
HBM).  Under torchrun each rank runs an independent replica (Mixtral-8x7B fits one GPU:
"replicas only"); value = all ranks' tokens / max-over-ranks time.

--impl reference times the CPU restatement of the same path (oracle/, the reference ships no
numeric implementation) on the host cores: one Mixtral-8x7B decoder layer decode step of B
sequences at mid-decode context, scaled by the layer count.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import torch

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "decode tokens/sec at prompt 512/gen 256"
UNIT = "tokens/s"
# HBM the planner keeps free beside weights + paged KV when sizing the resident batch: the engine's
# measured non-weight, non-KV peak (tools/mem_probe.py, profiles/r2_mem_probe.json: step buffers,
# graph pool, cuBLAS workspaces, the batched-prefill buffers, CUDA context) plus a 2 GB margin.
# Mixtral-8x7B holds 4.2 GB there; DeepSeek-V2-Lite 10.7 GB (B x 102400 logits, MLA scratch) keeps
# the round-1 14 GB.
RESERVE_GB = {"mixtral-8x7b": 6.25}


def reserve_bytes(args, arch) -> int:
    gb = args.reserve_gb if args.reserve_gb is not None else RESERVE_GB.get(arch.name, 14.0)
    return int(gb * 2**30)


def _ncu_traffic(config: str, gemm: str):
    """DRAM bytes (read + write) per launch of the dominant kernel from the committed ncu --set full
    capture (profiles/ncu_traffic.json, written by tools/ncu_traffic.py), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            rows = json.load(f)
        r = rows[config][gemm]
        return r["dram_bytes"], r["source"]
    except Exception:
        return None, None


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), float(p["bf16_tflops"]), float(p.get("bf16_tflops_sustained", p["bf16_tflops"])), "measured"
    except Exception:
        return 6650.0, 1590.0, 1400.0, "fallback"


class ClockSampler:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows: list[list[str]] = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                for line in out.stdout.strip().splitlines():
                    self.rows.append([c.strip() for c in line.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self) -> dict:
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in self.rows for n, v in zip(names, r[5:9]) if v.strip().lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    if ws > 1:
        import torch.distributed as dist

        backend = "nccl" if torch.cuda.is_available() else "gloo"
        if torch.cuda.is_available():  # bind the rank's GPU before NCCL's communicator is built
            torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")) % torch.cuda.device_count())
        dist.init_process_group(backend)
        return dist, dist.get_rank(), ws, int(os.environ.get("LOCAL_RANK", "0"))
    return None, 0, 1, 0


def _max_over_ranks(dist, v: float) -> float:
    if dist is None:
        return v
    t = torch.tensor([v], dtype=torch.float64, device="cuda" if torch.cuda.is_available() else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ------------------------------------------------------------------------------------------
# CPU arm (oracle port): one decoder layer decode step of B sequences, x L layers
# ------------------------------------------------------------------------------------------
def cpu_layer_sample(arch, B: int, ctx: int, reps: int, threads: int) -> tuple[float, str]:
    """The oracle port (oracle/moe_ref.py) timed on the host: one MoE decoder layer of B sequences
    at context `ctx`, scaled by the layer count (a full 93-471 GB model is impractical on CPU)."""
    from oracle import moe_ref as R

    torch.set_num_threads(threads)
    a = arch
    d = a.hidden
    g = torch.Generator().manual_seed(0)
    bf = torch.bfloat16

    def U(*shape, std=0.02):
        return (torch.rand(*shape, generator=g) * 2 - 1).mul_(std * math.sqrt(3)).to(bf)

    class _W:
        layers = []
    if a.family == "deepseek_v2":
        H, qk = a.n_heads, a.qk_nope_dim + a.qk_rope_dim
        fs = a.moe_ffn * a.n_shared
        W = dict(ln1=torch.ones(d, dtype=bf), ln2=torch.ones(d, dtype=bf),
                 kv_a=U(a.kv_lora_rank + a.qk_rope_dim, d), kv_a_norm=torch.ones(a.kv_lora_rank, dtype=bf),
                 kv_b=U(H * (a.qk_nope_dim + a.v_head_dim), a.kv_lora_rank), wo=U(d, H * a.v_head_dim),
                 router=U(a.n_experts, d), w_gate_up=U(a.n_experts, 2 * a.moe_ffn, d),
                 w_down=U(a.n_experts, d, a.moe_ffn), sh_gate_up=U(2 * fs, d), sh_down=U(d, fs))
        if a.q_lora_rank:
            W.update(q_a=U(a.q_lora_rank, d), q_a_norm=torch.ones(a.q_lora_rank, dtype=bf), q_b=U(H * qk, a.q_lora_rank))
        else:
            W["q_proj"] = U(H * qk, d)
        _W.layers = [None] * a.first_k_dense + [W]
        orc = R.DeepseekV2Oracle.__new__(R.DeepseekV2Oracle)
        orc.a, orc.w = a, _W()
        li = a.first_k_dense
        kc = U(B, H, ctx - 1, qk, std=1.0)
        vc = U(B, H, ctx - 1, a.v_head_dim, std=1.0)
        caches = lambda: ([None] * li + [kc], [None] * li + [vc])  # noqa: E731
        name = "DeepseekV2Oracle.layer_forward"
    else:
        hd = a.head_dim
        W = dict(ln1=torch.ones(d, dtype=bf), wq=U(a.n_heads * hd, d), wk=U(a.n_kv_heads * hd, d),
                 wv=U(a.n_kv_heads * hd, d), wo=U(d, a.n_heads * hd), ln2=torch.ones(d, dtype=bf),
                 router=U(a.n_experts, d), w_gate_up=U(a.n_experts, 2 * a.moe_ffn, d),
                 w_down=U(a.n_experts, d, a.moe_ffn))
        _W.layers = [W]
        orc = R.MixtralOracle.__new__(R.MixtralOracle)
        orc.a, orc.w = a, _W()
        li = 0
        kc = U(B, a.n_kv_heads, ctx - 1, hd, std=1.0)
        vc = U(B, a.n_kv_heads, ctx - 1, hd, std=1.0)
        caches = lambda: ([kc], [vc])  # noqa: E731
        name = "MixtralOracle.layer_forward"
    x = U(B, d, std=1.0)
    times = []
    for r in range(reps + 1):
        if a.family == "deepseek_v2":
            orc.kc, orc.vc = caches()
        else:
            orc.k_cache, orc.v_cache = caches()
        t0 = time.perf_counter()
        orc.layer_forward(li, x, ctx - 1)
        times.append(time.perf_counter() - t0)
    t_layer = statistics.median(times[1:])
    sample = (f"oracle/moe_ref.py {name}: one {a.name} MoE decoder layer, B={B} sequences (the run's batch), "
              f"context {ctx}, bf16 torch-CPU on {threads} threads of {_cpu_model()}, median of {reps}; "
              f"tokens/s = B / (t_layer x {a.layers} layers)")
    return B / (t_layer * a.layers), sample


def _cpu_model() -> str:
    """Host CPU model and the matrix/vector extensions torch's CPU kernels can use."""
    name, flags = "unknown CPU", set()
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name") and name == "unknown CPU":
                    name = line.split(":", 1)[1].strip()
                elif line.startswith("flags") and not flags:
                    flags = set(line.split(":", 1)[1].split())
    except OSError:
        pass
    ext = [x for x in ("avx512f", "avx512_bf16", "amx_bf16") if x in flags]
    return f"{name} ({', '.join(ext) or 'no AVX-512'})"


_BASELINE_CFG = {"mixtral-8x7b": "BASELINE configs[1]", "deepseek-v2-lite": "BASELINE configs[2], 1 GPU",
                 "tiny-mixtral": "BASELINE configs[0] model", "mixtral-8x22b": "BASELINE configs[3] model",
                 "deepseek-v2-236b": "BASELINE configs[4] model"}


def _workload_config(args, arch, world: int, ep: bool = False) -> dict:
    """The workload both arms are quoted on (the GPU arm's batch: the planner's largest resident B)."""
    from paper_2503_09716_b200.engine import resident_plan

    plan = resident_plan(arch, args.prompt_len, args.decode_len, B=args.batch, reserve_bytes=reserve_bytes(args, arch),
                         ep_world=world if ep else 1)
    where = (f"{world} B200 expert-parallel" if ep else "1 B200 resident")
    par = (f"ep{world}: experts {arch.n_experts // world} per rank, each rank's B sequences data-parallel, token "
           f"dispatch/combine fused into the permutation / down-GEMM kernels over NVLink peer memory (torch symmetric "
           f"memory), per-expert counts all-gathered over NCCL" if ep else f"replicas x{world}")
    return {"workload": f"{arch.name} decode phase, prompt {args.prompt_len} / gen {args.decode_len}, {where} "
                        f"({_BASELINE_CFG.get(arch.name, 'not a BASELINE config')});"
                        f" step = {args.decode_len} decode forwards of B={plan.B} sequences per GPU",
            "batch": plan.B, "b_a": plan.b_a, "b_e": plan.b_e, "kv_policy": "resident (paged, HBM)",
            "hbm_reserve_gb": reserve_bytes(args, arch) / 2**30,
            "parallelism": par, "l2": "inputs larger than L2 (all weights stream from HBM every forward)"}


def run_reference(args, dist, rank, world) -> None:
    from paper_2503_09716_b200.configs import get_arch

    if rank != 0:
        return
    arch = get_arch(args.config)
    threads = os.cpu_count() or 1
    cfg = _workload_config(args, arch, world)
    B = args.cpu_batch or cfg["batch"]  # the GPU arm's batch (one layer at the run's B)
    ctx = args.prompt_len + args.decode_len // 2
    vals = []
    sample = ""
    for _ in range(args.warmup):
        cpu_layer_sample(arch, B, ctx, 1, threads)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        v, sample = cpu_layer_sample(arch, B, ctx, 1, threads)
        vals.append(v)
    wall = time.perf_counter() - t0
    value = statistics.median(vals)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * wall / max(1, args.steps),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic", "config": cfg,
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port", "sample": sample,
                             "cpu_model": _cpu_model(), "batch": B},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------------------
# GPU arm
# ------------------------------------------------------------------------------------------
def kernel_breakdown(eng, reps: int = 2) -> dict:
    """Eager pass with CUDA events around every launch of one decode step on the engine stream
    (the stream the graph replays on): every libmgb entry point (by C-ABI name) and every cuBLAS
    call.  The stream is parked first so the host enqueues the whole step before the GPU starts;
    event gaps then time kernels, not Python launch latency."""
    from paper_2503_09716_b200 import _native as nat

    st = eng.stream
    pend: list[tuple[str, torch.cuda.Event, torch.cuda.Event]] = []

    def timed(name, fn):
        def inner(*a, **k):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            r = fn(*a, **k)
            e1.record(st)
            pend.append((name if isinstance(name, str) else name(a), e0, e1))
            return r
        return inner

    orig_call, mm, bmm = nat.call, torch.mm, torch.bmm
    try:
        # grouped GEMM launches are keyed by expert count (routed E vs shared / dense E = 1)
        nat.call = timed(lambda a: f"{a[0]}[E={a[5]}]" if a[0] == "mgb_moe_ffn" else
                         f"{a[0]}[E={a[4]}]" if a[0].startswith("mgb_moe_gemm") else a[0], orig_call)
        torch.mm = timed("cublas_gemm", mm)
        torch.bmm = timed("cublas_bmm", bmm)
        eng.serial_jobs = True  # one stream: concurrent side-stream kernels would blur the attribution
        saved = [t.clone() for t in (eng.buf.positions, eng.buf.step, eng.buf.next_ids, eng.buf.seq_lens)]
        for _ in range(reps):
            with torch.cuda.stream(st):
                torch.cuda._sleep(int(2e8))
                eng._step(record=False)
            torch.cuda.synchronize()
        for t, s in zip((eng.buf.positions, eng.buf.step, eng.buf.next_ids, eng.buf.seq_lens), saved):
            t.copy_(s)
    finally:
        nat.call, torch.mm, torch.bmm = orig_call, mm, bmm
        eng.serial_jobs = False
    recs: dict[str, list[float]] = {}
    for name, e0, e1 in pend:
        recs.setdefault(name.replace("mgb_", ""), []).append(e0.elapsed_time(e1))
    return {n: {"avg_ms": sum(v) / len(v), "per_step": len(v) // reps, "ms_per_step": sum(v) / reps}
            for n, v in recs.items()}


def use_ep(args, arch, world: int) -> bool:
    """Experts shard across the job's ranks for DeepSeek-V2 models (configs[2], [4]) and
    for any model whose weights do not fit one GPU (Mixtral-8x22B EP8, configs[3]); Mixtral-8x7B runs
    replicas.  --ep force: the EP path on a one-rank group; --ep off: never."""
    from paper_2503_09716_b200.engine import b200_hardware
    from paper_2503_09716_b200.planner import ModelSpec

    if args.ep == "off" or (world == 1 and args.ep != "force"):
        return False
    if arch.family == "deepseek_v2" or args.ep == "force":
        return True
    hbm = b200_hardware().m_g if torch.cuda.is_available() else 183_359 << 20
    return ModelSpec.from_document(arch.model_spec_document()).model_bytes > hbm - reserve_bytes(args, arch)


def run_ours(args, dist, rank, world) -> None:
    import gc

    from paper_2503_09716_b200.configs import get_arch

    torch.cuda.set_device(rank % torch.cuda.device_count())
    arch0 = get_arch(args.config)
    ep0 = use_ep(args, arch0, world)
    line = measure(args, arch0, dist, rank, world, args.steps, args.warmup, main=True, ep=ep0)
    # the other 1-GPU BASELINE configuration (configs[2], DeepSeek-V2-Lite) measured in the same run, so
    # the driver's bench records it too; same contract (device-timed decode steps, e2e through the
    # public API, roofline of the dominant GEMM), fewer steps
    extra = {}
    for name in [c for c in args.also.split(",") if c and c != args.config]:
        gc.collect()
        torch.cuda.empty_cache()
        # DeepSeek-V2-Lite is BASELINE configs[2]: expert-parallel across the job's GPUs (1 GPU: plain)
        ep = use_ep(args, get_arch(name), world)
        try:
            sub = measure(args, get_arch(name), dist, rank, world, args.also_steps, max(3, min(args.warmup, 3)),
                          main=False, ep=ep)
        except Exception as e:  # noqa: BLE001 -- report it in the line instead of losing the main result
            extra[name] = {"error": f"{type(e).__name__}: {str(e).splitlines()[0] if str(e) else ''}"[:300]}
            continue
        extra[name] = {k: sub[k] for k in ("value", "unit", "ms_per_step", "steps", "warmup", "forward_ms", "config", "graph",
                                           "e2e", "roofline", "expert_gemm", "incl_prefill", "kernel_hbm",
                                           "kernel_ms_per_forward", "clocks", "gpu_launches", "dtype")}
    if extra:
        line["also"] = extra
    if rank == 0:
        print(json.dumps(line), flush=True)


def measure(args, arch, dist, rank, world, steps: int, warmup: int, main: bool, ep: bool = False) -> dict:
    """Time one configuration (the bench contract: `warmup` untimed steps, then exactly `steps`
    device-timed decode phases, max over ranks); returns its JSON line.  ep: experts sharded over the
    job's ranks (PeerExpertParallel over symmetric memory), each rank decoding its own B sequences."""
    from paper_2503_09716_b200.engine import Engine, resident_plan

    plan = resident_plan(arch, args.prompt_len, args.decode_len, B=args.batch, reserve_bytes=reserve_bytes(args, arch),
                         ep_world=world if ep else 1)
    pep = None
    if ep:
        from paper_2503_09716_b200.ep import PeerExpertParallel

        rows = plan.B * arch.top_k  # this rank's routed rows; a receive buffer holds every source's worst case
        pep = PeerExpertParallel.from_symmetric_memory(arch.n_experts, dist.group.WORLD, world * rows, rows,
                                                       arch.hidden)
    eng = Engine(arch, plan, prompt_len=args.prompt_len, decode_len=args.decode_len, seed=0,
                 use_graph=True, ep=pep)
    B = eng.B
    N = args.decode_len
    eng.synthetic_prefill(seed=1)
    first = torch.randint(0, arch.vocab, (B,), generator=torch.Generator().manual_seed(7))
    first_pinned = first.to(torch.int32).pin_memory()
    eng.capture()

    def one_step():
        eng.reset(args.prompt_len)
        eng.buf.next_ids.copy_(first_pinned, non_blocking=True)
        for _ in range(N):
            eng.run_step()  # graph replay (host position checked against the planned context)

    for _ in range(warmup):
        one_step()
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(torch.cuda.current_device()) as clk:
        torch.cuda.synchronize()
        e0.record()
        for _ in range(steps):
            one_step()
        e1.record()
        torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    t = _max_over_ranks(dist, e0.elapsed_time(e1) / 1e3)
    tokens = B * N * steps * world
    value = tokens / t

    # ---- end-to-end through the public API (host tokens in, host tokens out) ----
    e2e_times = []
    for _ in range(args.e2e_steps):
        eng.reset(args.prompt_len)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        out = eng.decode(first_pinned, N)
        torch.cuda.synchronize()
        e2e_times.append(time.perf_counter() - t0)
    t_e2e = _max_over_ranks(dist, statistics.median(e2e_times))
    e2e_value = B * N * world / t_e2e

    # ---- the same decode step behind a real batched prefill of the B prompts (SURVEY.md §8d asks for
    # the incl.-prefill figure too): B x prompt_len tokens through Engine.prefill, device-timed ----
    incl = None
    if args.incl_prefill and eng.can_prefill():
        try:
            ids = torch.randint(0, arch.vocab, (B, args.prompt_len), generator=torch.Generator().manual_seed(11))
            torch.cuda.synchronize()
            p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            p0.record()
            eng.prefill(ids)
            p1.record()
            torch.cuda.synchronize()
            t_pf = _max_over_ranks(dist, p0.elapsed_time(p1) / 1e3)
            t_dec = t / steps
            incl = {"value": B * N * world / (t_pf + t_dec), "unit": UNIT, "prefill_ms": 1e3 * t_pf,
                    "decode_ms": 1e3 * t_dec, "prefill_tokens_per_s": B * args.prompt_len * world / t_pf,
                    "convention": f"B*{N} generated tokens / (batched prefill of B x {args.prompt_len} prompt tokens"
                                  f" + {N} decode forwards); the first generated token comes from the prefill"}
        except torch.OutOfMemoryError as e:  # report, do not lose the line
            incl = {"value": None, "unit": UNIT, "error": f"prefill out of memory: {str(e).splitlines()[0]}"}
            torch.cuda.empty_cache()

    # ---- per-kernel breakdown and roofline of the dominant kernel ----
    eng.reset(args.prompt_len + args.decode_len // 2)
    bd = kernel_breakdown(eng)
    hbm, tf_burst, tf_sust, src = _peaks()
    a = arch
    rows = B * a.top_k
    e_launch = arch.n_experts // world if ep else arch.n_experts  # experts per routed grouped launch
    k_active = e_launch  # every (local) expert is hit at these batch sizes
    nan = {"avg_ms": float("nan"), "ms_per_step": float("nan")}
    gu_bytes = k_active * 2 * a.moe_ffn * a.hidden * 2 + rows * a.hidden * 2 + rows * a.moe_ffn * 2
    dn_bytes = k_active * a.hidden * a.moe_ffn * 2 + rows * a.moe_ffn * 2 + rows * a.hidden * 2
    gu_flops = 2.0 * rows * a.hidden * 2 * a.moe_ffn
    dn_flops = 2.0 * rows * a.hidden * a.moe_ffn
    step_ms_eager = sum(v["ms_per_step"] for v in bd.values())
    tok_per_expert = rows / a.n_experts
    ridge = tf_burst * 1e12 / (hbm * 1e9)  # flop/B; expert GEMM intensity = tokens/expert flop/B
    ffn = bd.get(f"moe_ffn[E={e_launch}]")  # the fused launch (gate/up + SiLU*up + down), routed experts
    if ffn is not None:
        kname, kbytes, kflops, kr = ("mgb_moe_ffn (one tcgen05 CTA-pair launch: grouped gate/up + SiLU*up + down)",
                                     gu_bytes + dn_bytes, gu_flops + dn_flops, ffn)
        ffn_ms, gu_ms, dn_ms = ffn["avg_ms"], None, None
        traffic_key = "ffn"
    else:  # separate launches (EP path, MGB_FFN_FUSED=0)
        gu = bd.get(f"moe_gemm_gate_up[E={e_launch}]", nan)
        dn = bd.get(f"moe_gemm_down[E={e_launch}]", bd.get(f"moe_gemm_down_ep[E={e_launch}]", nan))
        kname, kbytes, kflops, kr = "mgb_moe_gemm_gate_up (tcgen05 grouped GEMM + SiLU*up)", gu_bytes, gu_flops, gu
        ffn_ms, gu_ms, dn_ms = gu["avg_ms"] + dn["avg_ms"], gu["avg_ms"], dn["avg_ms"]
        traffic_key = "gate_up"
    expert_tflops = (gu_flops + dn_flops) / (ffn_ms * 1e-3) / 1e12
    k_gbs = kbytes / (kr["avg_ms"] * 1e-3) / 1e9
    if tok_per_expert < ridge:
        roofline = {"kernel": kname, "bound": "hbm", "achieved": k_gbs, "peak": hbm, "unit": "GB/s", "frac": k_gbs / hbm}
    else:
        k_tf = kflops / (kr["avg_ms"] * 1e-3) / 1e12
        roofline = {"kernel": kname, "bound": "tensor", "achieved": k_tf, "peak": tf_burst, "unit": "TFLOP/s",
                    "frac": k_tf / tf_burst}
    traffic, traffic_src = _ncu_traffic(arch.name, traffic_key)
    roofline.update({"traffic": traffic, "traffic_source": traffic_src, "algorithmic_bytes_per_launch": kbytes,
                     "algorithmic_flops_per_launch": kflops, "avg_launch_ms": kr["avg_ms"], "peak_source": src,
                     "tokens_per_expert": tok_per_expert, "share_of_step": kr["ms_per_step"] / step_ms_eager})
    # achieved HBM bandwidth of the HBM-bound kernels (SURVEY.md §8d per-kernel algorithmic bytes;
    # attention at the breakdown's context, prompt_len + decode_len / 2 + 1)
    T, d, k, E = B, a.hidden, a.top_k, a.n_experts
    ctx_bd = args.prompt_len + args.decode_len // 2 + 1
    if a.family == "deepseek_v2":
        attn_name, attn_bytes = "decode_attn_mla", B * ctx_bd * (a.kv_lora_rank + a.qk_rope_dim) * 2
    else:
        attn_name = "decode_attn_gqa_sched" if "decode_attn_gqa_sched" in bd else "decode_attn_gqa"
        attn_bytes = B * ctx_bd * a.n_kv_heads * a.head_dim * 2 * 2
    shared = 2 if a.family == "deepseek_v2" else 0  # shared-expert rows read by the combine
    algo = {"router_topk": T * E * 4 + T * k * 12, "permute": T * d * 2 + T * k * d * 2,
            "unpermute_combine": T * k * d * 2 + T * d * 2 * (3 + (1 if shared else 0)), attn_name: attn_bytes,
            # fused residual add + RMSNorm + router + top-k + permute (route.cu): x and the attention
            # delta in, x_out and h out, router and norm weights, the k permuted copies of h, routing
            # records (topk idx/weight, dst_pos, src_token)
            "moe_route": T * d * 2 * 4 + (E + 1) * d * 2 + T * k * d * 2 + T * k * 16}
    kernel_hbm = {}
    for name, nbytes in algo.items():
        if name in bd:
            gbs = nbytes / (bd[name]["avg_ms"] * 1e-3) / 1e9
            kernel_hbm[name] = {"algorithmic_bytes": nbytes, "avg_ms": bd[name]["avg_ms"], "gbs": gbs, "frac": gbs / hbm}
    launches_per_step = eng.kernel_launches_per_step * N
    ctx_avg = args.prompt_len + args.decode_len / 2

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": steps, "warmup": warmup,
        "ms_per_step": 1e3 * t / steps, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "bf16", "data": "synthetic (random-init counter-based weights, synthetic prefill KV)",
        "config": _workload_config(args, arch, world, ep=ep),
        "graph": bool(eng.graph is not None),
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(first_pinned.numel() * 4),
                "d2h_bytes_per_step": int(out.numel() * out.element_size())},
        "roofline": roofline,
        "expert_gemm": {"tflops": expert_tflops, "tensor_util_of_bf16_peak": expert_tflops / tf_burst,
                        "tokens_per_expert": rows / a.n_experts, "ffn_ms": ffn_ms, "gate_up_ms": gu_ms, "down_ms": dn_ms,
                        "ffn_gbs": (gu_bytes + dn_bytes) / (ffn_ms * 1e-3) / 1e9},
        "incl_prefill": incl,
        "kernel_hbm": kernel_hbm,
        "kernel_ms_per_forward": {k: round(v["ms_per_step"], 4) for k, v in sorted(bd.items())},
        "forward_ms": 1e3 * t / steps / N, "context_avg": ctx_avg,
        "clocks": clk.summary(), "gpu_launches": launches_per_step * steps,
    }
    del eng
    if rank == 0 and main and args.cpu_baseline:
        cb = args.cpu_batch or B
        v, sample = cpu_layer_sample(arch, cb, int(ctx_avg), 2, os.cpu_count() or 1)
        line["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": os.cpu_count(), "kind": "port",
                                "sample": sample, "cpu_model": _cpu_model(), "batch": cb}
    return line


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="mixtral-8x7b")
    ap.add_argument("--batch", type=int, default=None, help="sequences per GPU (default: planner's largest)")
    ap.add_argument("--prompt-len", type=int, default=512)
    ap.add_argument("--decode-len", type=int, default=256)
    ap.add_argument("--reserve-gb", type=float, default=None,
                    help="HBM kept free beside weights + KV when sizing B (default: measured per model, RESERVE_GB)")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--cpu-batch", type=int, default=None, help="CPU arm batch (default: the GPU arm's B)")
    ap.add_argument("--no-cpu-baseline", dest="cpu_baseline", action="store_false")
    ap.add_argument("--also", default="deepseek-v2-lite",
                    help="comma-separated extra configs measured after the main one (\"\" = none)")
    ap.add_argument("--also-steps", type=int, default=3)
    ap.add_argument("--ep", default="auto", choices=["auto", "off", "force"],
                    help="auto: DeepSeek-V2-Lite runs expert-parallel over the job's GPUs when N > 1; force: also "
                         "at N = 1 (a one-rank NCCL group, the EP code path on one GPU)")
    ap.add_argument("--no-incl-prefill", dest="incl_prefill", action="store_false",
                    help="skip the batched-prefill pass behind the incl_prefill figure")
    args = ap.parse_args()
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # --gpus N without a launcher: start N ranks (one process per GPU) over torch.distributed.run
        # and exit with its status, so `python bench.py --gpus 8` measures 8 GPUs, not one
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", os.environ.get("MASTER_PORT", "29511"),
               os.path.abspath(__file__)] + sys.argv[1:]
        raise SystemExit(subprocess.call(cmd))
    if ws != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws}; launch one rank per GPU")
    dist, rank, world, local = _dist()
    if dist is None and args.ep == "force" and args.impl == "ours":  # one-rank group for the EP path
        import torch.distributed as tdist

        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", os.environ.get("MGB_EP_PORT", "29533"))
        torch.cuda.set_device(0)
        tdist.init_process_group("nccl", rank=0, world_size=1)
        dist = tdist
    if args.impl == "reference":
        run_reference(args, dist, rank, world)
    else:
        run_ours(args, dist, rank, world)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
