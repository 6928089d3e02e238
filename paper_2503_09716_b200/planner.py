"""Host-side mirror of the reference planner's engine-facing interface.

The engine consumes the reference's decision vector and sizes its HBM buffers with the
reference's memory model, so a plan produced by `moe-planner plan` drops straight in:
  - ModelSpec document      (reference: pkg/src/moe_planner/model_catalog.py:55-188)
  - WorkloadSpec / BatchingPlan (memory_model.py:35-89), incl. Python round() for omega*B
  - validate_plan           (memory_model.py:96-127)
  - cache_placement         (memory_model.py:147-164)
  - check_constraints, max_feasible_B (memory_model.py:182-277)
  - plan.json read/write    (cli.py:74-109)
  - HardwareProfile / latency tables + lookup (hw_profile.py:70-149,156-249,361-409)
Behaviour (including error classes' meaning) is identical; the implementation is independent.

Extension for B200 (not in the reference): kv_policy="resident" keeps every sequence's KV in
HBM (paged) instead of the reference's full KV offload; its constraint moves the KV term from
the host equation (Eq. 2) to the GPU equation (Eq. 3).
"""

from __future__ import annotations

import json
import math
from bisect import bisect_left
from dataclasses import asdict, dataclass, field, replace
from typing import Any, Mapping, Sequence

# ----------------------------------------------------------------------------------------
# model geometry
# ----------------------------------------------------------------------------------------
_REQUIRED = ("name", "num_layers", "experts_per_layer", "top_k", "shared_expert_bytes",
             "attention_weights_bytes", "expert_bytes", "kv_bytes_per_token_layer", "hidden_bytes_per_token",
             "attn_flops_base", "attn_flops_per_context", "expert_flops_per_token")
_OPTIONAL = ("attn_activation_bytes_per_token", "attn_activation_bytes_per_ctx_token",
             "expert_activation_bytes_per_token")
_POSITIVE = ("num_layers", "experts_per_layer", "top_k", "attention_weights_bytes", "expert_bytes",
             "kv_bytes_per_token_layer", "hidden_bytes_per_token", "attn_flops_base", "attn_flops_per_context",
             "expert_flops_per_token")


class SpecError(ValueError):
    pass


@dataclass(frozen=True)
class ModelSpec:
    name: str
    num_layers: int
    experts_per_layer: int
    top_k: int
    shared_expert_bytes: int
    attention_weights_bytes: int
    expert_bytes: int
    kv_bytes_per_token_layer: int
    hidden_bytes_per_token: int
    attn_flops_base: float
    attn_flops_per_context: float
    expert_flops_per_token: float
    attn_activation_bytes_per_token: float | None = None
    attn_activation_bytes_per_ctx_token: float = 0.0
    expert_activation_bytes_per_token: float | None = None

    def __post_init__(self) -> None:
        for f in _POSITIVE:
            if getattr(self, f) <= 0:
                raise SpecError(f"model spec field {f!r} must be positive")
        if self.shared_expert_bytes < 0 or self.attn_activation_bytes_per_ctx_token < 0:
            raise SpecError("byte fields must be non-negative")
        if self.top_k > self.experts_per_layer:
            raise SpecError("top_k exceeds experts_per_layer")

    @classmethod
    def from_document(cls, doc: Mapping[str, Any]) -> "ModelSpec":
        missing = [f for f in _REQUIRED if f not in doc]
        if missing:
            raise SpecError(f"model spec is missing required field {missing[0]!r}")
        return cls(**{f: doc[f] for f in _REQUIRED + _OPTIONAL if f in doc})

    @property
    def dense_bytes_per_layer(self) -> int:
        return self.attention_weights_bytes + self.shared_expert_bytes

    @property
    def model_bytes(self) -> int:
        return self.num_layers * (self.dense_bytes_per_layer + self.experts_per_layer * self.expert_bytes)

    @property
    def attn_activation_per_token(self) -> float:
        if self.attn_activation_bytes_per_token is not None:
            return self.attn_activation_bytes_per_token
        return 2.0 * self.hidden_bytes_per_token

    @property
    def expert_activation_per_token(self) -> float:
        if self.expert_activation_bytes_per_token is not None:
            return self.expert_activation_bytes_per_token
        return 2.0 * (2.0 * self.expert_bytes / (3.0 * self.hidden_bytes_per_token))


# ----------------------------------------------------------------------------------------
# hardware + latency tables
# ----------------------------------------------------------------------------------------
MODULE_KINDS = ("pre_attention", "attention_mechanism_gpu", "attention_mechanism_cpu", "post_attention",
                "expert", "router")


@dataclass(frozen=True)
class Hardware:
    m_g: int
    m_c: int
    bw_htod: float
    bw_dtoh: float
    gpu_peak_flops: float
    gpu_mem_bw: float
    gpu_launch_overhead: float
    cpu_attn_flops: float
    components: tuple = ()

    def to_document(self) -> dict[str, Any]:
        d = asdict(self)
        d["components"] = list(self.components)
        return d


@dataclass
class LatencyCurve:
    """Per-module latency samples (tokens, context, seconds), interpolated like the reference:
    piecewise-linear in tokens (clamped below, last-slope extrapolation above), linear in context
    between levels, clamped outside (hw_profile.py:361-409)."""

    module_kind: str
    entries: list = field(default_factory=list)

    def _levels(self) -> dict[int, list[tuple[int, float]]]:
        # derived once: a curve's samples are fixed after construction
        lv = self.__dict__.get("_lv")
        if lv is None or self.__dict__.get("_lv_n") != len(self.entries):
            lv = {}
            for t, c, s in sorted(self.entries, key=lambda e: (e[1], e[0])):
                lv.setdefault(int(c), []).append((int(t), float(s)))
            self.__dict__["_lv"], self.__dict__["_lv_n"] = lv, len(self.entries)
        return lv

    @staticmethod
    def _in_tokens(pts: list[tuple[int, float]], n: int) -> float:
        xs = [p[0] for p in pts]
        if n <= xs[0]:
            return pts[0][1]
        if n >= xs[-1]:
            (x0, y0), (x1, y1) = pts[-2], pts[-1]
            return y1 + (y1 - y0) / (x1 - x0) * (n - x1)
        i = bisect_left(xs, n)
        if xs[i] == n:
            return pts[i][1]
        (x0, y0), (x1, y1) = pts[i - 1], pts[i]
        return y0 + (n - x0) / (x1 - x0) * (y1 - y0)

    def __call__(self, tokens: int, context: int) -> float:
        lv = self._levels()
        cs = sorted(lv)
        if context <= cs[0]:
            return self._in_tokens(lv[cs[0]], tokens)
        if context >= cs[-1]:
            return self._in_tokens(lv[cs[-1]], tokens)
        i = bisect_left(cs, context)
        if cs[i] == context:
            return self._in_tokens(lv[cs[i]], tokens)
        c0, c1 = cs[i - 1], cs[i]
        a, b = self._in_tokens(lv[c0], tokens), self._in_tokens(lv[c1], tokens)
        return a + (context - c0) / (c1 - c0) * (b - a)


def profile_document(hw: Hardware, curves: Sequence[LatencyCurve]) -> dict[str, Any]:
    """Profile JSON accepted by the reference's ingest_profile (hw_profile.py:156-216)."""
    return {"hardware": hw.to_document(),
            "latency_tables": [{"module_kind": c.module_kind, "entries": [list(e) for e in c.entries]}
                               for c in curves]}


def load_profile_document(doc: Mapping[str, Any]) -> tuple[Hardware, list[LatencyCurve]]:
    h = doc["hardware"]
    hw = Hardware(**{k: h[k] for k in ("m_g", "m_c", "bw_htod", "bw_dtoh", "gpu_peak_flops", "gpu_mem_bw",
                                       "gpu_launch_overhead", "cpu_attn_flops")})
    curves = [LatencyCurve(t["module_kind"], [tuple(e) for e in t["entries"]]) for t in doc.get("latency_tables", [])]
    return hw, curves


# ----------------------------------------------------------------------------------------
# workload + plan
# ----------------------------------------------------------------------------------------
@dataclass(frozen=True)
class WorkloadSpec:
    prompt_len: int
    decode_len: int
    num_sequences: int
    phase: str = "decode"

    def __post_init__(self) -> None:
        if self.prompt_len < 1 or self.decode_len < 0 or self.num_sequences < 1:
            raise ValueError("invalid workload")
        if self.phase not in ("prefill", "decode"):
            raise ValueError(f"unknown phase {self.phase!r}")

    @property
    def max_context(self) -> int:
        return self.prompt_len + self.decode_len

    @property
    def tokens_per_seq_in_flight(self) -> int:
        return self.prompt_len if self.phase == "prefill" else 1

    def with_phase(self, phase: str) -> "WorkloadSpec":
        return replace(self, phase=phase)


@dataclass(frozen=True)
class BatchingPlan:
    """(B, b_a, b_e, omega, s_expert, s_params) — memory_model.py:66-89."""

    B: int
    b_a: int
    b_e: int
    omega: float
    s_expert: int
    s_params: int

    def cpu_sequences(self) -> int:
        return int(round(self.omega * self.B))  # Python round(): banker's rounding, as the reference

    def gpu_sequences(self) -> int:
        return self.B - self.cpu_sequences()

    def to_document(self) -> dict[str, Any]:
        return {"B": self.B, "b_a": self.b_a, "b_e": self.b_e, "omega": self.omega, "s_expert": self.s_expert,
                "s_params": self.s_params}

    @classmethod
    def from_document(cls, doc: Mapping[str, Any]) -> "BatchingPlan":
        if "plan" in doc:  # full evaluation document (cli.py:85-87)
            doc = doc["plan"]
        try:
            return cls(int(doc["B"]), int(doc["b_a"]), int(doc["b_e"]), float(doc["omega"]), int(doc["s_expert"]),
                       int(doc["s_params"]))
        except (KeyError, TypeError, ValueError) as exc:
            raise ValueError(f"malformed plan document: {exc}") from exc


def load_plan(path_or_doc) -> BatchingPlan:
    if isinstance(path_or_doc, BatchingPlan):
        return path_or_doc
    if isinstance(path_or_doc, Mapping):
        return BatchingPlan.from_document(path_or_doc)
    with open(path_or_doc, "r", encoding="utf-8") as f:
        return BatchingPlan.from_document(json.load(f))


class PlanError(ValueError):
    def __init__(self, fld: str, reason: str):
        super().__init__(f"invalid plan field {fld!r}: {reason}")
        self.field = fld


MIN_EXPERT_SLOTS = 2


@dataclass(frozen=True)
class Placement:
    dense_layers: int
    experts_per_layer: tuple
    cached_bytes: int
    uncached_expert_count: int


def placement(spec: ModelSpec, s_params: int) -> Placement:
    """Dense layers first, then experts round-robin across layers (memory_model.py:147-164)."""
    L, E, dense = spec.num_layers, spec.experts_per_layer, spec.dense_bytes_per_layer
    n_dense = min(L, s_params // dense) if dense > 0 else L
    n_exp = min(L * E, int((s_params - n_dense * dense) // spec.expert_bytes))
    q, r = divmod(n_exp, L)
    return Placement(n_dense, tuple(q + (l < r) for l in range(L)), n_dense * dense + n_exp * spec.expert_bytes,
                     L * E - n_exp)


def validate(spec: ModelSpec, plan: BatchingPlan) -> None:
    if plan.B < 1:
        raise PlanError("B", "must be >= 1")
    if plan.b_e < 1:
        raise PlanError("b_e", "must be >= 1")
    if not 0.0 <= plan.omega <= 1.0:
        raise PlanError("omega", "must be within [0, 1]")
    if abs(plan.omega / 0.1 - round(plan.omega / 0.1)) > 1e-9:
        raise PlanError("omega", "must be a multiple of 0.1")
    if plan.b_a < 1:
        raise PlanError("b_a", "must be >= 1")
    if plan.omega < 1.0 and plan.b_a > math.ceil((1.0 - plan.omega) * plan.B):
        raise PlanError("b_a", "exceeds the GPU share ceil((1 - omega) * B) of the batch")
    if plan.s_params < 0:
        raise PlanError("s_params", "must be >= 0")
    if plan.s_params > spec.model_bytes:
        raise PlanError("s_params", "exceeds the model size")
    if placement(spec, plan.s_params).uncached_expert_count > 0:
        if plan.s_expert < MIN_EXPERT_SLOTS * spec.expert_bytes:
            raise PlanError("s_expert", "below the double-buffering floor while uncached experts remain")
    elif plan.s_expert < 0:
        raise PlanError("s_expert", "must be >= 0")


@dataclass(frozen=True)
class Footprint:
    s_kv_cpu: int
    s_kv_gpu: int
    s_is: int
    host_total: int
    gpu_total: int
    host_feasible: bool
    gpu_feasible: bool

    @property
    def feasible(self) -> bool:
        return self.host_feasible and self.gpu_feasible


def footprint(spec: ModelSpec, hw: Hardware, wl: WorkloadSpec, plan: BatchingPlan,
              kv_policy: str = "offload") -> Footprint:
    """Eq. 2 (host) and Eq. 3 (GPU) of the paper, as memory_model.py:182-243 computes them."""
    prefill = wl.phase == "prefill"
    tif = wl.tokens_per_seq_in_flight
    ctx = wl.prompt_len if prefill else wl.max_context
    kv_all = plan.B * wl.max_context * spec.kv_bytes_per_token_layer * spec.num_layers
    kv_slice = 0 if (prefill or plan.omega >= 1.0) else plan.b_a * wl.max_context * spec.kv_bytes_per_token_layer
    s_is = int(plan.B * tif * spec.hidden_bytes_per_token + plan.b_a * tif * spec.attn_activation_per_token
               + plan.b_a * ctx * spec.attn_activation_bytes_per_ctx_token
               + plan.b_e * spec.expert_activation_per_token)
    if kv_policy == "resident":
        host = spec.model_bytes
        gpu = plan.s_params + plan.s_expert + spec.dense_bytes_per_layer + kv_all + s_is
        s_kv_cpu, s_kv_gpu = 0, kv_all
    else:
        host = kv_all + spec.model_bytes
        gpu = plan.s_params + plan.s_expert + spec.dense_bytes_per_layer + kv_slice + s_is
        s_kv_cpu, s_kv_gpu = kv_all, kv_slice
    return Footprint(s_kv_cpu, s_kv_gpu, s_is, host, gpu, host <= hw.m_c, gpu <= hw.m_g)


def largest_batch(spec: ModelSpec, hw: Hardware, wl: WorkloadSpec, template: BatchingPlan,
                  kv_policy: str = "offload") -> int:
    """Largest feasible B with the other plan fields fixed (monotone: doubling + bisection),
    memory_model.py:246-277.  Raises ValueError if even B=1 is infeasible."""
    ok = lambda B: footprint(spec, hw, wl, replace(template, B=B), kv_policy).feasible  # noqa: E731
    if not ok(1):
        raise ValueError("no batch size satisfies the host and GPU memory constraints")
    lo = 1
    while ok(lo * 2):
        lo *= 2
    hi = lo * 2 - 1
    while lo < hi:
        mid = (lo + hi + 1) // 2
        if ok(mid):
            lo = mid
        else:
            hi = mid - 1
    return lo
