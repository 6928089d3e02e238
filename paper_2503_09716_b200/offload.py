"""Host/HBM weight placement for module-based batching with offloaded weights (the prefetch
subsystem).

Placement follows the reference's cache_placement (memory_model.py:147-164): the dense modules
of the first `dense_layers` layers and the first `experts_per_layer[l]` experts of every layer
stay resident in HBM; everything else lives in pinned host memory as one contiguous blob per
module (one DMA per module, offload_dag.py:308-321,438-445).  Uncached modules are streamed on
the H2D copy engine into
  - a single dense buffer (one layer's attention weights), and
  - `slots = s_expert // expert_bytes` expert slots, each [gate_up(2f x d) | down(d x f)],
recycled exactly as the schedule's buffer edges say (copy k reuses the slot of copy k - slots).
Values are generated on the device with the same counter-based generator as the resident build
(so outputs are bit-identical to it) and then moved to pinned host memory.
"""

from __future__ import annotations

import torch

from .configs import ModelArch
from .hostmem import pinned_empty
from .planner import placement, ModelSpec
from .weights import DERIVED, deepseek_layer, dense_keys, derive_views, global_tensors, mixtral_layer

BF16 = torch.bfloat16


class OffloadedWeights:
    """Weights of either family (Mixtral, DeepSeek-V2) split between HBM and pinned host memory by
    the reference's cache placement.  DeepSeek-V2's dense first layers (first_k_dense MLP) and all
    norms / router gates are small and stay resident; the dense modules of a layer are its
    attention projections plus its shared experts (the reference's dense_bytes_per_layer)."""

    def __init__(self, arch: ModelArch, spec: ModelSpec, s_params: int, s_expert: int, seed: int = 0,
                 device: str = "cuda", extra_slots: int = 0, extra_dense: int = 0, source=None):
        a = arch
        d, f, E = a.hidden, a.moe_ffn, a.n_experts
        std = a.init_std
        bf = dict(dtype=BF16, device=device)
        self.arch = a
        self.place = placement(spec, s_params)
        if a.is_mla and self.place.dense_layers < a.first_k_dense:
            raise ValueError("DeepSeek-V2 offload keeps the dense first layers resident: s_params too small")
        self.n_slots = s_expert // spec.expert_bytes if spec.expert_bytes else 0
        if self.place.uncached_expert_count > 0 and self.n_slots < 2:
            raise ValueError("offloaded experts need at least 2 expert slots (double buffering)")
        self.embed, self.final_norm, self.lm_head = global_tensors(a, seed, device, source)
        build = deepseek_layer if a.is_mla else mixtral_layer
        self.dense_keys = dense_keys(a)
        self.dense_shapes: dict[str, tuple] | None = None
        self.dense_elems = 0
        self.expert_elems = 3 * d * f
        self.dense_bufs: list[torch.Tensor] = []
        # the plan's s_expert slots, then one slot per cross-step lookahead expert copy (engine.py)
        self.slots = torch.empty(max(self.n_slots, 0) + extra_slots, self.expert_elems, **bf)
        self.layers: list[dict] = []
        self.host_dense: list[torch.Tensor | None] = []
        self.host_experts: list[torch.Tensor | None] = []
        moe_first = a.first_k_dense if a.is_mla else 0
        for l in range(a.layers):
            # generated on the device (bit-identical to the resident build), or loaded from a checkpoint
            L = build(a, l, seed, device, source)
            if l >= moe_first and self.dense_shapes is None:
                self.dense_shapes = {k: tuple(L[k].shape) for k in self.dense_keys}
                self.dense_elems = sum(L[k].numel() for k in self.dense_keys)
                assert self.dense_elems * 2 == spec.dense_bytes_per_layer, "dense blob != reference dense bytes"
                if self.place.dense_layers < a.layers:  # the single dense buffer (+ the lookahead one)
                    self.dense_bufs = [torch.empty(self.dense_elems, **bf) for _ in range(1 + extra_dense)]
            # dense modules: resident, or one pinned blob (one DMA per layer, offload_dag.py:308-321)
            if l < self.place.dense_layers:
                self.host_dense.append(None)
            else:
                blob = pinned_empty(self.dense_elems)
                o = 0
                for k in self.dense_keys:
                    t = L.pop(k).reshape(-1)
                    blob[o:o + t.numel()].copy_(t)
                    o += t.numel()
                self.host_dense.append(blob)
                for k in DERIVED:
                    L.pop(k, None)
            # routed experts: keep the cached prefix in HBM, one pinned blob [gate_up | down] per other expert
            n_c = self.place.experts_per_layer[l]
            if "w_gate_up" in L and n_c < E:
                gu, dn = L["w_gate_up"], L["w_down"]
                blob = pinned_empty((E - n_c) * self.expert_elems).view(E - n_c, self.expert_elems)
                g = 2 * f * d
                blob[:, :g].copy_(gu[n_c:].reshape(E - n_c, g))
                blob[:, g:].copy_(dn[n_c:].reshape(E - n_c, d * f))
                self.host_experts.append(blob)
                L["w_gate_up"] = gu[:n_c].clone() if n_c > 0 else None
                L["w_down"] = dn[:n_c].clone() if n_c > 0 else None
                del gu, dn
            else:
                self.host_experts.append(None)
            self.layers.append(L)
        torch.cuda.synchronize()

    def dense_views(self, buf: int = 0) -> dict:
        """The streamed dense modules as views into a dense buffer."""
        out, o = {}, 0
        for k in self.dense_keys:
            shape = self.dense_shapes[k]
            n = 1
            for x in shape:
                n *= x
            out[k] = self.dense_bufs[buf][o:o + n].view(shape)
            o += n
        return derive_views(self.arch, out)

    def slot_views(self, s: int):
        a = self.arch
        d, f = a.hidden, a.moe_ffn
        buf = self.slots[s]
        return buf[:2 * f * d].view(1, 2 * f, d), buf[2 * f * d:].view(1, d, f)

    def host_bytes(self) -> int:
        n = sum(t.nbytes for t in self.host_dense if t is not None)
        return n + sum(t.nbytes for t in self.host_experts if t is not None)


OffloadedMixtralWeights = OffloadedWeights
