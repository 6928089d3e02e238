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
from .planner import placement, ModelSpec
from .weights import TID_EMBED, TID_LM_HEAD, fill_const_, fill_uniform_, tid

BF16 = torch.bfloat16


class OffloadedMixtralWeights:
    def __init__(self, arch: ModelArch, spec: ModelSpec, s_params: int, s_expert: int, seed: int = 0,
                 device: str = "cuda"):
        a = arch
        d, hd, f, E = a.hidden, a.head_dim, a.moe_ffn, a.n_experts
        qd, kvd = a.n_heads * hd, a.n_kv_heads * hd
        std = a.init_std
        bf = dict(dtype=BF16, device=device)
        self.arch = a
        self.place = placement(spec, s_params)
        self.n_slots = s_expert // spec.expert_bytes if spec.expert_bytes else 0
        if self.place.uncached_expert_count > 0 and self.n_slots < 2:
            raise ValueError("offloaded experts need at least 2 expert slots (double buffering)")
        self.embed = fill_uniform_(torch.empty(a.vocab, d, **bf), seed, TID_EMBED, std)
        self.final_norm = fill_const_(torch.empty(d, **bf), 1.0)
        self.lm_head = fill_uniform_(torch.empty(a.vocab, d, **bf), seed, TID_LM_HEAD, std)
        self.dense_elems = (qd + 2 * kvd) * d + d * qd
        self.expert_elems = 3 * d * f
        self.dense_buf = torch.empty(self.dense_elems, **bf) if self.place.dense_layers < a.layers else None
        self.slots = torch.empty(max(self.n_slots, 0), self.expert_elems, **bf)
        self.layers = []
        self.host_dense: list[torch.Tensor | None] = []
        self.host_experts: list[torch.Tensor | None] = []
        stage = torch.empty(max(self.dense_elems, self.expert_elems), **bf)
        for l in range(a.layers):
            L = dict(ln1=fill_const_(torch.empty(d, **bf), 1.0), ln2=fill_const_(torch.empty(d, **bf), 1.0),
                     router=fill_uniform_(torch.empty(E, d, **bf), seed, tid(l, "router"), std))
            # dense (attention) weights: resident or one pinned blob [wqkv | wo]
            dense = torch.empty(self.dense_elems, **bf) if l < self.place.dense_layers else stage[:self.dense_elems]
            wqkv = dense[:(qd + 2 * kvd) * d].view(qd + 2 * kvd, d)
            fill_uniform_(wqkv[:qd], seed, tid(l, "wq"), std)
            fill_uniform_(wqkv[qd:qd + kvd], seed, tid(l, "wk"), std)
            fill_uniform_(wqkv[qd + kvd:], seed, tid(l, "wv"), std)
            fill_uniform_(dense[(qd + 2 * kvd) * d:].view(d, qd), seed, tid(l, "wo"), std)
            if l < self.place.dense_layers:
                L["wqkv"], L["wo"] = wqkv, dense[(qd + 2 * kvd) * d:].view(d, qd)
                self.host_dense.append(None)
            else:
                self.host_dense.append(dense.cpu().pin_memory())
            # experts: generate the full per-layer tensors (tensor-id indexing), keep the cached
            # prefix in HBM, move the rest to one pinned blob per expert
            n_c = self.place.experts_per_layer[l]
            gu = fill_uniform_(torch.empty(E, 2 * f, d, **bf), seed, tid(l, "w_gate_up"), std)
            dn = fill_uniform_(torch.empty(E, d, f, **bf), seed, tid(l, "w_down"), std)
            L["w_gate_up"] = gu[:n_c].clone() if n_c > 0 else None
            L["w_down"] = dn[:n_c].clone() if n_c > 0 else None
            if n_c < E:
                blob = torch.empty(E - n_c, self.expert_elems, dtype=BF16).pin_memory()
                for e in range(n_c, E):
                    row = torch.cat([gu[e].reshape(-1), dn[e].reshape(-1)])
                    blob[e - n_c].copy_(row)
                self.host_experts.append(blob)
            else:
                self.host_experts.append(None)
            del gu, dn
            self.layers.append(L)
        torch.cuda.synchronize()

    # views into the streamed buffers
    def dense_views(self):
        a = self.arch
        d, hd = a.hidden, a.head_dim
        qd, kvd = a.n_heads * hd, a.n_kv_heads * hd
        return (self.dense_buf[:(qd + 2 * kvd) * d].view(qd + 2 * kvd, d),
                self.dense_buf[(qd + 2 * kvd) * d:].view(d, qd))

    def slot_views(self, s: int):
        a = self.arch
        d, f = a.hidden, a.moe_ffn
        buf = self.slots[s]
        return buf[:2 * f * d].view(1, 2 * f, d), buf[2 * f * d:].view(1, d, f)

    def host_bytes(self) -> int:
        n = sum(t.nbytes for t in self.host_dense if t is not None)
        return n + sum(t.nbytes for t in self.host_experts if t is not None)
