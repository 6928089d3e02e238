"""Generate the golden fixtures under tests/golden/ from the reference itself (run in the build
container, where /root/reference and HF transformers exist; the GPU box never runs this).

  PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

1. schedule_*.json  — the reference planner's serialized forward DAG (moe_planner
   build_forward_dag, offload_dag.py:514-533) for several (model, hardware, workload, plan,
   phase, routing) cases, plus the profile document it used and its critical path
   (plan_search.py:57-59).  tests/test_schedule.py rebuilds each with
   paper_2503_09716_b200.schedule and demands identical jobs and edges.
2. memory_model.json — footprints (memory_model.py:217-243), max_feasible_B (:246-277) and
   cache placements (:147-164) for a grid of plans.
3. hf_tiny_mixtral.pt — HF transformers 5.5.0 MixtralForCausalLM (sdpa attention, grouped_mm
   experts) run on the counter-based random-init weights of the tiny config: per-layer hidden
   states of one forward, router logits, and greedy generations.  Pins oracle/moe_ref.py.
"""

from __future__ import annotations

import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

import torch  # noqa: E402

import moe_planner as mp  # noqa: E402
from moe_planner.exec_sim import RoutingModel, sample_routing  # noqa: E402
from moe_planner.hw_profile import profile_to_document  # noqa: E402


def _dag_doc(dag):
    return {
        "nodes": [{"id": n.id, "kind": n.kind.value, "resource": n.resource.value if n.resource else None,
                   "duration": n.duration, "label": n.label, "layer": n.layer, "tokens": n.tokens, "seqs": n.seqs,
                   "nbytes": n.nbytes} for n in dag.nodes],
        "edges": [list(e) for e in dag.edges],
        "entry": dag.entry_id,
        "exit": dag.exit_id,
    }


def schedules():
    from paper_2503_09716_b200.configs import MIXTRAL_8X7B, TINY

    cases = []
    tiny = mp.preset("tiny-test")
    tiny_hw = mp.tiny_test_hw()
    wl_tiny = mp.WorkloadSpec(64, 32, 1024, "decode")
    e = tiny.expert_bytes
    cases.append(("tiny_decode_omega05", tiny, tiny_hw, wl_tiny, mp.BatchingPlan(64, 16, 40, 0.5, 2 * e, 0), None))
    cases.append(("tiny_decode_cached", tiny, tiny_hw, wl_tiny,
                  mp.BatchingPlan(32, 8, 16, 0.0, 3 * e, tiny.dense_bytes_per_layer + 3 * e), None))
    cases.append(("tiny_prefill", tiny, tiny_hw, wl_tiny.with_phase("prefill"),
                  mp.BatchingPlan(4, 2, 100, 0.0, 2 * e, 0), None))
    counts = [sample_routing(tiny, 48, RoutingModel("sampled", 0.3, 7), l) for l in range(tiny.num_layers)]
    cases.append(("tiny_decode_sampled_routing", tiny, tiny_hw, wl_tiny, mp.BatchingPlan(48, 16, 8, 0.0, 2 * e, 0),
                  counts))
    mix = mp.preset("mixtral-8x7b")
    hw_a = mp.a5000_like(256_000_000_000)
    wl_mix = mp.WorkloadSpec(512, 256, 10_000, "decode")
    cases.append(("mixtral_a5000_searched", mix, hw_a, wl_mix,
                  mp.BatchingPlan(1620, 256, 1024, 0.6, 8 * mix.expert_bytes, 20_000_000_000), None))
    ds = mp.preset("deepseek-v2-like")
    hw_b = mp.a5000_like(512_000_000_000)
    tmpl = mp.BatchingPlan(1, 16, 4096, 0.0, 8 * ds.expert_bytes, 0)
    ds_B = min(96, mp.max_feasible_B(ds, hw_b, wl_mix, tmpl))
    cases.append(("deepseek_a5000", ds, hw_b, wl_mix, mp.BatchingPlan(ds_B, 16, 4096, 0.0, 8 * ds.expert_bytes, 0),
                  None))
    # this framework's own model documents (configs.py) through the reference planner
    tiny_doc = mp.load_model_spec(TINY.model_spec_document())
    hw_big = mp.HardwareProfile(m_g=180_000_000_000, m_c=2_000_000_000_000, bw_htod=55e9, bw_dtoh=55e9,
                                gpu_peak_flops=1.6e15, gpu_mem_bw=6.5e12, gpu_launch_overhead=5e-6,
                                cpu_attn_flops=0.0)
    cases.append(("tinymixtral_b200_resident_weights", tiny_doc, hw_big, mp.WorkloadSpec(64, 32, 64, "decode"),
                  mp.BatchingPlan(64, 32, 16, 0.0, 0, tiny_doc.model_bytes), None))
    mix_doc = mp.load_model_spec(MIXTRAL_8X7B.model_spec_document())
    cases.append(("mixtral8x7b_b200_offload", mix_doc, hw_big, mp.WorkloadSpec(512, 256, 10_000, "decode"),
                  mp.BatchingPlan(512, 256, 4096, 0.0, 4 * mix_doc.expert_bytes, 60_000_000_000), None))
    out = []
    for name, model, hw, wl, plan, counts in cases:
        tables = mp.synth_profile(hw, model)
        layer = None
        if model.num_layers * model.experts_per_layer > 1000:
            # 60 x 160 experts: keep the fixture small -> one unserialized layer DAG (offload_dag.py:495-511)
            layer = 5
            dag = mp.build_layer_dag(model, hw, tables, wl, plan, layer_index=layer)
        else:
            dag = mp.build_forward_dag(model, hw, tables, wl, plan, expert_tokens=counts)
        doc = {
            "layer_index": layer,
            "name": name,
            "model": model.to_document(),
            "profile": profile_to_document(hw, tables),
            "workload": {"prompt_len": wl.prompt_len, "decode_len": wl.decode_len,
                         "num_sequences": wl.num_sequences, "phase": wl.phase.value},
            "plan": {"B": plan.B, "b_a": plan.b_a, "b_e": plan.b_e, "omega": plan.omega, "s_expert": plan.s_expert,
                     "s_params": plan.s_params},
            "expert_tokens": counts,
            "critical_path": mp.critical_path(dag),
            "dag": _dag_doc(dag),
        }
        path = os.path.join(HERE, f"schedule_{name}.json")
        with open(path, "w") as f:
            json.dump(doc, f, sort_keys=True)
        out.append((name, len(dag.nodes), len(dag.edges)))
    return out


def memory_model():
    from paper_2503_09716_b200.configs import DSV2_LITE, MIXTRAL_8X7B

    rows = []
    models = {"mixtral-8x7b": mp.preset("mixtral-8x7b"), "deepseek-v2-like": mp.preset("deepseek-v2-like"),
              "tiny-test": mp.preset("tiny-test"),
              "cfg-mixtral-8x7b": mp.load_model_spec(MIXTRAL_8X7B.model_spec_document()),
              "cfg-deepseek-v2-lite": mp.load_model_spec(DSV2_LITE.model_spec_document())}
    hws = {"a5000-256": mp.a5000_like(256_000_000_000), "a5000-512": mp.a5000_like(512_000_000_000),
           "tiny": mp.tiny_test_hw()}
    for mname, model in models.items():
        for hname, hw in hws.items():
            for phase in ("decode", "prefill"):
                wl = mp.WorkloadSpec(512 if mname != "tiny-test" else 64, 256 if mname != "tiny-test" else 32, 1000,
                                     phase)
                for slots in (2, 8):
                    for b_a in (16, 256):
                        for omega in (0.0, 0.5):
                            tmpl = mp.BatchingPlan(1, b_a, 1024, omega, slots * model.expert_bytes, 0)
                            try:
                                bmax = mp.max_feasible_B(model, hw, wl, tmpl)
                            except mp.NoFeasibleB:
                                bmax = None
                            B = max(b_a, 100)
                            plan = mp.BatchingPlan(B, b_a, 1024, omega, slots * model.expert_bytes,
                                                   model.model_bytes // 3)
                            fp = mp.check_constraints(model, hw, wl, plan)
                            pl = mp.cache_placement(model, plan.s_params)
                            rows.append({"model": model.to_document(), "hw": profile_to_document(hw, [])["hardware"],
                                         "workload": [wl.prompt_len, wl.decode_len, wl.num_sequences, phase],
                                         "template": [1, b_a, 1024, omega, slots * model.expert_bytes, 0],
                                         "max_feasible_B": bmax, "plan": [B, b_a, 1024, omega,
                                                                          slots * model.expert_bytes,
                                                                          model.model_bytes // 3],
                                         "footprint": [fp.s_kv_cpu, fp.s_kv_gpu, fp.s_is, fp.host_total, fp.gpu_total,
                                                       fp.host_feasible, fp.gpu_feasible],
                                         "placement": [pl.dense_layers, list(pl.experts_per_layer), pl.cached_bytes,
                                                       pl.uncached_expert_count],
                                         "cpu_sequences": plan.cpu_sequences()})
    # banker's rounding corner of cpu_sequences (memory_model.py:85-86)
    extra = [[B, om, mp.BatchingPlan(B, 1, 1, om, 0, 0).cpu_sequences()] for B in (1, 3, 5, 15, 25, 1620)
             for om in (0.1, 0.3, 0.5, 0.7, 0.9)]
    with open(os.path.join(HERE, "memory_model.json"), "w") as f:
        json.dump({"rows": rows, "cpu_sequences": extra}, f, sort_keys=True)
    return len(rows)


def hf_tiny():
    from transformers import MixtralConfig, MixtralForCausalLM

    from oracle import moe_ref as R
    from paper_2503_09716_b200.configs import TINY

    a = TINY
    cfg = MixtralConfig(vocab_size=a.vocab, hidden_size=a.hidden, intermediate_size=a.moe_ffn,
                        num_hidden_layers=a.layers, num_attention_heads=a.n_heads, num_key_value_heads=a.n_kv_heads,
                        head_dim=a.head_dim, num_local_experts=a.n_experts, num_experts_per_tok=a.top_k,
                        rope_theta=a.rope_theta, rms_norm_eps=a.rms_eps, max_position_embeddings=4096,
                        tie_word_embeddings=False)
    cfg._attn_implementation = "sdpa"
    torch.manual_seed(0)
    model = MixtralForCausalLM._from_config(cfg, dtype=torch.bfloat16, experts_implementation="grouped_mm").eval()
    W = R.make_mixtral_weights(a, seed=0)
    sd = {"model.embed_tokens.weight": W.embed, "model.norm.weight": W.final_norm, "lm_head.weight": W.lm_head}
    for l, L in enumerate(W.layers):
        p = f"model.layers.{l}."
        sd.update({p + "input_layernorm.weight": L["ln1"], p + "post_attention_layernorm.weight": L["ln2"],
                   p + "self_attn.q_proj.weight": L["wq"], p + "self_attn.k_proj.weight": L["wk"],
                   p + "self_attn.v_proj.weight": L["wv"], p + "self_attn.o_proj.weight": L["wo"],
                   p + "mlp.gate.weight": L["router"], p + "mlp.experts.gate_up_proj": L["w_gate_up"],
                   p + "mlp.experts.down_proj": L["w_down"]})
    missing, unexpected = model.load_state_dict(sd, strict=False)
    assert not unexpected, unexpected
    assert all("rotary" in m for m in missing), missing
    B, P, N = 4, 8, 8
    ids = torch.randint(0, a.vocab, (B, P), generator=torch.Generator().manual_seed(1))
    with torch.no_grad():
        out = model(ids, output_hidden_states=True, output_router_logits=True, use_cache=False)
        gen = model.generate(ids, max_new_tokens=N, min_new_tokens=N, do_sample=False, pad_token_id=0)
        # teacher-forced logits of the generated continuation (one forward over P+N-1 tokens)
        tf = model(gen[:, :-1], use_cache=False).logits[:, P - 1:, :]
    top = torch.topk(tf.float(), 16, dim=-1)
    doc = {
        "input_ids": ids,
        "hidden_states": [h[:, -1, :].clone() for h in out.hidden_states],  # last prompt position, per layer
        "router_logits": [r.view(B, P, -1)[:, -1, :].clone() for r in out.router_logits],
        "last_logits": out.logits[:, -1, :].clone(),
        "generated": gen,
        "tf_top16_values": top.values, "tf_top16_indices": top.indices,
        "meta": {"transformers": __import__("transformers").__version__, "attn": "sdpa",
                 "experts": "grouped_mm", "B": B, "P": P, "N": N},
    }
    torch.save(doc, os.path.join(HERE, "hf_tiny_mixtral.pt"))
    return gen


def hf_tiny_dsv2():
    """HF DeepseekV2ForCausalLM (MLA, group-limited routing, shared experts, dense layer 0) on the
    counter-based weights of configs.TINY_DSV2 (default rope: the YaRN scaling of the released
    checkpoints is a checkpoint property, not part of the path)."""
    from transformers import DeepseekV2Config, DeepseekV2ForCausalLM

    from oracle import moe_ref as R
    from paper_2503_09716_b200.configs import TINY_DSV2

    a = TINY_DSV2
    cfg = DeepseekV2Config(vocab_size=a.vocab, hidden_size=a.hidden, intermediate_size=a.dense_ffn,
                           moe_intermediate_size=a.moe_ffn, num_hidden_layers=a.layers, num_attention_heads=a.n_heads,
                           num_key_value_heads=a.n_heads, n_shared_experts=a.n_shared, n_routed_experts=a.n_experts,
                           routed_scaling_factor=a.routed_scaling, kv_lora_rank=a.kv_lora_rank, q_lora_rank=None,
                           qk_rope_head_dim=a.qk_rope_dim, v_head_dim=a.v_head_dim, qk_nope_head_dim=a.qk_nope_dim,
                           topk_method=a.topk_method, n_group=a.n_group, topk_group=a.topk_group,
                           num_experts_per_tok=a.top_k, first_k_dense_replace=a.first_k_dense, rms_norm_eps=a.rms_eps,
                           max_position_embeddings=4096, tie_word_embeddings=False,
                           rope_parameters={"rope_type": "default", "rope_theta": a.rope_theta})
    cfg._attn_implementation = "sdpa"
    model = DeepseekV2ForCausalLM._from_config(cfg, dtype=torch.bfloat16, experts_implementation="grouped_mm").eval()
    W = R.make_dsv2_weights(a, seed=0)
    sd = {"model.embed_tokens.weight": W.embed, "model.norm.weight": W.final_norm, "lm_head.weight": W.lm_head}
    for l, L in enumerate(W.layers):
        p = f"model.layers.{l}."
        sd.update({p + "input_layernorm.weight": L["ln1"], p + "post_attention_layernorm.weight": L["ln2"],
                   p + "self_attn.q_proj.weight": L["q_proj"], p + "self_attn.kv_a_proj_with_mqa.weight": L["kv_a"],
                   p + "self_attn.kv_a_layernorm.weight": L["kv_a_norm"], p + "self_attn.kv_b_proj.weight": L["kv_b"],
                   p + "self_attn.o_proj.weight": L["wo"]})
        if l < a.first_k_dense:
            f = a.dense_ffn
            sd.update({p + "mlp.gate_proj.weight": L["dense_gate_up"][:f], p + "mlp.up_proj.weight": L["dense_gate_up"][f:],
                       p + "mlp.down_proj.weight": L["dense_down"]})
        else:
            fs = a.moe_ffn * a.n_shared
            sd.update({p + "mlp.gate.weight": L["router"], p + "mlp.experts.gate_up_proj": L["w_gate_up"],
                       p + "mlp.experts.down_proj": L["w_down"],
                       p + "mlp.shared_experts.gate_proj.weight": L["sh_gate_up"][:fs],
                       p + "mlp.shared_experts.up_proj.weight": L["sh_gate_up"][fs:],
                       p + "mlp.shared_experts.down_proj.weight": L["sh_down"]})
    missing, unexpected = model.load_state_dict(sd, strict=False)
    assert not unexpected, unexpected
    assert all("rotary" in m for m in missing), missing
    # HF 5.5.0 DeepseekV2Moe.route_tokens_to_experts reads self.num_experts for
    # group_limited_greedy (modeling_deepseek_v2.py:112) but never sets it: supply the attribute.
    for layer in model.model.layers:
        if hasattr(layer.mlp, "experts"):
            layer.mlp.num_experts = a.n_experts
    B, P, N = 4, 6, 6
    ids = torch.randint(0, a.vocab, (B, P), generator=torch.Generator().manual_seed(2))
    with torch.no_grad():
        out = model(ids, output_hidden_states=True, use_cache=False)
        gen = model.generate(ids, max_new_tokens=N, min_new_tokens=N, do_sample=False, pad_token_id=0)
    doc = {"input_ids": ids, "hidden_states": [h[:, -1, :].clone() for h in out.hidden_states],
           "last_logits": out.logits[:, -1, :].clone(), "generated": gen,
           "meta": {"transformers": __import__("transformers").__version__, "attn": "sdpa", "B": B, "P": P, "N": N}}
    torch.save(doc, os.path.join(HERE, "hf_tiny_dsv2.pt"))
    return gen


if __name__ == "__main__":
    print("schedules", schedules())
    print("memory rows", memory_model())
    print("hf generate", hf_tiny().tolist())
    print("hf dsv2 generate", hf_tiny_dsv2().tolist())
