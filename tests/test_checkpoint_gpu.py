"""The engine on real on-disk weights: a HF safetensors checkpoint written by HF
transformers itself (random-init by HF, not by this framework's generator) is loaded through
paper_2503_09716_b200.checkpoint, and the engine's decode is compared with HF's own model on the
same tokens: teacher-forced logits within the bf16 tolerance, greedy argmax equal on every
safe-margin row; the same checkpoint with weights offloaded to pinned expert blobs runs bit-identical
to the resident load."""

import pytest
import torch

import hf_models
import parity_util as PU

pytestmark = pytest.mark.gpu


def _engine(path, B, P, N, use_graph, offload=False):
    from paper_2503_09716_b200.checkpoint import Checkpoint
    from paper_2503_09716_b200.engine import Engine
    from paper_2503_09716_b200.planner import BatchingPlan, ModelSpec

    a = Checkpoint(path).arch
    spec = ModelSpec.from_document(a.model_spec_document())
    if offload:
        plan = BatchingPlan(B, B // 2, 16, 0.0, 3 * spec.expert_bytes,
                            a.layers * spec.dense_bytes_per_layer + 10 * spec.expert_bytes)
    else:
        plan = BatchingPlan(B, B // 2, 16, 0.0, 0, spec.model_bytes)
    return Engine(None, plan, prompt_len=P, decode_len=N, use_graph=use_graph, checkpoint=path)


@pytest.mark.parametrize("family", ["mixtral", "deepseek_v2"])
def test_engine_from_checkpoint_matches_hf(tmp_path, family):
    m = hf_models.tiny_mixtral_hf() if family == "mixtral" else hf_models.tiny_dsv2_hf()
    path = hf_models.save(m, tmp_path / "ck")
    V = m.config.vocab_size
    B, P, N = 8, 12, 8
    ids = torch.randint(0, V, (B, P), generator=torch.Generator().manual_seed(4))
    with torch.no_grad():
        ref = m.generate(ids, max_new_tokens=N, min_new_tokens=N, do_sample=False, pad_token_id=0)
        lg_hf = m(ref).logits.float()  # teacher-forced logits at every position
    eng = _engine(path, B, P, N, use_graph=False)
    assert eng.w.layers[0]["ln1"].float().std() > 0  # real (non-unit) norms were loaded
    errs, checked = [], 0
    for pos in range(P + N - 1):
        le = eng.debug_forward(ref[:, pos], pos)["logits"].float().cpu()
        lo = lg_hf[:, pos]
        errs += PU.row_errs(le, lo).tolist()
        if pos >= P - 1:
            ok, n = PU.margin_filtered_equal(le, lo)
            assert ok, f"position {pos}: greedy argmax differs from HF on a safe-margin row"
            checked += n
    errs.sort()
    print(f"{family}: teacher-forced logits vs HF: median row err {errs[len(errs) // 2]:.2e}, "
          f"p90 {errs[int(0.9 * len(errs))]:.2e}; safe-margin rows checked {checked}")
    assert errs[len(errs) // 2] <= 2e-2 and checked > 0
    out = _engine(path, B, P, N, use_graph=True).generate(ids, N)  # batched prefill + graph decode
    prefix = PU.greedy_prefix(out, ref, P)
    print(f"{family}: identical greedy rows vs HF {int((prefix == N).sum())}/{B}, mean prefix {prefix.float().mean():.1f}")
    off = _engine(path, B, P, N, use_graph=True, offload=True)
    assert off.offload and off.w.host_bytes() > 0
    assert torch.equal(off.generate(ids, N), out)
