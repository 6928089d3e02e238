"""Scratch: layer-by-layer engine vs oracle comparison on the tiny config."""
import sys

import torch

sys.path.insert(0, ".")
from oracle import moe_ref as R  # noqa: E402
from paper_2503_09716_b200 import ops  # noqa: E402
from paper_2503_09716_b200.configs import TINY  # noqa: E402
from paper_2503_09716_b200.engine import Engine  # noqa: E402
from paper_2503_09716_b200.planner import BatchingPlan, ModelSpec  # noqa: E402

B, P, N = 8, 6, 10
mb = ModelSpec.from_document(TINY.model_spec_document()).model_bytes
eng = Engine(TINY, BatchingPlan(B, B // 2, 16, 0.0, 0, mb), prompt_len=P, decode_len=N, use_graph=False)
orc = R.MixtralOracle(TINY, R.make_mixtral_weights(TINY, 0))
toks = torch.randint(0, TINY.vocab, (B, P + N), generator=torch.Generator().manual_seed(1))
for pos in range(4):
    eng.buf.positions.fill_(pos)
    eng.buf.next_ids.copy_(toks[:, pos].to(torch.int32))
    ops.embed(eng.buf.next_ids, eng.w.embed, eng.buf.x)
    x = orc.w.embed[toks[:, pos]]
    print("pos", pos, "embed eq", torch.equal(eng.buf.x.cpu(), x))
    for l in range(TINY.layers):
        tr = {}
        x = orc.layer_forward(l, x, pos, tr)
        eng._issue_layer(l)
        torch.cuda.synchronize()
        b = eng.buf
        print(f"  L{l}: q {R.rel_err(b.q.cpu().view(B,-1), tr['q'].reshape(B,-1)):.2e} attn {R.rel_err(b.attn.cpu(), tr['attn']):.2e} "
              f"h2 {R.rel_err(b.h.cpu(), tr['h2']):.2e} idx_eq {torch.equal(eng.rws.topk_idx.cpu().long(), tr['topk_idx'])} "
              f"w {R.rel_err(eng.rws.topk_w.cpu(), tr['topk_w']):.2e} x_out {R.rel_err(b.x.cpu(), x):.2e}")
        if not torch.equal(eng.rws.topk_idx.cpu().long(), tr['topk_idx']):
            print("   eng idx", eng.rws.topk_idx.cpu().tolist())
            print("   orc idx", tr['topk_idx'].tolist())
            print("   orc logits", tr['logits'].float()[:2])
        b.x.copy_(x)  # re-sync residual stream so errors do not compound
