"""Vocab-parallel (tensor-parallel) head, NEXT-4 (§5: reductions invariant to the
TP degree).  tp ranks are emulated in one process: each runs tim_logprob_tp_partial on its own
contiguous copy of its W shard, the partial blocks are concatenated in rank order (what an
all-gather produces) and merged -- the result must be bit-identical to tim_logprob for every tp."""
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu
DEV = "cuda"


@pytest.mark.parametrize("N,d,V", [(700, 256, 4096), (300, 512, 151936), (1, 64, 2000)])
def test_tp_head_bitwise_equal_for_every_degree(tim, N, d, V):
    W = synth.head_weight(V, d, 5, device=DEV)
    ids = synth.token_ids(N, V, 5, device=DEV)
    H = synth.hidden_states(N, d, 5, device=DEV, weight=W, ids=ids, mode="peaked")
    ref_lp, ref_ent = tim.logprob(H, W, ids)
    S = tim.vocab_slices(V)
    for tp in (1, 2, 4, 8):
        if S % tp:
            continue
        parts = []
        for r in range(tp):
            a, b = tim.tp_vocab_range(V, tp, r)
            parts.append(tim.logprob_tp_partial(H, W[a:b].clone(), V, tp, r, ids))
        lp, ent = tim.logprob_tp_merge(torch.cat(parts), N, V, ids)
        assert torch.equal(lp.view(torch.int32), ref_lp.view(torch.int32)), tp
        assert torch.equal(ent.view(torch.int32), ref_ent.view(torch.int32)), tp
