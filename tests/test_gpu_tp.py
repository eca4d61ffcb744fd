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


def test_tp_head_in_library_collective_single_rank(tim):
    """tim_logprob_tp: partial + the library's NCCL all-gather of the slice partials + merge, on a
    libtim-owned communicator (world size 1 on this one-GPU box; the P >= 2 case runs in
    test_dist_nccl.py when several GPUs are visible): bitwise equal to tim_logprob."""
    import os
    import torch.distributed as dist
    own = not dist.is_initialized()
    if own:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29534")
        dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        comm = tim.Comm()
        N, d, V = 513, 512, 151936
        W = synth.head_weight(V, d, 6, device=DEV)
        ids = synth.token_ids(N, V, 6, device=DEV)
        H = synth.hidden_states(N, d, 6, device=DEV, weight=W, ids=ids, mode="peaked")
        ref_lp, ref_ent = tim.logprob(H, W, ids, temperature=0.8)
        lp, ent = tim.logprob_tp(H, W, V, ids, comm, temperature=0.8)
        assert torch.equal(lp.view(torch.int32), ref_lp.view(torch.int32))
        assert torch.equal(ent.view(torch.int32), ref_ent.view(torch.int32))
        with pytest.raises(ValueError):
            tim.logprob_tp(H, W[:-256], V, ids, comm)
        comm.close()
    finally:
        if own:
            dist.destroy_process_group()
