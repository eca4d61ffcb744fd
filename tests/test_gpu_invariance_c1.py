"""Batch invariance at the C1 shape (§3.1 P:202-207 -- the same
token must get bit-identical log-probs whether it is scored alone, as the rollout does, or inside a
large packed batch, as the trainer does).

* The full C1 batch (64 sequences x 4096 tokens, d = 2048, V = 151936) is scored once; packs of
  1, 2, 4, ..., 64 WHOLE sequences (the trainer's micro-batches) are scored separately and must be
  bitwise equal to the full batch on every token.
* 1,024 tokens of the batch are scored one at a time (the rollout's decode-step shape) and must be
  bitwise equal to their values in the full batch.
"""
import pytest
import torch

import synth

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
DEV = "cuda"


def _bits(t):
    return t.contiguous().view(torch.int32)


@pytest.fixture(scope="module")
def c1(tim):
    cfg = synth.CONFIGS["c1"]
    N = cfg.n_seq * cfg.seq_len
    W = synth.head_weight(cfg.vocab, cfg.hidden, cfg.seed, device=DEV)
    ids = synth.token_ids(N, cfg.vocab, cfg.seed, device=DEV)
    H = synth.hidden_states(N, cfg.hidden, cfg.seed, device=DEV, weight=W, ids=ids, mode="peaked")
    lp, ent = tim.logprob(H, W, ids)
    yield cfg, H, W, ids, _bits(lp), _bits(ent)
    del H, W
    torch.cuda.empty_cache()


@pytest.mark.parametrize("pack", [1, 2, 4, 8, 16, 32, 64])
def test_whole_sequence_packs_bitwise_equal_to_full_batch(tim, c1, pack):
    cfg, H, W, ids, ref_lp, ref_ent = c1
    L = cfg.seq_len
    for s0 in range(0, cfg.n_seq, pack):
        a, b = s0 * L, min(cfg.n_seq, s0 + pack) * L
        lp, ent = tim.logprob(H[a:b], W, ids[a:b])
        assert torch.equal(_bits(lp), ref_lp[a:b]), (pack, s0)
        assert torch.equal(_bits(ent), ref_ent[a:b]), (pack, s0)


def test_1024_single_token_calls_bitwise_equal_to_full_batch(tim, c1):
    cfg, H, W, ids, ref_lp, ref_ent = c1
    N = H.shape[0]
    g = torch.Generator().manual_seed(1024)
    rows = torch.randperm(N, generator=g)[:1024].tolist()
    lp1 = torch.empty(1024, dtype=torch.float32, device=DEV)
    ent1 = torch.empty(1024, dtype=torch.float32, device=DEV)
    for j, t in enumerate(rows):
        lp, ent = tim.logprob(H[t:t + 1], W, ids[t:t + 1])
        lp1[j] = lp[0]
        ent1[j] = ent[0]
    idx = torch.tensor(rows, device=DEV)
    assert torch.equal(_bits(lp1), ref_lp[idx])
    assert torch.equal(_bits(ent1), ref_ent[idx])
