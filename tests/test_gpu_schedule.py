"""The forward kernel's unit schedule never touches a row's arithmetic (§3.1 P:202-207,
DESIGN.md U20): the die-aware M-tile groups (pairs on one die of the B200 share an M-tile so its H
tile is cached in one die's L2) must give bitwise the same log-probs, entropies, samples and head
gradients as the cluster-id-order groups."""
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu
DEV = "cuda"


def _bits(t):
    return t.contiguous().view(torch.int32)


def test_die_map_probe_is_sane(tim):
    from paper_2605_14220_b200.tim import debug_die_map
    state, die = debug_die_map()
    assert state in (1, -1)
    if state == 1:
        n = torch.cuda.get_device_properties(0).multi_processor_count
        n1 = sum(die[:256])
        assert 0.3 * n <= n1 <= 0.7 * n


@pytest.mark.parametrize("N", [1024, 70000])
def test_die_groups_bitwise_equal_to_cluster_order(tim, N):
    from paper_2605_14220_b200.tim import debug_set_die_groups
    d, V = 4096, 151936                        # d = 4096: two pairs share each M-tile (G = 2)
    W = synth.head_weight(V, d, 41, device=DEV)
    ids = synth.token_ids(N, V, 41, device=DEV)
    H = synth.hidden_states(N, d, 41, device=DEV, weight=W, ids=ids, mode="peaked")
    keys = torch.arange(N, device=DEV, dtype=torch.int64) << 32
    try:
        debug_set_die_groups(False)
        lp0, ent0 = tim.logprob(H, W, ids)
        s0 = tim.sample(H, W, keys, seed=5)
        debug_set_die_groups(True)
        lp1, ent1 = tim.logprob(H, W, ids)
        s1 = tim.sample(H, W, keys, seed=5)
    finally:
        debug_set_die_groups(True)
    assert torch.equal(_bits(lp0), _bits(lp1)) and torch.equal(_bits(ent0), _bits(ent1))
    assert torch.equal(s0[0], s1[0]) and torch.equal(_bits(s0[1]), _bits(s1[1]))


def test_die_groups_head_backward_bitwise(tim):
    from paper_2605_14220_b200.tim import debug_set_die_groups
    N, d, V = 600, 4096, 151936
    W = synth.head_weight(V, d, 42, device=DEV)
    ids = synth.token_ids(N, V, 42, device=DEV)
    H = synth.hidden_states(N, d, 42, device=DEV, weight=W, ids=ids, mode="peaked")
    g = torch.randn(N, device=DEV, generator=torch.Generator(device=DEV).manual_seed(3))
    try:
        debug_set_die_groups(False)
        a = tim.head_backward(H, W, ids, grad_logp=g)
        debug_set_die_groups(True)
        b = tim.head_backward(H, W, ids, grad_logp=g)
    finally:
        debug_set_die_groups(True)
    assert torch.equal(a[0].view(torch.int32), b[0].view(torch.int32))
    assert torch.equal(a[1].view(torch.int32), b[1].view(torch.int32))
