"""The hot path is stream-ordered with caller-owned buffers, no host synchronisation and cached
workspaces, so one step (tim_logprob -> tim_correct -> tim_ppo_loss) can be captured in a CUDA
graph and replayed (launch-bound small batches, e.g. rollout-side scoring).  A replay must
reproduce the eager results bit for bit."""
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu
DEV = "cuda"


def test_step_captured_in_cuda_graph_is_bitwise_identical(tim):
    N_seq, L, d, V = 12, 300, 512, 8192
    cu = synth.cu_seqlens(N_seq, L, 3, variable=True)
    N = int(cu[-1])
    W = synth.head_weight(V, d, 3, device=DEV)
    ids = synth.token_ids(N, V, 3, device=DEV)
    H = synth.hidden_states(N, d, 3, device=DEV, weight=W, ids=ids, mode="peaked")
    mask = synth.resp_mask(cu, 40).to(DEV)
    cu = cu.to(DEV)
    lp0, _ = tim.logprob(H, W, ids)
    lp_roll = synth.perturb_laplace_mix(lp0, 3)
    adv = torch.randn(N, device=DEV, generator=torch.Generator(device=DEV).manual_seed(3))
    cfg = tim.PRESETS["tis-srs-k3-corr-ratio"]
    lp = torch.empty(N, device=DEV)
    ent = torch.empty(N, device=DEV)
    S = cu.numel() - 1
    cout = {"tis_w": torch.empty(N, device=DEV), "tok_keep": torch.empty(N, dtype=torch.uint8, device=DEV),
            "seq_keep": torch.empty(S, dtype=torch.uint8, device=DEV), "coeff": torch.empty(N, device=DEV),
            "seq_score": torch.empty(S, dtype=torch.float64, device=DEV),
            "stats_raw": torch.zeros(tim.STATS_BYTES, dtype=torch.uint8, device=DEV)}
    status = tim.new_status(DEV)
    pp = {}

    def step():
        tim.logprob(H, W, ids, out=(lp, ent), status=status)
        tim.correct(lp, lp_roll, cu, cfg, mask, status=status, return_stats=False, out=cout)
        pp["r"] = tim.ppo_loss(lp, lp_roll, adv, cu, tim.PPOConfig(), coeff=cout["coeff"], return_stats=False)

    step()
    torch.cuda.synchronize()
    ref = {k: v.clone() for k, v in cout.items()}
    ref["lp"], ref["ent"] = lp.clone(), ent.clone()
    ref_pp = {k: v.clone() for k, v in pp["r"].items() if isinstance(v, torch.Tensor)}

    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):  # warm the workspace caches on the capture stream's pool
        step()
    torch.cuda.current_stream().wait_stream(side)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        step()
    for _ in range(2):
        for t in list(cout.values()) + [lp, ent]:
            t.zero_()
        g.replay()
        torch.cuda.synchronize()
        assert tim.read_status(status) == (0, 0)
        assert torch.equal(lp.view(torch.int32), ref["lp"].view(torch.int32))
        assert torch.equal(ent.view(torch.int32), ref["ent"].view(torch.int32))
        for k in cout:
            assert torch.equal(cout[k].view(torch.uint8), ref[k].view(torch.uint8)), k
        for k, v in ref_pp.items():
            assert torch.equal(pp["r"][k].view(torch.uint8), v.view(torch.uint8)), k
