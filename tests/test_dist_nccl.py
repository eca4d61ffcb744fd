"""Multi-GPU (NCCL) invariance test: P in {1, 2, 4, 8} ranks, one GPU per rank.

The GPU-count half of the invariance claim (§3.1; BASELINE.json north_star
"bit-identical across batch shapes and GPU counts"): the global batch is cut
into P token shards with cuts inside sequences (tim.shard_range), every rank scores its rows with
tim_logprob, runs tim_correct / tim_ppo_loss with the library's NCCL exchange of exact partials
(tim.Comm), and rank 0 gathers the per-token outputs.  Everything -- logp, entropy, tis_w,
tok_keep, coeff, seq_keep, seq_score, the exact statistics, the PPO losses, histograms and
sequence losses -- must be BITWISE equal to the P = 1 run.  The vocab-parallel head over the same
communicator (tim_logprob_tp: the library's all-gather of slice partials) must equal tim_logprob.

Collected and run whenever >= 2 GPUs are visible (skipped on a 1-GPU box); the host-side logic
of the exchange is also covered at world size 2-3 over gloo on the CPU (test_dist_gloo.py).
"""
import os
import socket
import tempfile

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

N_GPU = torch.cuda.device_count() if torch.cuda.is_available() else 0
WORLDS = [p for p in (1, 2, 4, 8) if p <= N_GPU]
D, V, SEED = 512, 151936, 20260042


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _global_inputs():
    """Partition-independent global batch (host): variable-length sequences, the rollout side as
    the trainer's logp plus a seeded global perturbation vector."""
    import synth
    cu = synth.cu_seqlens(23, 3000, SEED, variable=True)
    n = int(cu[-1])
    mask = synth.resp_mask(cu, 200)
    g = torch.Generator().manual_seed(SEED)
    noise = torch.where(torch.rand(n, generator=g) < 0.5, 0.0, 2e-3 * torch.randn(n, generator=g)).float()
    adv = torch.randn(n, generator=g).float()
    return cu, mask, noise, adv, n


def _worker(rank, world, port, outdir):
    import torch.distributed as dist

    import synth
    from paper_2605_14220_b200 import tim

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    cu, mask, noise, adv, n = _global_inputs()
    a, b = tim.shard_range(n, world, rank)
    W = synth.head_weight(V, D, SEED, device=dev)
    H, ids = synth.global_rows(n, D, V, SEED, a, b, W, device=dev)
    lp, ent = tim.logprob(H, W, ids)
    roll = torch.clamp(lp + noise[a:b].to(dev), max=0.0)
    comm = tim.Comm()
    cfg = tim.CorrectConfig(tis=True, tis_cap=2.0, tok_rs=True, tok_lo=0.5, tok_hi=2.0, seq_rs=tim.SEQ_K3,
                            seq_agg=tim.AGG_MEAN, tau_seq=1e-6)
    res = tim.correct(lp, roll, cu.to(dev), cfg, mask[a:b].to(dev), tok_begin=a, comm=comm)
    pcfg = tim.PPOConfig(eps=0.2, hist_lo=-0.05, hist_hi=0.05, hist_bins=64)
    cur = torch.clamp(lp + 0.01 * noise[a:b].to(dev) * 50, max=0.0)
    ppo = tim.ppo_loss(cur, lp, adv[a:b].to(dev), cu.to(dev), pcfg, coeff=res["coeff"], tok_begin=a, comm=comm)
    # vocab-parallel head over the same communicator: every rank scores the SAME rows (this rank's
    # shard of the batch) against its W shard; the library all-gathers the slice partials
    S_v = tim.vocab_slices(V)
    if S_v % world == 0:
        vb, ve = tim.tp_vocab_range(V, world, rank)
        Hs, ids_s = synth.global_rows(n, D, V, SEED, 0, min(n, 1000), W, device=dev)
        tlp, tent = tim.logprob_tp(Hs, W[vb:ve].clone(), V, ids_s, comm)
        rlp, rent = tim.logprob(Hs, W, ids_s)
        assert torch.equal(tlp.view(torch.int32), rlp.view(torch.int32)), ("tp", world, rank)
        assert torch.equal(tent.view(torch.int32), rent.view(torch.int32)), ("tp", world, rank)
    torch.cuda.synchronize()
    local = {k: v.cpu() for k, v in (("logp", lp), ("entropy", ent), ("tis_w", res["tis_w"]),
                                       ("tok_keep", res["tok_keep"]), ("coeff", res["coeff"]),
                                       ("loss", ppo["loss"]), ("grad", ppo["grad"]), ("clipped", ppo["clipped"]))}
    parts = [None] * world
    dist.all_gather_object(parts, local)
    if rank == 0:
        out = {k: torch.cat([p[k] for p in parts]) for k in local}
        out.update({"seq_keep": res["seq_keep"].cpu(), "seq_score": res["seq_score"].cpu(), "stats": res["stats"],
                    "ppo_seq_loss": ppo["seq_loss"].cpu(), "ppo_hist": ppo["hist"].cpu(), "ppo_stats": ppo["stats"],
                    "cuts": [tim.shard_range(n, world, r) for r in range(world)]})
        torch.save(out, os.path.join(outdir, f"P{world}.pt"))
    comm.close()
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.skipif(N_GPU < 2, reason="needs >= 2 GPUs (one rank per GPU)")
def test_bitwise_equal_across_gpu_counts():
    import torch.multiprocessing as mp
    with tempfile.TemporaryDirectory() as d:
        for P in WORLDS:
            mp.spawn(_worker, args=(P, _free_port(), d), nprocs=P, join=True)
        ref = torch.load(os.path.join(d, "P1.pt"), weights_only=False)
        cu = _global_inputs()[0].numpy()
        for P in WORLDS[1:]:
            got = torch.load(os.path.join(d, f"P{P}.pt"), weights_only=False)
            # the shards really cut sequences
            assert any(int(a) not in set(cu.tolist()) for a, _ in got["cuts"][1:])
            for k in ("logp", "entropy", "tis_w", "coeff", "loss", "grad", "seq_score", "ppo_seq_loss"):
                x, y = ref[k], got[k]
                assert torch.equal(x.view(torch.int32 if x.dtype == torch.float32 else torch.int64),
                                   y.view(torch.int32 if y.dtype == torch.float32 else torch.int64)), (P, k)
            for k in ("tok_keep", "clipped", "seq_keep", "ppo_hist"):
                assert torch.equal(ref[k], got[k]), (P, k)
            assert ref["stats"] == got["stats"] and ref["ppo_stats"] == got["ppo_stats"], P
        assert 0 < ref["stats"]["n_seq_rejected"] < ref["stats"]["n_seq"]
