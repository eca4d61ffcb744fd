"""Small invocations of every kernel for compute-sanitizer (memcheck / racecheck / synccheck)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
from paper_2605_14220_b200 import tim

dev = torch.device("cuda")
cfg = synth.CONFIGS["toy"]
W = synth.head_weight(1000, 256, 1, device=dev)
ids = synth.token_ids(300, 1000, 1, device=dev)
H = synth.hidden_states(300, 256, 1, device=dev, weight=W, ids=ids, mode="peaked")
lp, ent = tim.logprob(H, W, ids)
sid, slp, sent = tim.sample(H, W, torch.arange(300, device=dev), seed=5)
g = torch.ones(256, dtype=torch.bfloat16, device=dev)
x = tim.rmsnorm(H, g)
cu = synth.cu_seqlens(3, 100).to(dev)
mask = synth.resp_mask(cu.cpu(), 10).to(dev)
roll = synth.perturb_laplace_mix(lp, 3)
res = tim.correct(lp, roll, cu, tim.PRESETS["tis-srs-k3-corr-ratio"], mask)
pp = tim.ppo_loss(lp, roll, torch.randn(300, device=dev), cu, tim.PPOConfig(), coeff=res["coeff"])
dh, dw = tim.head_backward(H, W, ids, torch.ones(300, device=dev), torch.full((300,), 0.01, device=dev))
lps, ents, lse2 = tim.logprob_saved(H, W, ids)
dh2, dw2 = tim.head_backward(H, W, ids, torch.ones(300, device=dev), saved=(ents, lse2))
lp5, _ = tim.logprob(H[:5], W, ids[:5])                       # small-batch H staging (pad_rows_kernel)
torch.cuda.synchronize()
print("sanitize run ok", float(lp.sum()), res["stats"]["n_seq_rejected"], pp["stats"]["n_clipped"], float(dh.abs().sum()))
# a larger correction / PPO call: several chunks per warp, so the per-warp TMA ring of the
# correction kernel wraps around (stages refilled), with variable-length sequences
cu2 = synth.cu_seqlens(256, 16384, variable=True, seed=11).to(dev)
n2 = int(cu2[-1])
den2 = -torch.rand(n2, device=dev) * 3
num2 = synth.perturb_laplace_mix(den2, 12)
mask2 = (torch.rand(n2, device=dev) > 0.2).to(torch.uint8)
res2 = tim.correct(num2, den2, cu2, tim.PRESETS["tis-srs-k3-corr-ratio"], mask2)
pp2 = tim.ppo_loss(num2, den2, torch.randn(n2, device=dev), cu2, tim.PPOConfig(), coeff=res2["coeff"])
torch.cuda.synchronize()
print("sanitize large run ok", n2, res2["stats"]["n_seq_rejected"], pp2["stats"]["n_clipped"])
# round 2: the fused one-launch correction (grid barriers), the d = 4096 head with die-aware
# M-tile groups (G = 2, the per-device die probe, shared::cluster id exchange), the TP head's
# library collective on a 1-rank communicator
tim.debug_set_correct_split(False)
res3 = tim.correct(num2, den2, cu2, tim.PRESETS["tis-srs-k3-corr-ratio"], mask2)
tim.debug_set_correct_split(True)
W4 = synth.head_weight(151936, 4096, 2, device=dev)
ids4 = synth.token_ids(600, 151936, 2, device=dev)
H4 = synth.hidden_states(600, 4096, 2, device=dev, weight=W4, ids=ids4, mode="peaked")
lp4, _ = tim.logprob(H4, W4, ids4)
import torch.distributed as dist
os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29541")
dist.init_process_group("gloo", rank=0, world_size=1)
comm = tim.Comm()
lpt, _ = tim.logprob_tp(H, W, 1000, ids, comm)
comm.close()
dist.destroy_process_group()
torch.cuda.synchronize()
print("sanitize round-2 run ok", int(res3["stats"]["n_seq_rejected"]), float(lp4.sum()), bool(torch.equal(lpt, lp)))
