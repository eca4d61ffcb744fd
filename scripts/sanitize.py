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
