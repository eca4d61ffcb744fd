"""SHA-256 digest of the log-prob / sampling / head-backward outputs on a 65,536-token slice of C1:
two builds that must be bitwise equal print the same digest (TIM_LIBRARY selects the build)."""
import hashlib
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2605_14220_b200 import tim  # noqa: E402

cfg = synth.CONFIGS["c1"]
N = 65536
W = synth.head_weight(cfg.vocab, cfg.hidden, cfg.seed, device="cuda")
ids = synth.token_ids(N, cfg.vocab, cfg.seed, device="cuda")
H = synth.hidden_states(N, cfg.hidden, cfg.seed, device="cuda", weight=W, ids=ids, mode="peaked")
lp, ent = tim.logprob(H, W, ids)
sid, slp, sent = tim.sample(H, W, torch.arange(N, device="cuda") << 32, seed=7)
dh, dw = tim.head_backward(H[:2048], W, ids[:2048], torch.ones(2048, device="cuda"),
                           torch.full((2048,), 0.01, device="cuda"))
h = hashlib.sha256()
for name, t in (("lp", lp), ("ent", ent), ("ids", sid), ("slp", slp), ("sent", sent), ("dh", dh), ("dw", dw)):
    h.update(t.contiguous().view(torch.uint8).cpu().numpy().tobytes())
    print(name, hashlib.sha256(t.contiguous().view(torch.uint8).cpu().numpy().tobytes()).hexdigest()[:12], end=" ")
print("all", h.hexdigest()[:16])
