"""Latency of tim_logprob / tim_sample for small token counts (rollout-side scoring) at a head shape."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2605_14220_b200 import tim  # noqa: E402

d, V = int(os.environ.get("D", "2048")), 151936
W = synth.head_weight(V, d, 1, device="cuda")
out = {"hidden": d, "vocab": V, "slices": tim.vocab_slices(V), "ms": {}}
for N in (1, 16, 64, 256, 1024, 4096, 16384):
    ids = synth.token_ids(N, V, 1, device="cuda")
    H = synth.hidden_states(N, d, 1, device="cuda")
    lp = torch.empty(N, device="cuda")
    ent = torch.empty(N, device="cuda")
    for _ in range(3):
        tim.logprob(H, W, ids, out=(lp, ent))
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    for _ in range(20):
        tim.logprob(H, W, ids, out=(lp, ent))
    b.record()
    torch.cuda.synchronize()
    out["ms"][N] = round(a.elapsed_time(b) / 20, 4)
print(json.dumps(out))
