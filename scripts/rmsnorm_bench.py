"""tim_rmsnorm bandwidth and tim_logprob_rmsnorm vs tim_logprob on the C1 batch (NEXT-4)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2605_14220_b200 import tim  # noqa: E402


def timed(fn, reps=10):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


cfg = synth.CONFIGS["c1"]
N, d, V = cfg.n_tok, cfg.hidden, cfg.vocab
W = synth.head_weight(V, d, cfg.seed, device="cuda")
ids = synth.token_ids(N, V, cfg.seed, device="cuda")
H = synth.hidden_states(N, d, cfg.seed, device="cuda")
g = (1.0 + 0.1 * torch.randn(d, device="cuda")).to(torch.bfloat16)
rms_ms = timed(lambda: tim.rmsnorm(H, g))
lp_ms = timed(lambda: tim.logprob(H, W, ids), reps=3)
lpr_ms = timed(lambda: tim.logprob_rmsnorm(H, g, W, ids), reps=3)
bytes_ = N * d * 2 * 2 + d * 2          # read h, write out (bf16), gamma
print(json.dumps({"n_tok": N, "hidden": d, "rmsnorm_ms": rms_ms, "rmsnorm_gbs": bytes_ / rms_ms / 1e6,
                  "algorithmic_bytes_per_token": 4 * d, "logprob_ms": lp_ms, "logprob_rmsnorm_ms": lpr_ms,
                  "prologue_share": (lpr_ms - lp_ms) / lpr_ms}))
