"""tim_sample on the C1 batch (for timing / ncu captures of the sampling twin)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2605_14220_b200 import tim  # noqa: E402

if os.environ.get("TUN"):  # h_policy,w_policy,sleep_waits,sync_slack
    tim.debug_set_tuning(*[int(x) for x in os.environ["TUN"].split(",")])
cfg = synth.CONFIGS[os.environ.get("CFG", "c1")]
W = synth.head_weight(cfg.vocab, cfg.hidden, cfg.seed, device="cuda")
ids = synth.token_ids(cfg.n_tok, cfg.vocab, cfg.seed, device="cuda")
H = synth.hidden_states(cfg.n_tok, cfg.hidden, cfg.seed, device="cuda", weight=W, ids=ids, mode="peaked")
keys = torch.arange(cfg.n_tok, device="cuda", dtype=torch.int64) << 32
reps = int(os.environ.get("REPS", "5"))
for _ in range(2):
    sid, slp, sent = tim.sample(H, W, keys, seed=20260001)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(reps):
    sid, slp, sent = tim.sample(H, W, keys, seed=20260001)
b.record()
torch.cuda.synchronize()
ms = a.elapsed_time(b) / reps
print({"ms": ms, "tokens_per_s": cfg.n_tok / (ms / 1e3), "ids_sum": int(sid.sum()), "lp_sum": float(slp.double().sum())})
