"""Sampling twin (C1) and forward under schedule knobs (tim_debug_set_tuning: W-window slack,
sleeping waits), interleaved in one process.  Results never change (ids_sum printed)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2605_14220_b200 import tim  # noqa: E402

cfg = synth.CONFIGS["c1"]
W = synth.head_weight(cfg.vocab, cfg.hidden, cfg.seed, device="cuda")
ids = synth.token_ids(cfg.n_tok, cfg.vocab, cfg.seed, device="cuda")
H = synth.hidden_states(cfg.n_tok, cfg.hidden, cfg.seed, device="cuda", weight=W, ids=ids, mode="peaked")
keys = torch.arange(cfg.n_tok, device="cuda", dtype=torch.int64) << 32


def timed(fn, reps=4):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        out = fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps, out


knobs = [tuple(int(x) for x in k.split(",")) for k in os.environ.get("KNOBS", "3,2,0,4 3,2,1,4 3,2,0,0 3,2,0,16 3,2,0,2").split()]
for rep in range(2):
    for k in knobs:
        tim.debug_set_tuning(*k)
        ms, (sid, _, _) = timed(lambda: tim.sample(H, W, keys, seed=20260001))
        fms, _ = timed(lambda: tim.logprob(H, W, ids))
        print(rep, "h,w,sleep,slack=%s" % (k,), "sample %.4f M" % (cfg.n_tok / ms / 1e3), "fwd %.4f M" % (cfg.n_tok / fms / 1e3),
              int(sid.sum()))
tim.debug_set_tuning(3, 2, 0, 4)
