"""Per-rank time of the vocab-parallel head (NEXT-4) on the C1 batch: one rank's
tim_logprob_tp_partial for tp = 1, 2, 4, 8 (rank 0 and the last rank), the merge of tp ranks'
partials, against tim_logprob.  Single GPU: the all-gather between ranks is not included."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2605_14220_b200 import tim  # noqa: E402


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        out = fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps, out


cfg = synth.CONFIGS["c1"]
N, d, V = cfg.n_tok, cfg.hidden, cfg.vocab
W = synth.head_weight(V, d, cfg.seed, device="cuda")
ids = synth.token_ids(N, V, cfg.seed, device="cuda")
H = synth.hidden_states(N, d, cfg.seed, device="cuda", weight=W, ids=ids, mode="peaked")
full_ms, (lp_ref, _) = timed(lambda: tim.logprob(H, W, ids))
out = {"n_tok": N, "hidden": d, "vocab": V, "logprob_ms": full_ms, "tp": {}}
for tp in (2, 4, 8):
    rows = {}
    parts = []
    for r in range(tp):
        b, e = tim.tp_vocab_range(V, tp, r)
        Ws = W[b:e].contiguous()
        if r in (0, tp - 1):
            ms, part = timed(lambda: tim.logprob_tp_partial(H, Ws, V, tp, r, ids))
            rows[r] = {"rows": e - b, "ms": ms}
        else:
            part = tim.logprob_tp_partial(H, Ws, V, tp, r, ids)
        parts.append(part)
    gathered = torch.cat(parts)
    mms, (lp, _) = timed(lambda: tim.logprob_tp_merge(gathered, N, V, ids))
    same = bool(torch.equal(lp.view(torch.int32), lp_ref.view(torch.int32)))
    worst = max(v["ms"] for v in rows.values())
    out["tp"][tp] = {"ranks": rows, "merge_ms": mms, "bitwise_equal_to_tp1": same,
                     "per_rank_speedup": full_ms / (worst + mms)}
print(json.dumps(out))
