"""Small-N latency probe: warm clocks first, then interleave token counts, with the small-batch
H staging (tim_debug_set_pad_small) on and off in the same process."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2605_14220_b200 import tim  # noqa: E402

d, V = int(os.environ.get("D", "2048")), 151936
W = synth.head_weight(V, d, 1, device="cuda")
Hbig = synth.hidden_states(256, d, 1, device="cuda")
ids_big = synth.token_ids(256, V, 1, device="cuda")
tim.logprob(Hbig[:1], W, ids_big[:1])      # size the workspace cache for the padded case


def t(N, reps=50):
    H, ids = Hbig[:N], ids_big[:N]
    lp = torch.empty(N, device="cuda")
    ent = torch.empty(N, device="cuda")
    for _ in range(5):
        tim.logprob(H, W, ids, out=(lp, ent))
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    for _ in range(reps):
        tim.logprob(H, W, ids, out=(lp, ent))
    b.record()
    torch.cuda.synchronize()
    return round(a.elapsed_time(b) / reps, 4), lp.clone()


for _ in range(400):          # ~60 ms of warm-up at full clocks
    t(256, 1)
print("rep N pad_on pad_off bitwise_equal")
for rep in range(3):
    for N in (1, 16, 64, 100, 128, 200, 256):
        tim.debug_set_pad_small(True)
        a, la = t(N)
        tim.debug_set_pad_small(False)
        b, lb = t(N)
        print(rep, N, a, b, torch.equal(la.view(torch.int32), lb.view(torch.int32)))
tim.debug_set_pad_small(True)
