"""One tim_head_backward_saved call on a BASELINE head shape (for ncu captures of the gradient
pass and the two tcgen05 GEMMs)."""
import argparse, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2605_14220_b200 import tim  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=14080)
ap.add_argument("--d", type=int, default=2048)
ap.add_argument("--reps", type=int, default=1)
a = ap.parse_args()
V = 151936
W = synth.head_weight(V, a.d, 1, device="cuda")
ids = synth.token_ids(a.n, V, 1, device="cuda")
H = synth.hidden_states(a.n, a.d, 1, device="cuda")
gl, ge = torch.randn(a.n, device="cuda"), torch.randn(a.n, device="cuda")
_, ent, lse2 = tim.logprob_saved(H, W, ids)
for _ in range(a.reps):
    tim.head_backward(H, W, ids, gl, ge, saved=(ent, lse2))
torch.cuda.synchronize()
