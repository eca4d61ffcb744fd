"""C2-shaped tim_logprob and tim_sample calls (for ncu metric comparisons of the two kernels)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2605_14220_b200 import tim  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 524288
d, V = int(os.environ.get("D", "4096")), 151936
W = synth.head_weight(V, d, 2, device="cuda")
ids = synth.token_ids(n, V, 2, device="cuda")
H = synth.hidden_states(n, d, 2, device="cuda", weight=W, ids=ids, mode="peaked")
keys = torch.arange(n, device="cuda", dtype=torch.int64) << 32
for _ in range(2):
    for name, fn in (("logprob", lambda: tim.logprob(H, W, ids)), ("sample", lambda: tim.sample(H, W, keys, seed=7))):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        print(f"{name}: {a.elapsed_time(b):.1f} ms {n / a.elapsed_time(b) * 1e3 / 1e6:.4f} Mtok/s", flush=True)
