"""Head backward (saved forward state, 14080 tokens) vs the GEMM progress-gate slack, interleaved;
digest of dH / dW must not depend on the slack."""
import hashlib, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2605_14220_b200 import tim  # noqa: E402

d = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
V, n = 151936, 14080
W = synth.head_weight(V, d, 1, device="cuda")
ids = synth.token_ids(n, V, 1, device="cuda")
H = synth.hidden_states(n, d, 1, device="cuda")
gl, ge = torch.randn(n, device="cuda"), torch.randn(n, device="cuda")
_, ent, lse2 = tim.logprob_saved(H, W, ids)
res = {}
for rep in range(3):
    for slack in (0, 8, 32, 128):
        tim.debug_set_gemm_slack(slack)
        tim.head_backward(H, W, ids, gl, ge, saved=(ent, lse2))
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(4):
            dh, dw = tim.head_backward(H, W, ids, gl, ge, saved=(ent, lse2))
        b.record()
        torch.cuda.synchronize()
        dig = hashlib.sha256(dh.cpu().numpy().tobytes() + dw.cpu().numpy().tobytes()).hexdigest()[:16]
        res.setdefault(slack, []).append(a.elapsed_time(b) / 4)
        print(f"d={d} rep {rep} slack {slack}: {a.elapsed_time(b) / 4:.3f} ms  digest {dig}", flush=True)
tim.debug_set_gemm_slack(32)
