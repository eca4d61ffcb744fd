"""Head backward (saved state, 14080 tokens): GEMM slack / L2-policy variants interleaved, with
ncu-free timing and a dH / dW digest that must not change."""
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
VARS = {"s0": (0, (1, 1, 2, 3)), "s32": (32, (1, 1, 2, 3)), "s128": (128, (1, 1, 2, 3)),
        "s32_dwA_normal": (32, (1, 1, 1, 3)), "s128_dwA_normal": (128, (1, 1, 1, 3)),
        "s128_all_normal": (128, (1, 1, 1, 1)), "s32_dhB_last": (32, (1, 3, 2, 3))}
for rep in range(3):
    for name, (slack, pol) in VARS.items():
        tim.debug_set_gemm_slack(slack)
        tim.debug_set_gemm_policy(*pol)
        tim.head_backward(H, W, ids, gl, ge, saved=(ent, lse2))
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(4):
            dh, dw = tim.head_backward(H, W, ids, gl, ge, saved=(ent, lse2))
        b.record()
        torch.cuda.synchronize()
        dig = hashlib.sha256(dh.cpu().numpy().tobytes() + dw.cpu().numpy().tobytes()).hexdigest()[:16]
        print(f"d={d} rep {rep} {name:18s}: {a.elapsed_time(b) / 4:.3f} ms  digest {dig}", flush=True)
