"""Debug: head backward (tcgen05 dH / dW GEMMs) vs torch fp32 matmuls of the same bf16 G."""
import torch, synth, sys
from paper_2605_14220_b200 import tim
DEV = "cuda"
for (N, d, V) in [(256, 256, 512), (300, 256, 5000), (1, 128, 257), (777, 512, 33000)]:
    W = synth.head_weight(V, d, 3, device=DEV)
    ids = synth.token_ids(N, V, 3, device=DEV)
    H = synth.hidden_states(N, d, 3, device=DEV, weight=W, ids=ids, mode="flat")
    gl = torch.randn(N, device=DEV)
    dh, dw = tim.head_backward(H, W, ids, gl)
    # reference through torch autograd on fp32 logits
    Hf = H.float().requires_grad_(True)
    Wf = W.float().requires_grad_(True)
    lp = torch.log_softmax(Hf @ Wf.T, dim=1).gather(1, ids[:, None])[:, 0]
    (lp * gl).sum().backward()
    eh = ((dh - Hf.grad).norm() / Hf.grad.norm()).item()
    ew = ((dw - Wf.grad).norm() / Wf.grad.norm()).item()
    print(f"N={N} d={d} V={V}: rel dH {eh:.2e} dW {ew:.2e}", flush=True)
