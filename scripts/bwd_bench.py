"""Time tim_head_backward (NEXT-3) on a BASELINE head shape and split it into its parts:
forward (tim_logprob), gradient epilogue kernel, and the two cuBLAS GEMMs (estimated from a
torch bf16 matmul of the same shapes).  Prints one JSON line."""
import argparse
import json
import sys
import os

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2605_14220_b200 import tim  # noqa: E402


def timed(fn, iters=5, warm=2):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / iters * 1e-3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=14080)
    ap.add_argument("--d", type=int, default=2048)
    ap.add_argument("--V", type=int, default=151936)
    args = ap.parse_args()
    N, d, V = args.n, args.d, args.V
    W = synth.head_weight(V, d, 1, device="cuda")
    ids = synth.token_ids(N, V, 1, device="cuda")
    H = synth.hidden_states(N, d, 1, device="cuda")
    gl = torch.randn(N, device="cuda")
    ge = torch.randn(N, device="cuda")
    t_bwd = timed(lambda: tim.head_backward(H, W, ids, gl, ge))
    t_fwd = timed(lambda: tim.logprob(H, W, ids))
    G = torch.randn(N, V, device="cuda").to(torch.bfloat16)
    t_dh = timed(lambda: torch.matmul(G, W))
    t_dw = timed(lambda: torch.matmul(G.t(), H))
    gemm = 2.0 * N * V * d
    out = {"n_tok": N, "hidden": d, "vocab": V, "ms_backward": t_bwd * 1e3, "ms_forward": t_fwd * 1e3,
           "ms_torch_dh_gemm": t_dh * 1e3, "ms_torch_dw_gemm": t_dw * 1e3,
           "ms_grad_kernel_est": (t_bwd - t_fwd - t_dh - t_dw) * 1e3,
           "tok_per_s_backward": N / t_bwd,
           "tflops_backward_4gemm": 4 * gemm / t_bwd / 1e12,
           "tflops_forward": gemm / t_fwd / 1e12}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
