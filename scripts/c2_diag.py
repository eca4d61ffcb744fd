"""C2-shaped tim_logprob calls: time per call and the number of progress gates that timed out
(diagnostics word in the workspace header).  argv: n_tok tuning(h,w,sleep,slack[,group]) reps"""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2605_14220_b200 import tim  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2097152
tun = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 and sys.argv[2] != "default" else None
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
d, V = int(os.environ.get("D", "4096")), 151936
if os.environ.get("MAXP"):
    tim.debug_set_kernel(True, int(os.environ["MAXP"]))
if os.environ.get("DIEG") is not None and hasattr(tim, "debug_set_die_groups"):
    tim.debug_set_die_groups(os.environ["DIEG"] == "1")
if tun:
    tim.debug_set_tuning(*tun[:4])
    if len(tun) > 4:
        tim.debug_set_schedule(tun[4], 0)
W = synth.head_weight(V, d, 2, device="cuda")
ids = synth.token_ids(n, V, 2, device="cuda")
H = synth.hidden_states(n, d, 2, device="cuda", weight=W, ids=ids, mode="peaked")
lp = torch.empty(n, device="cuda")
ent = torch.empty(n, device="cuda")
for r in range(reps):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    tim.logprob(H, W, ids, out=(lp, ent))
    b.record()
    torch.cuda.synchronize()
    ws = [v for k, v in tim._ws_cache.items() if k[2] == "logprob"][0]
    gates_off = int(ws[:64].view(torch.int64)[7].item())   # WsHeader.reserved[5]
    print(f"tuning={sys.argv[2] if len(sys.argv) > 2 else 'default'} rep {r}: {a.elapsed_time(b):.1f} ms "
          f"{n / a.elapsed_time(b) * 1e3 / 1e6:.4f} Mtok/s gates_timed_out={gates_off}", flush=True)
