"""The bench's C2 step (tim_logprob + tim_correct on the strong-scaling workload) repeated K times:
per-step log-prob kernel time (events on the launching stream) and the progress gates given up in
that launch (workspace diagnostics word).  argv: K [sync_slack]; env TUN=h,w,sleep,slack and DEMOTE=0/1 set the schedule knobs"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import synth
from paper_2605_14220_b200 import tim

K = int(sys.argv[1]) if len(sys.argv) > 1 else 12
if len(sys.argv) > 2:
    tim.debug_set_tuning(0, 0, 0, int(sys.argv[2]))
if os.environ.get("TUN"):  # h_policy,w_policy,sleep_waits,sync_slack
    tim.debug_set_tuning(*[int(x) for x in os.environ["TUN"].split(",")])
if os.environ.get("PERSIST") or os.environ.get("QUERY"):
    # cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, PERSIST MB); QUERY=1 only prints it
    import ctypes
    torch.cuda.init()
    torch.empty(1, device="cuda")  # the primary context exists before the limit is set
    rt = ctypes.CDLL("libcudart.so.12")
    lim0 = ctypes.c_size_t(0)
    rt.cudaDeviceGetLimit(ctypes.byref(lim0), 6)
    print(f"persisting L2 limit before: {lim0.value} B")
if os.environ.get("PERSIST"):
    mx = ctypes.c_int(0)
    rt.cudaDeviceGetAttribute(ctypes.byref(mx), 108, 0)  # cudaDevAttrMaxPersistingL2CacheSize
    want = min(int(os.environ["PERSIST"]) << 20, mx.value)
    err = rt.cudaDeviceSetLimit(6, ctypes.c_size_t(want))  # cudaLimitPersistingL2CacheSize
    lim = ctypes.c_size_t(0)
    rt.cudaDeviceGetLimit(ctypes.byref(lim), 6)
    print(f"persisting L2 limit: max {mx.value >> 20} MB, set {want >> 20} MB, err {err}, now {lim.value >> 20} MB")
if os.environ.get("DEMOTE"):
    tim.debug_set_schedule(0, os.environ["DEMOTE"] == "1")
dev = torch.device("cuda")
cfg = synth.CONFIGS[os.environ.get("CFG", "c2")]
W, H, ids, tb, cu, mask, n_glob = bench.build_workload(cfg, "strong", 1, 0, dev)
N = H.shape[0]
lp = torch.empty(N, device=dev)
ent = torch.empty(N, device=dev)
lp0, _ = tim.logprob(H, W, ids)
lp_roll = synth.perturb_laplace_mix(lp0, cfg.seed)
ccfg = tim.PRESETS["tis-srs-k3-corr-ratio"]
cur = torch.cuda.current_stream(dev)
ms = []
for k in range(K):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(cur)
    tim.logprob(H, W, ids, out=(lp, ent))
    b.record(cur)
    tim.correct(lp, lp_roll, cu, ccfg, mask, return_stats=False)
    torch.cuda.synchronize()
    ws = [v for kk, v in tim._ws_cache.items() if kk[2] == "logprob"][0]
    gates = int(ws[:64].view(torch.int64)[7].item())
    ms.append(a.elapsed_time(b))
    print(f"step {k}: {ms[-1]:.1f} ms  {N / ms[-1] * 1e3 / 1e6:.4f} Mtok/s  gates_given_up={gates}", flush=True)
s = sorted(ms)
print(f"median {s[len(s) // 2]:.1f} ms  min {s[0]:.1f}  max {s[-1]:.1f}  mean {sum(ms) / len(ms):.1f}")
