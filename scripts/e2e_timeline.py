"""Timeline of the host-input path (tim.logprob with pinned host H, C2 batch): CUDA events on the
copy stream (each H2D chunk) and on the compute stream (each chunk's tim_logprob), relative to the
first event, to show the copies hiding under the kernels (no nsys in this image)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import synth
from paper_2605_14220_b200 import tim

dev = torch.device("cuda")
cfg = synth.CONFIGS[os.environ.get("CFG", "c2")]
W, H, ids, tb, cu, mask, n_glob = bench.build_workload(cfg, "strong", 1, 0, dev)
Hh = H.cpu().pin_memory()
idsh = ids.cpu()
del H
torch.cuda.synchronize()
tim.logprob(Hh, W, idsh, device=dev)  # warm-up (workspaces, copy stream)
torch.cuda.synchronize()

# the same schedule as tim._logprob_from_host, with events around every copy and every launch
N, d = Hh.shape
cs = tim._copy_streams[str(dev)]
if os.environ.get("COMP") == "new":  # the kernels on a created (non-default) stream
    torch.cuda.set_stream(torch.cuda.Stream(dev))
comp = torch.cuda.current_stream(dev)
hd = torch.empty(N, d, dtype=torch.bfloat16, device=dev)
ids_d = idsh.to(dev)
lp = torch.empty(N, device=dev)
ent = torch.empty(N, device=dev)
cuts, a, step = [0], 0, tim._HOST_FIRST
while a < N:
    a = min(N, a + step)
    cuts.append(a)
    step = min(2 * step, tim._HOST_CHUNK)
ev = lambda: torch.cuda.Event(enable_timing=True)
t0 = ev()
t0.record(comp)
cs.wait_stream(comp)
cp_ev, k_ev = [], []


def copy(a, b):
    with torch.cuda.stream(cs):
        s, e = ev(), ev()
        s.record(cs)
        hd[a:b].copy_(Hh[a:b], non_blocking=True)
        e.record(cs)
        cp_ev.append((s, e))


def kernel(a, b, e_cp):
    comp.wait_event(e_cp)
    s, e = ev(), ev()
    s.record(comp)
    tim.logprob(hd[a:b], W, ids_d[a:b], out=(lp[a:b], ent[a:b]))
    e.record(comp)
    k_ev.append((s, e))


pairs = list(zip(cuts[:-1], cuts[1:]))
import time
print(f"# Hh pinned: {Hh.is_pinned()}, slice pinned: {Hh[8:16].is_pinned()}, comp {comp.cuda_stream:#x}, copy stream {cs.cuda_stream:#x}")
th0 = time.perf_counter()
if os.environ.get("ORDER") == "interleaved":  # copy i + 1 enqueued before kernel i
    copy(*pairs[0])
    for i, (a, b) in enumerate(pairs):
        if i + 1 < len(pairs):
            copy(*pairs[i + 1])
        kernel(a, b, cp_ev[i][1])
else:  # the library's order: every copy first, then the kernels
    for a, b in pairs:
        copy(a, b)
    for i, (a, b) in enumerate(pairs):
        kernel(a, b, cp_ev[i][1])
print(f"# host enqueue time {1e3 * (time.perf_counter() - th0):.1f} ms")
t1 = ev()
t1.record(comp)
torch.cuda.synchronize()
print(f"# host-input path, {cfg.name}: {N} rows in {len(cuts) - 1} chunks, H {N * d * 2 / 1e9:.2f} GB pinned host -> device")
print("# chunk  rows        H2D copy [start, end] ms      tim_logprob [start, end] ms")
for i, ((a, b), (s1, e1), (s2, e2)) in enumerate(zip(zip(cuts[:-1], cuts[1:]), cp_ev, k_ev)):
    print(f"  {i:3d}  {b - a:8d}   [{t0.elapsed_time(s1):9.2f}, {t0.elapsed_time(e1):9.2f}]   "
          f"[{t0.elapsed_time(s2):9.2f}, {t0.elapsed_time(e2):9.2f}]")
tot = t0.elapsed_time(t1)
cpy = sum(s.elapsed_time(e) for s, e in cp_ev)
ker = sum(s.elapsed_time(e) for s, e in k_ev)
print(f"# total {tot:.1f} ms; copies {cpy:.1f} ms ({N * d * 2 / cpy / 1e6:.1f} GB/s), kernels {ker:.1f} ms; "
      f"exposed (total - kernels) {tot - ker:.1f} ms")
