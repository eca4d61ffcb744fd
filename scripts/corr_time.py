"""Interleavable timing of the correction pass at N tokens (bench.correction_roofline's inputs):
median event time of the whole tim_correct and of pass 1 alone (tim_correct_local)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2605_14220_b200 import tim  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 27
reps = int(os.environ.get("REPS", "20"))
dev = torch.device("cuda")
S = n // 4096
cu = synth.cu_seqlens(S, 4096).to(dev)
g = torch.Generator(device=dev)
g.manual_seed(20260004)
den = -torch.empty(n, device=dev).exponential_(0.7, generator=g)
num = synth.perturb_laplace_mix(den, 20260004)
mask = (torch.arange(n, device=dev) % 4096 >= 1024).to(torch.uint8)
cfg = tim.PRESETS["tis-srs-k3-corr-ratio"]
if os.environ.get("SPLIT") and hasattr(tim, "debug_set_correct_split"):
    tim.debug_set_correct_split(os.environ["SPLIT"] == "1")
out = {"tis_w": torch.empty(n, dtype=torch.float32, device=dev),
       "tok_keep": torch.empty(n, dtype=torch.uint8, device=dev),
       "seq_keep": torch.empty(S, dtype=torch.uint8, device=dev),
       "coeff": torch.empty(n, dtype=torch.float32, device=dev),
       "seq_score": torch.empty(S, dtype=torch.float64, device=dev),
       "stats_raw": torch.zeros(tim.STATS_BYTES, dtype=torch.uint8, device=dev)}


def med(fn):
    for _ in range(3):
        fn()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for a, b in evs:
        a.record()
        fn()
        b.record()
    torch.cuda.synchronize()
    return sorted(a.elapsed_time(b) for a, b in evs)[reps // 2]


full = med(lambda: tim.correct(num, den, cu, cfg, mask, return_stats=False, out=out))
local = med(lambda: tim.correct_local(num, den, cu, cfg, mask))
print(f"full_ms {full:.4f} local_ms {local:.4f} full_GBps_18B {18 * n / full / 1e6:.1f} "
      f"local_GBps_18B {18 * n / local / 1e6:.1f}")
