"""Standalone tim_ppo_loss at N tokens (bench.ppo_roofline), for timing and ncu captures."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2605_14220_b200 import tim
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 27
peaks, src = bench._peaks()
print(bench.ppo_roofline(tim, torch.device("cuda"), n, peaks, src, reps=int(os.environ.get("REPS", "10"))))
