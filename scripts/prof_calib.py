"""Small driver for ncu: one Eq. 3 calibration over N bf16 activations (default 2e9 = 4 GB)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import cats_synth
import paper_2404_08763_b200 as cats

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2_000_000_000
acts = cats_synth.calib_acts(n, torch.bfloat16, seed=0, device="cuda")
t, info = cats.cats_calibrate_threshold(acts, 0.5)
torch.cuda.synchronize()
print(t, info)
