"""SM clock while the pass kernel runs back to back for ~3 s (nvidia-smi
sampled every 50 ms), plus the clock implied by clock64 vs globaltimer in a
tiny kernel launched between passes.  python tools/clock_probe.py"""
import os
import subprocess
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1704_07669_b200 as P
from paper_1704_07669_b200.synth import config_matrix

a = config_matrix("cfg2", device=torch.device("cuda:0"))
om = P.gaussian_matrix(10000, 60, seed=1)
sk = P.GpuSketch(10000, om, np.float32, rows_hint=a.shape[0])
smi = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,clocks_throttle_reasons.active",
                        "--format=csv,noheader,nounits", "-lms", "50"], stdout=subprocess.PIPE, text=True)
time.sleep(0.3)
t0 = time.time()
n = 0
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ev0.record()
while time.time() - t0 < 3.0:
    for _ in range(20):
        sk.reset()
        sk.push(a, 0, final=True)
        n += 1
    torch.cuda.synchronize()
ev1.record()
torch.cuda.synchronize()
smi.terminate()
out = smi.communicate()[0].strip().splitlines()
clk = [float(l.split(",")[0]) for l in out if l.strip()]
pw = [float(l.split(",")[1]) for l in out if l.strip()]
print(f"{n} passes, {ev0.elapsed_time(ev1) / n:.3f} ms/pass; nvidia-smi sm clock samples: n={len(clk)} "
      f"median {np.median(clk):.0f} min {min(clk):.0f} max {max(clk):.0f} MHz; power median {np.median(pw):.0f} W "
      f"max {max(pw):.0f}; reasons {sorted(set(l.split(',')[2].strip() for l in out if l.strip()))}")
