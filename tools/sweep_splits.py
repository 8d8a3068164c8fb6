#!/usr/bin/env python
"""Time the fused forward (cd_forward) for several forced split counts (design data for choose_splits)."""
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1911_05063_b200 import api as cd, synth

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
splits = [int(s) for s in sys.argv[2].split(",")] if len(sys.argv) > 2 else [0, 1, 2, 3, 4, 5, 6, 8, 10, 12, 16, 20, 24, 32]
# SWEEP_B=k: the config's first k batch elements (one rank's share of batch sharding)
X, Y = synth.config_inputs(cfg, B=int(os.environ["SWEEP_B"]) if os.environ.get("SWEEP_B") else None)
x, y = torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda()
tau = synth.CONFIGS[cfg]["tau"]
reps = 20 if cfg in ("c1", "c2", "c3") else 3
for s in splits:
    cd.set_forward_splits(s)
    for _ in range(2):
        cd.forward(x, y, tau=tau)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); b.record()
    tot = 0.0
    for _ in range(reps):
        cd.set_profile_events(a, b)
        cd.forward(x, y, tau=tau)
        cd.set_profile_events(None, None)
        torch.cuda.synchronize()
        tot += a.elapsed_time(b)
    print(f"{cfg} splits={s:3d} fused_kernel_ms={tot / reps:.4f}", flush=True)
cd.set_forward_splits(0)
