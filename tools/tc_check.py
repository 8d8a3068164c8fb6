#!/usr/bin/env python
"""Tensor-core forward (cd_set_forward_mode(3)) vs the FP32 fused forward: bitwise d / idx and the
partials, plus CUDA-event timings of both forwards.  python tools/tc_check.py [configs...]"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1911_05063_b200 import api as cd, synth, _lib

lib = _lib.load()


def run(x, y, mode, tau=0.01, reps=0):
    old = lib.cd_set_forward_mode(mode)
    try:
        out = cd.forward(x, y, tau=tau)
        torch.cuda.synchronize()
        ms = None
        if reps:
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(reps):
                cd.forward(x, y, tau=tau)
            b.record()
            torch.cuda.synchronize()
            ms = a.elapsed_time(b) / reps
        return out, ms
    finally:
        lib.cd_set_forward_mode(old)


cases = sys.argv[1:] or ["c1", "c2", "c3", "rand"]
for name in cases:
    if name == "rand":
        rng = np.random.default_rng(5)
        draws = [(int(rng.integers(1, 4)), int(rng.integers(1, 3000)), int(rng.integers(1, 3000))) for _ in range(8)]
        inputs = [(f"rand{B}x{N}x{M}", synth.uniform_pair(B, N, M, seed=k) if hasattr(synth, "uniform_pair") else
                   synth.shape_pair(B, N, M, config_index=300 + k)) for k, (B, N, M) in enumerate(draws)]
    else:
        inputs = [(name, synth.config_inputs(name))]
    for label, (X, Y) in inputs:
        x, y = torch.from_numpy(np.ascontiguousarray(X)).cuda(), torch.from_numpy(np.ascontiguousarray(Y)).cuda()
        reps = 20 if name in ("c2", "c3") else 0
        (f, fms) = run(x, y, 2, reps=reps)
        (t, tms) = run(x, y, 3, reps=reps)
        ok = [torch.equal(f[k], t[k]) for k in range(4)]
        pe = torch.equal(f[4], t[4])
        nd = int((f[0] != t[0]).sum() + (f[2] != t[2]).sum())
        ni = int((f[1] != t[1]).sum() + (f[3] != t[3]).sum())
        print(f"{label}: d/idx equal {ok} partials equal {pe} (diff d {nd}, idx {ni})"
              + (f"  fused {fms:.3f} ms  tensor {tms:.3f} ms" if reps else ""), flush=True)
