#!/usr/bin/env python
"""Experiment: c3 step as one stream vs the batch split in k parts on k streams (fork/join inside one
CUDA graph), so one part's epilogue / backward fills the tail waves of another part's fused forward.
usage: python tools/time_overlap.py [config] [splits-forced]"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1911_05063_b200 import api as cd, synth

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
X, Y = synth.config_inputs(cfg)
c = synth.CONFIGS[cfg]
B, N, M, tau = c["B"], c["N"], c["M"], c["tau"]
x, y = torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda()
one = torch.ones(1, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def part_step(xs, ys):
    d_xy, i_xy, d_yx, i_yx, part = cd.forward(xs, ys, tau=tau)
    gx, gy = cd.loss_backward(xs, ys, i_xy, i_yx, one)
    return part, gx, gy


def make(k):
    streams = [torch.cuda.Stream() for _ in range(k)]
    bounds = [B * i // k for i in range(k + 1)]

    def step():
        main = torch.cuda.current_stream()
        parts = []
        for i, s in enumerate(streams):
            s.wait_stream(main)
            with torch.cuda.stream(s):
                parts.append(part_step(x[bounds[i]:bounds[i + 1]], y[bounds[i]:bounds[i + 1]]))
        for s in streams:
            main.wait_stream(s)
        part = torch.cat([p[0] for p in parts])
        return cd.finalize(part, N, M)[1]
    return step


def timeit(step, K=50):
    for _ in range(3):
        step()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        step()
    g.replay()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    for i in range(K):
        flush.fill_(i & 255)
        ev[i][0].record()
        g.replay()
        ev[i][1].record()
    torch.cuda.synchronize()
    ts = sorted(a.elapsed_time(b) for a, b in ev)
    return ts[len(ts) // 2], sum(ts) / len(ts)


for forced in ([int(v) for v in sys.argv[2:]] or [0]):
    cd.set_forward_splits(forced)
    for k in (1, 2, 4):
        med, mean = timeit(make(k))
        print(f"{cfg} splits={forced or 'auto'} streams={k}: median {med:.4f} ms mean {mean:.4f} ms", flush=True)
cd.set_forward_splits(0)
