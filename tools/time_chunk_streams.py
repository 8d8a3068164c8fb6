#!/usr/bin/env python
"""Experiment: the e2e step's batch-range structure on the device alone (no copies): forward +
loss backward of ranges [4, 12, 12, 4] of c3 on one stream vs alternating over two streams (the next
range's fused kernel filling the previous range's tail wave), graph-captured, L2 flushed."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1911_05063_b200 import api as cd, synth

X, Y = synth.config_inputs("c3")
x, y = torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda()
one = torch.ones(1, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
B = 32


def make(bounds, nstreams):
    streams = [torch.cuda.Stream() for _ in range(nstreams)]

    def step():
        main = torch.cuda.current_stream()
        for s in streams:
            s.wait_stream(main)
        for i in range(len(bounds) - 1):
            s = streams[i % nstreams]
            with torch.cuda.stream(s):
                xs, ys = x[bounds[i]:bounds[i + 1]], y[bounds[i]:bounds[i + 1]]
                d_xy, i_xy, d_yx, i_yx, part = cd.forward(xs, ys, tau=0.01)
                cd.loss_backward(xs, ys, i_xy, i_yx, one)
        for s in streams:
            main.wait_stream(s)
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
    return ts[len(ts) // 2]


for bounds in ([0, 32], [0, 4, 16, 28, 32], [0, 8, 16, 24, 32], [0, 2, 10, 18, 26, 30, 32]):
    for ns in (1, 2):
        if ns > len(bounds) - 1:
            continue
        print(bounds, "streams", ns, "median ms %.4f" % timeit(make(bounds, ns)), flush=True)
