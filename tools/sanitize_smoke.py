#!/usr/bin/env python
"""Small ragged invocations of every C-ABI entry point (for compute-sanitizer memcheck/racecheck)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1911_05063_b200 import api as cd, synth

for (B, N, M) in [(1, 1, 1), (2, 3, 7), (2, 1000, 1030), (1, 2049, 513)]:
    X, Y = synth.uniform_pair(B, N, M, seed=N)
    x, y = torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda()
    d_xy, i_xy, d_yx, i_yx, part = cd.forward(x, y, tau=0.1)
    cd.finalize(part, N, M)
    cd.fscore_from_distances(d_xy, d_yx, 0.1)
    cd.backward(x, y, i_xy, i_yx, g_scalar=1.0, h_scalar=1.0)
    cd.forward(x, y, tau=0.1, q_slice=(0, max(1, N // 2)), r_slice=(M // 3, M))
    cd.forward(x, y, tau=0.1, algorithm="pruned")
    keys = cd.forward_rows(x, y, (0, N), tau=0.1)[2]
    cd.forward_cols(x, y, keys, (0, M), tau=0.1)
    cd.step_host(cd.pinned_copy(X).numpy(), cd.pinned_copy(Y).numpy(), tau=0.1)
    cd.loss_backward(x, y, i_xy, i_yx, torch.full((1,), 0.5, device="cuda"), 0.3, 1.7)
    st = cd.HostStepper(B, N, M, tau=0.1)
    st.step(cd.pinned_copy(X), cd.pinned_copy(Y))
V, F = synth.mesh_batch(2, subdiv=2)
rf, rb = synth.sampling_randoms(2, 777, seed=1)
v, f = torch.from_numpy(V).cuda(), torch.from_numpy(F).cuda()
pts, fi, ba = cd.sample_mesh(v, f, torch.from_numpy(rf).cuda(), torch.from_numpy(rb).cuda())
cd.sample_mesh_backward(f, fi, ba, V.shape[1], torch.ones_like(pts))
d, fi2, cl, ba2, pb, loss = cd.p2s_forward(pts.contiguous(), v, f)
cd.p2s_backward(pts, cl, fi2, ba2, f, V.shape[1], g_scalar=1.0)
cd.p2s_loss_backward(pts, cl, fi2, ba2, f, V.shape[1], torch.ones(1, device="cuda"))
cd.p2s_forward(pts.contiguous(), v, f, algorithm="pruned")                       # incl. the tie re-walk
far = (pts * 4.0 + 2.0).contiguous()
cd.p2s_forward(far, v, f, algorithm="pruned")
# backward both ways round the segment-sort limit, with a single-target segment
for (B, N, M) in [(3, 24576, 5), (1, 24577, 40)]:
    X, Y = synth.uniform_pair(B, N, M, seed=3)
    x, y = torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda()
    ixy = torch.zeros((B, N), dtype=torch.int32, device="cuda")
    iyx = torch.randint(0, N, (B, M), dtype=torch.int32, device="cuda")
    cd.backward(x, y, ixy, iyx, g_scalar=1.0, h_scalar=1.0)
torch.cuda.synchronize()
print("sanitize smoke ok")
