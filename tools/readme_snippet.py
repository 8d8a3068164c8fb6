#!/usr/bin/env python
"""The README usage snippet, executed (kept in sync with README.md)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1911_05063_b200 import api as cd

x = torch.randn(32, 16384, 3, device="cuda", requires_grad=True)   # B x N x 3 fp32
y = torch.randn(32, 16384, 3, device="cuda")                        # B x M x 3 fp32
loss = cd.chamfer(x, y)                  # mean over the batch of (1/N) sum d_xy + (1/M) sum d_yx
loss.backward()                          # argmin held fixed; gradients bit-identical to the fp64 oracle
d_xy, i_xy, d_yx, i_yx, part = cd.forward(x.detach(), y, tau=0.01)   # per-point squared distances + indices
cd_b, loss2, F, P, R = cd.finalize(part, 16384, 16384)               # per-batch CD, loss, F-score@tau
out = cd.forward(x.detach(), y, tau=0.01, algorithm="pruned")        # same results, far fewer pairs
assert torch.equal(out[0], d_xy) and torch.equal(out[3], i_yx)
assert abs(loss.item() - loss2.item()) <= 1e-6 * loss.item(), (loss.item(), loss2.item())
print("ok", loss.item(), float(F.mean()), tuple(x.grad.shape))
