#!/usr/bin/env python
"""Probe of the torch symmetric-memory calls distributed.PeerColKeys makes (one rank, NCCL, one GPU):
allocation, rendezvous, peer pointers, device barrier, and cd_forward_cols_peers reading the buffer
through the pointer the rendezvous returns."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist

os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29555")
dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
import torch.distributed._symmetric_memory as symm
from paper_1911_05063_b200 import api as cd, synth

grp = dist.group.WORLD
if hasattr(symm, "enable_symm_mem_for_group"):
    symm.enable_symm_mem_for_group(grp.group_name)
B, N, M = 2, 3000, 2500
buf = symm.empty(B, M, dtype=torch.int64, device=dev)
h = symm.rendezvous(buf, grp)
ptrs = [int(p) for p in h.buffer_ptrs]
print("buffer_ptrs", len(ptrs), ptrs[0] == buf.data_ptr())
X, Y = synth.shape_pair(B, N, M, config_index=52)
x, y = torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda()
full = cd.forward(x, y, tau=0.01)
cd.forward_rows(x, y, (0, N), tau=0.01, keys=buf)
h.barrier(channel=0)
d, i, _ = cd.forward_cols_peers(x, y, ptrs, (0, M), tau=0.01)
h.barrier(channel=0)
torch.cuda.synchronize()
print("peer resolve equals the full forward:", torch.equal(d, full[2]) and torch.equal(i, full[3]))
dist.destroy_process_group()
