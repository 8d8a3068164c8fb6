#!/usr/bin/env python
"""Per-rank work of a G-GPU run, timed on one GPU (device time, no collectives), and the efficiency
t(G = 1) / (G t(G)):
  batch sharding (default): forward (brute) + backward of the config's first B / G batch elements;
  query sharding (SHARD=query, the c5 design of distributed.query_sharded_step): rank 0's fused
  rows forward over X rows [0, N / G) against all of Y (column keys for every Y point), the column
  resolve of its Y rows [0, M / G) and the sliced backward.
python tools/time_batch_shard.py [c4] [G ...]"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1911_05063_b200 import api as cd, synth

cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
gs = [int(g) for g in sys.argv[2:]] or [1, 2, 4, 8]
Bfull = synth.CONFIGS[cfg]["B"]
tau = synth.CONFIGS[cfg]["tau"]
query = os.environ.get("SHARD") == "query"
t1 = None
if query:
    X, Y = synth.config_inputs(cfg)
    x, y = torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda()
    Bq, N, M = X.shape[0], X.shape[1], Y.shape[1]
    # the all-gathered indices a rank's backward reads (one full exact forward, outside the timing)
    _, i_xy_full, _, i_yx_full, _ = cd.forward(x, y, tau=tau, algorithm="pruned")
for G in gs:
    if query:
        B = Bq
        q, r = (0, N // G), (0, M // G)

        def step():
            d_xy, i_xy, keys, part = cd.forward_rows(x, y, q, tau=tau)
            d_yx, i_yx, part = cd.forward_cols(x, y, keys, r, tau=tau, partials=part)
            cd.backward(x, y, i_xy_full, i_yx_full, g_scalar=1.0 / (B * N), h_scalar=1.0 / (B * M), q_slice=q,
                        r_slice=r)
    else:
        B = Bfull // G
        X, Y = synth.config_inputs(cfg, B=B)
        x, y = torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda()

        def step():
            d_xy, i_xy, d_yx, i_yx, part = cd.forward(x, y, tau=tau)
            cd.backward(x, y, i_xy, i_yx, g_scalar=1.0 / (B * X.shape[1]), h_scalar=1.0 / (B * Y.shape[1]))

    for _ in range(1 if cfg == "c5" else 3):
        step()
    torch.cuda.synchronize()
    reps = 1 if cfg == "c5" else max(2, 40 // (Bfull // G))
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        step()
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / reps
    if G == 1:
        t1 = ms
    eff = (t1 / (G * ms)) if t1 else float("nan")
    print(f"{cfg} {'query' if query else 'batch'} G={G} B_local={B} step_ms={ms:.4f} efficiency_vs_G1={eff:.4f}", flush=True)
