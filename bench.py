#!/usr/bin/env python
"""bench.py — Chamfer fwd+bwd point-pairs/s on B200 (BASELINE.json metric), one JSON line.

A step is one pass of the whole hot path: cd_forward (both NN
directions + F-score hit counting at tau) -> [all-reduce of the B x 4 partials when N > 1] ->
cd_finalize (CD_b, loss, F) -> cd_backward of the loss (argmin fixed), all through the C ABI.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3] [--impl ours|reference]

Default workload on 1 GPU: config c3 (B=32, N=M=16,384, F-score at tau=0.01) — the largest
BASELINE.json config without a multi-GPU designation and the one naming F@0.01.  --gpus N > 1
(under torchrun) defaults to c5 (B=4, N=M=2^20) query-sharded across the ranks: STRONG scaling of
the north star's largest config (clouds broadcast from rank 0, X rows split, one MIN all-reduce of
the column keys, one partials all-reduce, all-gather of the index slices for the backward).
--config c4 splits its B=8 batch elements over the ranks (strong); other configs run their full
batch on every rank (weak).  For N > 1 the line also carries the same config on ONE GPU (rank 0
alone: the scaling fraction value_N / (N value_1)), the time inside collectives (max over ranks),
and c3 weak scaling (multi_gpu.c3_weak).  Inputs are seeded synthetic
ShapeNet-like clouds.  Timing: W untimed warm-up steps; K timed steps, each
bracketed by CUDA events on the launching stream with an L2 flush (256 MiB write) between steps
outside the events; barrier + synchronize on both sides; max over ranks.

--impl reference times the CPU oracle (oracle/, fp64 brute force) on the host cores on bounded
row samples of the same workload (the tier's reference arm; there is no installable reference).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_1911_05063_b200 import synth  # noqa: E402

METRIC = "Chamfer fwd+bwd point-pairs/sec at 1/2/4/8 B200; % of FP32 FMA peak"
UNIT = "directed point-pairs/s"
FP32_OPS_PER_PAIR = 6        # 3 FADD + 1 FMUL + 2 FFMA per directed pair
FLOPS_PER_PAIR = 8           # the same counting an FMA as 2 flops
SM_MAX_MHZ_FALLBACK = 1965.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None, help="timed steps (default: ~1 s of work per config)")
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default=None, choices=sorted(synth.CONFIGS),
                    help="default: c3 on 1 GPU; c5 (query-sharded strong scaling) on N > 1 GPUs")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="budget of the cpu_baseline oracle sample")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--colkey-exchange", choices=("nccl", "peer"), default="nccl",
                    help="query sharding's column-key exchange: NCCL all-reduce MIN, or peer reads of "
                         "symmetric-memory key arrays reduced inside the resolve kernel")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-clocks", action="store_true")
    ap.add_argument("--quiet", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="launch eagerly instead of replaying a CUDA graph")
    ap.add_argument("--no-pruned", action="store_true", help="skip the exact pruned (NEXT-2) comparison")
    ap.add_argument("--no-tc", action="store_true", help="skip the tensor-core forward (mode 3) comparison")
    ap.add_argument("--no-bwd-roofline", action="store_true", help="skip the separate backward timing")
    ap.add_argument("--no-extras", action="store_true", help="skip the NEXT-3 / NEXT-4 workload lines")
    ap.add_argument("--no-extra-lines", action="store_true", help="N > 1: skip the 1-GPU reference and c3 weak runs")
    ap.add_argument("--dist-backend", default="nccl", help="nccl (default); gloo only to exercise the multi-rank "
                    "logic when several ranks share one GPU")
    return ap.parse_args()


DEFAULT_STEPS = {"c1": 300, "c2": 300, "c3": 300, "c4": 20, "c5": 3}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ------------------------------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except (OSError, FileNotFoundError):
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.thread.join(timeout=2)
        sm, mx, reasons, power = [], None, set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
                power.append(float(parts[3]))
            except ValueError:
                continue
            for n, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return None
        loaded = [s for s in sm if mx is None or s >= 0.3 * mx] or sm
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm), "power_w_max": max(power) if power else None}


# ------------------------------------------------------------------------------------------ dist
def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


# ------------------------------------------------------------------------------------------ oracle timing
def _cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def oracle_sample(X, Y, budget_s: float, min_rows: int = 8):
    """Time the fp64 oracle brute force on row samples of both directions (bounded, ~budget_s).
    Returns (pairs/s, cores, description).  Rows are spread uniformly over all batch elements."""
    import oracle
    B, N, _ = X.shape
    M = Y.shape[1]
    threads = oracle.max_threads()
    # calibrate on a small sample
    rows = max(min_rows, threads * 32)
    t0 = time.perf_counter()
    oracle.nn(X, Y, rows=np.linspace(0, B * N - 1, rows).astype(np.int64))
    dt = max(time.perf_counter() - t0, 1e-4)
    rate = rows * M / dt
    per_dir_pairs = max(budget_s * rate / 2, rows * M)
    rx = int(min(B * N, max(min_rows, per_dir_pairs // M)))
    ry = int(min(B * M, max(min_rows, per_dir_pairs // N)))
    rows_x = np.linspace(0, B * N - 1, rx).astype(np.int64)
    rows_y = np.linspace(0, B * M - 1, ry).astype(np.int64)
    t0 = time.perf_counter()
    oracle.nn(X, Y, rows=rows_x, nthreads=threads)
    oracle.nn(Y, X, rows=rows_y, nthreads=threads)
    dt = time.perf_counter() - t0
    pairs = rx * M + ry * N
    desc = (f"fp64 brute-force oracle (oracle/chamfer_oracle.c, OpenMP) on {rx} X rows x {M} targets + {ry} Y rows "
            f"x {N} targets ({pairs:.3g} directed pairs, {dt:.1f} s) of the same workload; backward O(N+M) omitted")
    # single-core rate on a short sample (~1/8 of the budget), then the OpenMP default is restored
    r1 = int(max(min_rows, min(B * N, (budget_s / 8) * (rate / max(threads, 1)) / M)))
    t0 = time.perf_counter()
    oracle.nn(X, Y, rows=np.linspace(0, B * N - 1, r1).astype(np.int64), nthreads=1)
    one = r1 * M / max(time.perf_counter() - t0, 1e-6)
    oracle.nn(X[:, :1], Y[:, :1], nthreads=threads)
    return pairs / dt, threads, desc, dt, one


def run_reference(args):
    rank, world, local = dist_env()
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo", init_method="env://")
        if rank != 0:
            dist.barrier()
            dist.destroy_process_group()
            return
    c = synth.CONFIGS[args.config]
    X, Y = synth.config_inputs(args.config)
    budget = max(2.0, 150.0 / max(1, args.steps + args.warmup))
    vals = []
    for k in range(args.warmup + args.steps):
        v, cores, desc, dt, one = oracle_sample(X, Y, budget)
        if k >= args.warmup:
            vals.append(v)
    value = statistics.median(vals)
    B, N, M = c["B"], c["N"], c["M"]
    pairs = 2 * B * N * M
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 0, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": pairs / value * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": args.config, "desc": c["desc"], "B": B, "N": N, "M": M, "tau": c["tau"]},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": desc,
                         "value_1core": one, "cpu_model": _cpu_model()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


def _measured_peak(key, fallback):
    """(value, source) from the driver-written MEASURED_PEAKS.json, else the profiling guide's fallback."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            v = json.load(f).get(key)
        if v:
            return float(v), f"MEASURED_PEAKS.json {key}"
    except (OSError, ValueError):
        pass
    return fallback, "fallback (B200_PROFILING.md)"


def _traffic(kernel, cfg):
    """dram read+write bytes per launch of `kernel` (and its ncu FMA-pipe utilisation) from the
    committed ncu --set full capture."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(path) as f:
            d = json.load(f)
        e = d.get(f"{kernel}/{cfg}")
        if e is None:
            return None
        out = {"bytes_per_launch": e["dram_bytes_per_launch"], "source": "profiles/" + e["source"]}
        if "pipe_fma_pct" in e:
            out["ncu_pipe_fma_cycles_active_pct"] = e["pipe_fma_pct"]
        return out
    except (OSError, ValueError, KeyError):
        return None


COLL_NAMES = ("broadcast_clouds", "all_reduce_min_colkeys", "peer_barrier_keys_ready", "peer_barrier_keys_read",
              "all_reduce_partials", "all_gather_idx")


def _mean_ms(torch, fn, flush, K, warmup=1):
    """Mean device ms of K eager calls of fn (CUDA events on the launching stream, L2 flushed between)."""
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    for k in range(K):
        flush.fill_(k & 0xFF)
        ev[k][0].record()
        fn()
        ev[k][1].record()
    torch.cuda.synchronize()
    return sum(a.elapsed_time(b) for a, b in ev) / K


def multi_gpu_extras(cd, pdist, torch, dist, dev, flush, args, rank, world, value, X, Y, query_sharded,
                     strong_batch, loss_N):
    """N > 1 only: (a) the same config's full problem on ONE GPU (rank 0 alone, no collectives) and
    the scaling fraction value_N / (N x value_1); (b) c3 weak scaling (every rank its own batch of
    32, one partials all-reduce) with its own 1-GPU value — the two scaling regimes of SURVEY §8.e."""
    c = synth.CONFIGS[args.config]
    B, N, M, tau = c["B"], c["N"], c["M"], c["tau"]
    out = {}
    t = torch.zeros(2, dtype=torch.float64, device=dev)
    if rank == 0:
        if query_sharded:
            x1, y1 = torch.from_numpy(X).to(dev), torch.from_numpy(Y).to(dev)
        else:
            X1, Y1 = synth.config_inputs(args.config)
            x1, y1 = torch.from_numpy(X1).to(dev), torch.from_numpy(Y1).to(dev)

        loss1 = []

        def one():
            d_xy, i_xy, d_yx, i_yx, part = cd.forward(x1, y1, tau=tau)
            _, l1, _, _, _ = cd.finalize(part, N, M)
            cd.loss_backward(x1, y1, i_xy, i_yx, one_t)
            loss1[:] = [l1]
        one_t = torch.ones(1, dtype=torch.float32, device=dev)
        K1 = 2 if args.config == "c5" else max(3, min(args.steps, 20))
        t[0] = _mean_ms(torch, one, flush, K1)
        t[1] = float(loss1[0].item())
        del x1, y1
    dist.barrier()
    dist.broadcast(t, src=0)
    v1 = 2 * B * N * M / (t[0].item() * 1e-3)
    out["same_config_1gpu"] = {"value": v1, "ms_per_step": t[0].item(), "scaling_fraction": value / (world * v1),
                               "loss_1gpu": t[1].item(), "loss_bit_identical": t[1].item() == loss_N,
                               "note": "rank 0 alone, full problem, no collectives; fraction = value / (N x value_1gpu)"}
    if args.config != "c3":
        c3 = synth.CONFIGS["c3"]
        X3, Y3 = synth.config_inputs("c3", b0=rank * c3["B"], B=c3["B"])
        x3, y3 = torch.from_numpy(X3).to(dev), torch.from_numpy(Y3).to(dev)
        K3 = 50
        step3 = lambda: pdist.batch_sharded_step(cd, x3, y3, c3["B"] * world, rank * c3["B"], tau=c3["tau"])
        tt = torch.tensor([_mean_ms(torch, step3, flush, K3, warmup=3)], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t1 = torch.zeros(1, dtype=torch.float64, device=dev)
        if rank == 0:
            t1[0] = _mean_ms(torch, lambda: _c3_single(cd, x3, y3, c3), flush, K3, warmup=3)
        dist.barrier()
        dist.broadcast(t1, src=0)
        pairs3 = 2 * c3["B"] * world * c3["N"] * c3["M"]
        v3 = pairs3 / (tt.item() * 1e-3)
        v31 = 2 * c3["B"] * c3["N"] * c3["M"] / (t1.item() * 1e-3)
        out["c3_weak"] = {"value": v3, "unit": UNIT, "ms_per_step": tt.item(), "global_batch": c3["B"] * world,
                          "scaling": "weak", "value_1gpu": v31, "scaling_fraction": v3 / (world * v31),
                          "note": "each rank: the full c3 batch of 32 on its own batch elements; one B x 4 "
                                  "partials all-reduce; eager launches (no CUDA graph)"}
    return out


def _c3_single(cd, x, y, c3):
    d_xy, i_xy, d_yx, i_yx, part = cd.forward(x, y, tau=c3["tau"])
    cd.finalize(part, c3["N"], c3["M"])
    return cd.backward(x, y, i_xy, i_yx, g_scalar=1.0 / (c3["B"] * c3["N"]), h_scalar=1.0 / (c3["B"] * c3["M"]))


P2S_OPS_PER_PAIR = 44   # FP32-pipe lane ops per (point, face) of the p2s hot loop


def _timed(torch, fn, flush, K, warmup=2, graph=True):
    """Mean device ms of fn() over K replays (CUDA graph when possible), L2 flushed between steps."""
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    g = None
    if graph:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            fn()
        g.replay()
        torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    for k in range(K):
        flush.fill_(k & 0xFF)
        ev[k][0].record()
        if g is not None:
            g.replay()
        else:
            fn()
        ev[k][1].record()
    torch.cuda.synchronize()
    return sum(a.elapsed_time(b) for a, b in ev) / K


def measure_extras(cd, torch, dev, flush, args, K_extra):
    """NEXT-3 (point-to-surface loss fwd+bwd) and NEXT-4 (mesh -> sample -> Chamfer -> grad to
    vertices) steps on ShapeNet-like meshes (icosphere subdivision 5: 10,242 vertices, 20,480 faces)."""
    out = {}
    # NEXT-3: B=8 meshes, N=16,384 points each (c3-sized clouds), loss + grads to points and vertices
    B, N = 8, 16384
    V, F = synth.mesh_batch(B, subdiv=5, config_index=200)
    P = synth.shape_pair(B, N, 8, config_index=201)[0]
    v, f, p = torch.from_numpy(V).to(dev), torch.from_numpy(F).to(dev), torch.from_numpy(P).to(dev)
    Nv, Nf = V.shape[1], F.shape[0]

    def p2s_step():
        d, fi, cl, ba, pb, loss = cd.p2s_forward(p, v, f)
        cd.p2s_backward(p, cl, fi, ba, f, Nv, g=None, g_scalar=1.0 / (B * N))
        return loss

    ms = _timed(torch, p2s_step, flush, K_extra)
    fa, fb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fa.record()
    fb.record()
    torch.cuda.synchronize()
    cd.set_profile_events(fa, fb)
    cd.p2s_forward(p, v, f)
    cd.set_profile_events(None, None)
    torch.cuda.synchronize()
    kms = fa.elapsed_time(fb)
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    peak = sms * 128 * 1965e6 / 1e12
    pairs = B * N * Nf
    ach = P2S_OPS_PER_PAIR * pairs / (kms * 1e-3) / 1e12

    def p2s_step_pruned():
        d, fi, cl, ba, pb, loss = cd.p2s_forward(p, v, f, algorithm="pruned")
        cd.p2s_backward(p, cl, fi, ba, f, Nv, g=None, g_scalar=1.0 / (B * N))
        return loss

    ms_pr = _timed(torch, p2s_step_pruned, flush, K_extra)
    out["next3_point_to_surface"] = {
        "workload": f"B={B} meshes (icosphere-5: {Nv} verts, {Nf} faces) x N={N} points; loss + grads to points and vertices",
        "ms_per_step": ms, "point_face_pairs_per_s": pairs / (ms * 1e-3),
        "kernel": "p2s_kernel", "kernel_ms": kms,
        "roofline": {"bound": "alu", "unit": "Tops/s (FP32-pipe lane ops)", "achieved": ach, "peak": peak,
                     "frac": ach / peak, "algorithmic": f"{P2S_OPS_PER_PAIR} FP32-pipe ops per (point, face)"},
        "pruned": {"ms_per_step": ms_pr, "point_face_pairs_per_s_effective": pairs / (ms_pr * 1e-3),
                   "speedup_vs_brute": ms / ms_pr,
                   "note": "cd_p2s_forward_pruned (R26): same minima as the brute force; work-efficient, so "
                           "its rate is quoted in brute-force pairs per second"},
    }
    # NEXT-4: B=32 meshes -> N=16,384 samples each -> Chamfer vs Y (M=16,384) -> grad to vertices
    B, N, M = 32, 16384, 16384
    V, F = synth.mesh_batch(B, subdiv=5, config_index=210)
    Y = synth.shape_pair(B, 8, M, config_index=211)[1]
    rf, rb = synth.sampling_randoms(B, N, seed=212)
    v, f, y = torch.from_numpy(V).to(dev), torch.from_numpy(F).to(dev), torch.from_numpy(Y).to(dev)
    rft, rbt = torch.from_numpy(rf).to(dev), torch.from_numpy(rb).to(dev)
    Nv = V.shape[1]

    def pipe_step():
        pts, fi, ba = cd.sample_mesh(v, f, rft, rbt)
        d_xy, i_xy, d_yx, i_yx, part = cd.forward(pts, y, tau=0.01)
        _, loss, F1, _, _ = cd.finalize(part, N, M)
        gx, _ = cd.backward(pts, y, i_xy, i_yx, g_scalar=1.0 / (B * N), h_scalar=1.0 / (B * M))
        return cd.sample_mesh_backward(f, fi, ba, Nv, gx)

    ms = _timed(torch, pipe_step, flush, K_extra)

    def pipe_step_pruned():
        pts, fi, ba = cd.sample_mesh(v, f, rft, rbt)
        d_xy, i_xy, d_yx, i_yx, part = cd.forward(pts, y, tau=0.01, algorithm="pruned")
        _, loss, F1, _, _ = cd.finalize(part, N, M)
        gx, _ = cd.backward(pts, y, i_xy, i_yx, g_scalar=1.0 / (B * N), h_scalar=1.0 / (B * M))
        return cd.sample_mesh_backward(f, fi, ba, Nv, gx)

    ms_pr = _timed(torch, pipe_step_pruned, flush, K_extra)
    out["next4_sample_chamfer"] = {
        "workload": f"B={B} meshes (icosphere-5) -> N={N} samples -> Chamfer + F@0.01 vs M={M} -> grad to vertices",
        "ms_per_step": ms, "directed_pairs_per_s": 2 * B * N * M / (ms * 1e-3),
        "pruned_forward": {"ms_per_step": ms_pr, "directed_pairs_per_s_effective": 2 * B * N * M / (ms_pr * 1e-3),
                           "note": "same pipeline through cd_forward_pruned (results identical to the brute force)"},
    }
    return out


# ------------------------------------------------------------------------------------------ ours
def main():
    args = parse()
    if args.config is None:
        args.config = "c3" if int(os.environ.get("WORLD_SIZE", "1")) == 1 else "c5"
    if args.steps is None:
        args.steps = DEFAULT_STEPS[args.config]
    if args.impl == "reference":
        return run_reference(args)
    import torch
    import torch.distributed as dist

    from paper_1911_05063_b200 import api as cd
    from paper_1911_05063_b200 import distributed as pdist
    from paper_1911_05063_b200 import _lib

    rank, world, local = dist_env()
    if args.gpus != world and world > 1:
        log(f"warning: --gpus {args.gpus} but WORLD_SIZE={world}; using WORLD_SIZE")
    # one process per GPU; several ranks only share a GPU in the gloo logic check (--dist-backend gloo)
    gpu = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(gpu)
    dev = torch.device("cuda", gpu)
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", init_method="env://", device_id=dev)
        else:
            dist.init_process_group(args.dist_backend, init_method="env://")
    c = synth.CONFIGS[args.config]
    B, N, M, tau = c["B"], c["N"], c["M"], c["tau"]
    # partitioning per BASELINE.json configs: c5 query-sharded and c4 batch-sharded
    # (B = 8 split over the ranks) are STRONG scaling of the named problem; any other config under
    # N > 1 runs its full batch on every rank (weak scaling)
    query_sharded = args.config == "c5" and world > 1
    strong_batch = args.config == "c4" and world > 1
    if query_sharded:
        B_local, b0, B_global = B, 0, B
        X, Y = synth.config_inputs(args.config) if rank == 0 else (np.empty((B, N, 3), np.float32),
                                                                    np.empty((B, M, 3), np.float32))
        scaling = "strong"
    elif strong_batch:
        b0, b1 = pdist.shard_range(B, rank, world)
        B_local, B_global = b1 - b0, B
        if B_local < 1:
            raise SystemExit(f"c4 strong scaling needs at most B={B} ranks")
        X, Y = synth.config_inputs(args.config, b0=b0, B=B_local)
        scaling = "strong"
    else:
        B_local, b0, B_global = B, rank * B, B * world
        X, Y = synth.config_inputs(args.config, b0=b0, B=B_local)
        scaling = "weak"
    x = torch.from_numpy(X).to(dev)
    y = torch.from_numpy(Y).to(dev)
    w1 = w2 = 1.0
    pairs_total = 2 * B_global * N * M           # directed pairs of the whole job per step
    # the fused kernel evaluates each distance once for both directions: B*N*M evaluations per launch
    evals_fwd_launch = (B * N * M) // world if query_sharded else B_local * N * M
    prof = pdist.CollectiveTimer() if world > 1 else None
    # column-key exchange of query sharding: the NCCL all-reduce MIN (default), or --colkey-exchange
    # peer: symmetric-memory key arrays MIN-reduced inside the resolve kernel (cd_forward_cols_peers);
    # every rank must agree, so an unavailable peer path falls back to NCCL on all ranks
    peer = None
    if query_sharded and args.colkey_exchange == "peer":
        peer = pdist.PeerColKeys.create(B, M, dev)
        ok = torch.tensor([1 if peer is not None else 0], device=dev)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        if ok.item() == 0:
            peer = None
    colkey_exchange = ("peer reads of symmetric-memory key arrays, MIN fused into the resolve"
                       if peer is not None else f"{dist.get_backend()} all_reduce MIN") if query_sharded else None

    def step():
        if query_sharded:
            pdist.broadcast_clouds(x, y, src=0, prof=prof)
            return pdist.query_sharded_step(cd, x, y, tau=tau, w1=w1, w2=w2, prof=prof, peer=peer)
        return pdist.batch_sharded_step(cd, x, y, B_global, b0, tau=tau, w1=w1, w2=w2, prof=prof)

    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    for _ in range(args.warmup):
        out = step()
    torch.cuda.synchronize()
    if prof is not None:
        prof.reset()

    K = args.steps
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    fev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    for a, b in fev:   # materialise the cudaEvent handles (torch creates them lazily); libcd re-records them
        a.record()
        b.record()
    # single rank: the whole step (all kernels of rows a.1-a.8) is captured once into a CUDA graph and
    # replayed, so small configs are not bound by host launch overhead
    graph = None
    if world == 1 and not args.no_graph:
        gev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
        gev[0].record()
        gev[1].record()
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        cd.set_profile_events(*gev)
        with torch.cuda.graph(graph):
            out = step()
        cd.set_profile_events(None, None)
        for _ in range(args.warmup):
            graph.replay()
        torch.cuda.synchronize()
    sampler = ClockSampler(gpu) if not args.no_clocks else None
    if sampler:
        sampler.start()
        time.sleep(0.3)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    fwd_ms = []
    for k in range(K):
        flush.fill_(k & 0xFF)                     # L2 flush, outside the timed events
        if graph is not None:
            ev[k][0].record()
            graph.replay()
            ev[k][1].record()
            ev[k][1].synchronize()                # read the in-graph kernel events of this replay
            fwd_ms.append(gev[0].elapsed_time(gev[1]))
        else:
            cd.set_profile_events(*fev[k])
            ev[k][0].record()
            out = step()
            ev[k][1].record()
    cd.set_profile_events(None, None)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = sampler.stop() if sampler else None
    step_ms = [a.elapsed_time(b) for a, b in ev]
    if graph is None:
        fwd_ms = [a.elapsed_time(b) for a, b in fev]
    tot = torch.tensor([sum(step_ms), sum(fwd_ms)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tot, op=dist.ReduceOp.MAX)
    ms_per_step = tot[0].item() / K
    fwd_kernel_ms = tot[1].item() / K
    value = pairs_total / (ms_per_step * 1e-3)
    multi = None
    if world > 1:
        coll = prof.by_name_ms()
        ct = torch.tensor([sum(coll.values())] + [coll.get(n, 0.0) for n in COLL_NAMES], dtype=torch.float64,
                          device=dev)
        dist.all_reduce(ct, op=dist.ReduceOp.MAX)
        multi = {"ranks": dist.get_world_size(), "backend": dist.get_backend(), "colkey_exchange": colkey_exchange,
                 "collective_ms_per_step_max_rank": ct[0].item() / K,
                 "collective_share_of_step": ct[0].item() / K / ms_per_step,
                 "collectives_ms_per_step": {n: ct[i + 1].item() / K for i, n in enumerate(COLL_NAMES)
                                             if ct[i + 1].item() > 0},
                 "work_per_rank": ("B*N*M/world distance evaluations (X rows split; the fused kernel serves both "
                                   "directions)" if query_sharded else f"B_local={B_local} of B={B_global}")}
        if not args.no_extra_lines:
            multi.update(multi_gpu_extras(cd, pdist, torch, dist, dev, flush, args, rank, world, value, X, Y,
                                          query_sharded, strong_batch, float(out["loss"].item())))
    loss = float(out["loss"].item())

    # ---------------------------------------------------------------- exact pruned algorithm (NEXT-2)
    pruned = None
    if world == 1 and not args.no_pruned:
        class PrunedEngine:
            forward = staticmethod(lambda xx, yy, tau=None: cd.forward_pruned(xx, yy, tau=tau))
            finalize = staticmethod(cd.finalize)
            backward = staticmethod(cd.backward)

        def pstep():
            return pdist.batch_sharded_step(PrunedEngine, x, y, B_global, b0, tau=tau, w1=w1, w2=w2)

        for _ in range(args.warmup):
            pout = pstep()
        torch.cuda.synchronize()
        pgraph = None
        if not args.no_graph:
            pgraph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(pgraph):
                pout = pstep()
            for _ in range(args.warmup):
                pgraph.replay()
        torch.cuda.synchronize()
        pev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
        for k in range(K):
            flush.fill_(k & 0xFF)
            pev[k][0].record()
            if pgraph is not None:
                pgraph.replay()
            else:
                pout = pstep()
            pev[k][1].record()
        torch.cuda.synchronize()
        pms = sum(a.elapsed_time(b) for a, b in pev) / K
        ploss = float(pout["loss"].item())
        pruned = {"ms_per_step": pms, "value_effective": pairs_total / (pms * 1e-3), "unit": UNIT,
                  "speedup_vs_brute_step": ms_per_step / pms, "loss": ploss,
                  "loss_rel_diff_vs_brute": abs(ploss - loss) / max(abs(loss), 1e-300),
                  "note": ("cd_forward_pruned (exact: Hilbert-ordered tiles + lower-bound culling, SURVEY §8.f NEXT-2) "
                           "+ finalize + backward; effective = the same 2*B*N*M directed pairs / step time")}

    # ---------------------------------------------------------------- backward vs HBM roofline
    bwd_roof = None
    if not query_sharded and not args.no_bwd_roofline:
        d_xy0, i_xy0, d_yx0, i_yx0, _ = cd.forward(x, y, tau=tau)
        torch.cuda.synchronize()
        bms = _timed(torch, lambda: cd.backward(x, y, i_xy0, i_yx0, g_scalar=w1 / (B_global * N),
                                                h_scalar=w2 / (B_global * M)), flush, max(3, min(K, 50)))
        pts = B_local * (N + M)
        alg = 28 * pts   # read both clouds (12 B) + both index arrays (4 B) + write both gradients (12 B)
        hbm_peak = _measured_peak("hbm_gbs", 7700.0)
        nbl = cd.launch_count(_lib.CD_OP_BACKWARD, B_local, N, M)
        bwd_kern = ("cd_backward (seg_sort_grad: each (direction, batch) segment part sorted on chip, its targets' "
                    "gradients written by the same CTA: "
                    if max(N, M) <= 24576 else "cd_backward (keys+hist, radix passes, offsets, grad: ")
        bwd_roof = {"bound": "hbm", "kernel": f"{bwd_kern}{nbl} launches)", "ms": bms,
                    "achieved": alg / (bms * 1e-3) / 1e9, "peak": hbm_peak[0], "unit": "GB/s",
                    "frac": alg / (bms * 1e-3) / 1e9 / hbm_peak[0], "peak_source": hbm_peak[1],
                    "algorithmic": "28 B per point (clouds 12 + indices 4 + gradients 12); the sort (global key/value "
                                   "passes or the on-chip segment sort) and the partner gathers are extra traffic"}
        try:
            with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
                tb = json.load(f).get(f"backward/{args.config}")
        except (OSError, ValueError):
            tb = None
        if tb:
            gbs = tb["dram_bytes_per_call"] / (tb["ms_cold"] * 1e-3) / 1e9
            bwd_roof["dram_measured"] = {
                "bytes_per_call": tb["dram_bytes_per_call"], "ms_cold": tb["ms_cold"], "GB_s": gbs,
                "frac": gbs / hbm_peak[0], "source": "profiles/" + tb["source"],
                "note": "ncu dram__bytes_read+write summed over the backward's kernels (cold, serialised); "
                        "all DRAM traffic incl. the sort passes and the random coordinate gathers"}

    # ---------------------------------------------------------------- tensor-core forward (mode 3)
    tcf = None
    if world == 1 and not args.no_tc and not query_sharded:
        outs = {}
        times = {}
        for mode in (2, 3):
            old_mode = cd.set_forward_mode(mode)
            try:
                times[mode] = _timed(torch, lambda: cd.forward(x, y, tau=tau), flush, max(3, min(K, 50)))
                outs[mode] = cd.forward(x, y, tau=tau)
                torch.cuda.synchronize()
            finally:
                cd.set_forward_mode(old_mode)
        same = all(bool(torch.equal(a, b)) for a, b in zip(outs[2], outs[3]))
        tcf = {"forward_ms_tensor_core": times[3], "forward_ms_fp32_fused": times[2],
               "bit_identical_outputs": same,
               "note": ("cd_set_forward_mode(3): tcgen05 fp16-split MMA filter + exact fp32 re-scan (DESIGN.md "
                        "4.7, R27); not the default (its exactness rests on the measured tensor-core accumulation)")}

    # ---------------------------------------------------------------- NEXT-3 / NEXT-4 workloads
    extras = None
    if world == 1 and not args.no_extras:
        extras = measure_extras(cd, torch, dev, flush, args, K_extra=max(3, min(K, 50)))

    # ---------------------------------------------------------------- e2e through host buffers
    e2e = None
    if not args.no_e2e:
        xh = cd.pinned_copy(X)
        yh = cd.pinned_copy(Y)
        if world == 1:
            stepper = cd.HostStepper(B_local, N, M, tau=tau, w1=w1, w2=w2, device=dev, graph=not args.no_graph)

            def e2e_step():
                stepper.step(xh, yh)
            api_desc = (f"cd_step_host_overlapped via api.HostStepper (pinned host clouds -> H2D in {stepper.nchunks} "
                        "batch ranges on a copy stream, each range's forward starting as it lands and its loss "
                        "backward + gradient D2H following -> finalize -> D2H of loss and F; every step copies its "
                        "inputs and results" + ("; the call is captured once in a CUDA graph and replayed)"
                                                if not args.no_graph else ")"))
            h2d, d2h = int(X.nbytes + Y.nbytes), stepper.d2h_bytes()
        else:
            # the public API under torch.distributed: the clouds land from pinned host memory (rank 0 only
            # when query-sharded: the broadcast inside the step replicates them), the sharded step runs,
            # and loss + this rank's gradient rows return to pinned host memory
            own = rank == 0 or not query_sharded
            lh = cd.pinned_empty((1,))
            gxh = cd.pinned_empty((B_local, out["grad_x"].shape[1], 3))
            gyh = cd.pinned_empty((B_local, out["grad_y"].shape[1], 3))

            def e2e_step():
                if own:
                    x.copy_(xh, non_blocking=True)
                    y.copy_(yh, non_blocking=True)
                o = step()
                lh.copy_(o["loss"], non_blocking=True)
                gxh.copy_(o["grad_x"], non_blocking=True)
                gyh.copy_(o["grad_y"], non_blocking=True)
                stepper_loss[0] = lh
            stepper_loss = [None]
            api_desc = ("api + distributed.{} (pinned host clouds -> H2D{} -> sharded step with its collectives -> "
                        "D2H of loss and this rank's gradient rows)".format(
                            "query_sharded_step" if query_sharded else "batch_sharded_step",
                            " on rank 0, broadcast" if query_sharded else ""))
            h2d = int(X.nbytes + Y.nbytes) if own else 0
            d2h = 4 + 4 * (gxh.numel() + gyh.numel())
        for _ in range(max(1, args.warmup)):
            e2e_step()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        eev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
        for k in range(K):
            flush.fill_(k & 0xFF)
            eev[k][0].record()
            e2e_step()
            eev[k][1].record()
        torch.cuda.synchronize()
        et = torch.tensor([sum(a.elapsed_time(b) for a, b in eev)], dtype=torch.float64, device=dev)
        hd = torch.tensor([h2d, d2h], dtype=torch.float64, device=dev)
        if world > 1:
            dist.barrier()
            dist.all_reduce(et, op=dist.ReduceOp.MAX)
            dist.all_reduce(hd, op=dist.ReduceOp.SUM)
        e2e_ms = et.item() / K
        e2e = {"value": pairs_total / (e2e_ms * 1e-3), "unit": UNIT, "ms_per_step": e2e_ms,
               "h2d_bytes_per_step": int(hd[0].item()), "d2h_bytes_per_step": int(hd[1].item()),
               "api": api_desc,
               "loss_e2e": float(stepper.loss[0]) if world == 1 else float(stepper_loss[0][0])}

    # ---------------------------------------------------------------- roofline of the dominant kernel
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    sm_max = (clocks or {}).get("sm_max_mhz") or SM_MAX_MHZ_FALLBACK
    peak_ops = sms * 128 * sm_max * 1e6 / 1e12      # FP32-pipe lane ops/s, T
    achieved_ops = FP32_OPS_PER_PAIR * evals_fwd_launch / (fwd_kernel_ms * 1e-3) / 1e12
    roofline = {
        "bound": "alu", "kernel": "nn_fused_kernel", "unit": "Tops/s (FP32-pipe lane ops: FADD/FMUL/FFMA = 1)",
        "achieved": achieved_ops, "peak": peak_ops, "frac": achieved_ops / peak_ops,
        "peak_source": f"derived: {sms} SMs x 128 FP32 lanes x {sm_max:.0f} MHz (max SM clock); DESIGN.md §4.3",
        "algorithmic": (f"{FP32_OPS_PER_PAIR} FP32-pipe ops per distance evaluation x {evals_fwd_launch} evaluations "
                        "per launch (B*N*M: each distance serves both directions)"),
        "kernel_ms": fwd_kernel_ms, "kernel_share_of_step": fwd_kernel_ms / ms_per_step,
        "traffic": _traffic("nn_fused_kernel", args.config),
        "flops_view": {"achieved_tflops": FLOPS_PER_PAIR * evals_fwd_launch / (fwd_kernel_ms * 1e-3) / 1e12,
                       "peak_tflops": 2 * peak_ops},
    }
    if clocks and clocks.get("sm_mhz"):
        roofline["frac_at_sampled_clock"] = achieved_ops / (sms * 128 * clocks["sm_mhz"] * 1e6 / 1e12)

    # ---------------------------------------------------------------- cpu baseline (rank 0, N=1)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, cores, desc, dt, one = oracle_sample(X, Y, args.cpu_seconds)
        cpu = {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": desc, "value_1core": one,
               "cpu_model": _cpu_model()}

    launches = cd.launch_count(_lib.CD_OP_STEP, B_local, N, M)
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": args.warmup,
            "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": scaling, "vs_baseline": None,
            "dtype": "f32", "data": "synthetic (seeded ShapeNet-like deformed-icosphere surface samples, DESIGN.md §5)",
            "config": {"workload": args.config, "desc": c["desc"], "global_batch": B_global, "B_per_rank": B_local,
                       "N": N, "M": M, "tau": tau,
                       "parallelism": (f"query-sharded x{world}" if query_sharded else f"batch-sharded x{world}"),
                       "launch": "cuda_graph" if graph is not None else "eager",
                       "l2": "flushed between timed steps (256 MiB write outside the step events)"},
            # north-star "effective" view: directed pairs/s x 6 ops / FP32-pipe peak per GPU; can exceed 100
            # because the fused kernel evaluates each distance once for both directions
            "pct_fp32_fma_peak_effective": 100.0 * FP32_OPS_PER_PAIR * pairs_total / world / (ms_per_step * 1e-3) /
                                           (sms * 128 * sm_max * 1e6),
            "roofline": roofline,
            "roofline_backward": bwd_roof,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "pruned": pruned,
            "tensor_core_forward": tcf,
            "next_rows": extras,
            "multi_gpu": multi,
            "gpu_launches": launches * K,
            "gpu_launches_per_step": launches,
            "clocks": clocks,
            "loss": loss,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
