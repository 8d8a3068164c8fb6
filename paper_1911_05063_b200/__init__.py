"""B200-native batched exact nearest-neighbour Chamfer distance / backward / F-score.

The data-parallel hot path behind Kaolin's 3D point-cloud losses and metrics (PAPER.md:253-254,
§2.5 "Loss Functions and Metrics"), as hand-written sm_100a CUDA kernels behind the C ABI in
include/cd.h (libcd.so).  This package is the thin Python layer: ctypes marshalling plus a
torch.autograd wrapper; PyTorch provides device memory, streams and process groups only.
There is no CPU fallback: without a built libcd.so and an sm_100 GPU every compute call raises.
"""
from . import synth  # noqa: F401  (seeded inputs; no method arithmetic)

__all__ = ["p2s_forward", "p2s_backward", "point_to_surface", "PointToSurfaceFunction", "sample_mesh", "sample_mesh_backward", "sample_points", "SampleMeshFunction", "forward_pruned",
           "forward", "forward_rows", "forward_cols", "set_forward_mode", "finalize", "fscore", "fscore_from_distances", "backward", "chamfer", "step_host",
           "set_forward_splits", "ChamferFunction", "synth"]


def __getattr__(name):
    # torch-dependent API is imported lazily so `import paper_1911_05063_b200.synth` stays light
    if name in __all__ or name in ("workspace", "launch_count", "pinned_copy", "pinned_empty"):
        from . import api as _c
        return getattr(_c, name)
    raise AttributeError(name)
