"""ctypes binding of libcd.so (include/cd.h).  Argument marshalling only.

Loading fails loudly: there is no CPU fallback anywhere in this package.  If libcd.so is missing
(not built) or cannot be loaded, every compute call raises RuntimeError.
"""
from __future__ import annotations

import ctypes
import os
import re
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "lib", "libcd.so")
# experiment hook: load another in-tree build (e.g. a tuning variant); the product default is above
if os.environ.get("CD_LIB_VARIANT"):
    LIB_PATH = os.path.join(HERE, "lib", f"libcd_{os.environ['CD_LIB_VARIANT']}.so")
HEADER = os.path.join(os.path.dirname(HERE), "include", "cd.h")

CD_OK = 0
ABI_VERSION = 5
CD_OP_FORWARD, CD_OP_FSCORE, CD_OP_BACKWARD, CD_OP_STEP, CD_OP_FORWARD_PRUNED = 0, 1, 2, 3, 4
CD_OP_SAMPLE, CD_OP_SAMPLE_BACKWARD, CD_OP_P2S, CD_OP_P2S_BACKWARD, CD_OP_P2S_PRUNED = 5, 6, 7, 8, 9
STATUS_NAMES = {0: "CD_OK", 1: "CD_ERR_INVALID_VALUE", 2: "CD_ERR_MISALIGNED", 3: "CD_ERR_TOO_LARGE",
                4: "CD_ERR_UNSUPPORTED_DEVICE", 5: "CD_ERR_CUDA"}

_lock = threading.Lock()
_lib = None

vp = ctypes.c_void_p
i32 = ctypes.c_int
f32 = ctypes.c_float
sz = ctypes.c_size_t

_SIGS = {
    "cd_forward": ([vp, vp, i32, i32, i32, i32, i32, i32, i32, vp, vp, vp, vp, vp, f32, vp, sz, vp], i32),
    "cd_finalize": ([vp, i32, i32, i32, f32, f32, vp, vp, vp, vp, vp, vp], i32),
    "cd_fscore": ([vp, vp, i32, i32, i32, f32, vp, vp, vp, vp, sz, vp], i32),
    "cd_backward": ([vp, vp, i32, i32, i32, vp, vp, vp, vp, f32, f32, i32, i32, i32, i32, vp, vp, vp, sz, vp], i32),
    "cd_loss_backward": ([vp, vp, i32, i32, i32, vp, vp, vp, f32, f32, i32, i32, i32, i32, vp, vp, vp, sz, vp], i32),
    "cd_step_host": ([vp, vp, i32, i32, i32, f32, f32, f32, vp, vp, vp, vp, vp, sz, vp], i32),
    "cd_step_host_overlapped": ([vp, vp, i32, i32, i32, f32, f32, f32, vp, vp, vp, vp, i32, vp, sz, vp, vp, vp,
                                 vp], i32),
    "cd_workspace_size": ([i32, i32, i32, i32], sz),
    "cd_launch_count": ([i32, i32, i32, i32], i32),
    "cd_status_string": ([i32], ctypes.c_char_p),
    "cd_last_error_string": ([], ctypes.c_char_p),
    "cd_abi_version": ([], i32),
    "cd_set_forward_splits": ([i32], i32),
    "cd_set_profile_events": ([vp, vp], None),
    "cd_set_forward_mode": ([i32], i32),
    "cd_forward_pruned": ([vp, vp, i32, i32, i32, vp, vp, vp, vp, vp, f32, vp, sz, vp], i32),
    "cd_sample_mesh": ([vp, vp, i32, i32, i32, i32, vp, vp, vp, vp, vp, vp, sz, vp], i32),
    "cd_sample_mesh_backward": ([vp, vp, vp, i32, i32, i32, i32, vp, vp, vp, sz, vp], i32),
    "cd_sample_workspace_size": ([i32, i32, i32, i32, i32], sz),
    "cd_sample_launch_count": ([i32, i32, i32, i32, i32], i32),
    "cd_p2s_forward": ([vp, vp, vp, i32, i32, i32, i32, vp, vp, vp, vp, vp, vp, vp, sz, vp], i32),
    "cd_p2s_backward": ([vp, vp, vp, vp, vp, i32, i32, i32, i32, vp, f32, vp, vp, vp, sz, vp], i32),
    "cd_p2s_loss_backward": ([vp, vp, vp, vp, vp, i32, i32, i32, i32, vp, vp, vp, vp, sz, vp], i32),
    "cd_p2s_workspace_size": ([i32, i32, i32, i32, i32], sz),
    "cd_p2s_launch_count": ([i32, i32, i32, i32, i32], i32),
    "cd_p2s_forward_pruned": ([vp, vp, vp, i32, i32, i32, i32, vp, vp, vp, vp, vp, vp, vp, sz, vp], i32),
    "cd_forward_rows": ([vp, vp, i32, i32, i32, i32, i32, vp, vp, vp, vp, f32, vp, sz, vp], i32),
    "cd_forward_cols": ([vp, vp, i32, i32, i32, vp, i32, i32, vp, vp, vp, f32, vp, sz, vp], i32),
    "cd_forward_cols_peers": ([vp, vp, i32, i32, i32, vp, i32, i32, i32, vp, vp, vp, f32, vp, sz, vp], i32),
}


class CdError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


def declared_symbols(header: str = HEADER):
    """Function names declared in include/cd.h."""
    with open(header) as f:
        text = f.read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(cd_[a-z_0-9]+)\s*\(", text)))


def load():
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise RuntimeError(f"libcd.so not built ({LIB_PATH}); run `python -c 'import __graft_entry__ as g; "
                                   "g.build()'` — there is no CPU fallback")
            lib = ctypes.CDLL(LIB_PATH)
            for name, (args, res) in _SIGS.items():
                fn = getattr(lib, name)
                fn.argtypes = args
                fn.restype = res
            if lib.cd_abi_version() != ABI_VERSION:
                raise RuntimeError("libcd ABI version mismatch")
            _lib = lib
    return _lib


def check(status: int):
    if status != CD_OK:
        raise CdError(status, load().cd_last_error_string().decode())
