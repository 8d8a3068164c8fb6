"""C-ABI checks that need no GPU: the library loads, exports every symbol include/cd.h declares,
and validates arguments before touching CUDA (empty cloud -> domain error)."""
import ctypes
import os
import subprocess

import pytest

from paper_1911_05063_b200 import _lib

LIB = _lib.LIB_PATH


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(LIB):
        from paper_1911_05063_b200 import build
        build.build()
    return _lib.load()


def test_exports_every_declared_symbol(lib):
    declared = _lib.declared_symbols()
    assert {"cd_forward", "cd_backward", "cd_fscore", "cd_finalize", "cd_step_host"} <= set(declared)
    out = subprocess.run(["nm", "-D", "--defined-only", LIB], capture_output=True, text=True, check=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if line.strip()}
    missing = [s for s in declared if s not in exported]
    assert not missing, missing
    for s in declared:
        assert hasattr(lib, s)


def test_binding_declares_every_entry_point():
    """The ctypes binding (argument marshalling) carries a signature for every declared function, with
    the header's argument count, so a changed C signature cannot be called with stale arguments."""
    import re
    with open(_lib.HEADER) as f:
        text = re.sub(r"/\*.*?\*/", "", f.read(), flags=re.S)
    for name in _lib.declared_symbols():
        assert name in _lib._SIGS, name
        m = re.search(r"\b" + name + r"\s*\(([^)]*)\)", text)
        params = [p for p in m.group(1).split(",") if p.strip() and p.strip() != "void"]
        assert len(_lib._SIGS[name][0]) == len(params), (name, len(_lib._SIGS[name][0]), len(params))


def test_only_cd_symbols_exported():
    out = subprocess.run(["nm", "-D", "--defined-only", LIB], capture_output=True, text=True, check=True).stdout
    names = [line.split()[-1] for line in out.splitlines() if " T " in line]
    assert names and all(n.startswith("cd_") for n in names), names


def test_abi_version_and_status_strings(lib):
    assert lib.cd_abi_version() == 5
    assert lib.cd_status_string(0) == b"CD_OK"
    assert lib.cd_status_string(1) == b"CD_ERR_INVALID_VALUE"
    assert lib.cd_status_string(5) == b"CD_ERR_CUDA"


def test_workspace_sizes(lib):
    for op in range(4):
        assert lib.cd_workspace_size(op, 1, 1024, 1024) > 0
        assert lib.cd_workspace_size(op, 0, 1024, 1024) == 0      # empty batch
        assert lib.cd_workspace_size(op, 1, 0, 1024) == 0         # empty cloud
    assert lib.cd_workspace_size(0, 4, 1 << 20, 1 << 20) > lib.cd_workspace_size(0, 1, 1024, 1024)
    assert lib.cd_workspace_size(0, 1024, 1 << 21, 1 << 21) == 0  # B*(N+M) > 2^31-1


def test_launch_counts(lib):
    # fused forward: pack + fused + epilogue (row merge | column resolve) + partials
    assert lib.cd_launch_count(0, 32, 16384, 16384) == 4
    # backward, clouds of <= 24576 points: one launch sorts each segment part on chip and writes its
    # targets' gradients
    assert lib.cd_launch_count(2, 32, 16384, 16384) == 1
    assert lib.cd_launch_count(3, 32, 16384, 16384) == 4 + 1 + 1
    assert lib.cd_launch_count(2, 8, 24577, 100) == 2 * 3 + 2   # 15-bit segment-local keys: 2 passes of 8 bits
    # backward, larger clouds: keys+hist, radix passes x 3 kernels - 1 hist, offsets, grad
    assert lib.cd_launch_count(2, 8, 100000, 100000) == 2 * 3 + 2   # 17-bit local keys: 2 passes of 9 bits
    # c5: 20-bit local keys -> 3 passes of 7 bits (2 of 10 cost more)
    assert lib.cd_launch_count(2, 4, 1 << 20, 1 << 20) == 3 * 3 + 2


def _forward(lib, B=1, N=8, M=8, q=(0, 8), r=(0, 8), x=4, y=4, ws=256, wsb=1 << 30, tau=-1.0, dxy=64, ixy=64,
             dyx=64, iyx=64):
    v = ctypes.c_void_p
    return lib.cd_forward(v(x), v(y), B, N, M, q[0], q[1], r[0], r[1], v(dxy), v(ixy), v(dyx), v(iyx), None,
                          tau, v(ws), wsb, None)


def test_forward_validation_before_launch(lib):
    assert _forward(lib, N=0, q=(0, 0)) == 1
    assert b"empty cloud" in lib.cd_last_error_string()
    assert _forward(lib, B=0) == 1
    assert _forward(lib, x=0) == 1
    assert _forward(lib, q=(3, 2)) == 1
    assert _forward(lib, r=(0, 9)) == 1
    assert _forward(lib, dxy=0) == 1
    assert _forward(lib, tau=float("nan")) == 1
    assert _forward(lib, x=2) == 2       # misaligned cloud
    assert _forward(lib, ws=255) == 2    # misaligned workspace
    assert _forward(lib, wsb=16) == 3    # workspace too small
    assert _forward(lib, B=1 << 20, N=1 << 12, M=1 << 12, q=(0, 1 << 12), r=(0, 1 << 12)) == 3
    assert _forward(lib, B=65536, N=4, M=4, q=(0, 4), r=(0, 4)) == 3   # batch elements map to gridDim.y
    assert b"65535" in lib.cd_last_error_string()


def test_backward_and_fscore_validation(lib):
    v = ctypes.c_void_p
    assert lib.cd_backward(v(4), v(4), 1, 0, 4, v(4), v(4), None, None, 0.0, 0.0, 0, 0, 0, 4, v(4), v(4), v(256),
                           1 << 30, None) == 1
    assert lib.cd_backward(v(4), v(4), 1, 4, 4, v(4), v(4), None, None, 0.0, 0.0, 0, 5, 0, 4, v(4), v(4), v(256),
                           1 << 30, None) == 1
    assert lib.cd_fscore(v(4), v(4), 1, 4, 4, -0.5, v(4), None, None, v(256), 1 << 20, None) == 1
    assert lib.cd_finalize(None, 1, 4, 4, 1.0, 1.0, None, v(4), None, None, None, None) == 1
    # the loss backward: null upstream scalar, empty cloud, bad slice -> invalid value before any launch
    assert lib.cd_loss_backward(v(4), v(4), 1, 4, 4, v(4), v(4), None, 1.0, 1.0, 0, 4, 0, 4, v(4), v(4), v(256),
                                1 << 30, None) == 1
    assert b"grad_loss" in lib.cd_last_error_string()
    assert lib.cd_loss_backward(v(4), v(4), 1, 0, 4, v(4), v(4), v(4), 1.0, 1.0, 0, 0, 0, 4, v(4), v(4), v(256),
                                1 << 30, None) == 1
    assert lib.cd_loss_backward(v(4), v(4), 1, 4, 4, v(4), v(4), v(4), 1.0, 1.0, 0, 4, 0, 5, v(4), v(4), v(256),
                                1 << 30, None) == 1
    assert lib.cd_p2s_loss_backward(v(4), v(4), v(4), v(4), v(4), 1, 4, 3, 1, None, v(4), v(4), v(256), 1 << 30,
                                    None) == 1


@pytest.mark.skipif(os.environ.get("CUDA_VISIBLE_DEVICES", None) not in (None, "") and False, reason="")
def test_valid_call_without_gpu_reports_cuda_error(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present: covered by the gpu tests")
    assert _forward(lib) in (4, 5)   # no device: CD_ERR_CUDA (or unsupported device)
    assert lib.cd_last_error_string() != b""


def test_python_layer_fails_loudly_without_cuda():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_1911_05063_b200 import api as cd
    with pytest.raises(TypeError):
        cd.forward(torch.zeros(1, 4, 3), torch.zeros(1, 4, 3))
