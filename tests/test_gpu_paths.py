"""Randomised cross-check of the four forward paths (fused, per-direction, tensor-core filter, pruned):
bit-identical distances, indices and hit counts on random shapes and adversarial distributions
(duplicates, far clusters, dyadic lattices with exact ties, scaled and offset clouds), and a
deterministic backward.  The same generator as tools/stress.py (run there with 1500 draws)."""
import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_forward_paths_agree_random():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "stress.py"), "60", "3"], capture_output=True,
                       text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    assert "60 draws, 0 failures" in r.stdout, r.stdout[-3000:]
