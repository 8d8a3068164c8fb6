"""Race evidence on the GPU (compute-sanitizer is refused on this pool): every kernel
that communicates through shared memory / mbarriers re-runs byte-identically, with and without a
concurrent memory-bound kernel perturbing the timing (tools/race_stress.py; 50 reps there, 6 here)."""
import os
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def test_reruns_byte_identical():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
    import race_stress
    assert race_stress.run(reps=6, verbose=False) == 0
