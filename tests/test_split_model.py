"""CPU check of the tcgen05 engine's K-split cost model (mma_launch.cuh) on the bench
shapes, compiled host-only with nvcc: the choices DESIGN.md documents (HBM-bound
small batches take no extra split, C4 B = 64 four, the hint two, FTR twelve exact
splits; a forced split never drops below the exactness minimum)."""
import os
import shutil
import subprocess
import tempfile

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.mark.skipif(shutil.which("nvcc") is None, reason="nvcc not available")
def test_split_choices():
    with tempfile.TemporaryDirectory() as tmp:
        exe = os.path.join(tmp, "split_model")
        subprocess.run(["nvcc", "-std=c++17", "-O2", "-o", exe,
                        os.path.join(HERE, "native", "split_model.cu")],
                       check=True, capture_output=True, timeout=300)
        out = subprocess.run([exe], check=True, capture_output=True, text=True).stdout
    got = dict(line.split() for line in out.strip().splitlines())
    assert got == {"c2_b4": "1", "c2_b64": "1", "c4_b64": "4", "c4_b256": "1", "c5": "2",
                   "ftr": "12", "forced": "7", "forced_min": "5"}, got
