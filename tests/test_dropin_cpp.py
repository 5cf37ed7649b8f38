"""The C++ drop-in (shim/fqf_dropin.cpp, compiled against the reference's own
headers) running the reference's beamform/post tests restated in C++
(shim/test_dropin.cpp)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "shim", "build", "test_dropin")

needs_exe = pytest.mark.skipif(not os.path.exists(EXE), reason="shim not built (needs /root/reference)")


@needs_exe
def test_dropin_links_and_refuses_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    out = subprocess.run([EXE], capture_output=True, text=True, timeout=120)
    assert out.returncode != 0
    assert "no sm_100 (B200) CUDA device available" in out.stdout


@needs_exe
@pytest.mark.gpu
def test_dropin_reference_tests_pass_on_gpu():
    out = subprocess.run([EXE], capture_output=True, text=True, timeout=600)
    print(out.stdout)
    assert out.returncode == 0, out.stdout[-3000:]
