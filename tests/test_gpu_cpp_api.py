"""The C++ operator API as a reference user would call it (tests/cpp/):
compiled with g++ against include/dpb200 and libdpcuda.so, run on the GPU."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_cpp_example_known_answers(tmp_path):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    lib = os.path.join(ROOT, "paper_2101_12127_b200", "lib")
    exe = str(tmp_path / "example")
    subprocess.run(["g++", "-std=c++20", "-O2", f"-I{ROOT}/include", "-I/usr/local/cuda/include",
                    os.path.join(ROOT, "tests", "cpp", "example_operator_api.cpp"), "-o", exe, f"-L{lib}", "-ldpcuda",
                    f"-Wl,-rpath,{lib}", "-L/usr/local/cuda/lib64", "-lcudart"], check=True)
    out = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    # SURVEY.md Appendix A, via the C++ API
    assert "cfg1 root=map_and_batch batches=977 last=576 sum=1499999500000 fnv=8bc444c576bd14a5" in out.stdout
    assert "cfg2 restore_matches=1" in out.stdout
    # the reference's fingerprint of the same graph (golden, from the compiled reference)
    import json
    golden = json.load(open(os.path.join(ROOT, "tests", "golden", "golden.json")))["serialize"][0]
    assert f"fingerprint={golden['fingerprint']} roundtrip=1" in out.stdout
    assert "bucket rows=5000" in out.stdout
    # labels ride through the K9 chain: sum of i % 10 over 512 images
    assert "rrc images=512 label_sum=2296 " in out.stdout, out.stdout
    assert "float32[?,224,224,3]" in out.stdout or "224,224,3" in out.stdout
    assert "metrics /prefetch@0" in out.stdout
