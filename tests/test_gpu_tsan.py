"""ThreadSanitizer over the host runtime (the lock-free
lease / slot-release path had no TSAN run).  tests/cpp/stress_threads.cpp --
three threads calling GetNext on one iterator, three threads dropping the
batches after consumer-stream work, one thread taking checkpoints and
Metrics() -- is built with -fsanitize=thread against the TSAN build of the
engine (`make -C paper_2101_12127_b200/csrc tsan`) and must deliver every
batch exactly once with no data race reported in the engine's code."""
import os
import re
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_2101_12127_b200", "csrc")
TSAN_LIB = os.path.join(ROOT, "paper_2101_12127_b200", "build", "tsan")


def test_runtime_threads_under_tsan(tmp_path):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    subprocess.run(["make", "-C", CSRC, "-j8", "tsan"], check=True, capture_output=True)
    exe = str(tmp_path / "stress")
    subprocess.run(["g++", "-std=c++20", "-O1", "-g", "-fsanitize=thread", f"-I{ROOT}/include",
                    "-I/usr/local/cuda/include", os.path.join(ROOT, "tests", "cpp", "stress_threads.cpp"), "-o", exe,
                    f"-L{TSAN_LIB}", "-ldpcuda", f"-Wl,-rpath,{TSAN_LIB}", "-L/usr/local/cuda/lib64", "-lcudart"],
                   check=True)
    env = dict(os.environ, TSAN_OPTIONS="halt_on_error=0 exitcode=0 report_signal_unsafe=0")
    out = subprocess.run([exe], capture_output=True, text=True, timeout=900, env=env)
    assert "stress ok" in out.stdout, out.stdout + out.stderr[-4000:]
    # data races whose stacks touch the engine's own sources
    reports = out.stderr.split("==================")
    ours = [r for r in reports if "ThreadSanitizer: data race" in r and re.search(r"csrc/(engine/)?\w+\.(cpp|hpp|cu)", r)]
    assert not ours, ours[0][:6000]
