"""C++ drop-in headers (paper_2011_01805_b200/include/tiletensor_b200/*.hpp):
the reference's test expectations compiled against the unchanged
tiletensor:: API and run on the GPU (paper_2011_01805_b200/tests_cpp)."""
import subprocess

import pytest

from paper_2011_01805_b200 import build


def test_host_headers_compile():
    exe = build.build_host_tests()
    assert exe.exists()


@pytest.mark.gpu
def test_host_mirror_suite(gpu):
    exe = build.build_host_tests()
    proc = subprocess.run([str(exe)], capture_output=True, text=True, timeout=600)
    print(proc.stdout)
    print(proc.stderr[-4000:])
    assert proc.returncode == 0, proc.stderr[-4000:]
    assert "0 failed" in proc.stdout
