"""C++ drop-in headers (paper_2011_01805_b200/include/tiletensor_b200/*.hpp):
the reference's test expectations compiled against the unchanged
tiletensor:: API and run on the GPU (paper_2011_01805_b200/tests_cpp)."""
import subprocess

import pytest

from paper_2011_01805_b200 import build


def test_host_headers_compile():
    exe = build.build_host_tests()
    assert exe.exists()


def test_reference_include_names_compile(tmp_path):
    """A reference user's source, #include lines unchanged, builds against the
    drop-in headers (paper_2011_01805_b200/include/tiletensor/*.hpp forward to
    tiletensor_b200/*.hpp)."""
    src = tmp_path / "user.cpp"
    src.write_text(
        '#include "tiletensor/backend.hpp"\n#include "tiletensor/dense.hpp"\n'
        '#include "tiletensor/linalg.hpp"\n#include "tiletensor/nn.hpp"\n'
        '#include "tiletensor/rotate_sum.hpp"\n#include "tiletensor/shape.hpp"\n'
        '#include "tiletensor/tile_tensor.hpp"\n'
        "using namespace tiletensor;\n"
        "int main() { Session s(8192, 8); auto sh = parse_shape(\"[512/16,1024/32,*/16]\");\n"
        "  return format_shape(sh).empty() ? 1 : 0; }\n")
    root = build.ROOT
    proc = subprocess.run(["g++", "-std=c++20", "-fsyntax-only", "-I", str(root / "include"),
                           "-I", str(build.PKG / "include"), str(src)], capture_output=True, text=True)
    assert proc.returncode == 0, proc.stderr[-2000:]


@pytest.mark.gpu
def test_host_mirror_suite(gpu):
    exe = build.build_host_tests()
    proc = subprocess.run([str(exe)], capture_output=True, text=True, timeout=600)
    print(proc.stdout)
    print(proc.stderr[-4000:])
    assert proc.returncode == 0, proc.stderr[-4000:]
    assert "0 failed" in proc.stdout
