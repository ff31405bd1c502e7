"""The C ABI as a reference maintainer would consume it, on CPU:
compass_moe.h compiles together with the reference's compass_lab.h in either include order, as
C++ and as C (compass_lab.h defines cl_status unguarded; compass_moe.h includes it when it is on
the include path), and the runnable consumer (tests/integration/consumer.cpp) builds and links
against libcompass_moe.so. Running it needs a GPU: tests/test_gpu_integration.py."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_INC = "/root/reference/proj/include"
INC = os.path.join(ROOT, "include")


@pytest.mark.skipif(not os.path.exists(os.path.join(REF_INC, "compass_lab.h")), reason="reference headers absent")
@pytest.mark.parametrize("lang", ["c++", "c"])
@pytest.mark.parametrize("lab_first", [True, False])
def test_headers_compile_in_either_order(lang, lab_first):
    cc = "g++" if lang == "c++" else "gcc"
    std = "-std=c++17" if lang == "c++" else "-std=c11"
    cmd = [cc, "-x", lang, std, "-Wall", "-Werror", "-fsyntax-only", f"-I{INC}", f"-I{REF_INC}",
           os.path.join(ROOT, "tests", "integration", "include_order.cpp")] + (["-DLAB_FIRST"] if lab_first else [])
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


def test_consumer_builds_and_links(tmp_path):
    lib = os.path.join(ROOT, "paper_2509_09121_b200", "libcompass_moe.so")
    if not os.path.exists(lib) or not shutil.which("g++"):
        pytest.skip("library not built")
    extra = [f"-I{REF_INC}", "-DCOMPASS_HAVE_LAB"] if os.path.exists(os.path.join(REF_INC, "compass_lab.h")) else []
    exe = str(tmp_path / "consumer")
    r = subprocess.run(["g++", "-std=c++17", "-O1", "-Wall", "-Werror", f"-I{INC}", *extra,
                        os.path.join(ROOT, "tests", "integration", "consumer.cpp"), lib,
                        f"-Wl,-rpath,{os.path.dirname(lib)}", "-o", exe], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
