"""Native C++ unit tests of the host runtime (include/coserve/*.hpp), built with g++."""
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_host_cpp(tmp_path):
    exe = tmp_path / "test_host"
    src = os.path.join(ROOT, "tests", "cpp", "test_host.cpp")
    subprocess.check_call(["g++", "-std=c++17", "-O1", "-Wall", "-Werror", "-fsanitize=address,undefined",
                           "-I" + os.path.join(ROOT, "include"), src, "-o", str(exe)])
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "all host tests passed" in r.stdout
