"""CPU test of the host half of the 2-bit upload path (a1): the AVX-512 / AVX2 / scalar
packer in csrc/hostpack.cu compiled with the host compiler and checked base by base
(tests/cpp/hostpack_test.cpp); no GPU needed."""
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_hostpack_codes_and_validation(tmp_path):
    exe = tmp_path / "hostpack_test"
    csrc = os.path.join(ROOT, "paper_2002_04561_b200", "csrc")
    subprocess.check_call(["g++", "-O2", "-std=c++17", "-x", "c++", "-I", csrc, "-o", str(exe),
                           os.path.join(ROOT, "tests", "cpp", "hostpack_test.cpp"), "-x", "c++",
                           os.path.join(csrc, "hostpack.cu"), "-pthread"])
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "all ok" in out.stdout
