"""The C++ drop-in layer (include/ckrl_chunkrl.hpp -> libckrl_host.so): the reference's
known-answer cases restated in C++ (tests/cpp/test_dropin.cpp) through the reference's
signatures and exception types."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "build", "test_dropin")


def _build():
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "paper_2510_06710_b200", "host")], check=True)
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "tests", "cpp")], check=True)


def test_cpp_dropin_builds_and_links():
    """CPU: the header compiles, the library links against libckrl.so, the binary loads."""
    if not os.path.exists(os.path.join(ROOT, "paper_2510_06710_b200", "libckrl.so")):
        pytest.skip("libckrl.so not built")
    _build()
    out = subprocess.run([BIN, "--list"], check=True, capture_output=True, text=True).stdout
    assert "GRPO assembler: frozen slots never enter a trajectory" in out
    assert len(out.splitlines()) >= 20


@pytest.mark.gpu
def test_cpp_dropin_cases():
    if not os.path.exists(BIN):
        _build()
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    print(r.stderr)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]


def test_cpp_dropin_host_formats():
    """CPU: the host-only cases (trajectories dump, CKRL checkpoint) run without a device."""
    if not os.path.exists(os.path.join(ROOT, "paper_2510_06710_b200", "libckrl.so")):
        pytest.skip("libckrl.so not built")
    _build()
    r = subprocess.run([BIN, "dump_slab"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "[ ok ] dump_slab" in r.stdout
