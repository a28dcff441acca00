"""The C++ convlow API (drop-in for the reference's include/convlow/*.hpp),
built against libconvlow.so and run as a native test program
(tests/cpp/test_convlow.cpp): `cpu` mode here, `gpu` mode on the B200."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "build", "test_convlow")


def _build():
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "tests", "cpp")], check=True)


def test_cpp_api_cpu():
    _build()
    r = subprocess.run([BIN, "cpu"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.gpu
def test_cpp_api_gpu():
    _build()
    r = subprocess.run([BIN, "gpu"], capture_output=True, text=True, timeout=900)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
