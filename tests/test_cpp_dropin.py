"""The reference's hot-path tests restated in C++ against the drop-in headers
include/shellular/*.hpp (tests/cpp/test_dropin.cpp), driven from pytest."""
import os
import subprocess

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
CPP = os.path.join(HERE, "cpp")
BIN = os.path.join(CPP, "test_dropin")


def build():
    subprocess.run(["make", "-s", "-C", CPP], check=True)
    return BIN


def test_dropin_host_cases():
    """Reference arithmetic reached through the C ABI without device work."""
    out = subprocess.run([build(), "--host"], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert " 0 failed" in out.stdout


@pytest.mark.gpu
def test_dropin_device_cases():
    """Field / mesh / solve / homogenize cases of test_field/voxel/fem.cpp on the device."""
    out = subprocess.run([build()], capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stdout + out.stderr
    assert " 0 failed" in out.stdout
