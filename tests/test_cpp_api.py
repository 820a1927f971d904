"""The C++ host mirror (include/ffdp/voxreg.hpp) through its own parity suite
(tests/cpp/test_voxreg_api.cpp, built by paper_2509_25044_b200/build.py)."""
import os
import subprocess

import pytest

from paper_2509_25044_b200 import build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_cpp_mirror_compiles_against_the_abi():
    """The header-only mirror compiles (-Wall) and links against libffdp.so here (no GPU)."""
    b = build.build_cpp_tests()
    assert os.path.exists(b)


@pytest.mark.gpu
def test_cpp_mirror_parity_suite():
    b = build.build_cpp_tests()
    env = dict(os.environ, FFDP_GOLDEN_NIFTI=os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "nifti"))
    r = subprocess.run([b], capture_output=True, text=True, timeout=600, env=env)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert " 0 failed" in r.stdout


def test_cpp_plan_test_compiles():
    assert os.path.exists(build.build_cpp_plan_test())


@pytest.mark.gpu
def test_cpp_sharded_plan_threads_and_nccl():
    """ffdp_plan_* from C++: in-process groups of 1-4 ranks (threads sharing cuda:0) and
    NCCL at world 1 (world 2 with two devices) against the single-GPU step, bit for bit."""
    b = build.build_cpp_plan_test()
    r = subprocess.run([b], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert " 0 failed" in r.stdout
