"""Build recipe for libffdp.so (sm_100a) and the test oracle libraries.

    python -m paper_2509_25044_b200.build          # libffdp.so (+ oracle, + oracle/_ref if possible)

nvcc cross-compiles without a GPU. The .so files are written in-tree so they travel
with the gpurun snapshot; they are git-ignored.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
SOURCES = ["capi.cu", "sampler.cu", "lncc.cu", "mi.cu", "step_lncc.cu", "step_lncc2.cu", "step_lncc3.cu", "step_mi.cu", "smooth.cu", "resample.cu", "comm.cu", "plan.cu"]
LIB = os.path.join(HERE, "libffdp.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-fvisibility=hidden", "-shared"]


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build_lib(force: bool = False, verbose: bool = False) -> str:
    """One object per source (compiled in parallel, rebuilt when the source or a shared
    header changed), then one nvcc link into libffdp.so."""
    from concurrent.futures import ThreadPoolExecutor
    srcs = [os.path.join(CSRC, s) for s in SOURCES]
    headers = [os.path.join(CSRC, "ffdp_common.cuh"), os.path.join(ROOT, "include", "ffdp.h")]
    objdir = os.path.join(HERE, "build_obj")
    os.makedirs(objdir, exist_ok=True)
    objs = [os.path.join(objdir, os.path.basename(s)[:-3] + ".o") for s in srcs]
    cflags = [f for f in NVCC_FLAGS if f != "-shared"]

    def one(so):
        src, obj = so
        if force or _stale(obj, [src] + headers):
            cmd = [nvcc()] + cflags + ["-c", "-o", obj, src]
            if verbose:
                print(" ".join(cmd))
            subprocess.run(cmd, check=True)

    with ThreadPoolExecutor(max_workers=min(len(srcs), os.cpu_count() or 1)) as ex:
        list(ex.map(one, zip(srcs, objs)))
    if force or _stale(LIB, objs):
        cmd = [nvcc()] + ARCH + ["-shared", "-o", LIB] + objs + ["-ldl"]
        if verbose:
            print(" ".join(cmd))
        subprocess.run(cmd, check=True)
    return LIB


def build_oracle(verbose: bool = False) -> None:
    """The parity checker (test infrastructure): C restatement always, reference shim
    when /root/reference is present (prebuilt copies travel to the GPU box)."""
    od = os.path.join(ROOT, "oracle")
    subprocess.run(["make", "-s", "-C", od, "all"], check=True)
    if os.path.isdir("/root/reference/proj/include"):
        subprocess.run(["make", "-s", "-C", od, "ref"], check=True)


CPP_TEST_SRC = os.path.join(ROOT, "tests", "cpp", "test_voxreg_api.cpp")
CPP_TEST_BIN = os.path.join(ROOT, "tests", "cpp", "test_voxreg_api")


def build_cpp_tests(force: bool = False, verbose: bool = False) -> str:
    """The C++ parity suite of the host mirror (include/ffdp/voxreg.hpp), linked against
    libffdp.so and the oracle (test infrastructure) with $ORIGIN-relative rpaths."""
    cuda = os.path.dirname(os.path.dirname(nvcc()))
    deps = [CPP_TEST_SRC, os.path.join(ROOT, "include", "ffdp", "voxreg.hpp"),
            os.path.join(ROOT, "include", "ffdp", "nifti.hpp"), os.path.join(ROOT, "include", "ffdp.h"),
            LIB, os.path.join(ROOT, "oracle", "libffdp_oracle.so")]
    if force or _stale(CPP_TEST_BIN, deps):
        cmd = ["g++", "-O2", "-std=c++17", "-Wall", "-I" + os.path.join(ROOT, "include"),
               "-I" + os.path.join(cuda, "include"), CPP_TEST_SRC, "-o", CPP_TEST_BIN,
               "-L" + HERE, "-L" + os.path.join(ROOT, "oracle"), "-L" + os.path.join(cuda, "lib64"),
               "-lffdp", "-lffdp_oracle", "-lcudart",
               "-Wl,-rpath,$ORIGIN/../../paper_2509_25044_b200:$ORIGIN/../../oracle:" + os.path.join(cuda, "lib64")]
        if verbose:
            print(" ".join(cmd))
        subprocess.run(cmd, check=True)
    return CPP_TEST_BIN


def build_ref_backend(verbose: bool = False) -> None:
    """The reference's own driver linked through integration/voxreg/ffdp_backend.hpp
    (oracle/_ref/test_ref_backend; test infrastructure, needs /root/reference)."""
    if os.path.isdir("/root/reference/proj/include"):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "ref-backend"], check=True)


CPP_PLAN_SRC = os.path.join(ROOT, "tests", "cpp", "test_plan.cpp")
CPP_PLAN_BIN = os.path.join(ROOT, "tests", "cpp", "test_plan")


def build_cpp_plan_test(force: bool = False, verbose: bool = False) -> str:
    """The native sharded plan from C++ with one std::thread per rank (tests/cpp/test_plan.cpp)."""
    cuda = os.path.dirname(os.path.dirname(nvcc()))
    deps = [CPP_PLAN_SRC, os.path.join(ROOT, "include", "ffdp", "voxreg.hpp"), os.path.join(ROOT, "include", "ffdp.h"),
            LIB]
    if force or _stale(CPP_PLAN_BIN, deps):
        cmd = ["g++", "-O2", "-std=c++17", "-Wall", "-I" + os.path.join(ROOT, "include"),
               "-I" + os.path.join(cuda, "include"), CPP_PLAN_SRC, "-o", CPP_PLAN_BIN, "-L" + HERE,
               "-L" + os.path.join(cuda, "lib64"), "-lffdp", "-lcudart", "-lpthread",
               "-Wl,-rpath,$ORIGIN/../../paper_2509_25044_b200:" + os.path.join(cuda, "lib64")]
        if verbose:
            print(" ".join(cmd))
        subprocess.run(cmd, check=True)
    return CPP_PLAN_BIN


def build_all(verbose: bool = False) -> None:
    build_lib(verbose=verbose)
    build_oracle(verbose=verbose)
    build_cpp_tests(verbose=verbose)
    build_cpp_plan_test(verbose=verbose)
    build_ref_backend(verbose=verbose)


if __name__ == "__main__":
    build_all(verbose="-v" in sys.argv)
    print("built", LIB)
