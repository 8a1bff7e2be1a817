"""Test-only in-process NCCL stand-in (mock_nccl.cpp): build() compiles it next to this file."""
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "libmock_nccl.so")


def build():
    src = os.path.join(HERE, "mock_nccl.cpp")
    if not os.path.exists(SO) or os.path.getmtime(SO) < os.path.getmtime(src):
        subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-shared", "-Xcompiler", "-fPIC", "-std=c++17",
                               "-x", "cu", "-o", SO, src])
    return SO
