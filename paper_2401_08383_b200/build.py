"""Build recipe for libexflow_b200.so (nvcc -gencode arch=compute_100a,code=sm_100a)."""
import os
import subprocess

_HERE = os.path.dirname(os.path.abspath(__file__))


def build_library(jobs: int = 8) -> str:
    subprocess.run(["make", "-s", "-j", str(jobs), "-C", os.path.join(_HERE, "csrc")],
                   check=True)
    return os.path.join(_HERE, "libexflow_b200.so")
