"""Build liblopc.so in-tree with nvcc for sm_100a (no torch JIT cache)."""
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "csrc")
SO = os.path.join(HERE, "liblopc.so")
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-fmad=false", "-std=c++17",
              "-Xcompiler", "-fPIC", "-shared"]


def sources():
    return [os.path.join(SRC, f) for f in sorted(os.listdir(SRC))] + [
        os.path.join(os.path.dirname(HERE), "include", "lopc.h")]


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and os.path.exists(SO) and os.path.getmtime(SO) >= max(os.path.getmtime(p) for p in sources()):
        return SO
    cmd = ["nvcc", *NVCC_FLAGS, "-o", SO, os.path.join(SRC, "lopc_api.cu")]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    subprocess.check_call(cmd)
    return SO


if __name__ == "__main__":
    build(force=True, verbose=True)
