"""In-tree build of the native codec library (libsif.so) for sm_100a.

The library is a plain C ABI (include/sif.h) compiled by nvcc; it is loaded with ctypes
by `paper_2511_11608_b200._lib`.  The built .so lives next to this file so it travels
with the repository snapshot to the GPU box."""

import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libsif.so")
SOURCES = ["sif_lib.cu", "sif_enc.cu", "sif_post.cu", "sif_token.cu", "sif_decode.cu", "sif_synth.cu", "sif_common.cuh",
           "sif_crc_tables.cuh"]
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-Xcompiler", "-fPIC", "-shared", "-diag-suppress", "1835"]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(HERE, "csrc", s) for s in SOURCES] + [os.path.join(ROOT, "include", "sif.h")]
    return any(os.path.getmtime(p) > t for p in deps if os.path.exists(p))


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    nvcc = os.environ.get("NVCC", "nvcc")
    cmd = [nvcc, *NVCC_FLAGS, "-I", os.path.join(ROOT, "include"),
           os.path.join(HERE, "csrc", "sif_lib.cu"), "-o", LIB + ".tmp"]
    if verbose:
        print(" ".join(cmd))
    subprocess.run(cmd, check=True)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build(force=True, verbose=True))
