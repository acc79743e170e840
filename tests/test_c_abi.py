"""The C ABI from a plain C program (tests/c/abi_example.c): the one-call entry points
sif_encode_batched / sif_decode_batched, and the device-side length handoff between them.

CPU: the program compiles and links against include/sif.h + libsif.so (the INTEGRATION.md
binding).  GPU: it runs, and its payloads equal the reference's golden bytes (SURVEY.md
Appendix C: the 1x6 worked example's full hex; random_tensor(32, 32, seed=7) at s=0.9,
M=2/2, q=8, delta=0.01, seed=5 -> 784 bytes, sha256 prefix 160017cefefa418d), and its
decodes equal the oracle's decode of those bytes bit for bit."""

import hashlib
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "c", "abi_example.c")
LIBDIR = os.path.join(ROOT, "paper_2511_11608_b200")
WORKED_HEX = ("53494631010001000000060000000000003f0000000004000000000001000100010000803f000000400200000000000000020000"
              "001080010000803f0000804001000000000000000100000060007fba913f")


def _build(out_dir) -> str:
    import paper_2511_11608_b200.build as b

    b.build()
    exe = os.path.join(str(out_dir), "abi_example")
    cuda = os.environ.get("CUDA_HOME", "/usr/local/cuda")
    cmd = ["gcc", "-O2", "-std=c11", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
           "-I", os.path.join(cuda, "include"), SRC, "-o", exe, "-L", LIBDIR, "-lsif",
           "-L", os.path.join(cuda, "lib64"), "-lcudart", f"-Wl,-rpath,{LIBDIR}"]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return exe


def test_c_caller_compiles_and_links(tmp_path):
    exe = _build(tmp_path)
    assert os.path.exists(exe)


@pytest.mark.gpu
def test_c_caller_matches_reference_bytes(tmp_path):
    from oracle import sif_oracle as O

    exe = _build(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    lines = r.stdout.split("\n")
    assert "ok" in lines
    got = {}
    for ln in lines:
        parts = ln.split()
        if len(parts) == 3 and parts[0] in ("payload", "decoded"):
            got[(parts[0], int(parts[1]))] = bytes.fromhex(parts[2])
    p0, p1 = got[("payload", 0)], got[("payload", 1)]
    assert p0.hex() == WORKED_HEX
    assert len(p1) == 784 and hashlib.sha256(p1).hexdigest()[:16] == "160017cefefa418d"
    for i, p in ((0, p0), (1, p1)):
        ref = O.decode_bytes(p).reshape(-1).view(np.uint32)
        assert np.array_equal(np.frombuffer(got[("decoded", i)], dtype=np.uint32), ref), i
