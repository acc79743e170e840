"""The product path never routes through the CPU oracle (or any CPU fallback): no module of
the package imports `oracle`, the C ABI library is built from the CUDA sources only, and
importing the package does not load `oracle`."""

import ast
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2511_11608_b200")


def _imports(path):
    tree = ast.parse(open(path).read(), filename=path)
    for node in ast.walk(tree):
        if isinstance(node, ast.Import):
            for a in node.names:
                yield a.name
        elif isinstance(node, ast.ImportFrom):
            yield node.module or ""


def test_package_sources_do_not_import_oracle():
    for dirpath, _dirs, files in os.walk(PKG):
        for fn in files:
            if fn.endswith(".py"):
                p = os.path.join(dirpath, fn)
                bad = [m for m in _imports(p) if m == "oracle" or m.startswith("oracle.")]
                assert not bad, f"{p} imports {bad}"


def test_native_sources_are_cuda_only():
    csrc = os.path.join(PKG, "csrc")
    names = sorted(os.listdir(csrc))
    assert names and all(n.endswith((".cu", ".cuh")) for n in names), names


def test_import_does_not_load_oracle():
    code = "import sys, paper_2511_11608_b200; print(any(m == 'oracle' or m.startswith('oracle.') for m in sys.modules))"
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    assert r.stdout.strip().splitlines()[-1] == "False"
