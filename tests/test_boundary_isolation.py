"""The product package never reaches the oracle or the bench harness (task rule ③: only tests/,
__graft_entry__.smoke() and bench.py's CPU legs may touch oracle/), and the oracle shares no
code with the package (it imports nothing but numpy, the standard library and itself)."""
import ast
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_1907_00434_b200")
ORACLE = os.path.join(ROOT, "oracle")


def _imports(path):
    tree = ast.parse(open(path).read(), path)
    out = set()
    for n in ast.walk(tree):
        if isinstance(n, ast.Import):
            out.update(a.name.split(".")[0] for a in n.names)
        elif isinstance(n, ast.ImportFrom):
            out.add("." if n.level else (n.module or "").split(".")[0])
    return out


def _py_files(d):
    for dp, _, fs in os.walk(d):
        for f in fs:
            if f.endswith(".py"):
                yield os.path.join(dp, f)


def test_package_imports_no_oracle_or_bench():
    for f in _py_files(PKG):
        bad = _imports(f) & {"oracle", "bench", "benchkit", "tests"}
        assert not bad, (f, bad)


def test_native_sources_do_not_reference_the_oracle():
    csrc = os.path.join(PKG, "csrc")
    for f in os.listdir(csrc):
        text = open(os.path.join(csrc, f), errors="replace").read()
        assert "oracle/" not in text and "#include \"../../oracle" not in text, f


def test_oracle_imports_only_numpy_stdlib_and_itself():
    allowed = {".", "__future__", "numpy", "fractions", "itertools", "math", "dataclasses", "typing",
               "functools", "collections", "heapq", "bisect", "copy", "oracle"}
    for f in _py_files(ORACLE):
        bad = _imports(f) - allowed
        assert not bad, (f, bad)
