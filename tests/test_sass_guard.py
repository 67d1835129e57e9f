"""Static checks on the built sm_100a code (no GPU): the pinned rounding order and the TMA path.

The parity bar is bitwise, and it holds only if every multiply and add of the commit path is
rounded on its own (R17: two IEEE roundings per commit member).  A fused multiply-add anywhere
in the library (FFMA, or FFMA2 from ptxas contracting packed mul.rn.f32x2 + add.rn.f32x2)
would round once; the GPU tests would catch a mismatch only on inputs where it shows.  This
reads the SASS instead.  It also checks that the bulk kernels really issue TMA bulk copies and
mbarrier waits (B200_PROFILING.md's SASS mnemonics)."""
import os
import re
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_1907_00434_b200", "lib", "libmlfabric.so")
CUOBJDUMP = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"


@pytest.fixture(scope="module")
def sass():
    if not os.path.exists(LIB):
        pytest.skip("libmlfabric.so not built (run __graft_entry__.build())")
    if not os.path.exists(CUOBJDUMP):
        pytest.skip("needs cuobjdump")
    r = subprocess.run([CUOBJDUMP, "-sass", LIB], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    funcs, cur = {}, None
    for line in r.stdout.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            cur = m.group(1)
            funcs[cur] = []
        elif cur is not None:
            funcs[cur].append(line)
    assert funcs, "no device functions in the library"
    return funcs


def test_no_fused_multiply_add_anywhere(sass):
    bad = {f: [l.strip() for l in lines if re.search(r"\bFFMA2?\b", l)] for f, lines in sass.items()}
    bad = {f: v[:3] for f, v in bad.items() if v}
    assert not bad, f"fused multiply-adds would change the pinned roundings: {bad}"


def test_bulk_kernels_use_tma_and_mbarriers(sass):
    bulk = {f: lines for f, lines in sass.items() if "fused_commit_bulk" in f or "tree_reduce_bulk" in f
            or "fused_commit_momentum" in f}
    assert len(bulk) >= 5, sorted(sass)
    for f, lines in bulk.items():
        text = "\n".join(lines)
        assert "UBLKCP" in text, f"{f}: no TMA bulk copy"
        assert "SYNCS" in text, f"{f}: no mbarrier operations"


def test_packed_products_in_the_bf16_momentum_fold(sass):
    fs = [f for f in sass if "fused_commit_momentum_rr" in f and "Lb1E" in f]
    assert fs, sorted(sass)
    assert any(re.search(r"\bFMUL2\b", l) for l in sass[fs[0]])
