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


def _mzero_param_offset():
    """c[0x0] offset of MomentumArgs::mzero (the kernel parameter block starts at 0x380 on sm_100,
    where MomentumArgs::lr sits at 0x3b0): the layout of kernels.h's struct, computed here."""
    src = open(os.path.join(ROOT, "paper_1907_00434_b200", "csrc", "kernels.h")).read()
    K = int(re.search(r"kMaxOpsM\s*=\s*(\d+)", src).group(1))
    off = 64 + 8 * K                   # w h backup backup_h n src_off lr n_ops backup_after | op[K]
    off += K                           # flag[K]
    off = (off + 3) // 4 * 4 + 16 * K  # cA cB sh gm
    off = (off + 7) // 8 * 8 + 8       # sched
    return 0x380 + off


def _exact_products_only(lines, mzero_off):
    """Every FFMA2 adds a uniform register last loaded from the mzero parameter (-0.0): then
    fma.rn(a, b, -0) == mul.rn(a, b) bitwise (bulk.cu prod2), i.e. a product, not a fused sum."""
    last_def = {}
    for l in lines:
        m = re.search(r"\bLDCU (UR\d+), c\[0x0\]\[(0x[0-9a-f]+)\]", l)
        if m:
            last_def[m.group(1)] = int(m.group(2), 16)
            continue
        m = re.search(r"\b[A-Z0-9.]+ (UR\d+),", l)   # any other write to a uniform register
        if m and "FFMA2" not in l:
            last_def[m.group(1)] = None
        if re.search(r"\bFFMA2\b", l):
            a = re.search(r"FFMA2 [^;]*, (UR\d+)\.F32 ;", l)
            if not a or last_def.get(a.group(1)) != mzero_off:
                return False
    return True


def test_no_fused_multiply_add_anywhere(sass):
    """No FFMA anywhere; FFMA2 only as the exact packed product of the bf16 momentum fold's
    packed-sum instantiation (fused_commit_momentum_bh<..., true>), whose addend is -0."""
    mz = _mzero_param_offset()
    bad = {}
    for f, lines in sass.items():
        hits = [l.strip() for l in lines if re.search(r"\bFFMA2?\b", l)]
        if not hits:
            continue
        if "fused_commit_momentum_bh" in f and f.endswith("Lb1EEEvNS_12MomentumArgsE") \
                and not any(re.search(r"\bFFMA\b", l) for l in hits) and _exact_products_only(lines, mz):
            continue
        bad[f] = hits[:3]
    assert not bad, f"fused multiply-adds would change the pinned roundings: {bad}"


def test_packed_sum_momentum_fold_uses_exact_products(sass):
    fs = [f for f in sass if "fused_commit_momentum_bh" in f and f.endswith("Lb1EEEvNS_12MomentumArgsE")]
    assert fs, sorted(sass)
    text = "\n".join(sass[fs[0]])
    assert re.search(r"\bFFMA2\b", text) and re.search(r"\bFADD2\b", text)
    assert _exact_products_only(sass[fs[0]], _mzero_param_offset())


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
