"""The boundary from plain C99: compile tests/c_abi_check.c against include/mlfabric.h and
link it to libmlfabric.so with gcc, then run it (host-only planner calls; no GPU)."""
import os
import shutil
import subprocess

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(ROOT, "paper_1907_00434_b200", "lib")


@pytest.mark.skipif(shutil.which("gcc") is None, reason="needs gcc")
def test_c99_program_against_the_abi(tmp_path):
    exe = tmp_path / "c_abi_check"
    subprocess.run(["gcc", "-std=c99", "-Wall", "-Wextra", "-Werror", "-I", os.path.join(ROOT, "include"),
                    os.path.join(HERE, "c_abi_check.c"), "-o", str(exe), "-L", LIB, "-lmlfabric",
                    f"-Wl,-rpath,{LIB}"], check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=60)
    assert r.returncode == 0 and "C_ABI_OK" in r.stdout, r.stdout + r.stderr


@pytest.mark.gpu
def test_c99_program_runs_the_hot_path(tmp_path):
    # tests/c_abi_gpu.c: cudaMalloc + mlf_* only; its plan and pulled model vs the oracle
    import numpy as np

    import synthgen as sg
    from oracle.numerics import execute_plan
    from oracle.plan import Item, Params, make_net, plan as oracle_plan

    cuda = os.environ.get("CUDA_HOME", "/usr/local/cuda")
    exe, out = tmp_path / "c_abi_gpu", tmp_path / "out.bin"
    subprocess.run(["gcc", "-std=c99", "-Wall", "-Wextra", "-Werror", "-I", os.path.join(ROOT, "include"),
                    "-I", os.path.join(cuda, "include"), os.path.join(HERE, "c_abi_gpu.c"), "-o", str(exe),
                    "-L", LIB, "-lmlfabric", "-L", os.path.join(cuda, "lib64"), "-lcudart",
                    f"-Wl,-rpath,{LIB}", f"-Wl,-rpath,{os.path.join(cuda, 'lib64')}"], check=True)
    r = subprocess.run([str(exe), str(out)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and "C_GPU_OK" in r.stdout, r.stdout + r.stderr
    W, S, MB, v0 = 6, 100003, 10**6, 40
    raw = out.read_bytes()
    hdr = np.frombuffer(raw, np.int32, 4)
    o = 16
    order = np.frombuffer(raw, np.int32, W, o); o += 4 * W
    drop = np.frombuffer(raw, np.uint8, W, o); o += W
    group = np.frombuffer(raw, np.int32, W, o); o += 4 * W
    cfirst = np.frombuffer(raw, np.int32, W, o); o += 4 * W
    ccount = np.frombuffer(raw, np.int32, W, o); o += 4 * W
    w = np.frombuffer(raw, np.float32, S, o)
    net = make_net(7, [10 * MB, 5 * MB, 10 * MB, 5 * MB // 2, 10 * MB, 1 * MB, 0], [0] * 6 + [10 * MB])
    batch = [Item(i, S * 4, v0, 0, 1.0) for i in range(W)]
    p = oracle_plan(net, batch, Params(servers=[6], aggs=[0, 2], v_init=v0, tau_max=4))
    n, nc = int(hdr[0]), int(hdr[1])
    assert n == p["n_commit"] and list(order[:n]) == p["order"] and list(drop) == p["drop_reason"]
    assert list(group) == p["group"] and nc == p["n_server_commits"]
    assert list(cfirst[:nc]) == p["commit_first"] and list(ccount[:nc]) == p["commit_count"]
    assert int(hdr[2]) == n and int(hdr[3]) == 1            # version += n_commit; one fused launch
    idx = np.arange(S)
    wr, _, _ = execute_plan(sg.w0_values(0x4D4C46, idx), p,
                            lambda g: sg.update_values(0x4D4C46, g, 0, idx, sg.DTYPE_F32), 0.01)
    assert np.array_equal(w.view(np.uint32), wr.view(np.uint32))
