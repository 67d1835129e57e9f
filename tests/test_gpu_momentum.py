"""NEXT-1 on the GPU: momentum commits (Eq. 2, gamma > 0, aggregate form) through the C ABI.

Bitwise against oracle/momentum.weighted_f32 (the same weighted sums in the same fp32
order) and within 1e-6 (norm-relative) of the plain sequential Eq. 2 in float64.
"""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import synthgen as sg  # noqa: E402
from oracle.momentum import sequential_f64, weighted_f32  # noqa: E402
from oracle.numerics import commits_from_plan  # noqa: E402
from tests.test_gpu_parity import SEED, bits, random_plan  # noqa: E402

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_1907_00434_b200 import mlfabric as m
    from paper_1907_00434_b200.harness import Workload
    from synthgen import configs


def run_momentum(S, W, dtype, plan_d, gamma, lr=0.01, h_scale=1e-3):
    os.environ["MLF_COMMIT_IMPL"] = "bulk"
    dev = torch.device("cuda", 0)
    tdt = torch.bfloat16 if dtype == sg.DTYPE_BF16 else torch.float32
    slots = [torch.empty(S, dtype=tdt, device=dev) for _ in range(W)]
    for w, t in enumerate(slots):
        m.synth_fill(0, t.data_ptr(), S, dtype=dtype, seed=SEED, kind=1, a=w, b=0)
    wt = torch.empty(S, dtype=torch.float32, device=dev)
    m.synth_fill(0, wt.data_ptr(), S, dtype=m.MLF_F32, seed=SEED, kind=2)
    h0 = (sg.w0_values(SEED + 1, np.arange(S)) * np.float32(h_scale)).astype(np.float32)
    ht = torch.from_numpy(h0.copy()).to(dev)
    bk = torch.full((S,), float("nan"), device=dev)
    bh = torch.full((S,), float("nan"), device=dev)
    ctx = m.Context(device=0, model_shard=wt, update_slots=slots, lr=lr, model_elems=S, dtype=dtype,
                    backup_shard=bk, stream=torch.cuda.current_stream().cuda_stream, gamma=gamma,
                    history=ht, backup_history=bh)
    for w in range(W):
        ctx.submit(w, 0, 0, 1.0)
    ctx.execute(m.plan_from_dict(plan_d))
    ctx.sync()
    out = (wt.cpu().numpy(), ht.cpu().numpy(), bk.cpu().numpy(), bh.cpu().numpy())
    ctx.close()
    return out, h0


@pytest.mark.parametrize("gamma", [0.5, 0.9])
@pytest.mark.parametrize("dtype", [sg.DTYPE_F32, sg.DTYPE_BF16])
def test_momentum_random_plans(gamma, dtype):
    rng = np.random.default_rng(int(gamma * 10) + dtype)
    for trial in range(6):
        S = int(rng.choice([3, 8, 4099, 65_537, 200_003]))
        W = int(rng.integers(1, 20))
        p = random_plan(rng, W)
        (w, h, b, bh), h0 = run_momentum(S, W, dtype, p, gamma)
        idx = np.arange(S)
        w0 = sg.w0_values(SEED, idx)
        commits = commits_from_plan(p, lambda g: sg.update_values(SEED, g, 0, idx, dtype))
        wr, hr, bkr = weighted_f32(w0, h0, commits, 0.01, gamma, p["replica_boundary_commit"])
        assert np.array_equal(bits(w), bits(wr)) and np.array_equal(bits(h), bits(hr)), (trial, S, W)
        if p["replica_boundary_commit"] >= 0:
            assert np.array_equal(bits(b), bits(bkr[0])) and np.array_equal(bits(bh), bits(bkr[1]))
        else:
            assert np.all(np.isnan(b)) and np.all(np.isnan(bh))
        w64, h64, _ = sequential_f64(w0, h0, commits, 0.01, gamma)
        assert np.max(np.abs(w - w64)) <= 1e-6 * max(np.max(np.abs(w64)), 1e-30)


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_momentum_config2_every_element_vs_sequential_eq2(dtype):
    """The plain definition at full size (R21): config 2, gamma =
    0.9, tau = 32, two batches; EVERY one of the 25.6M elements of w and h on the GPU lies within
    the per-element forward error bound of sequential Eq. 2 in float64 (tests/momentum_bound.py),
    and the norm-relative error max|dw| / max|w64| is <= 1e-6 (the north star's fp32 target)."""
    from oracle.numerics import widen
    from tests.momentum_bound import sequential_with_bound
    cfg = configs.config(2, tau=32, gamma=0.9, dtype=dtype)
    wl = Workload(cfg, device=0)
    S, lr = cfg["S"], cfg["lr"]
    sdt = sg.DTYPE_BF16 if dtype == "bf16" else sg.DTYPE_F32
    plans = []
    for it in range(2):
        pb, pd, draws = wl.step(it)
        wl.ctx.sync()
        plans.append(pd)
    w_gpu = wl.w.cpu().numpy()
    h_gpu = wl.h.cpu().numpy()
    wl.ctx.close()
    assert sum(p["n_commit"] for p in plans) >= 48
    chunk = 1 << 22
    worst_w = worst_h = 0.0
    max_dw = max_w = 0.0
    for lo in range(0, S, chunk):
        idx = np.arange(lo, min(S, lo + chunk))
        w64 = sg.w0_values(cfg["seed"], idx)
        h64 = np.zeros(len(idx), np.float32)
        commits = []
        for it, pd in enumerate(plans):
            commits += commits_from_plan(pd, lambda g, it=it: sg.update_values(cfg["seed"], g, it, idx, sdt))
        w64, h64, bw, bh = sequential_with_bound(w64, h64, commits, lr, 0.9, widen)
        dw = np.abs(w_gpu[idx].astype(np.float64) - w64)
        dh = np.abs(h_gpu[idx].astype(np.float64) - h64)
        assert np.all(dw <= bw), (lo, float(np.max(dw / bw)))
        assert np.all(dh <= bh), (lo, float(np.max(dh / bh)))
        worst_w, worst_h = max(worst_w, float(np.max(dw / bw))), max(worst_h, float(np.max(dh / bh)))
        max_dw, max_w = max(max_dw, float(dw.max())), max(max_w, float(np.abs(w64).max()))
    assert max_dw <= 1e-6 * max_w, (max_dw, max_w)
    print(f"momentum {dtype}: worst |dw|/bound {worst_w:.3f}, |dh|/bound {worst_h:.3f}, "
          f"norm-relative {max_dw / max_w:.2e}")


@pytest.mark.parametrize("dtype,tau", [("f32", 32), ("bf16", 32), ("bf16", 4)])
def test_momentum_config2_full_size(dtype, tau):
    # fp32 takes the generic fold, all-bf16 operand lists the branch-free one (both kernels:
    # dynamic tiles at tau 4, round-robin at tau 32)
    cfg = configs.config(2, tau=tau, gamma=0.9, dtype=dtype)
    wl = Workload(cfg, device=0)
    S = cfg["S"]
    sdt = sg.DTYPE_BF16 if dtype == "bf16" else sg.DTYPE_F32
    rng = np.random.default_rng(9)
    idx = np.unique(np.concatenate([rng.integers(0, S, 20_000), np.arange(S - 9, S)]))
    w_ref = sg.w0_values(cfg["seed"], idx)
    h_ref = np.zeros(len(idx), np.float32)
    for it in range(3):
        pb, pd, draws = wl.step(it)
        wl.ctx.sync()
        commits = commits_from_plan(pd, lambda g: sg.update_values(cfg["seed"], g, it, idx, sdt))
        w_ref, h_ref, _ = weighted_f32(w_ref, h_ref, commits, cfg["lr"], 0.9)
        assert np.array_equal(bits(wl.w.cpu().numpy()[idx]), bits(w_ref))
        assert np.array_equal(bits(wl.h.cpu().numpy()[idx]), bits(h_ref))


def test_momentum_rejects_tree_mode_and_bad_gamma():
    dev = torch.device("cuda", 0)
    w = torch.zeros(64, device=dev)
    with pytest.raises(m.MlfError) as e:
        m.Context(device=0, model_shard=w, update_slots=[w], lr=0.1, model_elems=64, gamma=1.5, history=w)
    assert e.value.code == m.MLF_E_INVALID
    with pytest.raises(m.MlfError) as e:
        m.Context(device=0, model_shard=w, update_slots=[w], lr=0.1, model_elems=64, gamma=0.9)
    assert e.value.code == m.MLF_E_INVALID                 # no history buffer


def test_momentum_under_concurrent_copy_engine_traffic():
    # the momentum ring reuses stages like the commit ring (fence.proxy.async regression)
    S, W, gamma = 16_777_216, 24, 0.9
    rng = np.random.default_rng(5)
    p = random_plan(rng, W, n_commit=W, boundary=-1)
    dev = torch.device("cuda", 0)
    big_src = torch.ones(1 << 28, dtype=torch.float32, device=dev)
    big_dst = torch.empty_like(big_src)
    side = torch.cuda.Stream()
    torch.cuda.synchronize()
    for _ in range(40):                        # ~40 GiB: still running when the commit launches
        m.copy_engine(0, big_dst.data_ptr(), big_src.data_ptr(), big_src.numel() * 4, side.cuda_stream)
    (w, h, _, _), h0 = run_momentum(S, W, sg.DTYPE_F32, p, gamma)
    torch.cuda.synchronize()
    idx = np.unique(np.concatenate([rng.integers(0, S, 200_000), np.arange(S - 9, S)]))
    commits = commits_from_plan(p, lambda g: sg.update_values(SEED, g, 0, idx, sg.DTYPE_F32))
    wr, hr, _ = weighted_f32(sg.w0_values(SEED, idx), h0[idx], commits, 0.01, gamma, -1)
    assert np.array_equal(bits(w[idx]), bits(wr)) and np.array_equal(bits(h[idx]), bits(hr))
