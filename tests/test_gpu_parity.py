"""GPU parity: the CUDA path (through the C ABI) vs the oracle, element by element.

Bit-exact in pinned-order mode (R17): the kernel folds each commit's members
left to right in O(U) order with fp32 adds and applies w - (lr*x) with two
roundings, exactly like oracle/numerics.py, so fp32 and bf16 results must be
memcmp-equal; the exact-arithmetic variant additionally equals the exact rational
result for ANY order (data movement pinned independently of order).
"""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import synthgen as sg  # noqa: E402
from oracle.numerics import commit_batch, execute_plan  # noqa: E402
from oracle.plan import Item, Params, make_net, plan as oracle_plan  # noqa: E402

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_1907_00434_b200 import mlfabric as m
    from paper_1907_00434_b200.harness import Workload
    from synthgen import configs

SEED = 0x4D4C46


def bits(a):
    return np.ascontiguousarray(a).view(np.uint32)


def gpu_run(S, W, dtype, plan_d, *, lr=0.01, variant=0, iteration=0, backup=False, host_updates=False,
            impl="ldg", device=0):
    """Fill W slots + w0 on cuda:<device> with the generator, submit every worker, execute plan_d."""
    with torch.cuda.device(device):
        return _gpu_run(S, W, dtype, plan_d, lr, variant, iteration, backup, host_updates, impl, device)


def _gpu_run(S, W, dtype, plan_d, lr, variant, iteration, backup, host_updates, impl, device):
    os.environ["MLF_COMMIT_IMPL"] = impl                     # read at mlf_init
    dev = torch.device("cuda", device)
    tdt = torch.bfloat16 if dtype == sg.DTYPE_BF16 else torch.float32
    slots = [torch.empty(S, dtype=tdt, device=dev) for _ in range(W)]
    for w, t in enumerate(slots):
        m.synth_fill(device, t.data_ptr(), S, dtype=dtype, seed=SEED, kind=1, a=w, b=iteration, variant=variant)
    wt = torch.empty(S, dtype=torch.float32, device=dev)
    m.synth_fill(device, wt.data_ptr(), S, dtype=m.MLF_F32, seed=SEED, kind=2, variant=variant)
    bk = torch.full((S,), float("nan"), dtype=torch.float32, device=dev) if backup else None
    hosts = []
    if host_updates:
        for t in slots:
            hosts.append(t.cpu().pin_memory())
            t.zero_()
    ctx = m.Context(device=device, model_shard=wt, update_slots=slots, lr=lr, model_elems=S, dtype=dtype,
                    backup_shard=bk, stream=torch.cuda.current_stream(dev).cuda_stream)
    for w in range(W):
        ctx.submit(w, 0, 0, 1.0)
        if host_updates:
            ctx.set_update_host(w, hosts[w].data_ptr())
    pb = m.plan_from_dict(plan_d)
    ctx.execute(pb)
    ms = ctx.sync()
    out = wt.cpu().numpy()
    b = bk.cpu().numpy() if backup else None
    stats = ctx.stats()
    ctx.close()
    return out, b, ms, stats


def oracle_run(S, dtype, plan_d, *, lr=0.01, variant=0, iteration=0, idx=None):
    idx = np.arange(S) if idx is None else idx
    w0 = sg.w0_values(SEED, idx, ["normal", "exact"][variant])
    op = lambda g: sg.update_values(SEED, g, iteration, idx, dtype, ["normal", "exact"][variant])  # noqa: E731
    w, b, _ = execute_plan(w0, plan_d, op, lr)
    return w, b


def random_plan(rng, W, n_commit=None, max_group=4, boundary=None):
    n_commit = int(rng.integers(0, W + 1)) if n_commit is None else n_commit
    order = [int(x) for x in rng.permutation(W)[:n_commit]]
    first, count, pos = [], [], 0
    n_direct = int(rng.integers(0, n_commit + 1))
    for _ in range(n_direct):
        first.append(pos)
        count.append(1)
        pos += 1
    gid = 0
    group = [-1] * W
    for g in order[:n_direct]:
        group[g] = 0
    while pos < n_commit:
        c = int(min(rng.integers(1, max_group + 1), n_commit - pos))
        gid += 1
        first.append(pos)
        count.append(c)
        for q in range(pos, pos + c):
            group[order[q]] = gid
        pos += c
    if boundary is None:
        boundary = int(rng.integers(-1, len(first) + 1))
    return {"n_commit": n_commit, "order": order, "drop_reason": [0 if group[g] >= 0 else 1 for g in range(W)],
            "group": group, "n_direct": n_direct, "n_groups": gid, "group_node": [0] * gid,
            "n_server_commits": len(first), "commit_first": first, "commit_count": count,
            "replica_boundary_commit": boundary, "n_punted": 0, "punted": []}


def test_synth_fill_matches_generator():
    dev = torch.device("cuda", 0)
    n, off = 100_003, 12_345_678
    for dtype, tdt in ((sg.DTYPE_F32, torch.float32), (sg.DTYPE_BF16, torch.bfloat16)):
        for variant, vn in ((0, "normal"), (1, "exact")):
            t = torch.empty(n, dtype=tdt, device=dev)
            m.synth_fill(0, t.data_ptr(), n, elem_offset=off, dtype=dtype, seed=SEED, kind=1, a=7, b=3,
                         variant=variant)
            ref = sg.update_values(SEED, 7, 3, np.arange(off, off + n), dtype, vn)
            got = t.cpu().view(torch.int16 if dtype else torch.int32).numpy()
            assert np.array_equal(got.view(ref.dtype), ref)
    t = torch.empty(n, dtype=torch.float32, device=dev)
    m.synth_fill(0, t.data_ptr(), n, elem_offset=off, dtype=0, seed=SEED, kind=2)
    assert np.array_equal(bits(t.cpu().numpy()), bits(sg.w0_values(SEED, np.arange(off, off + n))))


IMPLS = ["ldg", "bulk"]


@pytest.mark.parametrize("impl", IMPLS)
@pytest.mark.parametrize("dtype", [sg.DTYPE_F32, sg.DTYPE_BF16])
def test_random_plans_bitwise(dtype, impl):
    rng = np.random.default_rng(dtype + 11)
    for trial in range(8):
        S = int(rng.choice([1, 3, 4, 9, 257, 2055, 4099, 65_537, 300_001]))
        W = int(rng.integers(1, 24))
        p = random_plan(rng, W)
        w, b, _, _ = gpu_run(S, W, dtype, p, backup=True, impl=impl)
        wr, br = oracle_run(S, dtype, p)
        assert np.array_equal(bits(w), bits(wr)), (trial, S, W)
        if p["replica_boundary_commit"] >= 0:
            assert np.array_equal(bits(b), bits(br))
        else:
            assert np.all(np.isnan(b))                     # no replica write


@pytest.mark.parametrize("tile", [1024, 2048, 4096, 8192])
@pytest.mark.parametrize("dtype", [sg.DTYPE_F32, sg.DTYPE_BF16])
def test_bulk_tiles_bitwise(tile, dtype):
    # every tile instantiation the adaptive choice can pick (1024 / 2048 / 4096) and the
    # 8192 override, with several tiles per CTA, ragged last tiles and a mirror boundary
    rng = np.random.default_rng(tile + dtype)
    os.environ["MLF_BULK_TILE"] = str(tile)
    try:
        for S in (tile * 148 * 3 + 4 * 97 + 5, 1_000_003):
            W = int(rng.integers(3, 20))
            p = random_plan(rng, W, n_commit=W, boundary=1)
            w, b, _, _ = gpu_run(S, W, dtype, p, backup=True, impl="bulk")
            wr, br = oracle_run(S, dtype, p)
            assert np.array_equal(bits(w), bits(wr)), (tile, S)
            assert np.array_equal(bits(b), bits(br)), (tile, S)
    finally:
        del os.environ["MLF_BULK_TILE"]


@pytest.mark.parametrize("dtype", [sg.DTYPE_F32, sg.DTYPE_BF16])
def test_bulk_contiguous_ranges_bitwise(dtype):
    # MLF_BULK_SCHED=contig: every CTA walks one contiguous range (ends not tile-aligned, ranges
    # shorter than a tile, ragged tails) — same bits as the oracle, mirror included
    rng = np.random.default_rng(77 + dtype)
    os.environ["MLF_BULK_SCHED"] = "contig"
    try:
        for S in (1, 9, 4099, 148 * 8 * 3 + 5, 300_001, 6_400_017):
            W = int(rng.integers(2, 20))
            p = random_plan(rng, W, n_commit=W, boundary=1)
            w, b, _, _ = gpu_run(S, W, dtype, p, backup=True, impl="bulk")
            wr, br = oracle_run(S, dtype, p)
            assert np.array_equal(bits(w), bits(wr)), S
            assert np.array_equal(bits(b), bits(br)), S
    finally:
        del os.environ["MLF_BULK_SCHED"]


@pytest.mark.parametrize("boundary", [0, 2, -1])
def test_bf16_16kb_layout_bitwise(boundary):
    # all-bf16 operand lists large enough for the 8192-element layout (16 KB bf16 copies, w
    # over two stages): bitwise equal to the 4096-element kernel on every element and to the
    # oracle on a sample, ragged tail and mirror boundary included
    rng = np.random.default_rng(77 + boundary)
    S, W = 8192 * 148 * 16 + 4 * 1237 + 5, 9
    p = random_plan(rng, W, n_commit=W, boundary=boundary)
    w_h, b_h, _, _ = gpu_run(S, W, sg.DTYPE_BF16, p, backup=True, impl="bulk")
    os.environ["MLF_BULK_BF16"] = "0"
    try:
        w_s, b_s, _, _ = gpu_run(S, W, sg.DTYPE_BF16, p, backup=True, impl="bulk")
    finally:
        del os.environ["MLF_BULK_BF16"]
    assert np.array_equal(bits(w_h), bits(w_s))
    assert np.array_equal(bits(b_h), bits(b_s)) if boundary >= 0 else np.all(np.isnan(b_h))
    idx = np.unique(np.concatenate([rng.integers(0, S, 100_000), np.arange(S - 13, S), np.arange(0, 9)]))
    wr, br = oracle_run(S, sg.DTYPE_BF16, p, idx=idx)
    assert np.array_equal(bits(w_h[idx]), bits(wr))
    if boundary >= 0:
        assert np.array_equal(bits(b_h[idx]), bits(br))


def test_distribution_on_one_gpu():
    # NEXT-4 with world = 1: the single view is filled from the single shard (ragged length)
    dev = torch.device("cuda", 0)
    S = 3_000_017
    w = torch.empty(S, dtype=torch.float32, device=dev)
    m.synth_fill(0, w.data_ptr(), S, dtype=m.MLF_F32, seed=SEED, kind=2)
    view = torch.full((-(-S // 64) * 64,), float("nan"), device=dev)
    ctx = m.Context(device=0, model_shard=w, update_slots=[], lr=0.0, model_elems=S, node_rank=[0], n_nodes=1,
                    stream=torch.cuda.current_stream().cuda_stream)
    dp = m.plan_distribution(1, [10**9], [10**9], [0, 0, 0], [0], S * 4)
    assert dp["n_direct"] == 3 and dp["t_total_ns"] == 0        # same node: zero-time pulls
    src = ctx.distribute(dp, [0, 0, 0], [view.data_ptr()], [w.data_ptr()], [0], [S])
    ctx.sync()
    assert src == -1 and torch.equal(view[:S].view(torch.int32), w.view(torch.int32))
    ctx.close()


def test_many_batches_dynamic_tile_counters():
    # 300 launches on one context with operand counts that switch between dynamic and
    # round-robin tiles (and between tile sizes): the tile counters must be back at zero before
    # every launch, or some tiles would be skipped or done twice
    dev = torch.device("cuda", 0)
    S, W, B = 20_000_003, 8, 300                      # 4096-element tiles: n >= 3 operands -> dynamic
    rng = np.random.default_rng(300)
    slots = [torch.empty(S, dtype=torch.float32, device=dev) for _ in range(W)]
    for k, t in enumerate(slots):
        m.synth_fill(0, t.data_ptr(), S, dtype=m.MLF_F32, seed=SEED, kind=1, a=k, b=0)
    wt = torch.empty(S, dtype=torch.float32, device=dev)
    m.synth_fill(0, wt.data_ptr(), S, dtype=m.MLF_F32, seed=SEED, kind=2)
    os.environ["MLF_COMMIT_IMPL"] = "bulk"
    ctx = m.Context(device=0, model_shard=wt, update_slots=slots, lr=0.01, model_elems=S,
                    stream=torch.cuda.current_stream().cuda_stream)
    idx = np.unique(np.concatenate([rng.integers(0, S, 20_000), np.arange(S - 9, S), np.arange(0, 9)]))
    ops = {k: sg.update_values(SEED, k, 0, idx, sg.DTYPE_F32) for k in range(W)}
    w_ref = sg.w0_values(SEED, idx)
    for b in range(B):
        n = int(rng.integers(1, W + 1))
        p = random_plan(rng, W, n_commit=n, boundary=-1)
        for k in range(W):
            ctx.submit(k, 0, 0, 1.0)
        ctx.execute(m.plan_from_dict(p))
        ctx.sync()
        w_ref, _, _ = execute_plan(w_ref, p, lambda g: ops[g], 0.01)
    assert np.array_equal(bits(wt.cpu().numpy()[idx]), bits(w_ref))
    ctx.close()


def test_double_buffered_batches_overlap_and_stay_exact():
    # two slot sets with host-resident updates: batch s+1 is submitted and its H2D starts
    # (mlf_release(ctx, 1)) while batch s still commits; the model after every batch equals
    # the oracle's sequential commits, and the pulled host copy matches the device model
    dev = torch.device("cuda", 0)
    S, W, B = 1_000_003, 6, 5
    slots = [torch.empty(S, dtype=torch.float32, device=dev) for _ in range(2 * W)]
    hosts = [torch.empty(S, dtype=torch.float32).pin_memory() for _ in range(2 * W)]
    wt = torch.empty(S, dtype=torch.float32, device=dev)
    m.synth_fill(0, wt.data_ptr(), S, dtype=m.MLF_F32, seed=SEED, kind=2)
    pulled = torch.empty(S, dtype=torch.float32).pin_memory()
    os.environ["MLF_COMMIT_IMPL"] = "bulk"
    ctx = m.Context(device=0, model_shard=wt, update_slots=slots, lr=0.01, model_elems=S,
                    worker_node=[i % W for i in range(2 * W)], n_nodes=W, node_rank=[0] * W,
                    stream=torch.cuda.current_stream().cuda_stream)
    for i in range(2 * W):
        ctx.set_update_host(i, hosts[i].data_ptr())
    ctx.set_pull_host(pulled.data_ptr())
    idx = np.unique(np.concatenate([np.random.default_rng(3).integers(0, S, 50_000), np.arange(S - 7, S)]))
    w_ref = sg.w0_values(SEED, idx)
    plan = {"n_commit": W, "order": list(range(W)), "drop_reason": [0] * W, "group": [0] * W, "n_direct": W,
            "n_groups": 0, "group_node": [], "n_server_commits": W, "commit_first": list(range(W)),
            "commit_count": [1] * W, "replica_boundary_commit": -1, "n_punted": 0, "punted": []}
    pbs = []
    for s in range(B):
        ctx.release(1)                                   # set s % 2 is free (batch s - 2 done)
        base = (s % 2) * W
        for k in range(W):                               # the producer writes its update for batch s
            t = torch.empty(S, dtype=torch.float32, device=dev)
            m.synth_fill(0, t.data_ptr(), S, dtype=m.MLF_F32, seed=SEED, kind=1, a=k, b=s)
            hosts[base + k].copy_(t.cpu())
            ctx.submit(base + k, 0, 0, 1.0)
        pbs.append(m.plan_from_dict(plan))
        ctx.execute(pbs[-1])
        w_ref, _, _ = execute_plan(w_ref, plan, lambda g: sg.update_values(SEED, g, s, idx, sg.DTYPE_F32), 0.01)
    ctx.sync()
    torch.cuda.synchronize()
    assert np.array_equal(bits(wt.cpu().numpy()[idx]), bits(w_ref))
    assert np.array_equal(bits(pulled.numpy()[idx]), bits(w_ref))
    with pytest.raises(m.MlfError) as e:
        ctx.release(-1)
    assert e.value.code == m.MLF_E_INVALID
    ctx.close()


@pytest.mark.parametrize("tile", [1024, 2048, 4096])
def test_bulk_commit_under_concurrent_copy_engine_traffic(tile):
    # regression: without fence.proxy.async between the empty-barrier wait and the bulk copy
    # that reuses a stage, concurrent copy-engine traffic (unrelated buffers, another stream)
    # let stages be overwritten before the consumers had read them (scripts/dbg_concurrent.py)
    dev = torch.device("cuda", 0)
    S, W = 16_777_216, 32
    rng = np.random.default_rng(tile)
    p = random_plan(rng, W, n_commit=W, boundary=-1)
    big_src = torch.ones(1 << 28, dtype=torch.float32, device=dev)
    big_dst = torch.empty_like(big_src)
    side = torch.cuda.Stream()
    os.environ["MLF_BULK_TILE"] = str(tile)
    try:
        os.environ["MLF_COMMIT_IMPL"] = "bulk"
        slots = [torch.empty(S, dtype=torch.float32, device=dev) for _ in range(W)]
        for w, t in enumerate(slots):
            m.synth_fill(0, t.data_ptr(), S, dtype=sg.DTYPE_F32, seed=SEED, kind=1, a=w, b=0)
        wt = torch.empty(S, dtype=torch.float32, device=dev)
        m.synth_fill(0, wt.data_ptr(), S, dtype=m.MLF_F32, seed=SEED, kind=2)
        torch.cuda.synchronize()
        ctx = m.Context(device=0, model_shard=wt, update_slots=slots, lr=0.01, model_elems=S,
                        stream=torch.cuda.current_stream().cuda_stream)
        for w in range(W):
            ctx.submit(w, 0, 0, 1.0)
        for _ in range(8):
            m.copy_engine(0, big_dst.data_ptr(), big_src.data_ptr(), big_src.numel() * 4, side.cuda_stream)
        ctx.execute(m.plan_from_dict(p))
        ctx.sync()
        torch.cuda.synchronize()
        ctx.close()
    finally:
        del os.environ["MLF_BULK_TILE"]
    idx = np.unique(np.concatenate([rng.integers(0, S, 200_000), np.arange(S - 9, S)]))
    wr, _ = oracle_run(S, sg.DTYPE_F32, p, idx=idx)
    assert np.array_equal(bits(wt.cpu().numpy()[idx]), bits(wr))


def test_contexts_on_two_devices_in_one_process():
    # the large-shared-memory opt-in is per device: a second device's first launch must set it
    if torch.cuda.device_count() < 2:
        pytest.skip("needs >= 2 GPUs")
    rng = np.random.default_rng(23)
    S, W = 300_007, 9
    p = random_plan(rng, W, n_commit=W, boundary=1)
    ref, bref = oracle_run(S, sg.DTYPE_F32, p)
    for device in (0, 1, 0):
        w, b, _, _ = gpu_run(S, W, sg.DTYPE_F32, p, impl="bulk", backup=True, device=device)
        assert np.array_equal(bits(w), bits(ref)) and np.array_equal(bits(b), bits(bref)), device


@pytest.mark.parametrize("impl", IMPLS)
def test_exact_variant_any_order(impl):
    rng = np.random.default_rng(3)
    S, W = 131_075, 256
    p = random_plan(rng, W, n_commit=256, max_group=16, boundary=3)
    w, b, _, _ = gpu_run(S, W, sg.DTYPE_F32, p, lr=2.0**-4, variant=1, backup=True, impl=impl)
    wr, br = oracle_run(S, sg.DTYPE_F32, p, lr=2.0**-4, variant=1)
    assert np.array_equal(bits(w), bits(wr)) and np.array_equal(bits(b), bits(br))
    # same updates in reverse order, all direct: identical bits (no rounding occurs)
    rev = random_plan(rng, W, n_commit=0)
    rev.update(order=p["order"][::-1], n_commit=256, n_direct=256, n_groups=0, group=[0] * W,
               commit_first=list(range(256)), commit_count=[1] * 256, n_server_commits=256,
               replica_boundary_commit=-1, drop_reason=[0] * W, group_node=[])
    w2, _, _, _ = gpu_run(S, W, sg.DTYPE_F32, rev, lr=2.0**-4, variant=1, impl=impl)
    assert np.array_equal(bits(w2), bits(w))


@pytest.mark.parametrize("impl", IMPLS)
def test_operand_list_longer_than_one_launch(impl):
    # > kMaxOps operands: split at commit boundaries, still one logical pass per commit
    rng = np.random.default_rng(5)
    S, W = 1031, 1100
    p = random_plan(rng, W, n_commit=1100, max_group=7, boundary=150)
    w, b, _, stats = gpu_run(S, W, sg.DTYPE_BF16, p, backup=True, impl=impl)
    wr, br = oracle_run(S, sg.DTYPE_BF16, p)
    assert np.array_equal(bits(w), bits(wr)) and np.array_equal(bits(b), bits(br))
    assert stats[0] == 2


@pytest.mark.parametrize("impl", IMPLS)
def test_degenerate_batches(impl):
    rng = np.random.default_rng(9)
    S = 5000
    empty = random_plan(rng, 6, n_commit=0, boundary=-1)
    w, _, _, stats = gpu_run(S, 6, sg.DTYPE_F32, empty, impl=impl)
    assert np.array_equal(bits(w), bits(sg.w0_values(SEED, np.arange(S)))) and stats[0] == 0
    snap = random_plan(rng, 6, n_commit=0, boundary=0)      # all dropped, carried items frozen
    w, b, _, _ = gpu_run(S, 6, sg.DTYPE_F32, snap, backup=True, impl=impl)
    assert np.array_equal(bits(b), bits(w))
    one = random_plan(rng, 1, n_commit=1, boundary=1)
    w, b, _, _ = gpu_run(1, 1, sg.DTYPE_F32, one, backup=True, impl=impl)
    wr, br = oracle_run(1, sg.DTYPE_F32, one)
    assert np.array_equal(bits(w), bits(wr)) and np.array_equal(bits(b), bits(br))


def test_host_resident_updates_move_only_when_committed():
    rng = np.random.default_rng(12)
    S, W = 70_001, 10
    p = random_plan(rng, W, n_commit=4, boundary=-1)
    w, _, _, stats = gpu_run(S, W, sg.DTYPE_F32, p, host_updates=True)
    wr, _ = oracle_run(S, sg.DTYPE_F32, p)
    assert np.array_equal(bits(w), bits(wr))
    assert stats[1] == 4 * S * 4                             # h2d bytes: committed updates only


@pytest.mark.parametrize("S", [9_000_011, 4 << 22, 1000])
def test_e2e_pipeline_h2d_commit_d2h(S):
    """mlf_set_pull_host: chunked H2D / commit / D2H overlap inside mlf_execute (incl. a ragged
    last chunk, an exact multiple of the chunk size and a single small chunk), with a mirror."""
    rng = np.random.default_rng(S % 97)
    W = 6
    p = random_plan(rng, W, n_commit=5, boundary=2)
    dev = torch.device("cuda", 0)
    slots = [torch.empty(S, device=dev) for _ in range(W)]
    hosts = []
    for w, t in enumerate(slots):
        m.synth_fill(0, t.data_ptr(), S, seed=SEED, kind=1, a=w, b=0)
        hosts.append(t.cpu().pin_memory())
        t.zero_()
    wt = torch.empty(S, device=dev)
    m.synth_fill(0, wt.data_ptr(), S, seed=SEED, kind=2)
    bk = torch.full((S,), float("nan"), device=dev)
    pulled = torch.full((S,), float("nan")).pin_memory()
    ctx = m.Context(device=0, model_shard=wt, update_slots=slots, lr=0.01, model_elems=S, backup_shard=bk,
                    stream=torch.cuda.current_stream().cuda_stream)
    ctx.set_pull_host(pulled.data_ptr())
    for w in range(W):
        ctx.submit(w, 0)
        ctx.set_update_host(w, hosts[w].data_ptr())
    ctx.execute(m.plan_from_dict(p))
    ctx.sync()
    wr, br = oracle_run(S, sg.DTYPE_F32, p)
    assert np.array_equal(bits(pulled.numpy()), bits(wr))
    assert np.array_equal(bits(wt.cpu().numpy()), bits(wr)) and np.array_equal(bits(bk.cpu().numpy()), bits(br))
    _, h2d, d2h = ctx.stats()
    assert h2d == 5 * S * 4 and d2h == S * 4
    ctx.close()


@pytest.mark.parametrize("nbytes", [16, 16384, 16400, 5 * 16384 + 48, 200_000_016])
def test_denominator_copy_kernels(nbytes):
    # the roofline denominators are measured with these kernels: they must copy exactly
    dev = torch.device("cuda", 0)
    src = torch.randint(0, 255, (nbytes,), dtype=torch.uint8, device=dev)
    for fn in (m.copy_kernel, m.copy_bulk, m.copy_engine):
        dst = torch.zeros(nbytes, dtype=torch.uint8, device=dev)
        fn(0, dst.data_ptr(), src.data_ptr(), nbytes, torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        assert torch.equal(dst, src), fn.__name__


@pytest.mark.parametrize("mode", [0, 1, 2])
def test_gather_modes_exact(mode):
    # get of the whole model from shards (TMA bulk / copy engine / SM loads): ragged shards,
    # an empty one, tails that are not 16-byte multiples, > 1 chunk per shard
    dev = torch.device("cuda", 0)
    S = 3 * 16384 + 1237
    src = torch.randn(S, device=dev)
    cuts = [0, 64, 64, 20000 + 7, 33333, S]        # shard begins (64-aligned except the ragged ones)
    begins, elems, ptrs = [], [], []
    for b, e in zip(cuts[:-1], cuts[1:]):
        begins.append(b)
        elems.append(e - b)
        ptrs.append(src[b:].data_ptr() if e > b else src.data_ptr())
    dst = torch.full((S,), float("nan"), device=dev)
    m.gather(0, dst.data_ptr(), ptrs, begins, elems, copy_engine=mode, stream=torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    assert torch.equal(dst.view(torch.int32), src.view(torch.int32))


def test_invalid_plan_rejected_without_device_work():
    dev = torch.device("cuda", 0)
    S = 64
    slots = [torch.zeros(S, device=dev) for _ in range(3)]
    wt = torch.ones(S, device=dev)
    ctx = m.Context(device=0, model_shard=wt, update_slots=slots, lr=0.5, model_elems=S,
                    stream=torch.cuda.current_stream().cuda_stream)
    ctx.submit(0, 0)
    ctx.submit(1, 0)
    with pytest.raises(m.MlfError) as e:
        ctx.submit(1, 0)
    assert e.value.code == m.MLF_E_STATE
    bad = random_plan(np.random.default_rng(0), 2, n_commit=2)
    bad["order"] = [0, 5]
    with pytest.raises(m.MlfError) as e:
        ctx.execute(m.plan_from_dict(bad))
    assert e.value.code == m.MLF_E_INVALID
    rep = random_plan(np.random.default_rng(0), 2, n_commit=2, boundary=1)
    with pytest.raises(m.MlfError) as e:                     # replica write without a backup shard
        ctx.execute(m.plan_from_dict(rep))
    assert e.value.code == m.MLF_E_INVALID
    assert ctx.stats()[0] == 0 and torch.all(wt == 1)
    ctx.close()


def test_submit_batch_equals_single_submits_and_is_all_or_nothing():
    """mlf_submit_batch = mlf_submit_update per worker in order (Table 1 push); a bad
    descriptor anywhere leaves the batch unchanged."""
    dev = torch.device("cuda", 0)
    S = 64
    slots = [torch.zeros(S, device=dev) for _ in range(6)]
    wt = torch.ones(S, device=dev)

    def view(c):
        b = c.batch_view()
        return [(b.node[i], b.bytes[i], b.version[i], b.t_avail_ns[i], b.norm[i]) for i in range(b.n)]

    kw = dict(device=0, model_shard=wt, update_slots=slots, lr=0.5, model_elems=S, worker_node=[3, 1, 4, 1, 5, 9],
              n_nodes=10, stream=torch.cuda.current_stream().cuda_stream)
    one, many = m.Context(**kw), m.Context(**kw)
    ws, vs, ts, ns = [4, 0, 2], [7, 5, 6], [10, 0, 30], [1.5, 0.25, 2.0]
    for w, v, t, nr in zip(ws, vs, ts, ns):
        one.submit(w, v, t, nr)
    many.submit_batch(ws, vs, ts, ns)
    assert view(one) == view(many) and len(view(many)) == 3
    for bad, code in (([1, 1], m.MLF_E_STATE),          # twice in one call
                      ([5, 0], m.MLF_E_STATE),          # already in the batch
                      ([5, 6], m.MLF_E_INVALID)):       # out of range
        with pytest.raises(m.MlfError) as e:
            many.submit_batch(bad, [0] * len(bad))
        assert e.value.code == code
        assert view(many) == view(one)
    with pytest.raises(m.MlfError) as e:                # negative t_avail
        many.submit_batch([1, 3], [0, 0], [0, -1])
    assert e.value.code == m.MLF_E_INVALID
    many.submit_batch([1, 3], [8, 9])                   # marks of the failed calls were undone
    one.submit(1, 8)
    one.submit(3, 9)
    assert view(one) == view(many) and len(view(many)) == 5
    many.submit_batch([], [])
    assert view(one) == view(many)
    one.close()
    many.close()


def test_executor_rejects_a_plan_beyond_the_delay_bound():
    """registerAsServer(tau_max) (Table 1): the executor re-checks (v + p) - v(g) <= tau_max for
    every committed update (R1) and rejects a stale plan before any device work."""
    dev = torch.device("cuda", 0)
    S = 64
    slots = [torch.ones(S, device=dev) for _ in range(3)]
    wt = torch.zeros(S, device=dev)
    ctx = m.Context(device=0, model_shard=wt, update_slots=slots, lr=1.0, model_elems=S, v0=10, tau_max=3,
                    stream=torch.cuda.current_stream().cuda_stream)
    for g, v in enumerate([10, 8, 10]):
        ctx.submit(g, v)
    # positions 1, 2, 3 commit versions 11, 12, 13: update 1 (v = 8) at position 2 has delay 4 > 3
    stale = {"n_commit": 3, "order": [0, 1, 2], "drop_reason": [0, 0, 0], "group": [0, 0, 0], "n_direct": 3,
             "n_groups": 0, "group_node": [], "n_server_commits": 3, "commit_first": [0, 1, 2],
             "commit_count": [1, 1, 1], "replica_boundary_commit": -1}
    with pytest.raises(m.MlfError) as e:
        ctx.execute(m.plan_from_dict(stale))
    assert e.value.code == m.MLF_E_INVALID and "tau_max" in str(e.value)
    assert ctx.stats()[0] == 0 and torch.all(wt == 0)
    # update 1 first: delays 3, 2, 3 are all within the bound
    ok = dict(stale, order=[1, 0, 2])
    ctx.execute(m.plan_from_dict(ok))
    ctx.sync()
    assert ctx.version() == 13 and torch.all(wt == -3)
    ctx.close()


@pytest.mark.parametrize("it_count", [3])
def test_config1_end_to_end_vs_oracle(it_count):
    os.environ["MLF_COMMIT_IMPL"] = "ldg"
    cfg = configs.config(1)
    wl = Workload(cfg, device=0)
    S = cfg["S"]
    idx = np.arange(S)
    w_ref = sg.w0_values(cfg["seed"], idx)
    for it in range(it_count):
        v_init = wl.v_init
        pb, pd, draws = wl.step(it)
        wl.ctx.sync()
        up, down, site = configs.network(cfg, it)
        batch = [Item(w, S * 4, d["version"], d["t_avail"], d["norm"]) for w, d in enumerate(draws)]
        op = oracle_plan(make_net(cfg["n_nodes"], up, down, None, site), batch,
                         Params(servers=cfg["servers"], aggs=cfg["aggs"], v_init=v_init, tau_max=cfg["tau"]))
        assert op == pd
        w_ref, _, _ = execute_plan(w_ref, op, lambda g: sg.update_values(cfg["seed"], g, it, idx), cfg["lr"])
        got = wl.w.cpu().numpy()
        assert np.array_equal(bits(got), bits(w_ref))
    assert wl.ctx.version() == wl.v_init


@pytest.mark.parametrize("impl", IMPLS)
@pytest.mark.parametrize("tau,dtype", [(4, "f32"), (32, "f32"), (32, "bf16")])
def test_config2_full_size_sampled(tau, dtype, impl):
    """BASELINE config 2 at full size (25.6M elements, 32 workers) in the launch configuration bench.py
    times; every element checked bitwise against the oracle at 20k sampled indices (incl. the tail)."""
    os.environ["MLF_COMMIT_IMPL"] = impl
    cfg = configs.config(2, tau=tau, dtype=dtype)
    wl = Workload(cfg, device=0)
    S = cfg["S"]
    rng = np.random.default_rng(tau)
    idx = np.unique(np.concatenate([rng.integers(0, S, 20_000), np.arange(S - 37, S), np.arange(0, 37)]))
    dt = sg.DTYPE_BF16 if dtype == "bf16" else sg.DTYPE_F32
    w_ref = sg.w0_values(cfg["seed"], idx)
    for it in range(2):
        v_init = wl.v_init
        pb, pd, draws = wl.step(it)
        wl.ctx.sync()
        # the plan the GPU executed is the oracle's plan of the same inputs
        up, down, site = configs.network(cfg, it)
        batch = [Item(cfg["worker_node"][g], S * cfg["e"], d["version"], d["t_avail"], d["norm"])
                 for g, d in enumerate(draws)]
        op = oracle_plan(make_net(cfg["n_nodes"], up, down, None, site), batch,
                         Params(servers=cfg["servers"], aggs=cfg["aggs"], v_init=v_init, tau_max=cfg["tau"]))
        assert op == pd, it
        w_ref, _, _ = execute_plan(w_ref, op, lambda g: sg.update_values(cfg["seed"], g, it, idx, dt), cfg["lr"])
        got = wl.w.cpu().numpy()[idx]
        assert np.array_equal(bits(got), bits(w_ref))
        assert pd["n_commit"] == min(tau, 32)


def test_context_holds_its_buffers():
    # the library borrows the buffers for the context's lifetime: the binding keeps them alive
    import gc
    import weakref
    w = torch.zeros(4099, device="cuda")
    slots = [torch.ones(4099, device="cuda") for _ in range(2)]
    refs = [weakref.ref(t) for t in (w, *slots)]
    with m.Context(device=0, model_shard=w, update_slots=slots, lr=0.5, model_elems=4099) as ctx:
        del w, slots
        gc.collect()
        assert all(r() is not None for r in refs)
        for g in range(2):
            ctx.submit(g, 0, 0, 1.0)
        p = {"n_commit": 2, "n_server_commits": 2, "order": [0, 1], "drop_reason": [0, 0], "group": [0, 0],
             "n_direct": 2, "n_groups": 0,
             "group_node": [], "commit_first": [0, 1], "commit_count": [1, 1], "replica_boundary_commit": -1}
        ctx.execute(m.plan_from_dict(p))
        ctx.sync()
        assert torch.equal(refs[0](), torch.full((4099,), -1.0, device="cuda"))
    gc.collect()
    assert all(r() is None for r in refs)
