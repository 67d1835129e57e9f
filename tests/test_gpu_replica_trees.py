"""NEXT-2 on the GPU: paper-faithful replica trees.

The replica model is updated by the plan's frozen replica commits — its own Alg. 3
grouping over carried ++ O(U) — and punted updates are retained across batches.  Both the
primary and the replica are compared bitwise with the oracle (oracle/numerics.commit_batch
applied to the plan's commits), over several batches with punting; the replica's own
grouping makes it differ from the primary only by fp32 rounding (checked <= 1e-6).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import synthgen as sg  # noqa: E402
from oracle.numerics import commit_batch, execute_plan  # noqa: E402
from tests.test_gpu_parity import bits  # noqa: E402

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_1907_00434_b200.harness import Workload
    from synthgen import configs


@pytest.mark.parametrize("div_max,dtype", [(10.0, "f32"), (40.0, "bf16"), (0.0, "f32")])
def test_replica_trees_bitwise_over_batches(div_max, dtype):
    # k' = 4 replica aggregators: the replica falls behind and punts, so retention is exercised
    cfg = configs.config(2, tau=32, with_replica=True, replica_mode=1, div_max=div_max, scale_S=300_007,
                         dtype=dtype, replica_aggs=4)
    wl = Workload(cfg, device=0)
    S = cfg["S"]
    idx = np.arange(S)
    dt = sg.DTYPE_BF16 if dtype == "bf16" else sg.DTYPE_F32
    data = lambda wid, it: sg.update_values(cfg["seed"], wid, it, idx, dt)  # noqa: E731
    primary = sg.w0_values(cfg["seed"], idx)
    replica = primary.copy()
    carried = []                       # (worker, iteration) of every carried item, in order
    punted_seen = 0
    roundings = 0                      # fp32 roundings on an element's chain, primary + replica (R17)
    for it in range(6):
        pb, pd, draws = wl.step(it)
        wl.ctx.sync()
        primary, _, _ = execute_plan(primary, pd, lambda g: data(g, it), cfg["lr"])
        items = carried + [(g, it) for g in pd["order"]]
        commits = [[data(*items[q]) for q in range(f, f + k)]
                   for f, k in zip(pd["replica_commit_first"], pd["replica_commit_count"])]
        replica, _ = commit_batch(replica, commits, cfg["lr"])
        carried = [items[i] for i in pd["punted"]]
        punted_seen += len(carried)
        # each commit: members - 1 adds, a product and a difference; a member counts one rounding
        roundings += pd["n_commit"] + 2 * pd["n_server_commits"]
        roundings += sum(pd["replica_commit_count"]) + 2 * len(pd["replica_commit_count"])
        assert np.array_equal(bits(wl.w.cpu().numpy()), bits(primary)), it
        assert np.array_equal(bits(wl.backup.cpu().numpy()), bits(replica)), it
        if not carried:
            # the replica holds the same updates with its own grouping: both are the exact sum up
            # to one fp32 rounding (<= 2^-24 of the largest magnitude, |w|) per operation on
            # either chain (first-order bound; DESIGN.md NEXT-2)
            tol = 2.0 ** -24 * float(np.max(np.abs(primary))) * roundings
            assert np.max(np.abs(replica - primary)) <= tol
    if div_max >= 10.0:
        assert punted_seen > 0         # retention across batches was exercised
    else:
        assert punted_seen == 0
