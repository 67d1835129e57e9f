"""The sharded (N > 1) path through the C ABI: 2 ranks (one process each; sharing cuda:0 when
the box has one GPU), IPC peer mappings, fold and tree modes, remote mirror stores —
bitwise against the oracle at sampled indices (tests/multigpu_check.py)."""
import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def _run(nproc, *args, timeout=600, extra_env=None):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--standalone", "--nnodes=1",
           f"--nproc-per-node={nproc}", os.path.join(HERE, "multigpu_check.py"), *args]
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", OMP_NUM_THREADS="1", **(extra_env or {}))
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, env=env)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    return r.stdout


@pytest.mark.parametrize("cid,extra", [(3, []), (4, ["--steps", "3"]), (5, ["--S", "300007", "--workers", "64"]),
                                        (3, ["--dtype", "bf16", "--kernel", "bulk"]),
                                        (3, ["--dtype", "bf16", "--kernel", "ldg", "--steps", "1"])])
def test_two_ranks_bitwise(cid, extra):
    out = _run(2, "--cid", str(cid), *extra)
    assert "MULTIGPU_OK fold" in out and "MULTIGPU_OK tree" in out and "MULTIGPU_OK staged" in out


def test_two_ranks_full_size_config3():
    # BASELINE config 3 at its stated size (64 workers x 143,667,240 fp32 = VGG-19) in the
    # bench's launch configuration (2 PS shards, bulk kernel), sampled outputs vs the oracle
    out = _run(2, "--cid", "3", "--S", "143667240", "--steps", "2", timeout=1200)
    assert "MULTIGPU_OK fold" in out and "MULTIGPU_OK tree" in out and "MULTIGPU_OK staged" in out


def test_two_ranks_full_size_config4():
    # config 4 as stated (128 workers, 25.6M fp32, N2 shares, C2 stragglers, re-planned every
    # batch) on 2 PS shards, sampled outputs vs the oracle planning the same batches
    out = _run(2, "--cid", "4", "--S", "25600000", "--steps", "2", timeout=1200)
    assert "MULTIGPU_OK fold" in out and "MULTIGPU_OK tree" in out and "MULTIGPU_OK staged" in out


def test_two_ranks_full_size_config5_updates():
    # config 5's 100M-element updates and replica mirror on the neighbour GPU, 64 of its 256
    # workers (the Python oracle plans 256 in ~2 minutes per batch)
    out = _run(2, "--cid", "5", "--S", "100000000", "--steps", "1", "--workers", "64", "--modes", "fold,tree",
               timeout=1200)
    assert "MULTIGPU_OK fold" in out and "MULTIGPU_OK tree" in out


def test_two_ranks_bf16_16kb_layout():
    # bf16 shards large enough for the 8192-element bf16 kernel (>= 16 tiles per CTA), operands
    # read over peer mappings (fold) and from the staging buffer (staged)
    out = _run(2, "--cid", "3", "--S", "40000000", "--steps", "1", "--dtype", "bf16", "--modes", "fold,staged",
               timeout=900)
    assert "MULTIGPU_OK fold" in out and "MULTIGPU_OK staged" in out


def test_two_ranks_staged_whole_slices():
    # MLF_STAGE_WHOLE=1: one copy-engine copy per remote operand slice, the fold in groups of
    # commits (the pre-batch mirror store in the first group only), bf16 and fp32
    for dt in ("f32", "bf16"):
        out = _run(2, "--cid", "5", "--S", "300007", "--modes", "staged", "--workers", "64", "--dtype", dt,
                   extra_env={"MLF_STAGE_WHOLE": "1"})
        assert "MULTIGPU_OK staged" in out


def test_two_ranks_staged_every_third_remote_operand():
    # MLF_STAGE_EVERY=3: a third of the remote operands staged by the copy engines, the rest read
    # over the peer mappings by the same kernel
    out = _run(2, "--cid", "3", "--S", "300007", "--modes", "staged", "--stage-mib", "4", "--workers", "32",
               extra_env={"MLF_STAGE_EVERY": "3"})
    assert "MULTIGPU_OK staged" in out
    # ... and with the first chunk folded straight from the peers while the copy engines pull
    # the second, 8 chunks
    out = _run(2, "--cid", "3", "--S", "300007", "--modes", "staged", "--workers", "32",
               extra_env={"MLF_STAGE_EVERY": "2", "MLF_STAGE_FIRST_DIRECT": "1", "MLF_STAGE_CHUNKS": "8"})
    assert "MULTIGPU_OK staged" in out
    # ... and the bench's mixed variant: 3 of every 4 remote operands staged, 3 chunks
    out = _run(2, "--cid", "3", "--S", "300007", "--modes", "staged", "--workers", "32",
               extra_env={"MLF_STAGE_SKIP": "4", "MLF_STAGE_FIRST_DIRECT": "1", "MLF_STAGE_CHUNKS": "3"})
    assert "MULTIGPU_OK staged" in out


def test_two_ranks_staged_minimum_chunk():
    # copy-engine staging with a 2 MiB buffer: 4096-element chunks, many of them, ragged tail
    out = _run(2, "--cid", "3", "--S", "300007", "--modes", "staged", "--stage-mib", "2", "--workers", "32")
    assert "MULTIGPU_OK staged" in out


def test_two_ranks_momentum_with_mirror():
    out = _run(2, "--cid", "5", "--S", "300007", "--gamma", "0.9", "--modes", "fold", "--workers", "64")
    assert "MULTIGPU_OK fold" in out


def test_two_ranks_replica_trees_with_retention():
    # config 5 (replica of shard j on GPU j+1), count-style Div_max so that updates are punted
    out = _run(2, "--cid", "5", "--S", "200003", "--steps", "4", "--replica-mode", "1", "--div-max", "20",
               "--workers", "32", "--modes", "fold,tree,staged")
    assert "MULTIGPU_OK fold" in out and "MULTIGPU_OK tree" in out and "MULTIGPU_OK staged" in out
    assert "punted_total=0" not in out


def test_two_ranks_host_resident_updates():
    # the e2e path: each rank stages its committed host-resident updates (phase 1), peers read them
    out = _run(2, "--cid", "3", "--S", "400009", "--steps", "2", "--host")
    assert "MULTIGPU_OK fold" in out and "MULTIGPU_OK tree" in out and "MULTIGPU_OK staged" in out


def test_two_ranks_allreduce_push_get():
    cmd = [sys.executable, "-m", "torch.distributed.run", "--standalone", "--nnodes=1", "--nproc-per-node=2",
           os.path.join(HERE, "allreduce_check.py"), "--S", "500009", "--workers", "8"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600,
                       env=dict(os.environ, MASTER_ADDR="127.0.0.1", OMP_NUM_THREADS="1"))
    assert r.returncode == 0 and "ALLREDUCE_OK" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]


def test_two_ranks_distribution_trees():
    # NEXT-4: model distribution along mlf_plan_distribution trees into every rank's view
    cmd = [sys.executable, "-m", "torch.distributed.run", "--standalone", "--nnodes=1", "--nproc-per-node=2",
           os.path.join(HERE, "distribute_check.py"), "--S", "1000003"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600,
                       env=dict(os.environ, MASTER_ADDR="127.0.0.1", OMP_NUM_THREADS="1"))
    assert r.returncode == 0 and "DISTRIBUTE_OK" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]
    assert "case degraded0: groups=1" in r.stdout


def test_two_gpus_multicast_get():
    # NVLS multicast fused get: needs one GPU per rank (the multicast object spans devices)
    if torch.cuda.device_count() < 2:
        pytest.skip("needs >= 2 GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--standalone", "--nnodes=1", "--nproc-per-node=2",
           os.path.join(HERE, "allreduce_check.py"), "--S", "1000003", "--workers", "4", "--multicast"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600,
                       env=dict(os.environ, MASTER_ADDR="127.0.0.1", OMP_NUM_THREADS="1"))
    assert r.returncode == 0 and "multicast=True" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]


def test_eight_ranks_sharing_the_visible_gpus():
    # world = 8 (the box size the north star names) on whatever GPUs are visible: 8 shards, 8
    # fused-get destinations, the 8-way plan — bitwise vs the oracle
    out = _run(8, "--cid", "3", "--S", "2000011", "--steps", "1", "--workers", "64", timeout=900)
    assert "MULTIGPU_OK fold" in out and "MULTIGPU_OK tree" in out and "MULTIGPU_OK staged" in out
    cmd = [sys.executable, "-m", "torch.distributed.run", "--standalone", "--nnodes=1", "--nproc-per-node=8",
           os.path.join(HERE, "allreduce_check.py"), "--S", "500009", "--workers", "8"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600,
                       env=dict(os.environ, MASTER_ADDR="127.0.0.1", OMP_NUM_THREADS="1"))
    assert r.returncode == 0 and "ALLREDUCE_OK" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]


def test_all_gpus_if_several():
    n = torch.cuda.device_count()
    if n < 4:
        pytest.skip("needs >= 4 GPUs")
    # 64 of config 5's 256 workers: the Python oracle plans every batch of every mode
    out = _run(4, "--cid", "5", "--S", "2000011", "--workers", "64", timeout=900)
    assert "MULTIGPU_OK fold" in out and "MULTIGPU_OK tree" in out and "MULTIGPU_OK staged" in out
    cmd = [sys.executable, "-m", "torch.distributed.run", "--standalone", "--nnodes=1", "--nproc-per-node=4",
           os.path.join(HERE, "distribute_check.py"), "--S", "2000011"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600,
                       env=dict(os.environ, MASTER_ADDR="127.0.0.1", OMP_NUM_THREADS="1"))
    assert r.returncode == 0 and "DISTRIBUTE_OK" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]
