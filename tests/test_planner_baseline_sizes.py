"""mlf_plan at BASELINE sizes vs the oracle (SURVEY §4.2 tier 2; Alg. 2, Alg. 3,
P:1816-1848 App. B.2, §5.3).

Config 4 (128 virtual workers, 8 PS shards, N2 NVLink shares, C2 stragglers, re-planned per
batch, 2 batches) and config 5 (256 workers, 8 shards, replica on the next GPU, Div_max 0,
1 batch).  The Python oracle needs minutes per batch at these sizes, so its plans are stored
in tests/golden/plans_config{4,5}_g8.json by scripts/gen_plan_golden.py, which calls only
oracle/; the inputs are regenerated here from the seeded synthgen recipe."""
import json
import os

import pytest

from paper_1907_00434_b200 import mlfabric as m
from synthgen import configs as cfgs

GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.mark.parametrize("cid", [4, 5])
def test_mlf_plan_equals_oracle_at_baseline_size(cid):
    gold = json.load(open(os.path.join(GOLD, f"plans_config{cid}_g8.json")))
    cfg = cfgs.config(cid, G=8)
    assert gold["seed"] == cfg["seed"] and gold["tau"] == cfg["tau"]
    for b in gold["batches"]:
        it, v_init, v_prev = b["iteration"], b["v_init"], b["v_prev"]
        draws = cfgs.batch_draws(cfg, it, v_init, v_prev)
        up, down, site = cfgs.network(cfg, it)
        batch = {"node": cfg["worker_node"], "size": [cfg["S"] * cfg["e"]] * cfg["W"],
                 "version": [d["version"] for d in draws], "t_avail": [d["t_avail"] for d in draws],
                 "norm": [d["norm"] for d in draws]}
        p = m.plan(cfg["n_nodes"], up, down, batch, cfg["servers"], site=site, aggs=cfg["aggs"],
                   replicas=cfg["replicas"], raggs=cfg["raggs"], v_init=v_init, tau_max=cfg["tau"],
                   div_max=cfg["div_max"], carried=b["carried"], shard_weights=[n for (_, n) in cfg["shards"]])
        assert p == b["plan"], it
        assert p["n_commit"] > 0
