"""Config 5: rescoring cost models against measured B200 times.

The reference simulator (`Simulate`) and the B200-calibrated model
(`rs_plan_predict_us`) are scored on committed per-program measurements
(`profiles/r01_programs_cal_*.json`, written by `bench.py --programs-out`):
top-k hit rates and the rank correlation between predicted and measured
times.
"""
import json
import os

import pytest

from common import ROOT
from paper_2110_10548_b200 import rescore


def test_spearman_matches_scipy():
    scipy_stats = pytest.importorskip("scipy.stats")
    xs = [3.0, 1.0, 2.0, 2.0, 5.0, 4.0]
    ys = [30.0, 12.0, 25.0, 19.0, 41.0, 47.0]
    assert abs(rescore.spearman(xs, ys) - scipy_stats.spearmanr(xs, ys)[0]) < 1e-12
    assert rescore.spearman([1.0, 1.0], [2.0, 3.0]) is None


def test_topk_hits_and_ties():
    rows = [{"instance": "a", "index": i, "sim_seconds": s, "measured_us": m, "text": f"p{i}"}
            for i, (s, m) in enumerate([(1.0, 9.0), (2.0, 5.0), (2.0, 7.0), (3.0, 8.0)])]
    out = rescore.topk(rows, ks=(1, 2, 3))
    assert out["top_k"] == {1: 0.0, 2: 1.0, 3: 1.0}
    assert out["detail"][0]["sim_rank_of_measured_best"] == 2
    assert out["detail"][0]["loss_if_sim_best"] == 9.0 / 5.0


@pytest.mark.parametrize("name", ["n1", "k4"])
def test_calibrated_model_ranks_measured_times_better(name):
    """On B200 the reference model (shared-switch division, no HBM level)
    orders the programs far from the measured order; the calibrated model,
    fed the executor's own traffic, tracks it (profiles/r01_programs_cal_*)."""
    rows = json.load(open(os.path.join(ROOT, "profiles", f"r01_programs_cal_{name}.json")))
    inst = lambda r: (tuple(r["request"]), json.dumps(r["matrix"]))  # noqa: E731
    ref = rescore.topk([{"instance": inst(r), "index": r["index"], "sim_seconds": r["sim_seconds"],
                         "measured_us": r["measured_us"], "text": r["text"]} for r in rows])
    cal = rescore.topk([{"instance": inst(r), "index": r["index"], "sim_seconds": r["calibrated_us"],
                         "measured_us": r["measured_us"], "text": r["text"]} for r in rows])
    assert cal["spearman"] > 0.9
    assert ref["spearman"] < 0.6
    assert cal["top_k"][1] >= ref["top_k"][1]
