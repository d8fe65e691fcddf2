#!/usr/bin/env python
"""Fit the B200-calibrated cost model (rs_plan_predict_us's form) to measured
per-program times and score it with leave-one-config-out validation.

Model per launch phase: latency (one value for one-GPU phases, one for
cross-GPU phases) + max per-GPU link bytes / link rate + max per-GPU HBM
bytes / HBM rate, summed over phases. Features come from the compiled plans
(planning-only contexts with the run's slot->GPU map); measured times from
`bench.py --programs-out` (configs 1-3). Prints the fitted constants and the
config-5 scores (top-k of the measured-best program, Spearman) per N.

  python tools/fit_cost_model.py profiles/r02_programs_n{1,2,4}.json
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2110_10548_b200 import executor, planner, rescore  # noqa: E402

WL = {"config1": ([2, 4], 64 << 20, "f32"), "config2": ([2, 4], 256 << 20, "bf16"),
      "config3": ([2, 2, 2], 64 << 20, "bf16")}


OPS = 5  # AllReduce, ReduceScatter, AllGather, Reduce, Broadcast (semantics.h:29-35)


def features(rows, world, per_op=False):
    """Per program: [n_local_phases, n_cross_phases, link_bytes_sum, hbm_bytes_sum]
    (per_op: link and HBM bytes split by the step's collective)."""
    K = 8
    slot_rank = [d * world // K for d in range(K)]
    ctx = executor.Context.virtual(K, slot_rank, world)
    cache = {}
    out = []
    for r in rows:
        axes, payload, dt = WL[r["config"]]
        key = (r["config"], tuple(r["request"]))
        if key not in cache:
            syn = planner.synthesize(planner.config_path("b200_sock"), axes, list(r["request"]), payload_bytes=payload)
            cache[key] = syn
        prog = cache[key].placements[r["matrix"]].programs[r["index"]]
        es = 2 if dt == "bf16" else 4
        plan = ctx.compile(prog, payload // es, dt)
        d = plan.describe()
        nl = nc = 0
        link = np.zeros(OPS if per_op else 1)
        hbm = np.zeros(OPS if per_op else 1)
        for st, (op, _) in zip(d["steps"], prog.steps):
            tx = max(max(rk["tx"], rk["rx"]) for rk in st["ranks"])
            hb = max(rk["hbm"] for rk in st["ranks"])
            if tx > 0:
                nc += 1
            else:
                nl += 1
            link[op if per_op else 0] += tx
            hbm[op if per_op else 0] += hb
        plan.close()
        out.append([nl, nc, *link, *hbm])
    ctx.close()
    return np.array(out, dtype=float)


def fit(X, y):
    """Least squares on relative error: minimise sum ((Xb - y) / y)^2 with
    b = [lat_local_us, lat_cross_us, 1/link (us per byte), 1/hbm]."""
    W = X / y[:, None]
    b, *_ = np.linalg.lstsq(W, np.ones_like(y), rcond=None)
    return np.maximum(b, 1e-12)


def score(rows, pred):
    res = rescore.topk([{"instance": (r["config"], tuple(r["request"]), r["matrix"]), "index": r["index"],
                         "sim_seconds": p, "measured_us": r["measured_us"], "text": r["text"]}
                        for r, p in zip(rows, pred)])
    return {"instances": res["instances"], "top_k": res["top_k"], "spearman": res["spearman"]}


def main():
    report = {}
    for path in sys.argv[1:]:
        rows = json.load(open(path))
        world = {"n1": 1, "n2": 2, "n4": 4}[os.path.basename(path).split("_")[-1].split(".")[0]]
        X = features(rows, world)
        Xo = features(rows, world, per_op=True)
        y = np.array([r["measured_us"] for r in rows])
        b = fit(X, y)
        bo = fit(Xo, y)
        per = {"params": {"lat_local_us": b[0], "lat_cross_us": b[1], "link_GBps": 1e-3 / b[2],
                          "hbm_GBps": 1e-3 / b[3]},
               "params_per_op": {"lat_local_us": bo[0], "lat_cross_us": bo[1],
                                 "link_GBps": [1e-3 / v for v in bo[2:2 + OPS]],
                                 "hbm_GBps": [1e-3 / v for v in bo[2 + OPS:]]},
               "fit_all": score(rows, X @ b),
               "fit_all_per_op": score(rows, Xo @ bo),
               "reference_simulate": score(rows, [r["sim_seconds"] for r in rows]),
               "calibrated_default": score(rows, [r["calibrated_us"] for r in rows])}
        # leave one config out: fit on the others, score the held-out config
        cv, cvo = {}, {}
        for held in sorted({r["config"] for r in rows}):
            tr = np.array([r["config"] != held for r in rows])
            if tr.sum() < 4:
                continue
            te = ~tr
            held_rows = [r for r, t in zip(rows, te) if t]
            cv[held] = score(held_rows, X[te] @ fit(X[tr], y[tr]))
            cvo[held] = score(held_rows, Xo[te] @ fit(Xo[tr], y[tr]))
        per["leave_one_config_out"] = cv
        per["leave_one_config_out_per_op"] = cvo
        mape = float(np.median(np.abs(X @ b - y) / y))
        per["median_abs_rel_error_fit_all"] = mape
        report[f"N={world}"] = per
        print(f"N={world}: params {json.dumps({k: round(v, 2) for k, v in per['params'].items()})}, "
              f"median |err| {mape:.3f}")
        for name in ("reference_simulate", "calibrated_default", "fit_all", "fit_all_per_op"):
            s = per[name]
            print(f"  {name:20s} instances {s['instances']:3d} top1 {s['top_k'][1]:.2f} top2 {s['top_k'][2]:.2f} "
                  f"top5 {s['top_k'][5]:.2f} rho {s['spearman']:.3f}")
        for tag, table in (("", cv), (" per-op", cvo)):
            for held, s in table.items():
                rho = s['spearman'] if s['spearman'] is None else round(s['spearman'], 3)
                print(f"  held-out {held}{tag:8s} instances {s['instances']:3d} top1 {s['top_k'][1]:.2f} top2 "
                      f"{s['top_k'][2]:.2f} top5 {s['top_k'][5]:.2f} rho {rho}")
    json.dump(report, open(os.path.join(ROOT, "profiles", "r02_cost_model_fit.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
