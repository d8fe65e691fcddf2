"""Config 5: rescoring the reference cost model against measured B200 times.

For each instance (placement, reduction request) the reference simulator
(`Simulate`, /root/reference/proj/src/simulator.cc:141-188) predicts a time
per synthesized program; `RankPrograms` (simulator.cc:190-213) sorts them
stably (ties keep emission order). An instance is a top-k *hit* when the
measured-fastest program is among the simulator's k fastest (the paper's
top-k, which it never defines precisely). The tie-aware
variant counts a hit when the measured-fastest program's predicted time is no
larger than the k-th smallest prediction.
"""
from __future__ import annotations

from collections import defaultdict

KS = (1, 2, 3, 5, 6, 10)


def _ranks(xs):
    """Average ranks (ties share the mean rank), 1-based."""
    order = sorted(range(len(xs)), key=lambda i: xs[i])
    ranks = [0.0] * len(xs)
    i = 0
    while i < len(order):
        j = i
        while j + 1 < len(order) and xs[order[j + 1]] == xs[order[i]]:
            j += 1
        for k in range(i, j + 1):
            ranks[order[k]] = (i + j) / 2.0 + 1.0
        i = j + 1
    return ranks


def spearman(xs, ys):
    """Spearman rank correlation (None when either side is constant)."""
    if len(xs) < 2:
        return None
    rx, ry = _ranks(xs), _ranks(ys)
    mx, my = sum(rx) / len(rx), sum(ry) / len(ry)
    sxy = sum((a - mx) * (b - my) for a, b in zip(rx, ry))
    sxx = sum((a - mx) ** 2 for a in rx)
    syy = sum((b - my) ** 2 for b in ry)
    if sxx == 0 or syy == 0:
        return None
    return sxy / (sxx * syy) ** 0.5


def topk(rows, ks=KS):
    """rows: iterable of dicts with keys instance (hashable), index (emission
    order), sim_seconds, measured_us. Returns per-k hit rates."""
    by = defaultdict(list)
    for r in rows:
        by[r["instance"]].append(r)
    strict = {k: 0 for k in ks}
    tie = {k: 0 for k in ks}
    detail = []
    rhos = []
    for inst, progs in by.items():
        ranked = sorted(progs, key=lambda r: (r["sim_seconds"], r["index"]))  # stable like RankPrograms
        best = min(progs, key=lambda r: (r["measured_us"], r["index"]))
        pos = next(i for i, r in enumerate(ranked) if r["index"] == best["index"])
        for k in ks:
            strict[k] += pos < k
            kth = ranked[min(k, len(ranked)) - 1]["sim_seconds"]
            tie[k] += best["sim_seconds"] <= kth
        sim_best = ranked[0]
        rho = spearman([r["sim_seconds"] for r in progs], [r["measured_us"] for r in progs])
        if rho is not None:
            rhos.append((rho, len(progs)))
        detail.append({"instance": inst, "programs": len(progs), "spearman": rho, "measured_best": best["text"],
                       "measured_best_us": best["measured_us"], "sim_rank_of_measured_best": pos + 1,
                       "sim_best": sim_best["text"], "sim_best_measured_us": sim_best["measured_us"],
                       "loss_if_sim_best": sim_best["measured_us"] / best["measured_us"]})
    n = max(1, len(by))
    # program-weighted mean rank correlation between predicted and measured
    # times (top-k alone saturates when one program wins every instance)
    wsum = sum(w for _, w in rhos)
    return {"instances": len(by), "top_k": {k: strict[k] / n for k in ks},
            "top_k_tie_aware": {k: tie[k] / n for k in ks},
            "spearman": (sum(r * w for r, w in rhos) / wsum) if wsum else None, "detail": detail}
