"""Regenerates the golden fixtures in tests/golden/ from the UNMODIFIED
reference built by oracle/Makefile (oracle/_ref/libredsynth_ref.so).

Run in the build container (needs /root/reference): `python tests/golden/make_golden.py`.
Fixtures:
  programs_<name>.json   the reference's synthesized program set (emission
                         order, text, lowered groups, simulated seconds)
  report_<name>.sha256   sha256 + size of the reference tool's JSON report
  refusals.json          mutated programs with the reference RunLowered's
                         status code, failing step, violation and message
  numeric_small.json     small-input numeric vectors produced by the C oracle
                         (oracle/numeric.c) for f32 / bf16 / i32, every program
                         of config 1 (K = 8, N = 37)
"""
import hashlib
import json
import os
import random
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import numeric, ref  # noqa: E402

CONFIGS = {
    # name: (system config, axes, reduce, payload bytes)
    "cfg1": ("configs/b200_sock.json", [2, 4], [0], 64 << 20),
    "cfg2_r1": ("configs/b200_sock.json", [2, 4], [1], 256 << 20),
    "cfg2_r01": ("configs/b200_sock.json", [2, 4], [0, 1], 256 << 20),
    "cfg3_r0": ("configs/b200_sock.json", [2, 2, 2], [0], 64 << 20),
    "cfg3_r1": ("configs/b200_sock.json", [2, 2, 2], [1], 64 << 20),
    "cfg3_r2": ("configs/b200_sock.json", [2, 2, 2], [2], 64 << 20),
    "cfg3_r01": ("configs/b200_sock.json", [2, 2, 2], [0, 1], 64 << 20),
    "cfg3_r02": ("configs/b200_sock.json", [2, 2, 2], [0, 2], 64 << 20),
    "cfg3_r12": ("configs/b200_sock.json", [2, 2, 2], [1, 2], 64 << 20),
    "k2_flat": ("configs/b200_flat2.json", [2], [0], 1 << 20),
    "k4_flat": ("configs/b200_flat4.json", [4], [0], 1 << 20),
    "k4_sock": ("configs/b200_sock4.json", [4], [0], 1 << 20),
    "k8_flat": ("configs/b200_flat8.json", [8], [0], 1 << 20),
    "k8_sock": ("configs/b200_sock.json", [8], [0], 1 << 20),
    "a100_2node_r0": ("/root/reference/proj/configs/a100_2node.json", [8, 4], [0], 4 << 30),
}


class P:  # minimal program object for oracle.numeric
    def __init__(self, steps):
        self.steps = steps


def main():
    assert ref.available(), "build the reference first: make -C oracle ref"
    for name, (cfg, axes, red, payload) in CONFIGS.items():
        path = cfg if cfg.startswith("/") else os.path.join(ROOT, cfg)
        doc = ref.synthesize(open(path).read(), axes, red, payload_bytes=payload)
        doc["config"] = {"system": cfg, "axes": axes, "reduce": red, "payload_bytes": payload}
        with open(os.path.join(HERE, f"programs_{name}.json"), "w") as f:
            json.dump(doc, f, separators=(",", ":"))
        text = ref.report(path, axes, red, payload)
        with open(os.path.join(HERE, f"report_{name}.sha256"), "w") as f:
            f.write(f"{hashlib.sha256(text.encode()).hexdigest()} {len(text.encode())}\n")

    # Refusals: mutate valid config-2 programs (op swap, group shuffle, member
    # drop, step duplication) and record the reference's verdict.
    rng = random.Random(20261018)
    progs = json.load(open(os.path.join(HERE, "programs_cfg2_r01.json")))["matrices"]
    cases = []
    while len(cases) < 300:
        m = rng.choice(progs)
        p = rng.choice(m["programs"])
        steps = [[s["op"], [list(g) for g in s["groups"]]] for s in p["steps"]]
        kind = rng.randrange(5)
        s = rng.randrange(len(steps))
        if kind == 0:
            steps[s][0] = rng.randrange(5)
        elif kind == 1 and len(steps) > 1:
            steps.insert(s, [steps[s][0], [list(g) for g in steps[s][1]]])
        elif kind == 2:
            g = rng.randrange(len(steps[s][1]))
            if len(steps[s][1][g]) > 1:
                steps[s][1][g].pop(rng.randrange(len(steps[s][1][g])))
        elif kind == 3:
            steps = steps[:s] + steps[s + 1:] or steps
        else:
            g = steps[s][1][rng.randrange(len(steps[s][1]))]
            rng.shuffle(g)
        code, state, fstep, fviol, msg = ref.run_lowered([(o, gs) for o, gs in steps], 8)
        final_full = None
        if code == 0:
            final_full = [[int(sum(int(b) << c for c, b in enumerate(state[d, r]))) for r in range(8)]
                          for d in range(8)]
        cases.append({"steps": steps, "code": code, "step": fstep if code else -1,
                      "violation": fviol if code else 0, "message": msg, "held": final_full})
    with open(os.path.join(HERE, "refusals.json"), "w") as f:
        json.dump(cases, f, separators=(",", ":"))

    # Small numeric vectors from the C oracle (config 1, K=8, N=37).
    K, N = 8, 37
    cfg1 = json.load(open(os.path.join(HERE, "programs_cfg1.json")))["matrices"]
    vectors = []
    for mi, m in enumerate(cfg1):
        for pi, p in enumerate(m["programs"]):
            steps = [(s["op"], s["groups"]) for s in p["steps"]]
            for dt in (numeric.F32, numeric.BF16, numeric.I32):
                bufs = numeric.synthetic_inputs(K, N, dt)
                numeric.execute(P(steps), K, bufs, dt, nthreads=1)
                vectors.append({"matrix": mi, "program": pi, "dtype": dt,
                                "out": [b.view(b.dtype).tolist() if dt != numeric.F32 else
                                        b.view("uint32").tolist() for b in bufs]})
    with open(os.path.join(HERE, "numeric_small.json"), "w") as f:
        json.dump({"K": K, "N": N, "seed_base": 1000, "vectors": vectors}, f, separators=(",", ":"))
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
