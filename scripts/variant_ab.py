"""Same-box A/B of variant builds of libmasw.so (development aid).

    python -m paper_2003_02256_b200.build --out=/tmp/v1.so -DMASW_FAST_SETTLE=0   (here)
    VARIANTS="base=paper_2003_02256_b200/libmasw.so,v1=/tmp/v1.so" \
        CONFIGS=ensemble,realistic,uniform ROUNDS=3 python scripts/variant_ab.py   (GPU box)

Each round runs every variant in its own process (MASW_LIB selects the library), in
alternating order, and records the library's own scan-kernel times (MASW_TIME_SCAN events)
plus a hash of the idx output; prints per variant and config the median scan time and
whether idx is bitwise identical to the first variant's.
"""
import hashlib
import json
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child(configs, reps):
    sys.path.insert(0, os.environ.get("MASW_TREE", ROOT))   # older trees: their own binding
    import numpy as np
    import torch
    import paper_2003_02256_b200 as masw
    import synth

    def dev(a):
        return torch.as_tensor(np.ascontiguousarray(a), device="cuda")

    out = {}
    for name in configs:
        kw = {"tier": 200.0} if name == "uniform" else {}
        w = synth.workload(name, **kw)
        m = w.models
        args = [dev(x) for x in (m.h, m.alpha, m.beta, m.rho)]
        lam, c = dev(w.lam), dev(w.c)
        ce = dev(w.ce) if w.ce is not None else None

        def run():
            if m.h.shape[0] > 1:
                return masw.masw_curves_ensemble(*args, lam, c, ce, flags=masw.TIME_SCAN).idx
            return masw.masw_curve(*[a[0] for a in args], lam, c, flags=masw.TIME_SCAN)[2]

        run()
        ts = []
        for _ in range(reps):
            idx = run()
            torch.cuda.synchronize()
            ts.append(masw.masw_last_scan_ms())
        h = hashlib.sha256(idx.cpu().numpy().tobytes()).hexdigest()[:16]
        alg, ev = masw.masw_last_work()
        out[name] = {"ms": ts, "idx": h, "alg": alg, "eval": ev}
    print("RESULT " + json.dumps(out), flush=True)


def main():
    if len(sys.argv) > 1 and sys.argv[1] == "--child":
        child(sys.argv[2].split(","), int(sys.argv[3]))
        return
    variants = [v.split("=", 1) for v in os.environ["VARIANTS"].split(",")]
    configs = os.environ.get("CONFIGS", "ensemble,realistic,uniform")
    rounds = int(os.environ.get("ROUNDS", "3"))
    reps = os.environ.get("REPS", "5")
    res = {n: {} for n, _ in variants}
    for k in range(rounds):
        order = variants if k % 2 == 0 else variants[::-1]
        for name, path in order:
            env = dict(os.environ)
            if os.path.isdir(path):   # a whole older tree (binding + library + synth)
                env["MASW_TREE"] = os.path.abspath(path)
                env.pop("MASW_LIB", None)
            else:
                env["MASW_LIB"] = os.path.abspath(path)
            p = subprocess.run([sys.executable, __file__, "--child", configs, reps], env=env,
                               capture_output=True, text=True)
            line = [x for x in p.stdout.splitlines() if x.startswith("RESULT ")]
            if p.returncode != 0 or not line:
                print(f"{name}: FAILED rc={p.returncode}\n{p.stderr[-2000:]}", flush=True)
                continue
            for cfg, v in json.loads(line[0][7:]).items():
                r = res[name].setdefault(cfg, {"ms": [], "idx": set(), "alg": v["alg"],
                                                "eval": v["eval"]})
                r["ms"] += v["ms"]
                r["idx"].add(v["idx"])
    base = variants[0][0]
    for cfg in configs.split(","):
        print(f"== {cfg}")
        b = res[base].get(cfg)
        for name, _ in variants:
            r = res[name].get(cfg)
            if not r:
                print(f"  {name:12s} missing")
                continue
            med = statistics.median(r["ms"])
            rel = med / statistics.median(b["ms"]) if b else float("nan")
            same = b is not None and r["idx"] == b["idx"]
            print(f"  {name:12s} {med:8.3f} ms  x{rel:.4f}  min {min(r['ms']):.3f}  "
                  f"idx {'same' if same else 'DIFF'}  eval/alg {r['eval'] / max(r['alg'], 1):.4f}",
                  flush=True)


if __name__ == "__main__":
    main()
