"""A/B of the fused-step variants over k and workloads (one GPU).

Times k_step(+k_lp3) per step (CUDA events inside orca_step_timed, L2-resident, after
warm-up) for each variant on the same evolving state.  Usage:
    python scripts/ablation_variants.py [--variants 0,3] [--ks 10,20,32] [--configs uniform_1m,dense]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1908_10107_b200 import orca as O  # noqa: E402
from paper_1908_10107_b200 import workloads as W  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--variants", default="0,3")
    ap.add_argument("--ks", default="10,20,32")
    ap.add_argument("--configs", default="uniform_1m,dense")
    ap.add_argument("--steps", type=int, default=8)
    ap.add_argument("--tag", default="")
    ap.add_argument("--ns", default="", help="agent counts (uniform-type configs), comma-separated")
    a = ap.parse_args()
    variants = [int(x) for x in a.variants.split(",")]
    jobs = []
    for cfg in a.configs.split(","):
        for n in ([int(x) for x in a.ns.split(",")] if a.ns else [None]):
            jobs.append((cfg, n))
    for cfg, nn in jobs:
        w = W.make(cfg, n=nn)
        for k in [int(x) for x in a.ks.split(",")]:
            p = dict(w["params"], maxNeighbors=k)
            ctx = O.Orca(p)
            ctx.set_agents(w["pos"], w["vel"], w["pref"])
            ctx.step(5)
            row = {"tag": a.tag, "config": cfg, "n": len(w["pos"]), "k": k}
            for v in variants:
                ctx.set_variant(v)
                ctx.step(2)
                ms = ctx.step_timed(a.steps)[0] / a.steps
                row[f"v{v}_ms"] = round(ms, 4)
            row["work"] = ctx.work()
            print(json.dumps(row), flush=True)
            ctx.close()


if __name__ == "__main__":
    main()
