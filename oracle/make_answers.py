"""Write canonical oracle answer files tests/golden/answers_sf<milli>_seed<seed>.json.

Calls ONLY oracle/sx_oracle (the CPU oracle CLI, which generates its own host
columns with gen/gen_cpu.c).  Used offline for sizes the GPU-box tests cannot
afford to recompute (SF10, SF100); the GPU parity tests and bench.py compare
against these files.

    python oracle/make_answers.py --sf-milli 100000 [--seed 42] [--queries q1,q6,q3,q9,q18]
"""
import argparse
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = os.path.join(os.path.dirname(HERE), "tests", "golden")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sf-milli", type=int, required=True)
    ap.add_argument("--seed", type=int, default=42)
    ap.add_argument("--queries", default="q1,q6,q3,q9,q18")
    args = ap.parse_args()
    path = os.path.join(GOLDEN, f"answers_sf{args.sf_milli}_seed{args.seed}.json")
    out = json.load(open(path)) if os.path.exists(path) else {
        "_about": "CPU-oracle answers (oracle/sx_oracle via oracle/make_answers.py); canonical rows as in oracle/__init__.py",
        "sf_milli": args.sf_milli, "seed": args.seed, "answers": {}, "oracle_seconds": {}}
    for q in args.queries.split(","):
        r = subprocess.run([os.path.join(HERE, "sx_oracle"), "--query", q, "--sf-milli", str(args.sf_milli),
                            "--seed", str(args.seed)], check=True, capture_output=True, text=True)
        d = json.loads(r.stdout.strip().splitlines()[-1])
        out["answers"][q] = d["rows"]
        out["oracle_seconds"][q] = d["seconds"][0]
        out["n_lineitem"] = d["n_lineitem"]
        with open(path, "w") as f:
            json.dump(out, f, indent=1)
        print(q, len(d["rows"]), d["seconds"], file=sys.stderr, flush=True)


if __name__ == "__main__":
    main()
