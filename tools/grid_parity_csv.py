"""Fill the parity column of a published grid / table CSV from the GPU parity run
(tests/test_gpu_published_sizes.py with GEMM_PARITY_OUT=...):

    python tools/grid_parity_csv.py GRID.csv PARITY.jsonl OUT.csv

parity_max_err_over_bound <- the uniform-input sampled-row check's max |err| / bound at that
shape; the row is only filled if the dyadic Freivalds check of every entry passed too (the
json line's "ok"), and it must have run the same plan the CSV row timed ("cfg" x "splits").
"""
import csv
import json
import sys


def main(grid, parity, out):
    res = {}
    for line in open(parity):
        d = json.loads(line)
        res[(d["m"], d["n"], d["k"])] = d
    rows = list(csv.DictReader(open(grid)))
    missing = []
    for r in rows:
        key = (int(r["m"]), int(r["n"]), int(r["k"]))
        d = res.get(key)
        plan = f"{r['cfg']} x{r['splits']}"
        if d is None or not d["ok"] or d["plan"] != plan:
            missing.append((key, plan, d and d["plan"]))
            continue
        r["parity_max_err_over_bound"] = f"{d['max_err_over_bound']:.3e}"
    with open(out, "w", newline="") as f:
        w = csv.DictWriter(f, fieldnames=list(rows[0].keys()))
        w.writeheader()
        w.writerows(rows)
    for m in missing:
        print("not filled:", m, file=sys.stderr)
    return 1 if missing else 0


if __name__ == "__main__":
    sys.exit(main(*sys.argv[1:4]))
