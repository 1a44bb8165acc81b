"""Join the config-3 timing sweep (tools/sweep.py tune) with the per-configuration ncu
metrics (tools/sweep.py ncu under `ncu --metrics ... --csv`) into the SURVEY §8(d) config-3
CSV: ... dmma_pipe_pct, bank_conflicts (duration-weighted / summed over a configuration's
launches, e.g. the hybrid's three kernels).

    python tools/config3_join.py TUNE.csv NCU.csv NCU_PASS.log OUT.csv
"""
import csv
import sys
from collections import defaultdict

DMMA = "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active"
BANK = "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum"
DUR = "gpu__time_duration.sum"
DRAM = "dram__bytes_read.sum"


def num(x):
    return float(x.replace(",", ""))


def main(tune_csv, ncu_csv, pass_log, out):
    # ncu long format: one row per (launch, metric)
    lines = open(ncu_csv).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    launches = defaultdict(dict)
    order = []
    for r in csv.DictReader(lines[start:]):
        lid = int(r["ID"])
        if lid not in launches:
            order.append(lid)
        launches[lid][r["Metric Name"]] = (r["Metric Value"], r["Metric Unit"])
        launches[lid]["_name"] = r["Kernel Name"]
    groups = []
    for line in open(pass_log):
        f = line.split()
        if len(f) == 3 and f[0].isdigit():
            groups.append((f[1], int(f[2])))
    per_cfg = {}
    it = iter(order)
    for name, n in groups:
        ids = [next(it) for _ in range(n)]
        durs = [num(launches[i][DUR][0]) for i in ids]
        dmma = sum(num(launches[i][DMMA][0]) * d for i, d in zip(ids, durs)) / sum(durs)
        bank = sum(num(launches[i][BANK][0]) for i in ids)
        per_cfg[name] = (dmma, bank)
    rows = list(csv.DictReader(open(tune_csv)))
    head = ["m", "n", "k", "alpha", "beta", "cfg", "bm", "bn", "bk", "wm", "wn", "e", "stages", "regs", "smem_bytes",
            "gpus", "best_s", "median_s", "tflops", "frac_peak_datasheet", "frac_peak_clock", "sm_mhz_mean",
            "power_w_mean", "dmma_pipe_pct", "bank_conflicts"]
    with open(out, "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(head)
        for r in rows:
            dm, bk = per_cfg.get(r["cfg"], (float("nan"), float("nan")))
            w.writerow([r[h] for h in head[:-2]] + [f"{dm:.2f}", f"{bk:.0f}"])
    print(f"{len(rows)} rows, {len(per_cfg)} configurations with ncu metrics -> {out}")


if __name__ == "__main__":
    main(*sys.argv[1:5])
