"""Summarise an ncu report (read here, no GPU needed): per captured kernel, the metrics the
roofline and DESIGN.md quote.

    python tools/ncu_summary.py REPORT.ncu-rep OUT.json
"""
import csv
import io
import json
import subprocess
import sys

KEYS = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active", "sm__cycles_elapsed.avg.per_second",
        "lts__t_sector_hit_rate.pct", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "launch__shared_mem_per_block_dynamic", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "smsp__inst_executed.sum"]


def main(rep, out):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    head, units, data = rows[0], rows[1], rows[2:]
    kernels = []
    for r in data:
        d = {}
        for k in KEYS:
            if k in head:
                i = head.index(k)
                d[k] = {"value": r[i], "unit": units[i]}
        kernels.append(d)

    def gb(d, k):
        try:
            v = float(d[k]["value"].replace(",", ""))
        except (KeyError, ValueError):
            return 0.0
        if v != v:      # ncu prints -nan for counters it could not collect on a launch
            return 0.0
        u = d[k]["unit"]
        return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}[u]

    total = {"dram_bytes": sum(gb(d, "dram__bytes_read.sum") + gb(d, "dram__bytes_write.sum") for d in kernels)}
    json.dump({"report": rep, "kernels": kernels, "total": total}, open(out, "w"), indent=1)
    print(json.dumps(total))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
