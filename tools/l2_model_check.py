"""f4: the paper's memory model (Eqs. (5)-(7), paper_1706_10086_b200/model.py l2_to_sm_bytes)
against ncu's L2 counters, one launch per configuration (ncu run by this script; GPU box):

    python tools/l2_model_check.py [N] > profiles/r02/l2_model_check_v1.jsonl

Per configuration: model L2->SM bytes 8*M*N*K*(1/BM + 1/BN) + the C store, ncu L2 read
bytes requested by the SMs (lts__t_sectors_srcunit_tex_op_read x 32 B: TMA and cp.async
loads both arrive as "tex" requests), all L2 read sectors, DRAM read bytes and the kernel time.
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1706_10086_b200 import model  # noqa: E402

CFGS = ["tma_64x64x32_w32x16_s3_splitk", "tma_64x64x16_w32x16_s6", "tma_128x128x16_w32x32_s4",
        "tma_256x64x16_w64x32_s4", "tma_64x128x16_w32x64_s4", "tma_32x64x32_w16x16_s3_splitk",
        "tma_64x32x32_w16x16_s4_splitk", "tma_32x32x32_w16x16_s4_splitk", "gen_64x64x16_w32x16_s4"]
METRICS = ["gpu__time_duration.sum", "lts__t_sectors_srcunit_tex_op_read.sum", "lts__t_sectors_op_read.sum",
           "dram__bytes_read.sum", "lts__t_sector_hit_rate.pct"]


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
    for name in CFGS:
        cmd = ["ncu", "--metrics", ",".join(METRICS), "--clock-control", "none", "-k", "regex:dgemm",
               "--launch-skip", "1", "--launch-count", "1", "--csv",
               sys.executable, os.path.join(ROOT, "tools", "one_launch_sp.py"), name, str(n), str(n), str(n), "1"]
        out = subprocess.run(cmd, capture_output=True, text=True, timeout=600).stdout
        rows = [r for r in csv.reader(io.StringIO(out[out.find('"ID"'):])) if r]
        head, vals = rows[0], rows[1:]
        got = {}
        for r in vals:
            rec = dict(zip(head, r))
            got[rec["Metric Name"]] = (float(rec["Metric Value"].replace(",", "")), rec["Metric Unit"])
        parts = name.split("_")[1].split("x")
        bm, bn = int(parts[0]), int(parts[1])
        pred = model.l2_to_sm_bytes(n, n, n, bm, bn)
        pred_read = pred - 8.0 * n * n          # the model's tile reads (its C store is a write)
        tex = got["lts__t_sectors_srcunit_tex_op_read.sum"][0] * 32
        scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}
        dram = got["dram__bytes_read.sum"][0] * scale.get(got["dram__bytes_read.sum"][1], 1.0)
        t = got["gpu__time_duration.sum"]
        print(json.dumps({"cfg": name, "n": n, "model_l2_to_sm_bytes": pred, "model_tile_read_bytes": pred_read,
                          "ncu_l2_tex_read_bytes": tex, "ratio_ncu_over_model_reads": tex / pred_read,
                          "ncu_l2_read_bytes_all": got["lts__t_sectors_op_read.sum"][0] * 32,
                          "ncu_dram_read_bytes": dram, "l2_hit_pct": got["lts__t_sector_hit_rate.pct"][0],
                          "time": t}), flush=True)


if __name__ == "__main__":
    main()
