"""Re-select a tuning table from a tuner log (lines "MxNxK cfg S=s: X TFLOP/s (median Y)")
with the tuner's current tie rule, without re-timing:
    python tools/retable.py TUNER_LOG OUT_TABLE"""
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1706_10086_b200 import gemm as G  # noqa: E402
from paper_1706_10086_b200 import tuner  # noqa: E402


def main(log, out):
    res = {}
    order = []
    for line in open(log):
        m = re.match(r"(\d+)x(\d+)x(\d+) (\S+) S=(\d+): ([\d.]+) TFLOP/s", line)
        if not m:
            continue
        shape = tuple(int(m.group(i)) for i in (1, 2, 3))
        if shape not in res:
            res[shape] = {}
            order.append(shape)
        fl = 2.0 * shape[0] * shape[1] * shape[2]
        res[shape][(G.cfg_id(m.group(4)), int(m.group(5)))] = fl / (float(m.group(6)) * 1e12)
    entries = []
    for shape in order:
        cfg, s = tuner.select(res[shape])
        entries.append((*shape, True, cfg, s))
        print(shape, G.cfg_name(cfg), s)
    tuner.write_table(out, entries)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
