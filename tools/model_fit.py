"""Offline replica of the size heuristic (csrc/gemm_f64.cu score_all / est_time) evaluated on
measured candidate timings (tools/heuristic_regret.py --dump): for each shape, which plan the
model picks among the timed candidates and its regret t_pick / t_best - 1.  Used to check a
change of the model's efficiencies against every dumped shape before it goes into the library.

    python tools/model_fit.py dump1.jsonl [dump2.jsonl ...] [--eff name=value ...]
"""
import argparse
import json
import math
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def lib_cands():
    """[(name, eff, eff_tail)] from k_tma_cands in csrc/gemm_f64.cu, in candidate order."""
    src = open(os.path.join(ROOT, "paper_1706_10086_b200", "csrc", "gemm_f64.cu")).read()
    body = src[src.index("static const Cand k_tma_cands[] = {"):]
    body = body[:body.index("};")]
    body = re.sub(r"//[^\n]*", "", body)
    out = []
    for m in re.finditer(r'\{"([^"]+)",\s*([0-9.]+)(?:,\s*([0-9.]+))?\}', body):
        out.append((m.group(1), float(m.group(2)), float(m.group(3)) if m.group(3) else 0.0))
    return out


def occupancy(c):
    """CTAs per SM from registers / shared memory / threads (B200: 64 K registers, 228 KB)."""
    warps = c["threads"] // 32
    per_warp = math.ceil(c["regs"] * 32 / 256) * 256
    by_regs = 65536 // (per_warp * warps) if c["regs"] else 1
    by_smem = (228 * 1024) // (c["smem_bytes"] + 1024)
    return max(1, min(by_regs, by_smem, 2048 // c["threads"], 32))


def est_time(d, occ, sms, M, N, K, S, eff):
    tiles = -(-M // d["bm"]) * -(-N // d["bn"])
    KT = -(-K // d["bk"])
    n, slots = tiles * S, sms * occ
    full, m = divmod(n, slots)
    units = float(full * occ)
    if m > 0:
        if occ == 1:
            units += 1.0
        else:
            c = -(-m // sms)
            if full == 0 and occ >= 3:
                c = occ
            units += c if c >= 2 else 1.0 / 0.6
    u = 16.0 / d["bk"]
    ksteps = -(-KT // S) + 2.0 * u     # model v4 (was 4 + 2 for a split)
    return units * d["bm"] * d["bn"] * ksteps * (d["bk"] / 16.0) / eff


def score_all(cfgs, cands, M, N, K, sms=148):
    out = []
    for name, eff, eff_tail in cands:
        d = cfgs.get(name)
        if d is None:
            continue
        occ = occupancy(d)
        KT = -(-K // d["bk"])
        if d["split_k"] == -2:
            tiles = -(-M // d["bm"]) * -(-N // d["bn"])
            G = sms * occ
            W, tail = divmod(tiles, G)
            u = 16.0 / d["bk"]
            ks = W * (KT + 4.0 * u) / eff
            if tail > 0:
                gsk = min(G, max(tail, tail * KT // 16))
                ks += (-(-(tail * KT) // gsk) + 12.0 * u) / (eff_tail if eff_tail > 0 else eff)
            out.append((ks * occ * d["bm"] * d["bn"] * (d["bk"] / 16.0), name, 1))
            continue
        if d["split_k"] == -1:
            tiles = -(-M // d["bm"]) * -(-N // d["bn"])
            G = max(1, min(sms * occ, tiles * KT))
            per_cta_tiles = -(-tiles // G) + 1.0
            t = (-(-(tiles * KT) // G) + (4.0 * per_cta_tiles + 6.0) * 16.0 / d["bk"]) * occ * d["bm"] * d["bn"] * (
                d["bk"] / 16.0) / eff
            out.append((t, name, 1))
            continue
        scap = 8 if d["split_k"] == -3 else 16
        smax = 1 if d["split_k"] == 1 else max(1, min(scap, KT // 2))
        for S in range(1, smax + 1):
            out.append((est_time(d, occ, sms, M, N, K, S, eff), name, S))
    return out


def pick(scored, measured):
    """The library's rule (first candidate > 0.1 % better than the best so far), restricted to
    the measured (cfg, S) pairs."""
    best_t, best = 1e300, None
    for t, name, S in scored:
        if f"{name}:{S}" not in measured:
            continue
        if t < best_t * 0.999:
            best_t, best = t, f"{name}:{S}"
    return best


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("dumps", nargs="+")
    ap.add_argument("--eff", nargs="*", default=[], help="name=value overrides of a candidate's eff")
    ap.add_argument("-v", action="store_true")
    a = ap.parse_args()
    cands = lib_cands()
    over = dict(kv.split("=") for kv in a.eff)
    cands = [(n, float(over.get(n, e)), et) for n, e, et in cands]
    cfgs, rows = {}, []
    for p in a.dumps:
        for line in open(p):
            r = json.loads(line)
            if "cfgs" in r:
                cfgs.update({c["name"]: c for c in r["cfgs"]})
            else:
                rows.append(r)
    regs = []
    for r in rows:
        M, N, K = r["shape"]
        times = r["times"]
        tbest = min(times.values())
        p = pick(score_all(cfgs, cands, M, N, K), times)
        reg = times[p] / tbest - 1.0 if p else float("nan")
        regs.append(reg)
        if a.v:
            bk = min(times, key=times.get)
            print(f"{M:6d} {N:6d} {K:6d}  pick {p:40s} best {bk:40s} regret {reg:7.4f}  (lib plan {r['plan']})")
    ok = [x for x in regs if x == x]
    print(f"shapes {len(ok)}  mean regret {sum(ok) / len(ok):.4f}  max {max(ok):.4f}  "
          f"> 5 %: {sum(x > 0.05 for x in ok)}")


if __name__ == "__main__":
    main()
