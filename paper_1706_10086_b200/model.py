"""The paper's performance model, evaluated for the B200 tile configurations.

PAPER.md §2 / §2.1 / §2.2:
  Eq. (2)  O(N)     = 3N^2 + 2N^3 ~ 2N^3                floating point operations
  Eq. (3)  B(e,t)   = N / (t*e)                         blocks per grid dimension
  Eq. (4)  P(N,t)   = 2N^3 / t * 1e-9                   GFLOP/s
  Eq. (5)  K(S,T)   = 2 T^2 S                           bytes of one A and one B tile
  Eq. (6)  M(N,T)   = N^2 (2N/T + 1)                    memory operations
  Eq. (7)  R(N,T)   = 2NT / (2N + T)  -> T  (N -> inf)  compute / memory ratio
  Eq. (8)  P(f,o,n) = f * o * n                         theoretical peak

B200 reading: a CTA tile is BM x BN (the paper's square tile T generalised
to a rectangle), a pipeline stage holds one BM x BK slab of A and one BK x BN slab of B
(8*(BM+BN)*BK bytes, the K(S,T) analog), and every element of C costs one read of a
BM-tile row panel and a BN-tile column panel per k-step: the L2 -> SM traffic is
8*M*N*K*(1/BM + 1/BN) bytes plus the C stream 8*M*N*(1 + [beta != 0]) (Eq. (6) with the C
store added, reading R14).  Peak = SMs x 128 FP64 FLOP/clk x f (Eq. (8); 128 measured by
gemm_peak_probe).

    python -m paper_1706_10086_b200.model [--n 16384] [--json]
"""

from __future__ import annotations

import argparse
import json


def flops_eq2(n: int) -> int:
    """Eq. (2): 3N^2 + 2N^3 (the exact count of alpha*A*B + beta*C is 2N^3 + 2N^2; reading R2)."""
    return 3 * n * n + 2 * n ** 3


def flops(m: int, n: int, k: int) -> int:
    """Eq. (4)'s convention generalised: 2MNK."""
    return 2 * m * n * k


def blocks(n: int, t: int, e: int) -> float:
    """Eq. (3): blocks per grid dimension, N / (t * e)."""
    return n / (t * e)


def gflops(n: int, seconds: float) -> float:
    """Eq. (4): 2N^3 / t * 1e-9."""
    return 2.0 * n ** 3 / seconds * 1e-9


def tile_bytes(s: int, t: int) -> int:
    """Eq. (5): K(S,T) = 2 T^2 S, the cache needed for one A and one B tile."""
    return 2 * t * t * s


def mem_ops(n: int, t: int) -> float:
    """Eq. (6): M(N,T) = N^2 (2N/T + 1)."""
    return n * n * (2.0 * n / t + 1.0)


def ratio(n: int, t: int) -> float:
    """Eq. (7): R(N,T) = 2NT / (2N + T)."""
    return 2.0 * n * t / (2.0 * n + t)


def peak(f_hz: float, o: float, n: int) -> float:
    """Eq. (8): P(f,o,n) = f * o * n (FLOP/s)."""
    return f_hz * o * n


# ---------------------------------------------------------------- B200 mapping
def stage_bytes(bm: int, bn: int, bk: int, s: int = 8) -> int:
    """Shared memory of one pipeline stage (A slab + B slab), the K(S,T) analog."""
    return s * (bm + bn) * bk


def l2_to_sm_bytes(m: int, n: int, k: int, bm: int, bn: int, beta_nonzero: bool = False, s: int = 8) -> float:
    """Tile traffic (Eq. (6) analog, C store included)."""
    return s * m * n * k * (1.0 / bm + 1.0 / bn) + s * m * n * (2.0 if beta_nonzero else 1.0)


def compulsory_bytes(m: int, n: int, k: int, beta_nonzero: bool = False, s: int = 8) -> int:
    return s * (m * k + k * n + m * n * (2 if beta_nonzero else 1))


def tile_intensity(bm: int, bn: int) -> float:
    """FLOP per L2->SM byte of a BM x BN tile (Eq. (7) analog for N -> infinity): 2/(8(1/BM+1/BN))."""
    return 2.0 / (8.0 * (1.0 / bm + 1.0 / bn))


B200_SMS = 148
B200_FP64_FLOP_PER_CLK_PER_SM = 128        # measured (gemm_peak_probe, profiles/r01_probe_peak_and_cfgs.json)
B200_MAX_HZ = 1.965e9


def b200_peak(f_hz: float = B200_MAX_HZ) -> float:
    return peak(f_hz, B200_FP64_FLOP_PER_CLK_PER_SM, B200_SMS)


def report(n: int = 16384, beta_nonzero: bool = False, cfgs=None):
    """One row per tile configuration: the model's bytes and ratios at N^3."""
    if cfgs is None:
        from . import gemm as G
        cfgs = G.cfgs()
    rows = []
    for c in cfgs:
        rows.append({
            "cfg": c["name"], "bm": c["bm"], "bn": c["bn"], "bk": c["bk"], "e": c["wm"] * c["wn"] // 32,
            "stage_bytes": stage_bytes(c["bm"], c["bn"], c["bk"]),
            "smem_bytes": c.get("smem_bytes"),
            "ctas": (-(-n // c["bm"])) * (-(-n // c["bn"])),
            "l2_to_sm_GB": l2_to_sm_bytes(n, n, n, c["bm"], c["bn"], beta_nonzero) / 1e9,
            "tile_flop_per_byte": tile_intensity(c["bm"], c["bn"]),
            "compulsory_GB": compulsory_bytes(n, n, n, beta_nonzero) / 1e9,
            "hbm_ridge_flop_per_byte": b200_peak() / 6.5514e12,
        })
    return rows


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=16384)
    ap.add_argument("--beta", action="store_true")
    ap.add_argument("--json", action="store_true")
    a = ap.parse_args(argv)
    rows = report(a.n, a.beta)
    if a.json:
        print(json.dumps(rows, indent=1))
        return 0
    print(f"N={a.n}: FLOPs 2N^3 = {flops(a.n, a.n, a.n):.4e} (Eq. (2) count {flops_eq2(a.n):.4e}); "
          f"B200 peak {b200_peak() / 1e12:.2f} TFLOP/s")
    for r in rows:
        print(f"{r['cfg']:36s} stage {r['stage_bytes'] / 1024:6.1f} KiB  CTAs {r['ctas']:7d}  "
              f"L2->SM {r['l2_to_sm_GB']:8.1f} GB  tile {r['tile_flop_per_byte']:5.1f} FLOP/B")
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
