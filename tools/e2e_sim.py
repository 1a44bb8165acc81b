"""Copy/compute simulation of gemm_f64_host (the e2e path): three in-order streams (H2D,
compute, D2H), PCIe at the measured rates (profiles/r01_e2e_probe.json: 55 / 53 GB/s
pinned), GEMM blocks timed with a wave model calibrated on the measured 16384^3 kernel
(240.8 ms: 111 waves of 256x64 tiles).  Used to choose the schedule geometry in
csrc/host_api.cu; prints the old and the implemented schedule and the best of a grid.

    python tools/e2e_sim.py [N] [--r02]
"""
import math
import sys

S = 148
RATE_SM = 2.479e11          # FLOP/s per SM inside a wave (calibrated: 16384^3 -> 240.8 ms)
TILE_OVH = 4e-6             # per-wave tile prologue/epilogue
LAUNCH = 6e-6
H2D, D2H = 55e9, 53e9


def gemm_t(M, N, K):
    tiles = math.ceil(M / 256) * math.ceil(N / 64)
    return math.ceil(tiles / S) * (256 * 64 * K * 2 / RATE_SM + TILE_OVH) + LAUNCH


# round 2: the large-shape plan is 64x64 tiles at two CTAs per SM (waves of 296 tiles),
# calibrated on the measured 16384^3 kernel (237.7 ms = 222 waves)
R_CTA64 = 64 * 64 * 16384 * 2 / (237.7e-3 / 222)


def gemm_t64(M, N, K):
    tiles = math.ceil(M / 64) * math.ceil(N / 64)
    return math.ceil(tiles / (2 * S)) * (64 * 64 * K * 2 / R_CTA64 + 3e-6) + 4e-6


def simulate(K, plan):
    th = tc = td = 0.0
    h_end, g_end, idle = {}, {}, 0.0
    for i, it in enumerate(plan):
        if it[0] == "h2d":
            th += it[1] / H2D
            h_end[i] = th
        elif it[0] == "gemm":
            start = max(tc, h_end[it[3]])
            idle += start - tc
            tc = start + gemm_t(it[1], it[2], K)
            g_end[i] = tc
        else:
            td = max(td, g_end[it[2]]) + it[1] / D2H
    return max(td, tc), idle


def schedule(M, N, K, R0, Ra, cb0, cb, Rp, Rlast, nlast):
    """The structure of host_impl: A[0:Ra], B block 0, GEMM(Ra rows), A[Ra:R0],
    GEMM(rest of block 0), B blocks 1.. each followed by its GEMM on R0 rows, then row
    panels of Rp rows (the last Rlast rows in nlast column blocks)."""
    plan = [("h2d", Ra * K * 8)]
    cols, c = [], 0
    while c < N:
        w = min(N - c, cb0 if not cols else cb)
        cols.append((c, w))
        c += w

    def block(hi, nr, nc):
        plan.append(("gemm", nr, nc, hi))
        plan.append(("d2h", nr * nc * 8, len(plan) - 1))

    for j, (c0, nc) in enumerate(cols):
        plan.append(("h2d", K * nc * 8))
        hi = len(plan) - 1
        if j == 0 and Ra < R0:
            block(hi, Ra, nc)
            plan.append(("h2d", (R0 - Ra) * K * 8))
            block(len(plan) - 1, R0 - Ra, nc)
        else:
            block(hi, R0, nc)
    rows, r = [], R0
    while r < M:
        rem = M - r
        nr = rem if (rem <= Rlast or Rlast == 0) else (rem - Rlast if rem <= Rlast + Rp else Rp)
        rows.append(nr)
        r += nr
    for p, nr in enumerate(rows):
        plan.append(("h2d", nr * K * 8))
        hi = len(plan) - 1
        nb = nlast if p == len(rows) - 1 else 1
        lcb = math.ceil(N / nb / 64) * 64
        for c0 in range(0, N, lcb):
            block(hi, nr, min(N, c0 + lcb) - c0)
    return plan


def main():
    global gemm_t
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
    if "--r02" in sys.argv:     # the round-2 kernel's wave model and a finer geometry grid
        gemm_t = gemm_t64
        t, idle = simulate(n, schedule(n, n, n, 3072, 768, 1024, 1536, 3840, 256, 2))
        print(f"implemented  {t * 1e3:7.2f} ms  {2 * n ** 3 / t / 1e12:6.2f} TFLOP/s  GPU idle {idle * 1e3:5.2f} ms"
              f"  (kernel alone {gemm_t(n, n, n) * 1e3:.1f} ms)")
        best = min((simulate(n, schedule(n, n, n, 64 * r0, 64 * ra, 64 * c0, 64 * cbt, 64 * rp, 64 * rl, 2))[0],
                    r0, ra, c0, cbt, rp, rl)
                   for r0 in (32, 37, 40, 44, 48, 52, 56) for ra in (4, 8, 12, 16) for c0 in (4, 8, 16, 24)
                   for cbt in (16, 24, 32, 37, 48) for rp in (37, 48, 60, 74) for rl in (4, 8))
        print(f"grid best    {best[0] * 1e3:7.2f} ms  (R0, Ra, cb0, cb, Rp, Rlast in 64-row/col tiles) = {best[1:]}")
        return
    kern = gemm_t(n, n, n)
    old = schedule(n, n, n, 2304, 2304, 2048, 2048, 2048, 2048, 2)      # round-1 first schedule
    new = schedule(n, n, n, 3072, 768, 1024, 1536, 3840, 256, 2)        # host_api.cu now
    for name, pl in (("previous", old), ("implemented", new)):
        t, idle = simulate(n, pl)
        print(f"{name:12s} {t * 1e3:7.2f} ms  {2 * n ** 3 / t / 1e12:6.2f} TFLOP/s  GPU idle {idle * 1e3:5.2f} ms"
              f"  (kernel alone {kern * 1e3:.1f} ms)")
    best = min((simulate(n, schedule(n, n, n, 256 * r0, 256 * ra, 64 * c0, 64 * cbt, 256 * rp, 256, 2))[0],
                r0, ra, c0, cbt, rp)
               for r0 in (10, 11, 12, 13) for ra in (1, 3, 6) for c0 in (4, 16, 24) for cbt in (16, 24, 32)
               for rp in (8, 15, 19))
    print(f"grid best    {best[0] * 1e3:7.2f} ms  (R0, Ra, cb0, cb, Rp in tiles) = {best[1:]}")


if __name__ == "__main__":
    main()
