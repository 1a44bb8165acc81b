import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_1706_10086_b200 import gemm as G
n = 2048
A = torch.ones((n, n), dtype=torch.float64, device="cuda")
B = torch.ones((n, n), dtype=torch.float64, device="cuda")
# B row k = k+1 so a missing / repeated k shows in the value
B = B * torch.arange(1, n + 1, dtype=torch.float64, device="cuda")[:, None]
for S in (2, 4):
    C = torch.zeros((n, n), dtype=torch.float64, device="cuda")
    G.gemm(A, B, C, 1.0, 0.0, cfg=G.cfg_id("tma_64x64x16_w32x16_s6_splitk"), splits=S)
    torch.cuda.synchronize()
    c = C.cpu().numpy()
    exp = n * (n + 1) / 2
    bad = np.argwhere(c != exp)
    print("S", S, "bad entries", len(bad), "unique diffs", np.unique(np.round(c[c != exp] - exp))[:20])
    if len(bad):
        tiles = set((int(i) // 64, int(j) // 64) for i, j in bad)
        print(" bad tiles", len(tiles), sorted(tiles)[:10])
        i, j = bad[0]
        ti, tj = i // 64 * 64, j // 64 * 64
        blk = c[ti:ti + 64, tj:tj + 64] != exp
        print(" pattern rows with bad in first bad tile", np.nonzero(blk.any(axis=1))[0][:64].tolist())
        print(" pattern cols", np.nonzero(blk.any(axis=0))[0][:64].tolist())
