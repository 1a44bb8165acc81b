import sys, numpy as np, torch
sys.path.insert(0, '.')
import oracle, synth
from paper_1706_10086_b200 import gemm as G
for n in (512, 1024, 2048):
    A, B, C0 = synth.problem(n, n, n, seed=3)
    ref = oracle.dgemm(1.0, A, B, 0.0, np.zeros((n, n)))
    dA, dB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    for name, S in (("tma_64x64x16_w32x16_s6", None), ("tma_64x64x16_w32x16_s6_splitk", 1), ("tma_64x64x16_w32x16_s6_splitk", 2), ("tma_64x64x16_w32x16_s6_splitk", 4), ("tma_128x64x16_w32x16_s6", None), ("tma_64x64x16_w64x32_s6", None)):
        dC = torch.zeros((n, n), dtype=torch.float64, device="cuda")
        G.gemm(dA, dB, dC, 1.0, 0.0, cfg=G.cfg_id(name), splits=S)
        torch.cuda.synchronize()
        err = np.abs(dC.cpu().numpy() - ref).max()
        print(n, name, S, "max abs err %.3e" % err, flush=True)
