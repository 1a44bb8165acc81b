"""Layout probes for the tcgen05 tf32 path (debugging aid)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
from paper_1706_10086_b200 import gemm as G

def run(A, B):
    M, K = A.shape; N = B.shape[1]
    dA = torch.from_numpy(A.astype(np.float32)).cuda(); dB = torch.from_numpy(B.astype(np.float32)).cuda()
    dC = torch.zeros((M, N), dtype=torch.float32, device="cuda")
    G.gemm_f32(dA, dB, dC, 1.0, 0.0); torch.cuda.synchronize()
    return dC.cpu().numpy()

np.set_printoptions(linewidth=200)
M = N = 128; K = 32
# P1: A = "k-selector" (A[i][k] = 1 iff k == i % 32), B[k][j] = 100*k + j  -> C[i][j] = 100*(i%32) + j
A = np.zeros((M, K)); A[np.arange(M), np.arange(M) % K] = 1
B = 100.0 * np.arange(K)[:, None] + np.arange(N)[None, :]
C = run(A, B); ref = A @ B
print("P1 ok", np.array_equal(C, ref)); print("C[0:4,0:8]\n", C[0:4, 0:8]); print("ref\n", ref[0:4, 0:8])
print("C[33,0:8]", C[33, 0:8], "C[64,0:8]", C[64, 0:8])
# P2: A[i][k] = i*1000 + k (exact), B = selector B[k][j] = 1 iff j == k
A = 1000.0 * np.arange(M)[:, None] + np.arange(K)[None, :]
B = np.zeros((K, N)); B[np.arange(K), np.arange(K)] = 1
C = run(A, B); ref = A @ B
print("P2 ok", np.array_equal(C, ref)); print("C[0:3,0:10]\n", C[0:3, 0:10]); print("C[5,0:34]", C[5, 0:34])
# P3: single nonzero A[i0][k0]=1, B[k0][j0]=1
for (i0, k0, j0) in [(0, 0, 0), (1, 0, 0), (0, 1, 0), (0, 0, 1), (9, 3, 5), (40, 17, 77), (100, 31, 127)]:
    A = np.zeros((M, K)); A[i0, k0] = 1; B = np.zeros((K, N)); B[k0, j0] = 1
    C = run(A, B); nz = np.argwhere(C != 0)
    print("P3", (i0, k0, j0), "nonzeros at", nz[:6].tolist(), "vals", C[C != 0][:6])
# P4: only B row k0 = ones, A col k0 = ones
for k0 in [0, 1, 4, 8, 9, 31]:
    A = np.zeros((M, K)); A[:, k0] = 1; B = np.zeros((K, N)); B[k0, :] = 1
    C = run(A, B)
    print("P4 k0", k0, "sum", C.sum(), "expected", M * N, "distinct", np.unique(C)[:5])
