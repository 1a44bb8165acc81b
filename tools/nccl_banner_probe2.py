"""Does the library's own NCCL communicator print NCCL's version banner on stdout?"""
import sys
import torch
sys.path.insert(0, ".")
from paper_1706_10086_b200 import gemm as G
torch.cuda.set_device(0)
c = G.Comm(0, 1)
x = torch.ones(8, dtype=torch.float64, device="cuda")
c.bcast(x)
torch.cuda.synchronize()
c.close()
print("probe done", file=sys.stderr)
