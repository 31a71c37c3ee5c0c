import sys, os
sys.path.insert(0, os.getcwd())
import torch
import bench
S, v = bench.make_shard(1024, 10_000_000, 1, torch.device("cuda", 0), torch.float32)
torch.cuda.synchronize()
print("free/total GB after S", [x / 1e9 for x in torch.cuda.mem_get_info()])
from paper_2310_17556_b200 import _lib
ctx = _lib.context_for(0, 1024, 10_000_000)
print("free after ctx", torch.cuda.mem_get_info()[0] / 1e9)
import paper_2310_17556_b200 as fsb
system = fsb.DampedSystem(fsb.ScoreMatrix(S), 1e-3, v)
print("free after system", torch.cuda.mem_get_info()[0] / 1e9)
sol = fsb.solve_chol(system)
print("ok", sol.rel_residual, "free", torch.cuda.mem_get_info()[0] / 1e9)
