cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r5r_build.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/r5r.csv python -c "
import sys; sys.path.insert(0,'.')
import torch, paper_2310_17556_b200 as fsb
S = torch.randn(1024, 1000000, device='cuda') / 32; v = torch.randn(1000000, device='cuda')
system = fsb.DampedSystem(fsb.ScoreMatrix(S), 1e-3, v)
torch.cuda.synchronize(); fsb.solve_chol(system, precision='fp64'); torch.cuda.synchronize()
fsb.solve_svd_direct(system); torch.cuda.synchronize()
fsb.residual(system, torch.zeros(1000000, dtype=torch.float64, device='cuda')); torch.cuda.synchronize()
" > gpurun_out/r5r.log 2>&1
