cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r5o_build.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r5o_routes.csv python -c "
import sys; sys.path.insert(0,'.')
import torch, paper_2310_17556_b200 as fsb
S = torch.randn(1024, 1000000, device='cuda') / 32; v = torch.randn(1000000, device='cuda')
system = fsb.DampedSystem(fsb.ScoreMatrix(S), 1e-3, v)
torch.cuda.synchronize(); print('EIGH'); fsb.solve_svd_eigh(system); torch.cuda.synchronize()
print('SVD'); fsb.solve_svd_direct(system); torch.cuda.synchronize()
" > gpurun_out/r5o.log 2>&1
