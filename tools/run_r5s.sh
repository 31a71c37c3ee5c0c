cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r5s_build.log 2>&1
FS_SVDA_GRAM=0 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 200 --csv --log-file gpurun_out/r5s.csv python -c "
import sys; sys.path.insert(0,'.')
import torch, paper_2310_17556_b200 as fsb
S = torch.randn(1024, 1000000, device='cuda') / 32; v = torch.randn(1000000, device='cuda')
system = fsb.DampedSystem(fsb.ScoreMatrix(S), 1e-3, v)
torch.cuda.synchronize(); fsb.solve_svd_direct(system); torch.cuda.synchronize()
" > gpurun_out/r5s.log 2>&1
