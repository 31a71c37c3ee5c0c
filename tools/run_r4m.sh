cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r4m_build.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'bjacobi_kernel' -c 1 -o gpurun_out/r4m_bj python -c "
import sys; sys.path.insert(0,'.')
import torch, paper_2310_17556_b200 as fsb
S = torch.randn(1024, 200000, device='cuda') / 32
w, U, sweeps = fsb.eigh_gram(fsb.ScoreMatrix(S), 'fp64'); torch.cuda.synchronize(); print('sweeps', sweeps)
" > gpurun_out/r4m_ncu.log 2>&1; echo "ncu rc=$?" >> gpurun_out/r4m_rc.txt
