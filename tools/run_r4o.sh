cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r4o_build.log 2>&1
for t in 1e-14 1e-12 1e-10 1e-8; do
  echo "tol $t" >> gpurun_out/r4o_eigh.log
  FS_SYEVJ_TOL=$t timeout 600 python tools/prof_eigh_stages.py >> gpurun_out/r4o_eigh.log 2>&1
  FS_SYEVJ_TOL=$t timeout 600 python -c "
import sys; sys.path.insert(0,'.')
import torch, paper_2310_17556_b200 as fsb
S = torch.randn(1024, 1000000, device='cuda') / 32
for p in ('f16x2','fp64'):
    w, U, sweeps = fsb.eigh_gram(fsb.ScoreMatrix(S), p); torch.cuda.synchronize(); print(p, 'sweeps', sweeps)
" >> gpurun_out/r4o_eigh.log 2>&1
done
