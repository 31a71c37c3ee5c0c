cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r5p_build.log 2>&1
timeout 600 python -c "
import sys, time; sys.path.insert(0,'.')
import torch, paper_2310_17556_b200 as fsb
for dt in (torch.float32, torch.float64):
    S = (torch.randn(1024, 1000000, device='cuda') / 32).to(dt)
    sm = fsb.ScoreMatrix(S)
    for i in range(4):
        torch.cuda.synchronize(); t0 = time.perf_counter(); G = fsb.gram_packed(sm, 1e-3, 'fp64'); torch.cuda.synchronize()
        print(dt, 'fp64 gram ms', round(1e3*(time.perf_counter()-t0), 2), flush=True)
    del S, sm; torch.cuda.empty_cache()
" > gpurun_out/r5p.log 2>&1
