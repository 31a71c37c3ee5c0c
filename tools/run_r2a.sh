cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_r2.py -x -q -m gpu > gpurun_out/r2_t1.log 2>&1
timeout 600 python tools/refine_headline.py > gpurun_out/r2_refine.log 2>&1
