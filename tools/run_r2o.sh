cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2o_build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_env_paths.py -q -m gpu -p no:cacheprovider > gpurun_out/r2o_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2o_rc.txt
timeout 1200 python tools/large_fit.py > gpurun_out/r2o_large.log 2>&1; echo "large rc=$?" >> gpurun_out/r2o_rc.txt
