cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2s_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_env_paths.py tests/test_gpu_parity.py -q -m gpu -p no:cacheprovider -k "potrf or host_entry or chunked" > gpurun_out/r2s_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2s_rc.txt
timeout 900 python tools/large_fit.py --potrf-ns 6144,8192,12288,16384 --skip-solve > gpurun_out/r2s_large.log 2>&1; echo "large rc=$?" >> gpurun_out/r2s_rc.txt
FS_POTRF_LOOKAHEAD=0 timeout 900 python tools/large_fit.py --potrf-ns 16384 --skip-solve > gpurun_out/r2s_large_nola.log 2>&1
