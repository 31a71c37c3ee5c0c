cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2r_build.log 2>&1
timeout 900 python tools/large_fit.py --potrf-ns 4096,6144,8192,12288,16384 --skip-solve > gpurun_out/r2r_large.log 2>&1; echo "large rc=$?" >> gpurun_out/r2r_rc.txt
timeout 600 ncu --set full --clock-control none -k regex:syrk_dmma_async -s 5 -c 1 -o gpurun_out/r2r_trail python tools/large_fit.py --potrf-ns 16384 --skip-solve > gpurun_out/r2r_ncu.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_env_paths.py -q -m gpu -p no:cacheprovider -k "host_entry or potrf or chunked" > gpurun_out/r2r_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2r_rc.txt
