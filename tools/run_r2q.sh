cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2q_build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_env_paths.py -q -m gpu -p no:cacheprovider -k potrf > gpurun_out/r2q_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2q_rc.txt
timeout 1200 python tools/large_fit.py --potrf-ns 2048,4096,8192,16384 > gpurun_out/r2q_large.log 2>&1; echo "large rc=$?" >> gpurun_out/r2q_rc.txt
FS_POTRF_BLOCKED_MINN=2048 timeout 600 python tools/large_fit.py --potrf-ns 2048,3072 --skip-solve > gpurun_out/r2q_small.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2q_potrf_launches.csv python tools/large_fit.py --potrf-ns 16384 --skip-solve > /dev/null 2>&1
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/r2q_alltests.log 2>&1; echo "alltests rc=$?" >> gpurun_out/r2q_rc.txt
