cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2p_build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_env_paths.py -q -m gpu -p no:cacheprovider > gpurun_out/r2p_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2p_rc.txt
for N in 2048 4096 8192; do
 for F in 100000 1; do
  FS_POTRF_FUSE_MAXN=$F timeout 600 python tools/large_fit.py --potrf-ns "" --n $N --m 200000 > gpurun_out/r2p_n${N}_f${F}.log 2>&1
 done
done
timeout 1200 python tools/large_fit.py --potrf-ns "" > gpurun_out/r2p_large.log 2>&1; echo "large rc=$?" >> gpurun_out/r2p_rc.txt
