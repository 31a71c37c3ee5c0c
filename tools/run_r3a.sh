cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r3a_build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_env_paths.py tests/test_gpu_parity.py -q -m gpu -p no:cacheprovider -k "trsv or refine or chol or host_entry" > gpurun_out/r3a_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r3a_rc.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/r3a_launches.csv python tools/prof_solve.py 1024 1000000 2 > /dev/null 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-modes > gpurun_out/r3a_bench.log 2>&1
