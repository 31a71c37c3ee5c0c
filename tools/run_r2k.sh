cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2k_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_r2.py -q -m gpu -x -p no:cacheprovider -k "trsv or refine or headline or chol" > gpurun_out/r2k_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2k_rc.txt
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-modes > gpurun_out/r2k_bench.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/r2k_launches.csv python tools/prof_solve.py 1024 1000000 2 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"cols_solve_y_cl|trsv_pair" -c 4 -o gpurun_out/r2k_xpass python tools/prof_solve.py 1024 1000000 1 > gpurun_out/r2k_ncu.log 2>&1
