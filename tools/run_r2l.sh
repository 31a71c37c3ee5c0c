cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2l_build.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-modes > gpurun_out/r2l_bench.log 2>&1
FS_CY_CLMIN=8 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-modes > gpurun_out/r2l_bench_cl8.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/r2l_launches.csv python tools/prof_solve.py 1024 1000000 2 > /dev/null 2>&1
FS_CY_CLMIN=8 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/r2l_launches_cl8.csv python tools/prof_solve.py 1024 1000000 2 > /dev/null 2>&1
timeout 1500 python -m pytest tests -q -m gpu -x -p no:cacheprovider > gpurun_out/r2l_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2l_rc.txt
