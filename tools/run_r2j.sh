cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2j_build.log 2>&1
FS_SYRK_DBG=768 timeout 300 python tools/prof_solve.py 1024 1000000 2 > gpurun_out/r2j_dbg768.log 2>&1
FS_SYRK_DBG=1792 timeout 300 python tools/prof_solve.py 1024 1000000 2 > gpurun_out/r2j_dbg1792.log 2>&1
FS_SYRK_DBG=768 timeout 300 python tools/prof_solve.py 256 1000000 2 > gpurun_out/r2j_dbg768_256.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-modes > gpurun_out/r2j_bench.log 2>&1
FS_F16_RING=0 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-modes > gpurun_out/r2j_bench_tiled.log 2>&1
FS_F16_RING=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/r2j_launches.csv python tools/prof_solve.py 1024 1000000 2 > /dev/null 2>&1
