cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r4g_build.log 2>&1
timeout 600 python __graft_entry__.py --smoke > gpurun_out/r4g_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r4g_rc.txt
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/r4g_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r4g_rc.txt
timeout 900 python bench.py > gpurun_out/r4g_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/r4g_rc.txt
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r4g_bench_ref.log 2>&1; echo "ref rc=$?" >> gpurun_out/r4g_rc.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'syrk_tc_kernel|retile16|cols_solve_y_cl|residual_cols|potrf_persistent|trsv_pair' -c 9 -o gpurun_out/r4g_full python tools/prof_solve.py 1024 1000000 1 > gpurun_out/r4g_ncu.log 2>&1; echo "ncu rc=$?" >> gpurun_out/r4g_rc.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/r4g_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-modes > gpurun_out/r4g_ncul.log 2>&1; echo "ncul rc=$?" >> gpurun_out/r4g_rc.txt
