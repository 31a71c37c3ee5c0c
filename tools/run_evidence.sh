# Evidence run of the current tree on one B200 (outputs under gpurun_out/ev_*): build, smoke, the
# GPU suite, bench (+ reference arm), ncu launch list and full capture, routes, n/m sweep, potrf.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ev_build.log 2>&1
timeout 600 python __graft_entry__.py --smoke > gpurun_out/ev_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/ev_rc.txt
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/ev_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/ev_rc.txt
timeout 900 python bench.py > gpurun_out/ev_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/ev_rc.txt
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/ev_bench_ref.log 2>&1; echo "ref rc=$?" >> gpurun_out/ev_rc.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/ev_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-modes > gpurun_out/ev_ncul.log 2>&1; echo "ncul rc=$?" >> gpurun_out/ev_rc.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'syrk_tc_kernel|retile16|cols_solve_y_cl|residual_cols|potrf_persistent|trsv_pair' -c 10 -o gpurun_out/ev_full python tools/prof_solve.py 1024 1000000 1 > gpurun_out/ev_ncu.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ev_rc.txt
timeout 900 python tools/prof_eigh.py > gpurun_out/ev_routes.log 2>&1; echo "routes rc=$?" >> gpurun_out/ev_rc.txt
timeout 1200 python tools/sweep.py gpurun_out/ev_sweep.json > gpurun_out/ev_sweep.log 2>&1; echo "sweep rc=$?" >> gpurun_out/ev_rc.txt
timeout 900 python tools/large_fit.py --skip-solve --potrf-ns 1024,2048,4096,6144,8192,12288,16384 > gpurun_out/ev_potrf.log 2>&1; echo "potrf rc=$?" >> gpurun_out/ev_rc.txt
