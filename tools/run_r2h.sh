cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2h_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -p no:cacheprovider -k "split_k_with_more or refinement_contracts" > gpurun_out/r2h_tests.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/r02_bench_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r2h_ncu_launch.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"syrk_tc_kernel|retile16|cols_solve_y_cl|residual_cols|potrf_persistent" -c 5 -o gpurun_out/r02_full python tools/prof_solve.py 1024 1000000 1 > gpurun_out/r2h_ncu_full.log 2>&1
timeout 1500 python tools/ref_conformance.py --out gpurun_out/r02_ref_conformance.json > gpurun_out/r2h_conf.log 2>&1
bash tools/sanitize.sh
