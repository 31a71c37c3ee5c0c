cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r3f_build.log 2>&1
timeout 600 python __graft_entry__.py --smoke > gpurun_out/r3f_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r3f_rc.txt
timeout 1800 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/r3f_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r3f_rc.txt
timeout 900 python bench.py > gpurun_out/r3f_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/r3f_rc.txt
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r3f_bench_ref.log 2>&1; echo "ref rc=$?" >> gpurun_out/r3f_rc.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/r02_bench_launches_final.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-modes > gpurun_out/r3f_ncu.log 2>&1
