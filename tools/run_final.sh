# full validation of the current tree on one B200: build, smoke, GPU suite, bench (+ reference arm),
# ncu launch list; outputs under gpurun_out/final_*
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/final_build.log 2>&1
timeout 600 python __graft_entry__.py --smoke > gpurun_out/final_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/final_rc.txt
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/final_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/final_rc.txt
timeout 900 python bench.py > gpurun_out/final_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/final_rc.txt
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/final_bench_ref.log 2>&1; echo "ref rc=$?" >> gpurun_out/final_rc.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/final_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-modes > gpurun_out/final_ncul.log 2>&1; echo "ncul rc=$?" >> gpurun_out/final_rc.txt
