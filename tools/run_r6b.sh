cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r6b_build.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'trsv' -c 4 --csv python tools/prof_solve.py 1024 1000000 1 2>/dev/null | grep trsv | awk -F'","' '{print $5, $NF}' > gpurun_out/r6b_ncu.log
for i in 1 2; do timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-modes --e2e-steps 0 2>/dev/null | grep '^{' | python -c "import sys,json; d=json.loads(sys.stdin.read()); s=d['stage_ms']; print(round(d['ms_per_step'],3), 'refine', round(s['refine'],3))" >> gpurun_out/r6b_bench.log; done
timeout 1800 python -m pytest tests -q -m gpu -p no:cacheprovider -x -k "trsv or potrf or pivot or chol or repeated or refine or fuzz or cho_ or workspace" > gpurun_out/r6b_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r6b_rc.txt
