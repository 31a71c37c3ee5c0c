cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r4q_build.log 2>&1
timeout 600 python tools/large_fit.py --skip-solve --potrf-ns 1024,2048,4096,6144 > gpurun_out/r4q_potrf.log 2>&1
for i in 1 2; do timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-modes --e2e-steps 0 2>/dev/null | grep '^{' | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['stage_ms']['potrf'])" >> gpurun_out/r4q_bench.log; done
timeout 1200 python -m pytest tests -q -m gpu -p no:cacheprovider -x -k "potrf or pivot or chol or repeated or fuzz" > gpurun_out/r4q_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r4q_rc.txt
