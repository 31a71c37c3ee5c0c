cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2t_build.log 2>&1
timeout 600 python __graft_entry__.py --smoke > gpurun_out/r2t_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r2t_rc.txt
timeout 1800 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/r2t_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2t_rc.txt
timeout 900 python bench.py > gpurun_out/r2t_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/r2t_rc.txt
timeout 600 python tools/prof_eigh.py > gpurun_out/r2t_eigh.log 2>&1
