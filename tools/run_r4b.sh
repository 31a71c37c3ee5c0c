cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r4b_build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_properties.py -q -m gpu -p no:cacheprovider --durations=10 > gpurun_out/r4b_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r4b_rc.txt
