cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r4a_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_r2.py tests/test_gpu_parity.py -q -m gpu -p no:cacheprovider -k "eigh or complex or svd" > gpurun_out/r4a_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r4a_rc.txt
timeout 600 python tools/prof_eigh.py > gpurun_out/r4a_prof_eigh.log 2>&1; echo "prof rc=$?" >> gpurun_out/r4a_rc.txt
