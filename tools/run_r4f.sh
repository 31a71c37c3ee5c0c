cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r4f_build.log 2>&1
timeout 300 python tools/prof_gram.py 1024 1000000 fp64 5 > gpurun_out/r4f_gram.log 2>&1
timeout 300 python tools/prof_gram.py 4096 200000 fp64 3 >> gpurun_out/r4f_gram.log 2>&1
timeout 300 python tools/gram_accuracy.py >> gpurun_out/r4f_acc.log 2>&1
timeout 1200 python -m pytest tests -q -m gpu -p no:cacheprovider -x -k "fp64 or dmma or gram or repeated" > gpurun_out/r4f_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r4f_rc.txt
