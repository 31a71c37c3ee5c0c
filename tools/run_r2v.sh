cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2v_build.log 2>&1
timeout 1200 python -m pytest tests -q -m gpu -p no:cacheprovider -k "eigh or eig or svd or complex or hermitian" > gpurun_out/r2v_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2v_rc.txt
timeout 600 python tools/prof_eigh.py > gpurun_out/r2v_eigh.log 2>&1
for n in 256 2048 4096; do timeout 600 python tools/prof_eigh.py $n 200000 > gpurun_out/r2v_eigh_$n.log 2>&1; done
