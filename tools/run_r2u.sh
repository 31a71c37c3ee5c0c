cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2u_build.log 2>&1
timeout 1200 python -m pytest tests -q -m gpu -p no:cacheprovider -k "eigh or eig or svd or complex or hermitian" > gpurun_out/r2u_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2u_rc.txt
timeout 600 python tools/prof_eigh.py > gpurun_out/r2u_eigh.log 2>&1
FS_SYEVJ_BLOCK=0 timeout 600 python tools/prof_eigh.py 1024 100000 > gpurun_out/r2u_eigh_scalar.log 2>&1
timeout 600 python tools/prof_eigh.py 1024 100000 > gpurun_out/r2u_eigh_small.log 2>&1
