cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r4n_build.log 2>&1
FS_SYEVJ_DBG=3 timeout 600 python tools/prof_eigh_stages.py > gpurun_out/r4n_eigh.log 2>&1
timeout 1200 python -m pytest tests -q -m gpu -p no:cacheprovider -x -k "eigh or jacobi or svd or syevj or routes or repeated or complex" > gpurun_out/r4n_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r4n_rc.txt
