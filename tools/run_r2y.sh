cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2y_build.log 2>&1
timeout 1200 python -m pytest tests -q -m gpu -p no:cacheprovider -k "svd or eigh or eig" > gpurun_out/r2y_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2y_rc.txt
timeout 1200 python tools/ref_conformance.py --out gpurun_out/r02_ref_conformance.json > gpurun_out/r2y_conf.log 2>&1; echo "conf rc=$?" >> gpurun_out/r2y_rc.txt
timeout 600 python tools/prof_eigh.py > gpurun_out/r2y_routes.log 2>&1
