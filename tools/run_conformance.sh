cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/cf_build.log 2>&1
timeout 1800 python tools/ref_conformance.py --all --out gpurun_out/cf_all.json > gpurun_out/cf.log 2>&1
timeout 1800 python tools/ref_conformance.py --out gpurun_out/cf_sel.json > gpurun_out/cf_sel.log 2>&1
