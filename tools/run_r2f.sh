cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_r2.py tests/test_multirank_gpu.py -q -m gpu > gpurun_out/r2_t2.log 2>&1
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_cli_fmat.py tests/test_all_finite_abi.py -q -m gpu > gpurun_out/r2_t3.log 2>&1
timeout 1500 python tools/ref_conformance.py --out gpurun_out/r02_ref_conformance.json > gpurun_out/r2_conf.log 2>&1
timeout 900 python bench.py > gpurun_out/r2_bench.log 2>&1
timeout 600 python __graft_entry__.py --smoke > gpurun_out/r2_smoke.log 2>&1
