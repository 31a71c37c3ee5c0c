cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2i_build.log 2>&1
FS_F16_RING=1 timeout 600 python tools/ring_check.py run /tmp/ring.npz > gpurun_out/r2i_ring.log 2>&1; echo "ring rc=$?" >> gpurun_out/r2i_rc.txt
FS_F16_RING=0 timeout 600 python tools/ring_check.py run /tmp/tiled.npz > gpurun_out/r2i_tiled.log 2>&1; echo "tiled rc=$?" >> gpurun_out/r2i_rc.txt
python tools/ring_check.py compare /tmp/ring.npz /tmp/tiled.npz > gpurun_out/r2i_compare.log 2>&1
FS_SYRK_DBG=256 timeout 300 python tools/prof_solve.py 1024 1000000 2 > gpurun_out/r2i_dbg.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2i_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/r2i_rc.txt
timeout 1500 python -m pytest tests -q -m gpu -x -p no:cacheprovider > gpurun_out/r2i_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2i_rc.txt
