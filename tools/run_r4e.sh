cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r4e_build.log 2>&1
bash tools/syrk_ablate.sh 0 8192 8 0 8192 8 > gpurun_out/r4e_ablate.log 2>&1
FS_SYRK_DBG=0 timeout 600 python tools/ring_check.py run /tmp/red.npz > gpurun_out/r4e_red.log 2>&1
FS_SYRK_DBG=8192 timeout 600 python tools/ring_check.py run /tmp/rmw.npz > gpurun_out/r4e_rmw.log 2>&1
python tools/ring_check.py compare /tmp/red.npz /tmp/rmw.npz > gpurun_out/r4e_cmp.log 2>&1
FS_PREC=tf32x3 bash tools/syrk_ablate.sh 0 8192 > gpurun_out/r4e_ablate_tf32.log 2>&1
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r4e_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/r4e_rc.txt
