cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2n_build.log 2>&1
FS_F16_RING=1 FS_SYRK_DBG=2816 timeout 300 python tools/prof_solve.py 1024 1000000 2 > gpurun_out/r2n_dbg.log 2>&1
FS_F16_RING=1 FS_SYRK_DBG=2048 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:syrk -c 4 --csv --log-file gpurun_out/r2n_launches.csv python tools/prof_solve.py 1024 1000000 2 > /dev/null 2>&1
FS_F16_RING=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:syrk -c 4 --csv --log-file gpurun_out/r2n_launches_conv.csv python tools/prof_solve.py 1024 1000000 2 > /dev/null 2>&1
