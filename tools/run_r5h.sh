cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r5h_build.log 2>&1
for shape in "4096 500000" "8192 250000"; do
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second,lts__t_sector_hit_rate.pct --clock-control none -k regex:syrk_tc_kernel -c 1 --csv python tools/prof_gram.py $shape f16x2 1 2>/dev/null | grep syrk_tc >> gpurun_out/r5h_ncu.csv
  timeout 300 python tools/prof_gram.py $shape f16x2 3 >> gpurun_out/r5h_time.log 2>&1
done
