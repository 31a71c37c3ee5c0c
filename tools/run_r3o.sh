cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for d in 0 4096; do
  FS_SYRK_DBG=$d timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:syrk_tc_kernel -c 2 --csv python tools/prof_solve.py 1024 1000000 1 2>/dev/null | grep syrk_tc_kernel | awk -F'","' -v d=$d '{print "dbg=" d, $(NF-2), $NF}'
  FS_SYRK_DBG=$d timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-modes 2>/dev/null | grep '^{' | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('bench dbg', d['value'], d['stage_ms']['gram'])"
done
