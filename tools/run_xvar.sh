cd $GRAFT_REPO_ROOT
for v in 7 6 8; do
  sed -i "s/constexpr int kCLXW = [0-9]*; /constexpr int kCLXW = $v; /" paper_2310_17556_b200/csrc/gemv.cu
  python -c "import paper_2310_17556_b200.build as b; b.build()" > /dev/null 2>&1
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:cols_solve -c 3 --csv python tools/prof_solve.py 1024 1000000 1 2>/dev/null | grep cols_solve | awk -F'","' -v v=$v '{print "XW=" v, $NF}'
done
