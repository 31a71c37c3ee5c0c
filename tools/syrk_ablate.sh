#!/bin/bash
# Ablation of the tcgen05 SYRK: FS_SYRK_DBG bits 1=no load, 2=no convert, 4=no MMA,
# 8=no fp64 flush, 16=no TMEM drain, 64=L2 prefetch on.  Times the Gram stage only
# (S_t is produced once, untimed) via tools/prof_syrk_only.py.
for d in "$@"; do
  printf "dbg=%-3s " "$d"; FS_SYRK_DBG=$d timeout 60 python tools/prof_syrk_only.py | tail -1
done
