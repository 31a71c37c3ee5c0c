cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nproc > gpurun_out/r4h_pageable.log
for w in 4 8 12 15; do FS_STAGE_WORKERS=$w timeout 300 python tools/prof_pageable.py >> gpurun_out/r4h_pageable.log 2>&1; done
timeout 600 python -m pytest tests -q -m gpu -p no:cacheprovider -k "staged or pageable" > gpurun_out/r4h_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r4h_rc.txt
