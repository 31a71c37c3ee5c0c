free -g; nproc; nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv
python - <<'PY'
import time, numpy as np
t=time.perf_counter()
rng=np.random.Generator(np.random.PCG64(0))
S=rng.standard_normal((1024,1000000),dtype=np.float32)
print("gen f32 1e9:", time.perf_counter()-t)
PY
python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -2
