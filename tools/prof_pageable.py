"""Time ScoreMatrix construction from a pageable 4.1 GB numpy array (the drop-in's host upload)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2310_17556_b200 as fsb
S = np.random.default_rng(0).standard_normal((1024, 1_000_000), dtype=np.float32)
for rep in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    sm = fsb.ScoreMatrix(S)
    torch.cuda.synchronize()
    print(f"workers={os.environ.get('FS_STAGE_WORKERS', 'default')} construct {1e3 * (time.perf_counter() - t0):.1f} ms", flush=True)
    del sm
