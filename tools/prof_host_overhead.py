"""Host-side cost of one solve_chol call (tiny device work): wall time per call, and a cProfile
of the Python path."""
import cProfile, os, pstats, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2310_17556_b200 as fsb
dev = torch.device("cuda", 0)
for n, m in ((8, 64), (1024, 1_000_000)):
    S = torch.randn(n, m, device=dev) / n ** 0.5
    v = torch.randn(m, device=dev)
    system = fsb.DampedSystem(fsb.ScoreMatrix(S), 1e-3, v)
    for _ in range(5):
        fsb.solve_chol(system)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(50):
        fsb.solve_chol(system)
    torch.cuda.synchronize()
    print(f"n={n} m={m}: {1e3 * (time.perf_counter() - t0) / 50:.3f} ms per call (wall)", flush=True)
S = torch.randn(8, 64, device=dev)
system = fsb.DampedSystem(fsb.ScoreMatrix(S), 1e-3, torch.randn(64, device=dev))
pr = cProfile.Profile()
pr.enable()
for _ in range(200):
    fsb.solve_chol(system)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(15)
