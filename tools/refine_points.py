import sys, json
sys.path.insert(0, '/root/repo')
sys.argv = ['x']
import importlib.util
spec = importlib.util.spec_from_file_location("sweep", "/root/repo/tools/sweep.py"); sw = importlib.util.module_from_spec(spec); spec.loader.exec_module(sw)
for n, m in ((1024, 1_000_000), (1024, 3_000_000), (1024, 10_000_000), (2048, 1_000_000)):
    print(json.dumps(sw.point(n, m, "f16x2")), flush=True)
