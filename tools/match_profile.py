"""Host profile of building the match table of a config (device matcher + download)."""
import cProfile, pstats, sys, time
sys.path.insert(0, '.')
import torch
from paper_2111_00655_b200 import workloads
name = sys.argv[1] if len(sys.argv) > 1 else 'random100k'
g = workloads.CONFIGS[name]()
bs = workloads.paper_backends(g) if name != 'random100k' else workloads.random_backends(g, 8, 1, 0)
for rep in range(3):
    bs.registry._tables.clear()
    torch.cuda.synchronize()
    pr = cProfile.Profile()
    t0 = time.perf_counter()
    pr.enable()
    t = bs.registry.match_table(g)
    pr.disable()
    torch.cuda.synchronize()
    print(rep, f"{1e3 * (time.perf_counter() - t0):.1f} ms", t.n_matches)
pstats.Stats(pr).sort_stats('tottime').print_stats(12)
