"""cProfile of the host side of one placement search (optimize + plan) on a config."""
import cProfile, pstats, sys, time
sys.path.insert(0, '.')
import paper_2111_00655_b200 as tp
from paper_2111_00655_b200 import workloads
name = sys.argv[1] if len(sys.argv) > 1 else 'random100k'
g = workloads.CONFIGS[name]()
bs = workloads.paper_backends(g) if name != 'random100k' else workloads.random_backends(g, 8, 1, 0)
res = tp.optimize(g, bs.registry, bs.measurer, 0.01, validate=False)  # warm
bs.registry._tables.clear()
pr = cProfile.Profile()
t0 = time.perf_counter()
pr.enable()
res = tp.optimize(g, bs.registry, bs.measurer, 0.01, validate=False)
t1 = time.perf_counter()
plan = tp.FitnessPlan(g, bs.registry, bs.measurer, res.placement, 0.01, bs.graph_backend, res.kernel_matches)
pr.disable()
t2 = time.perf_counter()
print(f"optimize {t1 - t0:.3f}s plan {t2 - t1:.3f}s device {res.device}")
pstats.Stats(pr).sort_stats('tottime').print_stats(25)
