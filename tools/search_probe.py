"""Phase times of one full placement search (bench.py's `search`) on a workload."""
import cProfile, os, pstats, sys, time
sys.path.insert(0, '.')
import torch
import paper_2111_00655_b200 as tp
from paper_2111_00655_b200 import workloads
from paper_2111_00655_b200.es_device import DeviceEvolution
name = sys.argv[1] if len(sys.argv) > 1 else 'random100k'
g = workloads.CONFIGS[name]()
bs = workloads.random_backends(g, 8, 1, 0) if name == 'random100k' else workloads.paper_backends(g, verify=False)
for rep in range(2):
    bs.registry._tables.clear()
    meas = tp.SimMeasurer(bs.measurer.profiles)
    torch.cuda.synchronize()
    pr = cProfile.Profile() if rep else None
    if pr: pr.enable()
    t0 = time.perf_counter()
    res = tp.optimize(g, bs.registry, meas, 0.01)
    t1 = time.perf_counter()
    if rep: os.environ['CB_PLAN_TIMING'] = '1'
    plan = tp.FitnessPlan(g, bs.registry, meas, res.placement, 0.01, bs.graph_backend, res.kernel_matches)
    os.environ.pop('CB_PLAN_TIMING', None)
    t2 = time.perf_counter()
    es = DeviceEvolution(plan, 65536, seed=0)
    t3 = time.perf_counter()
    es.initialize(); torch.cuda.synchronize()
    t4 = time.perf_counter()
    for _ in range(10): es.step()
    torch.cuda.synchronize()
    t5 = time.perf_counter()
    if pr: pr.disable()
    print(f"rep {rep}: optimize {t1-t0:.3f} {res.device['phases_s']} plan {t2-t1:.3f} es_ctor {t3-t2:.3f} init {t4-t3:.3f} 10 gens {t5-t4:.3f} total {t5-t0:.3f}", flush=True)
pstats.Stats(pr).sort_stats('cumtime').print_stats(18)
