"""A/B of the host pipeline (cb_fitness_host) on uniform random genomes."""
import os, sys, time
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2111_00655_b200 as tp
from paper_2111_00655_b200 import workloads
import bench
name, E = sys.argv[1], int(sys.argv[2])
vals = sys.argv[3].split(',')
g = workloads.CONFIGS[name]()
bs = workloads.random_backends(g, 8, 1, 0) if name == 'random100k' else workloads.paper_backends(g, verify=False)
res = tp.optimize(g, bs.registry, bs.measurer, 0.01, validate=False)
plan = tp.FitnessPlan(g, bs.registry, bs.measurer, res.placement, 0.01, bs.graph_backend, res.kernel_matches)
host = torch.empty((E, plan.words), dtype=torch.int64, pin_memory=True)
hn = host.numpy().view(np.uint64); hn[:] = bench.uniform_rows(E, plan.k, 1000)
fit = torch.empty(E, dtype=torch.float64, pin_memory=True).numpy()
plan.evaluate_packed(hn, fit)
ref = fit.copy()
for rep in range(3):
    for v in vals:
        os.environ['CB_HOST_CHUNK_PER_SM'] = v
        t0 = time.perf_counter(); plan.evaluate_packed(hn, fit); dt = time.perf_counter() - t0
        assert np.array_equal(fit, ref)
        print(name, E, 'per_sm', v, f'{dt*1e3:.1f} ms', f'{E/dt/1e6:.3f} M/s', flush=True)
