"""A/B of plan-time variants (environment variables read while the plan is
built), timed on one ES population in one process:
    python tools/plan_ab.py <workload> <genomes> VAR=a,b"""
import os, sys
sys.path.insert(0, '.')
import torch
import paper_2111_00655_b200 as tp
from paper_2111_00655_b200 import workloads
from paper_2111_00655_b200.es_device import DeviceEvolution
name, P = sys.argv[1], int(sys.argv[2])
var, vals = sys.argv[3].split('=')[0], sys.argv[3].split('=')[1].split(',')
g = workloads.CONFIGS[name]()
bs = workloads.paper_backends(g, verify=False) if name != 'random100k' else workloads.random_backends(g, 8, 1, 0)
res = tp.optimize(g, bs.registry, bs.measurer, 0.01, validate=False)
plans = {}
for v in vals:
    os.environ[var] = v
    plans[v] = tp.FitnessPlan(g, bs.registry, bs.measurer, res.placement, 0.01, bs.graph_backend,
                              res.kernel_matches)
es = DeviceEvolution(plans[vals[0]], P, seed=1)
es.initialize()
for _ in range(int(os.environ.get('AB_GENS', '1'))):
    es.step()
pop = es.pop[es.cur]
fit = torch.empty(P, dtype=torch.float64, device='cuda')
ref, times = None, {v: [] for v in vals}
for rep in range(3):
    for v in vals:
        plans[v].evaluate_device(pop.data_ptr(), P, fit.data_ptr())
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        plans[v].evaluate_device(pop.data_ptr(), P, fit.data_ptr())
        e1.record(); torch.cuda.synchronize()
        times[v].append(e0.elapsed_time(e1))
        if ref is None:
            ref = fit.clone()
        assert torch.equal(fit, ref), v
for v, ts in times.items():
    print(name, P, plans[v].kernel_name(), f'{var}={v}', ' '.join(f'{t:.2f}' for t in ts), f'min {min(ts):.2f} ms')
