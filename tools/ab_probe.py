"""A/B of fitness-kernel variants selected by environment variables, in one
process on one ES population (alternating, repeated):
    python tools/ab_probe.py <workload> <genomes> VAR=a,b [VAR2=...]"""
import os, sys, itertools
sys.path.insert(0, '.')
import torch
import paper_2111_00655_b200 as tp
from paper_2111_00655_b200 import workloads
from paper_2111_00655_b200.es_device import DeviceEvolution
name, P = sys.argv[1], int(sys.argv[2])
axes = [(kv.split('=')[0], kv.split('=')[1].split(',')) for kv in sys.argv[3:]]
g = workloads.CONFIGS[name]()
bs = workloads.paper_backends(g, verify=False) if name != 'random100k' else workloads.random_backends(g, 8, 1, 0)
res = tp.optimize(g, bs.registry, bs.measurer, 0.01, validate=False)
plan = tp.FitnessPlan(g, bs.registry, bs.measurer, res.placement, 0.01, bs.graph_backend, res.kernel_matches)
es = DeviceEvolution(plan, P, seed=1)
es.initialize()
for _ in range(int(os.environ.get('AB_GENS', '1'))):
    es.step()
pop = es.pop[es.cur]
fit = torch.empty(P, dtype=torch.float64, device='cuda')
ref = None
times = {}
for rep in range(3):
    for combo in itertools.product(*[v for _, v in axes]):
        for (k, _), v in zip(axes, combo):
            if k == 'POOL':  # plan-level knob: merged-sum pool entries in shared memory
                plan.set_pool(int(v))
            else:
                os.environ[k] = v
        plan.evaluate_device(pop.data_ptr(), P, fit.data_ptr())  # warm
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        plan.evaluate_device(pop.data_ptr(), P, fit.data_ptr())
        e1.record(); torch.cuda.synchronize()
        times.setdefault(combo, []).append(e0.elapsed_time(e1))
        if ref is None:
            ref = fit.clone()
        assert torch.equal(fit, ref), combo
for combo, ts in times.items():
    print(name, P, dict(zip([k for k, _ in axes], combo)), ' '.join(f'{t:.1f}' for t in ts), f'min {min(ts):.1f} ms')
