"""Time the fitness kernels (both paths) on a workload's DP placement."""
import sys
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2111_00655_b200 as tp
from paper_2111_00655_b200 import workloads
name = sys.argv[1] if len(sys.argv) > 1 else 'bert_base'
P = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 22
PATHS = sys.argv[3].split(',') if len(sys.argv) > 3 else ['auto', 'wide', 'unionfind']
g = workloads.CONFIGS[name]()
bs = workloads.paper_backends(g) if name != 'random100k' else workloads.random_backends(g, 8, 1, 0)
res = tp.optimize(g, bs.registry, bs.measurer, 0.01)
plan = tp.FitnessPlan(g, bs.registry, bs.measurer, res.placement, 0.01, bs.graph_backend, res.kernel_matches)
i = plan.info
print(name, 'k', plan.k, 'units', i.units, 'edges', i.edges, 'frontier', i.frontier_slots, 'dp', res.device)
for label, fill in (('random', None), ('sparse', 0.1), ('dense', 0.9)):
    rnd = lambda: torch.randint(-(1 << 63), (1 << 63) - 1, (P, plan.words), dtype=torch.int64, device='cuda')
    if fill is None:
        pop = rnd()
    elif fill < 0.5:  # density 1/8: AND of three random words
        pop = rnd() & rnd() & rnd()
    else:  # density 7/8
        pop = rnd() | rnd() | rnd()
    feas = np.zeros(plan.words, np.uint64)  # keep genomes feasible, as an ES population is
    for s_ in range(plan.k):
        if plan.rep_kind[s_] != 0:
            feas[s_ // 64] |= np.uint64(1) << np.uint64(s_ % 64)
    pop &= torch.from_numpy(feas.view(np.int64)).cuda()
    fit = torch.empty(P, dtype=torch.float64, device='cuda')
    out = {}
    for spec in PATHS:
        path, _, pool = spec.partition(':')
        if path.startswith('frontier') and not 0 < i.frontier_slots <= 32 or path == 'wide' and not i.frontier_slots:
            continue
        plan.set_path(path)
        if pool and path == 'anchor':
            plan.set_pool(int(pool))
        for _ in range(2):
            plan.evaluate_device(pop.data_ptr(), P, fit.data_ptr())
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            plan.evaluate_device(pop.data_ptr(), P, fit.data_ptr())
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 3
        out[spec] = (ms, fit.clone())
        print(f'  {label:7s} {spec:9s} {ms:8.2f} ms  {P/ms/1e3:10.3f} Mgenomes/s', flush=True)
    for k in out:
        assert torch.equal(out[k][1], out[PATHS[0]][1]), 'paths disagree'
    plan.set_path('auto')
