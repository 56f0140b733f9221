"""Does evaluating the ES population in lexicographic genome order (lanes of a
warp follow similar paths) speed up the frontier kernel?"""
import sys
sys.path.insert(0, '.')
import torch
import paper_2111_00655_b200 as tp
from paper_2111_00655_b200 import workloads
from paper_2111_00655_b200.es_device import DeviceEvolution
name = sys.argv[1] if len(sys.argv) > 1 else 'bert_base'
g = workloads.CONFIGS[name]()
bs = workloads.paper_backends(g)
res = tp.optimize(g, bs.registry, bs.measurer, 0.01)
plan = tp.FitnessPlan(g, bs.registry, bs.measurer, res.placement, 0.01, bs.graph_backend, res.kernel_matches)
P = 1 << 22
es = DeviceEvolution(plan, P, seed=0)
es.initialize()
def t_eval(pop):
    fit = torch.empty(P, dtype=torch.float64, device='cuda')
    for _ in range(2): plan.evaluate_device(pop.data_ptr(), P, fit.data_ptr())
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3): plan.evaluate_device(pop.data_ptr(), P, fit.data_ptr())
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 3, fit
def lexsort(pop):
    idx = torch.arange(P, device='cuda')
    for w in range(pop.shape[1] - 1, -1, -1):
        key = pop[idx, w] ^ (-(1 << 63))  # unsigned order
        idx = idx[torch.argsort(key, stable=True)]
    return pop[idx].contiguous()
for gen in (0, 5, 25, 100):
    while es.generation < gen:
        es.step()
    pop = es.pop[es.cur].clone()
    t0, f0 = t_eval(pop)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); sp = lexsort(pop); e1.record(); torch.cuda.synchronize()
    ts, f1 = t_eval(sp)
    uniq = torch.unique(pop, dim=0).shape[0]
    print(f'gen {gen:3d}: unsorted {t0:7.2f} ms  sorted {ts:7.2f} ms (sort {e0.elapsed_time(e1):6.2f} ms)  distinct {uniq/P:.3f}  same sum {torch.allclose(f0.sort().values, f1.sort().values)}')
