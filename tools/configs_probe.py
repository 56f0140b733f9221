"""Per-config timings of the whole search on one GPU: graph build, device
matching, pricing, DP, fitness plan, and device ES generations."""
import sys, time, json
sys.path.insert(0, '.')
import torch
import paper_2111_00655_b200 as tp
from paper_2111_00655_b200 import workloads
from paper_2111_00655_b200.cost import price_matches
from paper_2111_00655_b200.es_device import DeviceEvolution

configs = sys.argv[1:] or ['resnet50', 'bert_base', 'nasnet_a', 'nasrnn', 'random100k']
pops = {'resnet50': 1 << 20, 'bert_base': 1 << 20, 'nasnet_a': 1 << 18, 'nasrnn': 65536,
        'random100k': 1 << 20}
for name in configs:
    out = {'config': name}
    t0 = time.perf_counter()
    g = workloads.CONFIGS[name]()
    out['graph_s'] = time.perf_counter() - t0
    t0 = time.perf_counter()
    bs = workloads.paper_backends(g) if name != 'random100k' else workloads.random_backends(g, 8, 1, 0)
    out['registry_s'] = time.perf_counter() - t0
    for rep in range(2):
        bs.registry._tables.clear()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        table = bs.registry.match_table(g)
        t1 = time.perf_counter()
        price_matches(bs.measurer, bs.registry, table)
        t2 = time.perf_counter()
        res = tp.optimize(g, bs.registry, bs.measurer, 0.01, validate=False)
        t3 = time.perf_counter()
        plan = tp.FitnessPlan(g, bs.registry, bs.measurer, res.placement, 0.01, bs.graph_backend,
                              res.kernel_matches)
        t4 = time.perf_counter()
    out.update(nodes=len(g.nodes), matches=int(table.n_matches), match_s=t1 - t0,
               price_s=t2 - t1, optimize_s=t3 - t2, dp_device_ms=res.device['device_ms'],
               dp_levels=res.device['levels'], dp_launches=res.device['launches'],
               ties=res.device['ties'], window_safe=res.device['rounding_window_safe'],
               kernels=len(res.placement), dp_cost=res.cost_ms, plan_s=t4 - t3, k=plan.k,
               units=plan.info.units, edges=plan.info.edges, frontier=plan.info.frontier_slots,
               smem_path=plan.info.smem_path)
    P = pops[name]
    es = DeviceEvolution(plan, P, seed=0)
    es.initialize()
    for _ in range(2):
        es.step()
    torch.cuda.synchronize()
    es.enable_kernel_timing(True)
    t0 = time.perf_counter()
    for _ in range(5):
        es.step()
    torch.cuda.synchronize()
    kt = es.kernel_times_ms()
    out.update(population=P, gen_s=(time.perf_counter() - t0) / 5,
               fitness_ms=sum(kt['fitness']) / 5, breed_ms=sum(kt['breed']) / 5,
               evals_per_s=P / (sum(kt['fitness']) / 5 / 1e3), best=float(es.history_values().min()))
    print(json.dumps(out), flush=True)
