"""Fitness time of a device ES population (as the bench sweep measures it)."""
import sys
sys.path.insert(0, '.')
import torch
import paper_2111_00655_b200 as tp
from paper_2111_00655_b200 import workloads
from paper_2111_00655_b200.es_device import DeviceEvolution
name = sys.argv[1] if len(sys.argv) > 1 else 'random100k'
P = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 20
g = workloads.CONFIGS[name]()
bs = workloads.paper_backends(g) if name != 'random100k' else workloads.random_backends(g, 8, 1, 0)
res = tp.optimize(g, bs.registry, bs.measurer, 0.01, validate=False)
plan = tp.FitnessPlan(g, bs.registry, bs.measurer, res.placement, 0.01, bs.graph_backend, res.kernel_matches)
import os
if os.environ.get('CB_PATH'):
    plan.set_path(os.environ['CB_PATH'])
if os.environ.get('CB_POOL'):
    plan.set_pool(int(os.environ['CB_POOL']))
es = DeviceEvolution(plan, P, seed=1, fused=False)
es.initialize()
es.step()
es.enable_kernel_timing(True)
for _ in range(3):
    es.step()
kt = es.kernel_times_ms()
f = sum(kt['fitness']) / 3
dens = (es.pop[es.cur][:256].contiguous().view(torch.uint8).unsqueeze(-1).bitwise_and(torch.tensor([1 << i for i in range(8)], dtype=torch.uint8, device='cuda')) != 0).float().mean().item()
print(name, plan.kernel_name(), f"fitness {f:.2f} ms  {P / f / 1e3:.3f} M/s  density {dens:.3f}")
