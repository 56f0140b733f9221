"""Save a config's fitness-plan unit graph to gpurun_out/<config>_units.npz (one GPU)."""
import sys, os
sys.path.insert(0, '.')
import numpy as np
import paper_2111_00655_b200 as tp
from paper_2111_00655_b200 import workloads

os.makedirs('gpurun_out', exist_ok=True)
for name in sys.argv[1:] or ['random100k']:
    g = workloads.CONFIGS[name]()
    bs = workloads.paper_backends(g) if name != 'random100k' else workloads.random_backends(g, 8, 1, 0)
    res = tp.optimize(g, bs.registry, bs.measurer, 0.01, validate=False)
    plan = tp.FitnessPlan(g, bs.registry, bs.measurer, res.placement, 0.01, bs.graph_backend,
                          res.kernel_matches)
    ug = plan.unit_graph()
    np.savez_compressed(f'gpurun_out/{name}_units.npz', **{k: np.asarray(v) for k, v in ug.items()})
    print(name, len(ug['unit_bit']), len(ug['edges']), ug['frontier_needed'])
