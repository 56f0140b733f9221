"""The README's usage example, run as written (GPU)."""
import sys
sys.path.insert(0, '.')
import paper_2111_00655_b200 as tp          # drop-in for `import tensorplace as tp`
from paper_2111_00655_b200 import workloads

g = workloads.bert_base()                    # or tp.load_graph(...)
bs = workloads.paper_backends(g)             # registry + SimMeasurer (paper backend set)
res = tp.optimize(g, bs.registry, bs.measurer, 0.01)                  # device DP
es = tp.evolve(g, bs.registry, bs.measurer, res.placement, 0.01,     # reference-exact ES
               tp.ESConfig(), graph_backend=bs.graph_backend)
big = tp.evolve_device(g, bs.registry, bs.measurer, res.placement, 0.01,
                       population=1 << 20, generations=50)           # population-scale ES
print(res.cost_ms, es.cost_ms, big.cost_ms, len(big.placement))
