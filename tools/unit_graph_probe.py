"""Unit-graph statistics of each config's fitness plan (one GPU): genome
bits, units, edges, frontier width, static component sizes, degree."""
import sys, json, collections
sys.path.insert(0, '.')
import numpy as np
import paper_2111_00655_b200 as tp
from paper_2111_00655_b200 import workloads

configs = sys.argv[1:] or ['resnet50', 'bert_base', 'nasnet_a', 'nasrnn', 'random100k']
for name in configs:
    g = workloads.CONFIGS[name]()
    bs = workloads.paper_backends(g) if name != 'random100k' else workloads.random_backends(g, 8, 1, 0)
    res = tp.optimize(g, bs.registry, bs.measurer, 0.01, validate=False)
    plan = tp.FitnessPlan(g, bs.registry, bs.measurer, res.placement, 0.01, bs.graph_backend,
                          res.kernel_matches)
    ug = plan.unit_graph()
    m = len(ug['unit_bit'])
    par = list(range(m))
    def find(x):
        while par[x] != x:
            par[x] = par[par[x]]
            x = par[x]
        return x
    deg = np.zeros(m, np.int64)
    for a, b in ug['edges']:
        deg[a] += 1; deg[b] += 1
        ra, rb = find(int(a)), find(int(b))
        if ra != rb: par[max(ra, rb)] = min(ra, rb)
    comp_bits = collections.Counter()
    comp_units = collections.Counter()
    for u in range(m):
        r = find(u)
        comp_units[r] += 1
        if ug['unit_bit'][u] >= 0: comp_bits[r] += 1
    sizes = sorted(comp_bits.values(), reverse=True)
    hist = collections.Counter(min(s, 33) for s in sizes)
    span = [int(b - a) for a, b in ug['edges']]
    print(json.dumps({'config': name, 'k': plan.k, 'units': m, 'fixed': int((ug['unit_bit'] < 0).sum()),
                      'edges': len(ug['edges']), 'frontier_needed': ug['frontier_needed'],
                      'frontier_slots': plan.info.frontier_slots,
                      'components': len(comp_units), 'largest_comp_bits': sizes[:8],
                      'comp_bits_hist': dict(sorted(hist.items())), 'max_deg': int(deg.max()) if m else 0,
                      'mean_deg': float(deg.mean()) if m else 0, 'max_span': max(span) if span else 0,
                      'max_cnt': int(ug['unit_cnt'].max()) if m else 0}), flush=True)
