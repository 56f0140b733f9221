"""Device-resident evolutionary loop (es_device.DeviceEvolution)."""

import numpy as np
import pytest
import torch

import paper_2111_00655_b200 as tp
from conftest import build_case, golden, kernels_of
from oracle import OracleCase
from paper_2111_00655_b200.es_device import DeviceEvolution

pytestmark = pytest.mark.gpu


def _setup(name="bert_base"):
    case = [c for c in golden("models") if c["name"] == name][0]
    g, reg, meas = build_case(case)
    res = tp.optimize(g, reg, meas, case["epsilon"])
    plan = tp.FitnessPlan(g, reg, meas, res.placement, case["epsilon"],
                          case["es"]["graph_backend"], res.kernel_matches)
    return case, res, plan


@pytest.mark.parametrize("name", ["resnet50", "bert_base"])
def test_device_es_elitism_and_exact_fitness(gpu, name):
    case, res, plan = _setup(name)
    es = DeviceEvolution(plan, 4096, seed=3)
    es.initialize()
    for _ in range(15):
        es.step()
    hist = es.history_values()
    assert len(hist) == 16
    assert np.all(np.diff(hist) <= 0), "best cost must never increase (elitism)"
    assert hist[0] <= plan.seed_cost  # the DP seed is row 0 of generation 0
    # every stored fitness equals the oracle's graph-level cost of its genome
    pop = es.pop[es.cur].cpu().numpy().view(np.uint64)
    fit = es.fit[es.cur].cpu().numpy()
    oc = OracleCase(case)
    oc.price()
    want = oc.fitness(kernels_of(res.placement), case["es"]["graph_backend"], pop[:1024])
    assert np.array_equal(fit[:1024], want)
    best, bits = es.best()
    assert best == hist[-1]
    assert plan.evaluate([bits.tolist()])[0] == best
    # padding bits past the genome length stay clear
    if plan.k % 64:
        assert not np.any(pop[:, -1] >> np.uint64(plan.k % 64))


def test_breed_identity_without_mutation(gpu):
    _, _, plan = _setup("resnet50")
    es = DeviceEvolution(plan, 512, seed=1, mutation_rate=0.0)
    es.initialize()
    row = es.pop[es.cur][5].clone()
    es.pop[es.cur].copy_(row.expand_as(es.pop[es.cur]))
    es.fit[es.cur].fill_(1.0)
    es.elite.copy_(row.view(1, -1))
    es.step()
    assert torch.equal(es.pop[es.cur], row.expand_as(es.pop[es.cur]))


@pytest.mark.parametrize("name", ["resnet50", "bert_base"])
def test_fused_generation_matches_breed_then_fitness(gpu, name):
    """cb_es_generation's fused kernel (breed + packed anchor walk) produces
    the same children, fitness and history as cb_es_breed followed by the
    fitness kernel."""
    _, _, plan = _setup(name)
    assert plan.fused_generation()
    runs = []
    for fused in (True, False):
        es = DeviceEvolution(plan, 3000, seed=5, fused=fused)  # not a multiple of the CTA size
        assert es.fused == fused
        es.initialize()
        for _ in range(6):
            es.step()
        runs.append((es.pop[es.cur].clone(), es.fit[es.cur].clone(), es.history_values()))
    assert torch.equal(runs[0][0], runs[1][0])
    assert torch.equal(runs[0][1], runs[1][1])
    assert np.array_equal(runs[0][2], runs[1][2])
    plan.set_path("frontier")  # another walk: the generation falls back to two launches
    assert not plan.fused_generation()
    plan.set_path("auto")


@pytest.mark.parametrize("name", ["resnet50", "bert_base"])
def test_evolve_device_public_api(gpu, name):
    """evolve_device: DP-seeded device search through the package API; the
    decoded placement prices (host reference pricing) to the reported cost,
    which never exceeds the DP seed and reaches the reference evolve's
    result on these graphs."""
    case, res, plan = _setup(name)
    g, reg, meas = build_case(case)
    res = tp.optimize(g, reg, meas, case["epsilon"])
    out = tp.evolve_device(g, reg, meas, res.placement, case["epsilon"], population=8192,
                           generations=30, graph_backend=case["es"]["graph_backend"],
                           kernel_matches=res.kernel_matches)
    assert out.cost_ms <= out.seed_cost_ms
    assert out.cost_ms == tp.placement_cost_graphlevel(meas, g, out.placement, case["epsilon"],
                                                       reg.graph_backend_ids())
    assert [c for _, c in out.history] == sorted((c for _, c in out.history), reverse=True)
    assert out.genome_length == plan.k and out.evaluations == 8192 * 31


def test_elite_pick_kernel_follows_the_host_rule(gpu):
    """cb_elite_pick over gathered records: lowest fitness, first rank on
    ties, row copied, value (and history slot) written."""
    import ctypes

    import numpy as np
    import torch

    from paper_2111_00655_b200 import _native as nat
    from paper_2111_00655_b200.es_device import pick_elite_host
    rng = np.random.default_rng(0)
    for world, W in ((2, 1), (3, 5), (8, 1554)):
        fits = rng.choice([3.0, 1.5, 1.5, np.inf, 7.25], size=world)
        recs = np.empty((world, 1 + W), np.int64)
        recs[:, 0] = fits.view(np.int64)
        recs[:, 1:] = rng.integers(-(1 << 62), 1 << 62, size=(world, W))
        d = torch.from_numpy(recs).cuda()
        elite = torch.zeros(W, dtype=torch.int64, device="cuda")
        val = torch.zeros(1, dtype=torch.float64, device="cuda")
        hist = torch.zeros(1, dtype=torch.float64, device="cuda")
        nat.check(nat.lib().cb_elite_pick(ctypes.c_void_p(d.data_ptr()), world, W,
                                          ctypes.c_void_p(elite.data_ptr()),
                                          ctypes.c_void_p(val.data_ptr()),
                                          ctypes.c_void_p(hist.data_ptr()), ctypes.c_void_p(0)))
        best, want = pick_elite_host(recs)
        assert val.item() == want == hist.item()
        assert np.array_equal(elite.cpu().numpy(), recs[best, 1:])


@pytest.mark.parametrize("name", ["resnet50", "bert_base"])
def test_host_pipeline_chunks_match_one_launch(gpu, name):
    """cb_fitness_host over many chunks (two alternating compute streams,
    overlapped copies) returns exactly what one device launch returns, and
    the oracle agrees on a sample."""
    case, res, plan = _setup(name)
    n = 148 * 512 * 3 + 777  # > 3 chunks and a ragged tail
    rng = np.random.default_rng(3)
    feasible = np.array([k != 0 for k in plan.rep_kind], dtype=np.uint8)
    bits = (rng.random((n, plan.k)) < 0.5).astype(np.uint8)
    bits[: n // 2] &= feasible
    packed = np.packbits(bits, axis=1, bitorder="little")
    rows = np.zeros((n, plan.words * 8), np.uint8)
    rows[:, :packed.shape[1]] = packed
    rows = rows.view(np.uint64)
    host_rows = torch.empty((n, plan.words), dtype=torch.int64, pin_memory=True)
    host_rows.numpy().view(np.uint64)[:] = rows
    out = torch.empty(n, dtype=torch.float64, pin_memory=True).numpy()
    plan.evaluate_packed(host_rows.numpy().view(np.uint64), out)
    dev_rows = host_rows.cuda()
    dev_fit = torch.empty(n, dtype=torch.float64, device="cuda")
    plan.evaluate_device(dev_rows.data_ptr(), n, dev_fit.data_ptr())
    torch.cuda.synchronize()
    assert np.array_equal(out, dev_fit.cpu().numpy())
    oc = OracleCase(case)
    oc.price()
    sample = rng.choice(n, 256, replace=False)
    want = oc.fitness(kernels_of(res.placement), case["es"]["graph_backend"], bits[sample])
    assert np.array_equal(out[sample], want)
