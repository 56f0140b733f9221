"""Benchmark of the placement-search hot path (BASELINE.json metric:
placement-search wall time and fitness evals/sec).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl mine|reference]
    python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N

Workload (N=1, BASELINE.json configs[1]): BERT-base (seq 128) inference
graph, paper backend set (cuDNN / cuBLAS / TVM with rule-generated patterns
/ TensorRT as the graph inference library), op-level DP then evolutionary
search.  A step is one ES generation of the rank's population shard on the
GPU: tournament selection + two-point crossover + mutation (cb_es_breed)
and batched graph-level fitness of every genome (cb_fitness_device), plus
for N>1 the NCCL all-gather of the per-rank elites.  `value` is genomes
evaluated per second over all ranks (weak scaling: the shard per GPU is
fixed).  The shard is sized so the population exceeds L2 (inputs larger
than L2; no flush).  `e2e` prices a host-resident population through the
public API (FitnessPlan.evaluate_packed -> cb_fitness_host: pinned H2D,
fitness, D2H).  `search` reports the wall time of one full placement search
(match + price + DP + plan + ES generations).

--impl reference times the reference algorithm (the CPU oracle restating
tensorplace, oracle/oracle.c) on the host cores for the same workload.
"""

from __future__ import annotations

import argparse
import gc
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
# the CPU oracle's OpenMP threads sleep when idle instead of spinning next to
# host-side timings (set before libgomp loads)
os.environ.setdefault("OMP_WAIT_POLICY", "PASSIVE")

L2_BYTES = 126 * 1024 * 1024


def _peaks() -> tuple[float, str]:
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled while the timed region runs."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples: list[list[str]] = []
        self._stop = threading.Event()
        self._thread = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._thread.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._thread.join(timeout=10)

    def summary(self) -> dict:
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > i + 2 and s[i + 2].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


def build_workload(name: str):
    import paper_2111_00655_b200 as tp
    from paper_2111_00655_b200 import workloads
    g = workloads.CONFIGS[name]()
    from paper_2111_00655_b200 import _native
    bs = workloads.paper_backends(g, verify=_native.device_available()) if name != "random100k" else \
        workloads.random_backends(g, n_backends=8, n_graph=1, seed=0)
    return tp, g, bs


def shard_size(words: int, requested: int | None) -> int:
    if requested:
        return requested
    p = 1 << 20
    while p * words * 8 < 2 * L2_BYTES:
        p <<= 1
    return p


def run_mine(args) -> None:
    import numpy as np
    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # one GPU per rank; CB_BENCH_DIST_BACKEND=gloo (test only) lets several
    # ranks share the GPUs of a smaller box to exercise the N > 1 code path
    backend = os.environ.get("CB_BENCH_DIST_BACKEND", "nccl")
    local = local % max(torch.cuda.device_count(), 1) if backend != "nccl" else local
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    group = None
    if world > 1:
        import torch.distributed as dist
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
        group = dist.group.WORLD

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
        torch.cuda.synchronize(dev)

    from paper_2111_00655_b200.es_device import DeviceEvolution

    tp, g, bs = build_workload(args.workload)

    def search(P: int, gens: int, timed: bool):
        t = {}
        t0 = time.perf_counter()
        res = tp.optimize(g, bs.registry, bs.measurer, 0.01)
        t["dp_s"] = time.perf_counter() - t0
        plan = tp.FitnessPlan(g, bs.registry, bs.measurer, res.placement, 0.01, bs.graph_backend,
                              res.kernel_matches)
        es = DeviceEvolution(plan, P, seed=args.seed, device=dev, process_group=group)
        es.initialize()
        for _ in range(gens):
            es.step()
        torch.cuda.synchronize(dev)
        t["total_s"] = time.perf_counter() - t0
        t["es_s"] = t["total_s"] - t["dp_s"]
        return res, plan, es, t

    # warm search (module load, first launches), then the timed one on fresh objects
    bs.registry._tables.clear()
    search(4096, 2, False)
    bs.registry._tables.clear()
    res, plan, es0, search_t = search(args.search_population, args.search_generations, True)
    P = shard_size(plan.words, args.population)
    es = DeviceEvolution(plan, P, seed=args.seed, device=dev, process_group=group)
    es.initialize()
    for _ in range(args.warmup):
        es.step()
    barrier()
    es.enable_kernel_timing(True)
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        barrier()
        t_start.record()
        for _ in range(args.steps):
            es.step()
        t_end.record()
        barrier()
    ms = t_start.elapsed_time(t_end)
    kt = es.kernel_times_ms()
    mean = lambda xs: sum(xs) / len(xs) if xs else 0.0
    gen_ms, fit_ms, breed_ms = mean(kt["generation"]), mean(kt["fitness"]), mean(kt["breed"])
    best_cost, _ = es.best()

    # e2e through the public API with host buffers (pinned)
    rng = np.random.default_rng(rank)
    # the population the timed ES steps produced, now host-resident (pinned)
    host = torch.empty((P, plan.words), dtype=torch.int64, pin_memory=True)
    host.copy_(es.pop[es.cur])
    host_np = host.numpy().view(np.uint64)
    host_fit = torch.empty(P, dtype=torch.float64, pin_memory=True).numpy()
    plan.evaluate_packed(host_np, host_fit)  # warm
    barrier()
    t0 = time.perf_counter()
    for _ in range(args.e2e_steps):
        fit = plan.evaluate_packed(host_np, host_fit)
    e2e_s = time.perf_counter() - t0
    barrier()

    vals = torch.tensor([ms, e2e_s, gen_ms, fit_ms, breed_ms, search_t["total_s"]],
                        dtype=torch.float64, device=dev)
    if world > 1:
        import torch.distributed as dist
        dist.all_reduce(vals, op=dist.ReduceOp.MAX)
    ms, e2e_s, gen_ms, fit_ms, breed_ms, search_s = vals.tolist()
    if rank != 0:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()
        return
    step_ms = ms / args.steps
    evals_per_s = world * P * args.steps / (ms / 1e3)
    if es.fused:
        # fused breed + fitness: child row out, fitness out, two parent rows and
        # 2 x tournament 4-byte order keys gathered, per genome
        per_genome = 8 * plan.words + 8 + 2 * 8 * plan.words + 2 * es.tournament * 4
        dom_ms = gen_ms
    else:
        per_genome = plan.words * 8 + 8  # genome row in, fitness out
        dom_ms = fit_ms
    bytes_per_launch = P * per_genome
    peak, peak_src = _peaks()
    achieved = bytes_per_launch / (dom_ms / 1e3) / 1e9
    kernel_name = plan.generation_kernel_name() if es.fused else plan.kernel_name()
    traffic = None
    inst_per_genome = None
    prof = os.path.join(ROOT, "profiles", "fitness_ncu_summary.json")
    if os.path.exists(prof):
        try:
            with open(prof) as fh:
                d = json.load(fh)
            if d.get("workload") == args.workload and \
                    kernel_name.replace(" ", "") in d.get("kernel", "").replace(" ", ""):
                traffic = d.get("dram_bytes_per_launch_per_genome", 0) * P or None
                inst_per_genome = d.get("warp_instructions_per_genome")
        except (OSError, ValueError, KeyError):
            traffic = None
    sweep = None
    if world == 1 and not args.no_configs:
        sweep = config_sweep(dev)
    cpu = None  # last: its OpenMP pool must not compete with the sweep's host-side timings
    if world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(g, bs, res, plan, args)
    line = {
        "metric": "fitness_evals_per_sec",
        "value": evals_per_s,
        "unit": "genomes/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": step_ms,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "int128",
        "arithmetic": "u64 bit-genomes; exact 128-bit fixed-point cost sums (plan window), f64 region pricing",
        "data": "synthetic (BERT-base graph built op by op; simulated backend cost tables)",
        "config": {"workload": f"{args.workload}: op-level DP + evolutionary search",
                   "nodes": len(g.nodes), "dp_kernels": len(res.placement),
                   "genome_bits": plan.k, "genome_words": plan.words,
                   "population_per_gpu": P, "global_population": P * world,
                   "parallelism": f"population sharded over {world} GPU(s), "
                                  f"{'NCCL' if backend == 'nccl' else backend} all-gather of elites",
                   "l2": "population > L2 (no flush)"},
        "search": {"wall_s": search_s, "dp_s": search_t["dp_s"], "es_s": search_t["es_s"],
                   "es_population_per_gpu": args.search_population,
                   "es_generations": args.search_generations, "dp_cost_ms": res.cost_ms,
                   "best_cost_ms_after_timed_steps": best_cost},
        "kernels_ms": ({"generation_fused": gen_ms} if es.fused else
                       {"generation": gen_ms, "fitness": fit_ms, "breed": breed_ms}),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "kernel": kernel_name,
                     "peak_source": peak_src,
                     "algorithmic_bytes_per_launch": bytes_per_launch,
                     "algorithmic_bytes_per_genome": per_genome},
        "e2e": {"value": world * P * args.e2e_steps / e2e_s, "unit": "genomes/s",
                "h2d_bytes_per_step": P * plan.words * 8, "d2h_bytes_per_step": P * 8},
        "gpu_launches": args.steps * es.launches_per_generation,
        "clocks": clocks.summary(),
    }
    if cpu is not None:
        line["cpu_baseline"] = cpu
    if inst_per_genome:
        # the bound that binds: warp-instruction issue (4 schedulers per SM, one
        # instruction per cycle each), instructions per genome from the ncu capture
        # of the same kernel (profiles/fitness_ncu_summary.json)
        sms = torch.cuda.get_device_properties(dev).multi_processor_count
        mhz = line["clocks"].get("sm_mhz") or 1965.0
        peak_issue = sms * 4 * mhz * 1e6
        achieved_issue = inst_per_genome * P / (dom_ms / 1e3)
        line["issue_roofline"] = {"bound": "issue", "achieved": achieved_issue, "peak": peak_issue,
                                  "unit": "warp instructions/s", "frac": achieved_issue / peak_issue,
                                  "warp_instructions_per_genome": inst_per_genome,
                                  "source": "profiles/fitness_ncu_summary.json"}
    if sweep is not None:
        line["configs"] = sweep
    print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def _oracle_case(g, bs):
    from paper_2111_00655_b200.cost import profile_to_json
    from paper_2111_00655_b200.graph import graph_to_json
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from oracle import OracleCase  # checker / baseline only
    case = {"graph": graph_to_json(g),
            "backends": [[b.id, b.kind.value] for b in bs.registry.backends.values()],
            "patterns": [[bp.backend, bp.text(), bp.source.value] for bp in bs.registry.patterns],
            "profiles": {b: profile_to_json(p) for b, p in bs.measurer.profiles.items()},
            "epsilon": 0.01}
    return OracleCase(json.loads(json.dumps(case)))


def _random_packed(n: int, k: int, seed: int):
    """n random genomes of k bits as packed uint64 rows (padding bits clear)."""
    import numpy as np
    words = max(1, (k + 63) // 64)
    rows = np.random.default_rng(seed).integers(0, 1 << 63, size=(n, words), dtype=np.uint64)
    rows ^= np.random.default_rng(seed + 1).integers(0, 2, size=(n, words), dtype=np.uint64) << np.uint64(63)
    if k % 64:
        rows[:, -1] &= np.uint64((1 << (k % 64)) - 1)
    return rows


def cpu_baseline(g, bs, res, plan, args) -> dict:
    """The reference algorithm restated in C (oracle) on the host cores,
    bounded sample: fitness of `sample` random genomes."""
    import numpy as np
    oc = _oracle_case(g, bs)
    oc.price()
    kernels = [[a.backend_pattern.order, a.root, sorted(a.nodes)] for a in res.placement.assignments]
    threads = os.cpu_count() or 1
    sample = args.cpu_sample
    pop = _random_packed(sample, plan.k, 1)
    oc.fitness(kernels, bs.graph_backend, pop[:64], threads=threads)
    t0 = time.perf_counter()
    oc.fitness(kernels, bs.graph_backend, pop, threads=threads)
    dt = time.perf_counter() - t0
    return {"value": sample / dt, "unit": "genomes/s", "cores": threads, "kind": "port",
            "sample": f"{sample} random packed genomes of the {args.workload} DP placement "
                      f"({plan.k} bits), oracle/oracle.c or_fitness with {threads} OpenMP threads"}


# per-config sweep (BASELINE.json's five configs), one GPU: population for
# the search wall time, generations, population for the fitness rate, CPU
# sample for the oracle rate, and whether the oracle's covered-set DP (the
# reference's algorithm) is run for a parity check
SWEEP = {
    "resnet50": dict(search_pop=65536, gens=50, fit_pop=1 << 22, cpu=200_000, ref_dp=True),
    "bert_base": dict(search_pop=65536, gens=50, fit_pop=1 << 22, cpu=100_000, ref_dp=True),
    "nasnet_a": dict(search_pop=65536, gens=50, fit_pop=1 << 20, cpu=20_000, ref_dp=True),
    "nasrnn": dict(search_pop=65536, gens=50, fit_pop=65536, cpu=50_000, ref_dp=True),
    "random100k": dict(search_pop=65536, gens=10, fit_pop=1 << 20, cpu=200, ref_dp=False),
}


def config_sweep(dev) -> dict:
    """Search wall time, DP time, fitness rate and CPU-oracle rate for each
    BASELINE.json config (supplementary to the headline line)."""
    import numpy as np
    import torch
    from paper_2111_00655_b200.es_device import DeviceEvolution
    out = {}
    for name, cfg in SWEEP.items():
        tp, g, bs = build_workload(name)
        row = {"nodes": len(g.nodes)}
        for rep in range(2):  # first pass warms module loads, launches and allocations
            bs.registry._tables.clear()
            gc.collect()
            torch.cuda.synchronize(dev)
            t0 = time.perf_counter()
            res = tp.optimize(g, bs.registry, bs.measurer, 0.01, validate=False)
            t1 = time.perf_counter()
            plan = tp.FitnessPlan(g, bs.registry, bs.measurer, res.placement, 0.01, bs.graph_backend,
                                  res.kernel_matches)
            es = DeviceEvolution(plan, cfg["search_pop"], seed=0, device=dev)
            es.initialize()
            for _ in range(cfg["gens"] if rep else 2):
                es.step()
            torch.cuda.synchronize(dev)
            t2 = time.perf_counter()
        best, _ = es.best()
        # the matcher and pricing on their own (table cache cleared), host wall with syncs
        from paper_2111_00655_b200.cost import price_matches
        tm, tpr = [], []
        for _ in range(3):  # best of 3 (the first pays buffer allocation)
            bs.registry._tables.clear()
            torch.cuda.synchronize(dev)
            m0 = time.perf_counter()
            table = bs.registry.match_table(g)
            torch.cuda.synchronize(dev)
            m1 = time.perf_counter()
            price_matches(bs.measurer, bs.registry, table)
            torch.cuda.synchronize(dev)
            m2 = time.perf_counter()
            tm.append(m1 - m0)
            tpr.append(m2 - m1)
        row.update(matcher={"anchors": len(g.nodes), "patterns": len(bs.registry.patterns),
                            "matches": int(table.n_matches), "wall_ms": 1e3 * min(tm),
                            "anchors_per_s": len(g.nodes) / min(tm),
                            "note": "host wall incl. download of the match table"},
                   pricing={"matches": int(table.n_matches), "wall_ms": 1e3 * min(tpr)},
                   dp={"nodes": len(g.nodes), "device_ms": res.device["device_ms"],
                       "levels": res.device["levels"], "launches": res.device["launches"],
                       "nodes_per_s": len(g.nodes) / (res.device["device_ms"] / 1e3)})
        row.update(search_wall_s=t2 - t0, dp_s=t1 - t0, dp_device_ms=res.device["device_ms"],
                   es_population=cfg["search_pop"], es_generations=cfg["gens"],
                   dp_kernels=len(res.placement), dp_cost_ms=res.cost_ms, es_best_cost_ms=best,
                   rounding_window_safe=res.device["rounding_window_safe"],
                   genome_bits=plan.k, frontier_slots=plan.info.frontier_slots,
                   window_shift=plan.info.window_shift,
                   fitness_kernel=plan.kernel_name())
        P = cfg["fit_pop"]
        es = DeviceEvolution(plan, P, seed=1, device=dev, fused=False)  # the fitness kernel alone
        es.initialize()
        es.step()
        es.enable_kernel_timing(True)
        gens = 3
        for _ in range(gens):
            es.step()
        torch.cuda.synchronize(dev)
        kt = es.kernel_times_ms()
        fit_ms = sum(kt["fitness"]) / len(kt["fitness"])
        row.update(fitness_population=P, fitness_ms_per_generation=fit_ms,
                   fitness_evals_per_s=P / (fit_ms / 1e3))
        del es
        torch.cuda.empty_cache()
        # CPU oracle (reference algorithm in C), bounded sample, all host threads
        oc = _oracle_case(g, bs)
        oc.price()
        kernels = [[a.backend_pattern.order, a.root, sorted(a.nodes)] for a in res.placement.assignments]
        threads = os.cpu_count() or 1
        pop = np.random.default_rng(3).integers(0, 2, size=(cfg["cpu"], plan.k), dtype=np.uint8)
        t0 = time.perf_counter()
        oc.fitness(kernels, bs.graph_backend, pop, threads=threads)
        row["cpu_oracle_fitness_per_s"] = cfg["cpu"] / (time.perf_counter() - t0)
        row["cpu_threads"] = threads
        if name in ("resnet50", "bert_base"):
            # the reference's own search API, drop-in: tp.evolve with the default
            # ESConfig (population 32, 200 generations; reference draws replayed
            # exactly, each generation priced in one GPU batch)
            t0 = time.perf_counter()
            r2 = tp.optimize(g, bs.registry, bs.measurer, 0.01)
            ev = tp.evolve(g, bs.registry, bs.measurer, r2.placement, 0.01, tp.ESConfig(),
                           graph_backend=bs.graph_backend, kernel_matches=r2.kernel_matches)
            row["evolve_default"] = {"s": time.perf_counter() - t0, "cost_ms": ev.cost_ms,
                                     "evaluations": ev.evaluations,
                                     "note": "optimize + evolve(ESConfig()) through the public API"}
        if cfg["ref_dp"]:
            t0 = time.perf_counter()
            status, cost, ref_kernels = oc.dp(max_states=200_000)
            row["reference_dp"] = {"status": status, "s": time.perf_counter() - t0,
                                   "placement_identical": status == "ok" and ref_kernels == kernels
                                   and cost == res.cost_ms}
        else:
            row["reference_dp"] = {"status": "not run (covered-set state space of a 100k-node graph)"}
        out[name] = row
    return out


def run_reference(args) -> None:
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import numpy as np
    tp, g, bs = build_workload(args.workload)
    oc = _oracle_case(g, bs)
    t0 = time.perf_counter()
    oc.price()
    status, cost, kernels = oc.dp(max_states=2_000_000)
    dp_s = time.perf_counter() - t0
    threads = os.cpu_count() or 1
    k = sum(1 for _, _, _ in kernels) if kernels else 0
    # genome length: kernels not on graph backends
    gb = {b for b, kind in [[b.id, b.kind.value] for b in bs.registry.backends.values()]
          if kind == "graph_inference_library"}
    order_backend = [bp.backend for bp in bs.registry.patterns]
    k = sum(1 for o, _, _ in kernels if order_backend[o] not in gb)
    sample = args.ref_sample
    for _ in range(args.warmup):
        oc.fitness(kernels, bs.graph_backend, _random_packed(256, k, 2), threads=threads)
    times = []
    for step in range(args.steps):
        pop = _random_packed(sample, k, 100 + step)  # packed rows, as the GPU arm reads them
        t0 = time.perf_counter()
        oc.fitness(kernels, bs.graph_backend, pop, threads=threads)
        times.append(time.perf_counter() - t0)
    value = sample * len(times) / sum(times)
    line = {
        "impl": "reference",
        "metric": "fitness_evals_per_sec",
        "value": value,
        "unit": "genomes/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": 1e3 * sum(times) / len(times),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "arithmetic": "f64 with exact sums (Kulisch accumulator, fsum-equivalent rounding), CPU",
        "data": "synthetic (BERT-base graph; simulated backend cost tables)",
        "config": {"workload": f"{args.workload}: op-level DP + evolutionary search",
                   "nodes": len(g.nodes), "genome_bits": k, "dp_status": status,
                   "dp_cost_ms": cost, "dp_s": dp_s},
        "cpu_baseline": {"value": value, "unit": "genomes/s", "cores": threads, "kind": "port",
                         "sample": f"{sample} random packed genomes per step, oracle/oracle.c "
                                   f"(reference algorithm restated in C), {threads} threads"},
        "e2e": {"value": value, "unit": "genomes/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=("mine", "reference"), default="mine")
    ap.add_argument("--workload", default="bert_base")
    ap.add_argument("--population", type=int, default=None, help="genomes per GPU")
    ap.add_argument("--search-population", type=int, default=65536)
    ap.add_argument("--search-generations", type=int, default=50)
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--cpu-sample", type=int, default=2_000_000,
                    help="genomes in the CPU-baseline sample (~10 s of CPU work on BERT)")
    ap.add_argument("--ref-sample", type=int, default=400_000,
                    help="genomes per step of the --impl reference arm")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-configs", action="store_true", help="skip the five-config sweep")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_mine(args)


if __name__ == "__main__":
    main()
