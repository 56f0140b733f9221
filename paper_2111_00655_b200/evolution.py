"""Graph-level evolutionary search (API of tensorplace/evolution.py).

`evolve` reproduces the reference run exactly -- same seeded generator, same
sequence of draws for seeding, tournament selection, two-point crossover and
mutation, same fitness cache and elitism -- so histories and results are
identical.  What changes is fitness evaluation: every generation's
not-yet-seen genomes are packed into bit rows and priced in one batched GPU
launch (csrc/fitness.cu) against a plan of the DP placement built once by
the native runtime.  `es_device.DeviceEvolution` runs the whole loop on the
device for population-scale searches (and shards it across GPUs).
"""

from __future__ import annotations

import ctypes
import random
import time
from dataclasses import dataclass
from typing import Sequence

import numpy as np

from . import _native as nat
from .cost import Measurer, price_matches
from .errors import RegistryError
from .graph import ComputationGraph
from .placement import Assignment, PlacementStrategy
from .registry import BackendKind, PatternRegistry

Bits = tuple[int, ...]


@dataclass(frozen=True)
class ESConfig:
    population_size: int = 32
    generations: int = 200
    mutation_rate: float | None = None
    tournament_size: int = 4
    elitism: int = 1
    seed: int = 0
    time_budget_s: float | None = None

    def __post_init__(self):
        if self.population_size < 1 or self.generations < 0:
            raise ValueError("population_size and generations must be positive")
        if self.mutation_rate is not None and not 0.0 <= self.mutation_rate <= 1.0:
            raise ValueError("mutation_rate must be in [0, 1]")
        if self.tournament_size < 1 or self.elitism < 0:
            raise ValueError("tournament_size and elitism must be positive")
        if self.time_budget_s is not None and self.time_budget_s <= 0:
            raise ValueError("time_budget_s must be positive")


@dataclass
class ESResult:
    placement: PlacementStrategy
    cost_ms: float
    seed_cost_ms: float
    history: tuple[tuple[int, float], ...]
    evaluations: int
    genome_length: int


def eligible_slots(registry: PatternRegistry, dp_placement: PlacementStrategy) -> list[int]:
    return [i for i, a in enumerate(dp_placement.assignments)
            if registry.backend(a.backend_pattern.backend).kind
            is not BackendKind.GRAPH_INFERENCE_LIBRARY]


def resolve_graph_backend(registry: PatternRegistry, requested: str | None) -> str:
    ids = registry.graph_backend_ids()
    if requested is not None:
        if requested not in ids:
            raise RegistryError(f"backend '{requested}' is not a registered graph inference "
                                f"library (have: {list(ids)})")
        return requested
    if not ids:
        raise RegistryError("no graph inference library backend is registered")
    if len(ids) > 1:
        raise RegistryError(f"multiple graph inference libraries registered ({list(ids)}); "
                            f"a target must be named")
    return ids[0]


def _replacement(g: ComputationGraph, registry: PatternRegistry, a: Assignment,
                 target: str) -> list[Assignment] | None:
    for bp, m in registry.candidates_at(g, a.root):
        if bp.backend == target and m.nodes.node_ids == a.nodes:
            return [Assignment(a.nodes, bp, a.root)]
    singles = []
    for v in sorted(a.nodes):
        hit = next((bp for bp, m in registry.candidates_at(g, v)
                    if bp.backend == target and m.nodes.node_ids == frozenset((v,))), None)
        if hit is None:
            return None
        singles.append(Assignment(frozenset((v,)), hit, v))
    return singles


def decode_genome(g: ComputationGraph, registry: PatternRegistry,
                  dp_placement: PlacementStrategy, bits: Sequence[int],
                  graph_backend: str) -> PlacementStrategy | None:
    slots = eligible_slots(registry, dp_placement)
    if len(bits) != len(slots):
        raise ValueError(f"genome length {len(bits)} does not match {len(slots)} "
                         f"eligible kernels")
    flipped = {s for s, b in zip(slots, bits) if b}
    out: list[Assignment] = []
    for i, a in enumerate(dp_placement.assignments):
        if i not in flipped:
            out.append(a)
            continue
        rep = _replacement(g, registry, a, graph_backend)
        if rep is None:
            return None
        out.extend(rep)
    return PlacementStrategy(out)


def pack_genomes(genomes: Sequence[Sequence[int]], k: int, words: int) -> np.ndarray:
    """Rows of uint64 words, bit i of a genome at bit i%64 of word i//64."""
    n = len(genomes)
    if n == 0:
        return np.zeros((0, words), dtype=np.uint64)
    bits = np.asarray(genomes, dtype=np.uint8).reshape(n, k) if k else np.zeros((n, 0), np.uint8)
    packed = np.packbits(bits, axis=1, bitorder="little")
    buf = np.zeros((n, words * 8), dtype=np.uint8)
    buf[:, :packed.shape[1]] = packed
    return buf.view(np.uint64)


class FitnessPlan:
    """Device plan of a DP placement: prices offload genomes on the GPU.

    Built by the native runtime (cb_es_plan_create): eligible kernels in
    canonical order, their replacements on the target graph backend, the
    constant part of the cost and the dynamic region graph."""

    def __init__(self, g: ComputationGraph, registry: PatternRegistry, measurer: Measurer,
                 dp_placement: PlacementStrategy, epsilon: float, target: str,
                 kernel_matches: np.ndarray | None = None):
        self.g = g
        self.registry = registry
        self.target = target
        table = registry.match_table(g)
        self.table = table
        price_matches(measurer, registry, table)
        if kernel_matches is None:
            kernel_matches = self._locate(dp_placement)
        self.kernel_matches = nat.i32(kernel_matches)
        backends = list(registry.backends)
        is_graph = nat.u8([registry.backend(b).kind is BackendKind.GRAPH_INFERENCE_LIBRARY
                           for b in backends])
        alpha = np.zeros(len(backends))
        floor = np.ones(len(backends))
        for i, b in enumerate(backends):
            if is_graph[i]:
                alpha[i], floor[i] = measurer.region_params(b)
        raw = ctypes.c_void_p()
        nat.check(nat.lib().cb_es_plan_create(
            g.native, table.handle.raw, len(self.kernel_matches),
            nat.ptr(self.kernel_matches, nat.c_int32), len(backends),
            nat.ptr(is_graph, nat.c_uint8), nat.ptr(nat.f64(alpha), nat.c_double),
            nat.ptr(nat.f64(floor), nat.c_double), backends.index(target), float(epsilon),
            ctypes.byref(raw)))
        self.handle = nat.Handle(raw.value, "cb_es_plan_destroy")
        info = nat.ESPlanInfo()
        nat.check(nat.lib().cb_es_plan_query(self.handle.raw, ctypes.byref(info)))
        self.info = info
        self.k = info.genome_bits
        self.words = info.words
        self.seed_cost = info.seed_cost
        kind = np.empty(max(self.k, 1), np.int8)
        slot_kernel = np.empty(max(self.k, 1), np.int32)
        rep_ptr = np.empty(self.k + 1, np.int32)
        nat.check(nat.lib().cb_es_plan_slots(self.handle.raw, nat.ptr(slot_kernel, nat.c_int32),
                                             nat.ptr(kind, nat.c_int8),
                                             nat.ptr(rep_ptr, nat.c_int32), None))
        rep = np.empty(max(int(rep_ptr[-1]), 1), np.int32)
        nat.check(nat.lib().cb_es_plan_slots(self.handle.raw, None, None, None,
                                             nat.ptr(rep, nat.c_int32)))
        self.rep_kind = kind[:self.k]
        self.rep_ptr = rep_ptr
        self.rep_match = rep
        self.slot_kernel = slot_kernel[:self.k]

    def unit_graph(self) -> dict:
        """The plan's dynamic unit graph: genome bit per unit (-1 = fixed
        target-backend component), kernels per unit, edges (a < b) and the
        frontier width the thread-per-genome program needs."""
        m, e = self.info.units, self.info.edges
        bit = np.empty(max(m, 1), np.int32)
        cnt = np.empty(max(m, 1), np.int32)
        edges = np.empty((max(e, 1), 2), np.int32)
        need = nat.c_int32(0)
        nat.check(nat.lib().cb_es_plan_units(self.handle.raw, nat.ptr(bit, nat.c_int32),
                                             nat.ptr(cnt, nat.c_int32),
                                             nat.ptr(edges, nat.c_int32), ctypes.byref(need)))
        return {"unit_bit": bit[:m], "unit_cnt": cnt[:m], "edges": edges[:e],
                "frontier_needed": int(need.value)}

    def _locate(self, placement: PlacementStrategy) -> np.ndarray:
        """Match-table index of every assignment (same backend, same nodes)."""
        g, table = self.g, self.table
        backends = list(self.registry.backends)
        out = np.empty(len(placement.assignments), dtype=np.int32)
        pat_backend = table.patterns.compiled.backend
        for i, a in enumerate(placement.assignments):
            want = backends.index(a.backend_pattern.backend)
            hit = -1
            for m in table.group(g.index_of(a.root)):
                if int(pat_backend[table.pat[m]]) == want and table.node_set(m) == a.nodes:
                    hit = m
                    if int(table.pat[m]) == a.backend_pattern.order:
                        break
            if hit < 0:
                raise RegistryError(f"kernel {sorted(a.nodes)} on '{a.backend_pattern.backend}' "
                                    f"is not a registered match")
            out[i] = hit
        return out

    def set_path(self, path: str) -> None:
        """'auto' | 'frontier' / 'frontier_smem' (thread per genome, <= 32
        frontier slots; 'packed128': the packed-label walk in the plan's
        128-bit window; 'packed_anchor': the same with anchor labels, <= 8
        slots) | 'anchor' (thread per genome, lockstep, <= 64 slots) |
        'wide'
        (warp per genome, sparse walk, <= 128 slots) | 'unionfind'
        (warp/CTA per genome, any plan).  All give identical results;
        `auto` picks the packed anchor kernel for <= 8 slots, the
        packed-label frontier kernel for <= 16 slots (in the 128-bit window
        when the plan fits one), the
        anchor kernel up to 64, the wide kernel up to 128, else union-find."""
        code = {"auto": -1, "unionfind": 0, "frontier": 1, "frontier_smem": 2, "wide": 3,
                "anchor": 4, "packed128": 5, "packed_anchor": 6, "fsm": 7}[path]
        nat.check(nat.lib().cb_es_plan_set_path(self.handle.raw, code))

    def kernel_name(self) -> str:
        """The fitness kernel evaluate / evaluate_device launch."""
        return nat.lib().cb_es_plan_kernel(self.handle.raw).decode()

    def has_packed128(self) -> bool:
        """Whether the 'packed128' path applies (<= 16 frontier slots and
        every plan value inside a 128-bit window)."""
        return bool(self.info.packed_labels) and self.info.window_shift >= 0

    def fused_generation(self) -> bool:
        """Whether cb_es_generation runs breed + fitness as one kernel."""
        return bool(nat.lib().cb_es_generation_fused(self.handle.raw))

    def generation_kernel_name(self) -> str:
        """The kernel that prices a device ES generation."""
        name = self.kernel_name()
        if self.fused_generation():  # fitness_pa_kernel<F, W> -> fitness_pa_breed_kernel<F, words>
            f = name[name.index('<') + 1:].split(',')[0]
            return f"fitness_pa_breed_kernel<{f}, {self.words}>"
        return name

    def has_fsm(self) -> bool:
        """Whether the 'fsm' path applies (finite-state program built)."""
        return self.info.fsm_transitions > 0

    def has_packed_anchor(self) -> bool:
        """Whether the 'packed_anchor' path applies (<= 8 frontier slots,
        128-bit window)."""
        return self.info.packed_labels == 2 and self.info.window_shift >= 0

    def set_pool(self, entries: int) -> None:
        """Merged-component pool entries per genome of the anchor kernel
        (tuning / testing; results do not depend on it)."""
        nat.check(nat.lib().cb_es_plan_set_pool(self.handle.raw, int(entries)))

    def evaluate(self, genomes: Sequence[Sequence[int]]) -> np.ndarray:
        """Fitness of each genome (host buffers in, host results out)."""
        pop = pack_genomes(genomes, self.k, self.words)
        return self.evaluate_packed(pop)

    def evaluate_packed(self, pop: np.ndarray, out: np.ndarray | None = None) -> np.ndarray:
        """Fitness of packed genome rows held in host memory: chunked H2D /
        kernel / D2H pipeline (fully overlapped when `pop` and `out` are
        pinned, e.g. views of `torch.empty(..., pin_memory=True)`)."""
        pop = np.ascontiguousarray(pop, dtype=np.uint64)
        if out is None:
            out = np.empty(pop.shape[0], dtype=np.float64)
        assert out.dtype == np.float64 and out.flags.c_contiguous and len(out) == pop.shape[0]
        if pop.shape[0]:
            nat.check(nat.lib().cb_fitness_host(self.handle.raw, nat.ptr(pop, nat.c_uint64),
                                                pop.shape[0], nat.ptr(out, nat.c_double)))
        return out

    def evaluate_device(self, d_pop_ptr: int, n: int, d_fit_ptr: int, stream: int = 0) -> None:
        """Fitness of n packed genomes already resident on the device."""
        nat.check(nat.lib().cb_fitness_device(self.handle.raw, ctypes.c_void_p(d_pop_ptr), n,
                                              ctypes.c_void_p(d_fit_ptr),
                                              ctypes.c_void_p(stream)))

    def decode(self, bits: Sequence[int], placement: PlacementStrategy) -> PlacementStrategy | None:
        patterns = self.registry.patterns
        table, g = self.table, self.g
        flipped = {int(self.slot_kernel[s]): s for s, b in enumerate(bits) if b}
        out: list[Assignment] = []
        for i, a in enumerate(placement.assignments):
            s = flipped.get(i)
            if s is None:
                out.append(a)
                continue
            if self.rep_kind[s] == 0:
                return None
            for m in self.rep_match[self.rep_ptr[s]:self.rep_ptr[s + 1]]:
                nodes = table.node_set(int(m))
                out.append(Assignment(nodes, patterns[int(table.pat[m])],
                                      g.id_of(int(table.root[m]))))
        return PlacementStrategy(out)


def evolve(g: ComputationGraph, registry: PatternRegistry, measurer: Measurer,
           dp_placement: PlacementStrategy, epsilon: float, config: ESConfig,
           graph_backend: str | None = None, kernel_matches: np.ndarray | None = None) -> ESResult:
    """Graph-level search seeded with the DP placement; result cost never
    exceeds the seed cost (elitism)."""
    target = resolve_graph_backend(registry, graph_backend)
    plan = FitnessPlan(g, registry, measurer, dp_placement, epsilon, target, kernel_matches)
    slots = eligible_slots(registry, dp_placement)
    k = len(slots)
    assert k == plan.k, "plan and placement disagree on eligible kernels"
    seed_cost = plan.seed_cost
    if k == 0:
        return ESResult(dp_placement, seed_cost, seed_cost, (), 0, 0)

    cache: dict[Bits, float] = {}
    evaluations = 0

    def evaluate(pop: list[Bits]) -> list[float]:
        nonlocal evaluations
        fresh: list[Bits] = []
        seen: set[Bits] = set()
        for bits in pop:
            if bits not in cache and bits not in seen:
                seen.add(bits)
                fresh.append(bits)
        if fresh:
            for bits, val in zip(fresh, plan.evaluate(fresh)):
                cache[bits] = float(val)
            evaluations += len(fresh)
        return [cache[bits] for bits in pop]

    rng = random.Random(config.seed)
    rate = config.mutation_rate if config.mutation_rate is not None else 1.0 / k
    population: list[Bits] = [tuple([0] * k)]
    while len(population) < config.population_size:
        population.append(tuple(rng.randrange(2) for _ in range(k)))

    def pick(fits: list[float]) -> Bits:
        best = rng.randrange(len(population))
        for _ in range(config.tournament_size - 1):
            challenger = rng.randrange(len(population))
            if fits[challenger] < fits[best]:
                best = challenger
        return population[best]

    def cross(a: Bits, b: Bits) -> Bits:
        if k < 2:
            return a
        i, j = sorted((rng.randrange(k + 1), rng.randrange(k + 1)))
        return a[:i] + b[i:j] + a[j:]

    def mutate(bits: Bits) -> Bits:
        return tuple(1 - x if rng.random() < rate else x for x in bits)

    started = time.monotonic()
    fits = evaluate(population)
    best_bits, best_fit = population[0], float("inf")
    for bits, fit in zip(population, fits):
        if fit < best_fit:
            best_bits, best_fit = bits, fit
    history: list[tuple[int, float]] = [(0, best_fit)]
    for gen in range(1, config.generations + 1):
        if config.time_budget_s is not None and time.monotonic() - started > config.time_budget_s:
            break
        ranked = sorted(range(len(population)), key=lambda i: (fits[i], i))
        nxt: list[Bits] = [best_bits]
        nxt.extend(population[i] for i in ranked[:max(0, config.elitism - 1)])
        while len(nxt) < config.population_size:
            nxt.append(mutate(cross(pick(fits), pick(fits))))
        population = nxt[:config.population_size]
        fits = evaluate(population)
        for bits, fit in zip(population, fits):
            if fit < best_fit:
                best_bits, best_fit = bits, fit
        history.append((gen, best_fit))
    placement = plan.decode(best_bits, dp_placement)
    assert placement is not None
    final = evaluate([best_bits])[0]
    return ESResult(placement, final, seed_cost, tuple(history), evaluations, k)
