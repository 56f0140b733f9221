"""Population-scale graph-level search that stays on the GPU, optionally
sharded over the GPUs of one node.

Each rank owns a population shard of packed genomes (uint64 rows, same bit
layout as the reference's genome).  A generation is: the rank's best row
(device argmin) -> all-gather of every rank's best fitness and genome over
NCCL (NVLink) -> the global best becomes row 0 of every rank's next shard
(elitism, as in tensorplace/evolution.py:237-240) -> tournament selection,
two-point crossover and mutation of the remaining rows from the rank's own
shard (cb_es_breed) -> batched fitness of the new shard (cb_fitness_device).
No host synchronisation happens inside a generation; the per-generation best
cost is recorded in a device tensor.

Selection uses a counter-based generator (Philox) instead of Python's
Mersenne Twister, so runs are reproducible per (seed, rank) but do not
replay `evolution.evolve` draw for draw -- use `evolve` for that.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native as nat
from .evolution import FitnessPlan


def _torch():
    import torch
    return torch


def gather_records(record, group, out) -> None:
    """All-gather every rank's elite record ([fitness bits, genome row],
    int64, shape (1, 1 + W)) into `out` (world, 1 + W): the search's only
    collective, one call per generation.  NCCL uses the in-place tensor
    collective; other backends (gloo in the CPU tests) the list form."""
    import torch.distributed as dist
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(out, record, group=group)
    else:
        dist.all_gather(list(out.unbind(0)), record.view(-1), group=group)


def pick_elite_host(records: np.ndarray) -> tuple[int, float]:
    """The rule cb_elite_pick applies on the device, restated for host-side
    checks: the lowest fitness, first rank on ties."""
    fit = records[:, 0].astype(np.int64).view(np.float64)
    best = int(np.argmin(fit))  # first occurrence of the minimum
    return best, float(fit[best])


class DeviceEvolution:
    def __init__(self, plan: FitnessPlan, population: int, seed: int = 0, tournament: int = 4,
                 mutation_rate: float | None = None, device=None, process_group=None,
                 history_capacity: int = 4096, fused: bool = False):
        torch = _torch()
        if population < 2:
            raise ValueError("population must be at least 2")
        self.plan = plan
        self.P = int(population)
        self.W = plan.words
        self.k = plan.k
        self.seed = int(seed)
        self.tournament = int(tournament)
        self.rate = mutation_rate if mutation_rate is not None else (1.0 / self.k if self.k else 0.0)
        self.device = torch.device(device or "cuda")
        self.group = process_group
        if process_group is not None:
            import torch.distributed as dist
            self.rank = dist.get_rank(process_group)
            self.world = dist.get_world_size(process_group)
        else:
            self.rank, self.world = 0, 1
        opts = dict(dtype=torch.int64, device=self.device)
        self.pop = [torch.zeros((self.P, self.W), **opts), torch.zeros((self.P, self.W), **opts)]
        self.fit = [torch.empty(self.P, dtype=torch.float64, device=self.device) for _ in range(2)]
        self.cur = 0
        self.best_idx = torch.zeros(1, dtype=torch.int64, device=self.device)
        self.best_val = torch.zeros(1, dtype=torch.float64, device=self.device)
        self.elite_val = torch.full((1,), float("inf"), dtype=torch.float64, device=self.device)
        self.elite = torch.zeros((1, self.W), **opts)
        self.record = torch.zeros((1, 1 + self.W), **opts)
        self.gather_recs = torch.empty((self.world, 1 + self.W), **opts)
        self.history = torch.full((history_capacity,), float("inf"), dtype=torch.float64,
                                  device=self.device)
        self.generation = 0
        # fused=True: one breed + fitness kernel per generation when the plan
        # allows it (cb_es_generation).  Off by default: on B200 the separate
        # launches measured faster (BERT 27.4 vs 28.8 ms per 16.7 M genomes)
        # -- the walk is issue bound and the in-kernel breed adds to its issue
        # load more than it hides of the breed's memory latency.
        self.fused = bool(fused) and plan.fused_generation()
        # kernels of libcollage_b200.so per generation: fitness min/max and the
        # tournament order keys, (fused | breed + fitness), the two CUB argmin
        # kernels and their unpack
        # (+ the overflow list kernel when the anchor walk prices the plan);
        # torch's index_select / copies of the elite row are not counted
        self.launches_per_generation = self.launches_for(plan, self.fused)

    @staticmethod
    def launches_for(plan: FitnessPlan, fused: bool = False) -> int:
        """Kernels of libcollage_b200.so per generation: fitness min/max and the
        tournament order keys, (fused | breed + fitness), the two CUB argmin
        kernels and their unpack; torch's copies of the elite row are not counted."""
        return 6 if fused else 7

    # -- helpers -----------------------------------------------------------------------
    def _stream(self) -> int:
        return _torch().cuda.current_stream(self.device).cuda_stream

    @staticmethod
    def _ptr(t) -> ctypes.c_void_p:
        return ctypes.c_void_p(t.data_ptr())

    def initialize(self) -> None:
        """Row 0 of rank 0 is the all-zero genome (the DP placement itself);
        every other row is uniformly random."""
        with _torch().cuda.device(self.device):  # native launches use the current device
            self._initialize()

    def _initialize(self) -> None:
        torch = _torch()
        gen = torch.Generator(device=self.device)
        gen.manual_seed(self.seed * 1_000_003 + self.rank)
        words = torch.randint(-(1 << 62), 1 << 62, (self.P, self.W), generator=gen,
                              dtype=torch.int64, device=self.device)
        words ^= torch.randint(0, 4, (self.P, self.W), generator=gen, dtype=torch.int64,
                               device=self.device) << 62
        if self.k % 64:  # bits past the genome length stay clear
            words[:, -1] &= (1 << (self.k % 64)) - 1
        elif self.k == 0:
            words.zero_()
        self.pop[self.cur].copy_(words)
        if self.rank == 0:
            self.pop[self.cur][0].zero_()
        self._evaluate(self.cur)
        self._record_best()

    def _evaluate(self, which: int, stream: int | None = None) -> None:
        self.plan.evaluate_device(self.pop[which].data_ptr(), self.P, self.fit[which].data_ptr(),
                                  self._stream() if stream is None else stream)

    def _ptrs(self):
        # device pointers of the fixed buffers, as ctypes values (built once;
        # the tensors are never reallocated)
        p = getattr(self, "_ptr_cache", None)
        if p is None:
            p = self._ptr_cache = {
                "pop": [self._ptr(t) for t in self.pop], "fit": [self._ptr(t) for t in self.fit],
                "elite": self._ptr(self.elite), "best_idx": self._ptr(self.best_idx),
                "best_val": self._ptr(self.best_val), "history": self.history.data_ptr(),
                "hist_stride": self.history.element_size()}
        return p

    def _record_best(self, stream: int | None = None) -> None:
        if self.world == 1:
            # argmin, elite row and history entry in one native call
            p = self._ptrs()
            hist = (ctypes.c_void_p(p["history"] + self.generation * p["hist_stride"])
                    if self.generation < self.history.numel() else ctypes.c_void_p())
            nat.check(nat.lib().cb_argmin_elite(
                p["fit"][self.cur], self.P, p["pop"][self.cur], self.W, p["best_idx"],
                p["best_val"], p["elite"], hist,
                ctypes.c_void_p(self._stream() if stream is None else stream)))
            self.elite_val = self.best_val
            return
        # N > 1: one record per rank, one all-gather, the pick on the device
        p = self._ptrs()
        stream = self._stream() if stream is None else stream
        timing = getattr(self, "timing", False)
        if timing:
            torch = _torch()
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
            ev[0].record()
        nat.check(nat.lib().cb_elite_record(
            p["fit"][self.cur], self.P, p["pop"][self.cur], self.W, p["best_idx"], p["best_val"],
            self._ptr(self.record), ctypes.c_void_p(stream)))
        gather_records(self.record, self.group, self.gather_recs)
        hist = (ctypes.c_void_p(p["history"] + self.generation * p["hist_stride"])
                if self.generation < self.history.numel() else ctypes.c_void_p())
        nat.check(nat.lib().cb_elite_pick(
            self._ptr(self.gather_recs), self.world, self.W, p["elite"],
            self._ptr(self.elite_val), hist, ctypes.c_void_p(stream)))
        if timing:
            ev[1].record()
            self.exchange_events.append(tuple(ev))

    def enable_kernel_timing(self, on: bool = True) -> None:
        """Record CUDA events around the breed and fitness launches of every
        step (on the launching stream) for per-kernel durations."""
        self.timing = on
        self.kernel_events: list[tuple] = []
        self.exchange_events: list[tuple] = []

    def kernel_times_ms(self) -> dict[str, list[float]]:
        """Per-step device times: 'generation' (breed + fitness), and for the
        unfused path its 'breed' and 'fitness' parts."""
        torch = _torch()
        torch.cuda.synchronize(self.device)
        out = {"generation": [], "breed": [], "fitness": [],
               "exchange": [a.elapsed_time(b) for a, b in getattr(self, "exchange_events", [])]}
        for ev in self.kernel_events:
            out["generation"].append(ev[0].elapsed_time(ev[-1]))
            if len(ev) == 3:
                out["breed"].append(ev[0].elapsed_time(ev[1]))
                out["fitness"].append(ev[1].elapsed_time(ev[2]))
        return out

    def step(self) -> None:
        """One generation (no host synchronisation)."""
        with _torch().cuda.device(self.device):  # native launches use the current device
            self._step()

    def _step(self) -> None:
        self.generation += 1
        nxt = 1 - self.cur
        timing = getattr(self, "timing", False)
        if timing:
            torch = _torch()
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 if self.fused else 3)]
            ev[0].record()
        p = self._ptrs()
        stream = self._stream()
        args = (self.plan.handle.raw, p["pop"][self.cur], p["fit"][self.cur], self.P)
        rng = (ctypes.c_uint64(self.seed), ctypes.c_uint64(self.generation),
               ctypes.c_uint64(self.rank), self.tournament, float(self.rate),
               ctypes.c_void_p(stream))
        if self.fused:
            nat.check(nat.lib().cb_es_generation(*args, p["pop"][nxt], p["fit"][nxt], self.P,
                                                 p["elite"], 1, *rng))
            self.cur = nxt
        else:
            nat.check(nat.lib().cb_es_breed(*args, p["pop"][nxt], self.P, p["elite"], 1, *rng))
            if timing:
                ev[1].record()
            self.cur = nxt
            self._evaluate(self.cur, stream)
        if timing:
            ev[-1].record()
            self.kernel_events.append(tuple(ev))
        self._record_best(stream)

    def best(self) -> tuple[float, np.ndarray]:
        """(cost, genome bits) of the global best; synchronises."""
        bits = self.elite[0].cpu().numpy().view(np.uint8)
        unpacked = np.unpackbits(bits, bitorder="little")[:self.k]
        # the elite's own fitness (the history stops at its capacity)
        return float(self.elite_val.item()), unpacked

    def history_values(self) -> np.ndarray:
        return self.history[:min(self.generation + 1, self.history.numel())].cpu().numpy()


def evolve_device(g, registry, measurer, dp_placement, epsilon: float, population: int = 65536,
                  generations: int = 50, seed: int = 0, graph_backend: str | None = None,
                  kernel_matches=None, tournament: int = 4, mutation_rate: float | None = None,
                  device=None, process_group=None):
    """Population-scale graph-level search on the GPU (the device counterpart
    of `evolve`, tensorplace/evolution.py:195-250): the DP placement seeds
    row 0, every generation breeds and prices the whole population on the
    device (one shard per rank when `process_group` spans several GPUs, with
    an all-gather of the rank elites), and the best genome is decoded back
    into a placement.  Returns an `ESResult`; `evaluations` counts every
    priced genome (no fitness cache, unlike `evolve`)."""
    from .evolution import ESResult, FitnessPlan, resolve_graph_backend
    target = resolve_graph_backend(registry, graph_backend)
    plan = FitnessPlan(g, registry, measurer, dp_placement, epsilon, target, kernel_matches)
    seed_cost = plan.seed_cost
    if plan.k == 0:
        return ESResult(dp_placement, seed_cost, seed_cost, (), 0, 0)
    es = DeviceEvolution(plan, population, seed=seed, tournament=tournament,
                         mutation_rate=mutation_rate, device=device, process_group=process_group,
                         history_capacity=max(generations + 1, 1))
    es.initialize()
    for _ in range(generations):
        es.step()
    best, bits = es.best()
    placement = plan.decode(bits.tolist(), dp_placement)
    assert placement is not None  # the elite never regresses below the feasible seed
    hist = es.history_values()
    history = tuple((i, float(v)) for i, v in enumerate(hist))
    return ESResult(placement, best, seed_cost, history, population * (generations + 1), plan.k)
