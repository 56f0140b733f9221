"""bench.py --impl reference: the reference algorithm on the host cores,
fed from the committed case file, must not load the product library and
must print the contract's JSON line (CPU only)."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_line_without_product_library():
    cmd = [sys.executable, "bench.py", "--impl", "reference", "--workload", "random100k",
           "--steps", "1", "--warmup", "3", "--ref-sample", "16"]
    out = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["metric"] == "fitness_evals_per_sec"
    assert d["value"] > 0 and d["e2e"]["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] == "port"
    assert d["config"]["genome_bits"] == 99446 and d["reference_sample"]["dp_cost_ms"] == 22776.0808208
    # the same config dict as the GPU arm prints for this workload and N
    sys.path.insert(0, ROOT)
    import argparse
    import bench
    args = argparse.Namespace(workload="random100k", population=None)
    assert d["config"] == bench.workload_config(args, 1, 100000, 99446, 99446,
                                                bench.shard_size(1554, 1 << 20))
    assert d["product_library_loaded"] is False


def test_breed_follows_the_reference_operators():
    import numpy as np
    sys.path.insert(0, ROOT)
    import bench
    rng = np.random.default_rng(0)
    k, P = 200, 64
    pop = rng.integers(0, 2, size=(P, k), dtype=np.uint8)
    fits = rng.random(P)
    out = bench._breed(np.random.default_rng(1), pop, fits, k)
    assert out.shape == pop.shape
    assert np.array_equal(out[0], pop[int(np.argmin(fits))])  # elitism 1
    # with constant rows, a two-point crossover child is one block of the
    # other parent's value: at most 2 value changes along the genome, plus
    # about one mutation (probability 1/k per bit) adding at most 2 more
    pop = np.repeat(rng.integers(0, 2, size=(P, 1), dtype=np.uint8), k, axis=1)
    out = bench._breed(np.random.default_rng(2), pop, fits, k)
    changes = np.count_nonzero(np.diff(out[1:].astype(np.int8), axis=1), axis=1)
    assert np.median(changes) <= 4 and changes.max() <= 12
    flips = [min(np.count_nonzero(c != 0), np.count_nonzero(c != 1)) for c in out[1:]]
    assert any(0 < f < k for f in flips)  # some children mix both parents
