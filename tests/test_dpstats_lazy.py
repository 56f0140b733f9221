"""DPStats counters of a device pricing pass settle lazily (the reference's
per-candidate cache protocol is replayed only when a counter is read); the
object must still behave like the reference's plain dataclass."""

import copy
import dataclasses
import pickle

from paper_2111_00655_b200.dp import DPStats


def _lazy(calls=4, hits=1, comps=3):
    s = DPStats(nodes=3, pops=3)
    seen = []

    def settle(st):
        seen.append(1)
        st.measure_calls, st.cache_hits, st.computations = calls, hits, comps

    s.__dict__["_settle"] = settle
    return s, seen


def test_counters_settle_once_on_first_read():
    s, seen = _lazy()
    assert s.nodes == 3 and not seen  # other fields do not settle
    assert s.measure_calls == 4 and s.cache_hits == 1 and s.computations == 3
    assert s.measure_calls == s.cache_hits + s.computations
    assert len(seen) == 1


def test_plain_dataclass_behaviour():
    s, _ = _lazy()
    assert set(s.to_json()) == {f.name for f in dataclasses.fields(DPStats)}
    assert dataclasses.asdict(s)["computations"] == 3
    assert pickle.loads(pickle.dumps(s)) == s
    t, _ = _lazy()
    assert copy.deepcopy(t) == s
    assert "measure_calls=4" in repr(_lazy()[0])
