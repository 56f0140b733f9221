"""Process-wide interning of op kinds, attribute keys and string values, and
the typed encoding of attribute / literal values shared by the graph and
pattern compilers (tags as in include/collage_b200.h)."""

from __future__ import annotations

import math

TAG_INT = 0
TAG_FLOAT = 1
TAG_STR = 2
TAG_BOOL = 3
TAG_OTHER = 4

_INT64_MIN = -(1 << 63)
_INT64_MAX = (1 << 63) - 1


class Interner:
    def __init__(self):
        self._ids: dict[str, int] = {}

    def __call__(self, text: str) -> int:
        i = self._ids.get(text)
        if i is None:
            i = len(self._ids)
            self._ids[text] = i
        return i

    def get(self, text: str) -> int:
        """Id of `text`, or -1 if never interned (matches nothing)."""
        return self._ids.get(text, -1)

    def __len__(self) -> int:
        return len(self._ids)


OP_KINDS = Interner()
ATTR_KEYS = Interner()
STRINGS = Interner()


def encode_value(value) -> tuple[int, int, float]:
    """(tag, ival, fval) for an attribute value or a pattern literal.

    Equality on the device follows Python `==`: bools equal the ints 0/1,
    ints and floats compare by mathematical value, strings by content, and
    lists never equal a scalar literal.
    """
    if isinstance(value, bool):
        return TAG_BOOL, int(value), float(value)
    if isinstance(value, int):
        if _INT64_MIN <= value <= _INT64_MAX:
            return TAG_INT, value, 0.0
        # outside int64: keep exact equality against floats only
        f = float(value)
        if math.isfinite(f) and int(f) == value:
            return TAG_FLOAT, 0, f
        return TAG_OTHER, 0, 0.0
    if isinstance(value, float):
        return TAG_FLOAT, 0, value
    if isinstance(value, str):
        return TAG_STR, STRINGS(value), 0.0
    return TAG_OTHER, 0, 0.0
