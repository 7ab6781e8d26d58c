"""The counter-based random stream the walk kernel reproduces (host mirror).

Spec: reswalk rng.py:15-41 / _kernels.py:50-66.  The device copy is
csrc/fw_common.cuh; tests pin both to the known-answer table of SURVEY.md
Appendix A.  Replay stream ids: ``replay_sid(qid, step, lane)``
(_kernels.py:8-12), lane 1023 reserved for the PPR stop draw.
"""

import numpy as np

MASK64 = 0xFFFFFFFFFFFFFFFF
GOLDEN = 0x9E3779B97F4A7C15
MIX1 = 0xBF58476D1CE4E5B9
MIX2 = 0x94D049BB133111EB
TAG_REPLAY = 1 << 63
STOP_LANE = 1023
_INV53 = 1.0 / (1 << 53)


def mix64(z):
    z &= MASK64
    z = ((z ^ (z >> 30)) * MIX1) & MASK64
    z = ((z ^ (z >> 27)) * MIX2) & MASK64
    return z ^ (z >> 31)


def stream_base(key, stream_id):
    h = mix64((key & MASK64) + GOLDEN)
    return mix64(h ^ ((stream_id & MASK64) * MIX1 & MASK64))


def value_at(key, stream_id, counter):
    z = mix64((stream_base(key, stream_id) + (counter & MASK64) * GOLDEN) & MASK64)
    return (z >> 11) * _INV53


def replay_sid(qid, step, lane):
    if not (0 <= qid < 1 << 33 and 0 <= step < 1 << 20 and 0 <= lane < 1 << 10):
        raise ValueError("replay stream-id field overflow")
    return TAG_REPLAY | (qid << 30) | (step << 10) | lane


def mix64_np(z):
    """Vectorised mix64 over a uint64 array (wrapping arithmetic)."""
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * np.uint64(MIX1)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(MIX2)
    return z ^ (z >> np.uint64(31))


class RngStream:
    """One logical lane: ``next_uniform`` advances the counter by one."""

    __slots__ = ("key", "stream_id", "counter", "_base")

    def __init__(self, key, stream_id, counter=0):
        self.key = key & MASK64
        self.stream_id = stream_id & MASK64
        self.counter = counter
        self._base = stream_base(key, stream_id)

    def next_uniform(self):
        z = mix64((self._base + (self.counter & MASK64) * GOLDEN) & MASK64)
        self.counter += 1
        return (z >> 11) * _INV53


def make_stream(seed, stream_id):
    return RngStream(seed, stream_id)
