"""Walk applications as the engine consumes them (reswalk apps.py:17-59).

The per-step weight rules themselves live in the CUDA kernel
(csrc/fw_walk.cu ``elem_weight``, following _kernels.py:280-308): DeepWalk
and PPR use the edge weight (or 1), Node2Vec multiplies it by 1/a when the
neighbour is the previous vertex, 1 when it is also a neighbour of the
previous vertex and 1/b otherwise (first step first-order), MetaPath keeps
only edges labelled ``schema[step]``.  A query's start vertex is held in the
pool, not in its result row; ``length`` bounds the sampled vertices.
"""

from dataclasses import dataclass

from .errors import ValidationError

APPS = ("deepwalk", "ppr", "node2vec", "metapath")
APP_IDS = {name: i for i, name in enumerate(APPS)}  # apps.py:21-24


@dataclass
class WalkQuery:
    """Per-query walk state (apps.py:27-35); the GPU keeps it in registers."""

    query_id: int
    cur: int
    prev: int | None = None
    emitted: int = 0
    result_base: int = 0


@dataclass
class AppConfig:
    app: str = "deepwalk"
    length: int = 80                 # max sampled vertices per query
    stop_prob: float = 0.2           # ppr only
    a: float = 2.0                   # node2vec return parameter
    b: float = 0.5                   # node2vec in-out parameter
    schema: tuple = (0, 1, 2, 3, 4)  # metapath edge labels
    weighted: bool = True

    def validate(self):
        """Same rules and messages as apps.py:48-59."""
        if self.app not in APPS:
            raise ValidationError(f"unknown app {self.app!r}")
        if self.length < 1:
            raise ValidationError("walk length must be >= 1")
        if self.app == "ppr" and not 0.0 <= self.stop_prob <= 1.0:
            raise ValidationError("stop_prob must be in [0, 1]")
        if self.app == "node2vec" and (self.a <= 0 or self.b <= 0):
            raise ValidationError("node2vec parameters a, b must be positive")
        if self.app == "metapath" and len(self.schema) == 0:
            raise ValidationError("metapath needs a non-empty schema")
        return self
