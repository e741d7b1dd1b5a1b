"""Shift sequences (``/root/reference/pkg/src/sylvadi/shifts.py:31-67``).

Shift generation itself (Ritz values + greedy heuristic) is outside the hot
path; shifts are pinned in JSON files in the reference's
own layout and read back here, so every run shares bit-identical shifts.
"""

import json
from dataclasses import dataclass


@dataclass
class ShiftSequence:
    pairs: list
    cyclic: bool = True

    def __post_init__(self):
        self.pairs = [(complex(a), complex(b)) for a, b in self.pairs]
        if not self.pairs:
            raise ValueError("shift sequence must not be empty")

    def __len__(self):
        return len(self.pairs)

    def at(self, k):
        """(alpha_k, beta_k) for 1-based outer step k, reused cyclically."""
        i = k - 1
        if i >= len(self.pairs):
            if not self.cyclic:
                raise IndexError("shift sequence exhausted")
            i %= len(self.pairs)
        return self.pairs[i]

    def to_json(self, path):
        with open(path, "w") as fh:
            json.dump({"cyclic": self.cyclic,
                       "pairs": [[[a.real, a.imag], [b.real, b.imag]] for a, b in self.pairs]},
                      fh, indent=1)

    @classmethod
    def from_json(cls, path):
        with open(path) as fh:
            payload = json.load(fh)
        return cls(pairs=[(complex(*a), complex(*b)) for a, b in payload["pairs"]],
                   cyclic=bool(payload.get("cyclic", True)))
