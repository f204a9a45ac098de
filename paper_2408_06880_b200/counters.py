"""Logical work counters (same fields and update rules as the reference,
``pkg/src/slbm/counters.py:16-34`` and ``sparse.py:284-293``).

They are pure functions of cell counts, phase and step kind, so the engine
updates them on the host and never reads anything back from the device
for them.
"""

from __future__ import annotations

from dataclasses import asdict, dataclass


@dataclass
class Counters:
    steps: int = 0
    cells_visited: int = 0
    cells_visited_interior: int = 0
    cells_visited_frame: int = 0
    pdf_accesses: int = 0
    idx_reads: int = 0
    values_exchanged: int = 0
    messages: int = 0

    def add(self, other) -> None:
        for key, val in asdict(other).items() if isinstance(other, Counters) else vars(other).items():
            setattr(self, key, getattr(self, key) + val)

    def copy(self) -> "Counters":
        return Counters(**asdict(self))

    def as_dict(self) -> dict[str, int]:
        return asdict(self)

    def record_sweep(self, phase: str, cells: int, q: int, table_reads: bool) -> None:
        self.cells_visited += cells
        if phase == "interior":
            self.cells_visited_interior += cells
        elif phase == "frame":
            self.cells_visited_frame += cells
        self.pdf_accesses += 2 * q * cells
        if table_reads:
            self.idx_reads += (q - 1) * cells
