"""Run statistics (the reference's SortStats, stats.py:33-70).

Field meanings on the device:
  comparisons      key-vs-pivot classifications of the partition passes
                   (one three-way classification per live key per level)
  array_writes     element writes into the caller's array
  scratch_writes   element writes into the workspace (ping-pong partner,
                   ==p payload side buffer)
  element_writes   array_writes + scratch_writes; virtual_swaps = /3
  temp_high_water  workspace capacity in elements (the retained buffer)
  max_depth        deepest recursion level reached
  stages           segments partitioned or verified by the level kernels
  state_activations  device analogues of the machine states: partition
                   passes ("partition"), ==p runs retired ("eq_run"),
                   on-chip-sorted segments ("small")
  handler_activations  sorted / reversed verified bypasses and fallbacks
``gpu`` holds the raw device counters (levels, bytes, device ms).
"""

from __future__ import annotations

from dataclasses import dataclass, field


@dataclass
class SortStats:
    comparisons: int = 0
    element_writes: int = 0
    array_writes: int = 0
    scratch_writes: int = 0
    temp_high_water: int = 0
    max_depth: int = 0
    stages: int = 0
    state_activations: dict = field(default_factory=dict)
    handler_activations: dict = field(
        default_factory=lambda: {"sorted": 0, "reversed": 0, "fallbacks": 0})
    gpu: dict = field(default_factory=dict)

    @property
    def virtual_swaps(self) -> float:
        return self.element_writes / 3.0

    def as_dict(self) -> dict:
        return {
            "comparisons": self.comparisons,
            "element_writes": self.element_writes,
            "virtual_swaps": self.virtual_swaps,
            "temp_high_water": self.temp_high_water,
            "max_depth": self.max_depth,
            "stages": self.stages,
            "state_activations": dict(self.state_activations),
            "handler_activations": dict(self.handler_activations),
        }
