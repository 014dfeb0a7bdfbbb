"""Stage-level trace events of the sort (the trace half of the reference's
instrument.py:74-104, the part the sort path emits into).

``Sorter.trace`` takes any object with ``emit(kind, *payload)`` -- the
reference's own ``TraceSink`` works unchanged; this module provides an
equivalent sink and the event kinds.  The device recursion reports one
record per stage after every level (tsq_stage_record, include/tsq.h), and
the host turns them into the reference's event sequence:
``StateEnter("prescan", a, b)`` or ``HandlerEnter("sorted"|"reversed", a, b)``
[+ ``HandlerFallback``], then ``StageEnd(a, b, new_l, new_r)``, and a final
``StageEnd(0, n - 1, "root")`` (core.py:1676-1711, 1610-1611).  Per-element
``Compare`` / ``Write`` events have no device equivalent (a partition pass
moves every key of a level at once) and are not emitted.
"""

from __future__ import annotations

from dataclasses import dataclass

COMPARE = "Compare"
WRITE = "Write"
STATE_ENTER = "StateEnter"
STAGE_END = "StageEnd"
HANDLER_ENTER = "HandlerEnter"
HANDLER_FALLBACK = "HandlerFallback"


@dataclass(frozen=True)
class TraceEvent:
    kind: str
    payload: tuple

    def line(self) -> str:
        return f"{self.kind}\t" + "\t".join(str(p) for p in self.payload)


class TraceSink:
    """Collects stage-level trace events; dump as line-oriented text."""

    def __init__(self):
        self.events: list[TraceEvent] = []

    def emit(self, kind: str, *payload) -> None:
        self.events.append(TraceEvent(kind, payload))

    def dump(self) -> str:
        return "\n".join(e.line() for e in self.events)

    def kinds(self):
        return [e.kind for e in self.events]
