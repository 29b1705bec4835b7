"""Timeline documents for predicted or measured steps (`pkg/src/zeroppsim/render.py`).

``render_timeline(result, sched, format)`` emits the reference's two deterministic
formats -- an ASCII Gantt (one compute lane per device, a ``~`` comm sub-lane under
it) and a minimal SVG -- byte-identical to the reference for the same
:class:`SimResult` (pinned by tests/golden/render_*.txt).  ``chrome_trace`` is the
engine's addition for MEASURED steps: a Chrome/Perfetto trace-event JSON with one
process per device and compute / comm threads.

Glyphs: F forward, B input grad, W weight grad, r recompute, O optimizer, ~ comm,
. idle (`render.py:1-44`).  Zero-length tasks are not drawn.
"""

from __future__ import annotations

import json
import logging
from enum import Enum

from .config import ConfigError
from .simulation import SimResult
from .tasks import Schedule, TaskKind

__all__ = ["RenderFormat", "render_timeline", "render_ascii", "render_svg", "chrome_trace"]

log = logging.getLogger(__name__)

GLYPHS = {TaskKind.F: "F", TaskKind.B: "B", TaskKind.W: "W", TaskKind.R: "r", TaskKind.OPT: "O"}
FILLS = {TaskKind.F: "#4c72b0", TaskKind.B: "#dd8452", TaskKind.W: "#55a868", TaskKind.R: "#c44e52",
         TaskKind.OPT: "#8172b3"}
COMM_FILL = "#937860"
MAX_EXACT_COLUMNS = 4000   # beyond this the ASCII view switches to proportional columns
PROPORTIONAL_COLUMNS = 120


class RenderFormat(str, Enum):
    ASCII = "ascii"
    SVG = "svg"


def _lanes(result: SimResult, sched: Schedule):
    """[(compute cells, comm cells)] per device; cells = (start, end, task), by start."""
    out = []
    for tasks in sched.per_device:
        cells = {True: [], False: []}
        for t in tasks:
            s, e = result.task_times[t]
            if e > s:
                cells[t.is_compute].append((s, e, t))
        out.append(tuple(sorted(cells[k], key=lambda c: c[0]) for k in (True, False)))
    return out


def _exact_slot(result: SimResult, sched: Schedule) -> float | None:
    """Widest column such that every drawn task starts and ends on a column border."""
    lengths, marks = set(), set()
    for t in sched.tasks():
        s, e = result.task_times[t]
        if e > s:
            lengths.add(e - s)
            marks.update((s, e))
    if not lengths or min(lengths) <= 0:
        return None
    slot = min(lengths)
    if any(abs(m / slot - round(m / slot)) > 1e-6 for m in marks):
        return None
    return None if result.makespan / slot > MAX_EXACT_COLUMNS else slot


def _row(cells, width: int, col, glyph) -> str:
    row = ["."] * width
    for s, e, t in cells:
        a = col(s)
        b = max(col(e) - 1, a)
        for c in range(a, min(b, width - 1) + 1):
            row[c] = glyph(t)
    return "".join(row)


def render_ascii(result: SimResult, sched: Schedule) -> str:
    lanes = _lanes(result, sched)
    slot = _exact_slot(result, sched)
    if slot is None:
        log.warning("task durations are not commensurate; falling back to proportional column widths")
        width = PROPORTIONAL_COLUMNS
        k = width / result.makespan if result.makespan > 0 else 0.0
        col = lambda x: min(int(x * k), width)  # noqa: E731
        lines = [f"makespan={result.makespan:.10g} columns={width} (proportional)"]
    else:
        width = round(result.makespan / slot)
        col = lambda x: round(x / slot)  # noqa: E731
        lines = [f"makespan={result.makespan:.10g} columns={width} slot={slot:.10g}"]
    pad = len(f"d{len(lanes) - 1}") + 1
    for d, (compute, comm) in enumerate(lanes):
        lines.append(f"d{d}".ljust(pad) + "|" + _row(compute, width, col, lambda t: GLYPHS[t.kind]) + "|")
        if comm:
            lines.append("~".rjust(pad - 1).ljust(pad) + "|" + _row(comm, width, col, lambda t: "~") + "|")
    lines.append("legend: F=forward B=input-grad W=weight-grad r=recompute O=optimizer ~=comm .=idle")
    return "\n".join(lines) + "\n"


def render_svg(result: SimResult, sched: Schedule) -> str:
    lanes = _lanes(result, sched)
    W, H_ROW, H_COMM, GAP, X0 = 1000.0, 18, 8, 6, 40
    k = W / result.makespan if result.makespan > 0 else 0.0
    pitch = H_ROW + H_COMM + GAP

    def box(x, y, w, h, fill, title):
        return (f'<rect x="{x:.2f}" y="{y}" width="{max(w, 0.5):.2f}" height="{h}" fill="{fill}">'
                f'<title>{title}</title></rect>')

    doc = [f'<svg xmlns="http://www.w3.org/2000/svg" width="{X0 + W:.0f}" height="{len(lanes) * pitch + GAP}" '
           f'font-family="monospace" font-size="10">']
    for d, (compute, comm) in enumerate(lanes):
        y = GAP // 2 + d * pitch
        doc.append(f'<text x="2" y="{y + H_ROW - 5}">d{d}</text>')
        doc += [box(X0 + s * k, y, (e - s) * k, H_ROW, FILLS[t.kind], t.task_id) for s, e, t in compute]
        doc += [box(X0 + s * k, y + H_ROW + 1, (e - s) * k, H_COMM, COMM_FILL, t.task_id) for s, e, t in comm]
    doc.append("</svg>")
    return "\n".join(doc) + "\n"


def render_timeline(result: SimResult, sched: Schedule, format: RenderFormat = RenderFormat.ASCII) -> str:
    """Deterministic text rendering (`render.py:162-170`)."""
    try:
        fmt = RenderFormat(format)
    except ValueError:
        raise ConfigError(f"unknown render format: {format}") from None
    return render_ascii(result, sched) if fmt is RenderFormat.ASCII else render_svg(result, sched)


def chrome_trace(result: SimResult, sched: Schedule, time_unit_us: float = 1000.0) -> str:
    """Trace-event JSON (chrome://tracing, Perfetto).  ``time_unit_us`` converts the
    result's time unit to microseconds (1000 for measured milliseconds)."""
    ev = []
    for d, tasks in enumerate(sched.per_device):
        ev.append({"ph": "M", "pid": d, "name": "process_name", "args": {"name": f"device {d}"}})
        ev.append({"ph": "M", "pid": d, "tid": 0, "name": "thread_name", "args": {"name": "compute"}})
        ev.append({"ph": "M", "pid": d, "tid": 1, "name": "thread_name", "args": {"name": "comm"}})
        for t in tasks:
            if t not in result.task_times:
                continue
            s, e = result.task_times[t]
            ev.append({"ph": "X", "pid": d, "tid": 0 if t.is_compute else 1, "name": t.task_id,
                       "cat": t.kind.value, "ts": s * time_unit_us, "dur": max(e - s, 0.0) * time_unit_us})
    return json.dumps({"traceEvents": ev, "displayTimeUnit": "ms",
                       "otherData": {k: v for k, v in result.extras.items()
                                     if isinstance(v, (int, float, str))}})
