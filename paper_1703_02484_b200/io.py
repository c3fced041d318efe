"""Snapshot and per-step CSV files in the reference's formats, so runs of
this engine feed the reference's tools and vice versa.

  write_snapshot / read_snapshot        cli.py:263-310 (text, 17 significant digits)
  write_locality_flags / read_...       cli.py:313-321
  RunReport, aggregate, write_csv,
  read_csv, CSV_HEADER                  metrics.py:13-109

Host-side formatting only: a snapshot reads the positions back from the
device once.  Files are byte-identical to the reference's for the same
state (tests/test_io.py against files written by the reference,
tests/golden/make_golden_io.py).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .core import BrownsimError, ConfigError, PeriodicBox

CSV_HEADER = ("step,dt_used,step_ms,force_ms,maintain_ms,overlap_ms,"
              "overlap_iters,flip_passes,inversion_repairs,rollbacks")

# (csv column, StepStats attribute, is integer counter) -- metrics.py:18-29
_COLUMNS = [
    ("step", "step", True),
    ("dt_used", "dt_used", False),
    ("step_ms", "step_ms", False),
    ("force_ms", "force_ms", False),
    ("maintain_ms", "maintain_ms", False),
    ("overlap_ms", "overlap_ms", False),
    ("overlap_iters", "overlap_iterations", True),
    ("flip_passes", "flip_passes", True),
    ("inversion_repairs", "inversion_repairs", True),
    ("rollbacks", "rollbacks", True),
]

DEFAULT_WARMUP = 10  # metrics.py:31


def _g17(x) -> str:
    return format(float(x), ".17g")


# ---------------------------------------------------------------------------
# snapshots (cli.py:263-310)

def write_snapshot(system, t: float, path: str):
    """One particle per line, 'x y type', reals with 17 significant digits."""
    pos = np.asarray(system.positions, dtype=np.float64)
    types = np.asarray(system.type_of)
    lines = [f"# brownsim-snapshot v1 N={system.n} L={_g17(system.box.length)} t={_g17(t)}\n"]
    lines.extend(f"{_g17(x)} {_g17(y)} {int(k)}\n" for (x, y), k in zip(pos.tolist(), types.tolist()))
    with open(path, "w", encoding="utf-8") as fh:
        fh.writelines(lines)


def read_snapshot(path: str):
    """Inverse of write_snapshot: (positions, types, box, t); errors name the line."""
    with open(path, encoding="utf-8") as fh:
        header = fh.readline().rstrip("\n")
        parts = header.split()
        if parts[:3] != ["#", "brownsim-snapshot", "v1"]:
            raise BrownsimError(f"{path}:1: not a brownsim snapshot header: {header!r}")
        try:
            kv = dict(p.split("=", 1) for p in parts[3:])
            n = int(kv["N"])
            box = PeriodicBox(float(kv["L"]))
            t = float(kv["t"])
        except (KeyError, ValueError) as exc:
            raise BrownsimError(f"{path}:1: malformed header fields: {exc}") from exc
        positions = np.empty((n, 2), dtype=np.float64)
        types = np.empty(n, dtype=np.int32)
        for i in range(n):
            line = fh.readline()
            if not line:
                raise BrownsimError(f"{path}: truncated file, missing particle row {i}")
            cells = line.split()
            if len(cells) != 3:
                raise BrownsimError(f"{path}:{i + 2}: expected 'x y type', got {line!r}")
            try:
                positions[i, 0] = float(cells[0])
                positions[i, 1] = float(cells[1])
                types[i] = int(cells[2])
            except ValueError as exc:
                raise BrownsimError(f"{path}:{i + 2}: malformed row: {exc}") from exc
        if fh.readline().strip():
            raise BrownsimError(f"{path}: header says N={n} but more rows follow")
    return positions, types, box, t


def write_locality_flags(flags, path: str):
    with open(path, "w", encoding="utf-8") as fh:
        fh.writelines("1\n" if f else "0\n" for f in np.asarray(flags))


def read_locality_flags(path: str) -> np.ndarray:
    with open(path, encoding="utf-8") as fh:
        return np.array([line.strip() == "1" for line in fh if line.strip() != ""], dtype=bool)


# ---------------------------------------------------------------------------
# per-step series (metrics.py:34-109)

@dataclass
class RunReport:
    config_id: str
    n: int
    series: list = field(default_factory=list)
    warmup: int = DEFAULT_WARMUP

    def summary(self) -> dict:
        return aggregate(self.series, min(self.warmup, max(len(self.series) - 1, 0)))


def aggregate(series: list, warmup: int) -> dict:
    """Mean and max of every counter and timing over the post-warmup window."""
    if warmup >= len(series):
        raise ConfigError(f"warmup of {warmup} leaves no steps to aggregate (series has {len(series)})")
    window = series[warmup:]
    out = {}
    for name, attr, _ in _COLUMNS:
        if name == "step":
            continue
        vals = np.array([getattr(s, attr) for s in window], dtype=np.float64)
        out[f"mean_{name}"] = float(vals.mean())
        out[f"max_{name}"] = float(vals.max())
    out["steps"] = len(window)
    return out


def _fmt(x, integer: bool) -> str:
    return str(int(x)) if integer else _g17(x)


def write_csv(report: RunReport, path: str):
    """One row per step, then '#'-prefixed summary rows (mean/max per column)."""
    summary = report.summary() if len(report.series) > report.warmup else None
    with open(path, "w", encoding="utf-8") as fh:
        fh.write(CSV_HEADER + "\n")
        for s in report.series:
            fh.write(",".join(_fmt(getattr(s, attr), i) for _, attr, i in _COLUMNS) + "\n")
        fh.write(f"# config={report.config_id} n={report.n} warmup={report.warmup}\n")
        if summary is not None:
            for kind in ("mean", "max"):
                cells = [_g17(summary[f"{kind}_{name}"]) for name, _, _ in _COLUMNS if name != "step"]
                fh.write(f"# {kind}," + ",".join(cells) + "\n")


def read_csv(path: str) -> tuple:
    """Inverse of write_csv: (list of StepStats, parsed summary rows)."""
    from .dynamics import StepStats
    series, summary = [], {}
    with open(path, encoding="utf-8") as fh:
        header = fh.readline().rstrip("\n")
        if header != CSV_HEADER:
            raise BrownsimError(f"{path}: unexpected header {header!r}")
        for line in fh:
            line = line.rstrip("\n")
            if not line:
                continue
            if line.startswith("#"):
                body = line[1:].strip()
                kind = body.split(",", 1)[0]
                if kind in ("mean", "max"):
                    names = [name for name, _, _ in _COLUMNS if name != "step"]
                    for name, cell in zip(names, body.split(",")[1:]):
                        summary[f"{kind}_{name}"] = float(cell)
                continue
            kw = {attr: (int(cell) if integer else float(cell))
                  for (_, attr, integer), cell in zip(_COLUMNS, line.split(","))}
            series.append(StepStats(**kw))
    return series, summary
