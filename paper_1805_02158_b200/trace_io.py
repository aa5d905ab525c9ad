"""Trace CSV export in the reference's wire format (cli.py:281-298).

Header ``iter,cost,psnr,step_norm,gamma_abs_sum,elapsed_s``; floats ``%.17g``,
absent values as empty fields, elapsed with 6 decimals.  Consumers diff these
files (SPEC AC11 determinism), so the format is byte-identical to the
reference's for identical values.
"""

from __future__ import annotations

from pathlib import Path

from .errors import NativeFailure


def _field(value, fmt=".17g") -> str:
    return "" if value is None else format(value, fmt)


def trace_csv_lines(trace) -> list[str]:
    if not trace.records:
        raise ValueError("refusing to write an empty trace")
    lines = ["iter,cost,psnr,step_norm,gamma_abs_sum,elapsed_s"]
    for r in trace.records:
        lines.append(
            f"{r.iter},{_field(r.cost)},{_field(r.psnr)},"
            f"{_field(r.step_norm)},{_field(r.gamma_abs_sum)},{r.elapsed_s:.6f}"
        )
    return lines


def write_trace_csv(path, trace) -> None:
    """cli.py:285-298."""
    lines = trace_csv_lines(trace)
    try:
        Path(path).write_text("\n".join(lines) + "\n", encoding="ascii")
    except OSError as exc:
        raise NativeFailure(f"cannot write {path}: {exc}") from exc
