"""Matrix files in, reports out (reference ``rgsv/io.py``).

The formats are the reference's, so files written by either package are read
by the other and reports serialize to the same text:

* ``read_matrix`` (io.py:30-88): a Matrix Market file (dense ``array`` or
  ``coordinate``; real / integer / pattern / complex; general / symmetric /
  skew-symmetric / hermitian — coordinate entries are densified) or a
  headerless CSV whose cells are real or complex literals. The format is
  sniffed from the first line. The Matrix Market grammar is parsed here (the
  reference delegates to ``scipy.io.mmread``).
* ``write_matrix`` (io.py:91-96): dense real Matrix Market at 17 significant
  digits, column-major, which ``read_matrix`` round-trips bitwise.
* ``report_to_dict`` / ``write_report`` (io.py:120-264): JSON or CSV of a
  ``ComparativeReport``, ``GsvSpectrum``, ``BoundCertificate``,
  ``BasisResult`` or a list of the timing harness's ``BenchRecord``s, floats
  at ``.17g``.

Parsing and serialization are host work by nature; the parsed arrays go to
the device path through ``GmpPair`` / ``extract_basis`` unchanged. Complex
files are parsed faithfully and then rejected by the device path's
``ValidationError`` (no CPU fallback).
"""

from __future__ import annotations

import csv
import dataclasses
import json
import sys
from pathlib import Path

import numpy as np

from .errors import DimensionError, ParseError, ValidationError

MM_BANNER = "%%MatrixMarket"
_FIELDS = ("real", "double", "integer", "complex", "pattern")
_SYMMETRIES = ("general", "symmetric", "skew-symmetric", "hermitian")


def _checked(a: np.ndarray, name: str) -> np.ndarray:
    """The host half of core.as_matrix (core.py:43-57) for freshly parsed
    data: 2-D, nonempty, float64 / complex128, finite."""
    if a.ndim != 2:
        raise DimensionError(f"{name} must be 2-dimensional, got {a.ndim} dimensions")
    if a.shape[0] < 1 or a.shape[1] < 1:
        raise DimensionError(f"{name} must be nonempty, got shape {a.shape}")
    a = a.astype(np.complex128 if np.iscomplexobj(a) else np.float64, copy=False)
    if not np.isfinite(a).all():
        raise ValidationError(f"{name} contains non-finite entries")
    return np.ascontiguousarray(a)


def read_matrix(path) -> np.ndarray:
    """Matrix Market or headerless CSV -> validated dense host array
    (io.py:30-46)."""
    path = Path(path)
    try:
        with open(path, "r") as fh:
            text = fh.read()
    except (OSError, UnicodeDecodeError) as exc:
        raise ParseError(f"{path}: cannot read: {exc}") from exc
    if text.startswith(MM_BANNER):
        return _checked(_parse_matrix_market(text, path), str(path))
    return _checked(_parse_csv(text, path), str(path))


def _mm_fail(path, why: str):
    return ParseError(f"{path}: invalid Matrix Market file: {why}")


def _parse_matrix_market(text: str, path) -> np.ndarray:
    lines = text.splitlines()
    banner = lines[0].split()
    if len(banner) != 5 or banner[1].lower() != "matrix":
        raise _mm_fail(path, f"bad banner {lines[0]!r}")
    layout, field, symmetry = (w.lower() for w in banner[2:])
    if layout not in ("array", "coordinate"):
        raise _mm_fail(path, f"unknown format {layout!r}")
    if field not in _FIELDS:
        raise _mm_fail(path, f"unknown field {field!r}")
    if symmetry not in _SYMMETRIES:
        raise _mm_fail(path, f"unknown symmetry {symmetry!r}")
    if field == "pattern" and layout == "array":
        raise _mm_fail(path, "pattern field needs the coordinate format")
    if symmetry == "hermitian" and field != "complex":
        raise _mm_fail(path, "hermitian symmetry needs the complex field")
    body = [ln for ln in lines[1:] if ln.strip() and not ln.lstrip().startswith("%")]
    if not body:
        raise _mm_fail(path, "missing size line")
    try:
        size = [int(w) for w in body[0].split()]
    except ValueError:
        raise _mm_fail(path, f"bad size line {body[0]!r}") from None
    try:
        tokens = np.array(" ".join(body[1:]).split(), dtype=np.float64)
    except ValueError as exc:
        raise _mm_fail(path, f"non-numeric entry ({exc})") from None
    is_complex = field == "complex"
    dtype = np.complex128 if is_complex else np.float64

    def mirror(a):
        # fill the strict upper triangle from the stored lower one
        lower = np.tril(a, -1)
        if symmetry == "symmetric":
            return a + lower.T
        if symmetry == "skew-symmetric":
            return a - lower.T
        if symmetry == "hermitian":
            return a + lower.conj().T
        return a

    if layout == "array":
        if len(size) != 2 or min(size) < 0:
            raise _mm_fail(path, f"bad size line {body[0]!r}")
        rows, cols = size
        per = 2 if is_complex else 1
        if symmetry == "general":
            count = rows * cols
        else:
            if rows != cols:
                raise _mm_fail(path, "symmetric array must be square")
            count = rows * (rows + 1) // 2 if symmetry != "skew-symmetric" else rows * (rows - 1) // 2
        if tokens.size != count * per:
            raise _mm_fail(path, f"expected {count} entries, found {tokens.size // per}")
        vals = tokens.view(np.complex128) if is_complex else tokens
        if symmetry == "general":
            return vals.reshape(cols, rows).T.astype(dtype)  # file is column-major
        a = np.zeros((rows, cols), dtype=dtype)
        ii, jj = np.tril_indices(rows, -1 if symmetry == "skew-symmetric" else 0)
        order = np.lexsort((ii, jj))  # column by column of the lower triangle
        a[ii[order], jj[order]] = vals
        return mirror(a)

    if len(size) != 3 or min(size) < 0:
        raise _mm_fail(path, f"bad size line {body[0]!r}")
    rows, cols, nnz = size
    per = 2 + (0 if field == "pattern" else (2 if is_complex else 1))
    if tokens.size != nnz * per:
        raise _mm_fail(path, f"expected {nnz} entries of {per} fields")
    ent = tokens.reshape(nnz, per)
    ii = ent[:, 0].astype(np.int64) - 1
    jj = ent[:, 1].astype(np.int64) - 1
    if nnz and ((ent[:, 0] != ii + 1).any() or (ent[:, 1] != jj + 1).any() or ii.min() < 0
                or jj.min() < 0 or ii.max() >= rows or jj.max() >= cols):
        raise _mm_fail(path, "index out of range")
    if field == "pattern":
        vals = np.ones(nnz)
    elif is_complex:
        vals = ent[:, 2] + 1j * ent[:, 3]
    else:
        vals = ent[:, 2]
    a = np.zeros((rows, cols), dtype=dtype)
    np.add.at(a, (ii, jj), vals)  # repeated entries sum, as in scipy's COO
    if symmetry != "general":
        if rows != cols:
            raise _mm_fail(path, "symmetric matrix must be square")
        off = ii != jj
        sign = -1.0 if symmetry == "skew-symmetric" else 1.0
        mv = vals[off].conj() if symmetry == "hermitian" else vals[off]
        np.add.at(a, (jj[off], ii[off]), sign * mv)
    return a


def _parse_csv(text: str, path) -> np.ndarray:
    rows = []
    width = None
    for lineno, line in enumerate(text.splitlines(), start=1):
        line = line.strip()
        if not line:
            continue
        vals = []
        for col, cell in enumerate((c.strip() for c in line.split(",")), start=1):
            try:
                vals.append(float(cell))
            except ValueError:
                try:
                    vals.append(complex(cell))
                except ValueError:
                    raise ParseError(
                        f"{path}:{lineno}: column {col}: not a number: {cell!r}") from None
        if width is None:
            width = len(vals)
        elif len(vals) != width:
            raise ParseError(f"{path}:{lineno}: expected {width} columns, found {len(vals)}")
        rows.append(vals)
    if not rows:
        raise ParseError(f"{path}: no data rows")
    return np.array(rows)


def write_matrix(path, m) -> None:
    """Dense Matrix Market at full precision (io.py:91-96): the same text
    scipy's writer produces at precision 17 (``%.16e``-style mantissa,
    column-major), so files are interchangeable byte for byte."""
    if hasattr(m, "t") and hasattr(m, "rows"):  # a device.DevMatrix
        m = m.t
    if hasattr(m, "detach"):
        m = m.detach().cpu().numpy()
    a = _checked(np.asarray(m), "matrix")
    cplx = np.iscomplexobj(a)
    with open(path, "w") as fh:
        fh.write(f"{MM_BANNER} matrix array {'complex' if cplx else 'real'} general\n%\n")
        fh.write(f"{a.shape[0]} {a.shape[1]}\n")
        flat = a.T.reshape(-1)
        if cplx:
            fh.write("".join(f"{v.real:.16e} {v.imag:.16e}\n" for v in flat))
        else:
            fh.write("".join(f"{v:.16e}\n" for v in flat))


def _num(x) -> str:
    if x is None:
        return ""
    if isinstance(x, (bool, np.bool_)):
        return "true" if x else "false"
    if isinstance(x, (int, np.integer)):
        return str(int(x))
    return format(float(x), ".17g")


def _plain(x):
    if isinstance(x, np.ndarray):
        return [float(v) for v in x]
    if isinstance(x, np.integer):
        return int(x)
    if isinstance(x, np.floating):
        return float(x)
    if isinstance(x, np.bool_):
        return bool(x)
    return x


_BENCH_COLUMNS = ("method", "repetition", "seconds", "err_alpha", "err_beta", "residual1",
                  "residual2", "l1", "l2", "m", "p", "n")


def _kind(report) -> str:
    # late imports: io is a leaf the CLI pulls in before the device modules
    if isinstance(report, (list, tuple)):  # the timing harness's records (io.py:171-178)
        return "bench_records"
    from .analysis import ComparativeReport
    from .bounds import BoundCertificate
    from .engine import GsvSpectrum
    from .rangefinder import BasisResult

    for cls, kind in ((ComparativeReport, "comparative_report"), (GsvSpectrum, "spectrum"),
                      (BoundCertificate, "bound_certificate"), (BasisResult, "basis_result")):
        if isinstance(report, cls):
            return kind
    raise ValidationError(f"cannot serialize report of type {type(report).__name__}")


def _basis_columns(report) -> int:
    q = report.q
    return int(q.shape[1]) if hasattr(q, "shape") else int(q.cols)


def report_to_dict(report) -> dict:
    """JSON structure of a report object (io.py:120-180), key for key."""
    kind = _kind(report)
    if kind == "bench_records":
        return {"kind": kind,
                "records": [{k: _plain(v) for k, v in dataclasses.asdict(rec).items()}
                            for rec in report]}
    if kind == "comparative_report":
        spec = report.spectrum
        return {"kind": kind, "alphas": _plain(spec.alphas), "betas": _plain(spec.betas),
                "rho": _plain(report.rho), "theta": _plain(report.theta),
                "p1": _plain(report.p1), "p2": _plain(report.p2), "d1": report.d1,
                "d2": report.d2, "r": spec.r, "s": spec.s, "n": spec.n,
                "meta": dict(report.meta)}
    if kind == "spectrum":
        return {"kind": kind, "alphas": _plain(report.alphas), "betas": _plain(report.betas),
                "r": report.r, "s": report.s, "n": report.n}
    if kind == "bound_certificate":
        return {"kind": kind, "eta": report.eta, "e_script": report.e_script,
                "theta_bound": report.theta_bound, "p1_bounds": _plain(report.p1_bounds),
                "p2_bounds": _plain(report.p2_bounds), "d1_bound": report.d1_bound,
                "d2_bound": report.d2_bound, "vacuous": report.vacuous}
    return {"kind": kind, "columns": _basis_columns(report), "converged": report.converged,
            "iterations": report.iterations,
            "residual_history": [float(v) for v in report.residual_history],
            "block_widths": [int(w) for w in report.block_widths]}


def _csv_rows(report) -> list:
    """Per-index rows, then the scalar block (io.py:183-247)."""
    kind = _kind(report)
    if kind == "bench_records":  # one row per record (io.py:236-245)
        rows = [list(_BENCH_COLUMNS)]
        for rec in report:
            d = dataclasses.asdict(rec)
            rows.append([d[k] if isinstance(d[k], str) else _num(d[k]) for k in _BENCH_COLUMNS])
        return rows
    if kind == "comparative_report":
        spec = report.spectrum
        cols = (spec.alphas, spec.betas, report.rho, report.theta, report.p1, report.p2)
        rows = [["index", "alpha", "beta", "rho", "theta", "p1", "p2"]]
        rows += [[i + 1] + [_num(c[i]) for c in cols] for i in range(spec.n)]
        rows += [["d1", _num(report.d1)], ["d2", _num(report.d2)], ["r", spec.r], ["s", spec.s],
                 ["seed", report.meta.get("seed", "")], ["tol", _num(report.meta.get("tol"))]]
        return rows
    if kind == "spectrum":
        rows = [["index", "alpha", "beta"]]
        rows += [[i + 1, _num(report.alphas[i]), _num(report.betas[i])] for i in range(report.n)]
        return rows + [["r", report.r], ["s", report.s]]
    if kind == "bound_certificate":
        rows = [["index", "p1_bound", "p2_bound"]]
        rows += [[i + 1, _num(report.p1_bounds[i]), _num(report.p2_bounds[i])]
                 for i in range(report.p1_bounds.size)]
        for key in ("eta", "e_script", "theta_bound", "d1_bound", "d2_bound", "vacuous"):
            rows.append([key, _num(getattr(report, key))])
        return rows
    rows = [["iteration", "residual"]]
    rows += [[i, _num(res)] for i, res in enumerate(report.residual_history)]
    return rows + [["columns", _basis_columns(report)], ["converged", _num(report.converged)],
                   ["iterations", report.iterations]]


def write_report(report, path=None, fmt: str = "csv") -> None:
    """Serialize a report to ``path`` (stdout when None) as csv or json
    (io.py:250-264)."""
    if fmt not in ("csv", "json"):
        raise ValidationError(f"format must be 'csv' or 'json', got {fmt!r}")

    def emit(fh):
        if fmt == "json":
            json.dump(report_to_dict(report), fh, indent=2)
            fh.write("\n")
        else:
            csv.writer(fh, lineterminator="\n").writerows(_csv_rows(report))

    if path is None:
        emit(sys.stdout)
        return
    with open(path, "w", newline="") as fh:
        emit(fh)


__all__ = ["read_matrix", "write_matrix", "report_to_dict", "write_report"]
