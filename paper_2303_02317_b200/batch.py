"""Portfolio CSV batch front-end on the GPU path.

Mirrors the reference's ``cmd_batch`` / ``_batch_row_price`` (cli.py:727-842):
same header contract (``style,right,model,method,S,K,R,Y,V,E,T[,lambda]``),
same output (the input row plus ``price,status``, status ``ok`` or
``error:<column>``), same error-to-column mapping and exit codes -- but the
rows are parsed first and every group of rows with the same pricer is priced
by ONE device call (``fl_price_batch`` / ``fl_euro_approx``) instead of one
solver call per row.  Prices are formatted with ``repr(float)`` as the
reference does.

    python -m paper_2303_02317_b200.batch --csv portfolio.csv > priced.csv
"""

from __future__ import annotations

import argparse
import csv
import sys
from collections import defaultdict

import numpy as np

from . import _native
from .bsm import DEFAULT_LAMBDA
from .model import PricingError, StabilityError, UnsupportedCombinationError, ValidationError

__all__ = ["BATCH_HEADER", "price_rows", "price_csv", "main"]

BATCH_HEADER = ["style", "right", "model", "method", "S", "K", "R", "Y", "V", "E", "T"]  # cli.py:727-739

_FIELD_TO_COLUMN = {  # cli.py:741-750
    "spot": "S", "strike": "K", "rate": "R", "dividend_yield": "Y", "volatility": "V",
    "days_to_expiry": "E", "steps": "T", "lam": "lambda",
}

_COMBINATIONS = {  # cli.py:72-82
    ("european", "call", "binomial"): ("fast", "baseline", "gaussian", "closed-form"),
    ("american", "call", "binomial"): ("fast", "baseline"),
    ("american", "put", "bsm"): ("fast", "baseline"),
}

_NUMERIC = (("spot", 4, float), ("strike", 5, float), ("rate", 6, float), ("dividend_yield", 7, float),
            ("volatility", 8, float), ("days_to_expiry", 9, int), ("steps", 10, int))


def _status_of_exception(exc: Exception) -> str:
    """cmd_batch's mapping of a row's exception to its status cell (cli.py:825-836)."""
    if isinstance(exc, UnsupportedCombinationError):
        return "error:method"
    if isinstance(exc, ValidationError):
        return f"error:{_FIELD_TO_COLUMN.get(exc.field, exc.field)}"
    if isinstance(exc, StabilityError):
        return "error:lambda"
    if isinstance(exc, PricingError):
        return "error:S"
    raise exc  # anything else propagates, as in the reference


def _parse(row: list[str], has_lambda: bool):
    """(key, numbers, lam) for a row or raise the reference's exception
    (cli.py:753-794: numeric parse errors first, then the combination)."""
    style, right, model, method = (tok.strip() for tok in row[:4])
    num = {}
    for field, col, conv in _NUMERIC:
        try:
            num[field] = conv(row[col].strip())
        except ValueError:
            raise ValidationError(field, f"cannot parse {BATCH_HEADER[col]}={row[col]!r}") from None
    lam = None
    if has_lambda and len(row) > 11 and row[11].strip():
        try:
            lam = float(row[11])
        except ValueError:
            raise ValidationError("lam", f"cannot parse lambda={row[11]!r}") from None
    methods = _COMBINATIONS.get((style, right, model))
    if methods is None or method not in methods:
        raise UnsupportedCombinationError(
            f"unsupported combination: style={style} right={right} model={model} method={method}")
    return (style, right, model, method), num, lam


def price_rows(rows: list[list[str]], has_lambda: bool) -> list[tuple[str, str]]:
    """(price cell, status cell) per row; rows already length-checked."""
    out: list[tuple[str, str] | None] = [None] * len(rows)
    groups = defaultdict(list)  # (kind, method code, lam) -> row indices
    parsed = {}
    for i, row in enumerate(rows):
        try:
            key, num, lam = _parse(row, has_lambda)
        except Exception as exc:  # noqa: BLE001 -- mapped exactly like cmd_batch
            out[i] = ("", _status_of_exception(exc))
            continue
        parsed[i] = num
        style, right, model, method = key
        if model == "bsm":
            groups[(_native.KIND_PUT, method, DEFAULT_LAMBDA if lam is None else lam)].append(i)
        elif style == "american":
            groups[(_native.KIND_CALL, method, 0.0)].append(i)
        else:
            groups[(_native.KIND_EURO, method, 0.0)].append(i)
    for (kind, method, lam), idx in groups.items():
        cols = [np.array([parsed[i][f] for i in idx], dtype=np.float64)
                for f in ("spot", "strike", "rate", "dividend_yield", "volatility", "days_to_expiry")]
        T = np.array([parsed[i]["steps"] for i in idx], dtype=np.int64)
        if kind == _native.KIND_EURO and method in ("gaussian", "closed-form"):
            code = _native.METHOD_GAUSS if method == "gaussian" else _native.METHOD_CLOSED
            price, status = _native.euro_approx(*cols, T, code)
        else:
            code = _native.METHOD_FAST if method == "fast" else _native.METHOD_BASELINE
            res = _native.price_batch(np.int8(kind), *cols, T, lam=lam if kind == _native.KIND_PUT else DEFAULT_LAMBDA,
                                      method=code)
            price, status = res.price, res.status
        for k, i in enumerate(idx):
            err = _native.status_error(int(status[k]))
            out[i] = (repr(float(price[k])), "ok") if err is None else ("", _status_of_exception(err))
    return out  # type: ignore[return-value]


def price_csv(path: str, out=sys.stdout) -> int:
    """cmd_batch on the GPU path; returns the reference's exit code."""
    with open(path, newline="") as fh:
        reader = csv.reader(fh)
        header = next(reader, None)
        has_lambda = False
        if header is not None:
            header = [tok.strip() for tok in header]
        if header is None or header[: len(BATCH_HEADER)] != BATCH_HEADER:
            print("error: malformed header", file=sys.stderr)
            return 4
        if len(header) == len(BATCH_HEADER) + 1:
            if header[-1] != "lambda":
                print("error: malformed header", file=sys.stderr)
                return 4
            has_lambda = True
        elif len(header) != len(BATCH_HEADER):
            print("error: malformed header", file=sys.stderr)
            return 4
        rows = [row for row in reader if row]
    writer = csv.writer(out)
    writer.writerow([*header, "price", "status"])
    good = [r for r in rows if len(r) == len(header)]
    priced = iter(price_rows(good, has_lambda))
    for row in rows:
        if len(row) < len(header):
            writer.writerow([*row, "", f"error:{header[len(row)]}"])
        elif len(row) > len(header):
            writer.writerow([*row, "", f"error:{header[-1]}"])
        else:
            writer.writerow([*row, *next(priced)])
    return 0


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(description="price a portfolio CSV on the GPU (fftlattice batch format)")
    ap.add_argument("--csv", required=False)
    ap.add_argument("--parallel", action="store_true", help="accepted for compatibility (no effect)")
    args = ap.parse_args(argv)
    if not args.csv:
        raise OSError("batch requires --csv with the portfolio file")
    return price_csv(args.csv)


if __name__ == "__main__":
    sys.exit(main())
