"""The portfolio CSV front-end (batch.py) against the reference's own cmd_batch
output on the same file (tests/golden/portfolio*.csv, make_golden.py batch).
Header / row-shape / parse errors run on CPU; priced rows need the GPU."""

from __future__ import annotations

import csv
import io
import os

import pytest

from conftest import GOLDEN, price_close


def _read(text):
    return list(csv.reader(io.StringIO(text)))


def test_malformed_headers(tmp_path):
    from paper_2303_02317_b200 import batch

    for hdr in ("style,right,model,method,S,K,R,Y,V,E", "style,right,model,method,S,K,R,Y,V,E,T,lam",
                "style,right,model,method,S,K,R,Y,V,E,T,lambda,extra", ""):
        p = tmp_path / "p.csv"
        p.write_text(hdr + "\n")
        assert batch.price_csv(str(p), io.StringIO()) == 4, hdr


def test_unpriced_rows_match_reference(tmp_path):
    """Rows that fail before any pricing (shape, parse, combination) -- CPU only."""
    from paper_2303_02317_b200 import batch

    ref = _read(open(os.path.join(GOLDEN, "portfolio_ref.csv")).read())
    src = _read(open(os.path.join(GOLDEN, "portfolio.csv")).read())
    keep = [i for i, r in enumerate(ref[1:]) if r[-1] in ("error:method", "error:E", "error:T")
            or (r[-1] == "error:lambda" and r[11] == "abc") or len(src[1 + i]) != 12]
    p = tmp_path / "q.csv"
    with open(p, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(src[0])
        for i in keep:
            w.writerow(src[1 + i])
    out = io.StringIO()
    assert batch.price_csv(str(p), out) == 0
    got = _read(out.getvalue())
    assert got[0] == ref[0]
    assert got[1:] == [ref[1 + i] for i in keep]


@pytest.mark.gpu
def test_portfolio_matches_reference():
    from paper_2303_02317_b200 import batch

    ref = _read(open(os.path.join(GOLDEN, "portfolio_ref.csv")).read())
    out = io.StringIO()
    assert batch.price_csv(os.path.join(GOLDEN, "portfolio.csv"), out) == 0
    got = _read(out.getvalue())
    assert len(got) == len(ref) and got[0] == ref[0]
    for g, r in zip(got[1:], ref[1:]):
        assert g[:-2] == r[:-2] and g[-1] == r[-1], (g, r)
        if r[-1] == "ok":
            assert price_close(float(g[-2]), float(r[-2]), float(r[5])), (g, r)
