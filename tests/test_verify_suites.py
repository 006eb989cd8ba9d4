"""The on-device verify suites (verify.py) against the reference's own verify
output for the same seed (tests/golden/verify_ref.txt): every suite passes,
and the bsm-theorems weight identity (a host-side check) reports the same
worst ratio."""

from __future__ import annotations

import io
import os

import pytest

from conftest import GOLDEN


def _lines(text):
    return [ln.split() for ln in text.splitlines() if ln and not ln.startswith(" ")]


@pytest.mark.gpu
def test_verify_matches_reference():
    from paper_2303_02317_b200 import verify

    out = io.StringIO()
    rc = verify.run_suites(reps=6, steps=1024, seed=3, out=out)
    ref = _lines(open(os.path.join(GOLDEN, "verify_ref.txt")).read())
    got = _lines(out.getvalue())
    assert rc == 0, out.getvalue()
    assert [g[0] for g in got] == [r[0] for r in ref]
    assert [g[1] for g in got] == [r[1] for r in ref]
    # the weight identity is pure host arithmetic: identical worst ratio
    assert got[4][3] == ref[4][3]


def test_verify_argument_errors():
    import paper_2303_02317_b200 as fl
    from paper_2303_02317_b200 import verify

    with pytest.raises(fl.ValidationError):
        verify.run_suites(reps=-1)
    with pytest.raises(fl.ValidationError):
        verify.run_suites(reps=2, steps=10)
    assert verify.run_suites(reps=0) == 0
