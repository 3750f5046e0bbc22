"""GPU accuracy audit against fixtures made by the reference's own
oracle.py / kernels.py (tests/golden/make_golden_audit.py)."""

import numpy as np
import pytest

import paper_2502_00356_b200 as bg
from paper_2502_00356_b200 import audit

pytestmark = pytest.mark.gpu


def test_dynamic_window_oracle_points(golden):
    g = golden("audit")
    got = np.array([audit.oracle_log_bessel_k(bg.EvalPoint(a, b)) for a, b in zip(g["x"], g["nu"])])
    # same window search and 2^16-bin sum; libm + summation order differ at ~1e-15
    assert np.max(np.abs(got - g["oracle_log"]) / np.maximum(1.0, np.abs(g["oracle_log"]))) < 1e-12


def test_log10_grids(golden):
    g = golden("audit")
    o10 = audit.oracle_log10_grid(g["gn"], g["gx"], bins=2 ** 14)
    assert np.max(np.abs(o10 - g["oracle_log10_2p14"])) < 1e-12
    r10 = audit.refined_log10_grid(g["hn"], g["hx"])
    assert np.max(np.abs(r10 - g["refined_log10"])) < 1e-12
    p10 = audit.pure_integral_log10_grid(g["hn"], g["hx"])
    assert np.max(np.abs(p10 - g["pure_integral_log10"])) < 1e-11


def test_relative_error_and_heatmap():
    assert audit.relative_error(0.0, 2.0 ** -52) == pytest.approx(np.log10(2.0))
    assert audit.relative_error(0.0, 1e-9) == pytest.approx(6.65356, abs=1e-4)
    nus = np.linspace(0.001, 5.0, 20)
    xs = np.linspace(0.001, 0.1, 20)
    ref = audit.oracle_log10_grid(nus, xs)
    pure = audit.error_heatmap(nus, xs, "pure-integral", reference=ref)
    refined = audit.error_heatmap(nus, xs, "refined", reference=ref)
    assert pure.re.shape == (20, 20) and np.isfinite(pure.max_re)
    assert pure.max_re >= 5.0  # SPEC acceptance 2: the integral method fails at small x
    assert refined.max_re < pure.max_re
    import io

    buf = io.StringIO()
    refined.to_csv(buf)
    assert buf.getvalue().startswith("nu,x,re\n") and buf.getvalue().count("\n") == 401


def test_bound_finder_matches_reference_primitives(golden):
    g = golden("audit")
    found, curve = audit.find_upper_bound(return_curve=True)
    ours = np.array([ae for _, ae in curve])
    ref = g["bound_ae"]
    # same answer as the reference primitives (8; SPEC's claimed 9 is not what they give)
    assert found == 8.0 and float(g["bound_L"][np.argmax(ref <= 1e-9)]) == 8.0
    big = ref > 1e-9
    assert np.allclose(ours[big], ref[big], rtol=1e-6)
    assert np.all(ours[~big] < 1e-12)
