"""GPU tests of the SURVEY 8f 'next' rows built so far: device location
preprocessing (f2, bitwise equal to the host SPEC definitions) and the GP
consumer (f3: simulate / log_likelihood / predict / fit_mle on the generated
matrix, checked against the SPEC examples and a CPU oracle likelihood)."""

import math

import numpy as np
import pytest
import torch

import paper_2502_00356_b200 as bg
from paper_2502_00356_b200 import gp

pytestmark = pytest.mark.gpu


def test_normalize_device_matches_host():
    rng = np.random.default_rng(0)
    raw = rng.random((5000, 2)) * np.array([7.0, 3.0]) - 2.5
    host = bg.normalize_locations(bg.LocationSet(raw)).coords
    dev = bg.normalize_locations(torch.from_numpy(raw).cuda()).cpu().numpy()
    assert np.array_equal(host, dev)
    ex = torch.tensor([[10.0, 10.0], [10.0, 12.0], [11.0, 10.0]], dtype=torch.float64).cuda()
    assert np.array_equal(bg.normalize_locations(ex).cpu().numpy(), [[0, 0], [0, 1], [0.5, 0]])
    with pytest.raises(bg.DomainError, match="coincide"):
        bg.normalize_locations(torch.ones((3, 2), dtype=torch.float64).cuda())


@pytest.mark.parametrize("bits", [2, 10, 16, 31])
def test_morton_device_matches_host(bits):
    rng = np.random.default_rng(bits)
    s = bg.LocationSet(rng.random((4000, 2)), normalized=True)
    hs, hp = bg.morton_order(s, bits)
    dc, dp = bg.morton_order(torch.from_numpy(s.coords).cuda(), bits)
    assert np.array_equal(dp.cpu().numpy(), hp)
    assert np.array_equal(dc.cpu().numpy(), hs.coords)


def test_permutation_equivariance_bitwise():
    """Morton-reordering then generating Sigma equals P Sigma P^T bitwise."""
    rng = np.random.default_rng(3)
    s = bg.LocationSet(rng.random((700, 2)), normalized=True)
    theta = bg.MaternParams(1.0, 0.1, 1.5)
    full = bg.generate_covariance(s, theta, device="cuda").data
    ms, perm = bg.morton_order(s)
    permuted = bg.generate_covariance(ms, theta, device="cuda").data
    p = torch.from_numpy(perm).cuda()
    assert torch.equal(permuted, full[p][:, p])


def test_log_likelihood_spec_examples():
    one = bg.LocationSet(np.array([[0.5, 0.5]]))
    o = gp.Observations(one, np.array([0.0]))
    assert abs(gp.log_likelihood(o, bg.MaternParams(1.0, 0.1, 0.5)) + 0.5 * math.log(2 * math.pi)) < 1e-15
    o2 = gp.Observations(one, np.array([2.0]))
    v = gp.log_likelihood(o2, bg.MaternParams(4.0, 0.1, 0.5))
    assert abs(v - (-0.5 * (math.log(2 * math.pi) + math.log(4.0) + 1.0))) < 1e-14


def test_log_likelihood_vs_cpu(oracle):
    rng = np.random.default_rng(11)
    locs = bg.LocationSet(rng.random((300, 2)))
    obs = gp.simulate(locs, bg.MaternParams(1.0, 0.1, 1.5), seed=5)
    again = gp.simulate(locs, bg.MaternParams(1.0, 0.1, 1.5), seed=5)
    assert np.array_equal(obs.z, again.z)
    th = bg.MaternParams(0.8, 0.07, 1.2)
    sig = oracle.generate_covariance(locs.coords, 0.8, 0.07, 1.2)
    sign, logdet = np.linalg.slogdet(sig)
    ref = -0.5 * (300 * math.log(2 * math.pi) + logdet + obs.z @ np.linalg.solve(sig, obs.z))
    assert abs(gp.log_likelihood(obs, th) - ref) < 1e-8 * abs(ref)


def test_predict_interpolates_and_fit_improves():
    rng = np.random.default_rng(12)
    locs = bg.LocationSet(rng.random((200, 2)))
    truth = bg.MaternParams(1.0, 0.1, 0.5)
    obs = gp.simulate(locs, truth, seed=1)
    test = bg.LocationSet(locs.coords[:5].copy())
    pred, mspe = gp.predict(obs, truth, test, z_true=obs.z[:5])
    assert np.allclose(pred, obs.z[:5], atol=1e-8) and mspe < 1e-15
    fit = gp.fit_mle(obs, max_evals=60)
    assert fit.iterations >= 1 and fit.llh >= gp.log_likelihood(obs, gp.MLE_START)
