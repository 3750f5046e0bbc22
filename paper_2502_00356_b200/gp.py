"""Gaussian-process consumer of the covariance matrix.

The paper's end-to-end gains come from regenerating Sigma(theta) at every MLE
iteration; here every evaluation is one matrix generation on the
sm_100a kernel plus a cuSOLVER Cholesky (torch.linalg) on the same device:

    simulate      z = L u,  L = chol(Sigma(theta)),  u ~ N(0, I) seeded
    log_likelihood  -1/2 [N log 2pi + log|Sigma| + z^T Sigma^-1 z]  (two triangular solves)
    predict       kriging mean Sigma_test,train Sigma_train^-1 z  (+ MSPE)
    fit_mle       derivative-free simplex (Nelder-Mead) over log(theta) in the SPEC box

Optimiser bookkeeping runs on the host; the O(N^2) / O(N^3) work is on the GPU.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .besselk import DEFAULT_CONFIG, DomainError, QuadratureConfig
from .covariance import LocationSet, MaternParams, TileSpec, generate_covariance, generate_tile

LOG_2PI = math.log(2.0 * math.pi)
# start and box of the MLE search
MLE_START = MaternParams(1.0, 0.01, 0.5)
MLE_BOUNDS = ((0.01, 10.0), (0.005, 1.0), (0.1, 5.0))


def _torch():
    import torch

    return torch


@dataclass(frozen=True)
class Observations:
    locs: LocationSet
    z: np.ndarray

    def __post_init__(self):
        z = np.ascontiguousarray(self.z, dtype=np.float64).ravel()
        if z.size != len(self.locs):
            raise DomainError("length(z) must equal length(locs)")
        object.__setattr__(self, "z", z)


@dataclass
class FitResult:
    theta_hat: MaternParams
    llh: float
    iterations: int
    converged: bool
    trace: list = field(default_factory=list)


def _cholesky(locs, theta, cfg, device):
    torch = _torch()
    sigma = generate_covariance(locs, theta, cfg, device=device).data
    L, info = torch.linalg.cholesky_ex(sigma)
    if int(info) != 0:
        raise np.linalg.LinAlgError("covariance matrix is not positive definite")
    return L


def simulate(locs: LocationSet, theta: MaternParams, seed: int,
             cfg: QuadratureConfig = DEFAULT_CONFIG, device="cuda") -> Observations:
    """z = L u with u ~ N(0, I) from numpy's default_rng(seed) (same seed -> same z)."""
    torch = _torch()
    u = np.random.default_rng(seed).standard_normal(len(locs))
    L = _cholesky(locs, theta, cfg, device)
    z = (L @ torch.from_numpy(u).to(L.device)).cpu().numpy()
    return Observations(locs, z)


def log_likelihood(obs: Observations, theta: MaternParams,
                   cfg: QuadratureConfig = DEFAULT_CONFIG, device="cuda") -> float:
    """Exact Gaussian log-likelihood; -inf when Sigma(theta) is not positive definite."""
    torch = _torch()
    try:
        L = _cholesky(obs.locs, theta, cfg, device)
    except np.linalg.LinAlgError:
        return -math.inf
    z = torch.from_numpy(obs.z).to(L.device).unsqueeze(1)
    w = torch.linalg.solve_triangular(L, z, upper=False)
    logdet = 2.0 * torch.log(torch.diagonal(L)).sum()
    quad = (w * w).sum()
    return float(-0.5 * (obs.z.size * LOG_2PI + logdet + quad))


def predict(train: Observations, theta: MaternParams, test_locs: LocationSet,
            z_true=None, cfg: QuadratureConfig = DEFAULT_CONFIG, device="cuda"):
    """Kriging mean at test_locs; returns (predictions, mspe or None)."""
    torch = _torch()
    L = _cholesky(train.locs, theta, cfg, device)
    z = torch.from_numpy(train.z).to(L.device).unsqueeze(1)
    alpha = torch.cholesky_solve(z, L)
    spec = TileSpec(0, 0, len(test_locs), len(train.locs))
    k = generate_tile(spec, torch.from_numpy(test_locs.coords).to(L.device),
                      torch.from_numpy(train.locs.coords).to(L.device), theta, cfg)
    pred = (k @ alpha).squeeze(1).cpu().numpy()
    mspe = None if z_true is None else float(np.mean((pred - np.asarray(z_true)) ** 2))
    return pred, mspe


def fit_mle(obs: Observations, start: MaternParams = MLE_START, bounds=MLE_BOUNDS,
            cfg: QuadratureConfig = DEFAULT_CONFIG, device="cuda", max_evals: int = 1000,
            ftol: float = 1e-6) -> FitResult:
    """Maximise log_likelihood over log(theta) inside the box with Nelder-Mead; every
    objective evaluation regenerates Sigma on the GPU."""
    from scipy.optimize import minimize

    lo = np.log([b[0] for b in bounds])
    hi = np.log([b[1] for b in bounds])
    trace = []

    def objective(v):
        v = np.clip(v, lo, hi)
        th = MaternParams(*np.exp(v))
        llh = log_likelihood(obs, th, cfg, device)
        trace.append((th.sigma_sq, th.beta, th.nu, llh))
        return -llh if math.isfinite(llh) else 1e300

    x0 = np.clip(np.log([start.sigma_sq, start.beta, start.nu]), lo, hi)
    res = minimize(objective, x0, method="Nelder-Mead",
                   options={"maxfev": max_evals, "fatol": ftol, "xatol": 1e-8})
    best = min(trace, key=lambda t: -t[3])
    return FitResult(MaternParams(*best[:3]), best[3], len(trace), bool(res.success), trace)
