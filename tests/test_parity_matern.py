"""GPU parity of the Matern kernels (bgk_matern_tile / _covariance / _lower_tiles)
against the reference (golden matern_tile fixtures) and the CPU oracle.

Tolerance: max relative error <= 1e-10 per entry (BASELINE.json north_star);
layouts, mirroring, sharding and tile packing are checked BITWISE (entries are
pure functions of the location pair).
"""

import numpy as np
import pytest

from conftest import rel_err

pytestmark = pytest.mark.gpu

TOL = 1e-10


@pytest.fixture(scope="module")
def bg():
    import paper_2502_00356_b200 as bg

    return bg


def _golden_keys(g):
    return [k for k in g.files if k.startswith("nu") and k.count("_") == 1]


def test_golden_tiles_via_matern_tile(bg, golden):
    """bg.matern_tile with the reference's exact argument list vs kernels.matern_tile."""
    import torch

    g = golden("matern")
    locs = g["locs"]
    for key in _golden_keys(g):
        nu = float(key.split("_")[0][2:])
        beta = float(key.split("_")[1][4:])
        out = torch.empty((locs.shape[0], locs.shape[0]), dtype=torch.float64, device="cuda")
        bg.matern_tile(out, locs[:, 0], locs[:, 1], locs[:, 0], locs[:, 1],
                       float(g[key + "_s2"][0]), beta, nu, float(g[key + "_lp"][0]),
                       g[key + "_c"], g[key + "_a"], 9.0 / 40, 0.1, 2.0 ** -52, 15000)
        got = out.cpu().numpy()
        assert np.max(rel_err(got, g[key])) <= TOL, key
        # zero distance (diagonal and the duplicated location 7 == 3) gives sigma^2 exactly
        s2 = float(g[key + "_s2"][0])
        assert np.all(np.diag(got) == s2) and got[7, 3] == s2 and got[3, 7] == s2


def test_golden_tiles_via_generate_covariance(bg, golden):
    g = golden("matern")
    locs = g["locs"]
    for key in _golden_keys(g):
        nu = float(key.split("_")[0][2:])
        beta = float(key.split("_")[1][4:])
        theta = bg.MaternParams(float(g[key + "_s2"][0]), beta, nu)
        cov = bg.generate_covariance(locs, theta, device="cuda").to_numpy()
        assert np.max(rel_err(cov, g[key])) <= TOL, key
        assert np.array_equal(cov, cov.T)


@pytest.mark.parametrize("nu", [0.3, 0.8, 1.5, 1.7, 2.9, 0.5, 5.3, 19.5])
def test_covariance_vs_oracle(bg, oracle, nu):
    rng = np.random.default_rng(int(nu * 10))
    N = 700
    locs = rng.random((N, 2))
    locs[5] = locs[4] + 1e-3  # u = 0.014 < threshold: Temme branch
    theta = bg.MaternParams(1.3, 0.1, nu)
    cov = bg.generate_covariance(locs, theta, device="cuda").to_numpy()
    ref = oracle.generate_covariance(locs, 1.3, 0.1, nu, threads=8)
    assert np.max(rel_err(cov, ref)) <= TOL
    assert np.array_equal(cov, cov.T)
    assert np.all(np.diag(cov) == 1.3)


def test_m10_config_sample_vs_oracle(bg, oracle):
    """Rows of the M10 config (N=10K, nu=1.5, beta=0.1) against the oracle."""
    rng = np.random.default_rng(20250201)
    N = 10_000
    locs = rng.random((N, 2))
    theta = bg.MaternParams(1.0, 0.1, 1.5)
    cov = bg.generate_covariance(locs, theta, device="cuda")
    full = cov.data
    rows = [0, 1, 63, 64, 65, 4999, 5000, 9935, 9999]
    got = full[rows].cpu().numpy()
    ref = np.stack([oracle.generate_covariance(locs, 1.0, 0.1, 1.5, row_range=(r, r + 1),
                                               threads=8)[0] for r in rows])
    assert np.max(rel_err(got, ref)) <= TOL
    # symmetry of the whole device matrix, bitwise
    import torch

    assert bool(torch.equal(full, full.T))


def test_row_shards_union_bitwise(bg):
    """Union of G row-block shards == the 1-GPU full matrix, bitwise."""
    import torch

    rng = np.random.default_rng(11)
    N = 1000
    locs = rng.random((N, 2))
    theta = bg.MaternParams(1.0, 0.07, 1.7)
    full = bg.generate_covariance(locs, theta, device="cuda").data
    for G in (2, 3, 8):
        bounds = [N * g // G for g in range(G + 1)]
        parts = [bg.generate_covariance(locs, theta, device="cuda",
                                        rows=(bounds[g], bounds[g + 1])).data for g in range(G)]
        assert torch.equal(torch.cat(parts, 0), full)
    # odd, unaligned row range
    part = bg.generate_covariance(locs, theta, device="cuda", rows=(37, 611)).data
    assert torch.equal(part, full[37:611])


def test_host_output_blocks_bitwise(bg):
    rng = np.random.default_rng(12)
    N = 900
    locs = rng.random((N, 2))
    theta = bg.MaternParams(2.0, 0.2, 0.8)
    dev = bg.generate_covariance(locs, theta, device="cuda").to_numpy()
    host = bg.generate_covariance(locs, theta, host_block_bytes=64 * 8 * N).data
    assert isinstance(host, np.ndarray) and np.array_equal(host, dev)
    pinned = bg.empty_host_matrix(N, N)
    bg.generate_covariance(locs, theta, out=pinned)
    assert np.array_equal(pinned, dev)


@pytest.mark.parametrize("direct", [None, 0, 3])
@pytest.mark.parametrize("N,blk", [(4096, 64), (5003, 640), (4500, 1 << 30)])
def test_host_lower_mirrored_path_bitwise(bg, N, blk, direct, monkeypatch):
    # page-locked full-matrix output: only the lower triangle crosses PCIe and the
    # host mirrors it (covariance._full_host_lower_mirrored); must equal the device
    # matrix bit for bit, whatever the block size
    from paper_2502_00356_b200 import covariance as C

    assert N >= C._MIRROR_MIN_N
    monkeypatch.setattr(C, "_MIRROR_DIRECT", direct)  # upper blocks sent directly
    rng = np.random.default_rng(N)
    locs = rng.random((N, 2))
    locs[7] = locs[3]  # a duplicate location off the diagonal
    theta = bg.MaternParams(1.0, 0.1, 1.5)
    dev = bg.generate_covariance(locs, theta, device="cuda").to_numpy()
    pinned = bg.empty_host_matrix(N, N)
    pinned.fill(np.nan)
    bg.generate_covariance(locs, theta, out=pinned, host_block_bytes=blk * 8 * N)
    assert np.array_equal(pinned, dev)


@pytest.mark.parametrize("ts", [1, 7, 64, 100, 256])
def test_lower_tiles_layout_bitwise(bg, ts):
    rng = np.random.default_rng(13)
    N = 333
    locs = rng.random((N, 2))
    theta = bg.MaternParams(1.0, 0.1, 1.5)
    full = bg.generate_covariance(locs, theta, device="cuda").to_numpy()
    packed = bg.generate_covariance(locs, theta, tile_size=ts, layout="lower_tiles",
                                    device="cuda")
    T = -(-N // ts)
    assert packed.data.shape[0] == T * (T + 1) // 2
    for p in range(T):
        for q in range(p + 1):
            t = packed.tile(p, q)
            assert np.array_equal(t, full[p * ts:p * ts + t.shape[0], q * ts:q * ts + t.shape[1]])
    # a shard of the packed tile range
    l0, l1 = 3, min(T * (T + 1) // 2, 11)
    shard = bg.generate_covariance(locs, theta, tile_size=ts, layout="lower_tiles",
                                   device="cuda", tiles=(l0, l1)).to_numpy()
    assert np.array_equal(shard, packed.to_numpy()[l0:l1])


def test_generate_tile_layouts_and_scalar_equivalence(bg):
    rng = np.random.default_rng(14)
    rows = rng.random((37, 2))
    cols = rng.random((91, 2))
    theta = bg.MaternParams(1.0, 0.1, 1.5)
    spec = bg.TileSpec(0, 0, 37, 91)
    t_row = bg.generate_tile(spec, rows, cols, theta)
    t_col = bg.generate_tile(spec, rows, cols, theta, layout="col")
    assert t_col.flags.f_contiguous and np.array_equal(t_row, t_col)
    d = np.sqrt((rows[:, None, 0] - cols[None, :, 0]) ** 2 + (rows[:, None, 1] - cols[None, :, 1]) ** 2)
    # entrywise scalar construction through matern(r) -- bitwise
    flat = bg.matern_batch(d.ravel(), theta).reshape(d.shape)
    assert np.array_equal(flat, t_row)
    assert bg.matern(float(d[3, 5]), theta) == t_row[3, 5]
    assert bg.matern(0.0, theta) == 1.0


def test_matern_closed_form_nu_half(bg):
    """nu = 1/2: Sigma = sigma^2 exp(-r/beta) (<= 1e-7)."""
    rng = np.random.default_rng(15)
    locs = rng.random((400, 2))
    theta = bg.MaternParams(1.0, 0.1, 0.5)
    cov = bg.generate_covariance(locs, theta, device="cuda").to_numpy()
    d = np.sqrt(((locs[:, None, :] - locs[None, :, :]) ** 2).sum(-1))
    assert np.max(np.abs(cov - np.exp(-d / 0.1))) <= 1e-7
    # Cholesky succeeds (positive definite at desk scale)
    np.linalg.cholesky(cov)


def test_col_major_is_transpose(bg):
    import ctypes

    import torch

    from paper_2502_00356_b200 import _lib
    from paper_2502_00356_b200.covariance import _coords, matern_plan

    rng = np.random.default_rng(16)
    N = 300
    locs = rng.random((N, 2))
    theta = bg.MaternParams(1.0, 0.1, 2.9)
    full = bg.generate_covariance(locs, theta, device="cuda").data
    lx, ly = _coords(locs)
    r0, r1 = 45, 199
    out = torch.empty((N, r1 - r0), dtype=torch.float64, device="cuda")  # column block
    L = _lib.lib()
    plan = matern_plan(theta)
    rc = L.bgk_matern_covariance(ctypes.byref(plan), lx.data_ptr(), ly.data_ptr(), N, r0, r1,
                                 out.data_ptr(), r1 - r0, _lib.LAYOUT_COL_MAJOR,
                                 torch.cuda.current_stream().cuda_stream)
    _lib.check(rc, "cov col-major")
    assert torch.equal(out, full[:, r0:r1])


def test_nondefault_config_and_large_beta(bg, oracle):
    """bins=16 / t_upper=7 / a large range beta (all entries in the series branch)."""
    rng = np.random.default_rng(17)
    locs = rng.random((200, 2))
    for cfg_kw, beta in (({"bins": 16}, 0.1), ({"t_upper": 7.0}, 0.05), ({}, 50.0),
                         ({"small_x_threshold": 0.5}, 0.1)):
        cfg = bg.QuadratureConfig(**cfg_kw)
        theta = bg.MaternParams(1.0, beta, 1.2)
        cov = bg.generate_covariance(locs, theta, cfg, device="cuda").to_numpy()
        ref = oracle.generate_covariance(locs, 1.0, beta, 1.2, t0=cfg.t_lower, t1=cfg.t_upper,
                                         bins=cfg.bins, thr=cfg.small_x_threshold)
        assert np.max(rel_err(cov, ref)) <= TOL, cfg_kw


def test_sqrt_rn_fast(bg):
    """The classify pass's branch-free sqrt equals __dsqrt_rn bit for bit wherever it
    claims its range: random squared distances of the bench configs, random binades
    across the whole claimed range, and exact squares / perfect-square neighbours."""
    import torch

    from paper_2502_00356_b200 import _lib

    rng = np.random.default_rng(7)
    d = rng.random((1 << 20, 2)) - rng.random((1 << 20, 2))
    parts = [
        (d * d).sum(1),                                   # unit-square squared distances
        ((d * 1e3) ** 2).sum(1),                          # large coordinates
        np.ldexp(1.0 + rng.random(1 << 21), rng.integers(-960, 1020, 1 << 21)),
        np.arange(1, 1 << 20, dtype=np.float64) ** 2,     # exact squares
        np.nextafter(np.arange(1, 1 << 18, dtype=np.float64) ** 2, np.inf),
        np.nextafter(np.arange(1, 1 << 18, dtype=np.float64) ** 2, 0.0),
    ]
    x = torch.from_numpy(np.concatenate(parts)).cuda()
    fast = torch.empty_like(x)
    ref = torch.empty_like(x)
    _lib.check(_lib.lib().bgk_sqrt_rn_check(x.data_ptr(), x.numel(), fast.data_ptr(),
                                            ref.data_ptr(), None), "bgk_sqrt_rn_check")
    torch.cuda.synchronize()
    claimed = ~torch.isnan(fast)
    assert claimed.float().mean().item() > 0.99
    assert torch.equal(fast[claimed].view(torch.int64), ref[claimed].view(torch.int64))
    assert np.array_equal(ref.cpu().numpy().view(np.int64), np.sqrt(x.cpu().numpy()).view(np.int64))


@pytest.mark.parametrize("nu", [0.5, 1.0, 1.5, 2.5, 7.5])
def test_pow_mode_matches_general_power(bg, oracle, nu):
    """Half-integer / integer nu plans take u^nu = u^k sqrt(u)^half (pow_mode); the same
    plan with pow_mode cleared takes exp(nu ln u).  Both agree to rounding and both
    match the oracle; the three kernel paths of a plan (fast group, per-lane, mirror)
    stay bitwise symmetric."""
    import ctypes

    import torch

    from paper_2502_00356_b200 import _lib
    from paper_2502_00356_b200.covariance import _cov_launch, matern_plan

    rng = np.random.default_rng(11)
    N = 700
    locs = rng.random((N, 2))
    theta = bg.MaternParams(1.7, 0.1, nu)
    plan = matern_plan(theta)
    assert plan.pow_mode != 0
    general = _lib.BgkMaternPlan()
    ctypes.memmove(ctypes.byref(general), ctypes.byref(plan), ctypes.sizeof(plan))
    general.pow_mode = 0
    lxy = torch.from_numpy(np.ascontiguousarray(locs.T)).cuda()
    outs = []
    for p in (plan, general):
        out = torch.empty((N, N), dtype=torch.float64, device="cuda")
        _cov_launch(p, lxy[0], lxy[1], N, 0, N, out, N, _lib.LAYOUT_ROW_MAJOR)
        outs.append(out.cpu().numpy())
    fast, gen = outs
    assert np.array_equal(fast, fast.T) and np.array_equal(gen, gen.T)
    assert np.max(rel_err(fast, gen)) <= 1e-13
    ref = oracle.generate_covariance(locs, 1.7, 0.1, nu)
    assert np.max(rel_err(fast, ref)) <= TOL


def test_concurrent_streams_bitwise(bg):
    # re-entrancy: launches on two streams at once (persistent kernels with task
    # counters per stream) give the same matrices as one after the other
    import torch

    rng = np.random.default_rng(33)
    locs_a, locs_b = rng.random((3000, 2)), rng.random((2500, 2))
    th_a, th_b = bg.MaternParams(1.0, 0.1, 1.5), bg.MaternParams(2.0, 0.05, 0.8)
    ref_a = bg.generate_covariance(locs_a, th_a, device="cuda").data.clone()
    ref_b = bg.generate_covariance(locs_b, th_b, device="cuda").data.clone()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    torch.cuda.synchronize()
    with torch.cuda.stream(s1):
        a = bg.generate_covariance(locs_a, th_a, device="cuda").data
    with torch.cuda.stream(s2):
        b = bg.generate_covariance(locs_b, th_b, device="cuda").data
    torch.cuda.synchronize()
    assert torch.equal(a, ref_a) and torch.equal(b, ref_b)
