"""Pin the CPU oracle (oracle/fqf_oracle.c) to the reference's golden vectors.

The goldens come from the reference's own sources (oracle/_ref) and LAPACK;
see tests/golden/make_golden.py.  These run without a GPU.
"""
import numpy as np
import pytest

from oracle import oracle as O
from tests.golden_io import DAS_CASES, das_kwargs, load, rel_l2, rel_max


@pytest.mark.parametrize("name", DAS_CASES)
def test_oracle_das_matches_reference(name):
    meta, a = load(name)
    iq, oow = O.das(a["rf"], meta["fs"], meta["t0"], meta["angles"], a["elements"], meta["dims"],
                    meta["spacing"], meta["origin"], **das_kwargs(meta))
    # The restatement follows das_reconstruct's arithmetic order, so it agrees
    # to the last bits; 1e-12 is the reference's own bound
    # (test_beamform.cpp:385-424).
    assert rel_max(iq, a["iq"]) < 1e-12
    assert oow == meta["stats"]["out_of_window"]


def test_kat_golden_values():
    meta, a = load("das_kat")
    iq, _ = O.das(a["rf"], meta["fs"], meta["t0"], meta["angles"], a["elements"], meta["dims"],
                  meta["spacing"], meta["origin"], **das_kwargs(meta))
    # IQ[frame 0][voxel 0] and IQ[frame 1][voxel 0] of the
    # test_beamform.cpp:385-424 fixture, from the reference build.
    assert abs(iq[0, 0] - complex(0.21767054125126079, -0.23091352539589127)) < 1e-15
    assert abs(iq[1, 0] - complex(-0.2515352884279673, 0.01450684879472558)) < 1e-15


@pytest.mark.parametrize("name", ["demod_random", "demod_t0"])
def test_oracle_demod_matches_reference(name):
    meta, a = load(name)
    iq = O.rf_to_iq(a["rf"], meta["fs"], meta["t0"], meta["fc"], meta["taps"])
    assert np.array_equal(iq, a["iq"])  # same FP64 operations, same order


def test_oracle_demod_tone():
    # test_beamform.cpp:191-219: a tone at f_c demodulates to unit magnitude.
    fc, fs, T = 5e6, 20e6, 400
    t = np.arange(T) / fs
    rf = np.stack([np.cos(2 * np.pi * fc * t), np.cos(2 * np.pi * fc * t + np.pi / 3)], axis=1)
    iq = O.rf_to_iq(rf, fs, 0.0, fc)
    assert np.all(np.abs(iq[40:-40, 0] - 1.0) < 0.01)
    assert np.all(np.abs(iq[40:-40, 1] - np.exp(1j * np.pi / 3)) < 0.01)


def test_oracle_demod_rejects():
    rf = np.zeros((64, 1))
    with pytest.raises(O.OracleError):
        O.rf_to_iq(rf, 19e6, 0.0, 9.5e6)
    with pytest.raises(O.OracleError):
        O.rf_to_iq(rf, 20e6, 0.0, 5e6, 32)


def test_oracle_plan_chunks_matches_reference():
    meta, _ = load("plan_chunks")
    for case, plan in zip(meta["cases"], meta["plans"]):
        assert O.plan_chunks(*case) == [tuple(r) for r in plan]
    with pytest.raises(O.OracleError):
        O.plan_chunks(100, 5, 80)


def test_oracle_power_doppler():
    meta, a = load("pd_random")
    assert np.array_equal(O.power_doppler(a["iq"]), a["pd"])
    # test_post.cpp:283-316: unit phasors sum to exactly F.
    lattice = np.array([1, 1j, -1, -1j])
    iq = np.array([[lattice[(f + v) % 4] for v in range(30)] for f in range(100)])
    assert np.all(O.power_doppler(iq) == 100.0)
    assert np.all(O.power_doppler(2 * iq) == 400.0)


def _fro(x):
    return np.sqrt(np.sum(np.abs(x) ** 2))


@pytest.mark.parametrize("method", ["jacobi", "gram"])
def test_oracle_svd_static(method):
    meta, a = load("svd_static")
    x = a["iq"]
    F = x.shape[0]
    y, s, _ = O.svd_filter(x, 2, F, method=method)
    scale = _fro(x)
    assert abs(s[0] - scale) <= 1e-12 * scale
    if method == "jacobi":  # test_post.cpp:135-162 bounds hold for the SVD route
        assert _fro(y) <= 1e-9 * scale
        assert np.all(s[1:] <= 1e-9 * s[0])
    else:  # the Gram route squares the condition number: sqrt(eps) floor
        assert _fro(y) <= 1e-7 * scale
    y1, _, _ = O.svd_filter(x, 1, F, method=method)
    assert _fro(y1 - x) <= 1e-9 * scale


@pytest.mark.parametrize("method", ["jacobi", "gram"])
def test_oracle_svd_bands_match_lapack(method):
    meta, a = load("svd_bands")
    x = a["iq"]
    F = x.shape[0]
    y13, s, _ = O.svd_filter(x, 1, 3, method=method)
    y4, _, _ = O.svd_filter(x, 4, F, method=method)
    y25, _, _ = O.svd_filter(x, 2, 5, method=method)
    assert np.allclose(s, a["sigma"], rtol=1e-12, atol=0)
    assert abs(np.sum(s ** 2) - np.sum(np.abs(x) ** 2)) <= 1e-9 * np.sum(np.abs(x) ** 2)
    assert np.all(np.diff(s) <= 0) and np.all(s >= 0)
    assert rel_l2(y13, a["band13"]) < 1e-11
    assert rel_l2(y4, a["band4F"]) < 1e-11
    assert rel_l2(y25, a["band25"]) < 1e-11
    assert _fro(y13 + y4 - x) <= 1e-9 * _fro(x)


def test_oracle_svd_correlation_matches_lapack():
    meta, a = load("svd_corr")
    _, s, corr = O.svd_filter(a["iq"], 1, a["iq"].shape[0], want_corr=True)
    assert np.allclose(corr, corr.T, atol=1e-12)
    assert np.allclose(np.diag(corr), 1.0, atol=1e-12)
    assert np.all(np.abs(corr) <= 1 + 1e-12)
    assert np.allclose(corr, a["corr"], atol=1e-9)


@pytest.mark.parametrize("method", ["jacobi", "gram"])
def test_oracle_svd_vessel_fraction(method):
    meta, a = load("svd_vessel")
    x, vessel = a["iq"], a["vessel"]
    y, _, _ = O.svd_filter(x, 2, x.shape[0], method=method)
    assert rel_l2(y, a["band2"]) < 1e-9
    frac = lambda pd: pd[vessel].sum() / pd.sum()  # noqa: E731
    before, after = frac(O.power_doppler(x)), frac(O.power_doppler(y))
    assert before < 0.3 and after > 0.9  # test_post.cpp:220-251


def test_oracle_svd_rejects():
    x = np.array([[complex(f + 1, v) for v in range(16)] for f in range(3)])
    for lo, hi in [(0, 2), (1, 4), (3, 2)]:
        with pytest.raises(O.OracleError):
            O.svd_filter(x, lo, hi)
    with pytest.raises(O.OracleError):
        O.svd_filter(np.zeros((3, 16), complex), 1, 3)
    with pytest.raises(O.OracleError):
        O.svd_filter(np.ones((3, 2), complex), 1, 3)  # more frames than voxels


def test_oracle_heev_reconstructs():
    rng = np.random.default_rng(5)
    m = rng.standard_normal((12, 12)) + 1j * rng.standard_normal((12, 12))
    h = m @ m.conj().T
    w, v = O.heev(h.copy())
    assert np.allclose(v @ np.diag(w) @ v.conj().T, h, atol=1e-10 * np.abs(h).max())
    assert np.allclose(w, np.sort(np.linalg.eigvalsh(h))[::-1], rtol=1e-11)


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_ref_library_matches_its_goldens():
    meta, a = load("das_kat")
    iq, st = O.ref_das(a["rf"], meta["fs"], meta["t0"], meta["angles"], a["elements"],
                       meta["dims"], meta["spacing"], meta["origin"], fc=meta["fc"],
                       memory_budget=meta["memory_budget"])
    assert np.array_equal(iq, a["iq"])
    assert st == meta["stats"]


@pytest.mark.parametrize("name", ["linear2d", "matrix3d"])
def test_phantom_reference_chain_finds_the_vessel(name):
    # The SVD filter separates moving tissue from blood on the phantom
    # (cf. test_post.cpp:220-251): PD is concentrated inside the vessel.
    from tests import phantom_cases as PC
    pd, m, _ = PC.reference(name)
    c, ph = PC.case(name), PC.phantom(name)
    g = c.grid
    gt = O.ref_ground_truth_pd(ph.blood, g.dims, g.spacing, g.origin, PC.GT_SIGMA)
    inside, outside = pd[gt > 0.3].mean(), pd[gt < 0.01].mean()
    assert inside > 8 * outside
    assert np.isfinite(m["psnr"]) and -1 < m["ssim"] < 1


# ---------------------------------------------- RF synthesis (rf/simulate.cpp)

def _small_probe(n, v, fc, bw):
    """test_rf.cpp:31-43."""
    import paper_2509_05464_b200 as P
    el = np.array([[(i - (n - 1) / 2.0) * 0.4e-3, 0.0, 0.0] for i in range(n)])
    return P.Transducer(el, "test", 0.4e-3, fc, half_width=0.15e-3, subelements=v,
                        fractional_bandwidth=bw)


def _rel(a, b):
    return np.abs(a - b).max() / max(np.abs(a).max(), np.abs(b).max())


RF_CLOUD = (np.array([[1.0e-3, 0.3e-3, 8.0e-3], [-0.7e-3, 0.0, 11.0e-3], [0.2e-3, -0.2e-3, 9.5e-3]]),
            np.array([1.0, -0.7, 0.35]))


def test_oracle_rf_engine_matches_literal_reference():
    # test_rf.cpp:229-261: the banded-recurrence engine equals the literal
    # per-frequency synthesis to 1e-12.
    import paper_2509_05464_b200 as P
    td = _small_probe(3, 2, 5e6, 0.5)
    tx = P.plane_wave_delays(td, 3.0 * np.pi / 180.0, 1540.0)
    apod = np.array([1.0, 0.8, 1.2])
    pos, refl = RF_CLOUD
    eng = O.simulate_rf(pos, refl, td, tx.delays, apod, att=0.7, fs=20e6, duration=20e-6)
    lit = O.reference_rf(pos, refl, td, tx.delays, apod, att=0.7, fs=20e6, duration=20e-6)
    assert eng.shape == (400, 3)
    assert _rel(eng, lit) < 1e-12
    T, lo, hi, df = O.rf_passband(td, 20e6, 20e-6)
    sigma = 0.5 * 0.5 * 5e6 / np.sqrt(2 * np.log(2))
    span = np.sqrt(4 * np.log(10)) * sigma
    assert (lo, hi) == (max(1, int(np.ceil((5e6 - span) / df))),
                        min((T - 1) // 2, int(np.floor((5e6 + span) / df))))


def test_oracle_rf_elevation_within_knot_interpolation_error():
    # test_rf.cpp:263-291
    import paper_2509_05464_b200 as P
    td = _small_probe(3, 2, 5e6, 0.5)
    td.elevation_height, td.elevation_focus = 4.0e-3, 12.0e-3
    tx = P.plane_wave_delays(td, 0.0, 1540.0)
    pos = np.array([[1.0e-3, 0.5e-3, 8.0e-3], [-0.7e-3, -0.8e-3, 11.0e-3], [0.2e-3, 0.0, 9.5e-3]])
    refl = RF_CLOUD[1]
    eng = O.simulate_rf(pos, refl, td, tx.delays, tx.apodization)
    lit = O.reference_rf(pos, refl, td, tx.delays, tx.apodization)
    assert _rel(eng, lit) < 2e-3
    on = O.simulate_rf([[0.0, 0.0, 12e-3]], [1.0], td, tx.delays, tx.apodization)
    off = O.simulate_rf([[0.0, 1.5e-3, 12e-3]], [1.0], td, tx.delays, tx.apodization)
    assert np.abs(off).max() < 0.5 * np.abs(on).max()


def test_oracle_rf_blocks_and_linearity():
    # test_rf.cpp:312-386: doubling reflectivity doubles every sample
    # exactly; block partitioning leaves the frame unchanged.
    import paper_2509_05464_b200 as P
    td = _small_probe(4, 3, 5e6, 0.6)
    tx = P.plane_wave_delays(td, -2.0 * np.pi / 180.0, 1540.0)
    rng = np.random.default_rng(3)
    pos = np.stack([rng.uniform(-2e-3, 2e-3, 9), rng.uniform(-1e-3, 1e-3, 9),
                    rng.uniform(6e-3, 14e-3, 9)], axis=1)
    refl = rng.standard_normal(9)
    a = O.simulate_rf(pos, refl, td, tx.delays, tx.apodization)
    b = O.simulate_rf(pos, 2 * refl, td, tx.delays, tx.apodization)
    assert np.array_equal(2 * a, b)
    for blk in (1, 4):
        c = O.simulate_rf(pos, refl, td, tx.delays, tx.apodization, block_scatterers=blk)
        assert _rel(a, c) < 1e-12


# ------------------------------------------- RF synthesis vs the reference --

@pytest.mark.parametrize("name", ["rfsim_small", "rfsim_lens", "rfsim_matrix"])
def test_rfsim_restatement_matches_reference_simulator(name):
    """fqf_rfsim.c (the engine restatement) against the reference's own
    simulate_rf (simulate.cpp compiled with oracle/fftw_stub; fixtures in
    tests/golden/rfsim_*.npz from tests/golden/make_golden_rf.py)."""
    from tests.golden_io import load
    from tests.rf_cases import case_inputs
    meta, a = load(name)
    _, td, tx, inp = case_inputs(name)
    med = meta["medium"]
    got = O.simulate_rf(inp["positions"], inp["reflectivity"], td, tx.delays, tx.apodization,
                        c=med["c"], att=med["att"], fs=meta["fs"], duration=meta["duration"])
    ref = a["rf"]
    assert got.shape == ref.shape
    assert np.abs(got - ref).max() / np.abs(ref).max() < 1e-12
