"""GPU parity: the CUDA path (through the C ABI) against the reference's golden
vectors and the CPU oracle.  Runs on a B200 (``-m gpu``).

Tolerances (stated once, used below):
  IQ_REL_L2  = 1e-5  DAS / demod output vs FP64 reference (f32 IQ and
                     accumulation against the reference's FP64)
  IQ_REL_MAX = 1e-4  worst single voxel, relative to the volume's peak
  PD_REL_L2  = 1e-4  filtered power Doppler vs the FP64 restatement
  SIG_REL    = 1e-5  singular values from the FP64 Gram eigensolve
"""
import math

import numpy as np
import pytest

import paper_2509_05464_b200 as P
from oracle import oracle as O
from paper_2509_05464_b200 import workloads as W
from tests.golden_io import DAS_CASES, das_kwargs, load, rel_l2, rel_max

pytestmark = pytest.mark.gpu

IQ_REL_L2 = 1e-5
IQ_REL_MAX = 1e-4
PD_REL_L2 = 1e-4
SIG_REL = 1e-5


def gpu_das(meta, a, **over):
    kw = das_kwargs(meta)
    kw.update(over)
    bp = P.BeamformParams(c=kw["c"], center_frequency=kw["fc"], f_number=kw["f_number"],
                          interp_order=kw["interp_order"], lowpass_taps=kw["lowpass_taps"])
    opts = P.DasOptions(memory_budget_bytes=meta.get("memory_budget", 100_000_000),
                        matrix_budget_bytes=meta.get("matrix_budget", 512_000_000),
                        cache_matrices=meta.get("cache", True))
    grid = P.GridSpec(tuple(meta["dims"]), tuple(meta["spacing"]), tuple(meta["origin"]))
    return P.das_reconstruct_array(a["rf"], meta["fs"], meta["t0"], meta["angles"], grid,
                                   a["elements"], bp, opts, want_stats=True)


# ------------------------------------------------------------------ demod --

@pytest.mark.parametrize("name", ["demod_random", "demod_t0"])
def test_demod_matches_reference(name):
    meta, a = load(name)
    T, E = a["rf"].shape
    fr = P.RfFrame(a["rf"], meta["fs"], meta["t0"])
    iq = P.rf_to_iq(fr, meta["fc"], meta["taps"])
    assert iq.samples.shape == (T, E)
    assert rel_l2(iq.samples, a["iq"]) < IQ_REL_L2
    assert rel_max(iq.samples, a["iq"]) < IQ_REL_MAX


def test_demod_tone_and_rejections():
    fc, fs, T = 5e6, 20e6, 400
    t = np.arange(T) / fs
    rf = np.stack([np.cos(2 * np.pi * fc * t), np.cos(2 * np.pi * fc * t + np.pi / 3)], 1)
    iq = P.rf_to_iq(P.RfFrame(rf, fs), fc).samples
    assert np.all(np.abs(iq[40:-40, 0] - 1.0) < 0.01)  # test_beamform.cpp:191-219
    assert np.all(np.abs(iq[40:-40, 1] - np.exp(1j * np.pi / 3)) < 0.01)
    z = P.RfFrame(np.zeros((64, 1)), 19e6)
    for fcx, taps in [(9.5e6, 33), (0.0, 33), (5e6, 32), (5e6, 1)]:
        with pytest.raises(P.Error):
            P.rf_to_iq(z, fcx, taps)


def test_demod_linear_power_of_two_bitwise():
    meta, a = load("demod_random")
    one = P.rf_to_iq(P.RfFrame(a["rf"], 20e6), 5e6).samples
    two = P.rf_to_iq(P.RfFrame(2 * a["rf"], 20e6), 5e6).samples
    assert np.array_equal(two, 2 * one)  # test_beamform.cpp:238-243, exact in f32 too


# -------------------------------------------------------------------- DAS --

# DAS kernels (read at plan creation): the tensor-core default (das_tc) for
# the fixture's frame count and at 112 frames per pass (FQFG_DAS_SHAPE sets
# J), and das2 (FQFG_DAS_TC=0) with its default shape and the config-C shape
# (208 frames per pass, 16 + 8 warps, tile 4 x 8 x 2).
KERNEL_SHAPES = {"tc": {}, "tc-112": {"FQFG_DAS_SHAPE": "7,4,16,8"},
                 "das2": {"FQFG_DAS_TC": "0"},
                 "das2-c-shape": {"FQFG_DAS_TC": "0", "FQFG_DAS_SHAPE": "13,2,16,8,4,8,2"}}


def _kernel_env(monkeypatch, kernel):
    for k, v in KERNEL_SHAPES[kernel].items():
        monkeypatch.setenv(k, v)


@pytest.mark.parametrize("kernel", list(KERNEL_SHAPES))
@pytest.mark.parametrize("name", DAS_CASES)
def test_das_matches_reference(name, kernel, monkeypatch):
    """Every golden DAS fixture (the reference's own outputs): IQ within the
    f32 tolerance and DasStats exact, for the tensor-core default and das2
    (default and config-C production shape)."""
    _kernel_env(monkeypatch, kernel)
    meta, a = load(name)
    iq, st = gpu_das(meta, a)
    ref = a["iq"]
    assert iq.shape == ref.shape
    assert rel_l2(iq, ref) < IQ_REL_L2, name
    assert rel_max(iq, ref) < IQ_REL_MAX, name
    # DasStats parity (das.hpp:110-116): exact, the reference's own semantics.
    assert st.__dict__ == meta["stats"], (st.__dict__, meta["stats"])


def test_das_kat_golden_values():
    meta, a = load("das_kat")
    iq, _ = gpu_das(meta, a)
    scale = np.abs(a["iq"]).max()
    assert abs(iq[0, 0] - complex(0.21767054125126079, -0.23091352539589127)) < 1e-5 * scale
    assert abs(iq[1, 0] - complex(-0.2515352884279673, 0.01450684879472558)) < 1e-5 * scale


def test_das_partition_and_cache_invariance_bitwise():
    # test_beamform.cpp:426-462 / 520-558: the GPU path has no chunks; any
    # budget or caching choice must give the identical volume.
    meta, a = load("das_cached")
    base, _ = gpu_das(meta, a)
    n = int(np.prod(meta["dims"]))
    for budget in (16 * n * 2 * 4, 16 * 7 * 2):
        m = dict(meta, memory_budget=budget)
        iq, st = gpu_das(m, a)
        assert np.array_equal(iq, base)
    iq, st = gpu_das(dict(meta, cache=False), a)
    assert np.array_equal(iq, base)


def test_das_identical_transmits_mean():
    meta, a = load("das_identical")
    two, _ = gpu_das(meta, a)
    m1 = dict(meta, angles=meta["angles"][:1], t0=meta["t0"][:1])
    one, _ = gpu_das(m1, dict(a, rf=a["rf"][:, :1]))
    assert rel_max(two, one) < 1e-6


def test_das_linearity():
    meta, a = load("das_linearity")
    f1, f2 = a["rf"][0:1], a["rf"][1:2]
    v1, _ = gpu_das(meta, dict(a, rf=f1))
    v2, _ = gpu_das(meta, dict(a, rf=f2))
    vm, _ = gpu_das(meta, dict(a, rf=2 * f1 + f2))
    assert rel_max(vm, 2 * v1 + v2) < 1e-6  # reference bound 1e-9 in FP64


def test_das_power_of_two_exact_taps():
    # test_beamform.cpp:269-340: c = 1024, fs = 2^21, f_c = 2^18 put the echo
    # exactly on (40), half way (40.5) and past the recording.
    c, fs, fc = 1024.0, 2097152.0, 262144.0
    rng = np.random.default_rng(1)
    rf = rng.uniform(-1, 1, (1, 1, 128, 1))
    el = np.zeros((1, 3))
    for k, t0, interp in [(40.0, 0.0, 1), (40.5, 0.0, 1), (40.25, 0.0, 0), (200.0, 0.0, 1),
                          (40.0, 64.0 / fs, 1)]:
        z = k * c / (2.0 * fs)
        meta = dict(fs=fs, t0=[t0], angles=[0.0], dims=[1, 1, 1], spacing=[1e-3] * 3,
                    origin=[0.0, 0.0, z], fc=fc, c=c, f_number=0.0, interp_order=interp)
        iq, st = gpu_das(meta, dict(rf=rf, elements=el))
        ref, oow = O.das(rf, fs, [t0], [0.0], el, [1, 1, 1], [1e-3] * 3, [0.0, 0.0, z], c=c, fc=fc,
                         f_number=0.0, interp_order=interp)
        assert st.out_of_window == oow
        assert abs(iq[0, 0] - ref[0, 0]) <= 1e-6 * max(1.0, abs(ref[0, 0]))


def test_das_fnumber_aperture():
    # test_beamform.cpp:342-356: voxel at z = 3 mm, F# 1.5 -> half-aperture 1 mm.
    el = np.array([[0, 0, 0], [0.9e-3, 0, 0], [-0.9e-3, 0, 0], [1.1e-3, 0, 0], [-1.1e-3, 0, 0]])
    meta = dict(fs=20e6, t0=[0.0], angles=[0.0], dims=[1, 1, 1], spacing=[1e-4] * 3,
                origin=[0.0, 0.0, 3e-3], fc=5e6, f_number=1.5)
    for e, inside in enumerate([True, True, True, False, False]):
        rf = np.zeros((1, 1, 512, 5))
        rf[0, 0, :, e] = np.random.default_rng(e).uniform(-1, 1, 512)
        iq, _ = gpu_das(meta, dict(rf=rf, elements=el))
        assert (abs(iq[0, 0]) > 0) == inside


def test_das_rejections():
    meta, a = load("das_oow")
    with pytest.raises(P.Error):
        gpu_das(dict(meta, memory_budget=16), a)  # below one voxel row
    with pytest.raises(P.Error):
        gpu_das(dict(meta, dims=[0, 1, 1]), a)
    with pytest.raises(P.Error):
        gpu_das(dict(meta, fc=meta["fs"]), a)  # fs must exceed 2 f_c
    fr = P.RfFrame(np.zeros((32, 4)), 20e6, 0.0, P.TxEvent(0.0))
    other = P.RfFrame(np.zeros((32, 4)), 18e6, 0.0, P.TxEvent(0.0))
    td = P.Transducer(np.zeros((4, 3)))
    g = P.GridSpec((4, 1, 4), (2e-4,) * 3, (0, 0, 1e-3))
    bp = P.BeamformParams(center_frequency=5e6)
    with pytest.raises(P.Error):
        P.das_reconstruct([], g, td, bp)
    with pytest.raises(P.Error):
        P.das_reconstruct([[fr], [other]], g, td, bp)
    with pytest.raises(P.Error):
        P.das_reconstruct([[fr, fr], [fr]], g, td, bp)
    with pytest.raises(P.Error):
        P.das_reconstruct([[P.RfFrame(np.zeros((32, 3)), 20e6)]], g, td, bp)


def test_das_out_of_window_finite():
    meta, a = load("das_oow")
    iq, st = gpu_das(meta, a)
    assert st.out_of_window > 0 and np.all(np.isfinite(iq))


def test_das_matrix_probe_vs_oracle_large_window():
    # The small matrix-array workload (1024 elements, 3 angles, 20 frames):
    # several frames per lane-row and both f-number edges inside one tile.
    w = W.small()
    rng = np.random.default_rng(9)
    rf = rng.uniform(-1, 1, w.rf_shape()).astype(np.float32).astype(np.float64)
    g = w.grid
    iq, st = P.das_reconstruct_array(rf, w.fs, 0.0, w.angles, g, w.elements, w.bf(),
                                     want_stats=True)
    ref, oow = O.das(rf, w.fs, 0.0, w.angles, w.elements, g.dims, g.spacing, g.origin,
                     fc=w.fc)
    assert rel_l2(iq, ref) < IQ_REL_L2 and rel_max(iq, ref) < IQ_REL_MAX
    assert st.out_of_window == oow


@pytest.mark.parametrize("frames", [1, 17, 33, 100, 120, 209])
def test_das_frame_counts_vs_oracle(frames):
    # Every kernel instance (16*J frames per pass) and multi-pass splits.
    w = W.small()
    g = P.GridSpec((4, 3, 2), w.grid.spacing, w.grid.origin)
    rng = np.random.default_rng(frames)
    rf = rng.uniform(-1, 1, (frames, 1, w.n_samples, w.n_elements)).astype(np.float32)
    iq, _ = P.das_reconstruct_array(rf, w.fs, 0.0, [0.05], g, w.elements, w.bf())
    ref, _ = O.das(rf.astype(np.float64), w.fs, 0.0, [0.05], w.elements, g.dims, g.spacing,
                   g.origin, fc=w.fc)
    assert rel_l2(iq, ref) < IQ_REL_L2


def test_das_config_b_subgrid_vs_oracle():
    # Config B geometry (64^3 @ 0.2567 mm, 9 angles, T = 504) on a 10x8x3
    # sub-block at the deep corner, 2 frames.
    w = W.config("B")
    g0 = w.grid
    sp = g0.spacing
    g = P.GridSpec((10, 8, 3), sp, (g0.origin[0] + 40 * sp[0], g0.origin[1] + 50 * sp[1],
                                     g0.origin[2] + 60 * sp[2]))
    rng = np.random.default_rng(21)
    rf = rng.uniform(-1, 1, (2, w.n_angles, w.n_samples, w.n_elements)).astype(np.float32)
    iq, _ = P.das_reconstruct_array(rf, w.fs, 0.0, w.angles, g, w.elements, w.bf())
    ref, _ = O.das(rf.astype(np.float64), w.fs, 0.0, w.angles, w.elements, g.dims, g.spacing,
                   g.origin, fc=w.fc)
    assert rel_l2(iq, ref) < IQ_REL_L2 and rel_max(iq, ref) < IQ_REL_MAX


def test_das_files_roundtrip(tmp_path):
    meta, a = load("das_cached")
    el = a["elements"]
    frames = [[P.RfFrame(a["rf"][f, k], meta["fs"], meta["t0"][k], P.TxEvent(meta["angles"][k]))
               for k in range(a["rf"].shape[1])] for f in range(a["rf"].shape[0])]
    g = P.GridSpec(tuple(meta["dims"]), tuple(meta["spacing"]), tuple(meta["origin"]))
    opts = P.DasOptions(memory_budget_bytes=meta["memory_budget"], work_dir=str(tmp_path),
                        write_frames=True, keep_chunk_files=True)
    st = P.DasStats()
    vols = P.das_reconstruct(frames, g, P.Transducer(el), P.BeamformParams(center_frequency=5e6),
                             opts, st)
    assert st.chunks == 2
    for f in range(len(vols)):
        rd = P.read_iq_volume(str(tmp_path / f"Frame_{f + 1}.fqf"))
        assert rd.frame_index == f and rd.n_angles == 2 and np.array_equal(rd.values, vols[f].values)
    plan = P.plan_chunks(g.num_points(), 2, opts.memory_budget_bytes)
    again = P.assemble_frames(str(tmp_path), plan, g, len(vols))
    for f in range(len(vols)):
        assert np.array_equal(again[f].values, vols[f].values)
    (tmp_path / "IQ_CHUNK_2.fqf").unlink()
    with pytest.raises(P.Error, match="IQ_CHUNK_2"):
        P.assemble_frames(str(tmp_path), plan, g, len(vols))


# ------------------------------------------------------------ SVD filter --

def _vols(x, dims):
    g = P.GridSpec(tuple(dims), (1e-4,) * 3, (0, 0, 0))
    return [P.IqVolume(g, f, 1, x[f]) for f in range(x.shape[0])]


def test_svd_static_ensemble():
    meta, a = load("svd_static")
    x = a["iq"]
    F = x.shape[0]
    rep = P.SvdReport()
    high = P.svd_filter(_vols(x, meta["dims"]), 2, F, rep)
    scale = np.linalg.norm(x)
    assert abs(rep.singular_values[0] - scale) <= SIG_REL * scale
    assert np.linalg.norm(np.stack([v.values for v in high])) <= 1e-6 * scale
    assert rep.keep_lo == 2 and rep.keep_hi == F and rep.n_modes == F
    full = P.svd_filter(_vols(x, meta["dims"]), 1, F)
    assert rel_l2(np.stack([v.values for v in full]), x) < 1e-6


def test_svd_bands_match_lapack():
    meta, a = load("svd_bands")
    x = a["iq"]
    F = x.shape[0]
    rep = P.SvdReport()
    y13 = np.stack([v.values for v in P.svd_filter(_vols(x, meta["dims"]), 1, 3, rep)])
    y4 = np.stack([v.values for v in P.svd_filter(_vols(x, meta["dims"]), 4, F)])
    y25 = np.stack([v.values for v in P.svd_filter(_vols(x, meta["dims"]), 2, 5)])
    s = np.array(rep.singular_values)
    assert np.allclose(s, a["sigma"], rtol=SIG_REL)
    assert abs(np.sum(s ** 2) - np.sum(np.abs(x) ** 2)) <= 1e-6 * np.sum(np.abs(x) ** 2)
    assert rel_l2(y13, a["band13"]) < IQ_REL_L2
    assert rel_l2(y4, a["band4F"]) < IQ_REL_L2
    assert rel_l2(y25, a["band25"]) < IQ_REL_L2
    assert rel_l2(y13 + y4, x) < 1e-6


def test_svd_vessel_power_fraction():
    meta, a = load("svd_vessel")
    x, vessel = a["iq"], a["vessel"]
    y = np.stack([v.values for v in P.svd_filter(_vols(x, meta["dims"]), 2, x.shape[0])])
    assert rel_l2(y, a["band2"]) < 1e-4  # 40 dB tissue/blood: f32 input rounding x 100
    pd = P.power_doppler(_vols(y, meta["dims"])).data
    pd0 = P.power_doppler(_vols(x, meta["dims"])).data
    frac = lambda p: p[vessel].sum() / p.sum()  # noqa: E731
    assert frac(pd0) < 0.3 and frac(pd) > 0.9  # test_post.cpp:220-251


def test_svd_rejections():
    x = np.array([[complex(f + 1, v) for v in range(16)] for f in range(3)])
    vols = _vols(x, [4, 1, 4])
    for lo, hi in [(0, 2), (1, 4), (3, 2)]:
        with pytest.raises(P.Error):
            P.svd_filter(vols, lo, hi)
    with pytest.raises(P.Error):
        P.svd_filter([], 1, 1)
    with pytest.raises(P.Error):
        P.svd_filter(vols[:1], 1, 1)
    with pytest.raises(P.Error):
        P.svd_filter(_vols(np.zeros((3, 16), complex), [4, 1, 4]), 1, 3)
    with pytest.raises(P.Error):
        P.svd_filter(_vols(np.ones((3, 2), complex), [1, 1, 2]), 1, 3)


@pytest.mark.parametrize("lo,hi", [(2, 20), (1, 20), (3, 17), (1, 1), (5, 6), (2, 9)])
def test_svd_filter_pd_vs_oracle(lo, hi):
    # Clutter 20 dB above blood: rank-2 tissue + random blood, 20 frames.
    rng = np.random.default_rng(lo * 31 + hi)
    N, F = 3000, 20
    tissue = (rng.standard_normal((2, N)) + 1j * rng.standard_normal((2, N))) * 10
    mix = rng.standard_normal((F, 2)) + 1j * rng.standard_normal((F, 2))
    x = (mix @ tissue + rng.standard_normal((F, N)) + 1j * rng.standard_normal((F, N)))
    x = x.astype(np.complex64).astype(np.complex128)
    y_ref, s_ref, _ = O.svd_filter(x, lo, hi)
    y, s, pd = P.post.svd_filter_array(x, lo, hi, want_pd=True)
    assert np.allclose(s, s_ref, rtol=SIG_REL)
    assert rel_l2(y, y_ref) < IQ_REL_L2 * 10
    assert rel_l2(pd, O.power_doppler(y_ref)) < PD_REL_L2


def test_power_doppler():
    meta, a = load("pd_random")
    pd = P.post.power_doppler_array(a["iq"])
    assert rel_l2(pd, a["pd"]) < 1e-6
    lattice = np.array([1, 1j, -1, -1j])
    iq = np.array([[lattice[(f + v) % 4] for v in range(30)] for f in range(100)])
    assert np.all(P.post.power_doppler_array(iq) == 100.0)  # test_post.cpp:283-316
    assert np.all(P.post.power_doppler_array(2 * iq) == 400.0)
    with pytest.raises(P.Error):
        P.power_doppler([])


# ------------------------------------------------------ fused RF -> PD --

def test_reconstruct_pd_vs_oracle():
    import ctypes as C
    from paper_2509_05464_b200 import _native as N
    from paper_2509_05464_b200.beamform import _desc, _probe
    w = W.small()
    rng = np.random.default_rng(77)
    rf = rng.uniform(-1, 1, w.rf_shape()).astype(np.float32)
    g = w.grid
    iq_ref, _ = O.das(rf.astype(np.float64), w.fs, 0.0, w.angles, w.elements, g.dims, g.spacing,
                      g.origin, fc=w.fc)
    y_ref, s_ref, _ = O.svd_filter(iq_ref, 2, w.n_frames)
    pd_ref = O.power_doppler(y_ref)
    desc, keep = _desc(*rf.shape, w.fs, 0.0, w.angles)
    probe, el = _probe(w.elements)
    gc, bc = g._c(), w.bf()._c()
    pd = np.zeros(g.num_points())
    sig = np.zeros(w.n_frames)
    iq = np.zeros((w.n_frames, g.num_points(), 2), np.float32)
    N.check(N.load().fqfg_reconstruct_pd(C.byref(desc), rf.ctypes.data, C.byref(gc),
                                         C.byref(probe), C.byref(bc), 2, w.n_frames,
                                         pd.ctypes.data, sig.ctypes.data, iq.ctypes.data))
    assert rel_l2(iq[..., 0] + 1j * iq[..., 1], iq_ref) < IQ_REL_L2
    assert np.allclose(sig, s_ref, rtol=1e-4)
    assert rel_l2(pd, pd_ref) < PD_REL_L2


def test_pipeline_reconstructor_matches_host_api():
    import torch
    from paper_2509_05464_b200 import pipeline as PL
    w = W.small()
    rng = np.random.default_rng(5)
    rf = rng.uniform(-1, 1, w.rf_shape()).astype(np.float32)
    rec = PL.Reconstructor(w.fs, 0.0, w.angles, w.n_frames, w.n_samples, w.grid, w.elements,
                           w.bf())
    out = rec.step(torch.from_numpy(rf).cuda())
    torch.cuda.synchronize()
    iq, _ = P.das_reconstruct_array(rf, w.fs, 0.0, w.angles, w.grid, w.elements, w.bf())
    _, s, pd = P.post.svd_filter_array(iq, 2, w.n_frames, want_filtered=False, want_pd=True)
    assert np.array_equal(out.pd.cpu().numpy(), pd)
    assert rec.active_pairs > 0


def test_svd_report_mode_correlation_matches_lapack():
    # SvdReport::mode_correlation (svd.cpp:55-75) computed on device.
    meta, a = load("svd_corr")
    x = a["iq"]
    rep = P.SvdReport()
    P.svd_filter(_vols(x, meta["dims"]), 1, x.shape[0], rep)
    F = x.shape[0]
    c = np.array(rep.mode_correlation).reshape(F, F)
    assert np.allclose(c, c.T, atol=1e-12) and np.allclose(np.diag(c), 1.0)
    assert np.allclose(c, a["corr"], atol=1e-4)  # f32 ensemble vs FP64 LAPACK


def test_build_and_apply_delay_matrix_match_reference_formulas():
    # The explicit CSR operator (das.cpp:126-222) built and applied on the GPU.
    import ctypes as C
    from paper_2509_05464_b200 import _native as N
    meta, a = load("das_kat")
    el = a["elements"]
    g = P.GridSpec(tuple(meta["dims"]), tuple(meta["spacing"]), tuple(meta["origin"]))
    vox = np.array([g.point(v) for v in range(g.num_points())])
    probe = N.Probe(el.shape[0], np.ascontiguousarray(el).ctypes.data_as(C.POINTER(C.c_double)))
    bf = P.BeamformParams(center_frequency=meta["fc"])._c()
    n = vox.shape[0]
    rp = np.zeros(n + 1, np.uint64)
    oow, pad = C.c_uint64(), C.c_int()
    L = N.load()
    vv = np.ascontiguousarray(vox)
    N.check(L.fqfg_build_delay_matrix(vv.ctypes.data, n, meta["angles"][0], meta["t0"][0],
                                      meta["fs"], 64, C.byref(probe), C.byref(bf), rp.ctypes.data,
                                      None, None, C.byref(oow), C.byref(pad)))
    nnz = int(rp[-1])
    col = np.zeros(nnz, np.int32)
    val = np.zeros((nnz, 2))
    N.check(L.fqfg_build_delay_matrix(vv.ctypes.data, n, meta["angles"][0], meta["t0"][0],
                                      meta["fs"], 64, C.byref(probe), C.byref(bf), rp.ctypes.data,
                                      col.ctypes.data, val.ctypes.data, C.byref(oow), C.byref(pad)))
    iq = O.rf_to_iq(a["rf"][0, 0], meta["fs"], meta["t0"][0], meta["fc"])
    iq2 = np.ascontiguousarray(np.stack([iq.real, iq.imag], -1))
    y = np.zeros((n, 2))
    N.check(L.fqfg_apply_delay_matrix(n, rp.ctypes.data, col.ctypes.data, val.ctypes.data,
                                      iq2.ctypes.data, iq2.shape[0] * iq2.shape[1], y.ctypes.data))
    # One angle's row sums equal the FP64 literal DAS of that single angle.
    ref, _ = O.das(a["rf"][:1, :1], meta["fs"], meta["t0"][:1], meta["angles"][:1], el,
                   meta["dims"], meta["spacing"], meta["origin"], fc=meta["fc"])
    assert rel_max(y[:, 0] + 1j * y[:, 1], ref[0]) < 1e-12
    assert pad.value == 64


@pytest.mark.parametrize("F,N,v0,v1", [(7, 1000, 0, 1000), (100, 20000, 3, 19990),
                                       (200, 9000, 4096, 9000), (256, 5000, 17, 4999),
                                       (300, 3000, 0, 3000)])
def test_gram_dev_matches_fp64(F, N, v0, v1):
    # G = X^H X over a voxel range: FP64 accumulation of exact f32 products.
    import torch
    from paper_2509_05464_b200 import _native as N_
    rng = np.random.default_rng(F + N)
    x = (rng.standard_normal((F, N)) + 1j * rng.standard_normal((F, N))).astype(np.complex64)
    xs = x[:, v0:v1].astype(np.complex128)
    ref = xs.conj() @ xs.T
    L = N_.load()
    dx = torch.from_numpy(x.view(np.float32).reshape(F, N, 2)).cuda()
    g = torch.zeros((F, F, 2), dtype=torch.float64, device="cuda")
    work = torch.empty(L.fqfg_gram_work_bytes(F), dtype=torch.uint8, device="cuda")
    N_.check(L.fqfg_gram_dev(dx.data_ptr(), F, N, v0, v1, g.data_ptr(), work.data_ptr(), 0))
    torch.cuda.synchronize()
    gg = g.cpu().numpy()
    got = gg[..., 0] + 1j * gg[..., 1]
    assert np.abs(got - ref).max() / np.abs(ref).max() < 1e-12
    assert np.allclose(got, got.conj().T, atol=0)


@pytest.mark.parametrize("F,lo,hi,spread", [(200, 2, 200, 1e6), (200, 1, 200, 1e6),
                                             (200, 3, 200, 1e8), (200, 2, 198, 1e4),
                                             (100, 1, 99, 1.0), (40, 5, 40, 1e3),
                                             (200, 20, 150, 1e6), (2, 2, 2, 10.0)])
def test_eig_band_matches_full_eigensolve(F, lo, hi, spread):
    """fqfg_eig_band_dev (bisection + inverse iteration for the <= 8 vectors
    the band projection reads) against the full QL eigensolve: eigenvalues,
    the projector onto the selected modes, and the band-filtered PD."""
    import torch
    from paper_2509_05464_b200 import _native as N_
    rng = np.random.default_rng(F * 31 + lo)
    N = 4 * F + 64
    # clutter-like spectrum: a few dominant modes, then a long tail
    u = np.linalg.qr(rng.standard_normal((F, F)) + 1j * rng.standard_normal((F, F)))[0]
    s = spread ** (-np.linspace(0, 1, F) ** 0.3)
    a = rng.standard_normal((N, F)) + 1j * rng.standard_normal((N, F))
    x = ((a * s) @ u.conj().T).T.astype(np.complex64)  # [F][N]
    L = N_.load()
    dx = torch.from_numpy(np.ascontiguousarray(x).view(np.float32).reshape(F, N, 2)).cuda()
    work = torch.empty(L.fqfg_gram_work_bytes(F), dtype=torch.uint8, device="cuda")
    res = {}
    for name in ("full", "band"):
        g = torch.zeros((F, F, 2), dtype=torch.float64, device="cuda")
        N_.check(L.fqfg_gram_dev(dx.data_ptr(), F, N, 0, N, g.data_ptr(), work.data_ptr(), 0))
        w = torch.zeros(F, dtype=torch.float64, device="cuda")
        v = torch.zeros((F, F, 2), dtype=torch.float64, device="cuda")
        if name == "full":
            N_.check(L.fqfg_eig_dev(g.data_ptr(), F, w.data_ptr(), v.data_ptr(), 0))
        else:
            N_.check(L.fqfg_eig_band_dev(g.data_ptr(), F, lo, hi, w.data_ptr(), v.data_ptr(), 0))
        pd = torch.zeros(N, dtype=torch.float64, device="cuda")
        N_.check(L.fqfg_project_pd_dev(dx.data_ptr(), F, N, 0, N, v.data_ptr(), lo, hi, None,
                                       pd.data_ptr(), 0))
        torch.cuda.synchronize()
        vv = v.cpu().numpy()
        res[name] = (w.cpu().numpy(), vv[..., 0] + 1j * vv[..., 1], pd.cpu().numpy())
    wf, vf, pf = res["full"]
    wb, vb, pb = res["band"]
    assert np.all(np.diff(wb) <= 0)
    assert np.abs(wb - wf).max() <= 1e-12 * np.abs(wf).max()
    rb = hi - lo + 1
    modes = [j for j in range(F) if (lo - 1 <= j < hi) != (F - rb < rb)]
    if 0 < len(modes) <= 8:
        pf_ = vf[:, modes] @ vf[:, modes].conj().T
        pb_ = vb[:, modes] @ vb[:, modes].conj().T
        assert np.abs(pb_ - pf_).max() < 1e-9
    assert rel_l2(pb, pf) < 1e-10




@pytest.mark.parametrize("F,n,v0,v1", [(200, 9000, 0, 9000), (100, 20000, 1234, 17777),
                                       (256, 5000, 0, 5000), (20, 3000, 7, 2999),
                                       (20, 3000, 8, 2999), (200, 9000, 7, 9000),
                                       (137, 100, 0, 100), (64, 0, 0, 0)])
def test_gram_matches_fp64_reference(F, n, v0, v1):
    """The Casorati Gram of a voxel range (fqfg_gram_dev) against the FP64
    product of the same complex64 samples: Hermitian, finite, exact to FP64
    rounding; an empty range gives zeros."""
    import torch
    from paper_2509_05464_b200 import _native as N
    rng = np.random.default_rng(F + n)
    x = (rng.standard_normal((F, max(n, 1))) + 1j * rng.standard_normal((F, max(n, 1))))
    x = x.astype(np.complex64)[:, :n]
    xs = x[:, v0:v1].astype(np.complex128)
    ref = xs.conj() @ xs.T
    L = N.load()
    dx = torch.from_numpy(np.ascontiguousarray(x).view(np.float32).reshape(F, n, 2)).cuda() \
        if n else torch.zeros((F, 1, 2), device="cuda")
    w = torch.empty(L.fqfg_gram_work_bytes(F), dtype=torch.uint8, device="cuda")
    g = torch.full((F, F, 2), float("nan"), dtype=torch.float64, device="cuda")
    N.check(L.fqfg_gram_dev(dx.data_ptr(), F, n, v0, v1, g.data_ptr(), w.data_ptr(), 0))
    gg = g.cpu().numpy()
    g64 = gg[..., 0] + 1j * gg[..., 1]
    assert np.allclose(g64, g64.conj().T, atol=0) and np.all(np.isfinite(g64))
    if v1 == v0:
        assert np.all(g64 == 0)
        return
    scale = np.abs(ref).max()
    assert np.abs(g64 - ref).max() / scale < 1e-12


def _sharded_case(f_number):
    sp = 0.2567e-3
    w = W.Workload("sharded", W.matrix_probe(32), 3e6, 12e6, np.array([-6, 0, 6]) * W.DEG,
                   P.GridSpec((24, 20, 40), (sp, sp, sp), (-3.0e-3, -2.4e-3, 6e-3)), 504, 24)
    bf = w.bf()
    bf.f_number = f_number
    return w, bf


@pytest.mark.parametrize("f_number", [1.5, 0.0])
def test_depth_slab_sharding_replayed_on_one_gpu(f_number):
    """Depth-slab sharding replayed rank by rank on one GPU:
    each rank uploads only the RF samples fqfg_das_slab_samples names (the
    rest of its buffer is NaN), beamforms its slab like the unsharded run
    (bit-identically with das2; with the tensor-core DAS to fp32 rounding,
    its per-frame fp16 scale comes from the slab's own RF window), and the
    summed partial Grams give the unsharded PD."""
    import torch
    from paper_2509_05464_b200 import pipeline as PL
    w, bf = _sharded_case(f_number)
    rng = np.random.default_rng(31)
    h_rf = torch.from_numpy(rng.uniform(-1, 1, w.rf_shape()).astype(np.float32)).pin_memory()
    args = (w.fs, 0.0, w.angles, w.n_frames, w.n_samples, w.grid, w.elements, bf)
    full = PL.Reconstructor(*args)
    full.das_gram(h_rf.cuda())
    full_gram = full.gram.clone()  # fqfg_eig_dev overwrites the Gram
    full.finish()
    ref_pd = full.pd.clone()
    torch.cuda.synchronize()
    world = 3
    ranks = [PL.Reconstructor(*args, shard=(r, world)) for r in range(world)]
    assert ranks[0].k0 == 0 and ranks[-1].k1 == w.grid.dims[2]
    assert all(r.k1 > r.k0 for r in ranks)
    if f_number > 0:  # deeper slabs need later samples, shallower ones fewer
        assert ranks[0].t_end < w.n_samples and ranks[-1].t_begin > 0
    gram = torch.zeros_like(full_gram)
    for r in ranks:
        d_rf = torch.full(w.rf_shape(), float("nan"), dtype=torch.float32, device="cuda")
        nb = r.upload_rf(h_rf, d_rf)
        assert nb == w.n_frames * w.n_angles * (r.t_end - r.t_begin) * w.n_elements * 4
        r.das_gram(d_rf)
        torch.cuda.synchronize()
        if r.plan.tensor_cores:
            assert rel_l2(r.x[:, r.v0:r.v1].cpu().numpy(), full.x[:, r.v0:r.v1].cpu().numpy()) < 1e-6
        else:
            assert torch.equal(r.x[:, r.v0:r.v1], full.x[:, r.v0:r.v1])
        gram += r.gram
    tol = 1e-6 if full.plan.tensor_cores else 1e-12
    assert torch.allclose(gram, full_gram, rtol=tol, atol=tol * float(full_gram.abs().max()))
    pd = torch.zeros_like(full.pd)
    for r in ranks:
        r.gram.copy_(gram)
        r.finish()
        pd[r.v0:r.v1] = r.pd[r.v0:r.v1]
    torch.cuda.synchronize()
    assert rel_l2(pd.cpu().numpy(), ref_pd.cpu().numpy()) < (1e-6 if full.plan.tensor_cores else 1e-9)


@pytest.mark.parametrize("shape", ["1,16,8,4", "2,16,8,4", "4,12,8,4", "7,4,16,8", "13,2,16,8",
                                   "13,2,16,8,8,4,2", "13,2,16,8,2,16,2", "7,4,16,8,8,8,2"])
def test_das_kernel_shapes_agree(shape, monkeypatch):
    """Every compiled das2_kernel shape (frames per pass, warp split, voxel
    tile) sums each voxel's (element, angle) products in the same order, so
    the IQ is bitwise that of the default shape; all match the oracle."""
    monkeypatch.setenv("FQFG_DAS_TC", "0")
    w = W.small()
    rng = np.random.default_rng(12)
    rf = rng.uniform(-1, 1, w.rf_shape()).astype(np.float32)
    base, _ = P.das_reconstruct_array(rf, w.fs, 0.0, w.angles, w.grid, w.elements, w.bf())
    monkeypatch.setenv("FQFG_DAS_SHAPE", shape)
    got, _ = P.das_reconstruct_array(rf, w.fs, 0.0, w.angles, w.grid, w.elements, w.bf())
    assert np.array_equal(got, base)
    g = w.grid
    ref, _ = O.das(rf.astype(np.float64), w.fs, 0.0, w.angles, w.elements, g.dims, g.spacing,
                   g.origin, fc=w.fc)
    assert rel_l2(got, ref) < IQ_REL_L2


@pytest.mark.parametrize("J", [1, 2, 4, 7])
def test_das_tc_frames_per_pass_agree(J, monkeypatch):
    """The tensor-core DAS at every frames-per-pass width (MMA N = 16 J,
    several passes for small J) gives bitwise the IQ of the 208-frame pass:
    the per-frame fp16 scale, the K order of the MMAs and the accumulator
    restarts do not depend on N or the pass split; and it matches the oracle."""
    w = W.small()
    rng = np.random.default_rng(13)
    rf = rng.uniform(-1, 1, w.rf_shape()).astype(np.float32)
    monkeypatch.setenv("FQFG_DAS_SHAPE", "13,2,16,8")
    base, _ = P.das_reconstruct_array(rf, w.fs, 0.0, w.angles, w.grid, w.elements, w.bf())
    monkeypatch.setenv("FQFG_DAS_SHAPE", {1: "1,16,8,4", 2: "2,16,8,4", 4: "4,12,8,4",
                                          7: "7,4,16,8"}[J])
    got, _ = P.das_reconstruct_array(rf, w.fs, 0.0, w.angles, w.grid, w.elements, w.bf())
    assert np.array_equal(got, base)
    g = w.grid
    ref, _ = O.das(rf.astype(np.float64), w.fs, 0.0, w.angles, w.elements, g.dims, g.spacing,
                   g.origin, fc=w.fc)
    assert rel_l2(got, ref) < IQ_REL_L2


@pytest.mark.parametrize("spacing_mm,f_number", [(0.6, 0.0), (1.5, 0.0), (1.5, 1.0)])
def test_das_tc_long_windows_match_oracle_and_das2(spacing_mm, f_number, monkeypatch):
    """Coarse voxels: one 8 x 8 x 1 tile's tap rows for an (element, angle)
    span tens of samples, so the tensor-core DAS cuts each window into many
    16-row MMA parts (12-row stride; a tap pair belongs to exactly one part).
    IQ against the FP64 oracle and das2; the device K-block counter shows
    the parts were exercised."""
    from paper_2509_05464_b200.engine import Engine
    rng = np.random.default_rng(int(spacing_mm * 10) + int(f_number))
    F, T, fs, fc = 20, 400, 20e6, 5e6
    angles = np.array([-0.06, 0.0, 0.06])
    el = W.matrix_probe(4, 0.3e-3)
    sp = spacing_mm * 1e-3
    g = P.GridSpec((8, 8, 3), (sp, sp, sp), (-3.5 * sp, -3.5 * sp, 2e-3))
    rf = rng.uniform(-1, 1, (F, len(angles), T, el.shape[0])).astype(np.float32)
    bf = P.BeamformParams(c=1540.0, center_frequency=fc, f_number=f_number)
    tc, _ = P.das_reconstruct_array(rf, fs, 0.0, angles, g, el, bf)
    ref, _ = O.das(rf.astype(np.float64), fs, 0.0, angles, el, g.dims, g.spacing, g.origin, fc=fc,
                   f_number=f_number)
    assert rel_l2(tc, ref) < IQ_REL_L2
    assert rel_max(tc, ref) < IQ_REL_MAX
    eng = Engine(fs, 0.0, angles, F, T, g, el, bf)
    assert eng.info.mode == 2
    eng.run([rf], [np.zeros(g.num_points())])
    if f_number == 0:  # every (tile, element, angle) has taps: 3 x 16 x 3 windows
        assert eng.mma_blocks() > 2 * 3 * el.shape[0] * len(angles)
    monkeypatch.setenv("FQFG_DAS_TC", "0")
    das2, _ = P.das_reconstruct_array(rf, fs, 0.0, angles, g, el, bf)
    assert rel_l2(tc, das2) < 1e-5


@pytest.mark.parametrize("dims", [(11, 9, 3), (13, 17, 2), (8, 8, 1)])
def test_das_tc_ragged_grids_match_oracle_and_das2(dims, monkeypatch):
    """3-D grids whose x / y extents are not multiples of the 8 x 8 x 1 tile
    (partial tiles in x and y: their dead voxels carry NaN coordinates and
    must neither write nor contaminate the live ones) and a single-tile grid,
    through the tensor-core DAS, against the FP64 oracle and das2."""
    from paper_2509_05464_b200.engine import Engine
    rng = np.random.default_rng(sum(dims))
    F, T, fs, fc = 18, 320, 20e6, 5e6
    angles = np.array([-0.05, 0.02, 0.07])
    el = W.matrix_probe(4, 0.3e-3)
    sp = 0.1e-3
    g = P.GridSpec(dims, (sp, sp, sp), (-dims[0] / 2 * sp, -dims[1] / 2 * sp, 2e-3))
    rf = rng.uniform(-1, 1, (F, len(angles), T, el.shape[0])).astype(np.float32)
    bf = P.BeamformParams(c=1540.0, center_frequency=fc, f_number=1.0)
    tc, st = P.das_reconstruct_array(rf, fs, 0.0, angles, g, el, bf)
    ref, st_ref = O.das(rf.astype(np.float64), fs, 0.0, angles, el, g.dims, g.spacing, g.origin,
                        fc=fc, f_number=1.0)
    assert np.isfinite(tc).all()
    assert rel_l2(tc, ref) < IQ_REL_L2
    assert rel_max(tc, ref) < IQ_REL_MAX
    assert Engine(fs, 0.0, angles, F, T, g, el, bf).info.mode == 2
    monkeypatch.setenv("FQFG_DAS_TC", "0")
    das2, _ = P.das_reconstruct_array(rf, fs, 0.0, angles, g, el, bf)
    assert rel_l2(tc, das2) < 1e-5


@pytest.mark.parametrize("n_frames", [1, 17, 209])
def test_das_tc_frame_counts_match_oracle(n_frames):
    """Frame counts at the tensor-core DAS's pass boundaries: one frame (a
    16-frame group of 15 padding frames), one past a group, and one past the
    208-frame pass (a second pass of one frame) -- against the FP64 oracle."""
    rng = np.random.default_rng(n_frames)
    T, fs, fc = 256, 20e6, 5e6
    angles = np.array([-0.04, 0.03])
    el = W.matrix_probe(4, 0.3e-3)
    sp = 0.1e-3
    g = P.GridSpec((9, 8, 2), (sp, sp, sp), (-4.5 * sp, -4 * sp, 2e-3))
    rf = rng.uniform(-1, 1, (n_frames, len(angles), T, el.shape[0])).astype(np.float32)
    bf = P.BeamformParams(c=1540.0, center_frequency=fc, f_number=1.0)
    tc, _ = P.das_reconstruct_array(rf, fs, 0.0, angles, g, el, bf)
    ref, _ = O.das(rf.astype(np.float64), fs, 0.0, angles, el, g.dims, g.spacing, g.origin,
                   fc=fc, f_number=1.0)
    assert tc.shape == ref.shape
    assert rel_l2(tc, ref) < IQ_REL_L2
    assert rel_max(tc, ref) < IQ_REL_MAX


@pytest.mark.parametrize("n_angles", [6, 11, 13, 15, 16, 17])
def test_das_many_angles_match_oracle(n_angles):
    """Every shared-memory layout of the tensor-core DAS (table buffers x X
    slots, das_tc_slots): 4 x 5 (6 angles), 3 x 4 (11), 2 x 5 (13), 2 x 4 (15,
    config D; 16, the largest it takes) -- 4 x 6 and 4 x 4 are the 3- and
    9-angle cases elsewhere -- and 17 (das2 takes over), all against the FP64
    oracle."""
    from paper_2509_05464_b200.engine import Engine
    w = W.small()
    rng = np.random.default_rng(n_angles)
    angles = np.linspace(-0.12, 0.12, n_angles)
    F, T = 12, w.n_samples
    rf = rng.uniform(-1, 1, (F, n_angles, T, w.elements.shape[0])).astype(np.float32)
    iq, _ = P.das_reconstruct_array(rf, w.fs, 0.0, angles, w.grid, w.elements, w.bf())
    g = w.grid
    ref, _ = O.das(rf.astype(np.float64), w.fs, 0.0, angles, w.elements, g.dims, g.spacing,
                   g.origin, fc=w.fc)
    assert rel_l2(iq, ref) < IQ_REL_L2
    eng = Engine(w.fs, 0.0, angles, F, T, g, w.elements, w.bf())
    assert eng.info.mode == (2 if n_angles <= 16 else 0)


@pytest.mark.parametrize("taps", [17, 33, 65, 99])
def test_demod_filter_lengths_match_oracle(taps):
    """The fused demodulation (mix + FIR + transpose, up to 97 taps, 33-tap
    register-window path and the generic tap loop) and the two-kernel form
    (longer filters) against the FP64 oracle's rf_to_iq + DAS."""
    w = W.small()
    rng = np.random.default_rng(taps)
    rf = rng.uniform(-1, 1, w.rf_shape()).astype(np.float32)
    bf = w.bf()
    bf.lowpass_taps = taps
    got, _ = P.das_reconstruct_array(rf, w.fs, 0.0, w.angles, w.grid, w.elements, bf)
    g = w.grid
    ref, _ = O.das(rf.astype(np.float64), w.fs, 0.0, w.angles, w.elements, g.dims, g.spacing,
                   g.origin, fc=w.fc, lowpass_taps=taps)
    assert rel_l2(got, ref) < IQ_REL_L2


@pytest.mark.parametrize("F,E,A,dims,T", [
    (1, 1, 1, (1, 1, 1), 64),        # one frame, one element, one voxel
    (3, 5, 2, (9, 3, 5), 96),        # ragged everything: partial tiles in x, y, z
    (230, 16, 1, (6, 2, 3), 80),     # more frames than one pass (fpass 208): two passes
    (17, 33, 3, (11, 1, 13), 120),   # 2-D grid, E not a multiple of 32, F not a multiple of 16
])
@pytest.mark.parametrize("kernel", list(KERNEL_SHAPES))
def test_das_edge_shapes_match_oracle(F, E, A, dims, T, kernel, monkeypatch):
    """Shapes at the edges of the kernel's tiling (single voxel / element /
    frame, ragged tiles, multi-pass frame counts, 2-D grids) against the FP64
    oracle, with exact DasStats-style tap counts via the reference API; for
    the tensor-core default and das2."""
    _kernel_env(monkeypatch, kernel)
    rng = np.random.default_rng(F * 1000 + E)
    fs, fc = 20e6, 5e6
    el = np.stack([(np.arange(E) - (E - 1) / 2) * 0.3e-3, np.zeros(E), np.zeros(E)], axis=1)
    angles = np.linspace(-0.05, 0.05, A) if A > 1 else np.array([0.02])
    sp = 0.2e-3
    g = P.GridSpec(dims, (sp, sp, sp), (-(dims[0] - 1) * sp / 2, -(dims[1] - 1) * sp / 2, 1.5e-3))
    rf = rng.uniform(-1, 1, (F, A, T, E)).astype(np.float32)
    bf = P.BeamformParams(c=1540.0, center_frequency=fc, f_number=1.0)
    iq, _ = P.das_reconstruct_array(rf, fs, 0.0, angles, g, el, bf)
    ref, _ = O.das(rf.astype(np.float64), fs, 0.0, angles, el, g.dims, g.spacing, g.origin, fc=fc,
                   f_number=1.0)
    if np.abs(ref).max() == 0:
        assert np.abs(iq).max() == 0
        return
    assert rel_l2(iq, ref) < IQ_REL_L2
    assert rel_max(iq, ref) < IQ_REL_MAX


@pytest.mark.parametrize("F,N,lo,hi", [(2, 2, 2, 2), (2, 7, 1, 1), (3, 3, 2, 2), (5, 40, 1, 5),
                                       (12, 30, 4, 9), (40, 41, 2, 40)])
def test_svd_filter_edge_bands_match_oracle(F, N, lo, hi):
    """Smallest ensembles (F = 2, N = F), single-mode bands, the identity band
    and a mid band (both sides of the band larger than the rank-8 fast path)
    against the FP64 one-sided Jacobi restatement."""
    rng = np.random.default_rng(F * 100 + N)
    x = (rng.standard_normal((F, N)) + 1j * rng.standard_normal((F, N))).astype(np.complex64)
    y, s, pd = P.post.svd_filter_array(x, lo, hi, want_filtered=True, want_pd=True)
    y_ref, s_ref, _ = O.svd_filter(x.astype(np.complex128), lo, hi)
    assert np.allclose(s, s_ref, rtol=SIG_REL)
    assert rel_l2(y, y_ref) < 1e-5
    assert rel_l2(pd, O.power_doppler(y_ref)) < PD_REL_L2


# ---------------------------------------------- config-C geometry parity --

def _c_block(k0, by=8, bx=8, bz=4):
    """An 8 x 8 x 4 voxel block of the config-C grid (128^3 @ 0.2567 mm,
    matrix32x32, 9 angles, T = 768) centred laterally at plane k0, with the
    grid's own voxel coordinates."""
    w = W.config("C")
    g = w.grid
    nx, ny, _ = g.dims
    i0, j0 = nx // 2 - bx // 2, ny // 2 - by // 2
    sub = P.GridSpec((bx, by, bz), g.spacing,
                     tuple(g.origin[d] + (i0, j0, k0)[d] * g.spacing[d] for d in range(3)))
    return w, sub


@pytest.mark.parametrize("k0", [0, 62, 124])
def test_delay_matrix_bit_exact_vs_reference_at_config_c(k0):
    """build_delay_matrix (das.cpp:126-208) on the GPU against the reference's
    own, for the 1024-element probe and the config-C grid (shallow, mid,
    deep blocks; every angle): row_ptr, col_idx, out_of_window and the padded
    width are bit-exact; the complex weights agree to FP64 rounding."""
    import ctypes as C
    from paper_2509_05464_b200 import _native as N
    w, sub = _c_block(k0)
    vox = np.ascontiguousarray([sub.point(v) for v in range(sub.num_points())])
    el = np.ascontiguousarray(w.elements)
    probe = N.Probe(el.shape[0], el.ctypes.data_as(C.POINTER(C.c_double)))
    bf = w.bf()._c()
    L = N.load()
    n = vox.shape[0]
    for a in w.angles:
        rp_r, col_r, val_r, oow_r, pad_r = O.ref_build_delay_matrix(vox, a, 0.0, w.fs, w.n_samples,
                                                                    el, fc=w.fc)
        rp = np.zeros(n + 1, np.uint64)
        oow, pad = C.c_uint64(), C.c_int()
        N.check(L.fqfg_build_delay_matrix(vox.ctypes.data, n, a, 0.0, w.fs, w.n_samples,
                                          C.byref(probe), C.byref(bf), rp.ctypes.data, None, None,
                                          C.byref(oow), C.byref(pad)))
        nnz = int(rp[-1])
        col = np.zeros(nnz, np.int32)
        val = np.zeros((nnz, 2))
        N.check(L.fqfg_build_delay_matrix(vox.ctypes.data, n, a, 0.0, w.fs, w.n_samples,
                                          C.byref(probe), C.byref(bf), rp.ctypes.data,
                                          col.ctypes.data, val.ctypes.data, C.byref(oow),
                                          C.byref(pad)))
        assert nnz > 0
        assert np.array_equal(rp, rp_r)
        assert np.array_equal(col, col_r)
        assert oow.value == oow_r and pad.value == pad_r
        v = val[:, 0] + 1j * val[:, 1]
        assert np.max(np.abs(v - val_r)) <= 1e-14


@pytest.mark.parametrize("k0", [0, 62, 124])
def test_das_and_pd_at_config_c_geometry_match_reference(k0):
    """The benchmarked shape itself: config-C probe / angles / T = 768 / F =
    200 through the production kernel shape (208 frames per pass, 16 + 8
    warps, tile 4 x 8 x 2) and the F = 200 filter, on 8 x 8 x 4 blocks at the
    top, middle and bottom of the volume -- IQ against the reference's own
    das_reconstruct (oracle/_ref) and PD against the FP64 SVD-filter
    restatement + power_doppler of the reference IQ."""
    from paper_2509_05464_b200.engine import Engine
    w, sub = _c_block(k0)
    rng = np.random.default_rng(200 + k0)
    rf = rng.uniform(-1, 1, w.rf_shape()).astype(np.float32)
    eng = Engine(w.fs, 0.0, w.angles, w.n_frames, w.n_samples, sub, w.elements, w.bf())
    info = eng.info
    assert tuple(info.shape) == (13, 2, 16, 8)
    assert tuple(info.tile) == ((8, 8, 1) if info.mode == 2 else (4, 8, 2))
    assert info.frames_per_pass == 208 and info.n_passes == 1
    pd = np.zeros(sub.num_points())
    eng.run([rf], [pd])
    iq = eng.copy_iq()
    iq_ref, _ = O.ref_das(rf, w.fs, 0.0, w.angles, w.elements, sub.dims, sub.spacing, sub.origin,
                          fc=w.fc)
    assert rel_l2(iq, iq_ref) < IQ_REL_L2
    assert rel_max(iq, iq_ref) < IQ_REL_MAX
    y, _, _ = O.svd_filter(iq_ref, 2, w.n_frames, method="gram")
    assert rel_l2(pd, O.power_doppler(y)) < PD_REL_L2


def test_das_at_config_d_geometry(monkeypatch):
    """Config D's geometry (64 x 64 = 4096-element matrix, 15 angles over
    +-14 deg, T = 1176) through config D's production kernel shape (112
    frames per pass, 16 + 8 warps -- chosen there by the IQ memory budget),
    on an 8 x 8 x 4 block at mid depth of the 256 x 256 x 192 grid with 16
    frames: IQ against the reference's das_reconstruct, PD against the FP64
    filter restatement."""
    from paper_2509_05464_b200.engine import Engine
    monkeypatch.setenv("FQFG_DAS_SHAPE", "7,4,16,8")
    w = W.config("D")
    g = w.grid
    nx, ny, nz = g.dims
    i0, j0, k0 = nx // 2 - 4, ny // 2 - 4, nz // 2
    sub = P.GridSpec((8, 8, 4), g.spacing,
                     tuple(g.origin[d] + (i0, j0, k0)[d] * g.spacing[d] for d in range(3)))
    F = 16
    rng = np.random.default_rng(64)
    rf = rng.uniform(-1, 1, (F, w.n_angles, w.n_samples, w.n_elements)).astype(np.float32)
    eng = Engine(w.fs, 0.0, w.angles, F, w.n_samples, sub, w.elements, w.bf())
    assert tuple(eng.info.shape) == (7, 4, 16, 8) and eng.info.frames_per_pass == 112
    pd = np.zeros(sub.num_points())
    eng.run([rf], [pd])
    iq = eng.copy_iq()
    iq_ref, _ = O.ref_das(rf, w.fs, 0.0, w.angles, w.elements, sub.dims, sub.spacing, sub.origin,
                          fc=w.fc)
    assert rel_l2(iq, iq_ref) < IQ_REL_L2
    assert rel_max(iq, iq_ref) < IQ_REL_MAX
    y, _, _ = O.svd_filter(iq_ref, 2, F, method="gram")
    assert rel_l2(pd, O.power_doppler(y)) < PD_REL_L2


GRAM_TC_REL = 1e-7  # int8-digit tensor-core Gram vs exact FP64 (max entry, relative to max): 2e-8 measured, 7.5e-8 at 60 dB spread


@pytest.mark.parametrize("F,n,v0,v1,dyn", [(200, 9000, 0, 9000, 0), (100, 20000, 1234, 17777, 0),
                                           (256, 5000, 0, 5000, 0), (20, 3000, 7, 2999, 0),
                                           (200, 40000, 3, 39998, 60), (400, 3000, 0, 3000, 0),
                                           (137, 100, 0, 100, 30), (1, 50, 0, 50, 0),
                                           (64, 600000, 0, 600000, 40), (64, 0, 0, 0, 0)])
def test_gram_tensor_core_matches_fp64(F, n, v0, v1, dyn):
    """fqfg_gram_tc_dev (tcgen05.mma kind::i8, four 7-bit digits per sample,
    int32 TMEM accumulation, FP64 recombination) against the exact FP64
    product of the same complex64 samples; `dyn` dB of amplitude spread
    across voxels and frames (a clutter-dominated ensemble is far from
    uniform); several digit batches at 600k voxels; exactly Hermitian."""
    import torch
    from paper_2509_05464_b200 import _native as N
    rng = np.random.default_rng(F + n + dyn)
    m = max(n, 1)
    x = rng.standard_normal((F, m)) + 1j * rng.standard_normal((F, m))
    if dyn:
        x *= 10 ** (-dyn / 20 * rng.uniform(0, 1, (1, m)))
        x *= 10 ** (-dyn / 40 * rng.uniform(0, 1, (F, 1)))
    x = x.astype(np.complex64)[:, :n]
    xs = x[:, v0:v1].astype(np.complex128)
    ref = xs.conj() @ xs.T
    L = N.load()
    dx = torch.from_numpy(np.ascontiguousarray(x).view(np.float32).reshape(F, n, 2)).cuda() \
        if n else torch.zeros((F, 1, 2), device="cuda")
    w = torch.empty(L.fqfg_gram_tc_work_bytes(F), dtype=torch.uint8, device="cuda")
    g = torch.full((F, F, 2), float("nan"), dtype=torch.float64, device="cuda")
    N.check(L.fqfg_gram_tc_dev(dx.data_ptr(), F, n, v0, v1, g.data_ptr(), w.data_ptr(), 0))
    gg = g.cpu().numpy()
    gt = gg[..., 0] + 1j * gg[..., 1]
    assert np.all(np.isfinite(gt))
    assert np.array_equal(gt, gt.conj().T)
    if v1 == v0:
        assert np.all(gt == 0)
        return
    err = np.abs(gt - ref).max() / np.abs(ref).max()
    print(f"tensor-core Gram F={F} voxels={v1 - v0} dyn={dyn} dB: max rel error {err:.2e}")
    assert err < GRAM_TC_REL


@pytest.mark.parametrize("clutter_db", [40, 60, 80])
@pytest.mark.parametrize("gram", ["tc", "fp64"])
def test_filter_at_high_clutter_to_blood_ratios(clutter_db, gram):
    """The clutter filter alone at 40-80 dB clutter-to-blood power: a
    complex64 Casorati matrix (rank-1 tissue clutter moving slowly, 5 % of
    the voxels blood, noise 20 dB below blood), filtered on the GPU (Gram on
    the tensor cores or FP64, band eigensolve, one-pass PD) against the FP64
    restatement applied to the same complex64 samples.  Isolates what the
    f32 IQ of a full DAS adds at high ratios."""
    import torch
    from paper_2509_05464_b200 import _native as N
    F, n = 100, 20000
    rng = np.random.default_rng(clutter_db)
    amp = 10 ** (clutter_db / 20)
    t = np.arange(F)
    tissue = amp * (rng.standard_normal(n) + 1j * rng.standard_normal(n))[None, :] * \
        np.exp(1j * 0.01 * t)[:, None]
    vessel = rng.uniform(0, 1, n) < 0.05
    blood = np.where(vessel[None, :],
                     np.exp(1j * (0.7 * t[:, None] + rng.uniform(0, 6.28, n)[None, :])), 0)
    noise = 0.1 * (rng.standard_normal((F, n)) + 1j * rng.standard_normal((F, n)))
    x = (tissue + blood + noise).astype(np.complex64)
    y, _, _ = O.svd_filter(x.astype(np.complex128), 2, F, method="gram")
    pd_ref = O.power_doppler(y)
    L = N.load()
    dx = torch.from_numpy(np.ascontiguousarray(x).view(np.float32).reshape(F, n, 2)).cuda()
    g = torch.empty((F, F, 2), dtype=torch.float64, device="cuda")
    wv = torch.empty(F, dtype=torch.float64, device="cuda")
    v = torch.empty((F, F, 2), dtype=torch.float64, device="cuda")
    pd = torch.empty(n, dtype=torch.float64, device="cuda")
    if gram == "tc":
        w = torch.empty(L.fqfg_gram_tc_work_bytes(F), dtype=torch.uint8, device="cuda")
        N.check(L.fqfg_gram_tc_dev(dx.data_ptr(), F, n, 0, n, g.data_ptr(), w.data_ptr(), 0))
    else:
        w = torch.empty(L.fqfg_gram_work_bytes(F), dtype=torch.uint8, device="cuda")
        N.check(L.fqfg_gram_dev(dx.data_ptr(), F, n, 0, n, g.data_ptr(), w.data_ptr(), 0))
    N.check(L.fqfg_eig_band_dev(g.data_ptr(), F, 2, F, wv.data_ptr(), v.data_ptr(), 0))
    N.check(L.fqfg_project_pd_dev(dx.data_ptr(), F, n, 0, n, v.data_ptr(), 2, F, None,
                                  pd.data_ptr(), 0))
    err = rel_l2(pd.cpu().numpy(), pd_ref)
    print(f"filter at {clutter_db} dB clutter, {gram} Gram: PD rel-L2 {err:.2e}")
    assert err < PD_REL_L2
