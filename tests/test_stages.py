"""Stage file formats (paper_2509_05464_b200/stages.py) against the
reference's own writers compiled from /root/reference (oracle/_ref): every
file a stage writes is byte-identical to what run.cpp's writers produce for
the same values.  CPU only (no compute calls)."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2509_05464_b200 import post, stages
from paper_2509_05464_b200.beamform import GridSpec, IqVolume, RfFrame, TxEvent, write_iq_volume

needs_ref = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")


def _slurp(p):
    with open(p, "rb") as f:
        return f.read()


@needs_ref
@pytest.mark.parametrize("dims", [(7, 5, 3), (9, 1, 6), (1, 8, 1), (4, 6, 1), (1, 1, 1)])
def test_write_grid_bytes_match_reference(dims, tmp_path):
    rng = np.random.default_rng(sum(dims))
    data = rng.standard_normal(int(np.prod(dims))) * 10.0 ** rng.integers(-8, 8)
    sp, org = (0.2567e-3, 0.1e-3, 1.0 / 3.0), (-16.3e-3, 0.0, 0.01)
    stages.write_grid(str(tmp_path / "a.fqf"), post.VoxelGrid(dims, sp, org, data))
    O.ref_write_grid(tmp_path / "b.fqf", data, dims, sp, org)
    assert _slurp(tmp_path / "a.fqf") == _slurp(tmp_path / "b.fqf")
    back = stages.read_grid(str(tmp_path / "b.fqf"))
    assert tuple(back.dims) == dims and np.array_equal(back.data, data)
    assert back.spacing == sp and back.origin == org


@needs_ref
@pytest.mark.parametrize("dims", [(7, 1, 5), (1, 6, 4), (5, 4, 1), (1, 9, 1), (6, 1, 1),
                                  (1, 1, 1)])
def test_write_pgm_bytes_match_reference(dims, tmp_path):
    rng = np.random.default_rng(3 + sum(dims))
    data = rng.uniform(-0.2, 1.2, int(np.prod(dims)))
    data[:3] = [0.5 / 255, 1.5 / 255, 254.5 / 255][:min(3, data.size)]  # half-way roundings
    stages.write_pgm(str(tmp_path / "a.pgm"), post.VoxelGrid(dims, (1, 1, 1), (0, 0, 0), data))
    O.ref_write_pgm(tmp_path / "b.pgm", data, dims)
    assert _slurp(tmp_path / "a.pgm") == _slurp(tmp_path / "b.pgm")


@needs_ref
def test_write_pgm_rejects_full_volumes(tmp_path):
    with pytest.raises(Exception):
        stages.write_pgm(str(tmp_path / "a.pgm"),
                         post.VoxelGrid((3, 3, 3), (1, 1, 1), (0, 0, 0), np.zeros(27)))


@needs_ref
def test_iq_volume_bytes_match_reference(tmp_path):
    rng = np.random.default_rng(5)
    dims, sp, org = (4, 3, 2), (0.1e-3, 0.2e-3, 0.3e-3), (-1e-3, 0.0, 5e-3)
    iq = rng.standard_normal(24) + 1j * rng.standard_normal(24)
    write_iq_volume(str(tmp_path / "a.fqf"), IqVolume(GridSpec(dims, sp, org), 6, 9, iq))
    O.ref_write_iq_volume(tmp_path / "b.fqf", iq, dims, sp, org, 6, 9)
    assert _slurp(tmp_path / "a.fqf") == _slurp(tmp_path / "b.fqf")


@needs_ref
@pytest.mark.parametrize("same", [False, True])
def test_metrics_text_matches_reference(same):
    rng = np.random.default_rng(11)
    dims = (9, 1, 7)
    a = rng.uniform(0, 1, 63)
    b = a.copy() if same else np.clip(a + rng.normal(0, 0.05, 63), 0, 1)
    csv, js = O.ref_metrics_text(a, b, dims)
    m = O.ref_metrics(a, b, dims)
    rep = post.MetricsReport(mse=m["mse"], psnr=m["psnr"], ssim=m["ssim"])
    assert post.metrics_csv(rep) == csv
    assert post.metrics_json(rep) == js


def test_rf_and_particle_frames_round_trip(tmp_path):
    rng = np.random.default_rng(2)
    x = rng.uniform(-1, 1, (37, 5)).astype(np.float32).astype(np.float64)
    fr = RfFrame(x, 12e6, 1.25e-6, TxEvent(angle=-0.13962634015954636))
    p = str(tmp_path / stages.rf_frame_rel(3, 7).replace("/", "_"))
    stages.write_rf_frame(p, fr, 3)
    back, idx = stages.read_rf_frame(p)
    assert idx == 3 and np.array_equal(back.samples, x)
    assert back.sampling_rate == 12e6 and back.t0 == 1.25e-6
    assert back.tx.angle == -0.13962634015954636
    hdr = _slurp(p)[8:200].decode(errors="ignore")
    assert "kind=rf\n" in hdr and "angle=-0.13962634015954636\n" in hdr and "dtype=f32\n" in hdr
    pos = rng.standard_normal((11, 3))
    q = str(tmp_path / "particles.fqf")
    stages.write_particle_frame(q, pos, 4, 0.008)
    got, fi, t = stages.read_particle_frame(q)
    assert fi == 4 and t == 0.008 and np.array_equal(got, pos)
    assert "time=0.008\n" in _slurp(q)[8:120].decode(errors="ignore")


def test_stage_paths_follow_run_cpp():
    assert stages.rf_frame_rel(2, 0) == "rf/frame_0002_tx_00.fqf"  # test_pipeline.cpp:331
    assert stages.iq_frame_rel(0) == "beamform/Frame_1.fqf"
    assert stages.particle_frame_rel(12) == "particles/frame_0012.fqf"


@pytest.mark.parametrize("x,want", [
    (1.0, "1.0"), (0.5, "0.5"), (123.456, "123.456"), (1e-5, "1e-05"), (1e-4, "0.0001"),
    (1e15, "1e+15"), (123456789012345.0, "123456789012345.0"), (-2.5, "-2.5"),
    (3e100, "3e+100"), (0.0, "0.0"), (-0.0, "-0.0"), (float("nan"), "null"),
    (1234567.0, "1234567.0"), (0.000123, "0.000123"), (2.5e-8, "2.5e-08")])
def test_json_numbers_follow_nlohmann_format(x, want):
    """nlohmann::json dump of doubles (dtoa_impl::format_buffer, min_exp -4,
    max_exp 15); the vendored json.hpp is absent, so the rules are restated."""
    assert stages._json_number(x) == want


def test_svd_report_json_layout():
    rep = post.SvdReport(singular_values=[3.0, 1e-5], mode_correlation=[1.0, 0.25, 0.25, 1.0],
                         n_modes=2, keep_lo=2, keep_hi=2)
    s = stages.svd_report_json(rep)
    assert s == ('{\n  "keep": [\n    2,\n    2\n  ],\n  "mode_correlation": [\n    1.0,\n'
                 '    0.25,\n    0.25,\n    1.0\n  ],\n  "n_modes": 2,\n  "singular_values": [\n'
                 '    3.0,\n    1e-05\n  ]\n}\n')
    import json
    d = json.loads(s)
    assert d["keep"] == [2, 2] and d["singular_values"] == [3.0, 1e-5]
