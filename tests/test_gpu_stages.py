"""The beamform / post / metrics stage bodies on the GPU
(paper_2509_05464_b200/stages.py, run.cpp:397-507) over a micro stage
directory built from the flow phantoms of tests/phantom_cases.py:

* outputs are exactly the files run.cpp lists, and byte-identical across
  runs and between the two-stage and the fused (no IQ re-read) paths
  (test_pipeline.cpp:330-385's determinism checks);
* the pd / gt images and the metrics match the reference chain (the
  reference's das_reconstruct, the FP64 SVD restatement, the reference's
  render_db / ground_truth_pd / metrics) within the image-parity tolerances
  of tests/test_gpu_image.py; the gt grid file equals the reference writer's
  bytes for the reference's own ground truth.
"""
import json
import os

import numpy as np
import pytest

import paper_2509_05464_b200 as P
from oracle import oracle as O
from paper_2509_05464_b200 import stages as S
from tests import phantom_cases as PC
from tests.golden_io import rel_l2

pytestmark = pytest.mark.gpu

PD_REL_L2 = 1e-4
METRIC_ABS = 5e-4


def _slurp(p):
    with open(p, "rb") as f:
        return f.read()


def _stage_dir(root, name):
    c, ph = PC.case(name), PC.phantom(name)
    os.makedirs(os.path.join(root, "rf"), exist_ok=True)
    os.makedirs(os.path.join(root, "particles"), exist_ok=True)
    for f in range(c.F):
        for a in range(len(c.angles)):
            fr = P.RfFrame(ph.rf[f, a].astype(np.float64), c.fs, 0.0,
                           P.TxEvent(angle=float(c.angles[a])))
            S.write_rf_frame(os.path.join(root, S.rf_frame_rel(f, a)), fr, f)
        S.write_particle_frame(os.path.join(root, S.particle_frame_rel(f)), ph.blood[f], f,
                               f / 500.0)
    td = P.Transducer(np.asarray(c.elements), name, 0.3e-3, c.fc)
    return S.StageConfig(transducer=td, grid=c.grid, n_frames=c.F,
                         angles_deg=list(np.degrees(c.angles)), f_number=1.5, svd_lo=c.lo,
                         pd_dynamic_range_db=PC.DR_DB, ground_truth_sigma_voxels=PC.GT_SIGMA)


@pytest.mark.parametrize("name", PC.CASES)
def test_stages_outputs_match_reference_chain(name, tmp_path):
    c = PC.case(name)
    d1, d2 = str(tmp_path / "a"), str(tmp_path / "b")
    cfg = _stage_dir(d1, name)
    _stage_dir(d2, name)
    out1 = S.run_beamform(d1, cfg) + S.run_post(d1, cfg) + S.run_metrics(d1)
    for o in out1:
        assert os.path.exists(os.path.join(d1, o)), o
    assert sorted(os.listdir(os.path.join(d1, "beamform"))) == sorted(
        f"Frame_{f + 1}.fqf" for f in range(c.F))  # chunk stripes removed
    out2 = S.run_beamform_post(d2, cfg) + S.run_metrics(d2)
    assert sorted(out1) == sorted(out2)
    for o in out1:  # fused path: identical bytes
        assert _slurp(os.path.join(d1, o)) == _slurp(os.path.join(d2, o)), o
    pd_bytes = _slurp(os.path.join(d1, "post/pd.fqf"))
    os.remove(os.path.join(d1, "post/pd.fqf"))
    S.run_post(d1, cfg)
    assert _slurp(os.path.join(d1, "post/pd.fqf")) == pd_bytes  # rerun reproduces the bytes

    # against the reference chain
    pd_ref, m_ref, gimg_ref = PC.reference(name)
    img_ref = O.ref_render_db(pd_ref, c.grid.dims, PC.DR_DB, True)
    img = S.read_grid(os.path.join(d1, "post/pd.fqf")).data
    assert rel_l2(img, img_ref) < PD_REL_L2
    gt = S.read_grid(os.path.join(d1, "post/gt.fqf")).data
    assert np.abs(gt - gimg_ref).max() < 1e-9
    m = json.load(open(os.path.join(d1, "metrics/metrics.json")))
    assert abs(m["ssim"] - m_ref["ssim"]) < METRIC_ABS
    assert abs(m["psnr"] - m_ref["psnr"]) < METRIC_ABS
    rep = json.load(open(os.path.join(d1, "post/svd_report.json")))
    assert rep["keep"] == [c.lo, c.F] and rep["n_modes"] == c.F
    s = np.asarray(rep["singular_values"])
    assert np.all(np.diff(s) <= 0) and len(rep["mode_correlation"]) == c.F * c.F
    iq0 = P.read_iq_volume(os.path.join(d1, S.iq_frame_rel(0)))
    assert iq0.frame_index == 0 and iq0.n_angles == len(c.angles)
    # the reference writer's bytes for the reference's own ground truth
    O.ref_write_grid(tmp_path / "gt_ref.fqf", gimg_ref, c.grid.dims, c.grid.spacing,
                     c.grid.origin)
    ours = _slurp(os.path.join(d1, "post/gt.fqf"))
    ref = _slurp(tmp_path / "gt_ref.fqf")
    assert ours[:len(ref) - 8 * gimg_ref.size] == ref[:len(ref) - 8 * gimg_ref.size]  # header


def _cfg_text(cfg):
    g, td = cfg.grid, cfg.transducer
    el = np.asarray(td.elements, dtype=np.float64).reshape(-1)
    lines = {"n_frames": cfg.n_frames, "angles_deg": " ".join(repr(float(a)) for a in cfg.angles_deg),
             "sound_speed": cfg.sound_speed, "f_number": cfg.f_number,
             "lowpass_taps": cfg.lowpass_taps, "dims": " ".join(map(str, g.dims)),
             "spacing": " ".join(repr(float(v)) for v in g.spacing),
             "origin": " ".join(repr(float(v)) for v in g.origin),
             "center_frequency": repr(float(td.center_frequency)),
             "elements": " ".join(repr(float(v)) for v in el),
             "bmode_dr": cfg.bmode_dynamic_range_db, "pd_dr": cfg.pd_dynamic_range_db,
             "svd_lo": cfg.svd_lo, "svd_hi": cfg.svd_hi, "gt_sigma": cfg.ground_truth_sigma_voxels}
    return "\n".join(f"{k}={v}" for k, v in lines.items()) + "\n"


@pytest.mark.parametrize("name", PC.CASES)
def test_cpp_stage_body_over_engine_matches_python_stages(name, tmp_path):
    """The C++ stage body (shim/fqf_stages.cpp: run_beamform + run_post of
    run.cpp:397-487 over the reconstruction engine, the IQ ensemble kept on
    the GPU) writes the files the stage bodies write: IQ volumes, B-mode, gt,
    SVD report byte-identical; the PD grid within 1e-8 (the engine's
    tensor-core Gram and band eigensolve vs svd_filter's FP64 Gram and full
    eigensolve) and its graymap identical."""
    import ctypes as C
    lib = C.CDLL(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                              "shim", "build", "libfqf_dropin.so"))
    lib.fqfg_stage_last_error.restype = C.c_char_p
    d1, d2 = str(tmp_path / "py"), str(tmp_path / "cpp")
    cfg = _stage_dir(d1, name)
    _stage_dir(d2, name)
    out1 = S.run_beamform(d1, cfg) + S.run_post(d1, cfg)
    rc = lib.fqfg_stage_beamform_post(d2.encode(), _cfg_text(cfg).encode())
    assert rc == 0, lib.fqfg_stage_last_error().decode()
    for o in out1:
        a, b = os.path.join(d1, o), os.path.join(d2, o)
        assert os.path.exists(b), o
        if o == "post/pd.fqf":
            pa, pb = S.read_grid(a).data, S.read_grid(b).data
            assert rel_l2(pb, pa) < 1e-8
        else:
            assert _slurp(a) == _slurp(b), o
