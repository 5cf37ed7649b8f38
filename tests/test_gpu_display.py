"""Display and scoring on the GPU against the
reference's own render_db / bmode / mip / ground_truth_pd / metrics
(oracle/_ref) and the reference tests (test_post.cpp:318-501).

Tolerances: render/bmode/mip exact up to libm last-ulp differences
(DISP_ABS = 1e-14 on [0, 1] images); ground_truth_pd 1e-12 relative
(splat sums in 64-bit fixed point, deterministic); metrics 1e-12 (tree vs sequential
mean of the local SSIM)."""
import math

import numpy as np
import pytest

import paper_2509_05464_b200 as P
from oracle import oracle as O
from paper_2509_05464_b200 import post

pytestmark = pytest.mark.gpu

DISP_ABS = 1e-14
METRIC_REL = 1e-12


def vg(data, dims):
    return post.VoxelGrid(tuple(dims), (1e-3, 1e-3, 1e-3), (0.0, 0.0, 0.0),
                          np.asarray(data, np.float64).ravel())


@pytest.mark.parametrize("power", [0, 1])
@pytest.mark.parametrize("dims", [(7, 5, 3), (64, 1, 64), (33, 20, 17)])
def test_render_db_matches_reference(dims, power):
    rng = np.random.default_rng(sum(dims) + power)
    v = rng.standard_normal(int(np.prod(dims))) * np.exp(rng.uniform(-12, 2, int(np.prod(dims))))
    v[::7] = 0.0
    got = post.render_db(vg(v, dims), 60.0, power).data
    ref = O.ref_render_db(v, dims, 60.0, bool(power))
    assert np.max(np.abs(got - ref)) <= DISP_ABS


def test_render_db_reference_cases():
    # test_post.cpp:318-348
    v = vg([2.0, 1.0, 2e-9, 0.0], (4, 1, 1))
    amp = post.render_db(v, 60.0, post.DbScale.amplitude).data
    assert amp[0] == 1.0 and amp[2] == 0.0 and amp[3] == 0.0
    assert abs(amp[1] - (60.0 - 20.0 * math.log10(2.0)) / 60.0) <= 1e-14
    pw = post.render_db(v, 60.0, post.DbScale.power).data
    assert pw[0] == 1.0 and abs(pw[1] - (60.0 - 10.0 * math.log10(2.0)) / 60.0) <= 1e-14
    neg = post.render_db(vg([-4.0, 1.0], (2, 1, 1)), 60.0, post.DbScale.amplitude).data
    assert neg[0] == 1.0
    with pytest.raises(P.Error, match="nonzero volume"):
        post.render_db(vg([0.0, 0.0], (2, 1, 1)), 60.0, post.DbScale.amplitude)
    for dr in (0.0, -5.0):
        with pytest.raises(P.Error, match="dynamic range must be positive"):
            post.render_db(v, dr, post.DbScale.amplitude)


def test_bmode_matches_reference():
    dims = (24, 12, 9)
    rng = np.random.default_rng(4)
    iq = rng.standard_normal(int(np.prod(dims))) + 1j * rng.standard_normal(int(np.prod(dims)))
    g = P.GridSpec(dims, (1e-3,) * 3, (0.0, 0.0, 0.0))
    got = post.bmode(P.IqVolume(g, 0, 1, iq), 75.0).data
    assert np.max(np.abs(got - O.ref_bmode(iq, dims, 75.0))) <= DISP_ABS
    with pytest.raises(P.Error, match="bmode needs an IQ volume matching its grid"):
        post.bmode(P.IqVolume(g, 0, 1, iq[:-1]), 75.0)


@pytest.mark.parametrize("axis", [0, 1, 2])
def test_mip_matches_reference(axis):
    dims = (13, 7, 5)
    rng = np.random.default_rng(axis)
    v = rng.standard_normal(int(np.prod(dims)))
    m = post.mip(vg(v, dims), axis)
    want = list(dims)
    want[axis] = 1
    assert tuple(m.dims) == tuple(want)
    assert np.array_equal(m.data, O.ref_mip(v, dims, axis))
    assert m.data.max() == v.max()
    with pytest.raises(P.Error, match="mip axis must be 0, 1, or 2"):
        post.mip(vg(v, dims), 3)


def test_ground_truth_pd_matches_reference():
    from tests import phantom_cases as PC
    c, ph = PC.case("matrix3d"), PC.phantom("matrix3d")
    g = c.grid
    got = post.ground_truth_pd(ph.blood, g, 1.0).data
    ref = O.ref_ground_truth_pd(ph.blood, g.dims, g.spacing, g.origin, 1.0)
    assert got.max() == 1.0
    assert np.max(np.abs(got - ref)) <= 1e-12
    with pytest.raises(P.Error, match="kernel sigma must be positive"):
        post.ground_truth_pd(ph.blood, g, 0.0)
    with pytest.raises(P.Error, match="scatterer positions must be finite"):
        post.ground_truth_pd([np.array([[np.nan, 0.0, 0.0]])], g, 1.0)
    with pytest.raises(P.Error, match="needs at least one frame"):
        post.ground_truth_pd([], g, 1.0)


@pytest.mark.parametrize("dims", [(40, 1, 40), (16, 16, 16), (10, 12, 3), (64, 48, 1), (5, 1, 1)])
def test_metrics_match_reference(dims):
    rng = np.random.default_rng(dims[0] * 7 + dims[2])
    a = rng.uniform(0, 1, int(np.prod(dims)))
    b = np.clip(a + 0.1 * rng.standard_normal(a.size), 0, 1)
    got = post.metrics(vg(a, dims), vg(b, dims))
    ref = O.ref_metrics(a, b, dims)
    assert abs(got.mse - ref["mse"]) <= METRIC_REL * ref["mse"]
    assert abs(got.psnr - ref["psnr"]) <= METRIC_REL * abs(ref["psnr"])
    assert abs(got.ssim - ref["ssim"]) <= METRIC_REL
    same = post.metrics(vg(a, dims), vg(a, dims))  # test_post.cpp:470-478
    assert same.mse == 0.0 and math.isinf(same.psnr) and same.psnr > 0 and same.ssim == 1.0


def test_metrics_rejections_and_formats():
    with pytest.raises(P.Error, match="identical shape"):
        post.metrics(vg(np.zeros(4), (4, 1, 1)), vg(np.zeros(4), (2, 2, 1)))
    r = post.MetricsReport(0.25, 10 * math.log10(4.0), 0.5)
    assert post.metrics_csv(r) == "0.25,6.0205999132796242,0.5\n"
    assert post.metrics_json(post.MetricsReport(0.0, math.inf, 1.0)) == \
        '{"mse": 0, "psnr": "inf", "ssim": 1}\n'


def test_image_metrics_on_device_match_reference_chain():
    """The whole scoring chain on the GPU (PD -> render_db -> metrics vs the
    rendered ground truth) equals the reference's scoring of the same PD."""
    from tests import phantom_cases as PC
    c = PC.case("linear2d")
    g = c.grid
    pd_ref, m_ref, _ = PC.reference("linear2d")
    ph = PC.phantom("linear2d")
    gt = post.ground_truth_pd(ph.blood, g, PC.GT_SIGMA)
    gimg = post.render_db(gt, PC.DR_DB, post.DbScale.power)
    img = post.render_db(vg(pd_ref, g.dims), PC.DR_DB, post.DbScale.power)
    m = post.metrics(img, gimg)
    assert abs(m.ssim - m_ref["ssim"]) < 1e-9 and abs(m.psnr - m_ref["psnr"]) < 1e-9
