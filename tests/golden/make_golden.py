"""Regenerate tests/golden/*.npz from the REFERENCE (run in the build container).

Inputs are replayed exactly as the reference tests draw them (libstdc++
std::mt19937 / mt19937_64 via oracle/_ref's ref_mt19937_* helpers, in the same
order as proj/tests/test_beamform.cpp and test_post.cpp) or, for the larger
matrix-array / linear-array cases, from numpy's PCG64 with a stated seed.
Expected outputs come from the reference's own das_reconstruct / rf_to_iq /
plan_chunks / power_doppler (oracle/_ref/libfqf_ref.so, compiled from
/root/reference by oracle/Makefile) and, for the SVD filter whose Eigen
dependency is absent, from numpy.linalg.svd (LAPACK zgesdd).

Usage:  make -C oracle && python tests/golden/make_golden.py
"""
import json
import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", ".."))
from oracle import oracle as O  # noqa: E402

DEG = math.pi / 180.0


def small_probe(n):
    # test_beamform.cpp:34-47: pitch 0.3 mm, centred, y = z = 0.
    return np.array([[(i - (n - 1) / 2.0) * 0.3e-3, 0.0, 0.0] for i in range(n)])


def matrix32():
    # transducer.cpp:43-60: j outer, i inner, pitch 0.3 mm.
    return np.array([[(i - 15.5) * 0.3e-3, (j - 15.5) * 0.3e-3, 0.0]
                     for j in range(32) for i in range(32)])


def l11_4v():
    # transducer.cpp:26-41.
    return np.array([[(n - 63.5) * 0.3e-3, 0.0, 0.0] for n in range(128)])


def save(name, meta, **arrays):
    np.savez_compressed(os.path.join(HERE, name + ".npz"), meta=json.dumps(meta), **arrays)
    print("wrote", name, {k: v.shape for k, v in arrays.items()})


def numpy_rf(seed, shape):
    """RF for the larger cases: PCG64 uniform(-1, 1) rounded through f32 (the
    pipeline stores RF as f32, simulate.cpp:638-639).  Tests regenerate it
    from (seed, shape) instead of storing megabytes."""
    rng = np.random.default_rng(seed)
    return rng.uniform(-1, 1, size=shape).astype(np.float32).astype(np.float64)


def das_case(name, rf, fs, t0, angles, el, dims, spacing, origin, fc, rf_seed=None, **kw):
    opts = {k: kw.pop(k) for k in ("memory_budget", "matrix_budget", "cache") if k in kw}
    iq, stats = O.ref_das(rf, fs, t0, angles, el, dims, spacing, origin, fc=fc, **kw, **opts)
    meta = dict(fs=fs, t0=list(np.broadcast_to(t0, (len(angles),)).astype(float)),
                angles=list(map(float, angles)), dims=list(dims), spacing=list(spacing),
                origin=list(origin), fc=fc, stats=stats, **kw, **opts)
    if rf_seed is None:
        save(name, meta, rf=rf, elements=el, iq=iq)
    else:
        meta.update(rf_seed=rf_seed, rf_shape=list(rf.shape))
        save(name, meta, elements=el, iq=iq)
    return iq, stats


def main():
    # ---- test_beamform.cpp:385-424: literal-reference fixture (3 chunks) ----
    el8 = small_probe(8)
    F, A, T, E = 2, 2, 64, 8
    rf = O.ref_uniform(31, F * A * T * E).reshape(F, A, T, E)
    iq, st = das_case("das_kat", rf, 20e6, 0.25e-6, [-3 * DEG, 2 * DEG], el8, (7, 2, 5),
                      (0.2e-3, 0.3e-3, 0.2e-3), (-0.6e-3, -0.15e-3, 1.2e-3), 5e6,
                      memory_budget=16 * 24 * 2)
    assert st["chunks"] == 3 and st["matrix_builds"] == 6, st
    # Survey-recorded golden values.
    assert iq[0, 0] == complex(0.21767054125126079, -0.23091352539589127), iq[0, 0]
    assert iq[1, 0] == complex(-0.2515352884279673, 0.01450684879472558), iq[1, 0]
    das_case("das_kat_nearest", rf, 20e6, 0.25e-6, [-3 * DEG, 2 * DEG], el8, (7, 2, 5),
             (0.2e-3, 0.3e-3, 0.2e-3), (-0.6e-3, -0.15e-3, 1.2e-3), 5e6, interp_order=0)
    das_case("das_kat_fnum0", rf, 20e6, 0.25e-6, [-3 * DEG, 2 * DEG], el8, (7, 2, 5),
             (0.2e-3, 0.3e-3, 0.2e-3), (-0.6e-3, -0.15e-3, 1.2e-3), 5e6, f_number=0.0)

    # ---- 426-462: partition invariance (1 frame, 2 angles) ----
    rf = O.ref_uniform(41, 1 * 2 * 96 * 8).reshape(1, 2, 96, 8)
    das_case("das_partition", rf, 20e6, 0.0, [-2 * DEG, 3 * DEG], el8, (21, 1, 11),
             (0.15e-3, 0.2e-3, 0.25e-3), (-1.5e-3, 0.0, 1.5e-3), 5e6)

    # ---- 464-488: identical transmits ----
    el6 = small_probe(6)
    one = O.ref_uniform(47, 80 * 6).reshape(1, 1, 80, 6)
    das_case("das_identical", np.concatenate([one, one], axis=1), 20e6, 0.0, [0.0, 0.0], el6,
             (9, 1, 7), (0.2e-3, 0.2e-3, 0.2e-3), (-0.8e-3, 0.0, 1.0e-3), 5e6)

    # ---- 490-518: linearity (f1 then f2 drawn from one engine) ----
    both = O.ref_uniform(53, 2 * 72 * 6).reshape(2, 1, 72, 6)
    das_case("das_linearity", both, 20e6, 0.0, [1.5 * DEG], el6, (11, 1, 9),
             (0.15e-3, 0.2e-3, 0.2e-3), (-0.75e-3, 0.0, 0.8e-3), 5e6)

    # ---- 520-558: cached vs rebuilt, 2 chunks, 3 frames ----
    rf = O.ref_uniform(59, 3 * 2 * 64 * 6).reshape(3, 2, 64, 6)
    n = 10 * 1 * 8
    das_case("das_cached", rf, 20e6, 0.0, [-2 * DEG, 2 * DEG], el6, (10, 1, 8),
             (0.2e-3, 0.2e-3, 0.2e-3), (-0.9e-3, 0.0, 1.0e-3), 5e6,
             memory_budget=16 * ((n + 1) // 2) * 2)
    das_case("das_cached_off", rf, 20e6, 0.0, [-2 * DEG, 2 * DEG], el6, (10, 1, 8),
             (0.2e-3, 0.2e-3, 0.2e-3), (-0.9e-3, 0.0, 1.0e-3), 5e6,
             memory_budget=16 * ((n + 1) // 2) * 2, cache=False)

    # ---- 787-807: out-of-window echoes ----
    rf = O.ref_uniform(71, 24 * 4).reshape(1, 1, 24, 4)
    _, st = das_case("das_oow", rf, 20e6, 0.0, [0.0], small_probe(4), (3, 1, 4),
                     (0.2e-3, 0.2e-3, 2.0e-3), (-0.2e-3, 0.0, 1.0e-3), 5e6)
    assert st["out_of_window"] > 0

    # ---- matrix-array case (config B/C probe), numpy PCG64 RF ----
    rf = numpy_rf(20260816, (2, 3, 256, 1024))
    das_case("das_matrix32", rf, 12e6, 0.0, [-8 * DEG, 0.0, 8 * DEG], matrix32(), (6, 5, 4),
             (0.2567e-3, 0.2567e-3, 0.2567e-3), (-0.7e-3, -0.5e-3, 10.0e-3), 3e6,
             rf_seed=20260816)

    # ---- linear-array case (config A probe), numpy PCG64 RF, t0 != 0 ----
    rf = numpy_rf(7, (2, 3, 400, 128))
    das_case("das_l11", rf, 30.8e6, 1.0e-6, [-5 * DEG, 0.0, 5 * DEG], l11_4v(), (16, 1, 12),
             (0.1e-3, 0.1e-3, 0.1e-3), (-0.75e-3, 0.0, 5.0e-3), 7.7e6, rf_seed=7)

    # ---- demodulation: test_beamform.cpp:228-256 (random, 3 elements) ----
    rf = O.ref_uniform(17, 128 * 3).reshape(128, 3)
    save("demod_random", dict(fs=20e6, t0=0.0, fc=5e6, taps=33), rf=rf,
         iq=O.ref_rf_to_iq(rf, 20e6, 0.0, 5e6))
    rf = numpy_rf(3, (300, 64))
    save("demod_t0", dict(fs=12e6, t0=3.7e-6, fc=3e6, taps=21, rf_seed=3, rf_shape=[300, 64]),
         iq=O.ref_rf_to_iq(rf, 12e6, 3.7e-6, 3e6, 21))

    # ---- chunk plans: test_beamform.cpp:138-189 + random sweep (seed 3) ----
    cases = [(1_000_000, 5, 100_000_000), (1_000_000, 5, 10_000_000), (1, 5, 1_000), (3, 1, 24)]
    r = np.random.default_rng(3)
    for _ in range(60):
        na = int(r.integers(1, 8))
        cases.append((int(r.integers(1, 5001)), na, 16 * na + 1 + int(r.integers(0, 200_000))))
    plans = [O.ref_plan_chunks(*c) for c in cases]
    save("plan_chunks", dict(cases=cases, plans=plans))

    # ---- power Doppler on random complex (ref power_doppler) ----
    rng = np.random.default_rng(11)
    iq = rng.standard_normal((5, 24)) + 1j * rng.standard_normal((5, 24))
    save("pd_random", dict(dims=[4, 3, 2]), iq=iq, pd=O.ref_power_doppler(iq, (4, 3, 2)))

    # ---- SVD ensembles (test_post.cpp:135-251); expected from LAPACK ----
    def casorati_svd(x):
        u, s, vh = np.linalg.svd(x.T, full_matrices=False)  # X: N x F
        return u, s, vh

    def band(x, lo, hi):
        u, s, vh = casorati_svd(x)
        b = slice(lo - 1, hi)
        return ((u[:, b] * s[b]) @ vh[b, :]).T

    def corr_abs_u(x):
        u, _, _ = casorati_svd(x)
        m = np.abs(u)
        c = m - m.mean(axis=0)
        sd = np.sqrt((c * c).mean(axis=0))
        F = m.shape[1]
        out = np.eye(F)
        for i in range(F):
            for j in range(i + 1, F):
                den = sd[i] * sd[j]
                out[i, j] = out[j, i] = (c[:, i] @ c[:, j]) / (m.shape[0] * den) if den > 0 else 0
        return out

    # static ensemble, 10x1x20, 6 frames, mt19937_64(401)
    N = 200
    nz = O.ref_normal(401, 2 * N)
    pattern = nz[0::2] + 1j * nz[1::2]
    static = np.tile(pattern, (6, 1))
    u, s, vh = casorati_svd(static)
    save("svd_static", dict(dims=[10, 1, 20]), iq=static, sigma=s, band2=band(static, 2, 6))
    # bands, 15x2x10, 7 frames, mt19937_64(402), filled f outer / v inner
    N = 300
    nz = O.ref_normal(402, 2 * N * 7)
    ens = (nz[0::2] + 1j * nz[1::2]).reshape(7, N)
    _, s, _ = casorati_svd(ens)
    save("svd_bands", dict(dims=[15, 2, 10]), iq=ens, sigma=s, band13=band(ens, 1, 3),
         band4F=band(ens, 4, 7), band25=band(ens, 2, 5))
    # correlation, 12x1x14, 5 frames, mt19937_64(403)
    N = 168
    nz = O.ref_normal(403, 2 * N * 5)
    ens = (nz[0::2] + 1j * nz[1::2]).reshape(5, N)
    _, s, _ = casorati_svd(ens)
    save("svd_corr", dict(dims=[12, 1, 14]), iq=ens, sigma=s, corr=corr_abs_u(ens))
    # in-vessel, 20x1x20, 10 frames, mt19937_64(404): tissue first, then the
    # in-vessel increments in (frame, voxel) order from the same engine.
    N = 400
    vessel = np.array([(v % 20) in (8, 9) for v in range(N)])
    nz = O.ref_normal(404, 2 * N + 2 * 10 * int(vessel.sum()))
    tissue = (nz[0:2 * N:2] + 1j * nz[1:2 * N:2]) * 100.0
    at = 2 * N
    ens = np.zeros((10, N), dtype=complex)
    for f in range(10):
        for v in range(N):
            z = tissue[v]
            if vessel[v]:
                z = z + complex(nz[at], nz[at + 1])
                at += 2
            ens[f, v] = z
    _, s, _ = casorati_svd(ens)
    save("svd_vessel", dict(dims=[20, 1, 20]), iq=ens, sigma=s, band2=band(ens, 2, 10),
         vessel=vessel)


if __name__ == "__main__":
    main()
