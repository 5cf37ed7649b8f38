"""ctypes bindings for the CPU oracle (TEST INFRASTRUCTURE ONLY).

Two libraries, both built by ``oracle/Makefile``:

* ``liboracle.so`` -- this repo's FP64 C restatement of the reference hot path
  (``oracle/fqf_oracle.c``; every function cites the reference file:line it
  restates).
* ``_ref/libfqf_ref.so`` -- the reference's own unmodified C++ sources compiled
  in place (``oracle/ref_capi.cpp`` wraps ``rf_to_iq``, ``plan_chunks``,
  ``das_reconstruct``, ``power_doppler``, ``render_db`` and ``metrics``).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs import
this module.  The product package ``paper_2509_05464_b200`` never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libfqf_ref.so")

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")


class OracleError(RuntimeError):
    """A contract violation reported by the oracle (mirrors fqf::Error)."""


def build() -> None:
    """Compile liboracle.so (and _ref when /root/reference is present)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


_lib = None
_ref = None


class OTransducer(C.Structure):
    """oracle_transducer (fqf_oracle.h): the rf::Transducer fields the simulator reads."""
    _fields_ = [("n_elements", C.c_int), ("xyz", C.POINTER(C.c_double)),
                ("half_width", C.c_double), ("subelements", C.c_int), ("pitch", C.c_double),
                ("center_frequency", C.c_double), ("fractional_bandwidth", C.c_double),
                ("elevation_height", C.c_double), ("elevation_focus", C.c_double),
                ("elevation_core_weight", C.c_double), ("elevation_tail_weight", C.c_double),
                ("elevation_aperture_factor", C.c_double)]


class OMedium(C.Structure):
    _fields_ = [("c", C.c_double), ("attenuation_db_cm_mhz", C.c_double),
                ("min_fs_ratio", C.c_double)]


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(ORACLE_SO):
            build()
        L = C.CDLL(ORACLE_SO)
        L.oracle_last_error.restype = C.c_char_p
        L.oracle_rf_to_iq.argtypes = [_dp, C.c_int, C.c_int, C.c_double, C.c_double, C.c_double,
                                      C.c_int, _dp]
        L.oracle_plan_chunks.restype = C.c_long
        L.oracle_plan_chunks.argtypes = [C.c_size_t, C.c_int, C.c_size_t, C.c_void_p]
        L.oracle_das.argtypes = [_dp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, _dp, _dp,
                                 _dp, C.c_void_p, C.c_void_p, _dp, C.POINTER(C.c_uint64)]
        L.oracle_power_doppler.argtypes = [_dp, C.c_int, C.c_size_t, _dp]
        L.oracle_svd_filter.argtypes = [_dp, C.c_int, C.c_size_t, C.c_int, C.c_int, C.c_void_p,
                                        C.c_void_p, C.c_void_p]
        L.oracle_gram_filter.argtypes = [_dp, C.c_int, C.c_size_t, C.c_int, C.c_int, C.c_void_p,
                                         C.c_void_p]
        L.oracle_heev.argtypes = [_dp, C.c_int, _dp, _dp]
        pi = C.POINTER(C.c_int)
        L.oracle_simulate_rf.argtypes = [_dp, _dp, C.c_size_t, C.POINTER(OTransducer), _dp, _dp,
                                         C.POINTER(OMedium), C.c_double, C.c_double,
                                         C.c_size_t, _dp, pi, pi]
        L.oracle_reference_rf.argtypes = [_dp, _dp, C.c_size_t, C.POINTER(OTransducer), _dp, _dp,
                                          C.POINTER(OMedium), C.c_double, C.c_double, _dp, pi, pi]
        L.oracle_rf_passband.argtypes = [C.POINTER(OTransducer), C.c_double, C.c_double, pi, pi,
                                         pi, C.POINTER(C.c_double)]
        _lib = L
    return _lib


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref() -> C.CDLL:
    global _ref
    if _ref is None:
        if not os.path.exists(REF_SO):
            raise OracleError(f"{REF_SO} not built (needs /root/reference at build time)")
        L = C.CDLL(REF_SO)
        L.ref_last_error.restype = C.c_char_p
        L.ref_mt19937_uniform.argtypes = [C.c_uint32, C.c_size_t, C.c_double, C.c_double, _dp]
        L.ref_mt19937_64_normal.argtypes = [C.c_uint64, C.c_size_t, _dp]
        L.ref_rf_to_iq.argtypes = [_dp, C.c_int, C.c_int, C.c_double, C.c_double, C.c_double,
                                   C.c_int, _dp]
        L.ref_plan_chunks.restype = C.c_long
        L.ref_plan_chunks.argtypes = [C.c_size_t, C.c_int, C.c_size_t, C.c_void_p]
        L.ref_das.argtypes = [_dp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, _dp, _dp, _dp,
                              C.POINTER(C.c_int), _dp, _dp, C.c_double, C.c_double, C.c_double,
                              C.c_int, C.c_int, C.c_size_t, C.c_size_t, C.c_int, _dp,
                              C.POINTER(C.c_uint64)]
        L.ref_power_doppler.argtypes = [_dp, C.c_int, C.POINTER(C.c_int), _dp]
        _vp = C.c_void_p
        L.ref_simulate_rf.argtypes = [_dp, _dp, C.c_size_t, C.c_int, _dp, C.c_int, _dp, _dp, _dp,
                                      C.c_double, _dp, C.c_size_t, C.c_double, C.c_double,
                                      C.c_int, C.c_size_t, _vp, C.POINTER(C.c_int), _vp]
        L.ref_compose_frames.argtypes = [_dp, _dp, C.POINTER(C.c_int), _dp, _dp,
                                         C.POINTER(C.c_int), C.c_int, C.c_int, C.c_int, _dp,
                                         C.c_int, _dp, _dp, _dp, C.c_double, _dp, C.c_size_t,
                                         C.c_double, C.c_double, _vp, C.POINTER(C.c_int), _vp]
        L.ref_delay_matrix_build.restype = C.c_longlong
        L.ref_delay_matrix_build.argtypes = [_dp, C.c_size_t, C.c_double, C.c_double, C.c_double,
                                             C.c_int, C.c_int, _dp, C.c_double, C.c_double,
                                             C.c_double, C.c_int]
        L.ref_delay_matrix_fetch.argtypes = [C.c_void_p] * 3 + [C.POINTER(C.c_uint64),
                                                                C.POINTER(C.c_int)]
        L.ref_render_db.argtypes = [_dp, C.POINTER(C.c_int), C.c_double, C.c_int, _dp]
        L.ref_metrics.argtypes = [_dp, _dp, C.POINTER(C.c_int), _dp]
        L.ref_bmode.argtypes = [_dp, C.POINTER(C.c_int), C.c_double, _dp]
        L.ref_mip.argtypes = [_dp, C.POINTER(C.c_int), C.c_int, _dp]
        L.ref_ground_truth_pd.argtypes = [_dp, C.POINTER(C.c_int), C.c_int, C.POINTER(C.c_int),
                                          _dp, _dp, C.c_double, _dp]
        _cs = C.c_char_p
        L.ref_write_grid.argtypes = [_cs, C.POINTER(C.c_int), _dp, _dp, _dp]
        L.ref_write_pgm.argtypes = [_cs, C.POINTER(C.c_int), _dp]
        L.ref_write_iq_volume.argtypes = [_cs, C.POINTER(C.c_int), _dp, _dp, C.c_int, C.c_int, _dp]
        L.ref_metrics_text.argtypes = [_dp, _dp, C.POINTER(C.c_int), C.c_char_p, C.c_int,
                                       C.c_char_p, C.c_int]
        _ref = L
    return _ref


def _c(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _cplx_out(shape):
    return np.zeros(tuple(shape) + (2,), dtype=np.float64)


def _as_complex(a):
    return a[..., 0] + 1j * a[..., 1]


def _chk(rc, L, fn="oracle_last_error"):
    if rc:
        raise OracleError(getattr(L, fn)().decode())


# ------------------------------------------------------------------ oracle --

class _Grid(C.Structure):
    _fields_ = [("dims", C.c_int * 3), ("spacing", C.c_double * 3), ("origin", C.c_double * 3)]


class _Bf(C.Structure):
    _fields_ = [("c", C.c_double), ("fc", C.c_double), ("f_number", C.c_double),
                ("interp_order", C.c_int), ("lowpass_taps", C.c_int)]


def lowpass_kernel(fc, fs, taps):
    h = np.zeros(taps)
    L = lib()
    L.oracle_lowpass_kernel.argtypes = [C.c_double, C.c_double, C.c_int, _dp]
    L.oracle_lowpass_kernel(fc, fs, taps, h)
    return h


def rf_to_iq(rf, fs, t0, fc, taps=33):
    """rf [T][E] -> complex [T][E] (iq.cpp:34-82)."""
    rf = _c(rf)
    T, E = rf.shape
    out = _cplx_out((T, E))
    L = lib()
    _chk(L.oracle_rf_to_iq(rf, T, E, fs, t0, fc, taps, out), L)
    return _as_complex(out)


def plan_chunks(n, a, budget):
    L = lib()
    k = L.oracle_plan_chunks(n, a, budget, None)
    if k < 0:
        raise OracleError(L.oracle_last_error().decode())
    r = np.zeros(2 * k, dtype=np.uint64)
    L.oracle_plan_chunks(n, a, budget, r.ctypes.data)
    return [(int(r[2 * i]), int(r[2 * i + 1])) for i in range(k)]


def das(rf, fs, t0, angles, elements, dims, spacing, origin, c=1540.0, fc=None, f_number=1.5,
        interp_order=1, lowpass_taps=33):
    """Literal DAS; rf [F][A][T][E]. Returns (iq [F][N] complex, out_of_window)."""
    rf = _c(rf)
    F, A, T, E = rf.shape
    g = _Grid((C.c_int * 3)(*dims), (C.c_double * 3)(*spacing), (C.c_double * 3)(*origin))
    b = _Bf(c, fc, f_number, interp_order, lowpass_taps)
    N = int(np.prod(dims))
    out = _cplx_out((F, N))
    oow = C.c_uint64(0)
    L = lib()
    _chk(L.oracle_das(rf, F, A, T, E, fs, _c(np.broadcast_to(t0, (A,))), _c(angles),
                      _c(elements), C.byref(g), C.byref(b), out, C.byref(oow)), L)
    return _as_complex(out), int(oow.value)


def power_doppler(iq):
    """iq complex [F][N] -> PD [N] (render.cpp:23-42)."""
    iq = np.asarray(iq)
    F, N = iq.shape
    x = _c(np.stack([iq.real, iq.imag], axis=-1))
    pd = np.zeros(N)
    lib().oracle_power_doppler(x, F, N, pd)
    return pd


def svd_filter(iq, lo, hi, want_corr=False, method="jacobi"):
    """Casorati SVD filter (svd.cpp:29-93). Returns (filtered, sigma, corr|None)."""
    iq = np.asarray(iq)
    F, N = iq.shape
    x = _c(np.stack([iq.real, iq.imag], axis=-1))
    out = _cplx_out((F, N))
    sigma = np.zeros(F)
    L = lib()
    if method == "jacobi":
        corr = np.zeros((F, F)) if want_corr else None
        _chk(L.oracle_svd_filter(x, F, N, lo, hi, out.ctypes.data, sigma.ctypes.data,
                                 corr.ctypes.data if want_corr else None), L)
    else:
        corr = None
        _chk(L.oracle_gram_filter(x, F, N, lo, hi, out.ctypes.data, sigma.ctypes.data), L)
    return _as_complex(out), sigma, corr


def heev(a):
    a = np.asarray(a, dtype=np.complex128)
    F = a.shape[0]
    x = _c(np.stack([a.real, a.imag], axis=-1))
    w = np.zeros(F)
    v = _cplx_out((F, F))
    lib().oracle_heev(x, F, w, v)
    return w, _as_complex(v)


# --------------------------------------------------------------------- _ref --

def ref_uniform(seed, n, lo=-1.0, hi=1.0):
    out = np.zeros(n)
    ref().ref_mt19937_uniform(seed, n, lo, hi, out)
    return out


def ref_normal(seed, n):
    out = np.zeros(n)
    ref().ref_mt19937_64_normal(seed, n, out)
    return out


def ref_rf_to_iq(rf, fs, t0, fc, taps=33):
    rf = _c(rf)
    T, E = rf.shape
    out = _cplx_out((T, E))
    L = ref()
    _chk(L.ref_rf_to_iq(rf, T, E, fs, t0, fc, taps, out), L, "ref_last_error")
    return _as_complex(out)


def ref_plan_chunks(n, a, budget):
    L = ref()
    k = L.ref_plan_chunks(n, a, budget, None)
    if k < 0:
        raise OracleError(L.ref_last_error().decode())
    r = np.zeros(2 * k, dtype=np.uint64)
    L.ref_plan_chunks(n, a, budget, r.ctypes.data)
    return [(int(r[2 * i]), int(r[2 * i + 1])) for i in range(k)]


def ref_das(rf, fs, t0, angles, elements, dims, spacing, origin, c=1540.0, fc=None,
            f_number=1.5, interp_order=1, lowpass_taps=33, memory_budget=100_000_000,
            matrix_budget=512_000_000, cache=True):
    """The reference's das_reconstruct. Returns (iq [F][N] complex, stats dict)."""
    rf = _c(rf)
    F, A, T, E = rf.shape
    N = int(np.prod(dims))
    out = _cplx_out((F, N))
    st = (C.c_uint64 * 5)()
    L = ref()
    _chk(L.ref_das(rf, F, A, T, E, fs, _c(np.broadcast_to(t0, (A,))), _c(angles), _c(elements),
                   (C.c_int * 3)(*dims), _c(spacing), _c(origin), c, fc, f_number, interp_order,
                   lowpass_taps, memory_budget, matrix_budget, int(cache), out, st),
         L, "ref_last_error")
    keys = ("chunks", "matrix_builds", "out_of_window", "matrix_bytes_peak",
            "accumulator_bytes_peak")
    return _as_complex(out), dict(zip(keys, (int(v) for v in st)))


def ref_build_delay_matrix(voxels, angle, t0, fs, n_samples, elements, c=1540.0, fc=None,
                           f_number=1.5, interp_order=1):
    """The reference's build_delay_matrix: (row_ptr uint64 [n+1], col_idx int32
    [nnz], values complex [nnz], out_of_window, padded_samples)."""
    vox = _c(voxels).reshape(-1, 3)
    el = _c(elements).reshape(-1, 3)
    L = ref()
    nnz = L.ref_delay_matrix_build(vox, vox.shape[0], angle, t0, fs, n_samples, el.shape[0], el,
                                   c, fc, f_number, interp_order)
    if nnz < 0:
        raise OracleError(L.ref_last_error().decode())
    rp = np.zeros(vox.shape[0] + 1, np.uint64)
    col = np.zeros(nnz, np.int32)
    val = np.zeros((nnz, 2))
    oow, pad = C.c_uint64(), C.c_int()
    L.ref_delay_matrix_fetch(rp.ctypes.data_as(C.c_void_p), col.ctypes.data_as(C.c_void_p),
                             val.ctypes.data_as(C.c_void_p), C.byref(oow), C.byref(pad))
    return rp, col, val[:, 0] + 1j * val[:, 1], oow.value, pad.value


def _td_params(td):
    el = _c(np.asarray(td.elements, np.float64).reshape(-1, 3))
    tp = _c([td.half_width, td.pitch, td.center_frequency, td.fractional_bandwidth,
             td.elevation_height, td.elevation_focus, td.elevation_core_weight,
             td.elevation_tail_weight, td.elevation_aperture_factor])
    return el, tp


def ref_simulate_rf(positions, refl, td, delays, apod, angle=0.0, c=1540.0, att=0.5,
                    min_fs_ratio=4.0, budget=2_000_000_000, fs=20e6, duration=20e-6,
                    chunked=False, chunk_budget=0):
    """The reference's own rf::simulate_rf (or simulate_rf_chunked) from
    simulate.cpp, compiled with oracle/fftw_stub: (RF [T][E] float64, stats)."""
    L = ref()
    el, tp = _td_params(td)
    pos = _c(np.asarray(positions, np.float64).reshape(-1, 3))
    rr = _c(np.asarray(refl, np.float64).ravel())
    med = _c([c, att, min_fs_ratio])
    T = C.c_int()
    st = (C.c_uint64 * 4)()
    args = (pos, rr, pos.shape[0], el.shape[0], el, int(td.subelements), tp, _c(delays),
            _c(apod), angle, med, budget, fs, duration, int(chunked), chunk_budget)
    sp = C.cast(st, C.c_void_p)
    _chk(L.ref_simulate_rf(*args, None, C.byref(T), sp), L, "ref_last_error")
    out = np.zeros((T.value, el.shape[0]))
    _chk(L.ref_simulate_rf(*args, out.ctypes.data, C.byref(T), sp), L, "ref_last_error")
    keys = ("blocks", "frequencies", "peak_tracked_bytes", "pair_bin_products")
    return out, dict(zip(keys, (int(v) for v in st)))


def ref_compose_frames(tissue, flow, static_tissue, td, delays, apod, angle=0.0, c=1540.0,
                       att=0.5, min_fs_ratio=4.0, budget=2_000_000_000, fs=20e6,
                       duration=20e-6):
    """The reference's rf::compose_frames: tissue / flow = lists of
    (positions [n][3], reflectivity [n]); returns (RF [F][T][E], stats)."""
    L = ref()
    el, tp = _td_params(td)
    F = len(flow)
    tl = list(tissue) + [(np.zeros((0, 3)), np.zeros(0))] * (F - len(tissue))

    def cat(frames):
        pos = _c(np.concatenate([np.asarray(p, np.float64).reshape(-1, 3) for p, _ in frames]
                                + [np.zeros((1, 3))]))
        ref_ = _c(np.concatenate([np.asarray(r, np.float64).ravel() for _, r in frames]
                                 + [np.zeros(1)]))
        cnt = (C.c_int * F)(*[np.asarray(r).size for _, r in frames])
        return pos, ref_, cnt

    tp_, tr_, tc_ = cat(tl[:F])
    fp_, fr_, fc_ = cat(flow)
    T = C.c_int()
    st = (C.c_int * 2)()
    args = (tp_, tr_, tc_, fp_, fr_, fc_, F, int(static_tissue), el.shape[0], el,
            int(td.subelements), tp, _c(delays), _c(apod), angle, _c([c, att, min_fs_ratio]),
            budget, fs, duration)
    sp = C.cast(st, C.c_void_p)
    _chk(L.ref_compose_frames(*args, None, C.byref(T), sp), L, "ref_last_error")
    out = np.zeros((F, T.value, el.shape[0]))
    _chk(L.ref_compose_frames(*args, out.ctypes.data, C.byref(T), sp), L, "ref_last_error")
    return out, {"tissue_simulations": st[0], "flow_simulations": st[1]}


def ref_power_doppler(iq, dims):
    iq = np.asarray(iq)
    F, N = iq.shape
    x = _c(np.stack([iq.real, iq.imag], axis=-1))
    pd = np.zeros(N)
    L = ref()
    _chk(L.ref_power_doppler(x, F, (C.c_int * 3)(*dims), pd), L, "ref_last_error")
    return pd


def ref_render_db(vol, dims, dr_db=60.0, power=True):
    vol = _c(vol).ravel()
    out = np.zeros_like(vol)
    L = ref()
    _chk(L.ref_render_db(vol, (C.c_int * 3)(*dims), dr_db, int(power), out), L, "ref_last_error")
    return out


def ref_metrics(test, refimg, dims):
    out = np.zeros(3)
    L = ref()
    _chk(L.ref_metrics(_c(test).ravel(), _c(refimg).ravel(), (C.c_int * 3)(*dims), out), L,
         "ref_last_error")
    return {"mse": out[0], "psnr": out[1], "ssim": out[2]}


def ref_ground_truth_pd(positions_per_frame, dims, spacing, origin, sigma_voxels=1.0):
    """The reference's ground_truth_pd (render.cpp:106-145) over blood
    scatterer positions [frame] -> [n][3]."""
    counts = (C.c_int * len(positions_per_frame))(*[len(p) for p in positions_per_frame])
    xyz = _c(np.concatenate([np.asarray(p, np.float64).reshape(-1, 3)
                             for p in positions_per_frame]))
    out = np.zeros(int(np.prod(dims)))
    L = ref()
    _chk(L.ref_ground_truth_pd(xyz, counts, len(positions_per_frame), (C.c_int * 3)(*dims),
                               _c(spacing), _c(origin), sigma_voxels, out), L, "ref_last_error")
    return out


def ref_bmode(iq, dims, dr_db=75.0):
    """The reference's bmode (render.cpp:70-78) of a complex volume."""
    iq = np.asarray(iq, np.complex128).ravel()
    x = _c(np.stack([iq.real, iq.imag], axis=-1))
    out = np.zeros(iq.size)
    L = ref()
    _chk(L.ref_bmode(x, (C.c_int * 3)(*dims), dr_db, out), L, "ref_last_error")
    return out


def ref_mip(vol, dims, axis):
    """The reference's mip (render.cpp:80-104)."""
    od = list(dims)
    od[axis] = 1
    out = np.zeros(int(np.prod(od)))
    L = ref()
    _chk(L.ref_mip(_c(vol).ravel(), (C.c_int * 3)(*dims), axis, out), L, "ref_last_error")
    return out


def _otd(td):
    el = np.ascontiguousarray(np.asarray(td.elements, np.float64).reshape(-1, 3))
    t = OTransducer(el.shape[0], el.ctypes.data_as(C.POINTER(C.c_double)), td.half_width,
                    td.subelements, td.pitch, td.center_frequency, td.fractional_bandwidth,
                    td.elevation_height, td.elevation_focus, td.elevation_core_weight,
                    td.elevation_tail_weight, td.elevation_aperture_factor)
    return t, el


def rf_passband(td, fs, duration):
    t, keep = _otd(td)
    T, lo, hi, df = C.c_int(), C.c_int(), C.c_int(), C.c_double()
    rc = lib().oracle_rf_passband(C.byref(t), fs, duration, C.byref(T), C.byref(lo), C.byref(hi),
                                  C.byref(df))
    if rc:
        raise ValueError(f"passband error {rc}")
    return T.value, lo.value, hi.value, df.value


def _rf_call(fn, positions, refl, td, delays, apod, c, att, fs, duration, *extra):
    t, keep = _otd(td)
    pos = _c(np.asarray(positions, np.float64).reshape(-1, 3))
    rr = _c(refl)
    T, _, _, _ = rf_passband(td, fs, duration)
    out = np.zeros((T, t.n_elements))
    med = OMedium(c, att, 4.0)
    ns, nb = C.c_int(), C.c_int()
    rc = fn(pos, rr, pos.shape[0], C.byref(t), _c(delays), _c(apod), C.byref(med), fs, duration,
            *extra, out, C.byref(ns), C.byref(nb))
    if rc:
        raise ValueError(f"simulate error {rc}")
    return out


def simulate_rf(positions, refl, td, delays, apod, c=1540.0, att=0.5, fs=20e6, duration=20e-6,
                block_scatterers=0):
    """The simulate_rf engine restatement (fqf_rfsim.c): RF [T][E] float64."""
    return _rf_call(lib().oracle_simulate_rf, positions, refl, td, delays, apod, c, att, fs,
                    duration, int(block_scatterers))


def reference_rf(positions, refl, td, delays, apod, c=1540.0, att=0.5, fs=20e6, duration=20e-6):
    """test_rf.cpp:51-124 restated literally: RF [T][E] float64."""
    return _rf_call(lib().oracle_reference_rf, positions, refl, td, delays, apod, c, att, fs,
                    duration)


def ref_write_grid(path, data, dims, spacing, origin):
    """The reference's write_grid (grid.cpp:79-99) of a scalar f64 grid."""
    L = ref()
    _chk(L.ref_write_grid(str(path).encode(), (C.c_int * 3)(*dims), _c(spacing), _c(origin),
                          _c(data).ravel()), L, "ref_last_error")


def ref_write_pgm(path, data, dims):
    """The reference's write_pgm (render.cpp:147-175)."""
    L = ref()
    _chk(L.ref_write_pgm(str(path).encode(), (C.c_int * 3)(*dims), _c(data).ravel()), L,
         "ref_last_error")


def ref_write_iq_volume(path, iq, dims, spacing, origin, frame_index, n_angles):
    """The reference's write_iq_volume (das.cpp:395-407); iq complex [N]."""
    L = ref()
    z = np.ascontiguousarray(np.asarray(iq, np.complex128))
    _chk(L.ref_write_iq_volume(str(path).encode(), (C.c_int * 3)(*dims), _c(spacing), _c(origin),
                               int(frame_index), int(n_angles), z.view(np.float64).ravel()), L,
         "ref_last_error")


def ref_metrics_text(test, refimg, dims):
    """(metrics_csv, metrics_json) of the reference (metrics.cpp:114-126)."""
    L = ref()
    csv, js = C.create_string_buffer(512), C.create_string_buffer(512)
    _chk(L.ref_metrics_text(_c(test).ravel(), _c(refimg).ravel(), (C.c_int * 3)(*dims), csv, 512,
                            js, 512), L, "ref_last_error")
    return csv.value.decode(), js.value.decode()
