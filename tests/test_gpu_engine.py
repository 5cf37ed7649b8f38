"""The C++ reconstruction engine (fqfg_recon_*, csrc/recon.cu) on a B200:
RF -> power Doppler for sequences of ensembles through the C ABI, against the
FP64 oracle and the kernel-by-kernel path (tolerances as test_gpu_parity)."""
import ctypes as C
import os

import numpy as np
import pytest

import paper_2509_05464_b200 as P
from oracle import oracle as O
from paper_2509_05464_b200 import workloads as W
from paper_2509_05464_b200.engine import Engine
from tests.golden_io import rel_l2

pytestmark = pytest.mark.gpu

IQ_REL_L2 = 1e-5
PD_REL_L2 = 1e-4
SIG_REL = 1e-5


def _engine(w, **kw):
    return Engine(w.fs, 0.0, w.angles, w.n_frames, w.n_samples, w.grid, w.elements, w.bf(), **kw)


def _oracle_pd(w, rf):
    g = w.grid
    iq, _ = O.das(rf.astype(np.float64), w.fs, 0.0, w.angles, w.elements, g.dims, g.spacing,
                  g.origin, fc=w.fc)
    y, s, _ = O.svd_filter(iq, 2, w.n_frames)
    return iq, O.power_doppler(y), s


def test_engine_sequence_matches_oracle():
    """Three different ensembles through one engine (pageable host buffers):
    each PD and singular-value set against the FP64 oracle chain, and the
    IQ of the last one."""
    w = W.small()
    rng = np.random.default_rng(31)
    rfs = [rng.uniform(-1, 1, w.rf_shape()).astype(np.float32) for _ in range(3)]
    eng = _engine(w)
    pds = [np.full(w.grid.num_points(), np.nan) for _ in rfs]
    sig = [np.full(w.n_frames, np.nan) for _ in rfs]
    eng.run(rfs, pds, sig)
    for rf, pd, s in zip(rfs, pds, sig):
        iq_ref, pd_ref, s_ref = _oracle_pd(w, rf)
        assert rel_l2(pd, pd_ref) < PD_REL_L2
        assert np.max(np.abs(s - s_ref) / s_ref[0]) < SIG_REL
    assert rel_l2(eng.copy_iq(), iq_ref) < IQ_REL_L2
    info = eng.info
    assert (info.v_begin, info.v_end) == (0, w.grid.num_points())
    assert info.h2d_bytes_per_ensemble == w.n_frames * w.n_angles * (
        info.t_end - info.t_begin) * w.n_elements * 4


def test_engine_host_and_device_sources_agree_with_step():
    """Host RF through the ring (pinned), device-resident RF read in place,
    and (with the FP64 Gram) the kernel-by-kernel Reconstructor.step give the
    same PD bits; the default tensor-core Gram agrees to 1e-7."""
    import torch
    from paper_2509_05464_b200 import pipeline as PL
    w = W.small()
    rng = np.random.default_rng(5)
    rf = rng.uniform(-1, 1, w.rf_shape()).astype(np.float32)
    h_rf = torch.from_numpy(rf).pin_memory()
    d_rf = torch.from_numpy(rf).cuda()
    eng = _engine(w, gram_fp64=True)
    assert eng.info.gram_fp64 == 1
    pd_host = np.zeros(w.grid.num_points())
    eng.run([h_rf], [pd_host])
    d_pd = torch.zeros(w.grid.num_points(), dtype=torch.float64, device="cuda")
    eng.run_dev([d_rf, d_rf], d_pd)
    rec = PL.Reconstructor(w.fs, 0.0, w.angles, w.n_frames, w.n_samples, w.grid, w.elements,
                           w.bf(), keep_lo=2)
    ref = rec.step(d_rf).pd.cpu().numpy()
    assert np.array_equal(pd_host, ref)
    assert np.array_equal(d_pd.cpu().numpy(), ref)
    tc = _engine(w)
    assert tc.info.gram_fp64 == 0
    pd_tc = np.zeros(w.grid.num_points())
    tc.run([h_rf], [pd_tc])
    assert rel_l2(pd_tc, ref) < 1e-7


@pytest.mark.parametrize("shape,ring,xbuf,F", [("4,12,8,4", 32, 1, 150), ("4,12,8,4", 16, 2, 150),
                                               (None, 48, 0, 230), (None, 0, 1, 40)])
def test_engine_multipass_ring_reuse(shape, ring, xbuf, F, monkeypatch):
    """Frame passes (fpass 64 -> 3 passes, or 208 -> 2), a ring smaller than
    a pass (every slot reused several times per ensemble), one or two X
    buffers, four ensembles: every PD equals the kernel-by-kernel path."""
    import torch
    from paper_2509_05464_b200 import pipeline as PL
    if shape:
        monkeypatch.setenv("FQFG_DAS_SHAPE", shape)
    sp = 0.2567e-3
    w = W.Workload("mp", W.matrix_probe(16), 3e6, 12e6, np.array([-4, 0, 4]) * W.DEG,
                   P.GridSpec((16, 8, 10), (sp, sp, sp), (-2e-3, -1e-3, 8e-3)), 300, F)
    rng = np.random.default_rng(F + ring)
    rfs = [rng.uniform(-1, 1, w.rf_shape()).astype(np.float32) for _ in range(4)]
    eng = _engine(w, ring_frames=ring, x_buffers=xbuf, gram_fp64=True)
    pds = [np.zeros(w.grid.num_points()) for _ in rfs]
    eng.run(rfs, pds)
    info = eng.info
    assert info.n_passes == (3 if shape else (2 if F > 208 else 1))
    if ring:
        assert info.ring_frames == ring
    rec = PL.Reconstructor(w.fs, 0.0, w.angles, w.n_frames, w.n_samples, w.grid, w.elements,
                           w.bf(), keep_lo=2)
    for rf, pd in zip(rfs, pds):
        ref = rec.step(torch.from_numpy(rf).cuda()).pd.cpu().numpy()
        assert np.array_equal(pd, ref)


def test_engine_zero_ensemble_fails_like_svd_filter():
    w = W.small()
    eng = _engine(w)
    rf = np.zeros(w.rf_shape(), np.float32)
    with pytest.raises(P.Error, match="nonzero ensemble"):
        eng.run([rf], [np.zeros(w.grid.num_points())])


def test_reconstruct_pd_reuses_engine_and_matches_oracle():
    """The one-shot C entry fqfg_reconstruct_pd (cached engine): PD and IQ
    against the oracle, twice (the second call reuses the plan)."""
    from paper_2509_05464_b200 import _native as N
    from paper_2509_05464_b200.beamform import _desc, _probe
    w = W.small()
    rng = np.random.default_rng(77)
    for _ in range(2):
        rf = rng.uniform(-1, 1, w.rf_shape()).astype(np.float32)
        desc, keep = _desc(w.n_frames, w.n_angles, w.n_samples, w.n_elements, w.fs, 0.0, w.angles)
        probe, el = _probe(w.elements)
        gc, bc = w.grid._c(), w.bf()._c()
        pd = np.zeros(w.grid.num_points())
        iq = np.zeros((w.n_frames, w.grid.num_points()), np.complex64)
        N.check(N.load().fqfg_reconstruct_pd(C.byref(desc), rf.ctypes.data, C.byref(gc),
                                             C.byref(probe), C.byref(bc), 2, w.n_frames,
                                             pd.ctypes.data, None, iq.ctypes.data))
        iq_ref, pd_ref, _ = _oracle_pd(w, rf)
        assert rel_l2(pd, pd_ref) < PD_REL_L2
        assert rel_l2(iq, iq_ref) < IQ_REL_L2


def _sharded_worker(rank, world, port, rf, out):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    cudart = C.CDLL("libcudart.so")

    def allreduce(ptr, n, stream):
        # stream-ordered sum over the ranks, through host memory (gloo)
        buf = np.empty(n, np.float64)
        if cudart.cudaStreamSynchronize(C.c_void_p(stream)):
            return 1
        if cudart.cudaMemcpy(C.c_void_p(buf.ctypes.data), C.c_void_p(ptr), C.c_size_t(8 * n), 2):
            return 2
        t = torch.from_numpy(buf)
        dist.all_reduce(t)
        return int(cudart.cudaMemcpy(C.c_void_p(ptr), C.c_void_p(buf.ctypes.data),
                                     C.c_size_t(8 * n), 1))

    w = _shard_workload()
    eng = _engine(w, rank=rank, world=world, allreduce=allreduce)
    info = eng.info
    pd = np.zeros(w.grid.num_points())
    eng.run([rf, rf], [pd, pd])
    out[rank] = (info.v_begin, info.v_end, pd[info.v_begin:info.v_end].copy(), info.t_begin,
                 info.t_end)
    dist.destroy_process_group()


def _shard_workload():
    sp = 0.2567e-3
    return W.Workload("sh", W.matrix_probe(16), 3e6, 12e6, np.array([-4, 0, 4]) * W.DEG,
                      P.GridSpec((16, 8, 24), (sp, sp, sp), (-2e-3, -1e-3, 6e-3)), 400, 24)


def test_engine_depth_slabs_with_allreduce_callback():
    """world = 2 engines (two processes on one GPU, the Gram summed by a
    caller all-reduce over gloo): each rank reconstructs its depth slab from
    its RF window; together the slabs give the single-engine PD."""
    import torch.multiprocessing as mp
    w = _shard_workload()
    rf = np.random.default_rng(3).uniform(-1, 1, w.rf_shape()).astype(np.float32)
    ref = np.zeros(w.grid.num_points())
    _engine(w).run([rf], [ref])
    ctx = mp.get_context("spawn")
    with ctx.Manager() as m:
        out = m.dict()
        port = 29500 + os.getpid() % 1000
        procs = [ctx.Process(target=_sharded_worker, args=(r, 2, port, rf, out)) for r in range(2)]
        for p_ in procs:
            p_.start()
        for p_ in procs:
            p_.join(300)
        assert all(p_.exitcode == 0 for p_ in procs)
        res = dict(out)
    pd = np.zeros_like(ref)
    (a0, b0, p0, _, _), (a1, b1, p1, tb1, te1) = res[0], res[1]
    assert a0 == 0 and b0 == a1 and b1 == w.grid.num_points() and 0 < a1 < b1
    assert tb1 > 0  # the deep slab never reads the first echoes
    pd[a0:b0], pd[a1:b1] = p0, p1
    assert rel_l2(pd, ref) < 1e-7  # per-slab digit scales: the tensor-core Grams differ ~1e-9


def test_engine_rf_broadcast_path_on_one_rank():
    """The NVLink distribution mode (rf_broadcast: rank 0 uploads each RF
    chunk once and ncclBroadcast carries it to every rank) through a
    one-rank NCCL communicator: same PD bits as the plain host upload."""
    from paper_2509_05464_b200.engine import nccl_unique_id
    w = W.small()
    rng = np.random.default_rng(17)
    rfs = [rng.uniform(-1, 1, w.rf_shape()).astype(np.float32) for _ in range(2)]
    ref = [np.zeros(w.grid.num_points()) for _ in rfs]
    _engine(w).run(rfs, ref)
    eng = _engine(w, nccl_id=nccl_unique_id(), rf_broadcast=True, ring_frames=16)
    assert eng.info.nccl == 1
    got = [np.zeros(w.grid.num_points()) for _ in rfs]
    eng.run(rfs, got)
    for a, b in zip(got, ref):
        assert np.array_equal(a, b)


def test_engine_rank_windows_and_h2d_bytes():
    """Per-rank RF windows of a depth-slab split (world 2, callback
    all-reduce: nothing runs): deeper slabs read later samples, the slabs
    tile the grid, and with rf_broadcast-style accounting only rank 0 would
    upload.  (scripts/shard_plan.py prints the same at config C for N = 2,
    4, 8.)"""
    sp = 0.2567e-3
    w = W.Workload("sh", W.matrix_probe(16), 3e6, 12e6, np.array([-4, 0, 4]) * W.DEG,
                   P.GridSpec((16, 8, 24), (sp, sp, sp), (-2e-3, -1e-3, 6e-3)), 400, 24)
    infos = [_engine(w, rank=r, world=2, allreduce=lambda *a: 0).info for r in range(2)]
    assert infos[0].v_begin == 0 and infos[0].v_end == infos[1].v_begin
    assert infos[1].v_end == w.grid.num_points()
    assert infos[1].t_begin > infos[0].t_begin and infos[1].t_end >= infos[0].t_end
    for i in infos:
        assert i.h2d_bytes_per_ensemble == w.n_frames * w.n_angles * (i.t_end - i.t_begin) * \
            w.n_elements * 4


@pytest.mark.parametrize("F,E,A,dims,T", [
    (2, 7, 1, (3, 2, 2), 64),        # two frames, ragged tiles, E not a multiple of 32
    (17, 33, 3, (11, 1, 13), 120),   # 2-D grid, one 16-frame chunk + a partial one
    (230, 16, 2, (6, 4, 10), 80),    # two frame passes, 15 chunks, the last one partial
])
def test_engine_edge_shapes_match_oracle(F, E, A, dims, T):
    """The engine at the edges of its chunking and the kernels' tiling: PD
    and IQ against the FP64 oracle chain."""
    rng = np.random.default_rng(F * 31 + E)
    fs, fc = 20e6, 5e6
    el = np.stack([(np.arange(E) - (E - 1) / 2) * 0.3e-3, np.zeros(E), np.zeros(E)], axis=1)
    angles = np.linspace(-0.05, 0.05, A) if A > 1 else np.array([0.02])
    sp = 0.2e-3
    g = P.GridSpec(dims, (sp, sp, sp), (-(dims[0] - 1) * sp / 2, -(dims[1] - 1) * sp / 2, 1.5e-3))
    rf = rng.uniform(-1, 1, (F, A, T, E)).astype(np.float32)
    bp = P.BeamformParams(c=1540.0, center_frequency=fc, f_number=1.0)
    eng = Engine(fs, 0.0, angles, F, T, g, el, bp)
    pd = np.zeros(g.num_points())
    eng.run([rf], [pd])
    iq_ref, _ = O.das(rf.astype(np.float64), fs, 0.0, angles, el, g.dims, g.spacing, g.origin,
                      fc=fc, f_number=1.0)
    assert rel_l2(eng.copy_iq(), iq_ref) < IQ_REL_L2
    y, _, _ = O.svd_filter(iq_ref, 2, F)
    assert rel_l2(pd, O.power_doppler(y)) < PD_REL_L2
