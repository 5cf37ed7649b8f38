// recon.cu -- the reconstruction engine behind fqfg_recon_* (include/fqfgpu.h):
// the C++ host side of run_beamform + run_post (proj/src/pipeline/run.cpp:
// 397-487) fused on one device, RF in, power Doppler out, with the IQ
// ensemble never leaving HBM.
//
// One engine = one device = one depth slab of the grid (the whole grid when
// world = 1).  Per ensemble k (buffer b = k % nbuf):
//
//   copy stream   RF frames, 16 at a time, host -> a ring of chunk slots
//                 (only samples [t_begin, t_end) of each channel: what the
//                 slab's voxels can read through the FIR)
//   work stream   per chunk: wait for its upload, demodulate its frames into
//                 the frame-pass IQ buffer, release the ring slot; per frame
//                 pass: the DAS of the slab's planes into X[b] [F][N_slab]
//   filter stream Gram of X[b] -> [Gram all-reduce over the ranks] ->
//                 eigensolve (the vectors the band needs) -> projection +
//                 fused PD -> [PD slabs to rank 0] -> host
//
// The ring lets the upload of the next chunks (next pass, next ensemble)
// run during the DAS; the filter of ensemble k runs during the demod + DAS of
// ensemble k + 1 when two X buffers fit (nbuf = 2), else it overlaps only
// the next ensemble's first demodulation.  The only collectives are one F x
// F complex128 sum and the PD gather; they are NCCL (opened
// at run time, libnccl.so.2) or a caller-supplied all-reduce.
//
// Memory per rank (config C, one GPU): IQ pass 11.8 GB, X 2 x 3.4 GB, ring
// 2 ensembles x 4.4 GB; config D: IQ pass (112 frames) 65 GB, X 1 x 40 GB,
// ring sized to what is left.

#include <dlfcn.h>
#include <nccl.h>  // types only: the library is opened with dlopen

namespace {

constexpr int kChunk = 16;  // frames per upload / demodulation chunk (kFusedG)

struct NcclApi {
  bool ok = false;
  std::string why;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t,
                       cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*CommSplit)(ncclComm_t, int, int, ncclComm_t*, ncclConfig_t*) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl_api() {
  static NcclApi api = [] {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      a.why = dlerror() ? dlerror() : "dlopen(libnccl.so.2) failed";
      return a;
    }
    auto sym = [&](const char* n) { return dlsym(h, n); };
    a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(sym("ncclGetUniqueId"));
    a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(sym("ncclCommInitRank"));
    a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(sym("ncclCommDestroy"));
    a.AllReduce = reinterpret_cast<decltype(a.AllReduce)>(sym("ncclAllReduce"));
    a.Send = reinterpret_cast<decltype(a.Send)>(sym("ncclSend"));
    a.Recv = reinterpret_cast<decltype(a.Recv)>(sym("ncclRecv"));
    a.GroupStart = reinterpret_cast<decltype(a.GroupStart)>(sym("ncclGroupStart"));
    a.Broadcast = reinterpret_cast<decltype(a.Broadcast)>(sym("ncclBroadcast"));
    a.CommSplit = reinterpret_cast<decltype(a.CommSplit)>(sym("ncclCommSplit"));
    a.GroupEnd = reinterpret_cast<decltype(a.GroupEnd)>(sym("ncclGroupEnd"));
    a.GetErrorString = reinterpret_cast<decltype(a.GetErrorString)>(sym("ncclGetErrorString"));
    a.ok = a.GetUniqueId && a.CommInitRank && a.CommDestroy && a.AllReduce && a.Send && a.Recv &&
           a.GroupStart && a.GroupEnd && a.GetErrorString && a.Broadcast && a.CommSplit;
    if (!a.ok) a.why = "libnccl.so.2 lacks a required symbol";
    return a;
  }();
  return api;
}

#define NCK(x)                                                                     \
  do {                                                                             \
    ncclResult_t r_ = (x);                                                         \
    if (r_ != ncclSuccess)                                                         \
      fail(FQFG_ECUDA, "NCCL error %d (%s) at %s:%d", (int)r_,                     \
           nccl_api().GetErrorString(r_), __FILE__, __LINE__);                     \
  } while (0)

// Active (voxel, element) pairs per z-plane (das.cpp:165-168), exact: the
// depth-slab balance weight (the aperture widens with depth).
__global__ void plane_active_kernel(DasParams p, unsigned long long* out) {
  const size_t n = (size_t)p.nx * p.ny * p.nz;
  const size_t v = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= n) return;
  const int i = (int)(v % p.nx), j = (int)((v / p.nx) % p.ny), k = (int)(v / ((size_t)p.nx * p.ny));
  const double px = grid_coord(p.ox, i, p.sx), py = grid_coord(p.oy, j, p.sy),
               pz = grid_coord(p.oz, k, p.sz);
  unsigned long long c = 0;
  for (int e = 0; e < p.E; ++e) {
    const double ex = p.elem[3 * e], ey = p.elem[3 * e + 1], ez = p.elem[3 * e + 2];
    if (p.fnum > 0.0 && outside_aperture(px, py, pz, ex, ey, ez, p.fnum)) continue;
    ++c;
  }
  atomicAdd(out + k, c);
}

// The svd_filter nonzero check (svd.cpp:42) without a host round trip: trace
// of the (reduced) Gram = ||X||_F^2; flag[0] = 1 when it is not positive.
__global__ void gram_trace_check_kernel(const double2* g, int F, int* flag) {
  double t = 0.0;
  for (int i = threadIdx.x; i < F; i += 32) t += g[(size_t)i * F + i].x;
  for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  if (threadIdx.x == 0 && !(t > 0.0)) *flag = 1;
}

__global__ void sigma_kernel(const double* w, int F, double* s) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < F) s[i] = sqrt(fmax(w[i], 0.0));
}

// Planes [0, nz) into `parts` contiguous slabs of near-equal weight, cuts on
// multiples of `align` (the tile depth).
std::vector<std::pair<int, int>> balance_slabs(const std::vector<double>& w, int parts,
                                               int align) {
  const int nz = (int)w.size();
  std::vector<double> cum(nz + 1, 0.0);
  for (int k = 0; k < nz; ++k) cum[k + 1] = cum[k] + w[k];
  std::vector<int> cuts{0};
  for (int r = 1; r < parts; ++r) {
    const double target = cum[nz] * r / parts;
    int k = (int)(std::lower_bound(cum.begin(), cum.end(), target) - cum.begin());
    if (k > 0 && k <= nz && target - cum[k - 1] < cum[k] - target) --k;  // nearest cut
    k = (int)std::lround((double)k / align) * align;
    k = std::min(std::max(k, cuts.back()), nz);
    cuts.push_back(k);
  }
  cuts.push_back(nz);
  std::vector<std::pair<int, int>> s;
  for (int r = 0; r < parts; ++r) s.push_back({cuts[r], cuts[r + 1]});
  return s;
}

struct Ev {
  cudaEvent_t e = nullptr;
  explicit Ev(bool timing = false) {
    CK(cudaEventCreateWithFlags(&e, timing ? cudaEventDefault : cudaEventDisableTiming));
  }
  ~Ev() {
    if (e) cudaEventDestroy(e);
  }
  Ev(const Ev&) = delete;
  Ev& operator=(const Ev&) = delete;
};

}  // namespace

struct fqfg_recon_s {
  int device = 0;
  fqfg_das_plan_s P;
  int F = 0, A = 0, T = 0, E = 0;
  size_t N = 0;
  int lo = 2, hi = 0;
  int rank = 0, world = 1;
  std::vector<std::pair<int, int>> slabs;
  int k0 = 0, k1 = 0;
  size_t v0 = 0, nloc = 0;
  int row_lo = 1, row_hi = 0;   // IQ rows the slab reads (row = t + 1)
  int t_begin = 0, t_end = 0;   // RF samples they need
  uint64_t active_samples = 0;  // active (voxel, element, angle, frame) samples of the slab
  // device buffers
  std::vector<void*> allocs;
  size_t device_bytes = 0;
  void* work = nullptr;         // frame-pass IQ (+ staging for long filters)
  int nbuf = 1;
  float2* x[2] = {nullptr, nullptr};
  double2* gram[2] = {nullptr, nullptr};
  double2* v[2] = {nullptr, nullptr};
  double* w[2] = {nullptr, nullptr};
  double* sig[2] = {nullptr, nullptr};
  double* pd[2] = {nullptr, nullptr};
  double* pd_full = nullptr;    // rank 0 of a sharded NCCL run
  void* gwork = nullptr;
  void* eigwork = nullptr;
  void* scratch = nullptr;
  int* flags = nullptr;
  int max_flags = 0;
  float* ring = nullptr;
  int ring_chunks = 0;
  size_t chunk_floats = 0;
  size_t budget = 0;
  size_t h2d_per_ensemble = 0;
  int ring_frames_opt = 0;
  bool gram_fp64 = false;  // Gram engine: tensor cores (default) or FP64 CUDA cores
  cudaStream_t s_work = nullptr, s_copy = nullptr, s_post = nullptr;
  std::vector<std::unique_ptr<Ev>> ev_up, ev_rel;
  std::unique_ptr<Ev> das_done[2], post_done[2];
  // collectives
  ncclComm_t comm = nullptr;
  ncclComm_t rf_comm = nullptr;  // RF broadcast (its own communicator: the copy stream's
                                 // collectives never interleave with the filter stream's)
  bool rf_bcast = false;         // rank 0 uploads each chunk once; NVLink broadcast to all
  fqfg_allreduce_fn allreduce = nullptr;
  void* allreduce_user = nullptr;
  // instrumentation: events per DAS pass / demod / filter of the last run
  bool timing = false;
  std::vector<std::unique_ptr<Ev>> tev;
  size_t tev_used = 0;
  std::vector<std::array<int, 3>> tspans;  // (kind 0 demod / 1 das / 2 filter, ev a, ev b)
  double t_ms[4] = {0, 0, 0, 0};  // demod, DAS, filter spans; the whole run
  int last_b = -1;  // X buffer of the last ensemble reconstructed

  void* alloc(size_t bytes) {
    void* p = nullptr;
    if (cudaMalloc(&p, std::max<size_t>(bytes, 256)) != cudaSuccess) {
      cudaGetLastError();
      fail(FQFG_ENOMEM, "reconstruction engine: cannot allocate %.2f GB on device %d "
                        "(%.2f GB allocated so far)",
           bytes / 1e9, device, device_bytes / 1e9);
    }
    allocs.push_back(p);
    device_bytes += bytes;
    return p;
  }
  ~fqfg_recon_s() {
    if (s_work) cudaStreamSynchronize(s_work);
    if (s_post) cudaStreamSynchronize(s_post);
    if (s_copy) cudaStreamSynchronize(s_copy);
    if (rf_comm) nccl_api().CommDestroy(rf_comm);
    if (comm) nccl_api().CommDestroy(comm);
    for (void* p : allocs) cudaFree(p);
    ev_up.clear();
    ev_rel.clear();
    tev.clear();
    for (auto& e : das_done) e.reset();
    for (auto& e : post_done) e.reset();
    if (s_work) cudaStreamDestroy(s_work);
    if (s_copy) cudaStreamDestroy(s_copy);
    if (s_post) cudaStreamDestroy(s_post);
    free_plan(&P);
  }

  // Event pair around a span of work on stream `st` (instrumentation).
  int tmark(cudaStream_t st) {
    if (!timing) return -1;
    if (tev_used == tev.size()) tev.push_back(std::make_unique<Ev>(true));
    CK(cudaEventRecord(tev[tev_used]->e, st));
    return (int)tev_used++;
  }
  void tspan(int kind, int a, int b) {
    if (a >= 0 && b >= 0) tspans.push_back({kind, a, b});
  }

  void ensure_ring() {
    if (ring) return;
    const size_t frame_floats = (size_t)A * (t_end - t_begin) * E;
    chunk_floats = frame_floats * kChunk;
    // Two ensembles' worth of chunks when they fit (the next ensemble uploads
    // during this one's DAS), else what the budget leaves, at least 2 chunks.
    const int want = 2 * ((F + kChunk - 1) / kChunk);
    int fit = (int)std::min<size_t>((budget > device_bytes ? budget - device_bytes : 0) /
                                        std::max<size_t>(chunk_floats * sizeof(float), 1),
                                    (size_t)1 << 20);
    int n = std::max(2, std::min(want, fit));
    if (ring_frames_opt > 0) n = std::max(1, ring_frames_opt / kChunk);
    ring_chunks = n;
    ring = static_cast<float*>(alloc(chunk_floats * sizeof(float) * (size_t)n));
    for (int i = 0; i < n; ++i) {
      ev_up.push_back(std::make_unique<Ev>());
      ev_rel.push_back(std::make_unique<Ev>());
    }
  }

  // Gram -> [all-reduce] -> check -> eigensolve -> projection + PD -> host,
  // for the ensemble in X[b], on the filter stream.
  void filter(int b, int k, double* h_pd, double* h_sigma) {
    const int f0 = tmark(s_post);
    if (gram_fp64)
      run_gram(x[b], F, nloc, 0, nloc, gram[b], gwork, 0, s_post);
    else
      run_gram_tc(x[b], F, nloc, 0, nloc, gram[b], gwork, 0, s_post);
    if (world > 1) {
      if (comm) {
        NCK(nccl_api().AllReduce(gram[b], gram[b], (size_t)2 * F * F, ncclFloat64, ncclSum, comm,
                                 s_post));
      } else {
        const int rc = allreduce(allreduce_user, reinterpret_cast<double*>(gram[b]),
                                 (size_t)2 * F * F, (void*)s_post);
        require(rc == 0, "the all-reduce callback failed (%d)", rc);
      }
    }
    gram_trace_check_kernel<<<1, 32, 0, s_post>>>(gram[b], F, flags + k);
    CK_LAUNCH();
    run_eig_band(gram[b], F, lo, hi, w[b], v[b], eigwork, s_post);
    run_project(x[b], F, nloc, 0, nloc, v[b], lo, hi, nullptr, pd[b], scratch, s_post);
    const double* out = pd[b];
    size_t out_off = v0, out_n = nloc;
    if (world > 1 && comm) {
      NcclApi& nc = nccl_api();
      if (rank == 0) {
        CK(cudaMemcpyAsync(pd_full + v0, pd[b], nloc * sizeof(double), cudaMemcpyDeviceToDevice,
                           s_post));
        NCK(nc.GroupStart());
        for (int r = 1; r < world; ++r) {
          const size_t a = (size_t)slabs[r].first * P.p.nx * P.p.ny;
          const size_t n = (size_t)(slabs[r].second - slabs[r].first) * P.p.nx * P.p.ny;
          if (n) NCK(nc.Recv(pd_full + a, n, ncclFloat64, r, comm, s_post));
        }
        NCK(nc.GroupEnd());
        out = pd_full, out_off = 0, out_n = N;
      } else if (nloc) {
        NCK(nc.GroupStart());
        NCK(nc.Send(pd[b], nloc, ncclFloat64, 0, comm, s_post));
        NCK(nc.GroupEnd());
      }
    }
    if (h_pd && out_n)
      CK(cudaMemcpyAsync(h_pd + out_off, out, out_n * sizeof(double), cudaMemcpyDeviceToHost,
                         s_post));
    if (h_sigma) {
      sigma_kernel<<<(F + 127) / 128, 128, 0, s_post>>>(w[b], F, sig[b]);
      CK_LAUNCH();
      CK(cudaMemcpyAsync(h_sigma, sig[b], F * sizeof(double), cudaMemcpyDeviceToHost, s_post));
    }
    tspan(2, f0, tmark(s_post));
  }

  // Reconstruct n ensembles.  Host source: h_rf[k] (uploaded through the
  // ring); device source: d_rf[k] (resident [F][A][T][E], read in place).
  void run(int n, const float* const* h_rf, const float* const* d_rf, double* const* h_pd,
           double* const* h_sigma, double* d_pd_last) {
    CK(cudaSetDevice(device));
    require(n >= 0, "negative ensemble count");
    if (n == 0) return;
    const DasParams& p = P.p;
    if (n > max_flags) {
      flags = static_cast<int*>(alloc(sizeof(int) * (size_t)n));
      max_flags = n;
    }
    CK(cudaMemsetAsync(flags, 0, sizeof(int) * (size_t)n, s_work));
    if (P.d_kblocks) CK(cudaMemsetAsync(P.d_kblocks, 0, sizeof(unsigned long long), s_work));
    tspans.clear();
    tev_used = 0;
    // The streams start after whatever the caller enqueued before (legacy
    // default stream semantics are not assumed).
    const int t_start = tmark(s_work);
    {
      Ev start;
      CK(cudaEventRecord(start.e, s_work));
      CK(cudaStreamWaitEvent(s_post, start.e, 0));
      CK(cudaStreamWaitEvent(s_copy, start.e, 0));
    }
    static const float* const kNoRf[1] = {nullptr};
    const bool host = h_rf != nullptr || (rf_bcast && rank != 0 && !d_rf);
    if (host && !h_rf) h_rf = kNoRf;  // broadcast receivers read no host RF
    if (host) ensure_ring();
    const int rows = t_end - t_begin;
    const int per_pass = (p.fpass + kChunk - 1) / kChunk;
    // Uploads (host source): every chunk with valid frames, in order.
    struct Up {
      int k, pass, f_lo, nv;
    };
    std::vector<Up> ups;
    if (host)
      for (int k = 0; k < n; ++k)
        for (int pass = 0; pass < p.npass; ++pass) {
          const int nf = std::min(p.fpass, F - pass * p.fpass);
          for (int c = 0; c < per_pass; ++c)
            if (nf - c * kChunk > 0) ups.push_back({k, pass, c * kChunk, std::min(kChunk, nf - c * kChunk)});
        }
    size_t next_up = 0;
    auto enqueue_upload = [&]() {
      const Up& u = ups[next_up];
      const int slot = (int)(next_up % ring_chunks);
      if (next_up >= (size_t)ring_chunks) CK(cudaStreamWaitEvent(s_copy, ev_rel[slot]->e, 0));
      const int f = u.pass * p.fpass + u.f_lo;
      float* dst = ring + (size_t)slot * chunk_floats;
      if (rows > 0 && (!rf_bcast || rank == 0)) {
        const float* src = h_rf[u.k] + ((size_t)f * A * T + t_begin) * E;
        CK(cudaMemcpy2DAsync(dst, (size_t)rows * E * sizeof(float), src,
                             (size_t)T * E * sizeof(float), (size_t)rows * E * sizeof(float),
                             (size_t)u.nv * A, cudaMemcpyHostToDevice, s_copy));
      }
      if (rows > 0 && rf_bcast)  // one PCIe upload on rank 0, NVLink to every rank
        NCK(nccl_api().Broadcast(dst, dst, (size_t)u.nv * A * rows * E, ncclFloat32, 0, rf_comm,
                                 s_copy));
      CK(cudaEventRecord(ev_up[slot]->e, s_copy));
      ++next_up;
    };
    while (next_up < ups.size() && next_up < (size_t)ring_chunks) enqueue_upload();

    size_t up_i = 0;  // index into ups of the next chunk to demodulate
    for (int k = 0; k < n; ++k) {
      const int b = k % nbuf;
      for (int pass = 0; pass < p.npass; ++pass) {
        const int nf = std::min(p.fpass, F - pass * p.fpass);
        const int d0 = tmark(s_work);
        if (host) {
          for (int c = 0; c < per_pass; ++c) {
            const int f_lo = c * kChunk;
            const int nv = std::max(0, std::min(kChunk, nf - f_lo));
            if (nv > 0) {
              const int slot = (int)(up_i % ring_chunks);
              CK(cudaStreamWaitEvent(s_work, ev_up[slot]->e, 0));
              const RfSrc src{ring + (size_t)slot * chunk_floats, (long long)A * rows * E,
                              (long long)rows * E, t_begin, rows, f_lo};
              demod_frames(P, P.p, src, kChunk, nf, work, row_lo, row_hi, s_work);
              CK(cudaEventRecord(ev_rel[slot]->e, s_work));
              ++up_i;
              while (next_up < ups.size() && next_up < up_i + (size_t)ring_chunks)
                enqueue_upload();
            } else {  // padding frames of the pass: zeros
              const RfSrc src{ring, 0, 0, 0, 0, f_lo};
              demod_frames(P, P.p, src, kChunk, nf, work, row_lo, row_hi, s_work);
            }
          }
        } else {
          const float* rf = d_rf[k] + (size_t)pass * p.fpass * A * T * E;
          const RfSrc src{rf, (long long)A * T * E, (long long)T * E, 0, T, 0};
          demod_frames(P, P.p, src, p.fpass, nf, work, row_lo, row_hi, s_work);
        }
        demod_finish(P, P.p, nf, work, row_lo, row_hi, s_work);
        const int d1 = tmark(s_work);
        tspan(0, d0, d1);
        // X[b] is free once the filter of ensemble k - nbuf has read it.
        if (pass == 0 && k >= nbuf) CK(cudaStreamWaitEvent(s_work, post_done[b]->e, 0));
        const int a0 = tmark(s_work);
        das_pass(P, P.p, pass, k0, k1, work, x[b], v0, nloc, nullptr, s_work);
        tspan(1, a0, tmark(s_work));
      }
      CK(cudaEventRecord(das_done[b]->e, s_work));
      CK(cudaStreamWaitEvent(s_post, das_done[b]->e, 0));
      filter(b, k, h_pd ? h_pd[k] : nullptr, h_sigma ? h_sigma[k] : nullptr);
      if (d_pd_last && k == n - 1) {
        const double* src = (world > 1 && comm && rank == 0) ? pd_full : pd[b];
        const size_t cnt = (world > 1 && comm && rank == 0) ? N : nloc;
        CK(cudaMemcpyAsync(d_pd_last + ((world > 1 && comm && rank == 0) ? 0 : v0), src,
                           cnt * sizeof(double), cudaMemcpyDeviceToDevice, s_post));
      }
      CK(cudaEventRecord(post_done[b]->e, s_post));
    }
    // The run ends when all three streams have drained (PD on the host).
    {
      Ev end_post, end_copy;
      CK(cudaEventRecord(end_post.e, s_post));
      CK(cudaEventRecord(end_copy.e, s_copy));
      CK(cudaStreamWaitEvent(s_work, end_post.e, 0));
      CK(cudaStreamWaitEvent(s_work, end_copy.e, 0));
    }
    tspan(3, t_start, tmark(s_work));
    CK(cudaStreamSynchronize(s_post));
    CK(cudaStreamSynchronize(s_work));
    CK(cudaStreamSynchronize(s_copy));
    last_b = (n - 1) % nbuf;
    if (timing) {
      t_ms[0] = t_ms[1] = t_ms[2] = t_ms[3] = 0.0;
      for (auto& s : tspans) {
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, tev[s[1]]->e, tev[s[2]]->e));
        t_ms[s[0]] += ms;
      }
    }
    std::vector<int> hf(n);
    CK(cudaMemcpy(hf.data(), flags, sizeof(int) * (size_t)n, cudaMemcpyDeviceToHost));
    for (int k = 0; k < n; ++k)
      require(hf[k] == 0, "svd_filter needs a nonzero ensemble (ensemble %d)", k);
  }
};

namespace {

void build_recon(fqfg_recon_s& R, const fqfg_rf_desc* d, const fqfg_grid* g,
                 const fqfg_probe* pr, const fqfg_bf* bf, const fqfg_recon_opts& o) {
  CK(cudaGetDevice(&R.device));
  R.P.device = R.device;
  R.F = d->n_frames;
  R.A = d->n_angles;
  R.T = d->n_samples;
  R.E = d->n_elements;
  R.lo = o.keep_lo;
  R.hi = o.keep_hi > 0 ? o.keep_hi : d->n_frames;
  R.rank = o.rank;
  R.world = std::max(1, o.world);
  require(R.world >= 1 && R.rank >= 0 && R.rank < R.world, "rank %d outside world %d", R.rank,
          R.world);
  size_t free_b = 0, total_b = 0;
  CK(cudaMemGetInfo(&free_b, &total_b));
  R.budget = o.device_budget ? o.device_budget : (size_t)(0.92 * (double)free_b);
  R.ring_frames_opt = o.ring_frames;
  // Plan geometry first; the frame pass is sized below, once the slab's
  // readable rows are known.
  build_plan(d, g, pr, bf, R.P, 0);
  const DasParams& p = R.P.p;
  R.N = (size_t)p.nx * p.ny * p.nz;
  check_filter(R.F, R.N, R.lo, R.hi);
  // Depth slabs balanced by active aperture pairs per plane.
  std::vector<double> wpl(p.nz, 0.0);
  {
    unsigned long long* d_c = nullptr;
    CK(cudaMalloc(&d_c, sizeof(unsigned long long) * p.nz));
    CK(cudaMemset(d_c, 0, sizeof(unsigned long long) * p.nz));
    plane_active_kernel<<<(unsigned)((R.N + 255) / 256), 256>>>(p, d_c);
    CK_LAUNCH();
    std::vector<unsigned long long> hc(p.nz);
    CK(cudaMemcpy(hc.data(), d_c, sizeof(unsigned long long) * p.nz, cudaMemcpyDeviceToHost));
    cudaFree(d_c);
    for (int k = 0; k < p.nz; ++k) wpl[k] = (double)hc[k];
  }
  // Cut at any plane: the deep planes carry the most work, so tile-depth
  // alignment would cost balance (max / mean 1.11 at N = 8 for config C).
  R.slabs = balance_slabs(wpl, R.world, 1);
  R.k0 = R.slabs[R.rank].first;
  R.k1 = R.slabs[R.rank].second;
  R.v0 = (size_t)R.k0 * p.nx * p.ny;
  R.nloc = (size_t)(R.k1 - R.k0) * p.nx * p.ny;
  double act = 0.0;
  for (int k = R.k0; k < R.k1; ++k) act += wpl[k];
  R.active_samples = (uint64_t)act * (uint64_t)p.A * (uint64_t)p.F;
  if (R.k1 > R.k0) {
    slab_rows(R.P, R.k0, R.k1, R.row_lo, R.row_hi);
    const int mid = p.taps / 2;
    R.t_begin = std::max(0, R.row_lo - 1 - mid);
    R.t_end = std::min(p.T, std::max(R.t_begin, R.row_hi + mid));
  }
  R.rf_bcast = o.rf_broadcast != 0;
  if (R.rf_bcast) {
    // One upload for every rank: the union of the ranks' sample windows.
    int tb = p.T, te = 0;
    for (const auto& sl : R.slabs) {
      if (sl.second <= sl.first) continue;
      int rl, rh;
      slab_rows(R.P, sl.first, sl.second, rl, rh);
      const int mid = p.taps / 2;
      const int b = std::max(0, rl - 1 - mid), e = std::min(p.T, std::max(b, rh + mid));
      if (e > b) tb = std::min(tb, b), te = std::max(te, e);
    }
    if (te > tb) R.t_begin = tb, R.t_end = te;
  }
  // The pass IQ buffer holds only the slab's readable rows; the frame pass is
  // the largest whose IQ fits next to one X buffer, two RF chunks, the Gram
  // scratch and 2 GB of slack (config D: 208 frames per pass, 96 GB).
  {
    const int rows = R.row_lo <= R.row_hi ? R.row_hi - R.row_lo + 1 : 1;
    const size_t x1 = (size_t)R.F * std::max<size_t>(R.nloc, 1) * sizeof(float2);
    const size_t chunk2 = 2 * (size_t)kChunk * R.A * std::max(R.t_end - R.t_begin, 1) * R.E * 4;
    const size_t gw = o.gram_fp64 ? gram_splits(R.F) * (size_t)R.F * R.F * 16
                                  : gram_tc_work_bytes(R.F);
    const size_t other = x1 + chunk2 + gw + ((size_t)2 << 30);
    plan_shape(R.P, R.budget > other ? R.budget - other : 1, rows);
    R.P.p.iq_row0 = R.row_lo <= R.row_hi ? R.row_lo : 0;
    R.P.p.iq_rows = rows;
  }
  R.h2d_per_ensemble = (R.rf_bcast && R.rank != 0)
                           ? 0
                           : (size_t)R.F * R.A * (R.t_end - R.t_begin) * R.E * sizeof(float);
  // Buffers.
  const size_t gsz = (size_t)R.F * R.F * sizeof(double2);
  R.work = R.alloc(R.P.stage_bytes + R.P.iq_bytes);
  R.P.d_kblocks = static_cast<unsigned long long*>(R.alloc(sizeof(unsigned long long)));
  const size_t xbytes = (size_t)R.F * std::max<size_t>(R.nloc, 1) * sizeof(float2);
  const size_t ring_min = 2 * (size_t)kChunk * R.A * (R.t_end - R.t_begin) * R.E * sizeof(float);
  R.nbuf = R.device_bytes + 2 * xbytes + ring_min + (size_t)(1 << 30) <= R.budget ? 2 : 1;
  if (o.x_buffers == 1 || o.x_buffers == 2) R.nbuf = o.x_buffers;
  for (int b = 0; b < R.nbuf; ++b) R.x[b] = static_cast<float2*>(R.alloc(xbytes));
  for (int b = 0; b < 2; ++b) {
    R.gram[b] = static_cast<double2*>(R.alloc(gsz));
    R.v[b] = static_cast<double2*>(R.alloc(gsz));
    R.w[b] = static_cast<double*>(R.alloc(R.F * sizeof(double)));
    R.sig[b] = static_cast<double*>(R.alloc(R.F * sizeof(double)));
    R.pd[b] = static_cast<double*>(R.alloc(std::max<size_t>(R.nloc, 1) * sizeof(double)));
  }
  R.gram_fp64 = o.gram_fp64 != 0;
  R.gwork = R.alloc(R.gram_fp64 ? gram_splits(R.F) * gsz : gram_tc_work_bytes(R.F));
  R.eigwork = R.alloc(std::max(eig_work_bytes(R.F), gsz));
  R.scratch = R.alloc(filter_scratch_bytes(R.F));
  CK(cudaStreamCreateWithFlags(&R.s_work, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&R.s_copy, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&R.s_post, cudaStreamNonBlocking));
  for (int b = 0; b < 2; ++b) {
    R.das_done[b] = std::make_unique<Ev>();
    R.post_done[b] = std::make_unique<Ev>();
  }
  if (R.rf_bcast)
    require(o.nccl_id != nullptr, "the RF broadcast needs NCCL (an ncclUniqueId)");
  if (R.world > 1 || R.rf_bcast) {
    if (o.allreduce && !R.rf_bcast) {
      R.allreduce = o.allreduce;
      R.allreduce_user = o.allreduce_user;
    } else {
      require(o.nccl_id != nullptr,
              "a sharded engine (world %d) needs an ncclUniqueId or an all-reduce callback",
              R.world);
      NcclApi& nc = nccl_api();
      require(nc.ok, "NCCL unavailable: %s", nc.why.c_str());
      ncclUniqueId id;
      std::memcpy(&id, o.nccl_id, sizeof id);
      NCK(nc.CommInitRank(&R.comm, R.world, id, R.rank));
      if (R.rank == 0 && R.world > 1)
        R.pd_full = static_cast<double*>(R.alloc(R.N * sizeof(double)));
      if (R.rf_bcast) NCK(nc.CommSplit(R.comm, 0, R.rank, &R.rf_comm, nullptr));
    }
  }
  CK(cudaDeviceSynchronize());
}

// One engine per (host thread, device), rebuilt when the geometry changes: the
// plan cache of the one-shot fqfg_reconstruct_pd.
struct EngineCache {
  std::string key;
  fqfg_recon_s* R = nullptr;
  ~EngineCache() { delete R; }
};

std::string engine_key(const fqfg_rf_desc* d, const fqfg_grid* g, const fqfg_probe* pr,
                       const fqfg_bf* bf, int lo, int hi, int dev) {
  std::string k;
  auto put = [&](const void* p, size_t n) { k.append(static_cast<const char*>(p), n); };
  put(&dev, sizeof dev);
  put(&lo, sizeof lo);
  put(&hi, sizeof hi);
  put(&d->n_frames, 4 * sizeof(int));
  put(&d->sampling_rate, sizeof(double));
  put(d->t0, sizeof(double) * d->n_angles);
  put(d->angles, sizeof(double) * d->n_angles);
  put(g, sizeof *g);
  put(&pr->n_elements, sizeof(int));
  put(pr->xyz, sizeof(double) * 3 * pr->n_elements);
  put(bf, sizeof *bf);
  return k;
}

fqfg_recon_s* cached_engine(const fqfg_rf_desc* d, const fqfg_grid* g, const fqfg_probe* pr,
                            const fqfg_bf* bf, int lo, int hi) {
  static thread_local std::map<int, EngineCache> cache;
  int dev;
  CK(cudaGetDevice(&dev));
  EngineCache& c = cache[dev];
  const std::string key = engine_key(d, g, pr, bf, lo, hi, dev);
  if (c.R && c.key == key) return c.R;
  delete c.R;
  c.R = nullptr;
  fqfg_recon_opts o{};
  o.keep_lo = lo;
  o.keep_hi = hi;
  o.world = 1;
  auto R = std::make_unique<fqfg_recon_s>();
  build_recon(*R, d, g, pr, bf, o);
  c.R = R.release();
  c.key = key;
  return c.R;
}

}  // namespace

#pragma GCC visibility push(default)
extern "C" {

int fqfg_nccl_unique_id(void* out) {
  return guarded([&] {
    require(out != nullptr, "null output");
    NcclApi& nc = nccl_api();
    require(nc.ok, "NCCL unavailable: %s", nc.why.c_str());
    ncclUniqueId id;
    NCK(nc.GetUniqueId(&id));
    std::memcpy(out, &id, sizeof id);
  });
}

int fqfg_recon_create(const fqfg_rf_desc* d, const fqfg_grid* g, const fqfg_probe* pr,
                      const fqfg_bf* bf, const fqfg_recon_opts* opts, fqfg_recon* out) {
  return guarded([&] {
    require(out != nullptr, "engine output pointer is null");
    need_device();
    fqfg_recon_opts o{};
    o.keep_lo = 2;
    o.world = 1;
    if (opts) o = *opts;
    auto R = std::make_unique<fqfg_recon_s>();
    build_recon(*R, d, g, pr, bf, o);
    *out = R.release();
  });
}

int fqfg_recon_info_get(fqfg_recon R, fqfg_recon_info* info) {
  return guarded([&] {
    require(R && info, "null engine");
    info->k_begin = R->k0;
    info->k_end = R->k1;
    info->v_begin = R->v0;
    info->v_end = R->v0 + R->nloc;
    info->t_begin = R->t_begin;
    info->t_end = R->t_end;
    info->frames_per_pass = R->P.p.fpass;
    info->n_passes = R->P.p.npass;
    info->x_buffers = R->nbuf;
    info->ring_frames = R->ring_chunks * kChunk;
    info->device_bytes = R->device_bytes;
    info->h2d_bytes_per_ensemble = R->h2d_per_ensemble;
    info->active_samples = R->active_samples;
    info->tile[0] = R->P.TX;
    info->tile[1] = R->P.TY;
    info->tile[2] = R->P.TZ;
    info->shape[0] = R->P.J;
    info->shape[1] = R->P.VPW;
    info->shape[2] = R->P.NW;
    info->shape[3] = R->P.PW;
    info->mode = R->P.tc ? 2 : 0;
    info->nccl = R->comm != nullptr;
    info->gram_fp64 = R->gram_fp64 ? 1 : 0;
  });
}

int fqfg_recon_run(fqfg_recon R, int n, const float* const* rf, double* const* pd,
                   double* const* sigma) {
  return guarded([&] {
    require(R != nullptr, "null engine");
    require(n == 0 || rf != nullptr || (R->rf_bcast && R->rank != 0), "null RF list");
    for (int k = 0; k < n; ++k)
      require(rf[k] != nullptr || (R->rf_bcast && R->rank != 0), "RF of ensemble %d is null", k);
    R->run(n, rf, nullptr, pd, sigma, nullptr);
  });
}

int fqfg_recon_run_dev(fqfg_recon R, int n, const float* const* d_rf, double* d_pd_last) {
  return guarded([&] {
    require(R != nullptr, "null engine");
    require(n == 0 || d_rf != nullptr, "null RF list");
    for (int k = 0; k < n; ++k) require(d_rf[k] != nullptr, "RF of ensemble %d is null", k);
    R->run(n, nullptr, d_rf, nullptr, nullptr, d_pd_last);
  });
}

int fqfg_recon_set_timing(fqfg_recon R, int enable) {
  return guarded([&] {
    require(R != nullptr, "null engine");
    R->timing = enable != 0;
  });
}

int fqfg_recon_last_timing(fqfg_recon R, double* demod_ms, double* das_ms, double* filter_ms,
                           double* total_ms) {
  return guarded([&] {
    require(R != nullptr, "null engine");
    if (demod_ms) *demod_ms = R->t_ms[0];
    if (das_ms) *das_ms = R->t_ms[1];
    if (filter_ms) *filter_ms = R->t_ms[2];
    if (total_ms) *total_ms = R->t_ms[3];
  });
}

int fqfg_recon_mma_blocks(fqfg_recon R, unsigned long long* kblocks) {
  return guarded([&] {
    require(R != nullptr && kblocks != nullptr, "null argument");
    CK(cudaSetDevice(R->device));
    *kblocks = 0;
    if (R->P.tc && R->P.d_kblocks)
      CK(cudaMemcpy(kblocks, R->P.d_kblocks, sizeof(unsigned long long), cudaMemcpyDeviceToHost));
  });
}

int fqfg_recon_copy_iq(fqfg_recon R, size_t v_begin, size_t v_end, float* iq) {
  return guarded([&] {
    require(R != nullptr && iq != nullptr, "null argument");
    require(R->last_b >= 0, "no ensemble reconstructed yet");
    require(v_begin <= v_end && v_begin >= R->v0 && v_end <= R->v0 + R->nloc,
            "voxels [%zu, %zu) are not in this engine's slab [%zu, %zu)", v_begin, v_end, R->v0,
            R->v0 + R->nloc);
    CK(cudaSetDevice(R->device));
    const size_t n = v_end - v_begin;
    if (n == 0) return;
    CK(cudaMemcpy2D(iq, n * sizeof(float2), R->x[R->last_b] + (v_begin - R->v0),
                    R->nloc * sizeof(float2), n * sizeof(float2), (size_t)R->F,
                    cudaMemcpyDeviceToHost));
  });
}

int fqfg_reconstruct_pd(const fqfg_rf_desc* d, const float* rf, const fqfg_grid* grid,
                        const fqfg_probe* probe, const fqfg_bf* bf, int lo, int hi, double* pd_out,
                        double* sigma, float* iq_out) {
  return guarded([&] {
    check_rf(d, probe);
    check_grid(grid);
    size_t N = (size_t)grid->dims[0] * grid->dims[1] * grid->dims[2];
    check_filter(d->n_frames, N, lo, hi);
    require(pd_out != nullptr, "null PD output");
    need_device();
    fqfg_recon R = cached_engine(d, grid, probe, bf, lo, hi);
    const float* rfs[1] = {rf};
    double* pds[1] = {pd_out};
    double* sgs[1] = {sigma};
    R->run(1, rfs, nullptr, pds, sigma ? sgs : nullptr, nullptr);
    if (iq_out)
      CK(cudaMemcpy(iq_out, R->x[R->last_b], (size_t)d->n_frames * N * sizeof(float2),
                    cudaMemcpyDeviceToHost));
  });
}

int fqfg_recon_report(fqfg_recon R, double* sigma, double* mode_correlation) {
  return guarded([&] {
    require(R != nullptr, "null engine");
    require(R->last_b >= 0, "no ensemble reconstructed yet");
    require(R->world == 1, "the SVD report needs the whole ensemble on one engine (world 1)");
    CK(cudaSetDevice(R->device));
    const int F = R->F;
    const size_t gsz = (size_t)F * F * sizeof(double2);
    // SvdReport (svd.cpp:49-76) of the last ensemble, from the resident X:
    // exact FP64 Gram, full eigensolve, |U| = |X V| / sigma correlation.
    double2* g = static_cast<double2*>(tl_gram.get(2 * gsz + F * sizeof(double) + 1024));
    double2* v = g + (size_t)F * F;
    double* w = reinterpret_cast<double*>(v + (size_t)F * F);
    void* gw = tl_work.get(gram_splits(F) * gsz);
    void* ew = tl_eig.get(std::max(eig_work_bytes(F), gsz));
    cudaStream_t st = R->s_post;
    run_gram(R->x[R->last_b], F, R->nloc, 0, R->nloc, g, gw, 0, st);
    run_eig(g, F, w, v, ew, st);
    std::vector<double> hw(F), sg(F);
    CK(cudaMemcpyAsync(hw.data(), w, F * sizeof(double), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    for (int j = 0; j < F; ++j) sg[j] = std::sqrt(std::max(hw[j], 0.0));
    if (sigma) std::copy(sg.begin(), sg.end(), sigma);
    if (mode_correlation) run_mode_correlation(R->x[R->last_b], F, R->nloc, v, sg, mode_correlation, st);
    CK(cudaStreamSynchronize(st));
  });
}

void fqfg_recon_destroy(fqfg_recon R) {
  if (!R) return;
  cudaSetDevice(R->device);
  delete R;
}

}  // extern "C"
#pragma GCC visibility pop
