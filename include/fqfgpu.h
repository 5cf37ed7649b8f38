/*
 * fqfgpu.h -- C ABI of the B200 (sm_100a) reconstruction hot path.
 *
 * RF channel data -> IQ demodulation -> 3D plane-wave delay-and-sum with
 * angle compounding -> Casorati SVD clutter filter -> power Doppler.
 *
 * Each entry point replaces one function of the reference's C++ library
 * (proj/include/fqf/..., paths relative to /root/reference); the reference
 * has no plugin/FFI layer, so this ABI is what a C++ shim (or ctypes/cgo
 * binding) of those functions calls.  See INTEGRATION.md for the bindings.
 *
 *   fqfg_rf_to_iq          <- fqf::beamform::rf_to_iq          (beamform/iq.hpp:31,  src iq.cpp:34-82)
 *   fqfg_plan_chunks       <- fqf::beamform::plan_chunks       (beamform/das.hpp:49, src das.cpp:97-119)
 *   fqfg_das               <- fqf::beamform::das_reconstruct   (beamform/das.hpp:124-127, src das.cpp:224-356)
 *   fqfg_svd_filter        <- fqf::post::svd_filter            (post/svd.hpp:23-25,  src svd.cpp:29-93)
 *   fqfg_power_doppler     <- fqf::post::power_doppler         (post/render.hpp:13,  src render.cpp:23-42)
 *   fqfg_reconstruct_pd    <- run_beamform + run_post fused    (src pipeline/run.cpp:397-487)
 *
 * Conventions (mirroring the reference):
 *   - every call returns 0 on success, nonzero on failure; the message of the
 *     last failure on the calling thread is fqfg_last_error().  Contract
 *     violations return FQFG_EINVAL with the reference's require() message
 *     (core/error.hpp:30-33); CUDA failures return FQFG_ECUDA.
 *   - host-pointer entry points are synchronous, never retain inputs, and
 *     write outputs only on success (das.cpp:354, svd.cpp:49).
 *   - layouts: RF [frame][angle][t][element] f32, time-major per transmit
 *     (RfFrame, rf/simulate.hpp:22-37, stored as f32 at simulate.cpp:638);
 *     IQ volumes [frame][voxel] complex64 interleaved (re, im), voxel index
 *     i + nx*(j + ny*k) (GridSpec::point, das.hpp:28-32); the Casorati matrix
 *     column f is frame f (svd.cpp:38-41); PD f64 [voxel].
 *   - *_dev entry points take device pointers and a cudaStream_t (as void*),
 *     are asynchronous on that stream, and are what bench.py and the
 *     depth-slab multi-GPU driver use.
 *   - no CPU fallback: without a usable sm_100 device every compute entry
 *     point fails with FQFG_ENODEV.
 */
#ifndef FQFGPU_H
#define FQFGPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { FQFG_OK = 0, FQFG_EINVAL = 1, FQFG_ECUDA = 2, FQFG_ENODEV = 3, FQFG_ENOMEM = 4 };

/* Reconstruction grid (GridSpec, das.hpp:20-33). */
typedef struct {
  int dims[3];
  double spacing[3];
  double origin[3];
} fqfg_grid;

/* Probe element centres, [n_elements][3] metres (Transducer::elements,
 * transducer.hpp:13-31).  DAS reads only these (das.cpp:137-145). */
typedef struct {
  int n_elements;
  const double* xyz;
} fqfg_probe;

/* BeamformParams (das.hpp:76-82). */
typedef struct {
  double c;
  double center_frequency;
  double f_number;  /* <= 0 disables the receive aperture cut */
  int interp_order; /* 1 linear, 0 nearest */
  int lowpass_taps; /* odd, >= 3 */
} fqfg_bf;

/* Shape of an RF ensemble [n_frames][n_angles][n_samples][n_elements].  Per
 * angle slot: steering angle (TxEvent::angle) and start time t0 (RfFrame::t0);
 * das.cpp:249-251 requires them equal across frames, so they are per slot. */
typedef struct {
  int n_frames;
  int n_angles;
  int n_samples;
  int n_elements;
  double sampling_rate;
  const double* t0;     /* [n_angles] */
  const double* angles; /* [n_angles] radians */
} fqfg_rf_desc;

/* DasOptions (das.hpp:101-108), minus the file knobs which the host shim
 * honours itself (the GPU path keeps the ensemble resident). */
typedef struct {
  size_t memory_budget_bytes; /* 100'000'000 by default */
  size_t matrix_budget_bytes; /* 512'000'000 by default */
  int cache_matrices;         /* 1 by default */
} fqfg_das_opts;

/* DasStats (das.hpp:110-116), same semantics as the reference. */
typedef struct {
  uint64_t chunks;
  uint64_t matrix_builds;
  uint64_t out_of_window;
  uint64_t matrix_bytes_peak;
  uint64_t accumulator_bytes_peak;
} fqfg_das_stats;

const char* fqfg_last_error(void);
int fqfg_version(void);
/* Number of usable sm_100 devices (0 if none); never fails. */
int fqfg_device_count(void);
int fqfg_set_device(int device);

/* ---- host-buffer entry points (the drop-in surface) ---------------------- */

/* rf_to_iq over a batch of frames sharing fs/f_c: rf [batch][T][E] f32,
 * t0 [batch], iq [batch][T][E] complex64. */
int fqfg_rf_to_iq(const float* rf, int batch, int n_samples, int n_elements,
                  double sampling_rate, const double* t0, double center_frequency,
                  int lowpass_taps, float* iq);

/* plan_chunks: returns the chunk count in *n_chunks and, if ranges != NULL
 * (capacity 2*max_chunks), the [begin, end) voxel ranges. */
int fqfg_plan_chunks(size_t n_points, int n_angles, size_t budget_bytes, size_t* ranges,
                     size_t max_chunks, size_t* n_chunks);

/* das_reconstruct: rf [F][A][T][E] f32 -> iq_out [F][N] complex64.  stats may
 * be NULL. */
int fqfg_das(const fqfg_rf_desc* rf_desc, const float* rf, const fqfg_grid* grid,
             const fqfg_probe* probe, const fqfg_bf* bf, const fqfg_das_opts* opts,
             float* iq_out, fqfg_das_stats* stats);

/* svd_filter: iq [F][N] complex64 -> filtered [F][N] complex64 (may be
 * NULL), sigma [F] descending (may be NULL), pd [N] f64 = power Doppler of the
 * filtered ensemble (may be NULL), mode_correlation [F][F] = SvdReport's
 * Pearson correlation of the |U| columns (svd.cpp:55-75; may be NULL).
 * Band keep_lo..keep_hi, 1-based. */
int fqfg_svd_filter(const float* iq, int n_frames, size_t n_points, int keep_lo, int keep_hi,
                    float* filtered, double* sigma, double* pd, double* mode_correlation);

/* power_doppler: iq [F][N] complex64 -> pd [N] f64. */
int fqfg_power_doppler(const float* iq, int n_frames, size_t n_points, double* pd);

/* build_delay_matrix (das.hpp:86-88, das.cpp:126-208) for one transmit over
 * n voxels [n][3]: CSR row_ptr [n+1] (required), col_idx [nnz] = t*E + e and
 * values [nnz] complex128 (both NULL: count pass only -- read nnz from
 * row_ptr[n] and call again), out_of_window and padded_samples as
 * DelayMatrix reports them.  Computed on the GPU; the DAS path itself never
 * materialises these matrices. */
int fqfg_build_delay_matrix(const double* voxels, size_t n, double angle, double t0,
                            double sampling_rate, int n_samples, const fqfg_probe* probe,
                            const fqfg_bf* bf, uint64_t* row_ptr, int32_t* col_idx,
                            double* values, uint64_t* out_of_window, int* padded_samples);

/* apply_delay_matrix (das.hpp:90-92, das.cpp:210-222): out[r] = sum of
 * values[i] * iq[col_idx[i]] over row r, FP64 in entry order; iq has n_iq
 * complex128 samples ([T][E] time-major). */
int fqfg_apply_delay_matrix(size_t rows, const uint64_t* row_ptr, const int32_t* col_idx,
                            const double* values, const double* iq, size_t n_iq, double* out);

/* Fused RF -> PD (the benchmark path): demod + DAS + filter + PD without
 * moving the IQ ensemble to the host.  iq_out / sigma may be NULL. */
int fqfg_reconstruct_pd(const fqfg_rf_desc* rf_desc, const float* rf, const fqfg_grid* grid,
                        const fqfg_probe* probe, const fqfg_bf* bf, int keep_lo, int keep_hi,
                        double* pd_out, double* sigma, float* iq_out);

/* ---- device-resident entry points --------------------------------------- */

/* A DAS plan binds geometry, beamforming parameters and the per-angle tables
 * on one device; it is immutable and may be reused across ensembles. */
typedef struct fqfg_das_plan_s* fqfg_das_plan;

typedef struct {
  size_t n_points;          /* voxels */
  int frames_per_pass;      /* frames beamformed per pass (16 * J) */
  int n_passes;             /* ceil(F / frames_per_pass) */
  size_t work_bytes;        /* device scratch needed by fqfg_das_dev */
  uint64_t active_pairs;    /* (voxel, element, angle) triples inside the
                               f-number aperture, the DAS roofline's unit */
  int tile[3];              /* voxel tile of one CTA */
  int shape[4];             /* das2_kernel J, VPW, consumer warps, producer warps
                               (J also sets frames_per_pass = 16 J for das_tc) */
  int mode;                 /* DAS kernel: 0 das2 (CUDA-core gather), 2 das_tc (tensor
                               cores, the default); 1 is no longer used */
} fqfg_das_plan_info;

int fqfg_das_plan_create(const fqfg_rf_desc* rf_desc, const fqfg_grid* grid,
                         const fqfg_probe* probe, const fqfg_bf* bf, fqfg_das_plan* plan);
int fqfg_das_plan_info_get(fqfg_das_plan plan, fqfg_das_plan_info* info);
void fqfg_das_plan_destroy(fqfg_das_plan plan);

/* Beamform z-planes [k_begin, k_end) of the grid from device RF
 * [F][A][T][E] f32 into device x [F][N] complex64 (only the slab's voxels are
 * written).  work: work_bytes of device scratch.  counters (may be NULL):
 * device uint64[2] += {out_of_window, live taps}. */
int fqfg_das_dev(fqfg_das_plan plan, const float* d_rf, int k_begin, int k_end, float* d_x,
                 void* d_work, uint64_t* d_counters, void* stream);

/* RF samples [t_begin, t_end) of every channel that fqfg_das_dev(kb, ke)
 * reads (its delay window widened by the FIR half-length): a depth-slab rank
 * only needs these rows of the recording on its device. */
int fqfg_das_slab_samples(fqfg_das_plan plan, int k_begin, int k_end, int* t_begin, int* t_end);

/* Strided host -> device copy of the same byte range of n_slices equal slices
 * (e.g. RF samples [t_begin, t_end) of every [frame][angle] slice):
 * dst[i*slice_bytes + offset_bytes, + bytes) = src[same], async on `stream`. */
int fqfg_copy_slices_h2d(void* d_dst, const void* h_src, size_t n_slices, size_t slice_bytes,
                         size_t offset_bytes, size_t bytes, void* stream);

/* Partial Gram of a voxel range: d_gram [F][F] complex128 = X^H X over
 * voxels [v_begin, v_end) of d_x [F][N] complex64 (deterministic order).
 * d_work: fqfg_gram_work_bytes(F) bytes. */
size_t fqfg_gram_work_bytes(int n_frames);
int fqfg_gram_dev(const float* d_x, int n_frames, size_t n_points, size_t v_begin, size_t v_end,
                  double* d_gram, void* d_work, void* stream);

/* The same Gram on the tensor cores (tcgen05.mma kind::i8): every sample
 * scaled per frame by a power of two and split into four 7-bit digits (its
 * leading 28 bits), the 10 digit-level products with weight >= 128^-5 as
 * exact int32 GEMMs in TMEM, recombined in FP64 (relative error ~1e-9 of the
 * largest entry; the FP64 kernel above is exact).  d_work:
 * fqfg_gram_tc_work_bytes(F) bytes (F <= 1024). */
size_t fqfg_gram_tc_work_bytes(int n_frames);
int fqfg_gram_tc_dev(const float* d_x, int n_frames, size_t n_points, size_t v_begin,
                     size_t v_end, double* d_gram, void* d_work, void* stream);

/* Hermitian eigensolve of d_gram [F][F] complex128 (destroyed): d_w [F]
 * eigenvalues descending, d_v [F][F] complex128 eigenvectors (column j). */
int fqfg_eig_dev(double* d_gram, int n_frames, double* d_w, double* d_v, void* stream);

/* The eigensolve the band projection [keep_lo, keep_hi] needs: all
 * eigenvalues (descending, d_w) and only the eigenvector columns of d_v that
 * fqfg_project_pd_dev reads for that band (the band or its complement,
 * whichever is smaller); with <= 8 of them by bisection + inverse iteration,
 * else the full solve.  Other columns of d_v are unspecified. */
int fqfg_eig_band_dev(double* d_gram, int n_frames, int keep_lo, int keep_hi, double* d_w,
                      double* d_v, void* stream);

/* Band projection + fused power Doppler over voxels [v_begin, v_end):
 * Y = X V_b V_b^H (rank min(|b|, F-|b|) form), d_y [F][N] complex64 (may be
 * NULL: PD only), d_pd [N] f64 (may be NULL). */
int fqfg_project_pd_dev(const float* d_x, int n_frames, size_t n_points, size_t v_begin,
                        size_t v_end, const double* d_v, int keep_lo, int keep_hi, float* d_y,
                        double* d_pd, void* stream);

/* Instrumentation (bench.py): per-plan CUDA-event timing of the demod and DAS
 * kernels, summed over the fqfg_das_dev calls since set_timing(plan, 1) (the
 * getter waits for the last call's events), and a process-wide count of
 * kernel launches. */
int fqfg_das_plan_set_timing(fqfg_das_plan plan, int enable);
int fqfg_das_last_timing(fqfg_das_plan plan, double* demod_ms, double* das_ms);
uint64_t fqfg_launch_count(void);

/* Deterministic synthetic RF on device (bench input): uniform(-1, 1) from a
 * counter hash of (seed, index); d_rf has n floats. */
int fqfg_synth_rf_dev(float* d_rf, size_t n, uint64_t seed, void* stream);

/* ---- reconstruction engine (the C++ host of run_beamform + run_post,
 *      src/pipeline/run.cpp:397-487, over das_reconstruct das.hpp:124-127,
 *      svd_filter svd.hpp:23-25 and power_doppler render.hpp:13) ---------- */

/* One engine = one device = one depth slab of the grid (the whole grid when
 * world = 1).  It owns its plan, buffers and streams (created once, reused
 * for every ensemble): RF frames are uploaded 16 at a time (only the samples
 * the slab's voxels can read) into a ring of staging slots while the previous
 * frames are demodulated and beamformed; the filter of ensemble k runs during
 * the DAS of ensemble k + 1.  world > 1: the F x F Gram is summed over the
 * ranks (NCCL, or the caller's all-reduce) and rank 0 gathers the PD. */
typedef struct fqfg_recon_s* fqfg_recon;

/* Stream-ordered sum over the ranks of d_buf[count] (device, f64) on the
 * CUDA stream `stream`; returns 0 on success. */
typedef int (*fqfg_allreduce_fn)(void* user, double* d_buf, size_t count, void* stream);

typedef struct {
  int keep_lo, keep_hi;          /* retained band, 1-based (keep_hi 0: n_frames) */
  int rank, world;               /* this process's depth slab; world 1: whole grid */
  const void* nccl_id;           /* world > 1: fqfg_nccl_unique_id() of rank 0 (128 B) */
  fqfg_allreduce_fn allreduce;   /* world > 1 without NCCL (then no PD gather) */
  void* allreduce_user;
  size_t device_budget;          /* bytes it may allocate (0: 92 % of free memory) */
  int ring_frames;               /* RF staging capacity in frames (0: from the budget) */
  int x_buffers;                 /* IQ ensemble buffers: 0 auto (2 when they fit), 1, 2 */
  int gram_fp64;                 /* Gram engine: 0 tensor cores (fqfg_gram_tc_dev), 1 FP64 */
  int rf_broadcast;              /* 1: rank 0 uploads each RF chunk once (the union of the
                                    ranks' sample windows) and ncclBroadcast carries it to
                                    every rank over NVLink; other ranks pass no host RF.
                                    Needs nccl_id (world 1 allowed: a one-rank communicator) */
} fqfg_recon_opts;

typedef struct {
  int k_begin, k_end;            /* this rank's z-planes */
  size_t v_begin, v_end;         /* its voxels (x-fastest flat indices) */
  int t_begin, t_end;            /* RF samples of each channel it reads */
  int frames_per_pass, n_passes;
  int x_buffers;                 /* 2: the filter overlaps the next ensemble's DAS */
  int ring_frames;               /* RF staging capacity (0 until the first host run) */
  size_t device_bytes;           /* device memory it holds */
  size_t h2d_bytes_per_ensemble; /* host -> device RF bytes per ensemble */
  uint64_t active_samples;       /* active (voxel, element, angle, frame) samples of the slab */
  int tile[3];
  int shape[4];                  /* das2_kernel J, VPW, consumer warps, producer warps */
  int nccl;                      /* 1: collectives over NCCL */
  int gram_fp64;                 /* 1: FP64 CUDA-core Gram, 0: tensor cores */
  int mode;                      /* DAS kernel (fqfg_das_plan_info.mode) */
} fqfg_recon_info;

/* 128-byte ncclUniqueId for fqfg_recon_opts.nccl_id (rank 0 creates it and
 * shares it with the other ranks). */
int fqfg_nccl_unique_id(void* out);

int fqfg_recon_create(const fqfg_rf_desc* rf_desc, const fqfg_grid* grid,
                      const fqfg_probe* probe, const fqfg_bf* bf, const fqfg_recon_opts* opts,
                      fqfg_recon* engine);
int fqfg_recon_info_get(fqfg_recon engine, fqfg_recon_info* info);

/* Reconstruct n ensembles from host RF: rf[k] [F][A][T][E] f32 (page-locked
 * memory lets the uploads overlap the compute) -> pd[k] [N] f64 (rank 0 of a
 * NCCL run gets every voxel; otherwise each rank writes its voxels [v_begin,
 * v_end); NULL: none) and sigma[k] [F] descending (NULL: none).  Synchronous;
 * fails with svd_filter's message if an ensemble is all zero. */
int fqfg_recon_run(fqfg_recon engine, int n, const float* const* rf, double* const* pd,
                   double* const* sigma);

/* The same from device-resident RF d_rf[k] [F][A][T][E] (read in place, no
 * copies); the last ensemble's PD -> d_pd_last [N] device (may be NULL). */
int fqfg_recon_run_dev(fqfg_recon engine, int n, const float* const* d_rf, double* d_pd_last);

/* The IQ ensemble (DAS output, the Casorati matrix) of the last ensemble of
 * the last run for voxels [v_begin, v_end) of this engine's slab -> host iq
 * [F][v_end - v_begin] complex64. */
int fqfg_recon_copy_iq(fqfg_recon engine, size_t v_begin, size_t v_end, float* iq);

/* SvdReport (post/svd.hpp:10-16, svd.cpp:49-76) of the last ensemble of the
 * last run, from its resident IQ: sigma [F] (every singular value,
 * descending) and mode_correlation [F][F] (Pearson correlation of the |U|
 * columns; may be NULL).  world 1 engines only. */
int fqfg_recon_report(fqfg_recon engine, double* sigma, double* mode_correlation);

/* Instrumentation: CUDA-event time of the demodulation, DAS and filter spans
 * of the last run (ms, summed over its ensembles) and of the whole run (from
 * the first enqueued operation to the last result on the host). */
int fqfg_recon_set_timing(fqfg_recon engine, int enable);
int fqfg_recon_last_timing(fqfg_recon engine, double* demod_ms, double* das_ms,
                           double* filter_ms, double* total_ms);
/* Tensor-core DAS K blocks (3 tcgen05.mma of M 128 x N frames_per_pass x
 * K 16 each) issued by the last run (0 with das2): the roofline's MMA work. */
int fqfg_recon_mma_blocks(fqfg_recon engine, unsigned long long* kblocks);
void fqfg_recon_destroy(fqfg_recon engine);

/* ---- Display and scoring, FP64, host buffers ---- */

/* render_db (render.cpp:44-68, render.hpp:20-27): dB re the peak |v|,
 * clipped to [-dr_db, 0], mapped onto [0, 1]; power != 0: 10 log10, else
 * 20 log10.  Errors as the reference (empty volume, dr_db <= 0, all zero). */
int fqfg_render_db(const double* vol, const int* dims, double dr_db, int power, double* out);
/* Device variant over n values (stream-ordered; synchronises once to check
 * the peak). */
int fqfg_render_db_dev(const double* d_vol, size_t n, double dr_db, int power, double* d_out,
                       void* stream);

/* bmode (render.cpp:70-78): |IQ| of complex<double> [N][2], then render_db
 * in amplitude (20 log10). */
int fqfg_bmode(const double* iq, const int* dims, double dr_db, double* out);

/* mip (render.cpp:80-104): out has dims with dims[axis] = 1. */
int fqfg_mip(const double* vol, const int* dims, int axis, double* out);

/* ground_truth_pd (render.cpp:106-145): Gaussian splat (truncated at 3
 * sigma voxels) of the positions xyz [sum counts][3] of n_frames frames,
 * peak-normalised.  Contributions are added with FP64 atomics: equal to the
 * reference up to summation order. */
int fqfg_ground_truth_pd(const double* xyz, const int* counts, int n_frames,
                         const fqfg_grid* grid, double sigma_voxels, double* out);

/* metrics (metrics.cpp:84-101): mse, psnr (dB, +inf when identical), mean
 * local SSIM (11-tap Gaussian window, sigma 1.5, shrunk on short axes). */
int fqfg_metrics(const double* test, const double* reference, const int* dims,
                 double* mse_psnr_ssim);
int fqfg_metrics_dev(const double* d_test, const double* d_reference, const int* dims,
                     double* mse_psnr_ssim, void* stream);

/* ---- RF channel-data synthesis (rf/simulate.hpp) ---- */

/* rf::Transducer (transducer.hpp:13-31): the fields the simulator reads. */
typedef struct {
  int n_elements;
  const double* xyz;               /* [n_elements][3] element centres, m */
  double half_width;               /* element azimuth half-width b, m */
  int subelements;                 /* v per element */
  double pitch;
  double center_frequency;
  double fractional_bandwidth;     /* at -6 dB */
  double elevation_height;         /* <= 0: no lens */
  double elevation_focus;
  double elevation_core_weight;
  double elevation_tail_weight;
  double elevation_aperture_factor;
} fqfg_transducer;

/* rf::MediumParams (simulate.hpp:15-20). */
typedef struct {
  double c;
  double attenuation_db_cm_mhz;
  size_t scatterer_memory_budget;
  double min_fs_ratio;
} fqfg_medium;

/* rf::RfSimStats (simulate.hpp:39-44). */
typedef struct {
  int blocks;
  int frequencies;
  size_t peak_tracked_bytes;
  uint64_t pair_bin_products;
} fqfg_rfsim_stats;

/* rf::RfChunkPlan (simulate.hpp:63-68). */
typedef struct {
  int blocks;
  size_t block_scatterers;
  size_t per_scatterer_bytes;
  size_t fixed_bytes;
} fqfg_rf_chunk_plan;

/* plan_rf_chunks (simulate.hpp:70-72, simulate.cpp:389-416). */
int fqfg_plan_rf_chunks(const fqfg_transducer* t, size_t n_scatterers, const fqfg_medium* m,
                        double sampling_rate, double duration, size_t budget,
                        fqfg_rf_chunk_plan* out);

/* simulate_rf / simulate_rf_chunked (simulate.hpp:50-61): one plane-wave
 * transmit (tx_delays / tx_apod [n_elements]) of a scatterer cloud
 * (positions [n][3], reflectivity [n]) -> rf_out [T][n_elements] f64,
 * T = llround(fs * duration), t0 = 0.  chunked = 0: the reference's
 * single-pass rule (error unless the pair geometry fits the medium budget);
 * chunked = 1: budget (0 = the medium's) only sets the reported block plan --
 * the GPU streams scatterers regardless.  Errors as the reference. */
int fqfg_simulate_rf(const double* positions, const double* reflectivity, size_t n_scatterers,
                     const fqfg_transducer* t, const double* tx_delays, const double* tx_apod,
                     const fqfg_medium* m, double sampling_rate, double duration, int chunked,
                     size_t budget, double* rf_out, int* n_samples, fqfg_rfsim_stats* stats);

/* Device-resident variant (no validation beyond shapes, no host copies):
 * d_positions / d_reflectivity / d_elements / d_tx_delays / d_tx_apod are
 * device pointers; writes d_rf32 [T][E] f32 (nullable) and/or d_rf64. */
int fqfg_simulate_rf_dev(const double* d_positions, const double* d_reflectivity,
                         size_t n_scatterers, const fqfg_transducer* t, const double* d_elements,
                         const double* d_tx_delays, const double* d_tx_apod, const fqfg_medium* m,
                         double sampling_rate, double duration, float* d_rf32, double* d_rf64,
                         void* stream);

#ifdef __cplusplus
}
#endif

#endif
