/*
 * subsurf_b200.h -- C ABI of the B200-native SUBSURF time step.
 *
 * Plain pointers and sizes only.  Host arrays use the reference's ghost-padded
 * fp64 layout (Field4D, grid.hpp:91-119): P = (n1+2)(n2+2)(n3+2)(n4+2) doubles,
 *   idx = ((l*kMax + k)*jMax + j)*iMax + i,
 * per-face arrays hold 8 doubles per padded doxel in kFaceOffsets order
 * (grid.cpp:67-80, f = 2*axis + (sign > 0)).
 *
 * Every entry point replaces one reference function (cited below, file:line in
 * /root/reference/proj).  Errors: the reference throws; here a status code is
 * returned and ss_last_error() holds the message.  The C++ mirror
 * (include/subsurf_b200/subsurf.hpp) maps the codes back onto the reference's
 * exception types (errors.hpp:9-39).
 *
 * There is no CPU fallback: without a usable CUDA device every compute entry
 * point returns SS_ERR_CUDA.
 */
#ifndef SUBSURF_B200_H
#define SUBSURF_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SS_API __attribute__((visibility("default")))

typedef enum {
    SS_OK = 0,
    SS_ERR_VALIDATION = 1, /* ValidationError  (errors.hpp:15-18)            */
    SS_ERR_NOCONVERGE = 2, /* SolverError      (errors.hpp:26-33)            */
    SS_ERR_NONFINITE = 3,  /* NumericalError   (errors.hpp:36-39)            */
    SS_ERR_CUDA = 4,       /* device missing / CUDA runtime failure          */
    SS_ERR_NCCL = 5,       /* multi-GPU transport failure                    */
    SS_ERR_STATE = 6       /* API misuse (session not prepared, ...)         */
} ss_status;

/* GridSpec (grid.hpp:16-46) */
typedef struct {
    int n1, n2, n3, n4;
    double h1, h2, h3, h4;
} ss_grid;

/* CenterRow (io.hpp:23-27): frame 0-based, x,y,z 0-based doxel coordinates */
typedef struct {
    int frame;
    double x, y, z, radius;
} ss_center;

/* SegmentationParams (solver.hpp:77-85) flattened: SolverParams, SmoothingParams,
 * ThresholdParams, EdgeParams, InitParams, rescale_radius.  Field order is the
 * ABI; defaults are the reference's (cli.cpp:73-107). */
typedef struct {
    double tau, epsilon, omega, sor_tol;
    int sor_max_iter, n_steps, rescale_each_step;
    double sor_rel_tol;   /* extension: > 0 => sor_tol = rel * ||u^{n-1}||_2 per step */
    double sigma;
    int smooth_steps;
    double smooth_tol;
    int smooth_max_iter;
    double smooth_omega;
    double lambda, background;
    double K, delta, vartheta;
    double init_v, init_R;
    int init_profile;     /* 0 = peak, 1 = linear (seedinit.hpp:10) */
    double rescale_radius;/* NaN => per-row radii (std::nullopt); any other value is the
                           * explicit radius, r <= 0 included (a ball of at most one
                           * doxel: the rescale is a no-op, seedinit.cpp:73-88) */
} ss_seg_params;

/* per-step diagnostics line (solver.cpp:433-438) */
typedef struct {
    int iterations;
    double residual, tol, umin, umax;
} ss_step_diag;

SS_API const char* ss_last_error(void);
SS_API int ss_abi_version(void); /* 6 (round 2: ss_session_step_host_async / ss_session_wait) */
/* number of this library's kernel launches since load (process-wide) */
SS_API unsigned long long ss_launch_count(void);
/* 1 if a CUDA device is usable, else 0 (sets ss_last_error) */
SS_API int ss_device_available(void);

/* ---------------- per-call API: the reference's free functions ---------------- */

/* assemble_step (solver.hpp:50-51, solver.cpp:23-77).  G may be NULL (G == 1).
 * offdiag: 8*P, diag: P, abar: P (ghost rows zero, like the reference). */
SS_API ss_status ss_assemble_step(const ss_grid* g, const double* u_prev, const double* G,
                                  double tau, double epsilon, double* offdiag, double* diag,
                                  double* abar);
/* assemble_heat_step (solver.hpp:55, solver.cpp:79-116) */
SS_API ss_status ss_assemble_heat_step(const ss_grid* g, double dt, double* offdiag,
                                       double* diag, double* abar);
/* redblack_sor (solver.hpp:69-70, solver.cpp:379-397).  u: in = u_guess (its
 * ghosts are the Dirichlet data), out = result.  On SS_ERR_NOCONVERGE u holds
 * the last iterate and *iterations / *residual are set (SolverError fields).
 * workers > 1 is accepted and ignored (results are worker-count invariant,
 * solver.cpp:144-156). */
SS_API ss_status ss_redblack_sor(const ss_grid* g, const double* offdiag, const double* rhs,
                                 double* u, double omega, double sor_tol, int sor_max_iter,
                                 int workers, int* iterations, double* residual);
/* face_coefficients (edge.hpp:95-97, edge.cpp:73-99); G: 8*P, ghosts = 1 */
SS_API ss_status ss_face_coefficients(const ss_grid* g, const double* I0s, const double* ITs,
                                      double K, double delta, double vartheta, double* G);
/* heat_smooth (preprocess.hpp:23, preprocess.cpp:25-51) */
SS_API ss_status ss_heat_smooth(const ss_grid* g, const double* image, double sigma, int steps,
                                double omega, double sor_tol, int sor_max_iter, double* out);
/* local_threshold (preprocess.hpp:36-37, preprocess.cpp:53-102) */
SS_API ss_status ss_local_threshold(const ss_grid* g, const double* image, const ss_center* c,
                                    int n, double lambda, double background, double* out);
/* build_initial (seedinit.hpp:25-26, seedinit.cpp:42-66) */
SS_API ss_status ss_build_initial(const ss_grid* g, const ss_center* c, int n, double v,
                                  double R, int profile, double* u);
/* local_rescale (seedinit.hpp:32-33, seedinit.cpp:68-99); radius NaN => per-row radii
 * (std::nullopt), otherwise the explicit radius (r <= 0: no-op, as in the reference) */
SS_API ss_status ss_local_rescale(const ss_grid* g, double* u, const ss_center* c, int n,
                                  double radius);
/* apply_dirichlet (grid.cpp:126-136), apply_mirror_ghosts (grid.cpp:138-156),
 * interior_minmax (grid.cpp:158-171) on a padded host field */
SS_API ss_status ss_apply_dirichlet(const ss_grid* g, double* f, double value);
SS_API ss_status ss_apply_mirror_ghosts(const ss_grid* g, double* f);
SS_API ss_status ss_interior_minmax(const ss_grid* g, const double* f, double* lo, double* hi);
/* extract_mask (tracking.hpp:55, tracking.cpp:35-52): n4 frames of n1*n2*n3 bytes */
SS_API ss_status ss_extract_mask(const ss_grid* g, const double* u, double level,
                                 uint8_t* mask);
/* ---------------- cell tracking (tracking.hpp, tracking.cpp) ----------------
 * Frames are n4 volumes of n1*n2*n3 voxels, 0-based, x fastest (MaskFrames /
 * LabelField, tracking.hpp:14-34).  Per-voxel work (labelling, distance
 * transform, centres, predecessor candidates) runs on the GPU; the per-cell
 * linking on the host. */
typedef struct { /* CellRecord (tracking.hpp:36-42) */
    int frame, label;   /* 0-based frame, label 1..k */
    int cx, cy, cz;     /* 0-based centre voxel */
    int max_distance;   /* 26-neighbourhood BFS distance to background at the centre */
    long long voxel_count;
} ss_cell_record;
typedef struct { /* TrajectoryPoint (io.hpp:36-40) */
    int trajectory_id, frame;
    double x, y, z;
} ss_track_point;
/* label_components (tracking.hpp:59, tracking.cpp:69-127): labels n4*n1*n2*n3,
 * labels_per_frame n4 */
SS_API ss_status ss_label_components(const ss_grid* g, const uint8_t* mask, int32_t* labels,
                                     int* labels_per_frame);
/* distance_centers (tracking.hpp:64, tracking.cpp:189-215): one record per
 * (frame, label) in that order; *n_records = sum of labels_per_frame.  Fails with
 * SS_ERR_VALIDATION (and sets *n_records) when capacity is too small. */
SS_API ss_status ss_distance_centers(const ss_grid* g, const int32_t* labels,
                                     const int* labels_per_frame, ss_cell_record* out,
                                     int capacity, int* n_records);
/* backtrack_link (tracking.hpp:69-70, tracking.cpp:220-296): partial trajectories
 * as record indices (into the distance_centers order) with frames increasing;
 * chain c = record_index[chain_start[c] .. chain_start[c+1]-1], chain_start has
 * n_records + 1 entries; *n_chains set. */
SS_API ss_status ss_backtrack_link(const ss_grid* g, const int32_t* labels,
                                   const int* labels_per_frame, const ss_cell_record* records,
                                   int n_records, int* record_index, int* chain_start,
                                   int* n_chains);
/* track (tracking.hpp:81-82, tracking.cpp:374-401): extract_mask(u, level), the
 * whole pipeline, trajectory points in output order; *n_points set; fails with
 * SS_ERR_VALIDATION when capacity is too small. */
SS_API ss_status ss_track(const ss_grid* g, const double* u, double level, int window,
                          double radius, ss_track_point* out, int capacity, int* n_points);

/* segment (solver.hpp:91-92, solver.cpp:405-441).  u0 may be NULL
 * (build_initial); diags: n_steps entries or NULL.  On SS_ERR_NOCONVERGE the
 * failing step's diag holds the iterations and last residual, with tol = -1. */
SS_API ss_status ss_segment(const ss_grid* g, const double* image, const ss_center* c, int n,
                            const ss_seg_params* p, const double* u0, double* u_out,
                            ss_step_diag* diags);

/* ---------------- device-resident session (the performance boundary) ---------------- */
typedef struct ss_session ss_session;

SS_API ss_status ss_session_create(const ss_grid* g, int device, ss_session** out);
/* the grid split along l into n_slabs slabs on ONE device (Partition::create
 * semantics, parallel.cpp:9-19), exchanging halo planes by device copies:
 * the multi-GPU decomposition exercised on a single GPU (bit-identical to 1 slab) */
SS_API ss_status ss_session_create_group(const ss_grid* g, int n_slabs, int device, ss_session** out);
/* multi-GPU: one process per GPU.  Rank 0 calls ss_nccl_unique_id and shares the
 * 128 bytes (e.g. torch.distributed broadcast); every rank then creates its slab
 * session.  Host arrays of a distributed session are the rank's padded slab:
 * global planes l_begin-1 .. l_begin+l_count (ss_session_slab). */
SS_API ss_status ss_nccl_unique_id(uint8_t out[128]);
SS_API ss_status ss_session_create_dist(const ss_grid* g, int rank, int world, const uint8_t uid[128],
                                        int device, ss_session** out);
/* one rank's slab with the halo exchanges and all-gathers staged through the host and
 * the caller's callbacks (ABI 5): sendrecv sends `bytes` to rank `peer` and receives as many
 * from it; allgather concatenates every rank's `bytes` in rank order.  Return 0 on success.
 * Same messages as the NCCL transport, so results equal the single domain's bit for bit;
 * synchronous -- for running the multi-process path where one GPU serves several ranks
 * (tests), not a data path. */
typedef struct {
    void* ctx;
    int (*sendrecv)(void* ctx, int peer, const void* send, void* recv, size_t bytes);
    int (*allgather)(void* ctx, const void* local, void* all, size_t bytes);
} ss_host_comm;
SS_API ss_status ss_session_create_dist_host(const ss_grid* g, int rank, int world, const ss_host_comm* comm,
                                             int device, ss_session** out);
/* 1-based first owned slice, owned slice count (whole grid unless distributed), world size */
SS_API ss_status ss_session_slab(ss_session* s, int* l_begin, int* l_count, int* world);
SS_API ss_status ss_session_destroy(ss_session* s);
/* the cudaStream_t every kernel of this session is launched on */
SS_API void* ss_session_stream(ss_session* s);
/* segment() preamble (solver.cpp:408-426): u0 (or build_initial) + local_rescale,
 * local_threshold, heat_smooth x2, face_coefficients, apply_dirichlet. */
SS_API ss_status ss_session_prepare(ss_session* s, const double* image, const ss_center* c,
                                    int n, const ss_seg_params* p, const double* u0);
/* one time step of the loop body (solver.cpp:428-438): assemble_step,
 * redblack_sor (rhs = guess = u), local_rescale.  diag may be NULL; on
 * SS_ERR_NOCONVERGE it holds the iterations and the last residual. */
SS_API ss_status ss_session_step(ss_session* s, ss_step_diag* diag);
/* host <-> device copies of u (padded fp64, ghosts included) */
SS_API ss_status ss_session_set_u(ss_session* s, const double* host_u);
SS_API ss_status ss_session_get_u(ss_session* s, double* host_u);
SS_API ss_status ss_session_get_mask(ss_session* s, double level, uint8_t* mask);
/* track() on the session's device-resident u (no host round trip of u); single-process
 * sessions (one slab or an in-process slab group) */
SS_API ss_status ss_session_track(ss_session* s, double level, int window, double radius,
                                  ss_track_point* out, int capacity, int* n_points);
/* fixed-sweep mode (BASELINE config 4): assemble at the current u, then exactly
 * n_sweeps red+black sweeps with no stopping test; *residual = last residual.
 * Non-finite coefficients: SS_ERR_NONFINITE (solver.cpp:71-75). */
SS_API ss_status ss_session_fixed_sweeps(ss_session* s, int n_sweeps, double* residual);
/* one time step with the host's copy of u (ABI 5): u_in (or NULL: keep the device's u)
 * becomes the interior of u^{n-1}, then the time step of ss_session_step (n_sweeps = 0,
 * to tolerance) or ss_session_step_fixed (n_sweeps > 0), and the interior of u^n goes to
 * u_out (or NULL).  Host arrays are COMPACT interiors: n1*n2*n3*n4 doubles of the owned
 * slices, i fastest, no ghost layer (the ghosts are the session's Dirichlet data, 0 in
 * segment(), solver.cpp:425).  With page-locked u_in on a single-slab session the upload
 * streams in slice chunks and the assembly of each chunk starts as soon as its l+1
 * neighbour is in.  ss_session_set_u_interior / _get_u_interior: the copies alone. */
SS_API ss_status ss_session_step_host(ss_session* s, const double* u_in, double* u_out, int n_sweeps,
                                      ss_step_diag* diag);
/* ss_session_step_host with the result's download left in flight (ABI 6; one slab per
 * process -- a single domain or a distributed rank -- and page-locked u_in / u_out, else exactly ss_session_step_host): returns once the step is
 * computed and its D2H enqueued; u_out is complete after ss_session_wait (or any call that
 * reads it).  When the next call's u_in is this call's u_out, every upload chunk waits on
 * the device for its download chunk, so the D2H of step n and the H2D of step n + 1 run
 * concurrently in the two PCIe directions; the data still makes the full round trip. */
SS_API ss_status ss_session_step_host_async(ss_session* s, const double* u_in, double* u_out, int n_sweeps,
                                            ss_step_diag* diag);
/* wait for every transfer of ss_session_step_host_async and the session's stream */
SS_API ss_status ss_session_wait(ss_session* s);
SS_API ss_status ss_session_set_u_interior(ss_session* s, const double* u);
SS_API ss_status ss_session_get_u_interior(ss_session* s, double* u);
/* one time step of BASELINE config 4 (ABI 5): ss_session_step with exactly n_sweeps
 * sweeps and no stopping test in place of the solve to tolerance (assemble_step,
 * n_sweeps red+black sweeps, local_rescale).  The reference has no such mode: its
 * redblack_sor throws SolverError at max_iter and drops the iterate (solver.cpp:391-395);
 * this is that iterate (tests pin it against the reference, tests/golden/pins.json).
 * diag: iterations = n_sweeps, residual = the last residual, tol = 1.  diag == NULL (here
 * and in the host-buffer calls with n_sweeps > 0): no residual is evaluated at all. */
SS_API ss_status ss_session_step_fixed(ss_session* s, int n_sweeps, ss_step_diag* diag);
/* run_levelset_row (eoc.cpp:83-137): the EOC verification row n (10/20/40/80/160) on a
 * session created for the grid n^4 with h = 2.5/n; *err = space-time L2 error,
 * *sweeps = total SOR sweeps (may be NULL).  EocConfig defaults: omega 1.5, tol 1e-8. */
SS_API ss_status ss_session_eoc_row(ss_session* s, int n, double omega, double sor_tol, int sor_max_iter,
                                    double* err, long long* sweeps);
/* 0 = host-driven chunked loop, 1 = CUDA-graph conditional loop (default) */
SS_API ss_status ss_session_set_loop_mode(ss_session* s, int mode);
/* SOR kernel: 4 = auto (default: 3 when the solve's working set fits L2, else the TMA
 * two-pass with whole-row or 2D-tiled items, whichever keeps more lanes busy),
 * 1 = TMA-fed two-pass with whole-row items, 5 = TMA two-pass with 2D-tiled items
 * (tensor maps), 0 = plain LDG two-pass, 3 = resident (the whole solve in one
 * cooperative launch), 2 = two-iteration TMA wavefront (experimental; measured slower
 * on B200) */
SS_API ss_status ss_session_set_kernel(ss_session* s, int kernel);
/* kernel code (as above; 7 = one-sweep k-wavefront) the session's last segmentation
 * SOR solve ran after the support checks (-1: none yet) */
SS_API ss_status ss_session_sor_kernel(ss_session* s, int* kernel);
/* per-pass CUDA-event timing of the SOR kernels (forces the host-driven loop) */
SS_API ss_status ss_session_set_profiling(ss_session* s, int enable);
/* accumulated since the last call (then reset): total ms in red passes, black
 * passes, assembly kernels and rescale, and the number of each (profiling mode);
 * loop_ms / loop_passes: device time of the SOR loops (events around each CUDA-graph
 * solve, recorded in normal running at no cost) and the colour passes they ran;
 * halo_*: exchange time exposed vs overlapped (multi-slab, profiling mode) */
typedef struct {
    double red_ms, black_ms, assemble_ms, rescale_ms;
    long long red_n, black_n, assemble_n, rescale_n;
    long long sweeps; /* completed red+black sweeps */
    double loop_ms;
    long long loop_passes;
    /* multi-slab solves with the halo exchange on the comm stream (profiling mode):
     * halo_ms = device time of the exchanges (the comm stream, events around each),
     * halo_exposed_ms = how much of it the compute stream waited for after its interior
     * slices were done (the rest overlapped them), halo_n = exchanges timed */
    double halo_ms, halo_exposed_ms;
    long long halo_n;
} ss_profile;
SS_API ss_status ss_session_profile(ss_session* s, ss_profile* out);
/* the coefficients a step would assemble at the session's current u (the tile kernel of the
 * device-resident path, G included) as padded fp64 off-diagonals (8 * P; ghost doxels 0) --
 * what assemble_step (solver.cpp:23-77) returns in StepCoefficients::offdiag; single slab */
SS_API ss_status ss_session_assemble_export(ss_session* s, double* offdiag);
/* self-test of the assembly kernel's rsqrt tail (assemble_tile.cu): the largest relative
 * error of the hardware rsqrt.approx.f64 over every normal positive input high word; the
 * tail's exactness argument needs it below 2^-11 (two Newton steps then leave a few ulps) */
SS_API ss_status ss_selftest_rsqrt(double* eps0);
/* algorithmic bytes of one SOR colour pass: 28 B x interior doxels (SURVEY 8(d):
 * 56 B per doxel per red+black sweep) */
SS_API double ss_sor_pass_bytes(const ss_grid* g);

#ifdef __cplusplus
}
#endif
#endif
