/*
 * sfmcov_b200 — C ABI of the B200-native camera-covariance hot path.
 *
 * Drop-in boundary for the reference `sfmcov` library (arXiv 1808.02414,
 * /root/reference/proj).  The reference has no FFI or plugin registry; its
 * "operator API" is the free-function set in namespace sfmcov.  Each entry
 * point below replaces one of those functions (cited per declaration) with
 * plain pointers and sizes, no C++ or torch types.  include/sfmcov_b200.hpp
 * wraps this ABI back into the reference's C++ signatures, and
 * paper_1808_02414_b200/sfmcov.py into Python.
 *
 * Conventions
 *  - All arithmetic is FP64; indices int32 (observation ids < 2^31).
 *  - Cameras have P in {8, 9} parameters: P = 8 is the reference camera
 *    (r, C, c, k), include/sfmcov/types.hpp:28-39; P = 9 adds k2
 *    (u = f(1 + k1 rho + k2 rho^2) u_n), the BASELINE.json camera.
 *  - Matrix blocks are row-major within a block unless stated otherwise.
 *  - Return value = error kind (0 = ok), mirroring sfmcov::ErrorKind
 *    (include/sfmcov/error.hpp:9-16); the stage and the full
 *    "stage: message" text land in sfmcov_error, exactly as the reference's
 *    Error::what() would read.
 *  - Calls are synchronous and thread-safe per handle; a handle owns one
 *    CUDA device, one stream and a grow-only device workspace.
 *  - There is no CPU fallback: on a machine without a usable CUDA device
 *    sfmcov_cuda_create fails with SFMCOV_ERR_DEVICE.
 */
#ifndef SFMCOV_B200_H
#define SFMCOV_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* error kinds: include/sfmcov/error.hpp:9-16 (+ device, not in the reference) */
enum {
    SFMCOV_OK = 0,
    SFMCOV_ERR_IO = 1,
    SFMCOV_ERR_PARSE = 2,
    SFMCOV_ERR_INVARIANT = 3,
    SFMCOV_ERR_DEGENERATE = 4,
    SFMCOV_ERR_DIMENSION = 5,
    SFMCOV_ERR_SIZE_GUARD = 6,
    SFMCOV_ERR_DEVICE = 7
};

/* Scene, structure-of-arrays.  Replaces sfmcov::Reconstruction
 * (include/sfmcov/types.hpp:52-66).  Pointers are host or device memory
 * depending on the entry point; the caller owns them. */
typedef struct sfmcov_scene {
    int32_t n_cams;
    int32_t n_pts;
    int32_t n_obs;
    int32_t cam_params;        /* P: 8 or 9 */
    const double* cams;        /* n_cams x P: r(3) C(3) c|f k|k1 [k2] */
    const double* pts;         /* n_pts x 3 */
    const int32_t* obs_cam;    /* n_obs */
    const int32_t* obs_pt;     /* n_obs */
    const double* obs_u;       /* n_obs x 2, validated only; may be NULL */
    const double* obs_sigma;   /* n_obs x 4 (row-major 2x2); NULL = identity */
} sfmcov_scene;

/* sfmcov::CovarianceOptions (include/sfmcov/covariance.hpp:71-75). */
typedef struct sfmcov_options {
    int32_t threads;                  /* accepted and ignored (results never depend on it) */
    int32_t point_covariances;        /* sfmcov_cuda_compute_covariance_full only */
    int32_t camera_cross_covariances; /* sfmcov_cuda_compute_covariance_full only */
    int32_t reserved;
} sfmcov_options;

/* sfmcov::CovarianceDiagnostics (include/sfmcov/covariance.hpp:49-60).
 * On the Cholesky route min/max_pivot are taken over the Cholesky pivots
 * diag(L)^2 of the gauge-augmented camera matrix and |eig(E)| of the 7x7
 * border block; inertia is (P*n, 7) on success. */
typedef struct sfmcov_diagnostics {
    double scale_min;
    double scale_max;
    double min_pivot;
    double max_pivot;
    int32_t inertia_positive;
    int32_t inertia_negative;
    int32_t negative_eigenvalue_warnings;
    int32_t n_flagged;             /* total flagged columns */
    int64_t peak_dense_bytes;
    int64_t largest_dense_dim;     /* P*n + 7, as the reference reports */
    int64_t* flagged;              /* caller buffer for flagged column ids (may be NULL) */
    int64_t flagged_capacity;
} sfmcov_diagnostics;

typedef struct sfmcov_error {
    int32_t kind;
    char stage[32];
    char message[480];             /* "stage: message" */
} sfmcov_error;

typedef struct sfmcov_handle sfmcov_handle;

/* ---- lifecycle ----------------------------------------------------------- */
sfmcov_handle* sfmcov_cuda_create(int32_t device, sfmcov_error* err);
void sfmcov_cuda_destroy(sfmcov_handle* h);
/* The handle's CUDA stream (cudaStream_t) for callers that time or order work. */
void* sfmcov_cuda_stream(sfmcov_handle* h);
/* The handle's device ordinal. */
int32_t sfmcov_cuda_device(sfmcov_handle* h);
/* The i-th worker handle of h (same device, own stream and workspace;
 * created on first use, destroyed with h): batched independent problems. */
sfmcov_handle* sfmcov_cuda_worker(sfmcov_handle* h, int32_t i, sfmcov_error* err);

/* ---- full pipeline --------------------------------------------------------
 * Replaces sfmcov::compute_covariance (include/sfmcov/covariance.hpp:110-111,
 * src/covariance.cpp:323-350).  Host scene in, host per-camera blocks out:
 * cam_cov is n_cams x P x P (row-major blocks). */
int32_t sfmcov_cuda_compute_covariance(sfmcov_handle* h, const sfmcov_scene* scene,
                                       const sfmcov_options* opts, double* cam_cov,
                                       sfmcov_diagnostics* diag, sfmcov_error* err);

/* With the reference's optional outputs (CovarianceOptions::point_covariances
 * / camera_cross_covariances; covariance.cpp:283-348, result fields
 * point_cov and camera_matrix, covariance.hpp:62-69): point_cov is
 * n_pts x 3 x 3 (row-major blocks), camera_matrix the full (P n) x (P n)
 * camera covariance, column-major (symmetric up to the last bit, like the
 * reference's S Z_inv S); camera_cov equals its diagonal blocks bitwise when
 * it is requested.  A buffer may be NULL when its option is off. */
int32_t sfmcov_cuda_compute_covariance_full(sfmcov_handle* h, const sfmcov_scene* scene,
                                            const sfmcov_options* opts, double* cam_cov, double* point_cov,
                                            double* camera_matrix, sfmcov_diagnostics* diag,
                                            sfmcov_error* err);

/* Same, with every scene pointer and d_cam_cov in device memory of the
 * handle's device (inputs resident in HBM; used by the device-timed bench). */
int32_t sfmcov_cuda_compute_covariance_device(sfmcov_handle* h, const sfmcov_scene* d_scene,
                                              const sfmcov_options* opts, double* d_cam_cov,
                                              sfmcov_diagnostics* diag, sfmcov_error* err);

/* ---- stage entry points (host buffers; parity tests) ------------------- */

/* build_observation_index (src/scene.cpp:80-90) as CSR: ascending observation
 * ids per camera / per point.  off_* are int64 (n+1 / m+1). */
int32_t sfmcov_cuda_observation_index(sfmcov_handle* h, const sfmcov_scene* scene,
                                      int64_t* off_cam, int32_t* idx_cam,
                                      int64_t* off_pt, int32_t* idx_pt, sfmcov_error* err);

/* assemble_jacobian (include/sfmcov/projection.hpp:54, src/projection.cpp:80-105):
 * cam_blocks n_obs x 2 x P, point_blocks n_obs x 2 x 3, observation order. */
int32_t sfmcov_cuda_jacobian(sfmcov_handle* h, const sfmcov_scene* scene,
                             double* cam_blocks, double* point_blocks, sfmcov_error* err);

/* gauge_nullspace (include/sfmcov/nullspace.hpp:33, src/nullspace.cpp:64-68):
 * H is (P*n + 3m) x 7, row-major. */
int32_t sfmcov_cuda_nullspace(sfmcov_handle* h, const sfmcov_scene* scene, double* H,
                              sfmcov_error* err);

/* build_fisher_blocks + condition_columns (include/sfmcov/covariance.hpp:80-86,
 * src/covariance.cpp:33-116), unconditioned blocks: D n x P x P, A m x 3 x 3,
 * couplings n_obs x P x 3; s_a (P*n + 3m), s_b (7).  Any output may be NULL.
 * Like the reference function it does not run the scene validation, so a
 * non-SPD sigma fails in stage "fisher". */
int32_t sfmcov_cuda_fisher(sfmcov_handle* h, const sfmcov_scene* scene, double* D, double* A,
                           double* couplings, double* s_a, double* s_b,
                           sfmcov_diagnostics* diag, sfmcov_error* err);

/* schur_reduce on the conditioned system (include/sfmcov/covariance.hpp:94-95,
 * src/covariance.cpp:137-194): dense symmetric Z_p, (P*n+7)^2, column-major. */
int32_t sfmcov_cuda_schur(sfmcov_handle* h, const sfmcov_scene* scene, double* z_p,
                          sfmcov_error* err);

/* Dense gauge-free inversion kernel on an arbitrary SPD matrix (column-major
 * n x n, host): Cholesky + triangular inverse + diagonal-block extraction of
 * A^-1 with block size `block`.  blocks: (n / block) x block x block.  The
 * same device code path invert_schur's replacement uses. */
int32_t sfmcov_cuda_spd_inverse_blocks(sfmcov_handle* h, const double* a, int64_t n, int32_t block,
                                       double* blocks, double* min_pivot, double* max_pivot,
                                       sfmcov_error* err);

/* nullspace_residual (include/sfmcov/nullspace.hpp:36, src/nullspace.cpp:70-83):
 * max |J H| / (max |J| max |H|) over the scene's Jacobian (formed on the
 * GPU), H host (P*n + 3m) x b row-major, b >= 1. */
int32_t sfmcov_cuda_nullspace_residual(sfmcov_handle* h, const sfmcov_scene* scene, const double* H, int32_t b,
                                       double* residual, sfmcov_error* err);

/* ---- stage functions on a caller-supplied block system ------------------
 * The reference's BorderedSystem (include/sfmcov/covariance.hpp:36-47) as
 * arrays: D n x P x P, A m x 3 x 3 (row-major blocks), couplings
 * t x P x 3 in observation order with their obs_cam / obs_pt, border
 * (P*n + 3m) x b row-major (0 <= b <= 32).  Host buffers; the work runs on
 * the handle's device. */
/* condition_columns (covariance.hpp:86, src/covariance.cpp:84-116): s_a
 * (P*n + 3m), s_b (b), the flagged columns (ascending; n_flagged = total). */
int32_t sfmcov_cuda_condition_columns(sfmcov_handle* h, int32_t n, int32_t m, int32_t P, int32_t b, const double* D,
                                      const double* A, const double* border, double* s_a, double* s_b,
                                      int64_t* flagged, int64_t flagged_capacity, int64_t* n_flagged,
                                      sfmcov_error* err);
/* apply_conditioning (covariance.hpp:88, src/covariance.cpp:118-135), in place. */
int32_t sfmcov_cuda_apply_conditioning(sfmcov_handle* h, int32_t n, int32_t m, int32_t t, int32_t P, int32_t b,
                                       double* D, double* A, double* couplings, const int32_t* obs_cam,
                                       const int32_t* obs_pt, double* border, const double* s_a, const double* s_b,
                                       sfmcov_error* err);
/* schur_reduce (covariance.hpp:94-95, src/covariance.cpp:137-194): z_p
 * (P*n + b)^2 column-major, exactly symmetric; a_inv m x 3 x 3 (may be NULL).
 * A singular 3x3 point block fails in stage "schur" naming the point. */
int32_t sfmcov_cuda_schur_system(sfmcov_handle* h, int32_t n, int32_t m, int32_t t, int32_t P, int32_t b,
                                 const double* D, const double* A, const double* couplings, const int32_t* obs_cam,
                                 const int32_t* obs_pt, const double* border, double* z_p, double* a_inv,
                                 sfmcov_error* err);
/* invert_schur (covariance.hpp:100, src/covariance.cpp:196-257) on any
 * symmetric nonsingular matrix (dim x dim, column-major): the GPU Jacobi
 * eigendecomposition (eigen.cu), z_inv = V diag(1/lambda) V^T, symmetrised;
 * inertia from the signs of lambda, min/max_pivot = min/max |lambda| (the
 * reference reads them off Bunch-Kaufman pivots), the same 1e-12 ratio test. */
int32_t sfmcov_cuda_invert_symmetric(sfmcov_handle* h, const double* z, int64_t dim, double* z_inv,
                                     double* min_pivot, double* max_pivot, int32_t* inertia_positive,
                                     int32_t* inertia_negative, sfmcov_error* err);
/* extract_camera_covariances (covariance.hpp:104-105, src/covariance.cpp:259-279):
 * cam_cov[i] = S_i z_inv[ii] S_i (s_a may be NULL = unit), PSD warnings. */
int32_t sfmcov_cuda_extract_camera_blocks(sfmcov_handle* h, const double* z_inv, int64_t dim, int32_t n, int32_t P,
                                          const double* s_a, double* cam_cov, int32_t* warnings, sfmcov_error* err);
/* full_covariance (covariance.hpp:115, src/covariance.cpp:352-397): the
 * (P*n + 3m)^2 parameter covariance (column-major) as the parameter block of
 * the inverse of the conditioned bordered Fisher matrix, refused above
 * max_params with SFMCOV_ERR_SIZE_GUARD (stage "full-covariance"). */
int32_t sfmcov_cuda_full_covariance(sfmcov_handle* h, const sfmcov_scene* scene, int64_t max_params, double* sigma,
                                    sfmcov_error* err);

/* ---- multi-GPU (one process per GPU) --------------------------------------
 * The same pipeline with the Schur pair work and the dense inversion split
 * over ranks: chunks of the camera-pair-sorted observation-pair list per
 * rank + an NCCL all-reduce of the camera-pair blocks, and a 1D
 * block-cyclic fused Cholesky / triangular-inverse sweep (panel broadcast
 * over NVLink).  Every rank passes the same host scene and receives every
 * camera block.  Replaces compute_covariance (covariance.hpp:110-111) for
 * multi-GPU callers; NCCL is loaded at run time (libnccl.so.2). */
/* 128-byte NCCL unique id, created on rank 0 and sent to the others by the caller. */
int32_t sfmcov_nccl_unique_id(char* id128, sfmcov_error* err);
/* Attach the handle to rank `rank` of `nranks` (nranks = 1: no communicator). */
int32_t sfmcov_cuda_comm_init(sfmcov_handle* h, const char* id128, int32_t nranks, int32_t rank,
                              sfmcov_error* err);
int32_t sfmcov_cuda_compute_covariance_sharded(sfmcov_handle* h, const sfmcov_scene* scene,
                                               const sfmcov_options* opts, double* cam_cov,
                                               sfmcov_diagnostics* diag, sfmcov_error* err);
/* Same with every scene pointer and d_cam_cov in device memory. */
int32_t sfmcov_cuda_compute_covariance_sharded_device(sfmcov_handle* h, const sfmcov_scene* d_scene,
                                                      const sfmcov_options* opts, double* d_cam_cov,
                                                      sfmcov_diagnostics* diag, sfmcov_error* err);
/* Stage A of the multi-GPU path: 0 (default) = every rank runs validation ...
 * Schur factors on the whole scene (the single-GPU FP64 summation order; the
 * path stays within 1e-9 of the exact inverse at config 4), 1 = point-sharded
 * (each rank its points' sub-scene, per-camera sums all-reduced: less work per
 * rank, but the camera sums are added in another order and config 4's
 * ill-conditioned cameras then move by up to 1.2e-8). */
void sfmcov_cuda_set_sharded_stage_a(sfmcov_handle* h, int32_t on);
/* The distributed code path with `ranks` ranks emulated on this one device
 * (in-process copies instead of NCCL); for testing the multi-GPU path. */
int32_t sfmcov_cuda_compute_covariance_emulated(sfmcov_handle* h, const sfmcov_scene* scene,
                                                const sfmcov_options* opts, int32_t ranks, double* cam_cov,
                                                sfmcov_diagnostics* diag, sfmcov_error* err);
/* Host-only partition plans (no GPU needed): padded dimension of the
 * camera-aligned layout, the rank's local column count and which cameras'
 * blocks it extracts; and its chunk range of the sorted pair list. */
int32_t sfmcov_plan_dense(int32_t n_cams, int32_t cam_params, int32_t nranks, int32_t rank,
                          int32_t panel_blocks, int64_t* npad, int64_t* local_cols, int32_t* cam_owned);
int32_t sfmcov_plan_chunks(int64_t nchunks, int32_t nranks, int32_t rank, int64_t* begin, int64_t* end);

/* Verification: iterative refinement of the selected cameras' blocks
 * against the exact inverse of the bordered Fisher system
 * K = [[M, H], [H^T, 0]] (the FP64 D, A, couplings and H taken as exact data;
 * reference src/covariance.cpp:33-279, src/nullspace.cpp:14-62).  Runs the
 * product pipeline on the scene (its blocks for the selection -> base, may be
 * NULL), then `iters` steps of y += K~^-1 (e - K y) with double-double
 * residuals, K~^-1 being the FP64 solve through the pipeline's own factors.
 * refined / base: n_sel x P x P; history[k] = max over cameras of the
 * relative change of the block in step k (may be NULL).  Not on the product
 * path: the tests use it as the truth for the configs no CPU can invert. */
int32_t sfmcov_cuda_refine_covariance(sfmcov_handle* h, const sfmcov_scene* scene, const int32_t* cams,
                                      int32_t n_sel, int32_t iters, double* refined, double* base, double* history,
                                      sfmcov_error* err);

/* pseudoinverse_covariance (include/sfmcov/oracle.hpp:33-37, src/oracle.cpp:34-72):
 * the dense reference covariance for verification — Fisher matrix
 * (N = P n + 3 m params, refused above max_params with SFMCOV_ERR_SIZE_GUARD),
 * its eigendecomposition on the GPU (cuSOLVER syevd, loaded at run time; SVD
 * of a PSD matrix), the seven smallest dropped by count, Σ = V Λ^+ V^T.
 * cam_cov n x P x P; sigma_full N x N col-major (may be NULL); singular
 * values descending (N, may be NULL); gauge_gap = s[N-8] / s[N-7]. */
int32_t sfmcov_cuda_pseudoinverse_covariance(sfmcov_handle* h, const sfmcov_scene* scene, int64_t max_params,
                                             double* cam_cov, double* sigma_full, double* singular_values,
                                             double* gauge_gap, sfmcov_error* err);

/* Per-stage device times (ms) of the last pipeline call, in the order of
 * sfmcov_cuda_stage_name(i); returns the number of stages written. */
int32_t sfmcov_cuda_last_stage_times(sfmcov_handle* h, double* ms, int32_t capacity);
const char* sfmcov_cuda_stage_name(int32_t i);
/* Algorithmic counts of the last pipeline call (for roofline accounting):
 * [0] obs-pairs, [1] nonzero camera-pair blocks (incl. diagonal), [2] N = P*n,
 * [3] padded dense dim, [4] n_obs, [5] n_pts, [6] n_cams, [7] P,
 * [8] kernel launches of this library, [9] serial re-runs of the dense
 * stage after a pivot failure with overlapped streams. */
int32_t sfmcov_cuda_last_counts(sfmcov_handle* h, int64_t* counts, int32_t capacity);
/* Enable/disable per-stage event timing (off by default; adds syncs). */
void sfmcov_cuda_set_profiling(sfmcov_handle* h, int32_t on);

/* ---- sub-reconstructions (include/sfmcov/subrec.hpp, src/subrec.cpp) -----
 * Host planner with the reference's semantics and random draws, and the
 * batch of independent sub-scene covariances on the GPU (`workers` CUDA
 * handles of the handle's device in flight). */
/* build_view_graph: CSR over cameras (off n+1; neighbor / weight entries,
 * ascending neighbor); n_entries = 2 x #edges (written up to capacity). */
int32_t sfmcov_view_graph(const sfmcov_scene* scene, int32_t min_covis, int64_t* off, int32_t* nbr,
                          int32_t* weight, int64_t capacity, int64_t* n_entries, sfmcov_error* err);
/* The same graph on the device (the scene is validated first, as the
 * reference's planner entry points do): the co-visibility counts are the
 * camera-pair blocks' observation-pair counts of the covariance pipeline's
 * sorted pair list.  approximate_covariances / error_size_sweep use it. */
int32_t sfmcov_cuda_view_graph(sfmcov_handle* h, const sfmcov_scene* scene, int32_t min_covis, int64_t* off,
                               int32_t* nbr, int32_t* weight, int64_t capacity, int64_t* n_entries,
                               sfmcov_error* err);
/* extract_neighborhood: ascending global camera / point ids of the induced
 * sub-reconstruction (buffers of n_cams / n_pts capacity). */
int32_t sfmcov_extract_neighborhood(const sfmcov_scene* scene, int64_t center, int32_t k_bar, int32_t* cams,
                                    int64_t* n_cams, int32_t* pts, int64_t* n_pts, int32_t* truncated,
                                    sfmcov_error* err);
/* plan_coverage: subset s has cameras cams[subset_off[s] .. subset_off[s+1]). */
int32_t sfmcov_plan_coverage(const sfmcov_scene* scene, int32_t k_bar, uint64_t seed, int64_t* subset_off,
                             int64_t subset_capacity, int32_t* cams, int64_t cams_capacity, int64_t* n_subsets,
                             sfmcov_error* err);
/* approximate_covariances: per camera the kept block (n x P x P), its trace
 * and the producing subset id. */
int32_t sfmcov_cuda_approximate_covariances(sfmcov_handle* h, const sfmcov_scene* scene, int32_t k_bar,
                                            int32_t n_decompositions, uint64_t seed, int32_t workers,
                                            double* cam_cov, double* trace, int32_t* subset_id,
                                            sfmcov_error* err);
/* The same, one rank's share of a multi-GPU job ("trivial
 * multi-GPU job sharding"): every rank plans all coverings (deterministic),
 * computes only the subsets i of covering d with (i * n_decompositions + d)
 * mod nranks == rank, and returns its partial aggregate -- per camera the
 * smallest-trace block among its own subsets (trace +inf, subset -1 where
 * none).  Merging the ranks' partials by the smallest (trace, subset id)
 * gives exactly the single-call result.  On a failure failed_key receives
 * its place in the reference's order (src/subrec.cpp:202-222: covering d is
 * drawn, then its subsets computed, covering after covering):
 * d * 2^33 + (0 drawing | 1 computing) * 2^32 + the subset's index in d; -1
 * for a failure before any covering (validation, arguments, device).  The
 * merge reports the failure with the smallest key over all ranks, which is
 * the single call's error. */
int32_t sfmcov_cuda_approximate_covariances_shard(sfmcov_handle* h, const sfmcov_scene* scene, int32_t k_bar,
                                                  int32_t n_decompositions, uint64_t seed, int32_t workers,
                                                  int32_t nranks, int32_t rank, double* cam_cov, double* trace,
                                                  int32_t* subset_id, int64_t* failed_key, sfmcov_error* err);
/* monotonicity_check on the sub-reconstructions induced by two nested camera sets. */
int32_t sfmcov_cuda_monotonicity_check(sfmcov_handle* h, const sfmcov_scene* scene, const int32_t* small_cams,
                                       int64_t n_small, const int32_t* large_cams, int64_t n_large,
                                       double rel_tol, int32_t* violation_cams, double* trace_small,
                                       double* trace_large, int64_t* n_violations, int64_t* cameras_checked,
                                       sfmcov_error* err);

/* error_size_sweep: rows of (k_bar, subset_id, camera_id) in row_ints (3 per
 * row) and (err_relative, err_absolute, trace) in row_vals (3 per row). */
int32_t sfmcov_cuda_error_size_sweep(sfmcov_handle* h, const sfmcov_scene* scene, const int32_t* sizes,
                                     int32_t n_sizes, int32_t subsets_per_size, uint64_t seed, int32_t workers,
                                     int32_t* row_ints, double* row_vals, int64_t capacity, int64_t* n_rows,
                                     sfmcov_error* err);

/* ---- synthetic scenes (host only; harness, not the hot path) ------------
 * generate_cube_scene / generate_random_scene / transform_scene
 * (include/sfmcov/synthetic.hpp:17-28, src/synthetic.cpp:52-194) and the
 * BASELINE.json configs 1..5. */
typedef struct sfmcov_synth_scene sfmcov_synth_scene;
sfmcov_synth_scene* sfmcov_synth_cube(uint64_t seed, double noise_px, int32_t cam_params);
sfmcov_synth_scene* sfmcov_synth_random(int64_t n_cams, int64_t n_pts, double visibility,
                                        uint64_t seed, double noise_px, int32_t cam_params);
sfmcov_synth_scene* sfmcov_synth_config(int32_t config_index, uint64_t seed);
sfmcov_synth_scene* sfmcov_synth_transform(const sfmcov_synth_scene* in, const double* R3x3,
                                           const double* t3, double scale);
void sfmcov_synth_sizes(const sfmcov_synth_scene* s, int64_t* n, int64_t* m, int64_t* t, int32_t* P);
void sfmcov_synth_export(const sfmcov_synth_scene* s, double* cams, double* pts, int32_t* obs_cam,
                         int32_t* obs_pt, double* obs_u, double* obs_sigma);
void sfmcov_synth_free(sfmcov_synth_scene* s);
const char* sfmcov_synth_last_error(void);

/* ---- scene IO (include/sfmcov/scene_io.hpp, src/scene_io.cpp; host) --------
 * JSON in the reference's schema (sorted keys, compact, shortest round-trip
 * numbers, sigma omitted when identity; "k2" for P = 9 cameras) and a binary
 * format for large scenes.  Loaders return an owned scene (read it with
 * sfmcov_synth_sizes / _export, free with sfmcov_synth_free) or NULL with err
 * set (kinds io / parse, stage "load"; the reference's context strings).  The
 * scene invariants are checked by the CUDA library (the wrappers validate
 * after loading, as the reference's load ends with validate()). */
sfmcov_synth_scene* sfmcov_scene_load(const char* path, sfmcov_error* err);
int32_t sfmcov_scene_save(const sfmcov_scene* scene, const char* path, sfmcov_error* err);
sfmcov_synth_scene* sfmcov_scene_load_binary(const char* path, sfmcov_error* err);
int32_t sfmcov_scene_save_binary(const sfmcov_scene* scene, const char* path, sfmcov_error* err);

/* ---- covariance IO (include/sfmcov/covariance_io.hpp, src/covariance_io.cpp) --
 * Host only (libsfmcov_synth.so).  Blocks are P x P row-major, P in {8, 9}. */
/* pack_upper_triangle / unpack_upper_triangle (covariance_io.hpp:12-13): the
 * row-major upper triangle (0,0),(0,1),...,(P-1,P-1), P(P+1)/2 entries. */
void sfmcov_covio_pack_upper_triangle(const double* block, int32_t P, double* tri);
void sfmcov_covio_unpack_upper_triangle(const double* tri, int32_t P, double* block);
/* save_covariance_json (covariance_io.cpp:52-66): {"cameras":[{"cov":[...],
 * "id":i}...],"diagnostics":{...}} exactly as the reference's nlohmann dump
 * (sorted keys, compact, shortest round-trip doubles).  diag may be NULL
 * (zeros); its flagged buffer holds the flagged columns. */
int32_t sfmcov_covio_save_json(const char* path, int64_t n_cams, int32_t P, const double* cam_cov,
                               const sfmcov_diagnostics* diag, sfmcov_error* err);
/* load_covariance_json (covariance_io.cpp:68-101): fills up to `capacity`
 * blocks, *n_cams = the file's camera count (call again with a larger buffer
 * when it exceeds capacity); diag (may be NULL) gets the diagnostics and up to
 * flagged_capacity flagged columns (n_flagged = total).  Errors: io
 * (unreadable), parse ("invalid JSON" / "bad covariance file"). */
int32_t sfmcov_covio_load_json(const char* path, int32_t P, int64_t capacity, double* cam_cov, int64_t* n_cams,
                               sfmcov_diagnostics* diag, sfmcov_error* err);
/* save_covariance_csv (covariance_io.cpp:103-122): header id,cov_0_0,...,
 * one row per camera, %.17g. */
int32_t sfmcov_covio_save_csv(const char* path, int64_t n_cams, int32_t P, const double* cam_cov,
                              sfmcov_error* err);

#ifdef __cplusplus
}
#endif

#endif /* SFMCOV_B200_H */
