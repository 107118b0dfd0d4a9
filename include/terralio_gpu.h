/*
 * terralio_gpu.h — C-ABI of the B200-native RBF terrain hot path.
 *
 * This is the drop-in boundary between the reference's C++ class API
 * (terralio::terrain::TerrainModel & friends, /root/reference/proj/core) and
 * the sm_100a kernels in paper_2509_26222_b200/csrc. Plain C: opaque
 * handles, plain pointers + sizes, int status codes; no CUDA, torch or Eigen
 * types. A C++ shim (include/terralio_b200/terrain.hpp) and a ctypes binding
 * (paper_2509_26222_b200/_abi.py) rebuild the reference interface on top of
 * it; INTEGRATION.md shows the binding a proj/core maintainer adds.
 *
 * Conventions
 *  - Arrays are SoA `double*` (x[], y[], z[] …). Each data entry point takes
 *    a tlg_mem tag saying whether its pointers are host or device memory;
 *    host buffers are staged through pinned memory inside the call.
 *  - Status codes map 1:1 onto the reference's exceptions (see tlg_status);
 *    tlg_last_error() returns the thread's last message.
 *  - All device work is enqueued on the context's CUDA stream. Entry points
 *    that return host-visible results synchronise that stream.
 *  - There is no CPU fallback: every numeric result comes from a kernel;
 *    calls fail with TLG_CUDA_ERROR when no sm_100 device is present.
 *  - Jacobian rows use Eigen's column-major rows x 6 layout
 *    (CostEval::jacobian, scan_matcher.hpp:75): J[c * n + i].
 */
#ifndef TERRALIO_GPU_H_
#define TERRALIO_GPU_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TLG_ABI_VERSION 1

typedef enum tlg_status {
  TLG_OK = 0,
  TLG_INVALID_ARGUMENT = 1,     /* std::invalid_argument (kernel.cpp:18-24, center_select.cpp:10-15,22-24) */
  TLG_DOMAIN_ERROR = 2,         /* std::domain_error (kernel.cpp:29-31, terrain_model.cpp:98) */
  TLG_NO_SUPPORTED_CENTERS = 3, /* terrain::NoSupportedCenters (center_select.hpp:30-32) */
  TLG_RUNTIME_ERROR = 4,        /* std::runtime_error (terrain_model.cpp:289-295, snapshot.cpp) */
  TLG_CUDA_ERROR = 5,
  TLG_OUT_OF_MEMORY = 6,
  TLG_BUFFER_TOO_SMALL = 7
} tlg_status;

typedef enum tlg_mem { TLG_HOST = 0, TLG_DEVICE = 1 } tlg_mem;

/* terrain::KernelParams (kernel.hpp:12-24). */
typedef struct tlg_kernel_params {
  double sigma;         /* default 0.04 */
  double sigma_eps;     /* default 0.1  */
  double lambda;        /* default 1e-3 */
  double cutoff_radius; /* 0 = auto: max(cfg, 3 sigma_tilde) after finalize */
} tlg_kernel_params;

/* terrain::CenterSet minus the centre list (center_select.hpp:22-28). */
typedef struct tlg_center_params {
  double mesh_resolution;
  double accept_radius;
  int32_t accept_count;
  int32_t reserved;
  double roi_min_x, roi_min_y, roi_max_x, roi_max_y;
} tlg_center_params;

/* terrain::UpdateReport (terrain_model.hpp:21-26) + which solver ran. */
typedef struct tlg_update_report {
  uint64_t active_blocks;
  uint64_t active_centers;
  uint64_t born_centers;
  int32_t rejected;     /* inner solve failed; births persist, weights/blocks unchanged */
  int32_t solver;       /* 1 = one-shot Woodbury (m x m), 2 = information form (n x n) */
  double flops;         /* FP64 flops of the formulation run (DESIGN.md §4 F_W / F_I) */
} tlg_update_report;

/* Normal-equation block of the stacked manifold rows
 * (scan_matcher.cpp:296-299 A = J^T J, g = J^T r; :253 cost = |r|^2). */
typedef struct tlg_normal_eq {
  double A[21];   /* upper triangle of J^T J, row-major (i <= j) */
  double g[6];    /* J^T r */
  double cost;    /* sum r^2 */
  double valid;   /* number of supported (valid) rows */
} tlg_normal_eq;

typedef struct tlg_ctx tlg_ctx;
typedef struct tlg_model tlg_model;

/* ---- library / context ---------------------------------------------------- */
int tlg_abi_version(void);
const char* tlg_last_error(void);
/* device = CUDA ordinal; stream = the cudaStream_t every call of this context
 * is ordered on (NULL = the legacy default stream). Device inputs must be
 * ready on that stream; results are ready on it when a call returns with
 * host outputs, and ordered on it otherwise. */
tlg_status tlg_ctx_create(int device, void* stream, tlg_ctx** out);
tlg_status tlg_ctx_destroy(tlg_ctx* ctx);
tlg_status tlg_ctx_set_stream(tlg_ctx* ctx, void* stream);
tlg_status tlg_ctx_synchronize(tlg_ctx* ctx);
/* Number of kernels this context has launched (bench launch accounting). */
uint64_t tlg_ctx_launch_count(const tlg_ctx* ctx);
/* Per-kernel CUDA-event timing of the hot kernels (off by default).
 * kernel: 0 = manifold rows (K4), 1 = height/gradient eval (K3). */
tlg_status tlg_ctx_set_profiling(tlg_ctx* ctx, int enable);
tlg_status tlg_ctx_kernel_stats(tlg_ctx* ctx, int kernel, double* total_ms, uint64_t* launches);

/* ---- Batch-predict consumers ------------------------------ */
/* select_ground_points (pipeline.cpp:150-170): points p (sensor frame, SoA)
 * with FeatureKind codes kind (2 = Ground), pose R (row-major) / t; keeps, in
 * scan order, ground points whose world xy lies in [roi_min, roi_max], within
 * ground_radius of t_xy, first in their xy voxel (ground_voxel); at most
 * max_points. out_x/out_y/out_z need max_points capacity; *out_n = kept. */
tlg_status tlg_select_ground_points(tlg_ctx* ctx, const double* px, const double* py,
                                    const double* pz, const uint8_t* kind, size_t n,
                                    tlg_mem in_mem, const double R[9], const double t[3],
                                    const double roi_min[2], const double roi_max[2],
                                    double ground_radius, double ground_voxel,
                                    size_t max_points, double* out_x, double* out_y,
                                    double* out_z, tlg_mem out_mem, size_t* out_n);
/* terrain_error_histogram (metrics.cpp:199-232): errors |z - f(x, y)| (0.25 m
 * where unsupported), top floor(trim_fraction n) dropped, bins over
 * [0, 0.25]: edges[bins + 1], counts[bins], trimmed, overflow (host). */
tlg_status tlg_terrain_error_histogram(tlg_model* model, const double* x, const double* y,
                                       const double* z, size_t n, tlg_mem mem,
                                       double trim_fraction, int bins, double* edges,
                                       uint64_t* counts, uint64_t* trimmed, uint64_t* overflow);

/* ---- Feature correspondences -------------------------------- */
/* LocalMap (local_map.hpp:17-50): sliding window of frames, per-kind kNN
 * structures; build_correspondences (scan_matcher.cpp:44-183); feature rows
 * of total_cost (:185-216). FeatureKind codes: 0 edge, 1 planar, 2 ground. */
/* LM damped step (scan_matcher.cpp:300-305): delta = -(A + mu diag(A)^+ +
 * 1e-3 I)^-1 g by a pivoted LDL^T; ne may be the sum of the feature and
 * manifold normal equations. TLG_RUNTIME_ERROR when the step is not finite. */
tlg_status tlg_lm_step(tlg_ctx* ctx, const tlg_normal_eq* ne, double mu, double delta[6]);
/* Smallest eigenvalue of A (the degeneracy probe of lm_solve on the
 * feature-only normal matrix, scan_matcher.cpp:280-287). */
tlg_status tlg_ne_min_eigenvalue(tlg_ctx* ctx, const tlg_normal_eq* ne, double* lambda_min);
typedef struct tlg_map tlg_map;
typedef struct {
  double corr_gate, huber_delta, plane_fit_tol, plane_eig_ratio, edge_eig_ratio, edge_fit_tol,
      edge_min_extent, trim_ratio, trim_floor, ground_corr_voxel, ground_corr_radius;
} tlg_match_config; /* SolverConfig fields used by the association (scan_matcher.hpp:15-49) */
tlg_status tlg_match_config_default(tlg_match_config* cfg);
tlg_status tlg_map_create(tlg_ctx* ctx, double voxel_size, size_t window, tlg_map** out);
tlg_status tlg_map_destroy(tlg_map* map);
/* LocalMap::insert (local_map.cpp:19-45): sensor-frame points, kinds, labels
 * (NULL = -1), pose R (row-major) / t. */
tlg_status tlg_map_insert(tlg_map* map, const double* px, const double* py, const double* pz,
                          const uint8_t* kind, const int32_t* label, size_t n, tlg_mem mem,
                          const double R[9], const double t[3]);
/* Map points of one kind (0 edge, 1 planar) in map-id order: xyz (3 per
 * point) and labels on the host, up to cap; *count = total. */
tlg_status tlg_map_points(tlg_map* map, int kind, double* xyz, int32_t* labels, size_t cap,
                          size_t* count);
/* build_correspondences: the result stays in the map object (feature order
 * after the trims); *count = correspondences. */
tlg_status tlg_build_correspondences(tlg_map* map, const double* px, const double* py,
                                     const double* pz, const uint8_t* kind, size_t n,
                                     tlg_mem mem, const double R[9], const double t[3],
                                     const tlg_match_config* cfg, size_t* count);
/* The last correspondences on the host (any pointer may be NULL): kind (0
 * edge, 1 plane), feature index, params[7] (edge: point xyz, direction xyz;
 * plane: normal xyz, offset), weight, majority label, distance, plane fit
 * quality (smallest eigenvalue; 0 for edges). */
tlg_status tlg_correspondences_get(tlg_map* map, int32_t* kind, uint32_t* feature,
                                   double* params, double* weight, int32_t* label, double* dist,
                                   double* fitq, size_t cap);
/* total_cost's feature rows (scan_matcher.cpp:196-214) for n HOST
 * correspondences at pose (R, t): kind (0 edge -> 3 rows, 1 plane -> 1
 * row), p_sensor (3 per corr.), params (7 per corr., as
 * tlg_correspondences_get), weight. Host outputs r[rows] and J (column-major
 * rows x 6, ld = rows); *rows always set, TLG_BUFFER_TOO_SMALL when it
 * exceeds cap_rows. */
tlg_status tlg_feature_rows(tlg_ctx* ctx, const int32_t* kind, const double* p_sensor,
                            const double* params, const double* weight, size_t n,
                            const double R[9], const double t[3], double* r, double* J,
                            size_t cap_rows, size_t* rows);
/* Feature rows of total_cost at pose (R, t) for the last correspondences,
 * reduced to the normal equations (valid = rows). */
tlg_status tlg_feature_normal_eq(tlg_map* map, const double R[9], const double t[3],
                                 tlg_normal_eq* ne);

/* ---- kernel.cpp ------------------------------------------------------------- */
/* KernelParams::finalize (kernel.cpp:15-25): fills the auto cutoff, validates. */
tlg_status tlg_kernel_finalize(tlg_kernel_params* p);
/* kernel_eval (kernel.cpp:27-35) over n (x, c) pairs on the device:
 * out[i] = exp(-|x_i - c_i|^2 / (2 b^2)), exactly 0 when |x_i - c_i|^2 >
 * cutoff^2 (finalized params). TLG_DOMAIN_ERROR for a non-finite input or
 * bandwidth <= 0, before anything is written (the reference throws
 * std::domain_error). */
tlg_status tlg_kernel_eval(tlg_ctx* ctx, const tlg_kernel_params* p, const double* x,
                           const double* y, const double* cx, const double* cy, size_t n,
                           tlg_mem in_mem, double bandwidth, double* out, tlg_mem out_mem);

/* ---- center_select.cpp ------------------------------------------------------ */
/* supported_mesh_nodes (center_select.cpp:18-62): lattice nodes of `roi`
 * (i outer, j inner) with >= accept_count observation points within
 * accept_radius. Bit-exact node coordinates and order. z is only validated
 * (TerrainObservation::validate, :9-16). out_* in out_mem; *out_n always set;
 * TLG_BUFFER_TOO_SMALL when *out_n > cap. */
tlg_status tlg_supported_mesh_nodes(tlg_ctx* ctx, const double* x, const double* y,
                                    const double* z, size_t m, size_t z_len, tlg_mem in_mem,
                                    const tlg_center_params* params, double* out_x,
                                    double* out_y, size_t cap, size_t* out_n,
                                    tlg_mem out_mem);
/* select_centers (center_select.cpp:64-76): as above, TLG_NO_SUPPORTED_CENTERS
 * when empty. */
tlg_status tlg_select_centers(tlg_ctx* ctx, const double* x, const double* y, const double* z,
                              size_t m, size_t z_len, tlg_mem in_mem,
                              const tlg_center_params* params, double* out_x, double* out_y,
                              size_t cap, size_t* out_n, tlg_mem out_mem);

/* ---- TerrainModel ------------------------------------------------------------ */
/* TerrainModel(kernel, centers) (terrain_model.cpp:26-44). */
tlg_status tlg_model_create(tlg_ctx* ctx, const tlg_kernel_params* kernel,
                            const tlg_center_params* centers, const double* cx,
                            const double* cy, size_t n, tlg_mem mem, tlg_model** out);
tlg_status tlg_model_destroy(tlg_model* model);
tlg_status tlg_model_counts(const tlg_model* model, size_t* num_centers, size_t* num_blocks);
/* Diagnostics: which evaluation sweep the model's centres select — 0 generic
 * hash-grid sweep, 4..14 lattice window with runtime pair classes, 100 + g
 * compiled geometry g, 200 + g the same with boundary pairs summed without
 * the cutoff test (see below) — and whether the separable exp recurrence is
 * used. */
tlg_status tlg_model_sweep(tlg_model* model, int* kind, int* exp_recurrence);
/* kernel_eval returns exactly 0 beyond the cutoff (kernel.cpp:27-35). By
 * default height/gradient/manifold evaluation skips that test on window
 * boundary pairs when the kernel value at the cutoff makes every such pair's
 * contribution provably below 1e-11 x the window's largest |w| (paper
 * defaults: kappa_sigma(rho) = 6.8e-15); exact != 0 forces the per-pair
 * test. Neighbour ids (tlg_centers_near, tlg_moment_features) are always
 * exact. */
tlg_status tlg_model_set_exact_cutoff(tlg_model* model, int exact);
tlg_status tlg_model_kernel(const tlg_model* model, tlg_kernel_params* out);
tlg_status tlg_model_center_params(const tlg_model* model, tlg_center_params* out);
tlg_status tlg_model_get_centers(tlg_model* model, double* cx, double* cy, tlg_mem mem);
tlg_status tlg_model_get_weights(tlg_model* model, double* w, tlg_mem mem);
tlg_status tlg_model_set_weights(tlg_model* model, const double* w, tlg_mem mem);
tlg_status tlg_model_get_block_index(tlg_model* model, uint32_t* out, tlg_mem mem);
tlg_status tlg_model_block_size(const tlg_model* model, uint32_t block, size_t* n);
tlg_status tlg_model_get_block_members(const tlg_model* model, uint32_t block, uint32_t* out);
/* block_info_inverse(b): bn x bn column-major. */
tlg_status tlg_model_get_block_info_inverse(tlg_model* model, uint32_t block, double* out,
                                            tlg_mem mem);
tlg_status tlg_model_set_block_info_inverse(tlg_model* model, uint32_t block,
                                            const double* in, tlg_mem mem);

/* predict_height / predict_gradient (terrain_model.cpp:109-143), batched:
 * z[i] (0 when unsupported), supported[i] (1/0), grad_x/grad_y[i]. Any output
 * may be NULL. Non-finite queries: TLG_DOMAIN_ERROR (kernel.cpp:29-31). */
tlg_status tlg_eval(tlg_model* model, const double* x, const double* y, size_t n,
                    tlg_mem in_mem, double* z, uint8_t* supported, double* grad_x,
                    double* grad_y, tlg_mem out_mem);

/* moment_feature (terrain_model.cpp:97-107), batched as CSR over queries:
 * row_ptr[n+1], ids ascending per row, vals = s * kappa_sigma_tilde. */
tlg_status tlg_moment_features(tlg_model* model, const double* x, const double* y, size_t n,
                               tlg_mem in_mem, uint32_t* row_ptr, uint32_t* ids, double* vals,
                               size_t cap, size_t* nnz, tlg_mem out_mem);

/* Manifold soft-constraint rows, batched generalisation of
 * kin::manifold_residual/jacobian (contact.cpp:7-39) with the total_cost
 * weighting (scan_matcher.cpp:221-248): for lever arm h_i,
 *   xi = R h_i + t,  raw_i = xi_z - wheel_radius - f(xi_xy),
 *   J_i = [-df/dx, -df/dy, 1] [-R hat(h_i), I3],
 *   w_i = sqrt(huber/|raw|) if huber > 0 and |raw| > huber else 1,
 *   r_i = sqrt(lambda_M) w_i raw_i,  J row scaled alike; unsupported -> zero row.
 * R row-major 3x3 and t[3] are host arrays. Outputs r, J (J[c*n+i]), valid,
 * raw may be NULL; `ne` (host, may be NULL) receives the fused reduction. */
tlg_status tlg_manifold_rows(tlg_model* model, const double R[9], const double t[3],
                             const double* hx, const double* hy, const double* hz, size_t n,
                             tlg_mem in_mem, double wheel_radius, double lambda_M,
                             double huber_delta, double* r, double* J, uint8_t* valid,
                             double* raw, tlg_mem out_mem, tlg_normal_eq* ne);

/* ---- scans: lever arms binned once per scan ------------------------------
 * lm_solve evaluates the same scan's rows every LM iteration
 * (scan_matcher.cpp:276,315). tlg_scan_create copies the lever arms to the
 * device binned by the world cell of R0 h + t0, so later evaluations read
 * the weight grid warp-coherently. tlg_scan_manifold_rows is
 * tlg_manifold_rows over the scan; its rows come out in scan order: row k
 * belongs to input point perm[k] (tlg_scan_permutation). Results do not
 * depend on R0 (it only sets memory order). */
typedef struct tlg_scan tlg_scan;
tlg_status tlg_scan_create(tlg_model* model, const double R0[9], const double t0[3],
                           const double* hx, const double* hy, const double* hz, size_t n,
                           tlg_mem in_mem, tlg_scan** out);
tlg_status tlg_scan_destroy(tlg_scan* scan);
tlg_status tlg_scan_info(const tlg_scan* scan, size_t* n, double* bin_ms);
tlg_status tlg_scan_permutation(tlg_scan* scan, uint32_t* perm, tlg_mem out_mem);
tlg_status tlg_scan_manifold_rows(tlg_model* model, tlg_scan* scan, const double R[9],
                                  const double t[3], double wheel_radius, double lambda_M,
                                  double huber_delta, double* r, double* J, uint8_t* valid,
                                  double* raw, tlg_mem out_mem, tlg_normal_eq* ne);

/* recursive_update(obs, allow_birth) (terrain_model.cpp:145-253). */
tlg_status tlg_recursive_update(tlg_model* model, const double* x, const double* y,
                                const double* z, size_t m, size_t z_len, tlg_mem in_mem,
                                int allow_birth, tlg_update_report* report);

/* fit_batch_ridge (terrain_model.cpp:269-308). */
tlg_status tlg_fit_batch_ridge(tlg_ctx* ctx, const tlg_kernel_params* kernel,
                               const tlg_center_params* centers, const double* cx,
                               const double* cy, size_t n, const double* x, const double* y,
                               const double* z, size_t m, size_t z_len, tlg_mem mem,
                               tlg_model** out);

/* Point-sharded fit_batch_ridge (the reference's single-process
 * terrain_model.cpp:269-308 split at its one reduction): every rank creates
 * the model from the same centres (tlg_model_create), asks for the system
 * dimensions, assembles the partial system over its point shard into DEVICE
 * buffers H (elems doubles, lower band storage: element (i, j), 0 <= i - j,
 * at H[i + j * ld]) and b (n), the caller sums H and b over ranks (NCCL
 * all-reduce), and every rank solves: weights and info_inv blocks as
 * tlg_fit_batch_ridge computes them (within the stated tolerance; the
 * cross-rank summation order differs). add_lambda != 0 on exactly one rank.
 * An empty shard (m = 0) contributes zeros. */
tlg_status tlg_batch_ridge_system(tlg_model* model, size_t* n, size_t* ld, size_t* elems);
tlg_status tlg_batch_ridge_assemble(tlg_model* model, const double* x, const double* y,
                                    const double* z, size_t m, tlg_mem mem, double* H, size_t ld,
                                    double* b, int add_lambda);
tlg_status tlg_batch_ridge_solve(tlg_model* model, double* H, size_t ld, double* b);
/* Structural sparsity of that system, for the cross-rank reduction of the
 * partial systems: entry (i, j) can be nonzero only for centres within two
 * cutoffs (and the diagonal). *nnz = packed length (deterministic order, the
 * same on every rank for the same centres); pack gathers those entries of a
 * DEVICE H into a DEVICE packed[nnz]; unpack zeroes H and scatters them back.
 * Reducing packed instead of H moves ~nnz doubles instead of elems. */
tlg_status tlg_batch_ridge_pattern(tlg_model* model, size_t* nnz);
tlg_status tlg_batch_ridge_pack(tlg_model* model, const double* H, double* packed);
tlg_status tlg_batch_ridge_unpack(tlg_model* model, const double* packed, double* H);

/* Communicator for the sharded variants (SURVEY §8b tlg_comm_init): an NCCL
 * communicator over the ranks of one job (one process per GPU), created from
 * a TLG_COMM_ID_BYTES unique id that rank 0 makes (tlg_comm_unique_id) and
 * broadcasts out of band. NCCL is loaded at tlg_comm_unique_id / init time
 * (libnccl.so.2; TLG_RUNTIME_ERROR when absent). */
#define TLG_COMM_ID_BYTES 128
typedef struct tlg_comm tlg_comm;
tlg_status tlg_comm_unique_id(void* id);
tlg_status tlg_comm_init(tlg_ctx* ctx, const void* id, int rank, int size, tlg_comm** out);
tlg_status tlg_comm_destroy(tlg_comm* comm);
/* In-place SUM of the 29-double normal-equation block over the ranks: the one
 * exchange of a point-sharded LM cost evaluation (scan_matcher.cpp:296-299). */
tlg_status tlg_comm_allreduce_normal_eq(tlg_comm* comm, tlg_normal_eq* ne);
/* fit_batch_ridge over point shards in one call: assemble this rank's shard
 * (lambda I on rank 0), all-reduce the packed structural nonzeros and the
 * rhs, solve on every rank (every rank ends with the same model). */
tlg_status tlg_fit_batch_ridge_sharded(tlg_model* model, tlg_comm* comm, const double* x,
                                       const double* y, const double* z, size_t m, tlg_mem mem);

/* RBFT v1 snapshot (snapshot.cpp:7-126), byte-identical layout. */
tlg_status tlg_model_save(tlg_model* model, const char* path);
tlg_status tlg_model_load(tlg_ctx* ctx, const char* path, tlg_model** out);

#ifdef __cplusplus
}
#endif
#endif /* TERRALIO_GPU_H_ */
