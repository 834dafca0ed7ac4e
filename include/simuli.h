/*
 * simuli.h -- C ABI of the B200-native SimULi forward sensor-rendering hot path
 * (arXiv 2510.12901).  libsimuli.so implements it with hand-written CUDA for sm_100a.
 *
 * Citations: "P:n" = /root/reference/PAPER.md line n (section in brackets); readings of
 * silent or garbled passages are DESIGN.md §3 ledger items "A<n>".
 *
 * The five calls, in path order:
 *   simuli_build_tiles    Proc. ElevationTiling + ray table + culling SAT   [P:141-147, P:494-538]
 *   simuli_project        7-sigma-point UT projection, ray-based culling,  [P:129, P:134-147,
 *                         tile counts, depth keys, compositing records      P:544-562]
 *   simuli_bin_sort       duplication into (tile|depth) keys + radix sort  [P:129 "as in 3DGS",
 *                         + tile ranges                                     P:607 "Sort"]
 *   simuli_render_lidar   per-ray front-to-back compositing, LiDAR decode  [P:114-129, Eq. 1]
 *   simuli_render_camera  same for distorted rolling-shutter cameras       [P:112-129]
 *
 * ---- conventions (all calls) ----
 * Status: every call returns int32: SIMULI_OK (0) or an error code below; the message of
 *   the last error on the calling thread is simuli_last_error().  No exceptions cross the
 *   ABI.  No global mutable state besides that thread-local message; calls on distinct
 *   buffers / streams are thread-safe.
 * Ownership: the library never allocates or frees memory.  Every buffer is caller-owned:
 *   "host" pointers are ordinary CPU memory read/written during the call only; "device"
 *   pointers are CUDA global memory (e.g. torch tensors) that must stay alive until the
 *   enqueued work on `stream` has completed.  Scratch is the caller's `workspace`.
 * Asynchrony: device work is enqueued on the caller's cudaStream_t (passed as void*, NULL =
 *   legacy default stream); no call synchronises, except simuli_bin_sort with
 *   pair_capacity < 0 (documented there).  The forward kernels are launched with
 *   programmatic dependent launch (a kernel's CTAs may be scheduled while the previous
 *   kernel on the stream finishes; each waits for that kernel's completion before reading
 *   anything), so stream-order semantics are exactly those of plain launches
 *   (SIMULI_PDL=0 in the environment disables it).
 * Degenerate particles are not errors: zero / non-finite quaternion or scale, a sigma
 *   point closer than the minimum range / near plane, or a singular projected covariance
 *   make a particle "invalid": tile count 0, never rendered (A20).
 * Layouts: contiguous float32, row-major.  Quaternions are (w, x, y, z) and need not be
 *   unit (normalised inside).  Scales are post-activation standard deviations (m, > 0);
 *   opacity is post-sigmoid (A26).  SH coefficients are [n][(deg+1)^2][3]
 *   (coefficient-major, channel-minor), degree <= 3 (48 values at degree 3).
 *   Poses map sensor -> world.  LiDAR sensor frame: x forward, y left, z up (Eq. 3);
 *   camera frame: OpenCV (x right, y down, z forward) (A6).
 */
#ifndef SIMULI_H
#define SIMULI_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SIMULI_ABI_VERSION 12

enum {
  SIMULI_OK = 0,
  SIMULI_ERR_INVALID_ARGUMENT = 1, /* bad pointer / size / parameter                         */
  SIMULI_ERR_CAPACITY = 2,         /* a caller buffer is too small; *_required is filled    */
  SIMULI_ERR_CUDA = 3,             /* a CUDA launch / API call failed (message has the text) */
  SIMULI_ERR_UNSUPPORTED = 4       /* option not implemented (e.g. SH degree > 3)            */
};

enum { SIMULI_SENSOR_LIDAR = 0, SIMULI_SENSOR_CAMERA = 1 };
enum { SIMULI_CAM_PINHOLE_RADTAN = 0, SIMULI_CAM_FISHEYE_KB = 1 };

/* Thread-local text of the last error ("" if none).  Valid until the next call. */
const char* simuli_last_error(void);
int32_t simuli_abi_version(void);

/* Rigid pose, sensor -> world: x_world = R(q) x_sensor + t. */
typedef struct {
  float q[4]; /* w, x, y, z */
  float t[3];
} simuli_pose;

/* Spinning LiDAR (Fig. 3a; A5): every beam fires once per azimuth column;
 * column j (0 <= j < n_azimuth) fires at normalised time s_j = (j + 0.5)/n_azimuth of the
 * sweep, azimuth phi_j = wrap(azimuth_start + spin_direction (j + 0.5) 2 pi / n_azimuth).
 * Ray id = beam * n_azimuth + column (range-image layout). */
typedef struct {
  int32_t n_beams;
  const float* beam_elevation_rad; /* host [n_beams], any order, |omega| < pi/2         */
  int32_t n_azimuth;               /* columns per revolution (A)                          */
  float azimuth_start_rad;         /* phi_start in [-pi, pi)                              */
  int32_t spin_direction;          /* +1: azimuth increases with time, -1: decreases      */
  float min_range_m;               /* minimum range r_min (> 0)                           */
  float beam_divergence_rad;       /* theta_div >= 0 (App. C): every particle's
                                      covariance becomes Sigma_hat = Sigma + (theta r)^2
                                      (I - d d^T), d / r the direction / range from the sensor
                                      position at the mean's firing time (A27), used for the
                                      projection (sigma points from chol(Sigma_hat)) and the
                                      response, WITHOUT opacity compensation; 0 = off (the
                                      bitwise default path)                                 */
} simuli_lidar;

/* Tiling parameters: n_phi elevation tiles N_phi, M = max rays per tile,
 * r = 400 histogram bins, dense culling grid 1600 azimuth cells x 8 rows per elevation
 * tile (r^d_phi = 1600, r^d_omega = 8; A7, A10). */
typedef struct {
  int32_t n_phi;
  int32_t max_rays_per_tile;
  int32_t hist_bins;
  int32_t cull_az_cells;
  int32_t cull_rows_per_tile;
} simuli_tiling_params;

/* Output of simuli_build_tiles.  Host memory.  Call once with every array pointer NULL to
 * get the sizes, allocate, call again to fill (the sizing fields are rewritten). */
typedef struct {
  /* sizes / scalars (always written) */
  int32_t n_phi;            /* effective elevation tiles N_phi' <= requested n_phi         */
  int32_t n_theta;          /* azimuth tiles N_theta = clamp(ceil(H_max / M), 1, A)        */
  int32_t n_tiles;          /* n_phi * n_theta; tile id = elev_tile * n_theta + az_tile   */
  int32_t max_rays_in_tile; /* may exceed M when beams per tile do not divide M (A9)      */
  int32_t sat_rows, sat_cols; /* (8 n_phi + 1) x (1600 + 1)                              */
  int32_t n_rays, n_beams, n_azimuth;
  int32_t max_beams_per_elev_tile, max_cols_per_az_tile;
  float pi_f, two_pi_f;     /* (float)pi, (float)(2 pi)                                    */
  float az_tile_scale;      /* (float)(n_theta / 2pi)                                      */
  float az_cell_scale;      /* (float)(cull_az_cells / 2pi)                                */
  /* arrays (host, caller-allocated; NULL on the sizing call) */
  float* elev_bounds;       /* [n_phi+1] float32 boundaries T, strictly increasing         */
  float* cull_row_scale;    /* [n_phi] (float)(rows_per_tile / (T[k+1] - T[k]))             */
  float* ray_az;            /* [n_rays] phi_j                                              */
  float* ray_el;            /* [n_rays] omega_b                                            */
  float* ray_s;             /* [n_rays] firing time s_j in [0, 1)                          */
  int32_t* ray_tile;        /* [n_rays] render tile of each ray                             */
  int32_t* tile_ray_offsets;/* [n_tiles+1] CSR tile -> rays                                 */
  int32_t* tile_rays;       /* [n_rays] ray ids per tile, increasing                       */
  int32_t* sat;             /* [sat_rows*sat_cols] summed-area table of the dense ray mask */
  int32_t* elev_tile_beam_offsets; /* [n_phi+1] CSR elevation tile -> beams                */
  int32_t* elev_tile_beams;        /* [n_beams]                                             */
  int32_t* az_tile_col_offsets;    /* [n_theta+1] CSR azimuth tile -> columns               */
  int32_t* az_tile_cols;           /* [n_azimuth]                                           */
  float* beam_el_sorted;           /* [n_beams] beam elevations, ascending (exact culling)  */
  float* col_az_sorted;            /* [n_azimuth] column azimuths phi_j, ascending (ditto)  */
} simuli_tiling;

/* Proc. ElevationTiling with the corrections of A8: histogram of per-ray
 * elevations with r bins, one boundary per integer crossing of the normalised CDF
 * (integer-exact test), boundaries at the float32 midpoint of the beam gap, empty tiles
 * dropped, N_theta = ceil(H_max / M).  Also the ray table, tile -> ray CSR, dense ray
 * mask and its zero-padded summed-area table.  Host only, once per
 * sensor definition; the result is bit-exact and deterministic.
 * Errors: INVALID_ARGUMENT for n_beams/n_azimuth/n_phi/M/bins/cells < 1, n_phi > hist_bins
 * ("tile count exceeds histogram resolution"), |elevation| >= pi/2, |spin_direction| != 1.
 * All elevations identical -> a single elevation tile (not an error). */
int32_t simuli_build_tiles(const simuli_lidar* lidar, const simuli_tiling_params* params,
                           simuli_tiling* inout);

/* Device copy of a simuli_tiling (the caller uploads the arrays; the struct itself is
 * host memory holding device pointers). */
typedef struct {
  int32_t n_phi, n_theta, n_tiles, max_rays_in_tile, sat_rows, sat_cols;
  int32_t cull_az_cells, cull_rows_per_tile, n_rays, n_beams, n_azimuth;
  int32_t max_beams_per_elev_tile, max_cols_per_az_tile;
  float pi_f, two_pi_f, az_tile_scale, az_cell_scale;
  const float *elev_bounds, *cull_row_scale, *ray_az, *ray_el, *ray_s;
  const int32_t *ray_tile, *tile_ray_offsets, *tile_rays, *sat;
  const int32_t *elev_tile_beam_offsets, *elev_tile_beams, *az_tile_col_offsets, *az_tile_cols;
  const float *beam_el_sorted, *col_az_sorted;
} simuli_tiling_dev;

/* Gaussian particle set G_l or G_c: device pointers.
 * Scene graph (reading A29): particles of dynamic objects are stored in their
 * object's local frame.  actor_id [n] (device, or NULL = everything is static background)
 * gives -1 for the static background or the object index a in [0, n_actors); actor_pose
 * [n_actors] (device) is object a's SE(3) object -> world at the frame's timestamp t (the
 * sequence of poses + learned offsets is resolved by the caller).  simuli_project maps
 * each object particle to world coordinates first: mu_w = float32(R_a mu + t_a) (computed
 * in double, rounded once), q_w = q_a (x) q (so Sigma_w = R_a Sigma R_a^T), scales and SH
 * unchanged (SH stay in the world frame, A29); everything downstream (depth key, UT,
 * records) sees the world particle.  An id < -1 or >= n_actors makes the particle invalid. */
typedef struct {
  int64_t n;
  const float* means;   /* [n][3]              */
  const float* quats;   /* [n][4] (w,x,y,z)    */
  const float* scales;  /* [n][3]              */
  const float* opacity; /* [n]                 */
  const float* sh;      /* [n][(deg+1)^2][3]   */
  int32_t sh_degree;    /* 0..3                */
  const int32_t* actor_id;        /* [n] or NULL (A29)                 */
  const simuli_pose* actor_pose;  /* [n_actors] object -> world at t   */
  int32_t n_actors;
} simuli_gaussians;

/* Camera (A22).  model PINHOLE_RADTAN: k = (k1, k2, p1, p2, k3) (OpenCV);
 * FISHEYE_KB: k = (k1, k2, k3, k4, unused), theta_d = theta (1 + k1 th^2 + ... + k4 th^8).
 * Pixel centres at (i + 0.5, j + 0.5); rolling shutter: row j fires at s = (j + 0.5)/H
 * (top -> bottom); global shutter: s = 0.  tile_px must be 8 or 16 (the render and backward kernels' tile
 * shapes); simuli_project rejects any other value with SIMULI_ERR_UNSUPPORTED. */
typedef struct {
  int32_t model;
  int32_t width, height;
  float fx, fy, cx, cy;
  float k[5];
  int32_t rolling_shutter;
  float near_m;        /* near plane (KB: minimum distance; radtan: minimum depth z)   */
  float max_theta_rad; /* validity limit on the angle between a point and the optical
                          axis (both models; radtan is only meaningful inside its FOV)  */
  int32_t tile_px;
} simuli_camera;

/* Parameters shared by projection and rendering of one sensor frame. */
typedef struct {
  int32_t kind;                     /* SIMULI_SENSOR_LIDAR | SIMULI_SENSOR_CAMERA          */
  const simuli_lidar* lidar;        /* host struct (LiDAR)                                 */
  const simuli_tiling_dev* tiling;  /* host struct of device pointers (LiDAR)              */
  const simuli_camera* camera;      /* host struct (camera)                                */
  simuli_pose pose_start;           /* pose at s = 0 (start of the sweep / first row)      */
  simuli_pose pose_end;             /* pose at s = 1; lerp(t) + slerp(R) in between (A4)   */
  int32_t rs_iterations;            /* K firing-time fixed-point iterations (A3), >= 0     */
  float ut_alpha, ut_beta, ut_kappa;/* scaled-UT parameters (A1): default 1, 2, 0          */
  float extent_sigma;               /* box half-width in std-devs (A11): default 3         */
  int32_t enable_culling;           /* ray-based culling, LiDAR only (see below): 0 off,
                                       1 the paper's dense-grid SAT test (Proc.
                                       RayOccupancyCount / ProjectParticles), 2 exact
                                       ray containment per render tile (reading A32)      */
  int32_t write_all_records;        /* 1: write the record of every particle (invalid ->
                                       NaN box); 0: only particles with tile count > 0     */
} simuli_project_params;

/* Per-particle projection output (device, caller-allocated, n entries each).
 * record[g] = 20 float32: mu[3], M[9] (row-major, M = diag(1/s) R^T, the canonical
 * transform of P:129's 3D response), opacity, f[3] (SH features at the particle's
 * view direction, A17), box lo_a, hi_a, lo_b, hi_b (LiDAR: azimuth/elevation, may extend
 * past +-pi; camera: pixels).  tile_rect[g] = (row_lo, row_hi, col_start, n_cols): render
 * tiles rows row_lo..row_hi x the circular column run col_start.. (mod n_cols_total).
 * depth_key[g]: float32 range |mu - o_mid|, o_mid = t0 + 0.5 (t1 - t0), fixed op order
 * without FMA (A19).  tile_count[g] = rows * n_cols, 0 if invalid or culled. */
typedef struct {
  float* record;
  int32_t* tile_rect;
  float* depth_key;
  int32_t* tile_count;
  float* view_dir;  /* [n][3] or NULL: the view vector mu - o(s0) of each written record,
                       unnormalised (A17: the SH direction is its unit vector; A27: the
                       beam-divergence offset uses it whole; 0 if invalid) -- for the
                       backward (A31) */
} simuli_projected;

/* UT projection: 7 sigma points mu, mu +- sqrt(3+lambda) l_k (l_k = s_k R e_k,
 * A2) pushed through the time-dependent sensor model: each sigma point is projected with
 * the pose at its own firing time (K fixed-point iterations from s = 0, A3), LiDAR by
 * Eq. 3, cameras by the lens model; UT mean / covariance -> axis-aligned box of
 * extent_sigma std-devs (A11), rounded outward.  LiDAR, enable_culling = 1: ray-based
 * culling by the SAT rectangle count over the dense 1600 x 8-per-tile ray mask (Proc.
 * RayOccupancyCount / ProjectParticles) and the coarse tile rectangle of the
 * box; enable_culling = 2 (reading A32): the same idea at full resolution -- a spinning
 * LiDAR's rays are the product beams x columns (one firing time per column, A5), so the
 * render tiles containing a ray inside the box are exactly the elevation tiles of the
 * beams with lo_b <= omega_b <= hi_b times the azimuth tiles of the columns with phi_j in
 * the (seam-shifted, A12) azimuth interval: a rectangle, found by binary search in
 * beam_el_sorted / col_az_sorted; a particle with no such beam or column is culled.  The
 * lists then hold only (tile, particle) pairs with a ray inside the box; render outputs are
 * identical in all three modes (A12).  Camera: tiles of tile_px pixels, no culling.
 * Errors: INVALID_ARGUMENT (NULL / size mismatch / kind; actor_id set with n_actors < 1 or
 * actor_pose NULL), UNSUPPORTED (sh_degree > 3),
 * CUDA (launch failure).  Device pointers in `out` must hold n entries. */
int32_t simuli_project(const simuli_gaussians* gaussians, const simuli_project_params* params,
                       simuli_projected* out, void* stream);

/* Scratch bytes simuli_bin_sort needs for n particles, pair_capacity pairs, n_tiles. */
int32_t simuli_bin_sort_workspace_size(int64_t n, int64_t pair_capacity, int32_t n_tiles, size_t* bytes);

/* Tile-Gaussian duplication and sort "as in 3DGS": one pair per (tile, particle)
 * overlap, ordered by (tile, bits(depth_key), particle id) -- unique and deterministic --
 * and tile_ranges[t] = [begin, end) of tile t in the sorted arrays (0,0 if empty).
 * Implementation: the pairs are emitted as packed words (tile << b | depth bits - min,
 * particle id) with b the bit width of the depth-key range, and sorted by a stable LSD
 * onesweep radix sort with 8-bit digits (ceil((b + tile bits) / 8) passes, decided on the
 * device).
 * n_cols_total: N_theta (LiDAR) or ceil(W / tile_px) (camera).
 * sorted_ids: device [pair_capacity] (u32 particle ids); sorted_keys: device
 *   [pair_capacity] u64 (tile << 32 | depth bits) or NULL to skip; tile_ranges: device
 *   [n_tiles][2];
 * tile_order: device [n_tiles] or NULL -- the tiles ordered by decreasing list length
 *   (power-of-two buckets; a longest-first schedule for the render kernels, which is a
 *   performance hint only: results do not depend on it);
 * n_pairs_dev: device int64 (receives P).
 * n_pairs_max_dev: device int64 or NULL -- if given, raised to max(*n_pairs_max_dev, P) on
 *   the device (a sticky maximum over asynchronous calls: one later read checks a whole
 *   batch of scans against pair_capacity; the caller zeroes it).
 * pair_capacity >= 0: fully asynchronous; if P > pair_capacity only the first
 *   pair_capacity pairs are sorted and the result is INCOMPLETE -- the caller must check
 *   *n_pairs_dev <= pair_capacity and retry with larger buffers.
 * pair_capacity < 0: the call synchronises `stream` once after the scan; if P exceeds
 *   |pair_capacity| it returns SIMULI_ERR_CAPACITY with *pairs_required (host) = P. */
int32_t simuli_bin_sort(const simuli_projected* proj, int64_t n, int32_t n_tiles, int32_t n_cols_total,
                        void* workspace, size_t workspace_bytes, int64_t pair_capacity,
                        uint64_t* sorted_keys, uint32_t* sorted_ids, int32_t* tile_ranges, int32_t* tile_order,
                        int64_t* n_pairs_dev, int64_t* n_pairs_max_dev, int64_t* pairs_required, void* stream);

/* Compositing thresholds (A13, A14): skip alpha < alpha_min (default 1/255), clamp alpha
 * to alpha_max (0.99), stop a ray when T (1 - alpha) < T_min (1e-4) without compositing
 * that particle.
 * Features: sh == NULL -> each particle's record features f (SH evaluated once per particle
 * at its view direction, A17); sh != NULL -> Eq. 1 literally (A30): SH_i(d)
 * evaluated per (ray, particle) at the ray's unit direction d from sh (device, the
 * particle set's [n][(sh_degree+1)^2][3] coefficients, indexed by the sorted ids).
 * lidar_producers (LiDAR render only; outputs are identical for every value): the
 * pipeline shape per work item (<= 32 rays of one tile).  1, 2, 3 = a producer / consumer
 * pipeline with that many producer warps feeding one consumer warp (3: the shortest single
 * scan); 4 = one warp per item doing box tests, member pairs, responses and the per-ray
 * chain itself (the least SM resources per item: the highest throughput when several scans
 * are in flight, a long single scan); 0 = the default hybrid: the longest items (one per
 * SM) by the 3-producer pipeline, the rest one warp per item.  Other values:
 * INVALID_ARGUMENT. */
typedef struct {
  float alpha_min, alpha_max, T_min;
  const float* sh;
  int32_t sh_degree;
  int32_t lidar_producers;
} simuli_render_params;

/* Per-ray LiDAR outputs (device, [n_rays] each; any pointer may be NULL to skip it).
 * zeta [n_rays][3] = sum f_i alpha_i T_i; opacity omega = sum alpha_i T_i (Eq. 1);
 * depth_accum D = sum tau_i alpha_i T_i; depth = D / omega (0 if omega = 0, A16);
 * intensity gamma = zeta_0; raydrop beta_drop = softmax(zeta_1, zeta_2)_drop;
 * final_T; n_contrib; ray_od [n_rays][6] double (origin, unit direction) as used.
 * Workload counters: n_visited = list entries examined before the ray
 * stopped, n_inbox = entries whose box contained the ray. */
typedef struct {
  float* zeta;
  float* opacity;
  float* depth_accum;
  float* depth;
  float* intensity;
  float* raydrop;
  float* final_T;
  int32_t* n_contrib;
  double* ray_od;
  int32_t* n_visited;
  int32_t* n_inbox;
} simuli_lidar_out;

/* Per-ray front-to-back compositing, Eq. 1: for every ray (origin t(s_j),
 * direction R(s_j) u(phi_j, omega_b)) over its tile's sorted list, the particles whose box
 * contains the ray (A12) contribute alpha = min(alpha_max, sigma rho) with the 3D
 * response rho at tau_max, skipping tau < r_min (A15).  sorted_ids/tile_ranges/
 * tile_order (NULL = natural order) are simuli_bin_sort outputs; `proj` must hold the
 * records of every listed particle. */
int32_t simuli_render_lidar(const simuli_projected* proj, const uint32_t* sorted_ids, const int32_t* tile_ranges,
                            const int32_t* tile_order, const simuli_project_params* params,
                            const simuli_render_params* rparams, simuli_lidar_out* out, void* stream);

/* Per-pixel camera outputs (device, [H*W] each, row-major; NULL to skip): rgb [H*W][3] =
 * foreground colour c_f (before the environment map / bilateral grid of Eq. 2), opacity,
 * depth_accum, depth, final_T, n_contrib, ray_od [H*W][6] double.  Pixels whose ray is
 * outside the lens model's validity (theta > max_theta) are not rendered (omega = 0).
 * n_visited / n_inbox: workload counters as for LiDAR. */
typedef struct {
  float* rgb;
  float* opacity;
  float* depth_accum;
  float* depth;
  float* final_T;
  int32_t* n_contrib;
  double* ray_od;
  int32_t* n_visited;
  int32_t* n_inbox;
} simuli_camera_out;

int32_t simuli_render_camera(const simuli_projected* proj, const uint32_t* sorted_ids, const int32_t* tile_ranges,
                             const int32_t* tile_order, const simuli_project_params* params,
                             const simuli_render_params* rparams, simuli_camera_out* out, void* stream);

/* ---- Backward pass ("differentiable renderer", P:160-171 training; readings A31) ----
 * Gradients of a loss L with respect to the particle parameters, given the upstream
 * gradients of the rendered outputs.  The forward decisions (box membership A12, the
 * alpha_min / near skips A13, the T_min termination A14) are replayed with the same
 * float32 arithmetic as the render kernels and are not differentiated.  One exception: the
 * LiDAR backward cuts a list into 512-entry segments and enters segment s with T = the
 * product of the earlier segments' transmittance products (each formed from T = 1), whose
 * float32 rounding can differ from the forward's single running product; a ray whose T
 * crosses T_min within a few ulps of the threshold in a later segment can therefore
 * terminate one member earlier or later than in the forward (A23 flags such rays).  The
 * response
 * is: alpha = min(alpha_max, sigma rho(tau_max)) with tau_max and delta^2 of the
 * canonical transform M = diag(1/s) R(q/|q|)^T (clamped alpha: no gradient).  Features are
 * the per-particle SH at the projection's view direction (A17), held fixed (no gradient
 * through the direction); with rparams->sh (per-ray SH, A30) the features are SH_i(d) per
 * ray and the SH gradient sums Y_k(d) dL/dzeta alpha T over the rays (float atomics into
 * grad_out->sh); with beam divergence (A27) M = chol(Sigma_hat)^-1 is differentiated through
 * the Cholesky factor and Sigma_hat's view vector (the sensor position held at the mean's
 * firing time).
 * Upstream gradients (device, [n_rays] or [n_rays][3]; NULL = 0): LiDAR zeta, opacity
 * (omega), depth_accum (D), depth (D / omega), intensity (zeta_0), raydrop
 * (1 / (1 + exp(zeta_1 - zeta_2))); camera rgb (c_f), opacity, depth_accum, depth. */
typedef struct {
  const float *zeta, *opacity, *depth_accum, *depth, *intensity, *raydrop;
  /* optional: the forward's own zeta [R][3], opacity [R], depth_accum [R] outputs of this
     frame; given all three, the backward skips its first list pass (totals) */
  const float *fwd_zeta, *fwd_opacity, *fwd_depth_accum;
} simuli_lidar_grad_in;

typedef struct {
  const float *rgb, *opacity, *depth_accum, *depth;
  const float *fwd_rgb, *fwd_opacity, *fwd_depth_accum; /* optional, as above */
} simuli_camera_grad_in;

/* Per-particle parameter gradients (device, caller-allocated, n entries each; overwritten,
 * zero for particles that composite into no ray): means [n][3], quats [n][4] (w.r.t. the
 * unnormalised input quaternion), scales [n][3], opacity [n] (post-activation sigma),
 * sh [n][(deg+1)^2][3].  With a scene graph (simuli_gaussians.actor_id) means / quats are
 * the gradients of the OBJECT-frame inputs and actor_pose [n_actors][7] (device, or NULL
 * to skip) receives dL/dq_a (unnormalised, 4) and dL/dt_a (3) of every object pose
 * (A29, A31: R_w = R_a R_l, mu_w = R_a mu_l + t_a). */
typedef struct {
  float *means, *quats, *scales, *opacity, *sh;
  float* actor_pose;
} simuli_gaussian_grads;

/* Scratch bytes for the backward of n particles (16 floats each) plus the segment area of
 * the segmented list walk for up to pair_capacity pairs over n_tiles tiles (a smaller
 * workspace of at least 64 n bytes falls back to the unsegmented walk). */
int32_t simuli_backward_workspace_size(int64_t n, int64_t pair_capacity, int32_t n_tiles, size_t* bytes);

/* LiDAR backward.  gaussians / params / rparams / proj / sorted_ids / tile_ranges: exactly
 * the forward frame's (proj->view_dir must have been written by simuli_project).  Launches:
 * workspace clear, one warp per (tile, 32-ray chunk) replaying the tile's list twice
 * (totals, then gradients with suffix sums; warp-reduced float atomics into the workspace),
 * then one thread per particle for the parameter chain.  Asynchronous on `stream`;
 * gradient sums are in atomic (nondeterministic) order.
 * n = 0: returns SIMULI_OK without reading any other argument.
 * Errors: INVALID_ARGUMENT (NULL, view_dir missing, workspace below 64 n bytes, per-ray
 * SH of another degree, scene graph without poses), UNSUPPORTED (sh_degree > 3), CUDA. */
int32_t simuli_backward_lidar(const simuli_gaussians* gaussians, const simuli_projected* proj,
                              const uint32_t* sorted_ids, const int32_t* tile_ranges, const int32_t* tile_order,
                              const simuli_project_params* params, const simuli_render_params* rparams,
                              const simuli_lidar_grad_in* grad_in, simuli_gaussian_grads* grad_out,
                              void* workspace, size_t workspace_bytes, void* stream);

/* Camera backward: as simuli_backward_lidar, one CTA per tile (pixel per thread). */
int32_t simuli_backward_camera(const simuli_gaussians* gaussians, const simuli_projected* proj,
                               const uint32_t* sorted_ids, const int32_t* tile_ranges, const int32_t* tile_order,
                               const simuli_project_params* params, const simuli_render_params* rparams,
                               const simuli_camera_grad_in* grad_in, simuli_gaussian_grads* grad_out,
                               void* workspace, size_t workspace_bytes, void* stream);

/* Final camera colour, Eq. 2: c = A(omega c_f + (1 - omega) c_b(d)), with the
 * background c_b(d) from a learned environment map and A an affine colour transform from a
 * learned bilateral grid (readings A28):
 *  * env_map: device [env_h][env_w][3] float, equirectangular in the world frame (z up):
 *    longitude atan2(d_y, d_x) in [-pi, pi) -> [0, env_w), colatitude acos(d_z) in [0, pi]
 *    -> [0, env_h), texel centres at +0.5, bilinear, wrapping in longitude, clamped in
 *    colatitude; NULL -> c_b = 0.
 *  * grid: device [grid_d][grid_h][grid_w][12] float (16-byte aligned), row-major 3x4 affine matrices over
 *    (x / W, y / H, luminance), luminance = 0.299 r + 0.587 g + 0.114 b of the blended colour
 *    clamped to [0, 1], cell centres at +0.5, trilinear, clamped at the borders;
 *    c = M[:, :3] c_in + M[:, 3]; NULL -> A = identity.
 * d is the pixel's ray direction (the same inverse lens model and row time as
 * simuli_render_camera; (0, 0, 0) outside the lens validity).  rgb_fg [H*W][3] and opacity
 * [H*W] are simuli_render_camera's rgb / opacity; rgb_out [H*W][3] (may alias rgb_fg).
 * rgb_fg is Eq. 1's sum of SH alpha T, i.e. already omega times the opacity-normalised
 * foreground colour, so Eq. 2's "omega c_f" IS rgb_fg (A28: P:122 calls the step alpha
 * compositing; multiplying the sum by omega again would weight the foreground by omega^2):
 * c_in = rgb_fg + (1 - omega) c_b.
 * All device pointers, caller-owned; asynchronous on `stream`.  Errors: INVALID_ARGUMENT
 * (NULL / non-camera params / non-positive sizes with a non-NULL table). */
typedef struct {
  const float* env_map;
  int32_t env_h, env_w;
  const float* grid;
  int32_t grid_h, grid_w, grid_d;
} simuli_camera_compose;

int32_t simuli_compose_camera(const simuli_project_params* params, const simuli_camera_compose* compose,
                              const float* rgb_fg, const float* opacity, float* rgb_out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SIMULI_H */
