/*
 * oracle.h -- CPU ORACLE FOR THE SIMULI HOT PATH.  TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * legs may load this library.  The product (paper_2510_12901_b200/, include/simuli.h)
 * never links, imports or executes anything under oracle/, and this file shares no
 * code, header, constant table or helper with the product.
 *
 * Plain, slow, double-precision restatement of what SimULi (arXiv 2510.12901) computes
 * on its forward LiDAR / camera rendering path.  Citations: "P:n" = PAPER.md line n.
 * Readings of silent / garbled passages follow SURVEY.md §8(c) (ledger A1-A26) and are
 * listed in DESIGN.md §3.  Float32 appears only where the interface defines a float32
 * value (tile boundaries, ray angles, box edges, depth keys, tile maps); those steps are
 * written as explicit float operations (compiled with -ffp-contract=off, SSE math).
 */
#ifndef SIMULI_ORACLE_H
#define SIMULI_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Spinning LiDAR (A5, A6). Values are the float32 ABI values promoted. */
typedef struct {
  int32_t n_beams;
  const float* elev;        /* [n_beams] beam elevations (rad), any order          */
  int32_t n_az;             /* columns per revolution A                             */
  double az_start;          /* phi_start (rad)                                      */
  int32_t dir;              /* +1 ccw, -1 cw                                        */
  double r_min;             /* minimum range (m)                                    */
  double beam_div;          /* beam divergence theta_div (rad), App. C; 0 = off (A24) */
} or_lidar;

/* Camera (A22). model 0 = pinhole + radtan, 1 = KB fisheye. */
typedef struct {
  int32_t model, width, height;
  double fx, fy, cx, cy;
  double k[5];              /* radtan: k1 k2 p1 p2 k3 ; KB: k1 k2 k3 k4 (k[4] unused) */
  int32_t rolling;          /* 0 global (s=0), 1 rows top->bottom                    */
  double near_m, max_theta;
  int32_t tile_px;          /* power of two                                         */
} or_camera;

/* Tiling produced by Proc. ElevationTiling with the A8 corrections. */
typedef struct {
  int32_t n_phi, n_theta, n_tiles, max_rays_in_tile, sat_rows, sat_cols, n_rays;
  int32_t cull_rows_per_tile, cull_az_cells;
  float pi_f, two_pi_f, az_tile_scale, az_cell_scale;
  float* bounds;            /* [n_phi+1]  */
  float* cull_row_scale;    /* [n_phi]    */
  float* ray_az; float* ray_el; float* ray_s;  /* [n_rays], ray id = b*A + j */
  int32_t* ray_tile;        /* [n_rays]   */
  int32_t* tile_ray_offsets;/* [n_tiles+1] */
  int32_t* tile_rays;       /* [n_rays]   */
  int32_t* sat;             /* [sat_rows*sat_cols] */
  int32_t* ray_cell_row; int32_t* ray_cell_col; /* dense cell of each ray (diagnostic) */
  int32_t n_beams, n_az;    /* B, A: ray id = b*A + j                                       */
} or_tiling;

/* ---- primitives (exposed for pins) ---- */
void or_quat_to_rot(const double q[4], double R[9]);
/* App. C: Sigma_hat = Sigma + (theta r)^2 (I - d d^T), d = (mu - o)/r, r = |mu - o| */
void or_divergence_cov(const double Sigma[9], const double mu[3], const double o[3], double theta, double Sh[9]);
int  or_cholesky3(const double S[9], double L[9]);          /* S = L L^T, L lower; -1 if not SPD */
void or_lower_inverse3(const double L[9], double M[9]);      /* M = L^-1 (lower)                   */
int  or_sigma_points_sqrt(const double mu[3], const double Lsq[9], const double ut[3], double pts[21],
                          double wm[7], double wc[7]);        /* sigma points from the columns of Lsq */
void or_covariance(const double q[4], const double s[3], double Sigma[9]);
int  or_ut_weights(const double ut[3], double* spread, double wm[7], double wc[7]);
int  or_sigma_points(const double mu[3], const double q[4], const double s[3], const double ut[3],
                     double pts[21], double wm[7], double wc[7]);
void or_pose_at(const double pose0[7], const double pose1[7], double s, double R[9], double t[3]);
void or_lidar_point(const double x[3], const or_lidar* L, const double pose0[7], const double pose1[7],
                    int K, double out[4]);
int  or_camera_point(const double x[3], const or_camera* C, const double pose0[7], const double pose1[7],
                     int K, double out[4]);
int  or_camera_unproject(const or_camera* C, double u, double v, double dir[3]);
void or_sh_eval(const double* sh, int degree, const double dir[3], double out[3]);
void or_response(const double mu[3], const double Mrows[9], const double o[3], const double d[3], double out[2]);
int  or_ut_affine(const double mu[3], const double q[4], const double s[3], const double ut[3],
                  const double A[6], const double b[2], double mean[2], double cov[3]);
int  or_sat_query(const int32_t* sat, int32_t sat_cols, int32_t r_lo, int32_t r_hi, int32_t c_lo, int32_t c_hi);

/* ---- O7 tiling ---- */
int  or_build_tiling(const or_lidar* L, int32_t n_phi, int32_t M, int32_t hist_bins, int32_t cull_az,
                     int32_t cull_rows, or_tiling* out);
void or_free_tiling(or_tiling* t);
int32_t or_elev_tile(const or_tiling* t, float w);
int32_t or_az_col(const or_tiling* t, float phi);
int32_t or_dense_row(const or_tiling* t, float w);
int32_t or_dense_cell(const or_tiling* t, float phi);

/* ---- O1-O6, O9, O10 projection ---- */
typedef struct {
  int32_t* valid;           /* [n] 1 valid, 0 invalid                                    */
  int32_t* ambiguous;       /* [n] validity decision within a float32 margin (A23)        */
  double*  mean2d;          /* [n][2] UT mean (azimuth normalised into [-pi,pi))          */
  double*  cov2d;           /* [n][3] aa, ab, bb                                          */
  float*   box;             /* [n][4] lo_a, hi_a, lo_b, hi_b  (outward-rounded float32)   */
  double*  Mrows;           /* [n][9] M = diag(1/s) R^T                                    */
  double*  feat;            /* [n][3] SH features                                          */
  float*   key;             /* [n] float32 depth key (O10)                                 */
  double*  minrange;        /* [n] smallest sigma-point range / camera distance            */
  double*  viewdir;         /* [n][3] view vector mu - o(s0) (unnormalised; A17) or NULL    */
} or_proj_out;

typedef struct {
  int64_t n;
  const float *means, *quats, *scales, *opacity, *sh;
  int32_t sh_degree;
} or_gaussians;

int or_project_lidar(const or_gaussians* G, const or_lidar* L, const double pose0[7], const double pose1[7],
                     int K, const double ut[3], double extent_sigma, or_proj_out* out);
int or_project_camera(const or_gaussians* G, const or_camera* C, const double pose0[7], const double pose1[7],
                      int K, const double ut[3], double extent_sigma, or_proj_out* out);

/* ---- O8 culling + tile rect (from float32 boxes) ---- */
int or_cull_lidar(int64_t n, const int32_t* valid, const float* box, const or_tiling* t, int enable_cull,
                  int32_t* count, int32_t* rect);
int or_cull_camera(int64_t n, const int32_t* valid, const float* box, const or_camera* C,
                   int32_t* count, int32_t* rect);

/* ---- O11 binning ---- */
int64_t or_bin(int64_t n, const int32_t* count, const int32_t* rect, const float* key, int32_t n_tiles,
               int32_t n_cols_total, int64_t capacity, uint64_t* keys_out, uint32_t* ids_out, int32_t* ranges);

/* ---- O12 compositing ---- */
typedef struct {
  double near_tau, alpha_min, alpha_max, T_min;
  int32_t wrap;              /* 1: LiDAR azimuth wrap rules (O12), 0: camera plain box   */
  float pi_f, two_pi_f;
  int32_t flag_mode;         /* 1: compute A23 threshold flags                          */
  double eps_a, eps_b;       /* box-edge ambiguity margins (coordinate units)           */
  double eps_alpha, eps_T_rel, eps_tau;
  double eps_impact;         /* box-edge flags only when alpha*T of the particle > this  */
  double eps_amb_a, eps_amb_b; /* margins around validity-ambiguous particles' boxes       */
  const float* sh;           /* NULL: per-particle features feat (A17); else literal Eq. 1:
                                SH_i(d) per (ray, particle) at the ray direction (A30)   */
  int32_t sh_degree;
} or_render_params;

typedef struct {
  double* feat;   /* [R][3] zeta or colour */
  double* opacity; double* depth_accum; double* depth; double* T_final;
  int32_t* n_contrib; int32_t* flag;
  int64_t* scanned;  /* [R] list entries visited before stop (workload counter) */
  int64_t* inbox;    /* [R] box-passing entries                              */
} or_render_out;

int or_composite(int64_t n_gauss, const double* mu, const double* Mrows, const double* sigma, const double* feat,
                 const float* box, const int32_t* gamb,
                 const uint32_t* ids, const int32_t* ranges, int32_t n_rays, const int32_t* ray_tile,
                 const float* ray_a, const float* ray_b, const double* ray_od, const int32_t* ray_valid,
                 const or_render_params* p, or_render_out* out);
void or_decode_lidar(const double zeta[3], double out[2]);

/* ---- rays ---- */
void or_lidar_rays(const or_tiling* t, const double pose0[7], const double pose1[7], double* od);
void or_camera_rays(const or_camera* C, const double pose0[7], const double pose1[7], double* od,
                    int32_t* valid, float* pix_u, float* pix_v, int32_t* ray_tile);

void or_set_threads(int n);
int  or_get_threads(void);

/* O14: camera final colour, Eq. 2 (env map c_b + bilateral grid A; readings A28) */
int or_compose_camera(const or_camera* C, const double* ray_od, const double* rgb_fg, const double* omega,
                      const float* env, int32_t He, int32_t We, const float* grid, int32_t gh, int32_t gw,
                      int32_t gd, double* rgb_out);

/* O15: backward of Eq. 1 compositing ("differentiable renderer"; A31).  Per ray, the
 * forward contributions are collected in list order (same rules as or_composite) and
 * dL/d(mu, M, sigma, f) of every contributing particle accumulated from the upstream
 * gradients g_feat [R][3], g_opacity [R], g_daccum [R] (NULL = 0).  Outputs [n][3], [n][9],
 * [n], [n][3] are accumulated (caller zeroes); with p->sh (per-ray SH, A30) the features are
 * SH_g(d) per ray and d_sh [n][(deg+1)^2][3] accumulates dL/dSH directly. */
int or_backward_composite(const double* mu, const double* Mrows, const double* sigma, const double* feat,
                          const float* box, const uint32_t* ids, const int32_t* ranges, int32_t n_rays,
                          const int32_t* ray_tile, const float* ray_a, const float* ray_b, const double* ray_od,
                          const int32_t* ray_valid, const or_render_params* p, const double* g_feat,
                          const double* g_opacity, const double* g_daccum, double* d_mu, double* d_M,
                          double* d_sigma, double* d_feat, double* d_sh);
/* O16: chain to the particle parameters: M = diag(1/s) R(q/|q|)^T -> dq, ds;
 * f = SH(v) -> dSH (v = the projection's view direction, no gradient through v, A31). */
void or_backward_params(int64_t n, const float* quats, const float* scales, const double* viewdir,
                        int32_t sh_degree, const double* d_M, const double* d_feat, double* g_quats,
                        double* g_scales, double* g_sh);

/* O16 with the scene graph: gradients of the LOCAL particle parameters and of the object
 * poses (g_actor [n_actors][7] = dL/dq_a, dL/dt_a); d_mu / d_M are world-frame (O15). */
void or_backward_params_sg(int64_t n, const float* means, const float* quats, const float* scales,
                           const double* viewdir, int32_t sh_degree, const int32_t* actor_id, int32_t n_actors,
                           const double* actor_pose, double beam_div, const double* d_mu, const double* d_M,
                           const double* d_feat, double* g_means, double* g_quats, double* g_scales, double* g_sh,
                           double* g_actor);

/* O0: scene graph, object particles -> world at the frame's timestamp (A29) */
void or_actors_to_world(int64_t n, const float* means, const float* quats, const int32_t* actor_id,
                        int32_t n_actors, const double* actor_pose, float* means_w, float* quats_w);

#ifdef __cplusplus
}
#endif
#endif
